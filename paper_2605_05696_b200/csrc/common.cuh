// Shared device helpers for the irminsul_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/irminsul_b200.h"

namespace irm {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);

#define IRM_REQUIRE(cond, ...)          \
    do {                                \
        if (!(cond)) {                  \
            ::irm::set_error(__VA_ARGS__); \
            return IRM_EINVAL;          \
        }                               \
    } while (0)

#define IRM_CUDA_CHECK(expr)                                                        \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess) {                                                    \
            ::irm::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                             cudaGetErrorString(_e));                               \
            return IRM_ECUDA;                                                       \
        }                                                                           \
    } while (0)

// after every kernel launch of the library (one per launch): counts it, checks it
void count_launch();
#define IRM_LAUNCH_CHECK()          \
    do {                            \
        ::irm::count_launch();      \
        IRM_CUDA_CHECK(cudaGetLastError()); \
    } while (0)

int sm_count();

// ---------------------------------------------------------------- bit utils
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
    return (x << r) | (x >> (64 - r));
}

// ---------------------------------------------------------------- XXH64
// Published XXH64 algorithm (libxxhash 0.8.2, the library behind the
// reference's fingerprint.py:24-25).
constexpr uint64_t XP1 = 0x9E3779B185EBCA87ULL;
constexpr uint64_t XP2 = 0xC2B2AE3D27D4EB4FULL;
constexpr uint64_t XP3 = 0x165667B19E3779F9ULL;
constexpr uint64_t XP4 = 0x85EBCA77C2B2AE63ULL;
constexpr uint64_t XP5 = 0x27D4EB2F165667C5ULL;

__device__ __forceinline__ uint64_t xxh_round(uint64_t acc, uint64_t in) {
    acc += in * XP2;
    acc = rotl64(acc, 31);
    return acc * XP1;
}
__device__ __forceinline__ uint64_t xxh_merge(uint64_t acc, uint64_t v) {
    v = xxh_round(0, v);
    acc ^= v;
    return acc * XP1 + XP4;
}
__device__ __forceinline__ uint64_t xxh_avalanche(uint64_t h) {
    h ^= h >> 33;
    h *= XP2;
    h ^= h >> 29;
    h *= XP3;
    h ^= h >> 32;
    return h;
}

// XXH64 over n 32-bit words at a 4-byte-aligned address (token spans: the
// little-endian u32 encoding of fingerprint.py:16-21 is the memory image).
__device__ __forceinline__ uint64_t xxh64_words(const uint32_t *__restrict__ w, int64_t n,
                                                uint64_t seed) {
    const int64_t len = 4 * n;
    int64_t i = 0;
    uint64_t h;
    auto rd64 = [&](int64_t k) -> uint64_t {
        return (uint64_t)__ldg(w + k) | ((uint64_t)__ldg(w + k + 1) << 32);
    };
    if (n >= 8) {
        uint64_t v1 = seed + XP1 + XP2, v2 = seed + XP2, v3 = seed, v4 = seed - XP1;
        const int64_t stripes = n / 8;
        for (int64_t s = 0; s < stripes; ++s, i += 8) {
            v1 = xxh_round(v1, rd64(i));
            v2 = xxh_round(v2, rd64(i + 2));
            v3 = xxh_round(v3, rd64(i + 4));
            v4 = xxh_round(v4, rd64(i + 6));
        }
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = xxh_merge(h, v1);
        h = xxh_merge(h, v2);
        h = xxh_merge(h, v3);
        h = xxh_merge(h, v4);
    } else {
        h = seed + XP5;
    }
    h += (uint64_t)len;
    for (; i + 2 <= n; i += 2) {
        h ^= xxh_round(0, rd64(i));
        h = rotl64(h, 27) * XP1 + XP4;
    }
    if (i < n) {
        h ^= (uint64_t)__ldg(w + i) * XP1;
        h = rotl64(h, 23) * XP2 + XP3;
    }
    return xxh_avalanche(h);
}

// XXH64 of n 32-bit words computed by the 4 lanes of a quad: lane q of the
// quad runs accumulator v_{q+1} over every 32-byte stripe (the four lanes of
// a stripe are independent in XXH64), loads unrolled 4 stripes deep. Every
// lane of the warp must call this (shuffles), quads with n == 0 included;
// all 4 lanes of a quad return the hash.
__device__ __forceinline__ uint64_t xxh64_words_quad(const uint32_t *__restrict__ w, int64_t n,
                                                     uint64_t seed, int lane) {
    const int q = lane & 3, qb = lane & ~3;
    const int64_t stripes = n / 8;
    uint64_t v = q == 0 ? seed + XP1 + XP2 : q == 1 ? seed + XP2 : q == 2 ? seed : seed - XP1;
    const uint32_t *__restrict__ p = w + 2 * q;
    auto rd = [&](int64_t s) -> uint64_t {
        return (uint64_t)__ldg(p + 8 * s) | ((uint64_t)__ldg(p + 8 * s + 1) << 32);
    };
    int64_t s = 0;
    for (; s + 8 <= stripes; s += 8) {  // 8 stripes of loads in flight per lane
        uint64_t d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) d[u] = rd(s + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) v = xxh_round(v, d[u]);
    }
    for (; s + 4 <= stripes; s += 4) {
        const uint64_t d0 = rd(s), d1 = rd(s + 1), d2 = rd(s + 2), d3 = rd(s + 3);
        v = xxh_round(v, d0);
        v = xxh_round(v, d1);
        v = xxh_round(v, d2);
        v = xxh_round(v, d3);
    }
    for (; s < stripes; ++s) v = xxh_round(v, rd(s));
    const uint64_t v1 = __shfl_sync(0xffffffffu, v, qb), v2 = __shfl_sync(0xffffffffu, v, qb + 1);
    const uint64_t v3 = __shfl_sync(0xffffffffu, v, qb + 2), v4 = __shfl_sync(0xffffffffu, v, qb + 3);
    uint64_t h;
    if (stripes > 0) {
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = xxh_merge(h, v1);
        h = xxh_merge(h, v2);
        h = xxh_merge(h, v3);
        h = xxh_merge(h, v4);
    } else {
        h = seed + XP5;
    }
    h += (uint64_t)(4 * n);
    int64_t i = stripes * 8;
    for (; i + 2 <= n; i += 2) {
        h ^= xxh_round(0, (uint64_t)__ldg(w + i) | ((uint64_t)__ldg(w + i + 1) << 32));
        h = rotl64(h, 27) * XP1 + XP4;
    }
    if (i < n) {
        h ^= (uint64_t)__ldg(w + i) * XP1;
        h = rotl64(h, 23) * XP2 + XP3;
    }
    return xxh_avalanche(h);
}

// XXH64 over an arbitrary byte span (K2's byte entry point, for the KATs).
__device__ __forceinline__ uint64_t xxh64_bytes(const uint8_t *__restrict__ p, int64_t len,
                                                uint64_t seed) {
    auto rd64 = [&](int64_t k) -> uint64_t {
        uint64_t v = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) v |= (uint64_t)p[k + b] << (8 * b);
        return v;
    };
    auto rd32 = [&](int64_t k) -> uint64_t {
        uint64_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) v |= (uint64_t)p[k + b] << (8 * b);
        return v;
    };
    int64_t i = 0;
    uint64_t h;
    if (len >= 32) {
        uint64_t v1 = seed + XP1 + XP2, v2 = seed + XP2, v3 = seed, v4 = seed - XP1;
        for (; i + 32 <= len; i += 32) {
            v1 = xxh_round(v1, rd64(i));
            v2 = xxh_round(v2, rd64(i + 8));
            v3 = xxh_round(v3, rd64(i + 16));
            v4 = xxh_round(v4, rd64(i + 24));
        }
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = xxh_merge(h, v1);
        h = xxh_merge(h, v2);
        h = xxh_merge(h, v3);
        h = xxh_merge(h, v4);
    } else {
        h = seed + XP5;
    }
    h += (uint64_t)len;
    for (; i + 8 <= len; i += 8) {
        h ^= xxh_round(0, rd64(i));
        h = rotl64(h, 27) * XP1 + XP4;
    }
    if (i + 4 <= len) {
        h ^= rd32(i) * XP1;
        h = rotl64(h, 23) * XP2 + XP3;
        i += 4;
    }
    for (; i < len; ++i) {
        h ^= (uint64_t)p[i] * XP5;
        h = rotl64(h, 11) * XP1;
    }
    return xxh_avalanche(h);
}

// ---------------------------------------------------------------- block scan
// Exclusive scan of one int64 per thread across a block of BLOCK threads.
// The rotation of one (lo, hi) pair, rounded exactly as the oracle's C restatement
// (oracle/irm_oracle.c: lo*c - hi*s, lo*s + hi*c in separately rounded fp32
// products, no FMA contraction), so every K4 form agrees bit for bit.
__device__ __forceinline__ float rot_lo(float lo, float hi, float c, float s) {
    return __fsub_rn(__fmul_rn(lo, c), __fmul_rn(hi, s));
}
__device__ __forceinline__ float rot_hi(float lo, float hi, float c, float s) {
    return __fadd_rn(__fmul_rn(lo, s), __fmul_rn(hi, c));
}
__device__ __forceinline__ double rot_lo(double lo, double hi, double c, double s) { return lo * c - hi * s; }
__device__ __forceinline__ double rot_hi(double lo, double hi, double c, double s) { return lo * s + hi * c; }

template <int BLOCK>
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t *total,
                                                        int64_t *smem /*[BLOCK/32]*/) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) smem[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t s = lane < BLOCK / 32 ? smem[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += y;
        }
        if (lane < BLOCK / 32) smem[lane] = s;
    }
    __syncthreads();
    int64_t before = warp > 0 ? smem[warp - 1] : 0;
    *total = smem[BLOCK / 32 - 1];
    __syncthreads();
    return before + x - v;
}

}  // namespace irm
