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
// fp64: the reference's numpy expression, lo*cos - hi*sin / lo*sin + hi*cos, with every
// product rounded on its own (rotary.py:107) -- no FMA contraction
__device__ __forceinline__ double rot_lo(double lo, double hi, double c, double s) {
    return __dsub_rn(__dmul_rn(lo, c), __dmul_rn(hi, s));
}
__device__ __forceinline__ double rot_hi(double lo, double hi, double c, double s) {
    return __dadd_rn(__dmul_rn(lo, s), __dmul_rn(hi, c));
}

// ---------------------------------------------------------------- correctly rounded sincos
// sin / cos of an fp64 angle evaluated in double-double (~100 bits) and rounded once, so
// they equal the correctly rounded values the reference's rotary golden file holds
// (rotary_reference.csv, rotary.py:104: numpy/libm cos, sin; all 384 rotated golden values
// reproduce with correctly rounded cos/sin). CUDA's sincos is within 2 ulp, which left
// 1-ulp differences in fp64 rotations. Cost: ~1k fp64 flops per angle, evaluated per
// (chunk, frequency) -- not per row.
struct ddouble {
    double hi, lo;
};
__device__ __forceinline__ ddouble dd_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ ddouble dd_fast(double a, double b) {  // |a| >= |b|
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ ddouble dd_add(ddouble a, ddouble b) {
    ddouble s = dd_two_sum(a.hi, b.hi);
    const ddouble t = dd_two_sum(a.lo, b.lo);
    s = dd_fast(s.hi, __dadd_rn(s.lo, t.hi));
    return dd_fast(s.hi, __dadd_rn(s.lo, t.lo));
}
__device__ __forceinline__ ddouble dd_mul(ddouble a, ddouble b) {
    const double p = __dmul_rn(a.hi, b.hi);
    const double e = __fma_rn(a.hi, b.hi, -p);
    return dd_fast(p, __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, e)));
}

__device__ __forceinline__ void sincos_cr(double x, double *sn, double *cs) {
    // 1/n! as double-double, n = 0 .. 29
    constexpr double IF_HI[30] = {
        0x1.0p+0, 0x1.0p+0, 0x1.0p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5, 0x1.1111111111111p-7,
        0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19,
        0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33,
        0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41, 0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49,
        0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57, 0x1.e542ba4020225p-62, 0x1.71b8ef6dcf572p-66,
        0x1.0ce396db7f853p-70, 0x1.761b41316381ap-75, 0x1.f2cf01972f578p-80, 0x1.3f3ccdd165fa9p-84,
        0x1.88e85fc6a4e5ap-89, 0x1.d1ab1c2dccea3p-94, 0x1.0a18a2635085dp-98, 0x1.259f98b4358adp-103};
    constexpr double IF_LO[30] = {
        0.0, 0.0, 0.0, 0x1.5555555555555p-57, 0x1.5555555555555p-59, 0x1.1111111111111p-63,
        -0x1.f49f49f49f49fp-65, 0x1.a01a01a01a01ap-73, 0x1.a01a01a01a01ap-76, -0x1.c154f8ddc6c00p-73,
        0x1.cbbc05b4fa99ap-76, -0x1.c062e06d1f209p-80, -0x1.2aec959e14c06p-83, 0x1.f28e0cc748ebep-87,
        0x1.05d6f8a2efd1fp-92, 0x1.1d8656b0ee8cbp-97, 0x1.1d8656b0ee8cbp-101, 0x1.ac981465ddc6cp-103,
        0x1.eec01221a8b0bp-107, 0x1.2650f61dbdcb4p-112, 0x1.ea72b4afe3c2fp-120, -0x1.d043ae40c4647p-120,
        -0x1.aebcdbd20331cp-124, -0x1.3423c7d91404fp-130, -0x1.9ada5fcc1ab14p-135, -0x1.58ddadf344487p-139,
        -0x1.71c37ebd16540p-143, 0x1.054d0c78aea14p-149, 0x1.b9e2e28e1aa54p-153, 0x1.eaf8c39dd9bc5p-157};
    // pi/2 in four doubles; reduction r = x - k pi/2 (|x| < 2^40: k fits, the first step is exact)
    constexpr double P1 = 0x1.921fb54442d18p+0, P2 = 0x1.1a62633145c07p-54, P3 = -0x1.f1976b7ed8fbcp-110,
                     P4 = 0x1.4cf98e804177dp-164;
    const double k = rint(x * 0x1.45f306dc9c883p-1);
    const double p = __dmul_rn(k, P1);
    const double pe = __fma_rn(k, P1, -p);
    ddouble r = dd_fast(__dsub_rn(x, p), -pe);  // x - p exact (Sterbenz), -pe its correction
    const double q2 = __dmul_rn(k, P2);
    r = dd_add(r, {-q2, -__fma_rn(k, P2, -q2)});
    const double q3 = __dmul_rn(k, P3);
    r = dd_add(r, {-q3, -__fma_rn(k, P3, -q3)});
    r = dd_add(r, {-__dmul_rn(k, P4), 0.0});
    const ddouble z = dd_mul(r, r);
    ddouble s = {IF_HI[29], IF_LO[29]}, c = {IF_HI[28], IF_LO[28]};
    for (int n = 27; n >= 1; n -= 2) {  // sin: sum (-1)^i r^(2i+1)/(2i+1)!
        const ddouble t = dd_mul(z, s);
        s = dd_add({IF_HI[n], IF_LO[n]}, {-t.hi, -t.lo});
    }
    for (int n = 26; n >= 0; n -= 2) {  // cos: sum (-1)^i r^(2i)/(2i)!
        const ddouble t = dd_mul(z, c);
        c = dd_add({IF_HI[n], IF_LO[n]}, {-t.hi, -t.lo});
    }
    s = dd_mul(s, r);
    const int q = (int)(((long long)k % 4 + 4) % 4);
    const double sv = s.hi, cv = c.hi;
    *sn = q == 0 ? sv : q == 1 ? cv : q == 2 ? -sv : -cv;
    *cs = q == 0 ? cv : q == 1 ? -sv : q == 2 ? -cv : sv;
}

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
