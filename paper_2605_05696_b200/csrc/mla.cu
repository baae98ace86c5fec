// K5: fused absorbed-MLA reattach prefill on tcgen05 / TMEM (sm_100a).
//
// Absent from the reference ("R(delta)R(p_src) = R(p), fused in
// FlashMLA"; PAPER.md:469-476, 788-791 describe the production variant that
// fuses the rotation into the load path so the rotated k_r never reaches
// HBM). Semantics, restated in oracle/mla_ref.py:
//   S[r, k] = (q_c[r] . c_KV[k] + q_pe[r] . R(delta_k) kr_base[k]) * scale
//   causal: key k visible to the row of query position P iff k <= P
//   O[r] = softmax_k(S[r, :]) @ c_KV           (512-dim latent output)
// All heads share the single latent KV head, so rows are (query, head) pairs:
// one CTA owns 64 rows (4 queries x 16 heads) and streams 32-key KV tiles
// through a 4-stage ring.
//
// Tensor-core mapping (cta_group::1, M = 64):
//   QK : D = S  [64 x 32]  fp32 in TMEM (the half-subpartition lanes +16)
//        A = Q  [64 x 576] bf16 smem, K-major SW128 (9 pieces of 64 dims)
//        B = KV [32 x 576] bf16 smem, K-major SW128; piece 8 (k_r) is
//            rotated by R(delta) on its way into smem, in fp32 from an fp64
//            per-chunk angle table -- never written back to HBM
//   PV : D = O  [64 x 512] fp32 in TMEM (lanes +0, all 512 columns)
//        A = P  [64 x 32]  bf16 smem (softmax output), K-major SW64
//        B = V  = the same KV pieces 0..7 read MN-major (keys x dims)
// Warp roles: 0-3 softmax / O-correction (lazy rescale, threshold 2^8),
// 4-11 producers (cp.async + rotate), 12 the single-thread MMA issuer.
#include "common.cuh"
#include "tcgen05.cuh"
#include "cluster.cuh"
#include <cuda_bf16.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

namespace irm {
namespace mla {

constexpr int BM = 64;               // q-rows per CTA
constexpr int BN = 32;               // keys per KV tile
constexpr int NST = 4;               // KV ring stages
constexpr int DQK = 576, DV = 512;
constexpr int NPIECE = 9;            // 64-dim pieces of a 576-wide row
constexpr int QPIECE = BM * 128;     // 8 KB
constexpr int KPIECE = BN * 128;     // 4 KB
constexpr int KTILE = NPIECE * KPIECE;
constexpr int PTILE = BM * BN * 2;   // 4 KB, 64-byte rows (SW64)
constexpr int SMEM_Q = 0, SMEM_KV = NPIECE * QPIECE, SMEM_P = SMEM_KV + NST * KTILE;
constexpr int SMEM_BYTES = SMEM_P + 2 * PTILE;
constexpr int N_PROD = 256;          // rope producer threads (warps 4..11)
constexpr int GROUP = N_PROD / NST;  // rope group g (64 threads) owns ring stage g
constexpr int W_TMA = 12;            // c_KV gather warp (TMA tile::gather4)
constexpr int W_MMA = 13;
constexpr uint32_t CKV_TX = BN * DV * 2;  // c_KV bytes landed by TMA per tile
constexpr int THREADS = 32 * (W_MMA + 1);
constexpr uint32_t S_LANE = 16;      // S lives in the upper half-subpartition lanes
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units

struct Params {
    const __nv_bfloat16 *q;
    const __nv_bfloat16 *pool;
    const int32_t *kv_rows;   // [n_kv] pool row of key k (nullptr: identity)
    const int32_t *kv_chunk;  // [n_kv] chunk of key k (nullptr: no rotation)
    const float2 *chunk_cs;   // [n_chunks * 32] (cos, sin)(delta_c * inv_freq[j])
    __nv_bfloat16 *out;
    float *lse;
    int64_t n_rows;           // n_q * heads
    int32_t heads, n_kv, layout;
    int64_t q_pos0;
    float scale_log2;         // softmax scale * log2(e)
    int dbg;                  // IRM_MLA_DEBUG: per-role cycle breakdown of CTA 0
};

__device__ __forceinline__ uint32_t swz128(int row, int chunk) {  // SW128 byte offset (128-B rows)
    return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ uint32_t swz64(int row, int chunk) {   // SW64 byte offset (64-B rows)
    return (uint32_t)(row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
// Per-role cycle counters, printed for CTA 0 when IRM_MLA_DEBUG is set at run time, exist
// only in builds with -DIRM_MLA_PROF_MASK=<roles> (make EXTRA=-DIRM_MLA_PROF_MASK=15).
// Roles: 1 = 2-SM K loader, 2 = 2-SM MMA issuer, 4 = 2-SM softmax, 8 = 1-SM kernel.
#ifndef IRM_MLA_PROF_MASK
#define IRM_MLA_PROF_MASK 0
#endif
constexpr bool kProf = IRM_MLA_PROF_MASK != 0;
template <int ROLE>
__device__ __forceinline__ long long prof_clock() {
    if constexpr ((IRM_MLA_PROF_MASK & ROLE) != 0) return clock64();
    return 0;
}

__device__ __forceinline__ float ex2(float x) {  // 2^x, flush-to-zero; ex2(-inf) = 0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}


// Row max of raw scores with masked keys forced to -inf. Scores are scaled after the
// max (scale > 0), so the exponent is one FFMA per element: ex2(v * scale_log2 - m).
constexpr uint32_t NEG_INF_BITS = 0xff800000u;

__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}

// producers: the k_r part of KV tile `t` -- load kr_base, rotate by R(delta) in
// fp32 (cos/sin from the per-chunk fp64-angle table) -- into registers. Runs
// before the ring slot is free, so its two dependent L2 round trips
// (kv_chunk -> cs) overlap the wait.
struct RopeRegs {
    uint4 v[4];
};

__device__ __forceinline__ void rope_fetch(const Params &p, int t, int ptid, RopeRegs &rr) {
    if (p.layout == IRM_LAYOUT_HALF_SPLIT) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {  // (row, g): dims j = 8g..8g+7 pair with j + 32
            const int it = ptid + q * GROUP, r = it >> 2, g = it & 3;
            const int k = t * BN + r;
            uint4 a = make_uint4(0, 0, 0, 0), b = a;
            if (k < p.n_kv) {
                const int64_t prow = p.kv_rows ? (int64_t)__ldg(p.kv_rows + k) : (int64_t)k;
                const uint4 *src = reinterpret_cast<const uint4 *>(p.pool + prow * DQK + DV);
                a = __ldg(src + g);
                b = __ldg(src + g + 4);
                if (p.kv_chunk) {
                    const float4 *cs = reinterpret_cast<const float4 *>(p.chunk_cs + (int64_t)__ldg(p.kv_chunk + k) * 32 + 8 * g);
                    uint32_t *aw = reinterpret_cast<uint32_t *>(&a), *bw = reinterpret_cast<uint32_t *>(&b);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float4 c = __ldg(cs + e);  // (cos, sin) of pairs 2e and 2e + 1
                        const float l0 = bf_lo(aw[e]), l1 = bf_hi(aw[e]), h0 = bf_lo(bw[e]), h1 = bf_hi(bw[e]);
                        aw[e] = pack_bf2(l0 * c.x - h0 * c.y, l1 * c.z - h1 * c.w);
                        bw[e] = pack_bf2(l0 * c.y + h0 * c.x, l1 * c.w + h1 * c.z);
                    }
                }
            }
            rr.v[2 * q] = a;
            rr.v[2 * q + 1] = b;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // (row, c): pairs (2j, 2j+1), j = 4c..4c+3
            const int it = ptid + q * GROUP, r = it >> 3, c = it & 7;
            const int k = t * BN + r;
            uint4 a = make_uint4(0, 0, 0, 0);
            if (k < p.n_kv) {
                const int64_t prow = p.kv_rows ? (int64_t)__ldg(p.kv_rows + k) : (int64_t)k;
                a = __ldg(reinterpret_cast<const uint4 *>(p.pool + prow * DQK + DV) + c);
                if (p.kv_chunk) {
                    const float4 *cs = reinterpret_cast<const float4 *>(p.chunk_cs + (int64_t)__ldg(p.kv_chunk + k) * 32 + 4 * c);
                    uint32_t *aw = reinterpret_cast<uint32_t *>(&a);
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const float4 cc = __ldg(cs + e);
                        const float l0 = bf_lo(aw[2 * e]), h0 = bf_hi(aw[2 * e]);
                        const float l1 = bf_lo(aw[2 * e + 1]), h1 = bf_hi(aw[2 * e + 1]);
                        aw[2 * e] = pack_bf2(l0 * cc.x - h0 * cc.y, l0 * cc.y + h0 * cc.x);
                        aw[2 * e + 1] = pack_bf2(l1 * cc.z - h1 * cc.w, l1 * cc.w + h1 * cc.z);
                    }
                }
            }
            rr.v[q] = a;
        }
    }
}

// rope producers: write the rotated k_r (piece 8) of KV tile `t` into ring slot
// `tile` and publish it to the async proxy (c_KV arrives by TMA gather4)
__device__ __forceinline__ void store_rope(const Params &p, uint8_t *tile, int ptid, const RopeRegs &rr) {
    const uint32_t rope = smem_u32(tile) + 8 * KPIECE;
    if (p.layout == IRM_LAYOUT_HALF_SPLIT) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int it = ptid + q * GROUP, r = it >> 2, g = it & 3;
            sts128(rope + swz128(r, g), rr.v[2 * q]);
            sts128(rope + swz128(r, g + 4), rr.v[2 * q + 1]);
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int it = ptid + q * GROUP, r = it >> 3, c = it & 7;
            sts128(rope + swz128(r, c), rr.v[q]);
        }
    }
    fence_proxy_async_smem();
}

// BN consecutive pool rows x 64 columns -> one SW128 piece
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *tmap, int col, int row, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(tmap), "r"(col), "r"(row), "r"(smem_u32(bar))
        : "memory");
}

// 32 consecutive pool rows x several 64-column pieces in ONE TMA op (the pool seen as
// [piece][row][64 cols] with a 128-B piece stride): smem gets one 4 KB SW128 piece after
// another, exactly the layout of separate 2-D boxes, for 1/8 (K) or 1/4 (V) of the ops
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *tmap, int row, int piece, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(tmap), "r"(0), "r"(row), "r"(piece), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *tmap, int row, int piece, int group,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        ::"r"(dst), "l"(tmap), "r"(0), "r"(row), "r"(piece), "r"(group), "r"(smem_u32(bar))
        : "memory");
}

// .cta_group::2 forms: the data lands in the issuing CTA's smem, the transaction bytes
// complete on the LEADER CTA's mbarrier (bar = its shared::cluster address), so the peer's
// loads need no relay
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap *tmap, int row, int piece, int group,
                                                 uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst), "l"(tmap), "r"(0), "r"(row), "r"(piece), "r"(group), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap *tmap, int row, int piece,
                                                 uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst), "l"(tmap), "r"(0), "r"(row), "r"(piece), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_gather4_pair(uint32_t dst, const CUtensorMap *tmap, int col, int r0, int r1,
                                                 int r2, int r3, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(tmap), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *tmap, int col, int row, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(tmap), "r"(col), "r"(row), "r"(bar)
        : "memory");
}

// 4 arbitrary pool rows x 64 columns (128 B each) -> 512 B of a SW128 piece
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap *tmap, int col, int r0, int r1, int r2,
                                            int r3, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(tmap), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

static_assert(BN * 4 == 2 * GROUP && BN * 8 == 4 * GROUP, "rope work split assumes 2 / 4 items per producer");

__global__ void __launch_bounds__(THREADS, 1) mla_reattach_kernel(Params p, const __grid_constant__ CUtensorMap tmap_pool,
                                                                    const __grid_constant__ CUtensorMap tmap_tile) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bar_q, bar_kv_full[NST], bar_kv_empty[NST], bar_s_full[2], bar_p_full[2],
        bar_o_done[2];
    __shared__ uint32_t tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int64_t last_row = min(p.n_rows, row0 + BM) - 1;
    const int64_t max_pos = p.q_pos0 + last_row / p.heads;
    const int n_keys = (int)min((int64_t)p.n_kv, max_pos + 1);
    const int T = (n_keys + BN - 1) / BN;
    // CTAs of a wave start at scattered key tiles (any order is exact under the
    // online softmax), so concurrent CTAs do not hammer the same L2 lines
    const int toff = (int)(((uint32_t)blockIdx.x * 2654435761u) % (uint32_t)T);

    if (threadIdx.x == 0) {
        mbar_init(&bar_q, N_PROD);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&bar_kv_full[s], GROUP + 1);  // rope group + the TMA thread's expect_tx
            mbar_init(&bar_kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bar_s_full[s], 1);
            mbar_init(&bar_p_full[s], 128);
            mbar_init(&bar_o_done[s], 1);
        }
        fence_mbar_init();
    }
    if (warp == W_MMA) tc::tmem_alloc(&tmem_base, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tmem_base;

    if (warp >= 4 && warp < W_TMA) {
        // ------------------------------------------------------ Q (cp.async, once) + rope producers
        const int ptid = threadIdx.x - 128;
        const uint32_t qbase = smem_u32(smem + SMEM_Q);
        for (int i = ptid; i < BM * 72; i += N_PROD) {
            const int r = i / 72, c = i % 72;
            const int64_t grow = row0 + r;
            const bool ok = grow < p.n_rows;
            cp_async16(qbase + (c >> 3) * QPIECE + swz128(r, c & 7), p.q + (ok ? grow : 0) * DQK + c * 8, ok ? 16u : 0u);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        fence_proxy_async_smem();
        mbar_arrive(&bar_q);
        // NST independent rope groups: group g handles tiles g, g + NST, ... (ring stage g)
        const int g = ptid / GROUP, gtid = ptid % GROUP;
        long long c_wait = 0, c_load = 0, c0 = prof_clock<8>();
        for (int t = g; t < T; t += NST) {
            const int kt = (t + toff) % T;
            RopeRegs rr;
            rope_fetch(p, kt, gtid, rr);
            long long a = prof_clock<8>();
            if (t >= NST) mbar_wait(&bar_kv_empty[g], ((t / NST) - 1) & 1);
            long long b2 = prof_clock<8>();
            store_rope(p, smem + SMEM_KV + g * KTILE, gtid, rr);
            mbar_arrive(&bar_kv_full[g]);
            c_wait += b2 - a;
            c_load += prof_clock<8>() - b2;
        }
        if (kProf && p.dbg && blockIdx.x == 0 && gtid == 0)
            printf("rope g%d: wait_empty %lld store %lld total %lld (T=%d)\n", g, c_wait, c_load, prof_clock<8>() - c0, T);
    } else if (warp == W_TMA) {
        // ------------------------------------------------------ c_KV by TMA gather4 (paged rows)
        // lane i resolves the pool row of key i of the tile; lanes 0..7 each issue the
        // 8 gather4 (pieces 0..7) of rows 4i..4i+3
        long long c_wait = 0, c0 = prof_clock<8>();
        for (int t = 0; t < T; ++t) {
            const int st = t % NST, kt = (t + toff) % T;
            const int k = kt * BN + lane;
            const int row = k < p.n_kv ? (p.kv_rows ? __ldg(p.kv_rows + k) : k) : -1;  // -1: OOB, zero-filled
            long long a = prof_clock<8>();
            if (t >= NST) mbar_wait(&bar_kv_empty[st], ((t / NST) - 1) & 1);
            c_wait += prof_clock<8>() - a;
            if (lane == 0) mbar_arrive_expect_tx(&bar_kv_full[st], CKV_TX);
            __syncwarp();
            // a run of BN consecutive pool rows (the common case: chunks are contiguous in
            // the pool) goes as 8 tiled boxes; anything else as 64 gather4
            const int row0 = __shfl_sync(0xffffffffu, row, 0);
            if (__all_sync(0xffffffffu, row0 >= 0 && row == row0 + lane)) {
                if (lane == 0) {
                    const uint32_t dst = smem_u32(smem + SMEM_KV + st * KTILE);
#pragma unroll
                    for (int pc = 0; pc < 8; ++pc)
                        tma_load_2d(dst + pc * KPIECE, &tmap_tile, 64 * pc, row0, &bar_kv_full[st]);
                }
                continue;
            }
            const int r0 = __shfl_sync(0xffffffffu, row, 4 * (lane & 7));
            const int r1 = __shfl_sync(0xffffffffu, row, 4 * (lane & 7) + 1);
            const int r2 = __shfl_sync(0xffffffffu, row, 4 * (lane & 7) + 2);
            const int r3 = __shfl_sync(0xffffffffu, row, 4 * (lane & 7) + 3);
            if (lane < BN / 4) {
                const uint32_t dst = smem_u32(smem + SMEM_KV + st * KTILE) + lane * 512;
#pragma unroll
                for (int pc = 0; pc < 8; ++pc)
                    tma_gather4(dst + pc * KPIECE, &tmap_pool, 64 * pc, r0, r1, r2, r3, &bar_kv_full[st]);
            }
        }
        if (kProf && p.dbg && blockIdx.x == 0 && lane == 0)
            printf("tma: wait_empty %lld total %lld\n", c_wait, prof_clock<8>() - c0);
    } else if (warp == W_MMA) {
        // ------------------------------------------------------ MMA issuer
        // The warp stays converged (barrier waits by all lanes); one elected lane
        // issues each unrolled batch. Descriptors are built once: per MMA only the
        // 14-bit start-address field (bytes >> 4) advances, so a batch is a run of
        // UTCHMMA with immediate offsets.
        const uint32_t idesc_qk = tc::idesc_bf16(BM, BN, false, false);
        const uint32_t idesc_pv = tc::idesc_bf16(BM, 256, false, true);
        const uint64_t q_desc = tc::smem_desc_sw128(smem_u32(smem + SMEM_Q), 16, 1024);
        const uint64_t kv_desc = tc::smem_desc_sw128(smem_u32(smem + SMEM_KV), 16, 1024);
        const uint64_t v_desc = tc::smem_desc_sw128(smem_u32(smem + SMEM_KV), KPIECE, 1024);
        const uint64_t p_desc = tc::smem_desc_sw64(smem_u32(smem + SMEM_P), 16, 512);
        const uint32_t q_lo = (uint32_t)q_desc, q_hi = (uint32_t)(q_desc >> 32);
        const uint32_t kv_lo = (uint32_t)kv_desc, kv_hi = (uint32_t)(kv_desc >> 32);
        const uint32_t v_lo = (uint32_t)v_desc, v_hi = (uint32_t)(v_desc >> 32);
        const uint32_t p_lo = (uint32_t)p_desc, p_hi = (uint32_t)(p_desc >> 32);
        long long c_kv = 0, c_p = 0, c0 = prof_clock<8>();
        auto issue_qk = [&](int t) {
            const int st = t % NST;
            long long a = prof_clock<8>();
            mbar_wait(&bar_kv_full[st], (t / NST) & 1);
            c_kv += prof_clock<8>() - a;
            tc::fence_after();
            const uint32_t d = tbase + (S_LANE << 16) + (t & 1) * BN;
            if (tc::elect_one()) {
                uint32_t qa = q_lo, kb = kv_lo + ((st * KTILE) >> 4);  // see the 2-SM issue loop
#pragma unroll 1
                for (int pc = 0; pc < NPIECE; ++pc) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc::mma_bf16_ss_w(d, qa + 2 * k, q_hi, kb + 2 * k, kv_hi, idesc_qk, (pc | k) != 0);
                    qa += QPIECE >> 4;
                    kb += KPIECE >> 4;
                }
                tc::commit(&bar_s_full[t & 1]);
            }
            __syncwarp();
        };
        mbar_wait(&bar_q, 0);
        issue_qk(0);
        for (int t = 0; t < T; ++t) {
            // S buffer (t+1)&1 was consumed by softmax(t-1): its P(t-1) arrived before PV(t-1)
            if (t + 1 < T) issue_qk(t + 1);
            const int st = t % NST;
            long long a = prof_clock<8>();
            mbar_wait(&bar_p_full[t & 1], (t >> 1) & 1);
            c_p += prof_clock<8>() - a;
            tc::fence_after();
            const uint32_t pd = p_lo + (((t & 1) * PTILE) >> 4);
            const uint32_t vd = v_lo + ((st * KTILE) >> 4);
            if (tc::elect_one()) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int k = 0; k < BN / 16; ++k)
                        tc::mma_bf16_ss_w(tbase + h * 256, pd + ((k * 32) >> 4), p_hi,
                                          vd + ((4 * h * KPIECE + k * 2048) >> 4), v_hi, idesc_pv,
                                          (t > 0 || k > 0) ? 1u : 0u);
                }
                tc::commit(&bar_kv_empty[st]);
                tc::commit(&bar_o_done[t & 1]);
            }
            __syncwarp();
        }
        if (kProf && p.dbg && blockIdx.x == 0 && lane == 0)
            printf("mma: wait_kv %lld wait_p %lld total %lld\n", c_kv, c_p, prof_clock<8>() - c0);
    } else {
        // ------------------------------------------------------ softmax / correction (warps 0-3)
        const int w = warp;
        const int L = (lane >> 2) + 8 * (lane & 1);  // TMEM lane within the 16-lane group
        const int b = (lane >> 1) & 1;               // column parity of this thread
        const int r = 16 * w + L;                    // tile row
        const int64_t grow = row0 + r;
        const bool row_ok = grow < p.n_rows;
        const int64_t qpos = p.q_pos0 + (row_ok ? grow / p.heads : 0);
        const uint32_t s_lane = tbase + (((uint32_t)(32 * w) + S_LANE) << 16);
        const uint32_t o_lane = tbase + ((uint32_t)(32 * w) << 16);
        const uint32_t p_base = smem_u32(smem + SMEM_P);
        float m = -INFINITY, l = 0.f;
        long long c_s = 0, c_o = 0, c_r = 0, c0 = prof_clock<8>();
        for (int t = 0; t < T; ++t) {
            long long a = prof_clock<8>();
            mbar_wait(&bar_s_full[t & 1], (t >> 1) & 1);
            c_s += prof_clock<8>() - a;
            tc::fence_after();
            uint32_t v[16];
            tc::ld_16x64b_x16(s_lane + (t & 1) * BN, v);
            tc::wait_ld();
            float s[16];
            const int64_t kbase = (int64_t)((t + toff) % T) * BN + b;
            // the causal / length mask only touches diagonal and tail tiles
            if (!__all_sync(0xffffffffu, row_ok && kbase + 30 <= qpos && kbase + 30 < p.n_kv)) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t key = kbase + 2 * i;
                    if (!(row_ok && key <= qpos && key < p.n_kv)) v[i] = NEG_INF_BITS;
                }
            }
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int i = 0; i < 16; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(v[i]));
            float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
            mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
            float alpha = 1.f;
            const float m_new = fmaxf(m, mt);
            if (m_new > m + RESCALE_THRESHOLD) {  // lazy rescale: only when the max grows by > 2^8
                alpha = (m == -INFINITY) ? 0.f : ex2(m - m_new);
                m = m_new;
            }
            const float nm = (m == -INFINITY) ? 0.f : -m;  // fully masked so far: every v is -inf
            float ls[2] = {0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                s[i] = ex2(fmaf(__uint_as_float(v[i]), p.scale_log2, nm));
                ls[i & 1] += s[i];
            }
            float lsum = ls[0] + ls[1];
            lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
            l = l * alpha + lsum;
            // pack P: pairs of adjacent keys, thread b = 0 takes keys 0..15, b = 1 keys 16..31
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float other = __shfl_xor_sync(0xffffffffu, s[i], 2);
                const uint32_t pr = b == 0 ? pack_bf2(s[i], other) : pack_bf2(other, s[i]);
                if ((i >> 3) == b) pk[i & 7] = pr;
            }
            // P buffer t&1 is free once PV(t-2) completed
            a = prof_clock<8>();
            if (t >= 2) mbar_wait(&bar_o_done[t & 1], ((t >> 1) - 1) & 1);
            c_o += prof_clock<8>() - a;
            a = prof_clock<8>();
            if (t >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
                mbar_wait(&bar_o_done[(t - 1) & 1], ((t - 1) >> 1) & 1);  // O holds PV(0..t-1)
                tc::fence_after();
#pragma unroll 1
                for (int c = 0; c < DV / 64; ++c) {
                    uint32_t o[32];
                    tc::ld_16x64b_x32(o_lane + c * 64, o);
                    tc::wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tc::st_16x64b_x32(o_lane + c * 64, o);
                }
                tc::wait_st();
            }
            c_r += prof_clock<8>() - a;
            const uint32_t pt = p_base + (t & 1) * PTILE;
            sts128(pt + swz64(r, 2 * b), make_uint4(pk[0], pk[1], pk[2], pk[3]));
            sts128(pt + swz64(r, 2 * b + 1), make_uint4(pk[4], pk[5], pk[6], pk[7]));
            fence_proxy_async_smem();
            tc::fence_before();
            mbar_arrive(&bar_p_full[t & 1]);
        }
        if (kProf && p.dbg && blockIdx.x == 0 && lane == 0)
            printf("softmax w%d: wait_s %lld wait_o %lld rescale %lld total %lld\n", w, c_s, c_o, c_r, prof_clock<8>() - c0);
        // epilogue: O / l -> bf16, lse
        mbar_wait(&bar_o_done[(T - 1) & 1], ((T - 1) >> 1) & 1);
        tc::fence_after();
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
        for (int c = 0; c < DV / 64; ++c) {
            uint32_t o[32];
            tc::ld_16x64b_x32(o_lane + c * 64, o);
            tc::wait_ld();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float mine = __uint_as_float(o[i]) * inv_l;
                const float other = __shfl_xor_sync(0xffffffffu, mine, 2);
                const uint32_t pr = b == 0 ? pack_bf2(mine, other) : pack_bf2(other, mine);
                if ((i >> 4) == b) pk[i & 15] = pr;
            }
            if (row_ok) {
                uint4 *dst = reinterpret_cast<uint4 *>(p.out + grow * DV + c * 64 + 32 * b);
                dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                dst[2] = make_uint4(pk[8], pk[9], pk[10], pk[11]);
                dst[3] = make_uint4(pk[12], pk[13], pk[14], pk[15]);
            }
        }
        if (row_ok && b == 0 && p.lse) p.lse[grow] = (m + log2f(l)) * 0.69314718055994531f;
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == W_MMA) tc::tmem_dealloc(tbase, 512);
}

// ============================================================================
// CTA-pair (cta_group::2) variant: one cluster of 2 CTAs owns 128 rows and a
// 64-key tile per step. The leader CTA issues M = 128 MMAs whose A operand is
// split by rows (each CTA holds its 64 Q / P rows) and whose B operand is split
// by N (QK: each CTA holds 32 of the 64 keys; PV: each CTA holds 128 of each
// 256 latent dims). D lands in each CTA's TMEM in the 2x2 layout: S [64 x 64]
// in 32 columns (lanes 0-63 keys 0-31, lanes 64-127 keys 32-63), O [64 x 512]
// in 256 columns. Full tensor-core rate per SM, half the smem operand traffic
// per FLOP of the M = 64 kernel.
namespace p2 {

constexpr int PBN = 64;                     // keys per pair tile (QK N)
constexpr int VPIECE = 32 * 128;            // 4 KB: 32 keys x 64 dims (SW128)
constexpr int VTILE = 4 * VPIECE;           // V half-tile: 32 keys x this CTA's 256 latent dims
#ifndef IRM_MLA_VST
#define IRM_MLA_VST 4
#endif
constexpr int KST = 2, VST = IRM_MLA_VST;             // ring stages (V in half-tiles: PV(t) is two K=32 halves)
constexpr int PTILE2 = 64 * 128;            // P [64 rows x 64 keys] bf16, SW128
// Q pieces [0, QT) live in TMEM as the A operand of TS-mode QK MMAs (read by the tensor
// core from TMEM, not shared memory); pieces [QT, 9) stay in shared memory (SS mode)
#ifndef IRM_MLA_QT
#define IRM_MLA_QT 6
#endif
constexpr int QT = IRM_MLA_QT;
constexpr int S_Q = 0, S_K = (NPIECE - QT) * QPIECE, S_V = S_K + KST * KTILE, S_P = S_V + VST * VTILE;
constexpr int SMEM2 = S_P + 2 * PTILE2;     // 224 KB - QT x 8 KB
constexpr int W_KTMA = 8, W_MMA2 = 9, W_VTMA = 10;
constexpr int THREADS2 = 32 * 11;
constexpr uint32_t COL_S = 0, COL_O = 64;   // TMEM columns: S[2] x 32, O 2 x 128
constexpr uint32_t COL_Q = 320;             // Q pieces [0, QT): 32 columns each (bf16 pairs)
static_assert(COL_Q + 32 * QT <= 512, "TMEM holds at most 6 Q pieces next to S and O");

__device__ __forceinline__ void arrive_leader(uint64_t *bar, uint32_t rank) {
    if (rank == 0) mbar_arrive(bar);
    else cl::remote_arrive(cl::map_to(smem_u32(bar), 0));
}

// Rows of keys [k0, k0 + 32): one kv_rows read per lane, reused for every column piece.
struct Rows32 {
    int row;     // this lane's pool row (-1 past n_kv)
    int row0;    // lane 0's row
    bool contig; // all 32 rows form one ascending run -> one tiled TMA box per piece
};

__device__ __forceinline__ int key_row(const Params &p, int k) {
    return k < p.n_kv ? (p.kv_rows ? __ldg(p.kv_rows + k) : k) : -1;
}

__device__ __forceinline__ Rows32 rows32_resolve(int row, int lane) {
    Rows32 r;
    r.row = row;
    r.row0 = __shfl_sync(0xffffffffu, row, 0);
    r.contig = __all_sync(0xffffffffu, r.row0 >= 0 && row == r.row0 + lane);
    return r;
}

// TMA of the 32 rows of column piece `col_piece` into dst (a 32-row SW128 box): a tiled box
// for a contiguous run, else eight tile::gather4 ops (lanes 0-7, four rows each)
__device__ __forceinline__ void tma_rows32(const Rows32 &r, const CUtensorMap *tm_g4, const CUtensorMap *tm_tile,
                                           uint32_t dst, int col_piece, int lane, uint64_t *bar) {
    if (r.contig) {
        if (lane == 0) tma_load_2d(dst, tm_tile, 64 * col_piece, r.row0, bar);
        return;
    }
    const int g = lane & 7;
    const int r0 = __shfl_sync(0xffffffffu, r.row, 4 * g), r1 = __shfl_sync(0xffffffffu, r.row, 4 * g + 1);
    const int r2 = __shfl_sync(0xffffffffu, r.row, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, r.row, 4 * g + 3);
    if (lane < 8) tma_gather4(dst + lane * 512, tm_g4, 64 * col_piece, r0, r1, r2, r3, bar);
}

// the same 32 rows, completing on the leader's barrier (bar: shared::cluster address)
__device__ __forceinline__ void tma_rows32_pair(const Rows32 &r, const CUtensorMap *tm_g4, const CUtensorMap *tm_tile,
                                                uint32_t dst, int col_piece, int lane, uint32_t bar) {
    if (r.contig) {
        if (lane == 0) tma_load_2d_pair(dst, tm_tile, 64 * col_piece, r.row0, bar);
        return;
    }
    const int g = lane & 7;
    const int r0 = __shfl_sync(0xffffffffu, r.row, 4 * g), r1 = __shfl_sync(0xffffffffu, r.row, 4 * g + 1);
    const int r2 = __shfl_sync(0xffffffffu, r.row, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, r.row, 4 * g + 3);
    if (lane < 8) tma_gather4_pair(dst + lane * 512, tm_g4, 64 * col_piece, r0, r1, r2, r3, bar);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS2, 1)
mla_reattach_2sm_kernel(Params p, const __grid_constant__ CUtensorMap tmap_pool,
                        const __grid_constant__ CUtensorMap tmap_tile, const __grid_constant__ CUtensorMap tmap_k8,
                        const __grid_constant__ CUtensorMap tmap_v4) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t b_q, b_qpair, b_kfull[KST], b_krope[KST], b_vfull[VST],
        b_kempty[KST], b_vempty[VST], b_sfull[2], b_pfull[2], b_odone[2];
    __shared__ float sx[2][2][64];  // row-max exchange between the two key halves
    __shared__ float sl[2][64];     // final row-sum exchange
    __shared__ uint32_t tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cl::cta_rank();
    const int64_t prow0 = (int64_t)(blockIdx.x >> 1) * 128;  // first row of the pair
    const int64_t row0 = prow0 + 64 * rank;                 // first row of this CTA
    const int64_t last_row = min(p.n_rows, prow0 + 128) - 1;
    const int64_t max_pos = p.q_pos0 + last_row / p.heads;
    const int n_keys = (int)min((int64_t)p.n_kv, max_pos + 1);
    const int T = (n_keys + PBN - 1) / PBN;
    const int toff = (int)(((uint32_t)(blockIdx.x >> 1) * 2654435761u) % (uint32_t)T);

    if (threadIdx.x == 0) {
        mbar_init(&b_q, QT > 0 ? 256 : 128);  // smem Q (producers) + TMEM Q (softmax warps)
        mbar_init(&b_qpair, 1);
        for (int s = 0; s < KST; ++s) {
            // leader: its TMA expect_tx (both CTAs' c_KV bytes land here) + its rope group + the
            // peer's rope readiness (relayed); peer: b_krope collects its rope group
            mbar_init(&b_kfull[s], 2 + GROUP);
            mbar_init(&b_krope[s], GROUP);
            mbar_init(&b_kempty[s], 1);
        }
        for (int s = 0; s < VST; ++s) {
            mbar_init(&b_vfull[s], 1);  // leader: its expect_tx; the peer's bytes complete here too
            mbar_init(&b_vempty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&b_sfull[s], 1);
            mbar_init(&b_pfull[s], rank == 0 ? 128 + 1 : 128);  // local softmax threads (+ the peer's relay)
            mbar_init(&b_odone[s], 1);
        }
        fence_mbar_init();
    }
    if (warp == W_MMA2) tc2::tmem_alloc(&tmem_base, 512);
    tc::fence_before();
    cl::cluster_sync();
    tc::fence_after();
    const uint32_t tbase = tmem_base;

    if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ Q (once) + rope of this CTA's 32 keys
        const int ptid = threadIdx.x - 128;
        const uint32_t qbase = smem_u32(smem + S_Q);
        constexpr int QC = (NPIECE - QT) * 8;  // 16-byte chunks per row kept in smem
        for (int i = ptid; i < 64 * QC; i += 128) {
            const int r = i / QC, c = i % QC + QT * 8;
            const int64_t grow = row0 + r;
            const bool ok = grow < p.n_rows;
            cp_async16(qbase + ((c >> 3) - QT) * QPIECE + swz128(r, c & 7), p.q + (ok ? grow : 0) * DQK + c * 8,
                       ok ? 16u : 0u);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        fence_proxy_async_smem();
        mbar_arrive(&b_q);
        const int g = ptid / GROUP, gtid = ptid % GROUP;  // group g owns K stage g
        for (int t = g; t < T; t += KST) {
            const int kt = (t + toff) % T;
            RopeRegs rr;
            rope_fetch(p, 2 * kt + (int)rank, gtid, rr);  // keys kt*64 + 32*rank + [0, 32)
            if (t >= KST) mbar_wait(&b_kempty[g], ((t / KST) - 1) & 1);
            store_rope(p, smem + S_K + g * KTILE, gtid, rr);
            mbar_arrive(rank == 0 ? &b_kfull[g] : &b_krope[g]);
        }
    } else if (warp == W_KTMA) {
        // ------------------------------------------------ c_KV of this CTA's 32 keys (QK operand)
        long long c_e = 0, c0 = prof_clock<1>();
        int row_next = key_row(p, (toff % T) * PBN + 32 * (int)rank + lane);  // rows read one tile ahead
        for (int t = 0; t < T; ++t) {
            const int st = t % KST;
            const Rows32 rr = rows32_resolve(row_next, lane);
            if (t + 1 < T) row_next = key_row(p, ((t + 1 + toff) % T) * PBN + 32 * (int)rank + lane);
            long long a0 = prof_clock<1>();
            if (t >= KST) mbar_wait(&b_kempty[st], ((t / KST) - 1) & 1);
            c_e += prof_clock<1>() - a0;
            // both CTAs' c_KV bytes complete on the leader's b_kfull (peer: .cta_group::2 TMA)
            if (rank == 0 && lane == 0) mbar_arrive_expect_tx(&b_kfull[st], 2 * CKV_TX);
            __syncwarp();
            const uint32_t dst = smem_u32(smem + S_K + st * KTILE);
            const uint32_t kbar = cl::map_to(smem_u32(&b_kfull[st]), 0);
            if (rr.contig) {  // one op for the 8 c_KV pieces of 32 consecutive rows
                if (lane == 0) tma_load_3d_pair(dst, &tmap_k8, rr.row0, 0, kbar);
            } else {
                for (int pc = 0; pc < 8; ++pc)
                    tma_rows32_pair(rr, &tmap_pool, &tmap_tile, dst + pc * KPIECE, pc, lane, kbar);
            }
        }
        if (kProf && p.dbg && blockIdx.x < 2 && lane == 0)
            printf("2sm ktma cta%d: wait_empty %lld total %lld\n", (int)rank, c_e, prof_clock<1>() - c0);
    } else if (warp == W_VTMA) {
        // ------------------------------------------------ V: all 64 keys x this CTA's 256 latent dims
        // key half-tiles u = 2t + a: keys [64 kt + 32a, +32), rows read one half-tile ahead
        int row_next = key_row(p, (toff % T) * PBN + lane);
        long long c_ve = 0, c_vi = 0, c0v = prof_clock<1>();
        for (int u = 0; u < 2 * T; ++u) {
            const int st = u % VST;
            const Rows32 rr = rows32_resolve(row_next, lane);
            if (u + 1 < 2 * T) row_next = key_row(p, (((u + 1) / 2 + toff) % T) * PBN + 32 * ((u + 1) & 1) + lane);
            long long a0 = prof_clock<1>();
            if (u >= VST) mbar_wait(&b_vempty[st], ((u / VST) - 1) & 1);
            c_ve += prof_clock<1>() - a0;
            long long a1 = prof_clock<1>();
            // the leader's b_vfull[st] completes when BOTH CTAs' half-tiles have landed: the
            // leader expects 2 x VTILE bytes, the peer's TMA completes on that barrier directly
            if (rank == 0 && lane == 0) mbar_arrive_expect_tx(&b_vfull[st], 2 * (uint32_t)VTILE);
            __syncwarp();
            const uint32_t dst = smem_u32(smem + S_V + st * VTILE);
            const uint32_t vbar = cl::map_to(smem_u32(&b_vfull[st]), 0);
            if (rr.contig) {  // one op: pieces 4h + 2 rank + i, (h, i) in {0,1}^2
                if (lane == 0) tma_load_4d_pair(dst, &tmap_v4, rr.row0, 2 * (int)rank, 0, vbar);
            } else {
                for (int j = 0; j < 4; ++j) {
                    const int cpiece = (j >> 1) * 4 + 2 * (int)rank + (j & 1);  // dims [256h + 128 rank, +128)
                    tma_rows32_pair(rr, &tmap_pool, &tmap_tile, dst + j * VPIECE, cpiece, lane, vbar);
                }
            }
            c_vi += prof_clock<1>() - a1;
        }
        if (kProf && p.dbg && blockIdx.x < 2 && lane == 0)
            printf("2sm vtma cta%d: wait_empty %lld issue %lld total %lld\n", (int)rank, c_ve, c_vi, prof_clock<1>() - c0v);
    } else if (warp == W_MMA2) {
        if (rank != 0) {
            // ------------------------------------------------ peer: relay local data readiness to the leader
            const uint32_t q_l = cl::map_to(smem_u32(&b_qpair), 0);
            mbar_wait(&b_q, 0);
            if (lane == 0) cl::remote_arrive(q_l);
            auto relay_k = [&](int t) {  // the peer's rotated k_r is in smem
                mbar_wait(&b_krope[t % KST], (t / KST) & 1);
                if (lane == 0) cl::remote_arrive(cl::map_to(smem_u32(&b_kfull[t % KST]), 0));
            };
            relay_k(0);
            // forwarded in the leader's consumption order: K(t+1) for QK, then P(t) and V(t) for PV.
            // A cluster-scope release costs ~1.5K cycles; doing it here keeps it off the softmax path.
            for (int t = 0; t < T; ++t) {
                if (t + 1 < T) relay_k(t + 1);
                mbar_wait(&b_pfull[t & 1], (t >> 1) & 1);
                if (lane == 0) cl::remote_arrive(cl::map_to(smem_u32(&b_pfull[t & 1]), 0));
            }
        } else {
            // ------------------------------------------------ leader: MMA issue for the pair
            const uint32_t idesc_qk = tc::idesc_bf16(128, PBN, false, false);
            const uint32_t idesc_pv = tc::idesc_bf16(128, 256, false, true);
            const uint64_t q_desc = tc::smem_desc_sw128(smem_u32(smem + S_Q), 16, 1024);
            const uint64_t k_desc = tc::smem_desc_sw128(smem_u32(smem + S_K), 16, 1024);
            const uint64_t v_desc = tc::smem_desc_sw128(smem_u32(smem + S_V), VPIECE, 1024);
            const uint64_t p_desc = tc::smem_desc_sw128(smem_u32(smem + S_P), 16, 1024);
            const uint32_t q_lo = (uint32_t)q_desc, q_hi = (uint32_t)(q_desc >> 32);
            const uint32_t k_lo = (uint32_t)k_desc, k_hi = (uint32_t)(k_desc >> 32);
            const uint32_t v_lo = (uint32_t)v_desc, v_hi = (uint32_t)(v_desc >> 32);
            const uint32_t p_lo = (uint32_t)p_desc, p_hi = (uint32_t)(p_desc >> 32);
            mbar_wait(&b_q, 0);
            mbar_wait(&b_qpair, 0);
            long long c_k = 0, c_kp = 0, c_p = 0, c_v = 0, c_vl = 0, c0 = prof_clock<2>();
            auto issue_qk = [&](int t) {
                const int st = t % KST;
                long long a0 = prof_clock<2>();
                mbar_wait(&b_kfull[st], (t / KST) & 1);  // both CTAs' K tiles (bytes + rope)
                long long a1 = prof_clock<2>();
                c_k += a1 - a0;
                c_kp += prof_clock<2>() - a1;
                tc::fence_after();
                const uint32_t kd = k_lo + ((st * KTILE) >> 4);
                const uint32_t ds = tbase + COL_S + (t & 1) * 32;
                if (tc::elect_one()) {
                    // one 64-dim piece per iteration, descriptors advanced incrementally: a fully
                    // unrolled loop hoists all 72 descriptors into uniform registers and spills
                    uint32_t qa = q_lo, kb = kd, qt = tbase + COL_Q;
#pragma unroll 1
                    for (int pc = 0; pc < QT; ++pc) {  // A = Q from TMEM
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc2::mma_bf16_ts_w(ds, qt + 8 * k, kb + 2 * k, k_hi, idesc_qk, (pc | k) != 0);
                        qt += 32;
                        kb += KPIECE >> 4;
                    }
#pragma unroll 1
                    for (int pc = QT; pc < NPIECE; ++pc) {  // A = Q from shared memory
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc2::mma_bf16_ss_w(ds, qa + 2 * k, q_hi, kb + 2 * k, k_hi, idesc_qk, (pc | k) != 0);
                        qa += QPIECE >> 4;
                        kb += KPIECE >> 4;
                    }
                    tc2::commit_both(&b_sfull[t & 1]);
                    tc2::commit_both(&b_kempty[st]);
                }
                __syncwarp();
            };
            issue_qk(0);
            for (int t = 0; t < T; ++t) {
                if (t + 1 < T) issue_qk(t + 1);
                long long a0 = prof_clock<2>();
                mbar_wait(&b_pfull[t & 1], (t >> 1) & 1);
                c_p += prof_clock<2>() - a0;
                const uint32_t pd = p_lo + (((t & 1) * PTILE2) >> 4);
#pragma unroll 1
                for (int a = 0; a < 2; ++a) {  // PV over key half a, as soon as its V half-tile lands
                    const int u = 2 * t + a, vs = u % VST;
                    long long a1 = prof_clock<2>();
                    mbar_wait(&b_vfull[vs], (u / VST) & 1);  // both CTAs' V half-tiles
                    c_vl += prof_clock<2>() - a1;
                    c_v += prof_clock<2>() - a1;
                    tc::fence_after();
                    const uint32_t vd = v_lo + ((vs * VTILE) >> 4);
                    if (tc::elect_one()) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
#pragma unroll
                            for (int k = 0; k < 2; ++k)
                                tc2::mma_bf16_ss_w(tbase + COL_O + h * 128, pd + (((2 * a + k) * 32) >> 4), p_hi,
                                                   vd + ((2 * h * VPIECE + k * 2048) >> 4), v_hi, idesc_pv,
                                                   (t > 0 || a > 0 || k > 0) ? 1u : 0u);
                        }
                        tc2::commit_both(&b_vempty[vs]);
                        if (a == 1) tc2::commit_both(&b_odone[t & 1]);
                    }
                    __syncwarp();
                }
            }
            if (kProf && p.dbg && blockIdx.x == 0 && lane == 0)
                printf("2sm mma: wait_k %lld wait_kpair %lld wait_p %lld wait_v %lld (local %lld) total %lld T=%d\n", c_k, c_kp,
                       c_p, c_v, c_vl, prof_clock<2>() - c0, T);
        }
    } else {
        // ------------------------------------------------ softmax / correction (warps 0-3)
        const int w = warp;
        const int r = 32 * (w & 1) + lane;  // row of this CTA
        const int kh = w >> 1;              // key half (S) / latent-dim half (O)
        const int64_t grow = row0 + r;
        const bool row_ok = grow < p.n_rows;
        const int64_t qpos = p.q_pos0 + (row_ok ? grow / p.heads : 0);
        const uint32_t lane_base = tbase + ((uint32_t)(32 * w) << 16);
        const uint32_t p_base = smem_u32(smem + S_P);
        const uint32_t pfull_leader0 = cl::map_to(smem_u32(&b_pfull[0]), 0);
        const uint32_t pfull_leader1 = cl::map_to(smem_u32(&b_pfull[1]), 0);
        if constexpr (QT > 0) {
            // this thread's row of Q, pieces [0, QT), into its TMEM lane (rows are duplicated
            // across the lane halves: warps w and w + 2 hold the same rows, as the 2-SM TS
            // A operand expects)
            const uint4 *src = reinterpret_cast<const uint4 *>(p.q + (row_ok ? grow : 0) * DQK);
#pragma unroll 1
            for (int pc = 0; pc < QT; ++pc) {
                uint32_t qv[32];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint4 x = row_ok ? __ldg(src + 8 * pc + j) : make_uint4(0, 0, 0, 0);
                    qv[4 * j] = x.x;
                    qv[4 * j + 1] = x.y;
                    qv[4 * j + 2] = x.z;
                    qv[4 * j + 3] = x.w;
                }
                tc2::st_32x32b_x32(lane_base + COL_Q + 32 * pc, qv);
            }
            tc::wait_st();
            tc::fence_before();
            mbar_arrive(&b_q);
        }
        float m = -INFINITY, l = 0.f;
        long long c_s = 0, c_o = 0, c_x = 0, c_r = 0, c_e = 0, c_ld = 0, c_mx = 0, c_ex = 0, c0 = prof_clock<4>();
        for (int t = 0; t < T; ++t) {
            long long a0 = prof_clock<4>();
            mbar_wait(&b_sfull[t & 1], (t >> 1) & 1);
            c_s += prof_clock<4>() - a0;
            tc::fence_after();
            uint32_t v[32];
            long long b0 = prof_clock<4>();
            tc2::ld_32x32b_x32(lane_base + COL_S + (t & 1) * 32, v);
            tc::wait_ld();
            long long b1 = prof_clock<4>();
            c_ld += b1 - b0;
            const int64_t kbase = (int64_t)((t + toff) % T) * PBN + 32 * kh;
            if (!__all_sync(0xffffffffu, row_ok && kbase + 31 <= qpos && kbase + 31 < p.n_kv)) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int64_t key = kbase + i;
                    if (!(row_ok && key <= qpos && key < p.n_kv)) v[i] = NEG_INF_BITS;
                }
            }
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int i = 0; i < 32; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(v[i]));
            float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
            sx[t & 1][kh][r] = mt;  // exchange with the thread holding the other key half
            long long a1 = prof_clock<4>();
            c_mx += a1 - b1;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            c_x += prof_clock<4>() - a1;
            mt = fmaxf(mt, sx[t & 1][kh ^ 1][r]);
            float alpha = 1.f;
            const float m_new = fmaxf(m, mt);
            if (m_new > m + RESCALE_THRESHOLD) {
                alpha = (m == -INFINITY) ? 0.f : ex2(m - m_new);
                m = m_new;
            }
            const float nm = (m == -INFINITY) ? 0.f : -m;  // fully masked so far: every v is -inf
            float ls[2] = {0.f, 0.f};
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float e0 = ex2(fmaf(__uint_as_float(v[i]), p.scale_log2, nm));
                const float e1 = ex2(fmaf(__uint_as_float(v[i + 1]), p.scale_log2, nm));
                ls[(i >> 1) & 1] += e0 + e1;
                pk[i >> 1] = pack_bf2(e0, e1);
            }
            l = l * alpha + (ls[0] + ls[1]);
            long long a2 = prof_clock<4>();
            c_ex += a2 - a1;
            if (t >= 2) mbar_wait(&b_odone[t & 1], ((t >> 1) - 1) & 1);  // P buffer free
            c_o += prof_clock<4>() - a2;
            long long a3 = prof_clock<4>();
            if (t >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
                mbar_wait(&b_odone[(t - 1) & 1], ((t - 1) >> 1) & 1);  // O holds PV(0..t-1)
                tc::fence_after();
#pragma unroll 1
                for (int c = 0; c < 8; ++c) {
                    uint32_t o[32];
                    const uint32_t a = lane_base + COL_O + (c >> 2) * 128 + (c & 3) * 32;
                    tc2::ld_32x32b_x32(a, o);
                    tc::wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tc2::st_32x32b_x32(a, o);
                }
                tc::wait_st();
            }
            long long a4 = prof_clock<4>();
            c_r += a4 - a3;
            const uint32_t pt = p_base + (t & 1) * PTILE2;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                sts128(pt + swz128(r, 4 * kh + j), make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
            fence_proxy_async_smem();
            tc::fence_before();
            mbar_arrive(&b_pfull[t & 1]);  // local; the peer's relay forwards it to the leader
            c_e += prof_clock<4>() - a4;
        }
        if (kProf && p.dbg && blockIdx.x < 2 && lane == 0 && w == 0)
            printf("2sm softmax cta%d: wait_s %lld ld %lld mask %lld xchg+exp %lld wait_o %lld rescale %lld pstore %lld "
                   "total %lld\n", (int)rank, c_s, c_ld, c_mx, c_ex, c_o, c_r, c_e, prof_clock<4>() - c0);
        // epilogue: O / l -> bf16, lse (l summed over the two key halves)
        sl[kh][r] = l;
        mbar_wait(&b_odone[(T - 1) & 1], ((T - 1) >> 1) & 1);
        tc::fence_after();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        l += sl[kh ^ 1][r];
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
            const int h = c >> 2, q = c & 3;
            uint32_t o[32];
            tc2::ld_32x32b_x32(lane_base + COL_O + h * 128 + q * 32, o);
            tc::wait_ld();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2)
                pk[i >> 1] = pack_bf2(__uint_as_float(o[i]) * inv_l, __uint_as_float(o[i + 1]) * inv_l);
            if (row_ok) {
                uint4 *dst = reinterpret_cast<uint4 *>(p.out + grow * DV + 256 * h + 128 * kh + 32 * q);
                dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                dst[2] = make_uint4(pk[8], pk[9], pk[10], pk[11]);
                dst[3] = make_uint4(pk[12], pk[13], pk[14], pk[15]);
            }
        }
        if (row_ok && kh == 0 && p.lse) p.lse[grow] = (m + log2f(l)) * 0.69314718055994531f;
    }
    tc::fence_before();
    cl::cluster_sync();
    tc::fence_after();
    if (warp == W_MMA2) tc2::tmem_dealloc(tbase, 512);
}

}  // namespace p2

// ============================================================================
// v3: the CTA pair with V taken from the K tiles. Q pieces [0, QT3) in TMEM, 4 K stages,
// 3 S buffers (QK runs two tiles ahead of PV), and per tile only the OTHER CTA's keys'
// V pieces are loaded, straight into the K stage once QK(t) is done with it.
namespace p3 {
using namespace p2;
#undef IRM_MLA_QT_V3
#ifndef IRM_MLA_V3_QT
#define IRM_MLA_V3_QT 5
#endif
#ifndef IRM_MLA_V3_NS
#define IRM_MLA_V3_NS 3
#endif
constexpr int QT = IRM_MLA_V3_QT;
#ifndef IRM_MLA_V3_KST
#define IRM_MLA_V3_KST 4
#endif
#ifndef IRM_MLA_V3_NP
#define IRM_MLA_V3_NP 2
#endif
constexpr int KST = IRM_MLA_V3_KST, NS = IRM_MLA_V3_NS;  // S buffers: QK runs NS - 1 tiles ahead
constexpr int NP = IRM_MLA_V3_NP;  // P buffers: 1 frees smem for a fifth K stage
// P as the TMEM A operand of PV (TS mode), written over its own S buffer: the tensor core then
// reads only V from shared memory in PV. The 2-SM TS layout wants each row's 64 keys in both
// lane halves, so the two softmax warps holding a row's key halves swap them through shared
// memory (8 KB written + read per CTA per tile, instead of 8 KB of P written and 16 KB read by
// the MMAs)
// Default OFF: with P in TMEM the output differs from launch to launch in ~1-2K of 67M
// elements (up to 2e-3 abs) at the 128K/8K shape and launches occasionally fault when
// repeated back to back (tools/k5_stress.py); P through shared memory is bit-reproducible.
#ifndef IRM_MLA_V3_PT
#define IRM_MLA_V3_PT 0
#endif
constexpr bool PT = IRM_MLA_V3_PT != 0;
constexpr int XBUF = 2 * 2 * 64 * 64;  // P-half swap: [t & 1][key half][4 x 16 B][64 rows]
constexpr int S_Q = 0, S_K = (NPIECE - QT) * QPIECE, S_P = S_K + KST * KTILE;
constexpr int SMEM3 = S_P + (PT ? XBUF : NP * PTILE2);  // 192 KB (4 K stages, 2 P buffers)
constexpr uint32_t COL_S = 0, COL_O = 32 * NS, COL_Q = COL_O + 256;
static_assert(COL_Q + 32 * QT <= 512, "TMEM: S x 3, O, Q pieces");
constexpr uint32_t FV_TX = 4 * KPIECE;  // foreign V bytes per CTA per tile
// CTA pairs per shared key-tile order (the walk starts at a hashed tile; any order is exact
// under the online softmax)
#ifndef IRM_MLA_TGRP
#define IRM_MLA_TGRP 16
#endif

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS2, 1)
mla_reattach_2sm_v3_kernel(Params p, const __grid_constant__ CUtensorMap tmap_pool,
                           const __grid_constant__ CUtensorMap tmap_tile, const __grid_constant__ CUtensorMap tmap_k8,
                           const __grid_constant__ CUtensorMap tmap_k2) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t b_q, b_qpair, b_kfull[KST], b_krope[KST], b_qkdone[KST], b_vfull[KST],
        b_kempty[KST], b_sfull[NS], b_pfull[2], b_odone[2];
    __shared__ float sx[2][2][64];  // row-max exchange between the two key halves
    __shared__ float sl[2][64];     // final row-sum exchange
    __shared__ uint32_t tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cl::cta_rank();
    const int64_t prow0 = (int64_t)(blockIdx.x >> 1) * 128;  // first row of the pair
    const int64_t row0 = prow0 + 64 * rank;                 // first row of this CTA
    const int64_t last_row = min(p.n_rows, prow0 + 128) - 1;
    const int64_t max_pos = p.q_pos0 + last_row / p.heads;
    const int n_keys = (int)min((int64_t)p.n_kv, max_pos + 1);
    const int T = (n_keys + PBN - 1) / PBN;
    const int toff = (int)(((uint32_t)((blockIdx.x >> 1) / IRM_MLA_TGRP) * 2654435761u) % (uint32_t)T);

    if (threadIdx.x == 0) {
        mbar_init(&b_q, QT > 0 ? 256 : 128);  // smem Q (producers) + TMEM Q (softmax warps)
        mbar_init(&b_qpair, 1);
        for (int s = 0; s < KST; ++s) {
            // leader: its TMA expect_tx (both CTAs' c_KV bytes land here) + its rope group + the
            // peer's rope readiness (relayed); peer: b_krope collects its rope group
            mbar_init(&b_kfull[s], 2 + GROUP);
            mbar_init(&b_krope[s], GROUP);
            mbar_init(&b_kempty[s], 1);
        }
        for (int s = 0; s < KST; ++s) {
            mbar_init(&b_qkdone[s], 1);  // QK(t) done (multicast commit): the foreign V may overwrite
            mbar_init(&b_vfull[s], 1);   // leader: its expect_tx; the peer's bytes complete here too
        }
        for (int s = 0; s < NS; ++s) mbar_init(&b_sfull[s], 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&b_pfull[s], rank == 0 ? 128 + 1 : 128);  // local softmax threads (+ the peer's relay)
            mbar_init(&b_odone[s], 1);
        }
        fence_mbar_init();
    }
    if (warp == W_MMA2) tc2::tmem_alloc(&tmem_base, 512);
    tc::fence_before();
    cl::cluster_sync();
    tc::fence_after();
    const uint32_t tbase = tmem_base;

    if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ Q (once) + rope of this CTA's 32 keys
        const int ptid = threadIdx.x - 128;
        const uint32_t qbase = smem_u32(smem + S_Q);
        constexpr int QC = (NPIECE - QT) * 8;  // 16-byte chunks per row kept in smem
        for (int i = ptid; i < 64 * QC; i += 128) {
            const int r = i / QC, c = i % QC + QT * 8;
            const int64_t grow = row0 + r;
            const bool ok = grow < p.n_rows;
            cp_async16(qbase + ((c >> 3) - QT) * QPIECE + swz128(r, c & 7), p.q + (ok ? grow : 0) * DQK + c * 8,
                       ok ? 16u : 0u);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        fence_proxy_async_smem();
        mbar_arrive(&b_q);
        const int g = ptid / GROUP, gtid = ptid % GROUP;  // group g: tiles t = g (mod 2)
        for (int t = g; t < T; t += 2) {
            const int kt = (t + toff) % T, st = t % KST;
            RopeRegs rr;
            rope_fetch(p, 2 * kt + (int)rank, gtid, rr);  // keys kt*64 + 32*rank + [0, 32)
            if (t >= KST) mbar_wait(&b_kempty[st], ((t / KST) - 1) & 1);
            store_rope(p, smem + S_K + st * KTILE, gtid, rr);
            mbar_arrive(rank == 0 ? &b_kfull[st] : &b_krope[st]);
        }
    } else if (warp == W_KTMA) {
        // ------------------------------------------------ c_KV of this CTA's 32 keys (QK operand)
        long long c_e = 0, c0 = prof_clock<1>();
        int row_next = key_row(p, (toff % T) * PBN + 32 * (int)rank + lane);  // rows read one tile ahead
        for (int t = 0; t < T; ++t) {
            const int st = t % KST;
            const Rows32 rr = rows32_resolve(row_next, lane);
            if (t + 1 < T) row_next = key_row(p, ((t + 1 + toff) % T) * PBN + 32 * (int)rank + lane);
            long long a0 = prof_clock<1>();
            if (t >= KST) mbar_wait(&b_kempty[st], ((t / KST) - 1) & 1);
            c_e += prof_clock<1>() - a0;
            // both CTAs' c_KV bytes complete on the leader's b_kfull (peer: .cta_group::2 TMA)
            if (rank == 0 && lane == 0) mbar_arrive_expect_tx(&b_kfull[st], 2 * CKV_TX);
            __syncwarp();
            const uint32_t dst = smem_u32(smem + S_K + st * KTILE);
            const uint32_t kbar = cl::map_to(smem_u32(&b_kfull[st]), 0);
            if (rr.contig) {  // one op for the 8 c_KV pieces of 32 consecutive rows
                if (lane == 0) tma_load_3d_pair(dst, &tmap_k8, rr.row0, 0, kbar);
            } else {
                for (int pc = 0; pc < 8; ++pc)
                    tma_rows32_pair(rr, &tmap_pool, &tmap_tile, dst + pc * KPIECE, pc, lane, kbar);
            }
        }
        if (kProf && p.dbg && blockIdx.x < 2 && lane == 0)
            printf("2sm-v3 ktma cta%d: wait_empty %lld total %lld\n", (int)rank, c_e, prof_clock<1>() - c0);
    } else if (warp == W_VTMA) {
        // ------------------------------------------------ foreign V: the other CTA's 32 keys x my dims
        // PV over key half a reads, at K-stage slots 4h + 2a (+1), the half's own CTA's K pieces and,
        // in the other CTA, the same keys' pieces of ITS latent dims. So once QK(t) no longer needs
        // them, CTA r overwrites its slots 4h + 2(1 - r) (+1) with pieces 4h + 2r (+1) of the other
        // CTA's keys: V is never loaded for the CTA's own keys (16 KB per tile instead of 32 KB)
        int row_next = key_row(p, (toff % T) * PBN + 32 * (1 - (int)rank) + lane);
        for (int t = 0; t < T; ++t) {
            const int st = t % KST;
            const Rows32 rr = rows32_resolve(row_next, lane);
            if (t + 1 < T) row_next = key_row(p, ((t + 1 + toff) % T) * PBN + 32 * (1 - (int)rank) + lane);
            mbar_wait(&b_qkdone[st], (t / KST) & 1);
            if (rank == 0 && lane == 0) mbar_arrive_expect_tx(&b_vfull[st], 2 * FV_TX);
            __syncwarp();
            const uint32_t dst = smem_u32(smem + S_K + st * KTILE);
            const uint32_t vbar = cl::map_to(smem_u32(&b_vfull[st]), 0);
            const int src0 = 2 * (int)rank, dst0 = 2 * (1 - (int)rank);
            if (rr.contig) {  // two ops: pieces src0 + {0, 1} and 4 + src0 + {0, 1}
                if (lane == 0) {
                    tma_load_3d_pair(dst + dst0 * KPIECE, &tmap_k2, rr.row0, src0, vbar);
                    tma_load_3d_pair(dst + (4 + dst0) * KPIECE, &tmap_k2, rr.row0, 4 + src0, vbar);
                }
            } else {
                for (int j = 0; j < 4; ++j) {
                    const int off = (j >> 1) * 4 + (j & 1);
                    tma_rows32_pair(rr, &tmap_pool, &tmap_tile, dst + (dst0 + off) * KPIECE, src0 + off, lane, vbar);
                }
            }
        }
    } else if (warp == W_MMA2) {
        if (rank != 0) {
            // ------------------------------------------------ peer: relay local data readiness to the leader
            const uint32_t q_l = cl::map_to(smem_u32(&b_qpair), 0);
            mbar_wait(&b_q, 0);
            if (lane == 0) cl::remote_arrive(q_l);
            auto relay_k = [&](int t) {  // the peer's rotated k_r is in smem
                mbar_wait(&b_krope[t % KST], (t / KST) & 1);
                if (lane == 0) cl::remote_arrive(cl::map_to(smem_u32(&b_kfull[t % KST]), 0));
            };
            relay_k(0);
            // forwarded in the leader's consumption order: K(t+1) for QK, then P(t) and V(t) for PV.
            // A cluster-scope release costs ~1.5K cycles; doing it here keeps it off the softmax path.
            for (int t = 0; t < T; ++t) {
                if (t + 1 < T) relay_k(t + 1);
                mbar_wait(&b_pfull[t & 1], (t >> 1) & 1);
                if (lane == 0) cl::remote_arrive(cl::map_to(smem_u32(&b_pfull[t & 1]), 0));
            }
        } else {
            // ------------------------------------------------ leader: MMA issue for the pair
            const uint32_t idesc_qk = tc::idesc_bf16(128, PBN, false, false);
            const uint32_t idesc_pv = tc::idesc_bf16(128, 256, false, true);
            const uint64_t q_desc = tc::smem_desc_sw128(smem_u32(smem + S_Q), 16, 1024);
            const uint64_t k_desc = tc::smem_desc_sw128(smem_u32(smem + S_K), 16, 1024);
            const uint64_t kv_desc = tc::smem_desc_sw128(smem_u32(smem + S_K), KPIECE, 1024);  // MN-major view
            const uint32_t kv_lo = (uint32_t)kv_desc, kv_hi = (uint32_t)(kv_desc >> 32);
            const uint64_t p_desc = tc::smem_desc_sw128(smem_u32(smem + S_P), 16, 1024);
            const uint32_t q_lo = (uint32_t)q_desc, q_hi = (uint32_t)(q_desc >> 32);
            const uint32_t k_lo = (uint32_t)k_desc, k_hi = (uint32_t)(k_desc >> 32);
            const uint32_t p_lo = (uint32_t)p_desc, p_hi = (uint32_t)(p_desc >> 32);
            mbar_wait(&b_q, 0);
            mbar_wait(&b_qpair, 0);
            long long c_k = 0, c_kp = 0, c_p = 0, c_v = 0, c_vl = 0, c0 = prof_clock<2>();
            auto issue_qk = [&](int t) {
                const int st = t % KST;
                long long a0 = prof_clock<2>();
                mbar_wait(&b_kfull[st], (t / KST) & 1);  // both CTAs' K tiles (bytes + rope)
                long long a1 = prof_clock<2>();
                c_k += a1 - a0;
                c_kp += prof_clock<2>() - a1;
                tc::fence_after();
                const uint32_t kd = k_lo + ((st * KTILE) >> 4);
                const uint32_t ds = tbase + COL_S + (t % NS) * 32;
                if (tc::elect_one()) {
                    // one 64-dim piece per iteration, descriptors advanced incrementally: a fully
                    // unrolled loop hoists all 72 descriptors into uniform registers and spills
                    uint32_t qa = q_lo, kb = kd, qt = tbase + COL_Q;
#pragma unroll 1
                    for (int pc = 0; pc < QT; ++pc) {  // A = Q from TMEM
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc2::mma_bf16_ts_w(ds, qt + 8 * k, kb + 2 * k, k_hi, idesc_qk, (pc | k) != 0);
                        qt += 32;
                        kb += KPIECE >> 4;
                    }
#pragma unroll 1
                    for (int pc = QT; pc < NPIECE; ++pc) {  // A = Q from shared memory
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc2::mma_bf16_ss_w(ds, qa + 2 * k, q_hi, kb + 2 * k, k_hi, idesc_qk, (pc | k) != 0);
                        qa += QPIECE >> 4;
                        kb += KPIECE >> 4;
                    }
                    tc2::commit_both(&b_sfull[t % NS]);
                    tc2::commit_both(&b_qkdone[st]);
                }
                __syncwarp();
            };
            for (int t = 0; t < NS - 1 && t < T; ++t) issue_qk(t);
            for (int t = 0; t < T; ++t) {
#ifdef IRM_MLA_PT_WAIT_PV
                // experiment: with P in TMEM, QK(t + NS - 1) overwrites the columns PV(t - 1) reads P from;
                // wait for PV(t - 1) to complete before issuing it
                if (PT && t >= 1 && t + NS - 1 < T) {
                    mbar_wait(&b_odone[(t - 1) & 1], ((t - 1) >> 1) & 1);
                    tc::fence_after();
                }
#endif
                if (t + NS - 1 < T) issue_qk(t + NS - 1);  // reuses the S buffer softmax(t-1) has read
                const int st = t % KST;
                long long a0 = prof_clock<2>();
                mbar_wait(&b_pfull[t & 1], (t >> 1) & 1);
                long long a1 = prof_clock<2>();
                c_p += a1 - a0;
                mbar_wait(&b_vfull[st], (t / KST) & 1);  // both CTAs' foreign V in place
                c_v += prof_clock<2>() - a1;
                tc::fence_after();
                const uint32_t pd = p_lo + ((((t & 1) % NP) * PTILE2) >> 4);
                const uint32_t pt_col = tbase + COL_S + (t % NS) * 32;  // PT: P(t) over S(t)
                const uint32_t kd = kv_lo + ((st * KTILE) >> 4);
                if (tc::elect_one()) {
#pragma unroll
                    for (int a = 0; a < 2; ++a) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
#pragma unroll
                            for (int k = 0; k < 2; ++k) {
                                const uint32_t vb = kd + (((4 * h + 2 * a) * KPIECE + k * 2048) >> 4);
                                const uint32_t acc = (t > 0 || a > 0 || k > 0) ? 1u : 0u;
                                if constexpr (PT)  // keys 16 (2a + k) .. + 15: 8 bf16-pair columns
                                    tc2::mma_bf16_ts_w(tbase + COL_O + h * 128, pt_col + 8 * (2 * a + k), vb, kv_hi,
                                                       idesc_pv, acc);
                                else
                                    tc2::mma_bf16_ss_w(tbase + COL_O + h * 128, pd + (((2 * a + k) * 32) >> 4), p_hi,
                                                       vb, kv_hi, idesc_pv, acc);
                            }
                        }
                    }
                    tc2::commit_both(&b_kempty[st]);
                    tc2::commit_both(&b_odone[t & 1]);
                }
                __syncwarp();
            }
            if (kProf && p.dbg && blockIdx.x == 0 && lane == 0)
                printf("2sm-v3 mma: wait_k %lld wait_kpair %lld wait_p %lld wait_v %lld (local %lld) total %lld T=%d\n", c_k, c_kp,
                       c_p, c_v, c_vl, prof_clock<2>() - c0, T);
        }
    } else {
        // ------------------------------------------------ softmax / correction (warps 0-3)
        const int w = warp;
        const int r = 32 * (w & 1) + lane;  // row of this CTA
        const int kh = w >> 1;              // key half (S) / latent-dim half (O)
        const int64_t grow = row0 + r;
        const bool row_ok = grow < p.n_rows;
        const int64_t qpos = p.q_pos0 + (row_ok ? grow / p.heads : 0);
        const uint32_t lane_base = tbase + ((uint32_t)(32 * w) << 16);
        const uint32_t p_base = smem_u32(smem + S_P);
        const uint32_t pfull_leader0 = cl::map_to(smem_u32(&b_pfull[0]), 0);
        const uint32_t pfull_leader1 = cl::map_to(smem_u32(&b_pfull[1]), 0);
        if constexpr (QT > 0) {
            // this thread's row of Q, pieces [0, QT), into its TMEM lane (rows are duplicated
            // across the lane halves: warps w and w + 2 hold the same rows, as the 2-SM TS
            // A operand expects)
            const uint4 *src = reinterpret_cast<const uint4 *>(p.q + (row_ok ? grow : 0) * DQK);
#pragma unroll 1
            for (int pc = 0; pc < QT; ++pc) {
                uint32_t qv[32];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint4 x = row_ok ? __ldg(src + 8 * pc + j) : make_uint4(0, 0, 0, 0);
                    qv[4 * j] = x.x;
                    qv[4 * j + 1] = x.y;
                    qv[4 * j + 2] = x.z;
                    qv[4 * j + 3] = x.w;
                }
                tc2::st_32x32b_x32(lane_base + COL_Q + 32 * pc, qv);
            }
            tc::wait_st();
            tc::fence_before();
            mbar_arrive(&b_q);
        }
        float m = -INFINITY, l = 0.f;
        long long c_s = 0, c_o = 0, c_x = 0, c_r = 0, c_e = 0, c_ld = 0, c_mx = 0, c_ex = 0, c0 = prof_clock<4>();
        for (int t = 0; t < T; ++t) {
            long long a0 = prof_clock<4>();
            mbar_wait(&b_sfull[t % NS], (t / NS) & 1);
            c_s += prof_clock<4>() - a0;
            tc::fence_after();
            uint32_t v[32];
            long long b0 = prof_clock<4>();
            tc2::ld_32x32b_x32(lane_base + COL_S + (t % NS) * 32, v);
            tc::wait_ld();
            long long b1 = prof_clock<4>();
            c_ld += b1 - b0;
            const int64_t kbase = (int64_t)((t + toff) % T) * PBN + 32 * kh;
            if (!__all_sync(0xffffffffu, row_ok && kbase + 31 <= qpos && kbase + 31 < p.n_kv)) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int64_t key = kbase + i;
                    if (!(row_ok && key <= qpos && key < p.n_kv)) v[i] = NEG_INF_BITS;
                }
            }
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int i = 0; i < 32; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(v[i]));
            float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
            sx[t & 1][kh][r] = mt;  // exchange with the thread holding the other key half
            long long a1 = prof_clock<4>();
            c_mx += a1 - b1;
            asm volatile("bar.sync 1, 128;" ::: "memory");
            c_x += prof_clock<4>() - a1;
            mt = fmaxf(mt, sx[t & 1][kh ^ 1][r]);
            float alpha = 1.f;
            const float m_new = fmaxf(m, mt);
            if (m_new > m + RESCALE_THRESHOLD) {
                alpha = (m == -INFINITY) ? 0.f : ex2(m - m_new);
                m = m_new;
            }
            const float nm = (m == -INFINITY) ? 0.f : -m;  // fully masked so far: every v is -inf
            float ls[2] = {0.f, 0.f};
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float x0 = fmaf(__uint_as_float(v[i]), p.scale_log2, nm);
                const float x1 = fmaf(__uint_as_float(v[i + 1]), p.scale_log2, nm);
                const float e0 = ex2(x0);
                const float e1 = ex2(x1);
                ls[(i >> 1) & 1] += e0 + e1;
                pk[i >> 1] = pack_bf2(e0, e1);
            }
            l = l * alpha + (ls[0] + ls[1]);
            long long a2 = prof_clock<4>();
            c_ex += a2 - a1;
            // P buffer free (PT: S(t)'s buffer, read by PV(t - NS) before QK(t) overwrote it)
            if (!PT && NP == 2 && t >= 2) mbar_wait(&b_odone[t & 1], ((t >> 1) - 1) & 1);
            if (!PT && NP == 1 && t >= 1) mbar_wait(&b_odone[(t - 1) & 1], ((t - 1) >> 1) & 1);  // PV(t-1) read P
            c_o += prof_clock<4>() - a2;
            long long a3 = prof_clock<4>();
            if (t >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
                mbar_wait(&b_odone[(t - 1) & 1], ((t - 1) >> 1) & 1);  // O holds PV(0..t-1)
                tc::fence_after();
#pragma unroll 1
                for (int c = 0; c < 8; ++c) {
                    uint32_t o[32];
                    const uint32_t a = lane_base + COL_O + (c >> 2) * 128 + (c & 3) * 32;
                    tc2::ld_32x32b_x32(a, o);
                    tc::wait_ld();
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                    tc2::st_32x32b_x32(a, o);
                }
                tc::wait_st();
            }
            long long a4 = prof_clock<4>();
            c_r += a4 - a3;
            if constexpr (PT) {
                // swap key halves with warp w ^ 2 (same rows), then the row's 64 keys as 32 bf16-pair
                // columns over S(t) in this lane
                const uint32_t xb = p_base + (t & 1) * (XBUF / 2);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    sts128(xb + ((kh * 4 + j) * 64 + r) * 16,
                           make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
                asm volatile("bar.sync %0, 64;" ::"r"(2 + (w & 1)) : "memory");
                uint32_t px[16];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(px[4 * j]), "=r"(px[4 * j + 1]), "=r"(px[4 * j + 2]), "=r"(px[4 * j + 3])
                                 : "r"(xb + (((kh ^ 1) * 4 + j) * 64 + r) * 16));
                const uint32_t pcol = lane_base + COL_S + (t % NS) * 32;
                tc2::st_32x32b_x16(pcol + 16 * kh, pk);
                tc2::st_32x32b_x16(pcol + 16 * (kh ^ 1), px);
                tc::wait_st();
            } else {
                const uint32_t pt = p_base + ((t & 1) % NP) * PTILE2;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    sts128(pt + swz128(r, 4 * kh + j),
                           make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]));
                fence_proxy_async_smem();
            }
            tc::fence_before();
            mbar_arrive(&b_pfull[t & 1]);  // local; the peer's relay forwards it to the leader
            c_e += prof_clock<4>() - a4;
        }
        if (kProf && p.dbg && blockIdx.x < 2 && lane == 0 && w == 0)
            printf("2sm-v3 softmax cta%d: wait_s %lld ld %lld mask %lld xchg+exp %lld wait_o %lld rescale %lld pstore %lld "
                   "total %lld\n", (int)rank, c_s, c_ld, c_mx, c_ex, c_o, c_r, c_e, prof_clock<4>() - c0);
        // epilogue: O / l -> bf16, lse (l summed over the two key halves)
        sl[kh][r] = l;
        mbar_wait(&b_odone[(T - 1) & 1], ((T - 1) >> 1) & 1);
        tc::fence_after();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        l += sl[kh ^ 1][r];
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
            const int h = c >> 2, q = c & 3;
            uint32_t o[32];
            tc2::ld_32x32b_x32(lane_base + COL_O + h * 128 + q * 32, o);
            tc::wait_ld();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2)
                pk[i >> 1] = pack_bf2(__uint_as_float(o[i]) * inv_l, __uint_as_float(o[i + 1]) * inv_l);
            if (row_ok) {
                uint4 *dst = reinterpret_cast<uint4 *>(p.out + grow * DV + 256 * h + 128 * kh + 32 * q);
                dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                dst[2] = make_uint4(pk[8], pk[9], pk[10], pk[11]);
                dst[3] = make_uint4(pk[12], pk[13], pk[14], pk[15]);
            }
        }
        if (row_ok && kh == 0 && p.lse) p.lse[grow] = (m + log2f(l)) * 0.69314718055994531f;
    }
    tc::fence_before();
    cl::cluster_sync();
    tc::fence_after();
    if (warp == W_MMA2) tc2::tmem_dealloc(tbase, 512);
}

}  // namespace p3


__global__ void cossin_kernel(const int64_t *__restrict__ delta, int64_t n_chunks,
                              const double *__restrict__ inv_freq, float2 *__restrict__ cs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_chunks * 32) return;
    double s, c;
    sincos_cr((double)delta[i / 32] * inv_freq[i % 32], &s, &c);  // fp64 angle (|delta| up to 2^20)
    cs[i] = make_float2((float)c, (float)s);
}

}  // namespace mla
}  // namespace irm

using namespace irm;

extern "C" int irm_chunk_cossin(const int64_t *delta, int64_t n_chunks, const double *inv_freq, void *cs,
                                irm_stream_t stream) {
    IRM_REQUIRE(n_chunks >= 0, "n_chunks must be >= 0");
    if (n_chunks == 0) return IRM_OK;
    IRM_REQUIRE(delta && inv_freq && cs, "null pointer");
    mla::cossin_kernel<<<(unsigned)((n_chunks * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        delta, n_chunks, inv_freq, (float2 *)cs);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    return fn;
}

extern "C" int irm_mla_reattach_prefill(const void *q, int64_t n_q, int32_t heads, int64_t q_pos0,
                                        const void *pool, int64_t pool_rows, const int32_t *kv_rows,
                                        int32_t n_kv, const int32_t *kv_chunk, const void *chunk_cs,
                                        int32_t layout, float scale, void *out, float *lse, irm_stream_t stream) {
    IRM_REQUIRE(n_q >= 0 && heads >= 1 && n_kv >= 1 && q_pos0 >= 0, "bad sizes");
    IRM_REQUIRE(q_pos0 + n_q <= (int64_t)n_kv, "queries must be positions < n_kv (q_pos0 + n_q <= n_kv)");
    IRM_REQUIRE(layout == IRM_LAYOUT_HALF_SPLIT || layout == IRM_LAYOUT_INTERLEAVED, "bad layout");
    IRM_REQUIRE(!kv_chunk || chunk_cs, "kv_chunk requires chunk_cs");
    IRM_REQUIRE(pool_rows >= 1 && pool_rows < ((int64_t)1 << 31), "bad pool_rows");
    IRM_REQUIRE(kv_rows || pool_rows >= n_kv, "pool_rows < n_kv with identity kv_rows");
    if (n_q == 0) return IRM_OK;
    IRM_REQUIRE(q && pool && out, "null pointer");
    IRM_REQUIRE((((uintptr_t)q | (uintptr_t)pool | (uintptr_t)out) & 15) == 0, "16-byte alignment required");
    IRM_REQUIRE(!chunk_cs || ((uintptr_t)chunk_cs & 15) == 0, "chunk_cs must be 16-byte aligned");
    // pool as a 2-D tensor [pool_rows, 576] bf16 for TMA gather4: box = 64 columns x 1 row, SW128
    auto encode = get_encode_fn();
    if (!encode) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return IRM_ECUDA;
    }
    CUtensorMap tmap, tmap_tile;
    const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;  // none / 64 / 128 B: no difference
    const cuuint64_t strides[1] = {(cuuint64_t)mla::DQK * 2};
    const cuuint32_t estr[2] = {1, 1};
    for (int which = 0; which < 2; ++which) {
        // gather4 map: 64 columns x 1 row over the whole pool; tile map: 64 x BN rows over
        // the keys' row range (identity map: n_kv rows, so rows past the end are zero-filled)
        const cuuint64_t rows = which == 0 ? (cuuint64_t)pool_rows : (cuuint64_t)(kv_rows ? pool_rows : n_kv);
        const cuuint64_t dims[2] = {(cuuint64_t)mla::DQK, rows};
        const cuuint32_t box[2] = {64, which == 0 ? 1u : (cuuint32_t)mla::BN};
        CUresult cr = encode(which == 0 ? &tmap : &tmap_tile, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                             const_cast<void *>(pool), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, promo,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled failed (%d)", (int)cr);
            return IRM_ECUDA;
        }
    }
    // multi-piece maps over the same rows as tmap_tile: [piece][row][64 cols], piece stride 128 B
    //   k8: 8 pieces (the c_KV part of a row), box {64, 32, 8}
    //   v4: pieces p + 4 g for p in [0, 4), g in [0, 2), box {64, 32, 2, 2}
    CUtensorMap tmap_k8, tmap_v4, tmap_k2;
    {
        const cuuint64_t rows = (cuuint64_t)(kv_rows ? pool_rows : n_kv);
        const cuuint64_t dk[3] = {64, rows, 8};
        const cuuint64_t sk[2] = {(cuuint64_t)mla::DQK * 2, 128};
        const cuuint32_t bk[3] = {64, (cuuint32_t)mla::BN, 8};
        const cuuint32_t ek[3] = {1, 1, 1};
        CUresult cr = encode(&tmap_k8, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(pool), dk, sk, bk, ek,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const cuuint64_t dv[4] = {64, rows, 4, 2};
        const cuuint64_t sv[3] = {(cuuint64_t)mla::DQK * 2, 128, 512};
        const cuuint32_t bv[4] = {64, (cuuint32_t)mla::BN, 2, 2};
        const cuuint32_t ev[4] = {1, 1, 1, 1};
        if (cr == CUDA_SUCCESS)
            cr = encode(&tmap_v4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(pool), dv, sv, bv, ev,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const cuuint32_t b2[3] = {64, (cuuint32_t)mla::BN, 2};  // two adjacent pieces (v3 foreign V)
        if (cr == CUDA_SUCCESS)
            cr = encode(&tmap_k2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(pool), dk, sk, b2, ek,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled (multi-piece) failed (%d)", (int)cr);
            return IRM_ECUDA;
        }
    }
    mla::Params p{};
    p.q = (const __nv_bfloat16 *)q;
    p.pool = (const __nv_bfloat16 *)pool;
    p.kv_rows = kv_rows;
    p.kv_chunk = kv_chunk;
    p.chunk_cs = (const float2 *)chunk_cs;
    p.out = (__nv_bfloat16 *)out;
    p.lse = lse;
    p.n_rows = n_q * heads;
    p.heads = heads;
    p.n_kv = n_kv;
    p.layout = layout;
    p.q_pos0 = q_pos0;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.dbg = getenv("IRM_MLA_DEBUG") != nullptr;
    // default: the CTA pair with V from the K tiles (v3); IRM_MLA_V2 = the pair with a separate
    // V ring, IRM_MLA_1SM = the single-CTA kernel (both kept for comparison and tests)
    if (getenv("IRM_MLA_1SM") == nullptr && getenv("IRM_MLA_V2") == nullptr) {
        const int smem = mla::p3::SMEM3 + 1024;
        IRM_CUDA_CHECK(cudaFuncSetAttribute(mla::p3::mla_reattach_2sm_v3_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int64_t grid = 2 * ((p.n_rows + 127) / 128);
        mla::p3::mla_reattach_2sm_v3_kernel<<<(unsigned)grid, mla::p2::THREADS2, smem, (cudaStream_t)stream>>>(
            p, tmap, tmap_tile, tmap_k8, tmap_k2);
        IRM_LAUNCH_CHECK();
        return IRM_OK;
    }
    if (getenv("IRM_MLA_1SM") == nullptr) {  // CTA-pair (cta_group::2) kernel: 128 rows per cluster
        const int smem = mla::p2::SMEM2 + 1024;
        IRM_CUDA_CHECK(cudaFuncSetAttribute(mla::p2::mla_reattach_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        const int64_t grid = 2 * ((p.n_rows + 127) / 128);
        mla::p2::mla_reattach_2sm_kernel<<<(unsigned)grid, mla::p2::THREADS2, smem, (cudaStream_t)stream>>>(
            p, tmap, tmap_tile, tmap_k8, tmap_v4);
        IRM_LAUNCH_CHECK();
        return IRM_OK;
    }
    const int smem = mla::SMEM_BYTES + 1024;
    IRM_CUDA_CHECK(cudaFuncSetAttribute(mla::mla_reattach_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t grid = (p.n_rows + mla::BM - 1) / mla::BM;
    mla::mla_reattach_kernel<<<(unsigned)grid, mla::THREADS, smem, (cudaStream_t)stream>>>(p, tmap, tmap_tile);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}
