// K4 fan-out: one source read, many rotated destinations.
//
// In a reattach wave several requests hit the same stored chunk (the shared
// body of the agent_meta workload: 8 requests per wave reattach the same
// ~193 entries, each at its own delta = p_dest - p_src). KvRegistry.materialize
// (reference registry.py:146-166) is a pure function of (entry, p_dest), so the
// B200 form reads each (entry, layer) slab from HBM once per wave:
//
//   irm_group_by_source   the wave's compacted hit list -> groups of hits that
//                         share a source run (src_row, len), members listed
//                         contiguously per group (one CTA, a hash table in a
//                         caller-owned, zero-initialised workspace that the
//                         call leaves zeroed again; no host synchronisation)
//   irm_rotate_gather_fanout
//                         persistent CTAs walk (group, layer, tile, member):
//                         the members of a tile are served back to back, each
//                         by its own 1-D bulk load of the tile (TMA engine; the
//                         first from HBM, the rest hit L2 -- evict_last hint),
//                         an in-place k_r rotation by the member's R(delta)
//                         (fp32 on fp64-derived cos/sin, staged with the tile)
//                         and a bulk store (evict_first hint). Warp-specialised
//                         for bf16 / 64-wide k_r: a producer warp (iterator +
//                         loads), rotation warps (one 8-pair unit per thread), a
//                         storer warp (stores; hands stages back once read).
//
// HBM traffic per wave = unique source rows + all destination rows (x layers
// x row bytes), against 2 x all destination rows for the plain gather. The
// launch is then bound by HBM WRITE bandwidth (8.15 of its 9.2 GB are writes
// on the config-2 wave): ~4.9 TB/s of writes, where a 1:1 copy reaches 6.5
// TB/s combined (tools/k4_fan_bench.py, profiles/r02_k4_fanout.md). Two
// source-once forms measured slower: threads copying the source tile into
// per-member output stages (2.7 ms against 1.68 ms here) and the TMA engine
// copying it shared -> shared inside the CTA (2.63 ms): an SM moves 36 KB
// between its own stages more slowly than it re-reads them from L2. A third,
// round-robin source-once form (each stage serves all members of its tile,
// the pristine k_r kept aside, stages interleaved so a stage is rewritten only
// after its previous store left) ran 1.67-1.73 ms: no faster than this form,
// so L2 re-reads are not what holds the launch at ~5.4 TB/s combined.
#include <algorithm>
#include <cuda_bf16.h>
#include <stdlib.h>
#include <type_traits>
#include "common.cuh"
#include "tma.cuh"

namespace irm {

// ------------------------------------------------------------------ grouping
constexpr int GB_THREADS = 1024;

struct GroupWs {
    unsigned long long *key;  // [T] (src + 1) << 24 | len, 0 = empty
    int32_t *cnt;             // [T] members
    uint32_t *first;          // [T] 0x7FFFFFFF - smallest member index (atomicMax; 0 = unset)
    int32_t *off;             // [T] member offset of the group
    int32_t *slot;            // [n] slot of member i
    int32_t *rank;            // [n] rank of member i within its group
    int64_t tmask;
    int64_t bytes;
};

static GroupWs carve_group_ws(void *ws, int64_t n) {
    int64_t t = 2;
    while (t < 2 * std::max<int64_t>(n, 1)) t <<= 1;
    GroupWs w{};
    char *p = (char *)ws;
    int64_t o = 0;
    auto take = [&](int64_t bytes) {
        char *q = p ? p + o : nullptr;
        o = (o + bytes + 255) / 256 * 256;
        return q;
    };
    w.key = (unsigned long long *)take(t * 8);
    w.cnt = (int32_t *)take(t * 4);
    w.first = (uint32_t *)take(t * 4);
    w.off = (int32_t *)take(t * 4);
    w.slot = (int32_t *)take(n * 4);
    w.rank = (int32_t *)take(n * 4);
    w.tmask = t - 1;
    w.bytes = o;
    return w;
}

__device__ __forceinline__ unsigned long long group_key(int64_t src, int32_t len) {
    // rows below 2^39 and lengths below 2^24 pack exactly; anything else is one "bad" group that
    // the gather's bounds check flags and skips
    if (src < 0 || src >= (1LL << 39) || len < 0 || len >= (1 << 24)) return ~0ULL;
    return ((unsigned long long)(src + 1) << 24) | (unsigned long long)len;
}

__global__ void __launch_bounds__(GB_THREADS)
group_by_source_kernel(const int64_t *__restrict__ src, const int64_t *__restrict__ dst,
                       const int32_t *__restrict__ len, const int64_t *__restrict__ delta, int64_t n_cap,
                       const int64_t *__restrict__ n_dev, GroupWs w, int64_t *__restrict__ g_src,
                       int32_t *__restrict__ g_len, int32_t *__restrict__ g_first, int32_t *__restrict__ g_count,
                       int64_t *__restrict__ m_dst, int64_t *__restrict__ m_delta, int64_t *__restrict__ n_groups) {
    __shared__ int64_t sm[GB_THREADS / 32];
    const int64_t n = n_dev ? min(n_cap, *n_dev) : n_cap;
    // 1: claim a slot per distinct source run; count members; remember the first member
    for (int64_t i = threadIdx.x; i < n; i += GB_THREADS) {
        const unsigned long long key = group_key(src[i], len[i]);
        uint64_t idx = ((key * 0x9E3779B97F4A7C15ULL) >> 20) & (uint64_t)w.tmask;
        for (;;) {
            unsigned long long k = ((volatile unsigned long long *)w.key)[idx];
            if (k == 0) {
                k = atomicCAS(&w.key[idx], 0ULL, key);
                if (k == 0) k = key;  // claimed
            }
            if (k == key) break;
            idx = (idx + 1) & (uint64_t)w.tmask;
        }
        w.slot[i] = (int32_t)idx;
        w.rank[i] = atomicAdd(&w.cnt[idx], 1);
        atomicMax(&w.first[idx], 0x7FFFFFFFu - (uint32_t)i);
    }
    __syncthreads();
    // 2: groups in the order of their first member; member offsets by an exclusive scan
    int64_t gbase = 0, mbase = 0;
    for (int64_t i0 = 0; i0 < n; i0 += GB_THREADS) {
        const int64_t i = i0 + threadIdx.x;
        bool lead = false;
        int32_t c = 0, s = 0;
        if (i < n) {
            s = w.slot[i];
            lead = (int64_t)(0x7FFFFFFFu - w.first[s]) == i;
            if (lead) c = w.cnt[s];
        }
        int64_t tg, tm;
        const int64_t eg = block_exclusive_scan<GB_THREADS>(lead ? 1 : 0, &tg, sm);
        const int64_t em = block_exclusive_scan<GB_THREADS>((int64_t)c, &tm, sm);
        if (lead) {
            const int64_t g = gbase + eg, mo = mbase + em;
            g_src[g] = src[i];
            g_len[g] = len[i];
            g_first[g] = (int32_t)mo;
            g_count[g] = c;
            w.off[s] = (int32_t)mo;
        }
        gbase += tg;
        mbase += tm;
    }
    __syncthreads();
    // 3: scatter the members
    for (int64_t i = threadIdx.x; i < n; i += GB_THREADS) {
        const int64_t pos = (int64_t)w.off[w.slot[i]] + w.rank[i];
        m_dst[pos] = dst[i];
        m_delta[pos] = delta[i];
    }
    __syncthreads();
    // 4: leave the workspace zeroed for the next call
    for (int64_t i = threadIdx.x; i < n; i += GB_THREADS) {
        const int32_t s = w.slot[i];
        w.key[s] = 0;
        w.cnt[s] = 0;
        w.first[s] = 0;
        w.off[s] = 0;
        w.slot[i] = 0;
        w.rank[i] = 0;
    }
    if (threadIdx.x == 0) *n_groups = gbase;
}

// ------------------------------------------------------------------ fan-out gather
template <typename T> struct FanElem;
template <> struct FanElem<__nv_bfloat16> {
    static __device__ __forceinline__ float ld(const __nv_bfloat16 *p) { return __bfloat162float(*p); }
    static __device__ __forceinline__ void st(__nv_bfloat16 *p, float v) { *p = __float2bfloat16_rn(v); }
};
template <> struct FanElem<float> {
    static __device__ __forceinline__ float ld(const float *p) { return *p; }
    static __device__ __forceinline__ void st(float *p, float v) { *p = v; }
};

__global__ void member_cossin_kernel(const int64_t *__restrict__ delta, int64_t n_cap,
                                     const int64_t *__restrict__ n_dev, int half,
                                     const double *__restrict__ inv_freq, float2 *__restrict__ cs,
                                     unsigned long long *__restrict__ work) {
    if (work && blockIdx.x == 0 && threadIdx.x == 0) *work = 0;  // the gather's item counter, per launch
    const int64_t n = n_dev ? min(n_cap, *n_dev) : n_cap;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * half;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / half;
        const int j = (int)(i - c * half);
        double s, co;
        sincos_cr((double)delta[c] * inv_freq[j], &s, &co);  // fp64 angle
        cs[i] = make_float2((float)co, (float)s);
    }
}

struct FanArgs {
    const char *pool;
    char *out;
    int64_t pool_rows, out_rows;  // per layer (= the layer strides)
    int32_t layers, ckv, kr, row_bytes, ckv_bytes;
    const int64_t *g_src;
    const int32_t *g_len, *g_first, *g_count;
    const int64_t *m_dst;
    const float2 *cs;
    int64_t n_groups, n_items;
    const int64_t *n_groups_dev;
    int32_t layout;
    unsigned long long *status;  // sticky: 1 source run out of the pool, 2 destination run out of `out`
    unsigned long long *work;    // dynamic item counter (nullable: static round robin)
    int32_t rounds;              // > 1: the grid is rounds x the resident CTAs and each CTA retires after
                                 // its share of the items, so kernels of other streams get SMs in between
};

// Reload form: the same fan-out, but every member's tile is brought in by its own
// bulk copy (the first from HBM, the rest from L2: the CTA walks the members of a
// tile back to back) and rotated in place, so the SM threads only touch k_r.
template <int ROWS>
struct ReloadIter {
    int64_t item, g, src, dst, quota = INT64_MAX;
    int32_t l, tile, ntiles, len, m, m0, mc;
    __device__ __forceinline__ bool member_ok(const FanArgs &a, bool report) {
        dst = __ldg(a.m_dst + m0 + m);
        const bool ok = dst >= 0 && dst + len <= a.out_rows;
        if (!ok && report && tile == 0 && l == 0 && a.status) atomicOr(a.status, 2ULL);
        return ok;
    }
    __device__ __forceinline__ bool next_member(const FanArgs &a, bool report) {  // from m (inclusive)
        for (; m < mc; ++m)
            if (member_ok(a, report)) return true;
        return false;
    }
    __device__ __forceinline__ void load_item(const FanArgs &a, bool report) {
        while (item < a.n_items) {
            g = item / a.layers;
            l = (int32_t)(item - g * a.layers);
            len = __ldg(a.g_len + g);
            src = __ldg(a.g_src + g);
            m0 = __ldg(a.g_first + g);
            mc = __ldg(a.g_count + g);
            const bool ok = src >= 0 && len >= 0 && src + len <= a.pool_rows;
            if (!ok && report && l == 0 && a.status) atomicOr(a.status, 1ULL);
            ntiles = ok ? (len + ROWS - 1) / ROWS : 0;
            for (tile = 0; tile < ntiles; ++tile) {
                m = 0;
                if (next_member(a, report)) return;
            }
            advance(a);
        }
    }
    // the next (group, layer) item: first blockIdx.x, then dynamically from the shared
    // counter when the launch has one (items vary 1..16 tiles x members: a static round
    // robin left the slowest CTA ~25 % behind the mean)
    __device__ __forceinline__ void advance(const FanArgs &a) {
        if (--quota <= 0) item = a.n_items;  // this CTA's share is done: retire
        else if (a.work) item = (int64_t)atomicAdd(a.work, 1ULL) + gridDim.x;
        else item += gridDim.x;
    }
    __device__ __forceinline__ void start(const FanArgs &a, bool report) {
        item = blockIdx.x;
        if (a.rounds > 1) quota = (a.n_items + gridDim.x - 1) / gridDim.x;
        load_item(a, report);
    }
    __device__ __forceinline__ void next(const FanArgs &a, bool report) {
        ++m;
        if (next_member(a, report)) return;
        while (++tile < ntiles) {
            m = 0;
            if (next_member(a, report)) return;
        }
        advance(a);
        load_item(a, report);
    }
    __device__ __forceinline__ bool valid(const FanArgs &a) const { return item < a.n_items; }
};

// D: stores kept in flight -- a stage is refilled once the store issued D tiles ago has
// left it, so loads run STAGES - D tiles ahead (the members' reloads mostly hit L2)
template <typename T, int ROWS, int STAGES, int D, int THREADS, bool VEC>
__global__ void __launch_bounds__(THREADS)
rotate_gather_reload_kernel(FanArgs a) {
    static_assert(D >= 1 && D < STAGES, "stores in flight");
    static_assert(!VEC || ROWS * 4 <= THREADS, "one k_r unit per thread");
    if (a.n_groups_dev) a.n_items = min(a.n_groups, *a.n_groups_dev) * a.layers;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const int64_t stage_bytes = (int64_t)ROWS * a.row_bytes;
    const int half = a.kr / 2;
    const uint32_t cs_bytes = (uint32_t)(half * sizeof(float2));
    // each stage also receives its member's (cos, sin) table by the same mbarrier: the
    // table (n_members x 256 B) does not stay in the L1 that the stages leave free
    float2 *cs_stage = reinterpret_cast<float2 *>(smem + STAGES * stage_bytes);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](const ReloadIter<ROWS> &it, int stage) {
        const int32_t r0 = it.tile * ROWS;
        const int32_t rows = min(ROWS, it.len - r0);
        const uint32_t bytes = (uint32_t)(rows * a.row_bytes);
        const char *src = a.pool + ((int64_t)it.l * a.pool_rows + it.src + r0) * a.row_bytes;
        mbar_arrive_expect_tx(&full[stage], bytes + cs_bytes);
        bulk_g2s(smem + stage * stage_bytes, src, bytes, &full[stage]);
        bulk_g2s(cs_stage + stage * half, a.cs + (int64_t)(it.m0 + it.m) * half, cs_bytes, &full[stage]);
    };

    ReloadIter<ROWS> prod, cons;
    cons.start(a, threadIdx.x == 0);
    if (threadIdx.x == 0) {
        prod.start(a, false);
        for (int s = 0; s < STAGES - D + 1 && prod.valid(a); ++s) {
            issue(prod, s);
            prod.next(a, false);
        }
    }
    for (int64_t t = 0; cons.valid(a); ++t) {
        const int stage = (int)(t % STAGES);
        const int32_t r0 = cons.tile * ROWS;
        const int32_t rows = min(ROWS, cons.len - r0);
        mbar_wait(&full[stage], (uint32_t)((t / STAGES) & 1));
        uint8_t *tile = smem + stage * stage_bytes;
        const float2 *cs = cs_stage + stage * half;
        if (VEC) {
            // bf16, 64-wide k_r: a unit = 8 rotation pairs (j = 8u .. 8u+7) of one row, two
            // 16-byte words in shared memory, cos/sin as four 16-byte loads (L1-resident table)
            if (threadIdx.x < rows * 4) {
                const int r = threadIdx.x >> 2, u = threadIdx.x & 3;
                const float4 *c4 = reinterpret_cast<const float4 *>(cs + 8 * u);
                float4 e[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) e[q] = c4[q];
                uint4 *k = reinterpret_cast<uint4 *>(tile + (int64_t)r * a.row_bytes + a.ckv_bytes);
                const bool il = a.layout == IRM_LAYOUT_INTERLEAVED;
                uint4 w0 = k[il ? 2 * u : u], w1 = k[il ? 2 * u + 1 : u + 4];
                __nv_bfloat162 *p0 = reinterpret_cast<__nv_bfloat162 *>(&w0);
                __nv_bfloat162 *p1 = reinterpret_cast<__nv_bfloat162 *>(&w1);
                const float *ef = reinterpret_cast<const float *>(e);  // (cos, sin) x 8
                if (il) {  // pairs (2j, 2j+1): word w0 holds j = 8u..8u+3, w1 j = 8u+4..8u+7
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        __nv_bfloat162 &p = q < 4 ? p0[q] : p1[q - 4];
                        const float2 v = __bfloat1622float2(p);
                        const float c = ef[2 * q], sn = ef[2 * q + 1];
                        p = __floats2bfloat162_rn(rot_lo(v.x, v.y, c, sn), rot_hi(v.x, v.y, c, sn));
                    }
                } else {  // pairs (j, j + 32): w0 = lo[8u..8u+7], w1 = hi[8u..8u+7]
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 lo = __bfloat1622float2(p0[q]), hi = __bfloat1622float2(p1[q]);
                        const float c0 = ef[4 * q], s0 = ef[4 * q + 1], c1 = ef[4 * q + 2], s1 = ef[4 * q + 3];
                        p0[q] = __floats2bfloat162_rn(rot_lo(lo.x, hi.x, c0, s0), rot_lo(lo.y, hi.y, c1, s1));
                        p1[q] = __floats2bfloat162_rn(rot_hi(lo.x, hi.x, c0, s0), rot_hi(lo.y, hi.y, c1, s1));
                    }
                }
                k[il ? 2 * u : u] = w0;
                k[il ? 2 * u + 1 : u + 4] = w1;
            }
        } else {
            for (int i = threadIdx.x; i < rows * half; i += THREADS) {
                const int r = i / half, j = i - r * half;
                const int ilo = a.layout == IRM_LAYOUT_INTERLEAVED ? 2 * j : j;
                const int ihi = a.layout == IRM_LAYOUT_INTERLEAVED ? 2 * j + 1 : j + half;
                T *k = reinterpret_cast<T *>(tile + (int64_t)r * a.row_bytes + a.ckv_bytes);
                const float lo = FanElem<T>::ld(k + ilo), hi = FanElem<T>::ld(k + ihi);
                const float2 e = cs[j];
                FanElem<T>::st(k + ilo, rot_lo(lo, hi, e.x, e.y));
                FanElem<T>::st(k + ihi, rot_hi(lo, hi, e.x, e.y));
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            bulk_s2g(a.out + ((int64_t)cons.l * a.out_rows + cons.dst + r0) * a.row_bytes, tile,
                     (uint32_t)(rows * a.row_bytes));
            bulk_commit();
            // tile t + STAGES - D + 1 goes into the stage of tile t - D + 1 ... first those
            // stages never used yet (t < D - 1), then the one whose store left D tiles ago
            const int64_t nt = t + STAGES - D + 1;
            if (prod.valid(a)) {
                if (t >= D - 1) bulk_wait_read<D - 1>();  // store t - D + 1 has left its stage
                issue(prod, (int)(nt % STAGES));
                prod.next(a, false);
            }
        }
        cons.next(a, threadIdx.x == 0);
    }
    if (threadIdx.x == 0) bulk_wait<0>();
}

// Warp-specialised reload form (bf16, 64-wide k_r): a producer warp walks the
// (group, layer, tile, member) sequence and issues each tile's bulk load together
// with its member's (cos, sin) table and a stage record (store address, bytes);
// NROT rotation warps rotate k_r in place, one 8-pair unit per thread; a storer
// warp issues each tile's bulk store and hands the stage back once the store has
// left it (D stores in flight). Iterator loads (group / member metadata, L2
// latency) never sit between a tile's arrival and its store.
struct StageRec {
    int64_t out_off;  // byte offset of the tile's destination in out
    uint32_t bytes;   // 0: end of work
    int32_t rows;
};

template <int ROWS, int STAGES, int D, int HINT>
__global__ void __launch_bounds__(64 + ROWS * 4)
rotate_gather_ws_kernel(FanArgs a) {
    constexpr int NROT = ROWS * 4 / 32;  // rotation warps: one 8-pair unit per thread
    static_assert(ROWS * 4 % 32 == 0 && D >= 1 && D < STAGES, "shape");
    if (a.n_groups_dev) a.n_items = min(a.n_groups, *a.n_groups_dev) * a.layers;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[STAGES], rotated[STAGES], empty[STAGES];
    __shared__ StageRec rec[STAGES];
    const int64_t stage_bytes = (int64_t)ROWS * a.row_bytes;
    float2 *cs_stage = reinterpret_cast<float2 *>(smem + STAGES * stage_bytes);  // 32 (cos, sin) per stage
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&rotated[s], NROT);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {  // ---------------------------------------------------- producer
        if (lane != 0) return;
        ReloadIter<ROWS> it;
        it.start(a, true);
        int64_t t = 0;
        for (;; ++t) {
            const int s = (int)(t % STAGES);
            if (t >= STAGES) mbar_wait(&empty[s], (uint32_t)(((t / STAGES) - 1) & 1));
            if (!it.valid(a)) {
                rec[s].bytes = 0;
                mbar_arrive(&full[s]);  // release: the record is visible to whoever waits the phase
                return;
            }
            const int32_t r0 = it.tile * ROWS;
            const int32_t rows = min(ROWS, it.len - r0);
            const uint32_t bytes = (uint32_t)(rows * a.row_bytes);
            rec[s].out_off = ((int64_t)it.l * a.out_rows + it.dst + r0) * a.row_bytes;
            rec[s].bytes = bytes;
            rec[s].rows = rows;
            mbar_arrive_expect_tx(&full[s], bytes + 256);
            if (HINT & 1)  // sources are re-read by the tile's other members: keep them in L2
                bulk_g2s_hint(smem + s * stage_bytes,
                              a.pool + ((int64_t)it.l * a.pool_rows + it.src + r0) * a.row_bytes, bytes, &full[s],
                              l2_policy_evict_last());
            else
                bulk_g2s(smem + s * stage_bytes, a.pool + ((int64_t)it.l * a.pool_rows + it.src + r0) * a.row_bytes,
                         bytes, &full[s]);
            bulk_g2s(cs_stage + s * 32, a.cs + (int64_t)(it.m0 + it.m) * 32, 256, &full[s]);
            it.next(a, true);
        }
    }
    if (warp == 1) {  // ---------------------------------------------------- storer
        if (lane != 0) return;
        for (int64_t t = 0;; ++t) {
            const int s = (int)(t % STAGES);
            mbar_wait(&rotated[s], (uint32_t)((t / STAGES) & 1));
            const uint32_t bytes = rec[s].bytes;
            if (bytes == 0) break;
            if (HINT & 2)  // destinations are not re-read by this launch
                bulk_s2g_hint(a.out + rec[s].out_off, smem + s * stage_bytes, bytes, l2_policy_evict_first());
            else
                bulk_s2g(a.out + rec[s].out_off, smem + s * stage_bytes, bytes);
            bulk_commit();
            if (t >= D - 1) {
                bulk_wait_read<D - 1>();  // store t - D + 1 has left its stage
                mbar_arrive(&empty[(int)((t - D + 1) % STAGES)]);
            }
        }
        bulk_wait<0>();
        return;
    }
    // ------------------------------------------------------------------------ rotation warps
    const int tid = threadIdx.x - 64;
    const int r = tid >> 2, u = tid & 3;
    const bool il = a.layout == IRM_LAYOUT_INTERLEAVED;
    for (int64_t t = 0;; ++t) {
        const int s = (int)(t % STAGES);
        mbar_wait(&full[s], (uint32_t)((t / STAGES) & 1));
        const uint32_t bytes = rec[s].bytes;
        if (bytes != 0 && r < rec[s].rows) {
            const float4 *c4 = reinterpret_cast<const float4 *>(cs_stage + s * 32 + 8 * u);
            float4 e[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) e[q] = c4[q];
            uint4 *k = reinterpret_cast<uint4 *>(smem + s * stage_bytes + (int64_t)r * a.row_bytes + a.ckv_bytes);
            uint4 w0 = k[il ? 2 * u : u], w1 = k[il ? 2 * u + 1 : u + 4];
            __nv_bfloat162 *p0 = reinterpret_cast<__nv_bfloat162 *>(&w0);
            __nv_bfloat162 *p1 = reinterpret_cast<__nv_bfloat162 *>(&w1);
            const float *ef = reinterpret_cast<const float *>(e);
            if (il) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    __nv_bfloat162 &p = q < 4 ? p0[q] : p1[q - 4];
                    const float2 v = __bfloat1622float2(p);
                    const float c = ef[2 * q], sn = ef[2 * q + 1];
                    p = __floats2bfloat162_rn(rot_lo(v.x, v.y, c, sn), rot_hi(v.x, v.y, c, sn));
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 lo = __bfloat1622float2(p0[q]), hi = __bfloat1622float2(p1[q]);
                    const float c0 = ef[4 * q], s0 = ef[4 * q + 1], c1 = ef[4 * q + 2], s1 = ef[4 * q + 3];
                    p0[q] = __floats2bfloat162_rn(rot_lo(lo.x, hi.x, c0, s0), rot_lo(lo.y, hi.y, c1, s1));
                    p1[q] = __floats2bfloat162_rn(rot_hi(lo.x, hi.x, c0, s0), rot_hi(lo.y, hi.y, c1, s1));
                }
            }
            k[il ? 2 * u : u] = w0;
            k[il ? 2 * u + 1 : u + 4] = w1;
            fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rotated[s]);
        if (bytes == 0) return;
    }
}

template <int ROWS, int STAGES, int D, int HINT = 0>
static int launch_ws(const FanArgs &a, int max_sms, cudaStream_t st) {
    auto kern = rotate_gather_ws_kernel<ROWS, STAGES, D, HINT>;
    constexpr int threads = 64 + ROWS * 4;
    const int smem = STAGES * (ROWS * a.row_bytes + 256);
    IRM_REQUIRE(smem <= 227 * 1024, "stages do not fit in shared memory (row_bytes %d)", a.row_bytes);
    IRM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    IRM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    if (per_sm < 1) per_sm = 1;
    int sms = sm_count();
    if (max_sms > 0) sms = std::min(sms, max_sms);
    int64_t grid = (int64_t)sms * per_sm * (a.rounds > 1 ? a.rounds : 1);
    if (grid > a.n_items) grid = a.n_items;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, threads, smem, st>>>(a);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

template <typename T, int ROWS, int STAGES, int D>
static int launch_reload(const FanArgs &a_in, int max_sms, cudaStream_t st) {
    FanArgs a = a_in;
    a.work = nullptr;  // producer and consumers walk the item sequence independently: static schedule
    a.rounds = 1;
    // the vectorised k_r path: bf16, 64-wide k_r, 16-byte aligned c_KV
    const bool vec = std::is_same<T, __nv_bfloat16>::value && a.kr == 64 && a.ckv_bytes % 16 == 0 &&
                     ROWS * 4 <= 256;
    auto kern = vec ? rotate_gather_reload_kernel<T, ROWS, STAGES, D, 256, (ROWS * 4 <= 256)>
                    : rotate_gather_reload_kernel<T, ROWS, STAGES, D, 256, false>;
    const int smem = STAGES * (ROWS * a.row_bytes + (a.kr / 2) * (int)sizeof(float2));
    IRM_REQUIRE(smem <= 227 * 1024, "reload stages do not fit in shared memory (row_bytes %d)", a.row_bytes);
    IRM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    IRM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    if (per_sm < 1) per_sm = 1;
    int sms = sm_count();
    if (max_sms > 0) sms = std::min(sms, max_sms);
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > a.n_items) grid = a.n_items;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, 256, smem, st>>>(a);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

template <typename T>
static int dispatch_fanout(const FanArgs &a, int max_sms, cudaStream_t st) {
    const bool ws_ok = std::is_same<T, __nv_bfloat16>::value && a.kr == 64 && a.ckv_bytes % 16 == 0 &&
                       6 * (32 * a.row_bytes + 256) <= 227 * 1024;
    if (const char *v = getenv("IRM_FAN_VARIANT")) {  // tuning hook (tools/k4_fan_bench.py)
        const int var = atoi(v);
        if (var == 1) return launch_reload<T, 48, 4, 2>(a, max_sms, st);
        if (var == 2) return launch_reload<T, 32, 6, 3>(a, max_sms, st);
        if (ws_ok) {
            if (var == 3) return launch_ws<48, 4, 2, 3>(a, max_sms, st);
            if (var == 4) return launch_ws<24, 8, 4, 3>(a, max_sms, st);
            if (var == 5) return launch_ws<16, 12, 6, 3>(a, max_sms, st);
            if (var == 6) return launch_ws<32, 6, 3, 0>(a, max_sms, st);
        }
    }
    // default: warp-specialised, 32-row tiles, 6 stages, 3 stores in flight, L2 hints
    // (tools/k4_fan_bench.py: 1.68-1.70 ms on the config-2 wave at 148 and 120 SMs)
    if (ws_ok) return launch_ws<32, 6, 3, 3>(a, max_sms, st);
    for (int rows : {32, 16, 8, 4, 1})
        if (6 * (rows * a.row_bytes + (a.kr / 2) * (int)sizeof(float2)) <= 227 * 1024) {
            if (rows == 32) return launch_reload<T, 32, 6, 3>(a, max_sms, st);
            if (rows == 16) return launch_reload<T, 16, 6, 3>(a, max_sms, st);
            if (rows == 8) return launch_reload<T, 8, 6, 3>(a, max_sms, st);
            if (rows == 4) return launch_reload<T, 4, 6, 3>(a, max_sms, st);
            return launch_reload<T, 1, 6, 3>(a, max_sms, st);
        }
    IRM_REQUIRE(false, "row too wide for the fan-out gather (%d bytes)", a.row_bytes);
    return IRM_EINVAL;
}

}  // namespace irm

using namespace irm;

extern "C" int64_t irm_group_workspace_bytes(int64_t n) {
    if (n < 0) return -1;
    return carve_group_ws(nullptr, n).bytes;
}

extern "C" int irm_group_by_source(const int64_t *src_row, const int64_t *dst_row, const int32_t *len,
                                   const int64_t *delta, int64_t n, const int64_t *n_dev, int64_t *g_src,
                                   int32_t *g_len, int32_t *g_first, int32_t *g_count, int64_t *m_dst,
                                   int64_t *m_delta, int64_t *n_groups, void *ws, int64_t ws_bytes,
                                   irm_stream_t stream) {
    IRM_REQUIRE(n >= 0 && n < (1LL << 31), "n must be in [0, 2^31)");
    IRM_REQUIRE(n_groups != nullptr, "null n_groups");
    GroupWs w = carve_group_ws(ws, n);
    if (!ws || ws_bytes < w.bytes) {
        set_error("group workspace %lld < %lld", (long long)ws_bytes, (long long)w.bytes);
        return IRM_ECAPACITY;
    }
    IRM_REQUIRE(n == 0 || (src_row && dst_row && len && delta && g_src && g_len && g_first && g_count && m_dst &&
                           m_delta),
                "null pointer");
    group_by_source_kernel<<<1, GB_THREADS, 0, (cudaStream_t)stream>>>(
        src_row, dst_row, len, delta, n, n_dev, w, g_src, g_len, g_first, g_count, m_dst, m_delta, n_groups);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int64_t irm_fanout_workspace_bytes(int64_t n_members, int32_t kr_dim) {
    if (n_members < 0 || kr_dim < 0) return -1;
    return ((n_members * (kr_dim / 2) * (int64_t)sizeof(float2) + 255) / 256) * 256 + 256;
}

extern "C" int irm_rotate_gather_fanout(const void *pool, int64_t pool_layer_stride, void *out,
                                        int64_t out_layer_stride, int32_t layers, int32_t ckv_dim, int32_t kr_dim,
                                        const int64_t *g_src, const int32_t *g_len, const int32_t *g_first,
                                        const int32_t *g_count, int64_t n_groups, const int64_t *n_groups_dev,
                                        const int64_t *m_dst, const int64_t *m_delta, int64_t n_members,
                                        const int64_t *n_members_dev, const double *inv_freq, int32_t layout,
                                        int32_t dtype, int32_t max_sms, int32_t cta_rounds, uint64_t *status, void *ws,
                                        int64_t ws_bytes, irm_stream_t stream) {
    IRM_REQUIRE(n_groups >= 0 && n_members >= 0 && layers >= 1 && ckv_dim >= 0 && kr_dim >= 4 && kr_dim % 4 == 0,
                "bad sizes (layers >= 1, kr_dim a multiple of 4)");
    IRM_REQUIRE(layout == IRM_LAYOUT_HALF_SPLIT || layout == IRM_LAYOUT_INTERLEAVED, "bad layout");
    IRM_REQUIRE(dtype == IRM_DTYPE_BF16 || dtype == IRM_DTYPE_F32, "fan-out gather: bf16 or f32 pools");
    IRM_REQUIRE(max_sms >= 0, "max_sms must be >= 0");
    IRM_REQUIRE(cta_rounds >= 1, "cta_rounds must be >= 1");
    if (n_groups == 0 || n_members == 0) return IRM_OK;
    IRM_REQUIRE(pool && out && g_src && g_len && g_first && g_count && m_dst && m_delta && inv_freq && ws,
                "null pointer");
    const int esz = dtype == IRM_DTYPE_F32 ? 4 : 2;
    IRM_REQUIRE((ckv_dim * esz) % 16 == 0 && ((ckv_dim + kr_dim) * esz) % 16 == 0,
                "fan-out gather: c_KV and row bytes must be multiples of 16");
    IRM_REQUIRE((((uintptr_t)pool) | ((uintptr_t)out)) % 16 == 0, "pool/out must be 16-byte aligned");
    if (ws_bytes < irm_fanout_workspace_bytes(n_members, kr_dim)) {
        set_error("fan-out workspace too small");
        return IRM_ECAPACITY;
    }
    cudaStream_t st = (cudaStream_t)stream;
    float2 *cs = reinterpret_cast<float2 *>(ws);
    const int half = kr_dim / 2;
    const int64_t grid = std::min<int64_t>((n_members * half + 255) / 256, (int64_t)sm_count() * 8);
    const int64_t cs_bytes = ((n_members * half * (int64_t)sizeof(float2) + 255) / 256) * 256;
    unsigned long long *work = reinterpret_cast<unsigned long long *>((char *)ws + cs_bytes);  // the spare 256 B
    member_cossin_kernel<<<(unsigned)std::max<int64_t>(grid, 1), 256, 0, st>>>(m_delta, n_members, n_members_dev,
                                                                               half, inv_freq, cs, work);
    IRM_LAUNCH_CHECK();
    FanArgs a{};
    a.pool = (const char *)pool;
    a.out = (char *)out;
    a.pool_rows = pool_layer_stride;
    a.out_rows = out_layer_stride;
    a.layers = layers;
    a.ckv = ckv_dim;
    a.kr = kr_dim;
    a.row_bytes = (ckv_dim + kr_dim) * esz;
    a.ckv_bytes = ckv_dim * esz;
    a.g_src = g_src;
    a.g_len = g_len;
    a.g_first = g_first;
    a.g_count = g_count;
    a.m_dst = m_dst;
    a.cs = cs;
    a.n_groups = n_groups;
    a.n_items = n_groups * layers;
    a.n_groups_dev = n_groups_dev;
    a.layout = layout;
    a.status = (unsigned long long *)status;
    a.work = getenv("IRM_FAN_STATIC") ? nullptr : work;  // tuning hook: the static round robin
    a.rounds = cta_rounds;
    if (dtype == IRM_DTYPE_BF16) return dispatch_fanout<__nv_bfloat16>(a, max_sms, st);
    return dispatch_fanout<float>(a, max_sms, st);
}
