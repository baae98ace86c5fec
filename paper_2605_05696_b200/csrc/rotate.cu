// K4: delta-rotation rotate + gather, and the per-row producer rotation.
//
// Replaces KvRegistry.materialize (reference registry.py:146-166) over a
// paged latent pool: per hit chunk and layer, the position-free c_KV rows are
// copied verbatim and the 64-wide k_r rows are rotated by R(delta), delta =
// p_dest - p_src uniform per chunk (rotary.py:98-108 with positions = delta).
//
// HBM-bound: 1152 B read + 1152 B written per bf16 row. A persistent CTA
// streams contiguous row tiles of one (chunk, layer) slab through shared
// memory with 1-D bulk async copies (TMA engine, mbarrier completion), rotates
// the k_r columns in shared memory in fp32 (cos/sin from an fp64 angle per
// chunk: fp32 angles fail the 1e-5 bar at |delta| ~ 2^20), and writes the tile
// back with a bulk store. STAGES tiles are in flight per CTA.
#include <algorithm>
#include <cuda.h>
#include <string.h>
#include "common.cuh"
#include "tma.cuh"
#include <cuda_bf16.h>
#include <stdlib.h>

namespace irm {

// ------------------------------------------------------------ element traits
template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
    using CS = float2;
    using Acc = float;
    static __device__ __forceinline__ float load(__nv_bfloat16 v) { return __bfloat162float(v); }
    static __device__ __forceinline__ __nv_bfloat16 store(float v, int) { return __float2bfloat16_rn(v); }
};
template <> struct Elem<float> {
    using CS = float2;
    using Acc = float;
    static __device__ __forceinline__ float load(float v) { return v; }
    static __device__ __forceinline__ float store(float v, int) { return v; }
};

__device__ __forceinline__ double round_bf16_f64(double x) {
    // single RNE rounding of f64 onto the bf16 grid (rotary.py:63-87)
    if (!isfinite(x) || x == 0.0) return x;
    int e;
    frexp(x, &e);
    const int ue = max(e - 8, -133);
    double q = ldexp(rint(ldexp(x, -ue)), ue);
    const double bf16_max = ldexp(2.0 - ldexp(1.0, -7), 127);
    if (fabs(q) > bf16_max) q = copysign(__longlong_as_double(0x7ff0000000000000LL), q);
    return q;
}

template <> struct Elem<double> {
    using CS = double2;
    using Acc = double;
    static __device__ __forceinline__ double load(double v) { return v; }
    static __device__ __forceinline__ double store(double v, int round) {
        if (round == IRM_ROUND_F32) return (double)__double2float_rn(v);
        if (round == IRM_ROUND_BF16) return round_bf16_f64(v);
        return v;
    }
};

template <typename CS>
__device__ __forceinline__ CS make_cs(double a);
template <> __device__ __forceinline__ float2 make_cs<float2>(double a) {
    double s, c;
    sincos_cr(a, &s, &c);
    return make_float2((float)c, (float)s);
}
template <> __device__ __forceinline__ double2 make_cs<double2>(double a) {
    double s, c;
    sincos_cr(a, &s, &c);
    return make_double2(c, s);
}

// per chunk: cs[c*half + j] = (cos, sin)(delta[c] * inv_freq[j]), angle in fp64
template <typename CS>
__global__ void chunk_cossin_kernel(const int64_t *__restrict__ delta, int64_t n_chunks, int half,
                                    const double *__restrict__ inv_freq, CS *__restrict__ cs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_chunks * half) return;
    const int64_t c = i / half;
    const int j = (int)(i - c * half);
    cs[i] = make_cs<CS>((double)delta[c] * inv_freq[j]);
}

template <typename T>
__device__ __forceinline__ void rotate_pair(T *row_kr, int j, int half, int layout,
                                            typename Elem<T>::CS cs, int round) {
    using A = typename Elem<T>::Acc;
    const int ilo = layout == IRM_LAYOUT_INTERLEAVED ? 2 * j : j;
    const int ihi = layout == IRM_LAYOUT_INTERLEAVED ? 2 * j + 1 : j + half;
    const A lo = Elem<T>::load(row_kr[ilo]);
    const A hi = Elem<T>::load(row_kr[ihi]);
    const A c = (A)cs.x, s = (A)cs.y;
    row_kr[ilo] = Elem<T>::store(rot_lo(lo, hi, c, s), round);
    row_kr[ihi] = Elem<T>::store(rot_hi(lo, hi, c, s), round);
}

// ------------------------------------------------------------ TMA-staged kernel
struct GatherArgs {
    const char *pool;
    char *out;
    int64_t pool_ls, out_ls;  // layer strides in rows
    int32_t layers, ckv, kr, row_bytes;
    const int64_t *src_row, *dst_row, *delta;
    const int32_t *len;
    int64_t n_chunks, n_items;
    const int64_t *n_dev;  // optional device-side chunk count (<= n_chunks): graph-friendly compaction
    int32_t layout, round;
    unsigned long long *status;  // optional sticky flags: 1 source run outside the pool, 2 destination outside out
};

// A chunk's rows must lie inside the pool and the output (the layer strides are the row
// counts): out-of-range work is skipped and reported, never read or written.
__device__ __forceinline__ bool chunk_in_bounds(const GatherArgs &a, int64_t c, bool report) {
    const int64_t len = __ldg(a.len + c), s = __ldg(a.src_row + c), d = __ldg(a.dst_row + c);
    const bool src_ok = s >= 0 && len >= 0 && s + len <= a.pool_ls;
    const bool dst_ok = d >= 0 && d + len <= a.out_ls;
    if (report && a.status && !(src_ok && dst_ok))
        atomicOr(a.status, (src_ok ? 0ULL : 1ULL) | (dst_ok ? 0ULL : 2ULL));
    return src_ok && dst_ok;
}

template <int ROWS>
struct TileIter {
    int64_t item, c;
    int32_t l, tile, ntiles;
    __device__ __forceinline__ void load(const GatherArgs &a, bool report) {
        while (item < a.n_items) {
            c = item / a.layers;
            l = (int32_t)(item - c * a.layers);
            ntiles = chunk_in_bounds(a, c, report && l == 0) ? (__ldg(a.len + c) + ROWS - 1) / ROWS : 0;
            if (ntiles > 0) return;
            item += gridDim.x;
        }
    }
    __device__ __forceinline__ void start(const GatherArgs &a, bool report) {
        item = blockIdx.x;
        tile = 0;
        load(a, report);
    }
    __device__ __forceinline__ void next(const GatherArgs &a, bool report) {
        if (++tile >= ntiles) {
            tile = 0;
            item += gridDim.x;
            load(a, report);
        }
    }
    __device__ __forceinline__ bool valid(const GatherArgs &a) const { return item < a.n_items; }
};

template <typename T, int ROWS, int STAGES, int THREADS>
__global__ void __launch_bounds__(THREADS)
rotate_gather_tma_kernel(GatherArgs a, const typename Elem<T>::CS *__restrict__ cs) {
    if (a.n_dev) a.n_items = min(a.n_chunks, *a.n_dev) * a.layers;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const int64_t stage_bytes = (int64_t)ROWS * a.row_bytes;
    const int row_elems = a.ckv + a.kr;
    const int half = a.kr / 2;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](const TileIter<ROWS> &it, int stage) {
        const int32_t r0 = it.tile * ROWS;
        const int32_t rows = min(ROWS, __ldg(a.len + it.c) - r0);
        const uint32_t bytes = (uint32_t)(rows * a.row_bytes);
        const char *src = a.pool + ((int64_t)it.l * a.pool_ls + __ldg(a.src_row + it.c) + r0) * a.row_bytes;
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(smem + stage * stage_bytes, src, bytes, &full[stage]);
    };

    // producer iterator (thread 0) runs STAGES-1 tiles ahead of the consumers
    TileIter<ROWS> prod, cons;
    cons.start(a, threadIdx.x == 0);
    if (threadIdx.x == 0) {
        prod.start(a, false);
        for (int s = 0; s < STAGES && prod.valid(a); ++s) {
            issue(prod, s);
            prod.next(a, false);
        }
    }
    for (int64_t t = 0; cons.valid(a); ++t) {
        const int stage = (int)(t % STAGES);
        const int32_t r0 = cons.tile * ROWS;
        const int32_t rows = min(ROWS, __ldg(a.len + cons.c) - r0);
        mbar_wait(&full[stage], (uint32_t)((t / STAGES) & 1));
        T *tile = reinterpret_cast<T *>(smem + stage * stage_bytes);
        const typename Elem<T>::CS *ccs = cs + cons.c * half;
        for (int i = threadIdx.x; i < rows * half; i += THREADS) {
            const int r = i / half, j = i - r * half;
            rotate_pair<T>(tile + (int64_t)r * row_elems + a.ckv, j, half, a.layout, ccs[j], a.round);
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            char *dst = a.out + ((int64_t)cons.l * a.out_ls + __ldg(a.dst_row + cons.c) + r0) * a.row_bytes;
            bulk_s2g(dst, tile, (uint32_t)(rows * a.row_bytes));
            bulk_commit();
            if (t >= 1 && prod.valid(a)) {
                bulk_wait_read<1>();  // the store of tile t-1 has left its stage
                issue(prod, (int)((t - 1) % STAGES));
                prod.next(a, false);
            }
        }
        cons.next(a, threadIdx.x == 0);
    }
    if (threadIdx.x == 0) bulk_wait<0>();
}

// ------------------------------------------------------------ generic fallback
// any dims / alignment: one CTA per (chunk, layer) item, one warp per row
template <typename T>
__global__ void rotate_gather_generic_kernel(GatherArgs a, const typename Elem<T>::CS *__restrict__ cs) {
    if (a.n_dev) a.n_items = min(a.n_chunks, *a.n_dev) * a.layers;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int row_elems = a.ckv + a.kr, half = a.kr / 2;
    for (int64_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
        const int64_t c = item / a.layers;
        const int32_t l = (int32_t)(item - c * a.layers);
        if (!chunk_in_bounds(a, c, threadIdx.x == 0 && l == 0)) continue;
        for (int32_t r = warp; r < a.len[c]; r += nwarp) {
            const T *src = reinterpret_cast<const T *>(a.pool) + ((int64_t)l * a.pool_ls + a.src_row[c] + r) * row_elems;
            T *dst = reinterpret_cast<T *>(a.out) + ((int64_t)l * a.out_ls + a.dst_row[c] + r) * row_elems;
            for (int e = lane; e < row_elems; e += 32) dst[e] = src[e];
            __syncwarp();
            for (int j = lane; j < half; j += 32) rotate_pair<T>(dst + a.ckv, j, half, a.layout, cs[c * half + j], a.round);
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------ per-row rotation
// One thread per (row, frequency): the angle's cos/sin are computed once and applied to
// the row in every layer (the producer rotates kr_raw of all layers by the same p_src + i,
// registry.py:131-133). fp64 rows take correctly rounded cos/sin (sincos_cr: the
// reference's f64 values bit for bit); fp32/bf16 rows round CUDA's fp64 sincos to fp32.
template <typename CS>
__device__ __forceinline__ CS row_cs(double a);
template <> __device__ __forceinline__ double2 row_cs<double2>(double a) {
    double s, c;
    sincos_cr(a, &s, &c);
    return make_double2(c, s);
}
template <> __device__ __forceinline__ float2 row_cs<float2>(double a) {
    double s, c;
    sincos(a, &s, &c);
    return make_float2((float)c, (float)s);
}

template <typename T>
// rows / out may be the same buffer (in place): every element is read, then written, by one
// thread only, so the non-aliasing promise holds for every access the compiler may reorder
__global__ void rotate_rows_kernel(const T *__restrict__ rows, int64_t rs, int64_t rls, T *__restrict__ out,
                                   int64_t os, int64_t ols, int64_t n, int half, int layers,
                                   const double *__restrict__ pos, const double *__restrict__ inv_freq,
                                   int layout, int round) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * half) return;
    const int64_t r = i / half;
    const int j = (int)(i - r * half);
    const int ilo = layout == IRM_LAYOUT_INTERLEAVED ? 2 * j : j;
    const int ihi = layout == IRM_LAYOUT_INTERLEAVED ? 2 * j + 1 : j + half;
    using A = typename Elem<T>::Acc;
    const auto cs = row_cs<typename Elem<T>::CS>(pos[r] * inv_freq[j]);
    for (int l = 0; l < layers; ++l) {
        const T *src = rows + l * rls + r * rs;
        T *dst = out + l * ols + r * os;
        const A lo = Elem<T>::load(src[ilo]), hi = Elem<T>::load(src[ihi]);
        dst[ilo] = Elem<T>::store(rot_lo(lo, hi, (A)cs.x, (A)cs.y), round);
        dst[ihi] = Elem<T>::store(rot_hi(lo, hi, (A)cs.x, (A)cs.y), round);
    }
}

// bf16, 64-wide rotary rows, 16-byte aligned: one thread per (row, 8-pair unit) -- eight
// cos/sin pairs computed once, then two 16-byte loads / stores per layer (the pairs of
// j = 8u .. 8u+7: interleaved words 2u, 2u+1; half-split words u (lo) and u+4 (hi))
template <int LSPLIT>
__global__ void rotate_rows_bf16x8_kernel(const __nv_bfloat16 *__restrict__ rows, int64_t rs, int64_t rls,
                                          __nv_bfloat16 *__restrict__ out, int64_t os, int64_t ols, int64_t n,
                                          int layers, const double *__restrict__ pos,
                                          const double *__restrict__ inv_freq, int layout) {
    // LSPLIT threads share a (row, unit): thread ls takes layers ls, ls + LSPLIT, ... (more loads in flight)
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * 4 * LSPLIT) return;
    const int ls = (int)(i % LSPLIT);
    const int64_t r = (i / LSPLIT) >> 2;
    const int u = (int)((i / LSPLIT) & 3);
    float c[8], sn[8];
    const double p = pos[r];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        double s_, c_;
        sincos(p * inv_freq[8 * u + q], &s_, &c_);
        c[q] = (float)c_;
        sn[q] = (float)s_;
    }
    const bool il = layout == IRM_LAYOUT_INTERLEAVED;
    const int w0i = il ? 2 * u : u, w1i = il ? 2 * u + 1 : u + 4;
#pragma unroll 3
    for (int l = ls; l < layers; l += LSPLIT) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rows + l * rls + r * rs);
        uint4 *dst = reinterpret_cast<uint4 *>(out + l * ols + r * os);
        uint4 w0 = src[w0i], w1 = src[w1i];
        __nv_bfloat162 *p0 = reinterpret_cast<__nv_bfloat162 *>(&w0);
        __nv_bfloat162 *p1 = reinterpret_cast<__nv_bfloat162 *>(&w1);
        if (il) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                __nv_bfloat162 &pp = q < 4 ? p0[q] : p1[q - 4];
                const float2 v = __bfloat1622float2(pp);
                pp = __floats2bfloat162_rn(rot_lo(v.x, v.y, c[q], sn[q]), rot_hi(v.x, v.y, c[q], sn[q]));
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 lo = __bfloat1622float2(p0[q]), hi = __bfloat1622float2(p1[q]);
                p0[q] = __floats2bfloat162_rn(rot_lo(lo.x, hi.x, c[2 * q], sn[2 * q]),
                                              rot_lo(lo.y, hi.y, c[2 * q + 1], sn[2 * q + 1]));
                p1[q] = __floats2bfloat162_rn(rot_hi(lo.x, hi.x, c[2 * q], sn[2 * q]),
                                              rot_hi(lo.y, hi.y, c[2 * q + 1], sn[2 * q + 1]));
            }
        }
        dst[w0i] = w0;
        dst[w1i] = w1;
    }
}

// ------------------------------------------------------------ host launchers
constexpr int RG_THREADS = 256;
constexpr int RG_STAGES = 4;

template <typename T, int ROWS, int STAGES = RG_STAGES>
static int launch_tma(const GatherArgs &a, const typename Elem<T>::CS *cs, int max_sms, cudaStream_t st) {
    auto kern = rotate_gather_tma_kernel<T, ROWS, STAGES, RG_THREADS>;
    const int smem = STAGES * ROWS * a.row_bytes;
    IRM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    IRM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RG_THREADS, smem));
    if (per_sm < 1) per_sm = 1;
    int sms = sm_count();
    if (max_sms > 0) sms = std::min(sms, max_sms);
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > a.n_items) grid = a.n_items;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, RG_THREADS, smem, st>>>(a, cs);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

template <typename T>
static int launch_gather(const GatherArgs &a, void *ws, const int64_t *delta, const double *inv_freq,
                         int max_sms, cudaStream_t st) {
    using CS = typename Elem<T>::CS;
    const int half = a.kr / 2;
    CS *cs = reinterpret_cast<CS *>(ws);
    const int64_t ncs = a.n_chunks * half;
    if (ncs > 0) {
        chunk_cossin_kernel<CS><<<(unsigned)((ncs + 255) / 256), 256, 0, st>>>(delta, a.n_chunks, half, inv_freq, cs);
        IRM_LAUNCH_CHECK();
    }
    const bool tma_ok = (a.row_bytes % 16 == 0) && (((uintptr_t)a.pool | (uintptr_t)a.out) % 16 == 0);
    if (tma_ok) {
        // rows per tile so that one pipeline stage is ~36 KB (4 stages: 144 KB, one CTA per SM;
        // 18 KB stages with 3 CTAs per SM ran 2-5 % slower, tools/k4_tune.py)
        const int rows_fit = 36864 / a.row_bytes;
        if (const char *v = getenv("IRM_RG_VARIANT")) {  // tuning hook: rows x stages
            const int var = atoi(v);
            if (var == 1) return launch_tma<T, 8, 8>(a, cs, max_sms, st);
            if (var == 2) return launch_tma<T, 16, 6>(a, cs, max_sms, st);
            if (var == 3) return launch_tma<T, 32, 3>(a, cs, max_sms, st);
            if (var == 4) return launch_tma<T, 32, 4>(a, cs, max_sms, st);
            if (var == 5) return launch_tma<T, 8, 12>(a, cs, max_sms, st);
            if (var == 6) return launch_tma<T, 16, 8>(a, cs, max_sms, st);
            if (var == 7) return launch_tma<T, 32, 5>(a, cs, max_sms, st);
            if (var == 8) return launch_tma<T, 32, 6>(a, cs, max_sms, st);
            if (var == 9) return launch_tma<T, 64, 3>(a, cs, max_sms, st);
            if (var == 10) return launch_tma<T, 48, 4>(a, cs, max_sms, st);
            if (var == 11) return launch_tma<T, 24, 6>(a, cs, max_sms, st);
        }
        if (rows_fit >= 32) return launch_tma<T, 32>(a, cs, max_sms, st);
        if (rows_fit >= 16) return launch_tma<T, 16>(a, cs, max_sms, st);
        if (rows_fit >= 8) return launch_tma<T, 8>(a, cs, max_sms, st);
        if (a.row_bytes <= 49152) return launch_tma<T, 1>(a, cs, max_sms, st);
    }
    int64_t grid = (int64_t)sm_count() * 8;
    if (grid > a.n_items) grid = a.n_items;
    rotate_gather_generic_kernel<T><<<(unsigned)grid, 256, 0, st>>>(a, cs);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

}  // namespace irm

using namespace irm;

extern "C" int64_t irm_rotate_gather_workspace_bytes(int64_t n_chunks, int32_t kr_dim) {
    if (n_chunks < 0 || kr_dim < 0) return -1;
    const int64_t cs = ((n_chunks * (kr_dim / 2) * (int64_t)sizeof(double2) + 255) / 256) * 256;
    return cs + 256;
}

extern "C" int irm_rotate_gather(const void *pool, int64_t pool_layer_stride, void *out,
                                 int64_t out_layer_stride, int32_t layers, int32_t ckv_dim,
                                 int32_t kr_dim, const int64_t *src_row, const int64_t *dst_row,
                                 const int32_t *len, const int64_t *delta, int64_t n_chunks,
                                 const int64_t *n_chunks_dev, const double *inv_freq, int32_t layout,
                                 int32_t dtype, int32_t out_round, int32_t max_sms, uint64_t *status, void *ws,
                                 int64_t ws_bytes, irm_stream_t stream) {
    IRM_REQUIRE(n_chunks >= 0 && layers >= 1 && ckv_dim >= 0 && kr_dim >= 0 && kr_dim % 2 == 0,
                "bad sizes (layers >= 1, kr_dim even)");
    IRM_REQUIRE(layout == IRM_LAYOUT_HALF_SPLIT || layout == IRM_LAYOUT_INTERLEAVED, "bad layout");
    IRM_REQUIRE(dtype >= IRM_DTYPE_F64 && dtype <= IRM_DTYPE_BF16, "bad dtype");
    IRM_REQUIRE(out_round == IRM_ROUND_NONE || dtype == IRM_DTYPE_F64,
                "out_round applies to f64 pools only");
    IRM_REQUIRE(out_round >= 0 && out_round <= 2, "bad out_round");
    IRM_REQUIRE(max_sms >= 0, "max_sms must be >= 0");
    if (n_chunks == 0) return IRM_OK;
    IRM_REQUIRE(pool && out && src_row && dst_row && len && delta && inv_freq && ws, "null pointer");
    if (ws_bytes < irm_rotate_gather_workspace_bytes(n_chunks, kr_dim)) {
        set_error("rotate_gather workspace too small");
        return IRM_ECAPACITY;
    }
    const int esz = dtype == IRM_DTYPE_F64 ? 8 : dtype == IRM_DTYPE_F32 ? 4 : 2;
    GatherArgs a{};
    a.pool = (const char *)pool;
    a.out = (char *)out;
    a.pool_ls = pool_layer_stride;
    a.out_ls = out_layer_stride;
    a.layers = layers;
    a.ckv = ckv_dim;
    a.kr = kr_dim;
    a.row_bytes = (ckv_dim + kr_dim) * esz;
    a.src_row = src_row;
    a.dst_row = dst_row;
    a.delta = delta;
    a.len = len;
    a.n_chunks = n_chunks;
    a.n_items = n_chunks * layers;
    a.n_dev = n_chunks_dev;
    a.layout = layout;
    a.round = out_round;
    a.status = (unsigned long long *)status;
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == IRM_DTYPE_BF16) return launch_gather<__nv_bfloat16>(a, ws, delta, inv_freq, max_sms, st);
    if (dtype == IRM_DTYPE_F32) return launch_gather<float>(a, ws, delta, inv_freq, max_sms, st);
    return launch_gather<double>(a, ws, delta, inv_freq, max_sms, st);
}

extern "C" int irm_rotate_rows_layered(const void *rows, int64_t row_stride, int64_t rows_layer_stride, void *out,
                                       int64_t out_stride, int64_t out_layer_stride, int32_t layers, int64_t n,
                                       int32_t dim, const double *positions, const double *inv_freq, int32_t layout,
                                       int32_t dtype, int32_t out_round, irm_stream_t stream) {
    IRM_REQUIRE(n >= 0 && dim >= 0 && dim % 2 == 0 && layers >= 1, "bad sizes (dim even, layers >= 1)");
    IRM_REQUIRE(layout == IRM_LAYOUT_HALF_SPLIT || layout == IRM_LAYOUT_INTERLEAVED, "bad layout");
    IRM_REQUIRE(out_round == IRM_ROUND_NONE || dtype == IRM_DTYPE_F64, "out_round applies to f64 only");
    if (n == 0 || dim == 0) return IRM_OK;
    IRM_REQUIRE(rows && out && positions && inv_freq, "null pointer");
    const int half = dim / 2;
    const unsigned grid = (unsigned)((n * half + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    const bool vec = dtype == IRM_DTYPE_BF16 && dim == 64 && out_round == IRM_ROUND_NONE && row_stride % 8 == 0 &&
                     out_stride % 8 == 0 && rows_layer_stride % 8 == 0 && out_layer_stride % 8 == 0 &&
                     ((((uintptr_t)rows) | ((uintptr_t)out)) & 15) == 0;
    const int lsplit = getenv("IRM_PROD_LSPLIT") ? atoi(getenv("IRM_PROD_LSPLIT")) : (layers >= 9 ? 3 : 1);
    if (vec && lsplit == 3)
        rotate_rows_bf16x8_kernel<3><<<(unsigned)((n * 12 + 255) / 256), 256, 0, st>>>(
            (const __nv_bfloat16 *)rows, row_stride, rows_layer_stride, (__nv_bfloat16 *)out, out_stride,
            out_layer_stride, n, layers, positions, inv_freq, layout);
    else if (vec)
        rotate_rows_bf16x8_kernel<1><<<(unsigned)((n * 4 + 255) / 256), 256, 0, st>>>(
            (const __nv_bfloat16 *)rows, row_stride, rows_layer_stride, (__nv_bfloat16 *)out, out_stride,
            out_layer_stride, n, layers, positions, inv_freq, layout);
    else if (dtype == IRM_DTYPE_BF16)
        rotate_rows_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
            (const __nv_bfloat16 *)rows, row_stride, rows_layer_stride, (__nv_bfloat16 *)out, out_stride,
            out_layer_stride, n, half, layers, positions, inv_freq, layout, out_round);
    else if (dtype == IRM_DTYPE_F32)
        rotate_rows_kernel<float><<<grid, 256, 0, st>>>((const float *)rows, row_stride, rows_layer_stride,
                                                        (float *)out, out_stride, out_layer_stride, n, half,
                                                        layers, positions, inv_freq, layout, out_round);
    else if (dtype == IRM_DTYPE_F64)
        rotate_rows_kernel<double><<<grid, 256, 0, st>>>((const double *)rows, row_stride, rows_layer_stride,
                                                         (double *)out, out_stride, out_layer_stride, n, half,
                                                         layers, positions, inv_freq, layout, out_round);
    else
        IRM_REQUIRE(false, "bad dtype");
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_rotate_rows(const void *rows, int64_t row_stride, void *out, int64_t out_stride,
                               int64_t n, int32_t dim, const double *positions,
                               const double *inv_freq, int32_t layout, int32_t dtype,
                               int32_t out_round, irm_stream_t stream) {
    return irm_rotate_rows_layered(rows, row_stride, 0, out, out_stride, 0, 1, n, dim, positions, inv_freq, layout,
                                   dtype, out_round, stream);
}

// Elementwise store rounding of f64 values (rotary.py:63-95: round_bf16 / f32 cast).
namespace irm {
__global__ void round_f64_kernel(const double *__restrict__ x, double *__restrict__ y, int64_t n, int mode) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = Elem<double>::store(x[i], mode);
}
}  // namespace irm

extern "C" int irm_round_f64(const double *x, double *y, int64_t n, int32_t mode, irm_stream_t stream) {
    IRM_REQUIRE(n >= 0 && mode >= 0 && mode <= 2, "bad arguments");
    if (n == 0) return IRM_OK;
    IRM_REQUIRE(x && y, "null pointer");
    irm::round_f64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, y, n, mode);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

// Replica fetch (K6): copy runs of latent rows whose source lives in another GPU's pool,
// addressed through peer (CUDA IPC / NVLink) mappings. One CTA per (run, layer) item,
// grid-stride; 16-byte loads straight from peer memory, 16-byte stores to the local pool.
namespace irm {
__global__ void copy_runs_kernel(const int64_t *__restrict__ src_addr, int64_t src_ls, char *__restrict__ dst,
                                 int64_t dst_ls, const int64_t *__restrict__ dst_row, const int32_t *__restrict__ len,
                                 int64_t n_runs, const int64_t *__restrict__ n_runs_dev, int layers, int row_bytes) {
    if (n_runs_dev) n_runs = min(n_runs, *n_runs_dev);
    const int64_t items = n_runs * layers;
    const int vec = row_bytes / 16;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t c = it / layers;
        const int l = (int)(it - c * layers);
        const int64_t n16 = (int64_t)__ldg(len + c) * vec;
        const uint4 *s = reinterpret_cast<const uint4 *>((const char *)__ldg(src_addr + c) + l * src_ls);
        uint4 *d = reinterpret_cast<uint4 *>(dst + l * dst_ls + __ldg(dst_row + c) * (int64_t)row_bytes);
        for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
    }
}
}  // namespace irm

extern "C" int irm_copy_runs(const int64_t *src_addr, int64_t src_layer_stride, void *dst, int64_t dst_layer_stride,
                             const int64_t *dst_row, const int32_t *len, int64_t n_runs, const int64_t *n_runs_dev,
                             int32_t layers, int32_t row_bytes, irm_stream_t stream) {
    IRM_REQUIRE(n_runs >= 0 && layers >= 1 && row_bytes > 0 && row_bytes % 16 == 0, "bad sizes");
    IRM_REQUIRE(src_layer_stride % 16 == 0 && dst_layer_stride % 16 == 0, "layer strides must be 16-byte multiples");
    if (n_runs == 0) return IRM_OK;
    IRM_REQUIRE(src_addr && dst && dst_row && len, "null pointer");
    IRM_REQUIRE(((uintptr_t)dst & 15) == 0, "dst must be 16-byte aligned");
    int64_t grid = std::min<int64_t>(n_runs * layers, (int64_t)sm_count() * 8);
    irm::copy_runs_kernel<<<(unsigned)std::max<int64_t>(grid, 1), 256, 0, (cudaStream_t)stream>>>(
        src_addr, src_layer_stride, (char *)dst, dst_layer_stride, dst_row, len, n_runs, n_runs_dev, layers, row_bytes);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

// ---------------------------------------------------------------- peer pool mapping (K6)
// The pool a peer process exports is mapped into this process on the CURRENT device with
// lazy peer enabling, so kernels launched on this rank's GPU read the peer's HBM over
// NVLink (the IPC handle is opened from the reader's device, not the owner's).
extern "C" int irm_peer_export(const void *ptr, void *handle, int64_t *offset) {
    IRM_REQUIRE(ptr && handle && offset, "null pointer");
    // driver entry point fetched through the runtime: the library does not link libcuda
    using range_fn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
    static range_fn get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        IRM_REQUIRE(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                        q == cudaDriverEntryPointSuccess && fn,
                    "cuMemGetAddressRange unavailable");
        get_range = (range_fn)fn;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    CUresult r = get_range(&base, &size, (CUdeviceptr)ptr);
    IRM_REQUIRE(r == CUDA_SUCCESS, "cuMemGetAddressRange failed (%d): not a device allocation", (int)r);
    static_assert(sizeof(cudaIpcMemHandle_t) == IRM_PEER_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    IRM_CUDA_CHECK(cudaIpcGetMemHandle(&h, (void *)base));
    memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((CUdeviceptr)ptr - base);
    return IRM_OK;
}

extern "C" int irm_peer_open(const void *handle, int64_t offset, void **ptr) {
    IRM_REQUIRE(handle && ptr && offset >= 0, "bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *base = nullptr;
    IRM_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr = (char *)base + offset;
    return IRM_OK;
}
