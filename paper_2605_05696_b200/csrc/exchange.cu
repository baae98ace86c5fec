// K6 exchange: the device side of one lookup wave over the hash-sharded store
// (shard.ShardedStore.lookup_insert). The reference has one
// in-process dict (registry.py:113-140, first writer wins in engine order,
// engine.py:197-223); sharded by fingerprint prefix, a wave's lookups become
//
//   irm_exchange_pack    queries -> [G, cap] owner buckets (fp, order, p, len),
//                        stable: bucket slots in query order; unused slots carry
//                        padding order keys above every real key
//   (all-to-all of the buckets: NCCL over NVLink, torch.distributed)
//   irm_exchange_split   received rows -> the K3 query arrays of the owner
//   (K3: irm_store_lookup_insert on the owner's shard; the winner is the smallest
//    order key, whatever the array order)
//   irm_exchange_reply   first writers get rows of the owner's sub-range of their
//                        own pool (bump allocation per writer in slot order), every
//                        entry's global row is recorded, and each slot's answer
//                        (hit, p_src, global row, fresh) is written in place
//   (reverse all-to-all)
//   irm_exchange_unpack  answers back to query order
//
// Each step is one launch with no host synchronisation (graph-capturable); the
// bucket bookkeeping and the per-writer scans run in one CTA so the slot order,
// and with it every row assignment, is deterministic.
#include "common.cuh"

namespace irm {
namespace xchg {

constexpr int XT = 1024;
constexpr int64_t PAD_ORDER = 1LL << 62;  // = shard.PAD_ORDER
constexpr int MAX_WORLD = 32;

__device__ __forceinline__ int owner_of(uint64_t fp, int world) {
    return (int)(((fp >> 32) * (uint64_t)world) >> 32);
}

__global__ void __launch_bounds__(XT) pack_kernel(const uint64_t *__restrict__ fp, const int64_t *__restrict__ order,
                                                  const int64_t *__restrict__ p, const int32_t *__restrict__ len,
                                                  const uint8_t *__restrict__ probe, int64_t n, int world, int rank,
                                                  int64_t cap, int64_t *__restrict__ send, int64_t *__restrict__ dest,
                                                  unsigned long long *__restrict__ flags) {
    __shared__ int64_t base[MAX_WORLD], tile_tot[MAX_WORLD];
    __shared__ int32_t woff[XT / 32][MAX_WORLD + 1];
    const int64_t m = (int64_t)world * cap;
    for (int64_t s = threadIdx.x; s < m; s += XT) {  // every slot padding first; real rows overwrite
        int64_t *r = send + 4 * s;
        r[0] = 0;
        r[1] = PAD_ORDER + (int64_t)rank * m + s;  // unique, above every real key
        r[2] = 0;
        r[3] = 0;
    }
    if (threadIdx.x < MAX_WORLD) base[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    bool over = false;
    for (int64_t b = 0; b < n; b += XT) {
        const int64_t i = b + threadIdx.x;
        int o = world;  // not probed
        if (i < n && (!probe || probe[i])) o = owner_of(fp[i], world);
        int myrank = 0;
        for (int k = 0; k < world; ++k) {  // per owner: this lane's rank among the warp's queries to it
            const unsigned msk = __ballot_sync(0xffffffffu, o == k);
            if (o == k) myrank = __popc(msk & lt);
            if (lane == 0) woff[w][k] = __popc(msk);
        }
        __syncthreads();
        if (threadIdx.x < world) {  // per owner: exclusive prefix over the warps (query order)
            int64_t run = 0;
            for (int ww = 0; ww < XT / 32; ++ww) {
                const int32_t c = woff[ww][threadIdx.x];
                woff[ww][threadIdx.x] = (int32_t)run;
                run += c;
            }
            tile_tot[threadIdx.x] = run;
        }
        __syncthreads();
        if (i < n) {
            int64_t d = -1;
            if (o < world) {
                const int64_t pos = base[o] + woff[w][o] + myrank;
                if (pos < cap) {
                    d = (int64_t)o * cap + pos;
                    int64_t *r = send + 4 * d;
                    r[0] = (int64_t)fp[i];
                    r[1] = order[i];
                    r[2] = p[i];
                    r[3] = (int64_t)len[i];
                } else {
                    over = true;  // the bucket is full: the query goes unanswered (flag 1)
                }
            }
            dest[i] = d;
        }
        __syncthreads();
        if (threadIdx.x < world) base[threadIdx.x] += tile_tot[threadIdx.x];
        __syncthreads();
    }
    if (__any_sync(0xffffffffu, over) && lane == 0) atomicOr(flags, 1ULL);
}

__global__ void split_kernel(const int64_t *__restrict__ recv, int64_t m, uint64_t *__restrict__ fp,
                             int64_t *__restrict__ order, int64_t *__restrict__ p, int32_t *__restrict__ len,
                             uint8_t *__restrict__ real) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t *r = recv + 4 * s;
        fp[s] = (uint64_t)r[0];
        order[s] = r[1];
        p[s] = r[2];
        len[s] = (int32_t)r[3];
        real[s] = r[1] < PAD_ORDER ? 1 : 0;
    }
}

__global__ void __launch_bounds__(XT) reply_kernel(const int64_t *__restrict__ recv, int world, int64_t cap,
                                                   const int32_t *__restrict__ hit, const int64_t *__restrict__ entry,
                                                   const int64_t *__restrict__ p_src,
                                                   const int64_t *__restrict__ n_before, int64_t base_row,
                                                   int64_t region, int64_t *__restrict__ next,
                                                   int64_t *__restrict__ e_grow, int64_t n_egrow,
                                                   unsigned long long *__restrict__ flags,
                                                   int64_t *__restrict__ reply) {
    __shared__ int64_t sm[XT / 32];
    const int64_t m = (int64_t)world * cap;
    // 1: first writers' rows, per writer w (slots [w cap, (w + 1) cap), its queries in order):
    //    lrow = base + next[w] + exclusive scan of the novel lengths; global row = w << 40 | lrow
    for (int wr = 0; wr < world; ++wr) {
        const int64_t start = next[wr];
        int64_t run = 0;
        for (int64_t t = 0; t < cap; t += XT) {
            const int64_t s = (int64_t)wr * cap + t + threadIdx.x;
            const bool novel = t + threadIdx.x < cap && hit[s] == 0;
            const int64_t L = novel ? recv[4 * s + 3] : 0;
            int64_t tot;
            const int64_t ex = block_exclusive_scan<XT>(L, &tot, sm);
            if (novel) {
                const int64_t e = entry[s];
                if (e >= 0 && e < n_egrow) e_grow[e] = ((int64_t)wr << 40) | (base_row + start + run + ex);
            }
            run += tot;
        }
        if (threadIdx.x == 0) {
            next[wr] = start + run;
            if (start + run > region) atomicOr(flags, 2ULL);  // the writer's sub-range is full
        }
        __syncthreads();
    }
    // 2: every slot's answer (e_grow of this wave's new entries is visible after the barrier)
    const int64_t nb = *n_before;
    for (int64_t s = threadIdx.x; s < m; s += XT) {
        const int32_t h = hit[s];
        const int64_t e = entry[s];
        int64_t *r = reply + 4 * s;
        r[0] = h;
        r[1] = p_src[s];
        r[2] = (e >= 0 && e < n_egrow) ? e_grow[e] : -1;
        r[3] = (h == 1 && e >= nb) ? 1 : 0;  // fresh: an entry this very exchange created
    }
}

__global__ void unpack_kernel(const int64_t *__restrict__ back, const int64_t *__restrict__ dest, int64_t n,
                              int64_t cap, int32_t *__restrict__ hit, int64_t *__restrict__ p_src,
                              int64_t *__restrict__ row, int64_t *__restrict__ owner, uint8_t *__restrict__ fresh) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = dest[i];
        if (d >= 0) {
            const int64_t *r = back + 4 * d;
            hit[i] = (int32_t)r[0];
            p_src[i] = r[1];
            row[i] = r[2];
            owner[i] = d / cap;
            fresh[i] = r[3] == 1 ? 1 : 0;
        } else {
            hit[i] = -1;
            p_src[i] = 0;
            row[i] = -1;
            owner[i] = -1;
            fresh[i] = 0;
        }
    }
}

}  // namespace xchg
}  // namespace irm

using namespace irm;

static unsigned grid_for(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 4L * sm_count() ? 4L * sm_count() : g));
}

extern "C" int irm_exchange_pack(const uint64_t *q_fp, const int64_t *q_order, const int64_t *q_p,
                                 const int32_t *q_len, const uint8_t *q_probe, int64_t n, int32_t world,
                                 int32_t rank, int64_t cap, int64_t *send, int64_t *dest, uint64_t *flags,
                                 irm_stream_t stream) {
    IRM_REQUIRE(n >= 0 && cap >= 0, "bad sizes");
    IRM_REQUIRE(world >= 1 && world <= xchg::MAX_WORLD && rank >= 0 && rank < world, "bad world / rank");
    IRM_REQUIRE(send && flags && (n == 0 || (q_fp && q_order && q_p && q_len && dest)), "null pointer");
    if ((int64_t)world * cap == 0 && n == 0) return IRM_OK;
    xchg::pack_kernel<<<1, xchg::XT, 0, (cudaStream_t)stream>>>(q_fp, q_order, q_p, q_len, q_probe, n, world, rank,
                                                               cap, send, dest, (unsigned long long *)flags);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_exchange_split(const int64_t *recv, int64_t m, uint64_t *fp, int64_t *order, int64_t *p,
                                  int32_t *len, uint8_t *real, irm_stream_t stream) {
    IRM_REQUIRE(m >= 0, "bad sizes");
    if (m == 0) return IRM_OK;
    IRM_REQUIRE(recv && fp && order && p && len && real, "null pointer");
    xchg::split_kernel<<<grid_for(m), 256, 0, (cudaStream_t)stream>>>(recv, m, fp, order, p, len, real);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_exchange_reply(const int64_t *recv, int32_t world, int64_t cap, const int32_t *hit,
                                  const int64_t *entry, const int64_t *p_src, const int64_t *n_before,
                                  int64_t base_row, int64_t region, int64_t *next, int64_t *e_grow, int64_t n_egrow,
                                  uint64_t *flags, int64_t *reply, irm_stream_t stream) {
    IRM_REQUIRE(world >= 1 && cap >= 0 && n_egrow >= 0, "bad sizes");
    if ((int64_t)world * cap == 0) return IRM_OK;
    IRM_REQUIRE(recv && hit && entry && p_src && n_before && next && e_grow && flags && reply, "null pointer");
    xchg::reply_kernel<<<1, xchg::XT, 0, (cudaStream_t)stream>>>(recv, world, cap, hit, entry, p_src, n_before,
                                                                base_row, region, next, e_grow, n_egrow,
                                                                (unsigned long long *)flags, reply);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_exchange_unpack(const int64_t *back, const int64_t *dest, int64_t n, int64_t cap, int32_t *hit,
                                   int64_t *p_src, int64_t *row, int64_t *owner, uint8_t *fresh,
                                   irm_stream_t stream) {
    IRM_REQUIRE(n >= 0 && cap >= 0, "bad sizes");
    if (n == 0) return IRM_OK;
    IRM_REQUIRE(back && dest && hit && p_src && row && owner && fresh, "null pointer");
    xchg::unpack_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(back, dest, n, cap, hit, p_src, row, owner,
                                                                       fresh);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}
