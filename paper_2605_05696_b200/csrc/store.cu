// K3: the content-hash chunk store on the device.
//
// Replaces KvRegistry.lookup / insert (reference registry.py:113-140) and the
// per-chunk probe/insert of engine.serve (engine.py:197-223) with a batched,
// order-exact operation: the reference serves chunks one at a time with
// first-writer-wins, which equals "per fingerprint, the query with the
// smallest (request, chunk) order key writes; everyone else hits it".
//
// Table: open addressing, linear probing, keys claimed with atomicCAS, the
// batch winner elected with atomicMin on the order key. Entry indices and
// pool rows of new entries are assigned by an exclusive scan in query order,
// so insert_epoch (registry.py:83,137) and pool layout are deterministic.
#include "common.cuh"
#include <algorithm>

namespace irm {

constexpr int ST_BLOCK = 512;
enum : int8_t { Q_NOVEL = 0, Q_HIT_OLD = 1, Q_HIT_BATCH = 2, Q_SKIP = 3 };
enum : int64_t { ERR_TABLE_FULL = 1, ERR_ENTRIES_FULL = 2, ERR_POOL_FULL = 4 };

__device__ __forceinline__ uint64_t slot_hash(uint64_t fp) {
    // fingerprints are already xxh64 outputs; fold the high bits in anyway
    return (fp ^ (fp >> 31)) * 0x9E3779B97F4A7C15ULL;
}

// Find or claim the slot of fp. Returns n_slots for the EMPTY-key side slot,
// -1 when the table is full.
__device__ __forceinline__ int64_t find_slot(const irm_store_view &st, uint64_t fp, bool claim) {
    if (fp == IRM_EMPTY_KEY) return st.n_slots;
    const uint64_t m = (uint64_t)st.n_slots - 1;
    uint64_t idx = (slot_hash(fp) >> 17) & m;
    for (int64_t probe = 0; probe < st.n_slots; ++probe, idx = (idx + 1) & m) {
        uint64_t k = ((volatile uint64_t *)st.slot_key)[idx];
        if (k == fp) return (int64_t)idx;
        if (k == IRM_EMPTY_KEY) {
            if (!claim) return -1;
            k = atomicCAS((unsigned long long *)&st.slot_key[idx], (unsigned long long)IRM_EMPTY_KEY,
                          (unsigned long long)fp);
            if (k == IRM_EMPTY_KEY || k == fp) return (int64_t)idx;
        }
    }
    return -1;
}

__global__ void store_reset_kernel(irm_store_view st) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < st.n_slots) st.slot_key[i] = IRM_EMPTY_KEY;
    if (i <= st.n_slots) {
        st.slot_order[i] = INT64_MAX;
        st.slot_entry[i] = -1;
    }
    if (i < 4) st.counters[i] = 0;
}

__global__ void store_claim_kernel(irm_store_view st, const uint64_t *__restrict__ q_fp,
                                   const int64_t *__restrict__ q_order,
                                   const uint8_t *__restrict__ q_probe, int64_t n,
                                   int64_t *__restrict__ q_slot) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (q_probe && !q_probe[i]) {
        q_slot[i] = -2;
        return;
    }
    const int64_t s = find_slot(st, q_fp[i], true);
    q_slot[i] = s;
    if (s < 0) {
        atomicOr((unsigned long long *)&st.counters[2], (unsigned long long)ERR_TABLE_FULL);
        return;
    }
    if (st.slot_entry[s] < 0) atomicMin((long long *)&st.slot_order[s], (long long)q_order[i]);
}

// state per query + per-block totals of (new entries, new rows)
__global__ void __launch_bounds__(ST_BLOCK)
store_decide_kernel(irm_store_view st, const int64_t *__restrict__ q_order,
                    const int32_t *__restrict__ q_len, int64_t n,
                    const int64_t *__restrict__ q_slot, int8_t *__restrict__ q_state,
                    int64_t *__restrict__ blk_cnt, int64_t *__restrict__ blk_rows) {
    __shared__ int64_t sm[ST_BLOCK / 32];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int8_t state = Q_SKIP;
    if (i < n) {
        const int64_t s = q_slot[i];
        if (s >= 0) {
            if (st.slot_entry[s] >= 0) state = Q_HIT_OLD;
            else if (st.slot_order[s] == q_order[i]) state = Q_NOVEL;
            else state = Q_HIT_BATCH;
        }
        q_state[i] = state;
    }
    int64_t tot_c, tot_r;
    block_exclusive_scan<ST_BLOCK>(state == Q_NOVEL ? 1 : 0, &tot_c, sm);
    block_exclusive_scan<ST_BLOCK>(state == Q_NOVEL ? (int64_t)q_len[i] : 0, &tot_r, sm);
    if (threadIdx.x == 0) {
        blk_cnt[blockIdx.x] = tot_c;
        blk_rows[blockIdx.x] = tot_r;
    }
}

// exclusive scan of the block totals (single block, tiles of ST_BLOCK)
__global__ void __launch_bounds__(ST_BLOCK)
store_blockscan_kernel(int64_t nb, int64_t *__restrict__ blk_cnt, int64_t *__restrict__ blk_rows,
                       int64_t *__restrict__ totals) {
    __shared__ int64_t sm[ST_BLOCK / 32];
    int64_t cc = 0, cr = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += ST_BLOCK) {
        const int64_t b = b0 + threadIdx.x;
        const int64_t vc = b < nb ? blk_cnt[b] : 0, vr = b < nb ? blk_rows[b] : 0;
        int64_t tc, tr;
        const int64_t ec = block_exclusive_scan<ST_BLOCK>(vc, &tc, sm);
        const int64_t er = block_exclusive_scan<ST_BLOCK>(vr, &tr, sm);
        if (b < nb) {
            blk_cnt[b] = cc + ec;
            blk_rows[b] = cr + er;
        }
        cc += tc;
        cr += tr;
    }
    if (threadIdx.x == 0) {
        totals[0] = cc;
        totals[1] = cr;
    }
}

__global__ void __launch_bounds__(ST_BLOCK)
store_commit_kernel(irm_store_view st, const uint64_t *__restrict__ q_fp,
                    const int64_t *__restrict__ q_p, const int32_t *__restrict__ q_len, int64_t n,
                    const int64_t *__restrict__ q_slot, const int8_t *__restrict__ q_state,
                    const int64_t *__restrict__ blk_cnt, const int64_t *__restrict__ blk_rows,
                    const int64_t *__restrict__ totals, int32_t *__restrict__ q_hit,
                    int64_t *__restrict__ q_entry, int64_t *__restrict__ q_p_src,
                    int64_t *__restrict__ q_row) {
    __shared__ int64_t sm[ST_BLOCK / 32];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int8_t state = i < n ? q_state[i] : Q_SKIP;
    int64_t tc, tr;
    const int64_t ec = block_exclusive_scan<ST_BLOCK>(state == Q_NOVEL ? 1 : 0, &tc, sm);
    const int64_t er = block_exclusive_scan<ST_BLOCK>(state == Q_NOVEL ? (int64_t)q_len[i] : 0, &tr, sm);
    // counters are bumped only by the resolve kernel, after every commit block
    const int64_t n_before = st.counters[0], rows_before = st.counters[1];
    if (i >= n) return;
    if (state == Q_NOVEL) {
        const int64_t e = n_before + blk_cnt[blockIdx.x] + ec;
        const int64_t row = rows_before + blk_rows[blockIdx.x] + er;
        const int64_t s = q_slot[i];
        // the entry's rows must fit the latent pool (pool_rows 0: unbounded); an entry that
        // does not fit is never published, so nothing ever reads past the pool
        const bool fits = st.pool_rows <= 0 || row + q_len[i] <= st.pool_rows;
        if (e < st.max_entries && fits) {
            st.e_fp[e] = q_fp[i];
            st.e_p_src[e] = q_p[i];
            st.e_len[e] = q_len[i];
            st.e_row[e] = row;
            st.slot_entry[s] = e;
        } else {
            atomicOr((unsigned long long *)&st.counters[2],
                     (unsigned long long)(fits ? ERR_ENTRIES_FULL : ERR_POOL_FULL));
        }
        st.slot_order[s] = INT64_MAX;
        q_hit[i] = 0;
        q_entry[i] = e;
        q_p_src[i] = q_p[i];
        q_row[i] = fits ? row : -1;
    } else if (state == Q_SKIP) {
        q_hit[i] = -1;
        q_entry[i] = -1;
        q_p_src[i] = 0;
        q_row[i] = -1;
    }
}

// hits: resolve after all new entries are published; also bump the counters
__global__ void store_resolve_kernel(irm_store_view st, int64_t n,
                                     const int64_t *__restrict__ q_slot,
                                     const int8_t *__restrict__ q_state,
                                     const int64_t *__restrict__ totals, int32_t *__restrict__ q_hit,
                                     int64_t *__restrict__ q_entry, int64_t *__restrict__ q_p_src,
                                     int64_t *__restrict__ q_row) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        const int64_t ne = st.counters[0] + totals[0];
        st.counters[0] = ne < st.max_entries ? ne : st.max_entries;
        st.counters[1] += totals[1];
    }
    if (i >= n) return;
    const int8_t state = q_state[i];
    if (state != Q_HIT_OLD && state != Q_HIT_BATCH) return;
    const int64_t e = st.slot_entry[q_slot[i]];
    q_hit[i] = 1;
    q_entry[i] = e;
    q_p_src[i] = e >= 0 ? st.e_p_src[e] : 0;
    q_row[i] = e >= 0 ? st.e_row[e] : -1;
}

__global__ void store_lookup_kernel(irm_store_view st, const uint64_t *__restrict__ q_fp, int64_t n,
                                    int64_t *__restrict__ q_entry) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t s = find_slot(st, q_fp[i], false);
    q_entry[i] = s >= 0 ? st.slot_entry[s] : -1;
}

struct StoreWs {
    int64_t *q_slot, *blk_cnt, *blk_rows, *totals;
    int8_t *q_state;
    int64_t bytes;
};

static StoreWs carve_store_ws(void *ws, int64_t n) {
    const int64_t nb = (n + ST_BLOCK - 1) / ST_BLOCK + 1;
    StoreWs w{};
    char *p = (char *)ws;
    int64_t o = 0;
    auto take = [&](int64_t bytes) {
        char *q = p ? p + o : nullptr;
        o = (o + bytes + 255) / 256 * 256;
        return q;
    };
    w.q_slot = (int64_t *)take(n * sizeof(int64_t));
    w.blk_cnt = (int64_t *)take(nb * sizeof(int64_t));
    w.blk_rows = (int64_t *)take(nb * sizeof(int64_t));
    w.totals = (int64_t *)take(2 * sizeof(int64_t));
    w.q_state = (int8_t *)take(n);
    w.bytes = o;
    return w;
}

static int check_view(const irm_store_view *st) {
    IRM_REQUIRE(st != nullptr, "null store view");
    IRM_REQUIRE(st->n_slots >= 2 && (st->n_slots & (st->n_slots - 1)) == 0,
                "n_slots must be a power of two >= 2");
    IRM_REQUIRE(st->slot_key && st->slot_order && st->slot_entry && st->counters,
                "null store arrays");
    IRM_REQUIRE(st->e_fp && st->e_p_src && st->e_len && st->e_row && st->max_entries > 0,
                "null entry arrays");
    return IRM_OK;
}

}  // namespace irm

using namespace irm;

extern "C" int irm_store_reset(const irm_store_view *st, irm_stream_t stream) {
    if (int rc = check_view(st)) return rc;
    const int64_t n = st->n_slots + 1;
    store_reset_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*st);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int64_t irm_store_workspace_bytes(int64_t n) {
    if (n < 0) return -1;
    return carve_store_ws(nullptr, n).bytes;
}

extern "C" int irm_store_lookup_insert(const irm_store_view *st, const uint64_t *q_fp,
                                       const int64_t *q_order, const int64_t *q_p,
                                       const int32_t *q_len, const uint8_t *q_probe, int64_t n,
                                       int32_t *q_hit, int64_t *q_entry, int64_t *q_p_src,
                                       int64_t *q_row, void *ws, int64_t ws_bytes,
                                       irm_stream_t stream) {
    if (int rc = check_view(st)) return rc;
    IRM_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return IRM_OK;
    IRM_REQUIRE(q_fp && q_order && q_p && q_len && q_hit && q_entry && q_p_src && q_row,
                "null query arrays");
    StoreWs w = carve_store_ws(ws, n);
    if (!ws || ws_bytes < w.bytes) {
        set_error("store workspace %lld < %lld", (long long)ws_bytes, (long long)w.bytes);
        return IRM_ECAPACITY;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned nb = (unsigned)((n + ST_BLOCK - 1) / ST_BLOCK);
    store_claim_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(*st, q_fp, q_order, q_probe, n,
                                                                   w.q_slot);
    IRM_LAUNCH_CHECK();
    store_decide_kernel<<<nb, ST_BLOCK, 0, s>>>(*st, q_order, q_len, n, w.q_slot, w.q_state,
                                                w.blk_cnt, w.blk_rows);
    IRM_LAUNCH_CHECK();
    store_blockscan_kernel<<<1, ST_BLOCK, 0, s>>>(nb, w.blk_cnt, w.blk_rows, w.totals);
    IRM_LAUNCH_CHECK();
    store_commit_kernel<<<nb, ST_BLOCK, 0, s>>>(*st, q_fp, q_p, q_len, n, w.q_slot, w.q_state,
                                                w.blk_cnt, w.blk_rows, w.totals, q_hit, q_entry,
                                                q_p_src, q_row);
    IRM_LAUNCH_CHECK();
    store_resolve_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        *st, n, w.q_slot, w.q_state, w.totals, q_hit, q_entry, q_p_src, q_row);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_store_lookup(const irm_store_view *st, const uint64_t *q_fp, int64_t n,
                                int64_t *q_entry, irm_stream_t stream) {
    if (int rc = check_view(st)) return rc;
    IRM_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return IRM_OK;
    IRM_REQUIRE(q_fp && q_entry, "null query arrays");
    store_lookup_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*st, q_fp, n,
                                                                                      q_entry);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

// ---------------------------------------------------------------- wave plan / hit compaction
// The per-chunk glue around K3 in the warm-serve step (engine.py:181-223 batched over a
// wave): which request owns each chunk slot, its absolute position, whether it is probed
// (carve-out, engine.py:186-189), its global order key; and after the lookup, the hits
// compacted in slot order into K4's work list with their count left on the device.
namespace irm {

__global__ void wave_plan_kernel(const int64_t *__restrict__ chunk_off, int32_t n_req,
                                 const int32_t *__restrict__ start, const int64_t *__restrict__ meta_len,
                                 int64_t cap, int64_t carve, int64_t order0, int64_t *__restrict__ req,
                                 int64_t *__restrict__ p_abs, uint8_t *__restrict__ probe,
                                 int64_t *__restrict__ order) {
    const int64_t total = chunk_off[n_req];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = n_req - 1;  // the last request with chunk_off[r] <= i (clamped)
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(chunk_off + mid) <= i) lo = mid;
            else hi = mid - 1;
        }
        const int64_t p = __ldg(meta_len + lo) + start[i];
        req[i] = lo;
        p_abs[i] = p;
        probe[i] = (i < total && p >= carve) ? 1 : 0;
        order[i] = order0 + i;
    }
}

constexpr int WC_BLOCK = 1024;

__global__ void __launch_bounds__(WC_BLOCK)
wave_compact_kernel(const int32_t *__restrict__ hit, const int64_t *__restrict__ row,
                    const int64_t *__restrict__ req, const int64_t *__restrict__ p_abs,
                    const int64_t *__restrict__ p_src, const int32_t *__restrict__ len, int64_t cap,
                    int64_t req_stride, int64_t *__restrict__ src_out, int64_t *__restrict__ dst_out,
                    int32_t *__restrict__ len_out, int64_t *__restrict__ delta_out, int64_t *__restrict__ n_hit,
                    int32_t *__restrict__ length_out, int64_t *__restrict__ hit_tokens,
                    unsigned long long *__restrict__ status) {
    __shared__ int64_t sm[WC_BLOCK / 32];
    int64_t base = 0, tokens = 0;
    for (int64_t i0 = 0; i0 < cap; i0 += WC_BLOCK) {
        const int64_t i = i0 + threadIdx.x;
        const int32_t l = i < cap ? len[i] : 0;
        bool h = i < cap && hit[i] == 1;
        if (h && (p_abs[i] < 0 || p_abs[i] + l > req_stride)) {  // would spill into the next request's rows
            h = false;
            if (status) atomicOr(status, 4ULL);
        }
        if (i < cap) length_out[i] = h ? l : 0;
        int64_t tot;
        const int64_t k = base + block_exclusive_scan<WC_BLOCK>(h ? 1 : 0, &tot, sm);
        if (h) {
            const int64_t pa = p_abs[i];
            src_out[k] = row[i];
            dst_out[k] = req[i] * req_stride + pa;
            len_out[k] = l;
            delta_out[k] = pa - p_src[i];
            tokens += l;
        }
        base += tot;
    }
    int64_t ttot;
    block_exclusive_scan<WC_BLOCK>(tokens, &ttot, sm);
    if (threadIdx.x == 0) {
        *n_hit = base;
        if (hit_tokens) *hit_tokens += ttot;
    }
}

// Phase 1 -> phase 2 on the device (engine.py:170-179): request r's tail is
// tok[off[r] + m[r], off[r+1]) where m[r] is the K0 prefix match; the tails are
// packed into one CSR stream set for K1, and the request's marker spans
// (request-relative [s, e)) become tail-relative pins: spans with e - 1 >= m only, rebased to
// (max(s - m, 0), e - m), each pinning start - 1 (if > 0) and end - 1
// (chunking.py:149-161); a dropped pin is -1, which K1 ignores.
__global__ void __launch_bounds__(WC_BLOCK)
wave_rebase_plan_kernel(const int64_t *__restrict__ off, const int64_t *__restrict__ m, int32_t n_req,
                        const int64_t *__restrict__ span_off, const int64_t *__restrict__ spans,
                        int64_t *__restrict__ tail_off, int64_t *__restrict__ pin_off, int64_t *__restrict__ pins) {
    __shared__ int64_t sm[WC_BLOCK / 32];
    int64_t base = 0;
    for (int32_t r0 = 0; r0 < n_req; r0 += WC_BLOCK) {
        const int32_t r = r0 + threadIdx.x;
        const int64_t len = r < n_req ? max(off[r + 1] - off[r] - m[r], (int64_t)0) : 0;
        int64_t tot;
        const int64_t ex = block_exclusive_scan<WC_BLOCK>(len, &tot, sm);
        if (r < n_req) {
            tail_off[r] = base + ex;
            pin_off[r] = 2 * span_off[r];
            const int64_t mr = m[r];
            for (int64_t k = span_off[r]; k < span_off[r + 1]; ++k) {
                const int64_t s = spans[2 * k], e = spans[2 * k + 1];  // request-relative [s, e)
                const bool keep = e - 1 >= mr;
                const int64_t rs = max(s - mr, (int64_t)0), re = e - mr;
                pins[2 * k] = keep && rs > 0 ? rs - 1 : -1;
                pins[2 * k + 1] = keep ? re - 1 : -1;
            }
        }
        base += tot;
    }
    if (threadIdx.x == 0) {
        tail_off[n_req] = base;
        pin_off[n_req] = 2 * span_off[n_req];
    }
}

__global__ void wave_rebase_copy_kernel(const uint32_t *__restrict__ tok, const int64_t *__restrict__ off,
                                        const int64_t *__restrict__ m, int32_t n_req, int64_t cap,
                                        const int64_t *__restrict__ tail_off, uint32_t *__restrict__ tail) {
    const int64_t total = off[n_req];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < min(total, cap);
         i += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = n_req - 1;  // the request holding token i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(off + mid) <= i) lo = mid;
            else hi = mid - 1;
        }
        const int64_t j = i - off[lo] - m[lo];
        if (j >= 0) tail[tail_off[lo] + j] = tok[i];
    }
}

}  // namespace irm

extern "C" int irm_wave_rebase(const uint32_t *tok, const int64_t *off, const int64_t *m, int32_t n_req, int64_t cap,
                               const int64_t *span_off, const int64_t *spans, uint32_t *tail, int64_t *tail_off,
                               int64_t *pin_off, int64_t *pins, irm_stream_t stream) {
    IRM_REQUIRE(n_req >= 1 && cap >= 0, "bad sizes");
    IRM_REQUIRE(tok && off && m && span_off && tail && tail_off && pin_off, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    irm::wave_rebase_plan_kernel<<<1, irm::WC_BLOCK, 0, s>>>(off, m, n_req, span_off, spans, tail_off, pin_off, pins);
    IRM_LAUNCH_CHECK();
    const int64_t grid = std::min<int64_t>((cap + 255) / 256, (int64_t)irm::sm_count() * 8);
    irm::wave_rebase_copy_kernel<<<(unsigned)std::max<int64_t>(grid, 1), 256, 0, s>>>(tok, off, m, n_req, cap, tail_off,
                                                                                      tail);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_wave_plan(const int64_t *chunk_off, int32_t n_req, const int32_t *start,
                             const int64_t *meta_len, int64_t cap, int64_t carve, int64_t order0, int64_t *req,
                             int64_t *p_abs, uint8_t *probe, int64_t *order, irm_stream_t stream) {
    IRM_REQUIRE(n_req >= 1 && cap >= 0, "bad sizes");
    if (cap == 0) return IRM_OK;
    IRM_REQUIRE(chunk_off && start && meta_len && req && p_abs && probe && order, "null pointer");
    const int64_t grid = std::min<int64_t>((cap + 255) / 256, (int64_t)irm::sm_count() * 4);
    irm::wave_plan_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(chunk_off, n_req, start, meta_len, cap,
                                                                            carve, order0, req, p_abs, probe, order);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_wave_compact(const int32_t *hit, const int64_t *row, const int64_t *req, const int64_t *p_abs,
                                const int64_t *p_src, const int32_t *len, int64_t cap, int64_t req_stride,
                                int64_t *src_out, int64_t *dst_out, int32_t *len_out, int64_t *delta_out,
                                int64_t *n_hit, int32_t *length_out, int64_t *hit_tokens, uint64_t *status,
                                irm_stream_t stream) {
    IRM_REQUIRE(cap >= 0 && req_stride >= 0, "bad sizes");
    IRM_REQUIRE(n_hit && (cap == 0 || (hit && row && req && p_abs && p_src && len && src_out && dst_out &&
                                       len_out && delta_out && length_out)),
                "null pointer");
    irm::wave_compact_kernel<<<1, irm::WC_BLOCK, 0, (cudaStream_t)stream>>>(
        hit, row, req, p_abs, p_src, len, cap, req_stride, src_out, dst_out, len_out, delta_out, n_hit, length_out,
        hit_tokens, (unsigned long long *)status);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}
