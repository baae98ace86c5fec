/*
 * irminsul_b200.h -- C ABI of the B200-native cache-reattach hot path.
 *
 * The reference (Irminsul, /root/reference/pkg/src/irminsul) is a pure-Python
 * package with no FFI; its "operator API" is a set of module functions. Each
 * entry point below is the batched, device-resident replacement for one of
 * them (file:line cited per function). The Python drop-in modules in
 * paper_2605_05696_b200/ bind these through ctypes with the reference's own
 * signatures.
 *
 * Conventions
 *  - Every pointer argument is DEVICE memory owned by the caller (torch
 *    tensors), unless the name ends in _h. No entry point allocates.
 *  - Every call is asynchronous on `stream` (a cudaStream_t) and returns
 *    IRM_OK (0), IRM_EINVAL (1: bad argument -> ValueError), IRM_ECUDA
 *    (2: CUDA error -> RuntimeError) or IRM_ECAPACITY (3: output/workspace
 *    too small -> ValueError). irm_last_error() gives a message.
 *  - Entry points are re-entrant across streams; calls that mutate one store
 *    must be ordered on one stream by the caller (single-writer, like
 *    registry.py:95-101).
 */
#ifndef IRMINSUL_B200_H
#define IRMINSUL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *irm_stream_t; /* == cudaStream_t */

#define IRM_OK 0
#define IRM_EINVAL 1
#define IRM_ECUDA 2
#define IRM_ECAPACITY 3

#define IRM_FORCED_NONE 0       /* chunking.py:31 Forced.NONE */
#define IRM_FORCED_MAX_CLAMP 1  /* chunking.py:32 */
#define IRM_FORCED_MARKER 2     /* chunking.py:33 */
#define IRM_FORCED_STREAM_END 3 /* chunking.py:34 */

#define IRM_LAYOUT_HALF_SPLIT 0  /* rotary.py:98-108 (DSv3-form, reference) */
#define IRM_LAYOUT_INTERLEAVED 1 /* DSv2-form: pairs (2j, 2j+1) */

#define IRM_DTYPE_F64 0
#define IRM_DTYPE_F32 1
#define IRM_DTYPE_BF16 2

#define IRM_ROUND_NONE 0 /* rotary.py:90-95 _store(): F64 */
#define IRM_ROUND_F32 1  /*                            F32 */
#define IRM_ROUND_BF16 2 /*                            BF16E (single RNE rounding) */

int irm_abi_version(void);
const char *irm_last_error(void);
int irm_device_sm_count(void);
/* Kernels this library has launched (or recorded into a CUDA graph being
 * captured) in this process: the caller's evidence of its own GPU launches. */
int64_t irm_launch_count(void);

/* ---- constants (rng.py:17-38, chunking.py:64-86) ---------------------- */
/* Gear table: out[i] = splitmix64 output i+1 of `seed`, 65,536 entries.
 * Replaces chunking.build_gear_table / gear_table (chunking.py:64-76). */
int irm_gear_table(uint64_t seed, uint64_t *out, irm_stream_t stream);

/* ---- K1: CDC + xxh64 (chunking.py:89-133 + fingerprint.py:28-30) -------
 * tok:        all streams' u32 tokens, concatenated.
 * stream_off: [n_streams+1] token offsets (int64).
 * pin_off:    [n_streams+1] offsets into pins; pins of one stream are
 *             stream-relative token indices, sorted ascending (duplicates and
 *             out-of-range values allowed: they never match, like `t in
 *             markers`). A pin forces a boundary after token t and resets the
 *             rolling state (chunking.py:116-118). marker_pinned=0 ignores them.
 * Outputs (dense, stream-major, chunk order): c_start (stream-relative),
 * c_len, c_fp, c_forced; chunk_off[n_streams+1] gets the per-stream CSR
 * offsets (chunk_off[n_streams] = total chunks).
 * cap must be >= irm_cdc_chunk_bound(); ws_bytes >= irm_cdc_workspace_bytes(). */
int64_t irm_cdc_chunk_bound(int64_t n_tokens, int32_t n_streams, int64_t n_pins, int32_t min_size);
int64_t irm_cdc_workspace_bytes(int64_t n_tokens, int32_t n_streams, int64_t n_pins, int32_t min_size);
int irm_cdc_xxh64(const uint32_t *tok, int64_t n_tokens, const int64_t *stream_off,
                  int32_t n_streams, const int64_t *pin_off, const int64_t *pins, int64_t n_pins,
                  int32_t mask_exponent, int32_t min_size, int32_t max_size, int32_t marker_pinned,
                  const uint64_t *gear, int32_t *c_start, int32_t *c_len, uint64_t *c_fp,
                  uint8_t *c_forced, int64_t *chunk_off, int64_t cap, void *ws, int64_t ws_bytes,
                  irm_stream_t stream);
/* The same, with the Gear table given by its generating seed (ChunkerParams.gear_seed,
 * chunking.py:42,64-66): g_t = splitmix64 output (tok & 0xFFFF) + 1 of gear_seed is
 * computed in the kernel instead of read from a table (identical results). */
int irm_cdc_xxh64_seeded(const uint32_t *tok, int64_t n_tokens, const int64_t *stream_off,
                         int32_t n_streams, const int64_t *pin_off, const int64_t *pins, int64_t n_pins,
                         int32_t mask_exponent, int32_t min_size, int32_t max_size, int32_t marker_pinned,
                         uint64_t gear_seed, int32_t *c_start, int32_t *c_len, uint64_t *c_fp,
                         uint8_t *c_forced, int64_t *chunk_off, int64_t cap, void *ws, int64_t ws_bytes,
                         irm_stream_t stream);

/* ---- K2: batched xxh64 over byte spans (fingerprint.py:24-50) ----------
 * out[i] = XXH64(base + off[i], len[i] bytes, seed). Token spans: off/len x4. */
int irm_xxh64_spans(const uint8_t *base, const int64_t *off, const int64_t *len, int64_t n,
                    uint64_t seed, uint64_t *out, irm_stream_t stream);

/* ---- Ingest: JSONL traces -> flattened token CSR (host; model.py:80-170) ----
 * Lines split on \n, \r\n and \r when universal_newlines (a text file), on \n
 * only otherwise (an in-memory stream). irm_trace_scan validates every record
 * exactly as model._parse_request does
 * (same error precedence; on IRM_EINVAL err_line / err_field name the line and
 * field, irm_last_error() the message) and writes sizes[4] = {requests, tokens,
 * segments, string bytes}. irm_trace_fill then writes, in caller buffers:
 *   tokens [tokens] u32           the flattened request tokens (flatten, :80-87)
 *   req_tok_off / req_seg_off [requests + 1], req_turn [requests]
 *   req_session [2 x requests]    (offset, length) of session_id in strings
 *   seg_kind [segments]           index into system, header, history, tool, doc,
 *                                 marker, body, other
 *   seg_tok_off [segments]        start of the segment within its request
 *   seg_shared [2 x segments]     (offset, length) of shared_id, offset -1 = null
 *   strings [string bytes]        UTF-8 */
int irm_trace_scan(const char *text, int64_t len, int32_t universal_newlines, int64_t *sizes, int64_t *err_line,
                   char *err_field, int32_t field_cap);
int irm_trace_fill(const char *text, int64_t len, int32_t universal_newlines, uint32_t *tokens, int64_t *req_tok_off,
                   int64_t *req_seg_off,
                   int64_t *req_turn, int64_t *req_session, uint8_t *seg_kind, int64_t *seg_tok_off,
                   int64_t *seg_shared, char *strings);

/* ---- K0: exact-prefix index (radix.py:31-89; engine.py:170, 228) -------
 * Every prefix of every inserted sequence is a key of an open-addressing
 * table holding the smallest insert epoch that reaches it (the radix tree's
 * earliest-inserted witness). Caller-owned; initialise with irm_prefix_reset(). */
typedef struct {
    uint64_t *slots;      /* [2 x n_slots] slot i = (slots[2i] prefix key or
                           IRM_EMPTY_KEY, slots[2i+1] (int64) the smallest insert
                           epoch with this prefix): key and epoch share one 32-B
                           sector, so an insert is one random DRAM access        */
    int64_t n_slots;      /* power of two, >= 2 x the distinct prefixes stored  */
    int64_t *counters;    /* [2]: slots used, flags (1 table full: error; 4 a hash
                           collision was resolved by an exact scan: informational;
                           sticky)                                             */
    uint64_t hash_key;    /* keys the prefix hash (polynomial base and mixing);
                           fixed for the index's life. 1 = degenerate keys (every
                           prefix of one length collides): a test hook for the
                           exact fallback                                      */
} irm_prefix_view;

int irm_prefix_reset(const irm_prefix_view *ix, irm_stream_t stream);
int64_t irm_prefix_workspace_bytes(int64_t n_tokens, int32_t n_seq);
/* A batch of n_seq operations, in order, on sequences tok[seq_off[i],
 * seq_off[i+1]) (seq_off relative to tok; n_tokens = seq_off[n_seq]).
 *   op_insert[i] != 0: insert sequence i with epoch op_epoch[i]
 *     (RadixTree.insert, radix.py:31-58);
 *   op_query[i] != 0 (nullptr: all): m[i] = the longest prefix of sequence i
 *     shared with a sequence inserted with an epoch < op_epoch[i] (before the
 *     batch or earlier in it), wit[i] = the smallest such epoch reaching depth
 *     m[i]; m = 0, wit = -1 when nothing matches (match_prefix, radix.py:60-83).
 * Every answer is checked token by token against the witness's tokens at
 * arena + wit_off[wit] (wit_len[wit] tokens; the caller keeps each inserted
 * sequence there, including this batch's, indexed by epoch); a mismatch (hash
 * collision) is answered again by an exact scan of the sequences with epochs
 * < op_epoch[i] and sets flag 4: answers are always exact. */
int irm_prefix_match_insert(const irm_prefix_view *ix, const uint32_t *tok, const int64_t *seq_off,
                            int32_t n_seq, int64_t n_tokens, const int64_t *op_epoch,
                            const uint8_t *op_insert, const uint8_t *op_query, const uint32_t *arena,
                            const int64_t *wit_off, const int64_t *wit_len, int64_t *m, int64_t *wit,
                            void *ws, int64_t ws_bytes, irm_stream_t stream);

/* Graph-capturable wave form of phase 1 (engine.py:170, 228): append the n_seq
 * sequences tok[seq_off[r], seq_off[r+1]) to the token arena at *arena_used,
 * record wit_off / wit_len for epochs *epoch_next + r, write those epochs to
 * op_epoch (for irm_prefix_match_insert with every op inserting and querying),
 * then advance *arena_used and *epoch_next -- all on the device. A wave that
 * would overflow the arena (arena_cap tokens) or the epoch arrays (wit_cap) is
 * not appended: op_epoch = -1 (nothing matched or inserted) and flag 1. */
int irm_prefix_wave_prepare(const irm_prefix_view *ix, uint32_t *arena, int64_t arena_cap, int64_t *arena_used,
                            int64_t *wit_off, int64_t *wit_len, int64_t wit_cap, int64_t *epoch_next,
                            const uint32_t *tok, const int64_t *seq_off, int32_t n_seq, int64_t *op_epoch,
                            irm_stream_t stream);

/* ---- K3: content-hash chunk store (registry.py:113-140) ----------------
 * Open-addressing table fingerprint -> entry, plus entry arrays, all caller
 * owned. Initialise with irm_store_reset(). First writer wins by the
 * smallest order key (registry.py:128-130 + engine.py's sequential order). */
typedef struct {
    uint64_t *slot_key;   /* [n_slots]   fingerprint or IRM_EMPTY_KEY          */
    int64_t *slot_order;  /* [n_slots+1] batch claim (atomicMin), INT64_MAX idle */
    int64_t *slot_entry;  /* [n_slots+1] entry index or -1; [n_slots] = fp==EMPTY */
    int64_t n_slots;      /* power of two                                       */
    uint64_t *e_fp;       /* [max_entries]                                      */
    int64_t *e_p_src;     /* [max_entries] absolute source position (registry.py:82) */
    int32_t *e_len;       /* [max_entries] chunk length                         */
    int64_t *e_row;       /* [max_entries] first row in the latent pool         */
    int64_t max_entries;
    int64_t *counters;    /* [4]: n_entries, pool rows used, error flags (1 table
                           full, 2 entries full, 4 pool rows exhausted; sticky),
                           reserved                                            */
    int64_t pool_rows;    /* rows of the latent pool new entries are allocated in;
                           an entry whose rows would pass it is not published
                           (flag 4, q_row = -1). 0: unbounded                  */
} irm_store_view;
#define IRM_EMPTY_KEY 0xFFFFFFFFFFFFFFFFULL

int irm_store_reset(const irm_store_view *st, irm_stream_t stream);
/* Batched lookup-or-insert of n queries, given in ascending q_order (the
 * sequential serve order: request, then chunk). For probed queries
 * (q_probe != 0; 0 = carve-out, engine.py:184-196: neither probed nor
 * inserted):
 *   q_hit = 1 and the entry's (p_src, row) if the fingerprint was stored
 *     before the batch or inserted by an earlier query of the batch;
 *   q_hit = 0 if this query is the first writer: a new entry is appended
 *     with p_src = q_p, len = q_len, row = pool rows allocated in order.
 * Unprobed queries get q_hit = -1. */
int64_t irm_store_workspace_bytes(int64_t n);
int irm_store_lookup_insert(const irm_store_view *st, const uint64_t *q_fp,
                            const int64_t *q_order, const int64_t *q_p, const int32_t *q_len,
                            const uint8_t *q_probe, int64_t n, int32_t *q_hit, int64_t *q_entry,
                            int64_t *q_p_src, int64_t *q_row, void *ws, int64_t ws_bytes,
                            irm_stream_t stream);
/* Read-only batched lookup (registry.py:116-117): q_entry = -1 on miss. */
int irm_store_lookup(const irm_store_view *st, const uint64_t *q_fp, int64_t n, int64_t *q_entry,
                     irm_stream_t stream);
/* Warm-serve step glue around K3 (engine.py:181-223 batched over a wave of
 * n_req requests whose chunk table is CSR chunk_off[n_req+1], cap slots):
 * irm_wave_plan gives, per slot i < cap, req[i] = the owning request (clamped
 * to n_req-1 past the end), p_abs[i] = meta_len[req] + start[i], probe[i] =
 * (i < chunk_off[n_req] && p_abs >= carve) (the carve-out, engine.py:186-189),
 * order[i] = order0 + i. irm_wave_compact lists the slots with hit[i] == 1 in
 * slot order as K4 work (src = row, dst = req*req_stride + p_abs, len,
 * delta = p_abs - p_src), n_hit[0] = their count, length_out[i] = len if hit
 * else 0, and adds the hit tokens to *hit_tokens (if not null). A hit whose
 * rows [p_abs, p_abs + len) leave [0, req_stride) is not listed (it would
 * write into the next request's rows) and sets bit 4 of *status (nullable). */
/* Phase 1 -> phase 2 glue (engine.py:170-179): with m[r] the prefix match of
 * request r = tok[off[r], off[r+1]), packs the tails tok[off[r] + m[r], off[r+1])
 * into `tail` (CSR tail_off[n_req+1]; cap = the token capacity of tok) and
 * rebases the request's marker spans (span_off[n_req+1], spans[2k], [2k+1] =
 * request-relative [start, end), ascending) into tail-relative pins (pin_off = 2 span_off):
 * spans with end - 1 >= m only, as (max(start - m, 0), end - m), each pinning
 * start - 1 (if > 0) and end - 1 (marker_pin_offsets, chunking.py:149-161);
 * dropped pins are -1 (ignored by K1). */
int irm_wave_rebase(const uint32_t *tok, const int64_t *off, const int64_t *m, int32_t n_req, int64_t cap,
                    const int64_t *span_off, const int64_t *spans, uint32_t *tail, int64_t *tail_off,
                    int64_t *pin_off, int64_t *pins, irm_stream_t stream);
int irm_wave_plan(const int64_t *chunk_off, int32_t n_req, const int32_t *start, const int64_t *meta_len,
                  int64_t cap, int64_t carve, int64_t order0, int64_t *req, int64_t *p_abs, uint8_t *probe,
                  int64_t *order, irm_stream_t stream);
int irm_wave_compact(const int32_t *hit, const int64_t *row, const int64_t *req, const int64_t *p_abs,
                     const int64_t *p_src, const int32_t *len, int64_t cap, int64_t req_stride, int64_t *src_out,
                     int64_t *dst_out, int32_t *len_out, int64_t *delta_out, int64_t *n_hit, int32_t *length_out,
                     int64_t *hit_tokens, uint64_t *status, irm_stream_t stream);

/* ---- K4: delta-rotation rotate + gather (registry.py:146-166) ----------
 * For each chunk c and layer l: rows [src_row[c], +len[c]) of the pool are
 * copied to rows [dst_row[c], +len[c]) of out. Each row is ckv_dim latent
 * values copied verbatim followed by kr_dim rotary values rotated by
 * R(delta[c]) (angle = delta * inv_freq[j] in fp64, rotary.py:98-108).
 * pool/out element (row r, layer l) at base + (l*layer_stride + r) * row_dim.
 * dtype: element type of pool and out. out_round: IRM_ROUND_* applied to
 * the rotated values (f64 pools only; BF16E/F32 store emulation).
 * n_chunks_dev (nullable): device-side count of the leading chunks to process
 * (<= n_chunks), so a compacted hit list needs no host synchronisation.
 * Bounds: pool_layer_stride / out_layer_stride are the row counts of one layer;
 * a chunk whose source run leaves the pool or whose destination run leaves out
 * is skipped and reported in *status (nullable, sticky OR: 1 source, 2
 * destination) -- never read or written out of range.
 * max_sms: spread the persistent CTAs over at most this many SMs (0 = all), per
 * call, so a CUDA graph captures it with its launch (the reattach pipeline
 * leaves ~20 SMs to CDC/lookup of the next wave running concurrently; the
 * gather holds the HBM roofline down to ~120 SMs, profiles/r01d_k4_sms.md). */
int64_t irm_rotate_gather_workspace_bytes(int64_t n_chunks, int32_t kr_dim);
int irm_rotate_gather(const void *pool, int64_t pool_layer_stride, void *out,
                      int64_t out_layer_stride, int32_t layers, int32_t ckv_dim, int32_t kr_dim,
                      const int64_t *src_row, const int64_t *dst_row, const int32_t *len,
                      const int64_t *delta, int64_t n_chunks, const int64_t *n_chunks_dev,
                      const double *inv_freq, int32_t layout, int32_t dtype, int32_t out_round,
                      int32_t max_sms, uint64_t *status, void *ws, int64_t ws_bytes, irm_stream_t stream);
/* K4 fan-out form. materialize (registry.py:146-166) is a pure function of
 * (entry, p_dest): when several hits of a wave share a source run, its rows are
 * read from HBM once and written once per destination.
 * irm_group_by_source: the first n = min(n, *n_dev) (n_dev nullable) K4 work
 * items (src_row, dst_row, len, delta, e.g. irm_wave_compact's output) grouped
 * by source run (src_row, len): group g = (g_src, g_len, g_first, g_count), its
 * members m_dst / m_delta[g_first .. g_first + g_count); groups in the order of
 * their first item; *n_groups = the group count (device). ws: at least
 * irm_group_workspace_bytes(n) bytes, ZERO-FILLED before the first call; every
 * call leaves it zeroed. n < 2^31.
 * irm_rotate_gather_fanout: for each group g < min(n_groups, *n_groups_dev),
 * layer l and member m: rows [g_src, +g_len) of the pool -> rows [m_dst,
 * +g_len) of out, c_KV verbatim, k_r rotated by R(m_delta) (fp64 angle, fp32
 * rotation), bf16 or f32 pools, kr_dim a multiple of 4. n_members(_dev) bounds
 * the member table; ws at
 * least irm_fanout_workspace_bytes(n_members, kr_dim). Bounds, status and
 * max_sms as irm_rotate_gather. Items are handed out dynamically (an atomic
 * counter in ws). cta_rounds > 1: the grid is cta_rounds x the resident CTAs and
 * each CTA retires after its share of the items, so kernels of a higher-priority
 * stream (the next wave's front in the reattach pipeline) get SMs in between. */
int64_t irm_group_workspace_bytes(int64_t n);
int irm_group_by_source(const int64_t *src_row, const int64_t *dst_row, const int32_t *len, const int64_t *delta,
                        int64_t n, const int64_t *n_dev, int64_t *g_src, int32_t *g_len, int32_t *g_first,
                        int32_t *g_count, int64_t *m_dst, int64_t *m_delta, int64_t *n_groups, void *ws,
                        int64_t ws_bytes, irm_stream_t stream);
int64_t irm_fanout_workspace_bytes(int64_t n_members, int32_t kr_dim);
int irm_rotate_gather_fanout(const void *pool, int64_t pool_layer_stride, void *out, int64_t out_layer_stride,
                             int32_t layers, int32_t ckv_dim, int32_t kr_dim, const int64_t *g_src,
                             const int32_t *g_len, const int32_t *g_first, const int32_t *g_count, int64_t n_groups,
                             const int64_t *n_groups_dev, const int64_t *m_dst, const int64_t *m_delta,
                             int64_t n_members, const int64_t *n_members_dev, const double *inv_freq,
                             int32_t layout, int32_t dtype, int32_t max_sms, int32_t cta_rounds, uint64_t *status,
                             void *ws, int64_t ws_bytes, irm_stream_t stream);
/* K6 replica fetch: for run c < min(n_runs, *n_runs_dev), copy len[c] rows of
 * row_bytes from src_addr[c] + l * src_layer_stride (a device address, normally
 * inside a peer GPU's pool mapped through CUDA IPC over NVLink) to
 * dst + l * dst_layer_stride + dst_row[c] * row_bytes, for every layer l.
 * Replaces the reference's in-process dict sharing of registry rows
 * (registry.py:126-140) when the store is sharded across GPUs. */
int irm_copy_runs(const int64_t *src_addr, int64_t src_layer_stride, void *dst, int64_t dst_layer_stride,
                  const int64_t *dst_row, const int32_t *len, int64_t n_runs, const int64_t *n_runs_dev,
                  int32_t layers, int32_t row_bytes, irm_stream_t stream);
/* Peer pool mapping for irm_copy_runs: irm_peer_export writes the
 * IRM_PEER_HANDLE_BYTES-byte IPC handle of the device allocation holding `ptr` and
 * the byte offset of `ptr` in it; another process on any GPU of the node passes
 * both to irm_peer_open, which maps the allocation on the caller's CURRENT device
 * (peer access over NVLink enabled lazily) and returns the address of `ptr` there.
 * Mappings live until the process exits. Replaces the reference's in-process
 * sharing of registry rows (registry.py:126-140). */
#define IRM_PEER_HANDLE_BYTES 64
int irm_peer_export(const void *ptr, void *handle, int64_t *offset);
int irm_peer_open(const void *handle, int64_t offset, void **ptr);
/* K6 lookup exchange over the hash-sharded store (replaces the in-process dict
 * of registry.py:113-140 across G GPUs; first writer = smallest order key, as
 * engine.py:197-223 inserts in order). One wave:
 *   irm_exchange_pack: probed query i (q_probe nullptr: all) goes to slot
 *     owner * cap + k of send [world * cap, 4] = (fp, order, p, len), owner =
 *     ((fp >> 32) * world) >> 32, k = its rank among this rank's queries to that
 *     owner (query order); dest[i] = the slot, or -1 (not probed, or the bucket
 *     is full: flags |= 1). Unused slots: order = 2^62 + rank * world * cap + slot.
 *   (all-to-all of the send buffers: recv [world * cap, 4])
 *   irm_exchange_split: recv -> K3 query arrays (real = order < 2^62).
 *   (irm_store_lookup_insert on this rank's shard)
 *   irm_exchange_reply: novel slots of writer w get rows base_row + next[w] + ...
 *     (lengths scanned in slot order; next[w] advances; past region: flags |= 2);
 *     e_grow[entry] = w << 40 | row; reply [world * cap, 4] = (hit, p_src,
 *     e_grow[entry] or -1, fresh = hit on an entry >= *n_before).
 *   (reverse all-to-all: back)
 *   irm_exchange_unpack: back[dest[i]] -> hit / p_src / row / owner / fresh of
 *     query i (dest -1: hit -1, row -1, owner -1).
 * world <= 32. One CTA for pack and reply (deterministic slot order). */
int irm_exchange_pack(const uint64_t *q_fp, const int64_t *q_order, const int64_t *q_p, const int32_t *q_len,
                      const uint8_t *q_probe, int64_t n, int32_t world, int32_t rank, int64_t cap, int64_t *send,
                      int64_t *dest, uint64_t *flags, irm_stream_t stream);
int irm_exchange_split(const int64_t *recv, int64_t m, uint64_t *fp, int64_t *order, int64_t *p, int32_t *len,
                       uint8_t *real, irm_stream_t stream);
int irm_exchange_reply(const int64_t *recv, int32_t world, int64_t cap, const int32_t *hit, const int64_t *entry,
                       const int64_t *p_src, const int64_t *n_before, int64_t base_row, int64_t region, int64_t *next,
                       int64_t *e_grow, int64_t n_egrow, uint64_t *flags, int64_t *reply, irm_stream_t stream);
int irm_exchange_unpack(const int64_t *back, const int64_t *dest, int64_t n, int64_t cap, int32_t *hit,
                        int64_t *p_src, int64_t *row, int64_t *owner, uint8_t *fresh, irm_stream_t stream);
/* Per-row absolute rotation (producer side of the store, registry.py:131-133
 * with rotary.py:98-108): out[i] = R(positions[i]) rows[i] for the dim-wide
 * rotary rows at rows + i*row_stride (elements). out may alias rows. fp64 rows
 * use correctly rounded cos/sin (the reference's f64 values bit for bit). */
int irm_rotate_rows(const void *rows, int64_t row_stride, void *out, int64_t out_stride,
                    int64_t n, int32_t dim, const double *positions, const double *inv_freq,
                    int32_t layout, int32_t dtype, int32_t out_round, irm_stream_t stream);
/* The same over `layers` layers at rows + l*rows_layer_stride (out: out_layer_stride),
 * every layer's row i rotated by positions[i]: cos/sin evaluated once per (row,
 * frequency) -- the batched producer of a multi-layer latent pool. */
int irm_rotate_rows_layered(const void *rows, int64_t row_stride, int64_t rows_layer_stride, void *out,
                            int64_t out_stride, int64_t out_layer_stride, int32_t layers, int64_t n, int32_t dim,
                            const double *positions, const double *inv_freq, int32_t layout, int32_t dtype,
                            int32_t out_round, irm_stream_t stream);
/* Elementwise store rounding of f64 values: IRM_ROUND_F32 (f32 cast) or
 * IRM_ROUND_BF16 (rotary.py:63-87 round_bf16, single RNE incl. subnormals). */
int irm_round_f64(const double *x, double *y, int64_t n, int32_t mode, irm_stream_t stream);

/* ---- K5: fused absorbed-MLA reattach prefill ----
 * No reference implementation exists ("deliberate
 * follow-up"); semantics restated in oracle/mla_ref.py:
 *   S[r,k] = (q[r,:512] . c_KV[k] + q[r,512:] . R(delta_k) kr_base[k]) * scale
 *   causal (key k visible to query position P iff k <= P), O = softmax(S) c_KV
 * q    [n_q, heads, 576] bf16 (absorbed q_nope || rotated q_pe); query i at
 *      position q_pos0 + i (q_pos0 + n_q <= n_kv)
 * pool [pool_rows, 576] bf16 latent rows (c_KV || kr_base); key k at pool
 *      row kv_rows[k] (NULL: row k), gathered by TMA (tile::gather4)
 * kv_chunk [n_kv] chunk of key k and chunk_cs [n_chunks*32] float2 from
 *      irm_chunk_cossin(): k_r is rotated by R(delta) in shared memory on its
 *      way to the tensor cores and never written back (NULL: no rotation)
 * out  [n_q, heads, 512] bf16; lse [n_q, heads] fp32 natural log (nullable) */
int irm_chunk_cossin(const int64_t *delta, int64_t n_chunks, const double *inv_freq, void *cs,
                     irm_stream_t stream);
int irm_mla_reattach_prefill(const void *q, int64_t n_q, int32_t heads, int64_t q_pos0,
                             const void *pool, int64_t pool_rows, const int32_t *kv_rows, int32_t n_kv,
                             const int32_t *kv_chunk, const void *chunk_cs, int32_t layout,
                             float scale, void *out, float *lse, irm_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
