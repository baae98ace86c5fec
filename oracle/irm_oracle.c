/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the cache-reattach hot path.
 *
 * A plain-C restatement of the reference algorithm (Irminsul, pure-Python
 * simulator under /root/reference/pkg/src/irminsul). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product path (paper_2605_05696_b200) never does.
 *
 * Parity is pinned against golden vectors generated from the reference
 * itself (tests/golden/make_golden.py) and the reference's own KATs.
 *
 *   splitmix64      <- src/rng.py:17-24  (splitmix64_next), :27-38 (SplitMix64)
 *   gear table      <- src/chunking.py:64-76
 *   canonical marker<- src/chunking.py:79-86
 *   xxh64           <- src/fingerprint.py:24-30 -> python-xxhash 3.7.0
 *                      (bundled libxxhash 0.8.2, XXH64, seed 0); restated from
 *                      the published XXH64 specification
 *   cdc_chunk       <- src/chunking.py:89-133 (hot loop 113-128)
 *   materialize     <- src/registry.py:146-166 + src/rotary.py:98-108
 *                      (bf16 pool variant used as the CPU baseline arm)
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>
#include <pthread.h>
#include <unistd.h>

/* Minimal dynamic parallel-for over [0, n) on pthreads (no OpenMP runtime in
 * this image). Work items are claimed one at a time from an atomic counter. */
typedef void (*par_body_fn)(int64_t i, void *ctx);
typedef struct { int64_t n; int64_t next; par_body_fn fn; void *ctx; } par_job;
static void *par_worker(void *arg) {
    par_job *j = (par_job *)arg;
    for (;;) {
        int64_t i = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (i >= j->n) break;
        j->fn(i, j->ctx);
    }
    return NULL;
}
static void par_for(int64_t n, int32_t n_threads, par_body_fn fn, void *ctx) {
    if (n_threads <= 0) n_threads = (int32_t)sysconf(_SC_NPROCESSORS_ONLN);
    if (n_threads > 256) n_threads = 256;
    if (n_threads > n) n_threads = (int32_t)(n > 0 ? n : 1);
    par_job job = {n, 0, fn, ctx};
    pthread_t th[256];
    for (int32_t t = 1; t < n_threads; ++t) pthread_create(&th[t], NULL, par_worker, &job);
    par_worker(&job);
    for (int32_t t = 1; t < n_threads; ++t) pthread_join(th[t], NULL);
}

#define GEAR_SIZE 65536

/* ---------------- splitmix64 (src/rng.py:17-24) ---------------- */
static inline uint64_t sm64_next(uint64_t *state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void oracle_splitmix64_fill(uint64_t seed, int64_t n, uint64_t *out) {
    uint64_t s = seed;
    for (int64_t i = 0; i < n; ++i) out[i] = sm64_next(&s);
}

/* src/rng.py:41-51 */
uint64_t oracle_derive_seed(uint64_t seed, const uint64_t *labels, int32_t n) {
    uint64_t state = seed;
    for (int32_t i = 0; i < n; ++i) {
        state ^= labels[i];
        uint64_t s2 = state;
        state = sm64_next(&s2);  /* returns output, not the advanced state */
    }
    return state;
}

/* src/chunking.py:64-66 */
void oracle_gear_table(uint64_t seed, uint64_t *out) {
    oracle_splitmix64_fill(seed, GEAR_SIZE, out);
}

/* src/chunking.py:79-86: SplitMix64(SplitMix64(seed ^ 64).next_u64()).fill(64) & 0xFFFFFFFF */
void oracle_canonical_marker(uint64_t seed, uint32_t *out) {
    uint64_t s = seed ^ 64ULL;
    uint64_t s2 = sm64_next(&s);
    for (int i = 0; i < 64; ++i) out[i] = (uint32_t)(sm64_next(&s2) & 0xFFFFFFFFULL);
}

/* ---------------- XXH64 (libxxhash 0.8.2 semantics) ---------------- */
#define P1 0x9E3779B185EBCA87ULL
#define P2 0xC2B2AE3D27D4EB4FULL
#define P3 0x165667B19E3779F9ULL
#define P4 0x85EBCA77C2B2AE63ULL
#define P5 0x27D4EB2F165667C5ULL

static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
static inline uint64_t rd64(const uint8_t *p) { uint64_t v; memcpy(&v, p, 8); return v; }
static inline uint32_t rd32(const uint8_t *p) { uint32_t v; memcpy(&v, p, 4); return v; }
static inline uint64_t xround(uint64_t acc, uint64_t in) {
    acc += in * P2; acc = rotl64(acc, 31); return acc * P1;
}
static inline uint64_t xmerge(uint64_t acc, uint64_t v) {
    v = xround(0, v); acc ^= v; return acc * P1 + P4;
}

uint64_t oracle_xxh64(const uint8_t *p, int64_t len, uint64_t seed) {
    const uint8_t *end = p + len;
    uint64_t h;
    if (len >= 32) {
        const uint8_t *limit = end - 32;
        uint64_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
        do {
            v1 = xround(v1, rd64(p)); v2 = xround(v2, rd64(p + 8));
            v3 = xround(v3, rd64(p + 16)); v4 = xround(v4, rd64(p + 24));
            p += 32;
        } while (p <= limit);
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = xmerge(h, v1); h = xmerge(h, v2); h = xmerge(h, v3); h = xmerge(h, v4);
    } else {
        h = seed + P5;
    }
    h += (uint64_t)len;
    while (p + 8 <= end) { h ^= xround(0, rd64(p)); h = rotl64(h, 27) * P1 + P4; p += 8; }
    if (p + 4 <= end) { h ^= (uint64_t)rd32(p) * P1; h = rotl64(h, 23) * P2 + P3; p += 4; }
    while (p < end) { h ^= (uint64_t)(*p) * P5; h = rotl64(h, 11) * P1; ++p; }
    h ^= h >> 33; h *= P2; h ^= h >> 29; h *= P3; h ^= h >> 32;
    return h;
}

/* src/fingerprint.py:28-30: xxh64 seed 0 over the LE u32 encoding (x86 is LE) */
uint64_t oracle_fingerprint(const uint32_t *tok, int64_t n) {
    return oracle_xxh64((const uint8_t *)tok, 4 * n, 0);
}

/* ---------------- CDC (src/chunking.py:89-133) ----------------
 * pins: sorted ascending, duplicates allowed, any values (out-of-range ones
 * never match a token index, exactly like `t in markers`).
 * forced codes: 0 none, 1 max_clamp, 2 marker, 3 stream_end (Forced enum order).
 * Returns the number of chunks, or -1 if cap is exceeded. */
int64_t oracle_cdc_chunk(const uint32_t *tok, int64_t n, const int64_t *pins, int64_t n_pins,
                         int32_t k, int32_t min_size, int32_t max_size, const uint64_t *gear,
                         int32_t *c_start, int32_t *c_len, uint64_t *c_fp, uint8_t *c_forced,
                         int64_t cap) {
    if (n == 0) return 0;
    const uint64_t mask = (1ULL << k) - 1;
    uint64_t h = 0;
    int64_t start = 0, nc = 0, pi = 0;
    while (pi < n_pins && pins[pi] < 0) ++pi;
    for (int64_t t = 0; t < n; ++t) {
        h = rotl64(h, 1) + gear[tok[t] & 0xFFFF];
        int64_t since = t - start + 1;
        int forced;
        while (pi < n_pins && pins[pi] < t) ++pi;
        if (pi < n_pins && pins[pi] == t) { forced = 2; h = 0; }
        else if (since == max_size) forced = 1;
        else if (since >= min_size && (h & mask) == 0) forced = 0;
        else continue;
        if (nc >= cap) return -1;
        c_start[nc] = (int32_t)start; c_len[nc] = (int32_t)since;
        c_fp[nc] = oracle_fingerprint(tok + start, since); c_forced[nc] = (uint8_t)forced;
        ++nc; start = t + 1;
    }
    if (start < n) {
        if (nc >= cap) return -1;
        c_start[nc] = (int32_t)start; c_len[nc] = (int32_t)(n - start);
        c_fp[nc] = oracle_fingerprint(tok + start, n - start); c_forced[nc] = 3; ++nc;
    }
    return nc;
}

/* Per-token rolling state h_t (for white-box tests of the scan decomposition). */
void oracle_gear_states(const uint32_t *tok, int64_t n, const int64_t *pins, int64_t n_pins,
                        const uint64_t *gear, uint64_t *h_out) {
    uint64_t h = 0; int64_t pi = 0;
    for (int64_t t = 0; t < n; ++t) {
        h = rotl64(h, 1) + gear[tok[t] & 0xFFFF];
        h_out[t] = h;
        while (pi < n_pins && pins[pi] < t) ++pi;
        if (pi < n_pins && pins[pi] == t) h = 0;
    }
}

/* Batched CDC over CSR streams, threaded across streams (the CPU baseline arm).
 * Chunks of stream s go to [out_off[s], out_off[s+1]) (a caller bound, e.g.
 * n_s/min_size + 2 + pins); counts[s] receives the chunk count (-1 on overflow). */
typedef struct {
    const uint32_t *tok; const int64_t *stream_off; const int64_t *pin_off; const int64_t *pins;
    int32_t k, min_size, max_size; const uint64_t *gear; const int64_t *out_off;
    int32_t *c_start, *c_len; uint64_t *c_fp; uint8_t *c_forced; int64_t *counts;
} cdc_batch_ctx;
static void cdc_batch_body(int64_t s, void *p) {
    cdc_batch_ctx *c = (cdc_batch_ctx *)p;
    int64_t o = c->out_off[s];
    c->counts[s] = oracle_cdc_chunk(c->tok + c->stream_off[s], c->stream_off[s + 1] - c->stream_off[s],
                                    c->pins + c->pin_off[s], c->pin_off[s + 1] - c->pin_off[s],
                                    c->k, c->min_size, c->max_size, c->gear, c->c_start + o,
                                    c->c_len + o, c->c_fp + o, c->c_forced + o,
                                    c->out_off[s + 1] - o);
}
int64_t oracle_cdc_batch(const uint32_t *tok, const int64_t *stream_off, int32_t n_streams,
                         const int64_t *pin_off, const int64_t *pins,
                         int32_t k, int32_t min_size, int32_t max_size, const uint64_t *gear,
                         const int64_t *out_off, int32_t *c_start, int32_t *c_len,
                         uint64_t *c_fp, uint8_t *c_forced, int64_t *counts, int32_t n_threads) {
    cdc_batch_ctx ctx = {tok, stream_off, pin_off, pins, k, min_size, max_size, gear, out_off,
                         c_start, c_len, c_fp, c_forced, counts};
    par_for(n_streams, n_threads, cdc_batch_body, &ctx);
    int64_t total = 0;
    for (int32_t s = 0; s < n_streams; ++s) total += counts[s] < 0 ? 0 : counts[s];
    return total;
}

/* ---------------- rotate + gather baseline (bf16 pool) ----------------
 * The CPU arm of K4: per hit chunk, copy c_KV (512 bf16) verbatim and rotate
 * k_r (64 bf16, half-split or interleaved) by delta with fp64 angles, fp32 math,
 * bf16 RNE store -- the same work the GPU kernel does, per layer.
 * pool/out: [layers][rows][576] bf16 (row stride 576). */
static inline float bf2f(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }
static inline uint16_t f2bf(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    if ((u & 0x7FFFFFFF) > 0x7F800000) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7FFF + ((u >> 16) & 1);
    return (uint16_t)(u >> 16);
}

typedef struct {
    const uint16_t *pool; int64_t pool_rows; uint16_t *out; int64_t out_rows; int32_t layers;
    const int64_t *src_row, *dst_row; const int32_t *len; const int64_t *delta;
    const double *inv_freq; int32_t interleaved;
} rot_ctx;
static void rot_body(int64_t c, void *p) {
    rot_ctx *x = (rot_ctx *)p;
    float cs[32], sn[32];
    for (int j = 0; j < 32; ++j) {
        double a = (double)x->delta[c] * x->inv_freq[j];
        cs[j] = (float)cos(a); sn[j] = (float)sin(a);
    }
    for (int32_t l = 0; l < x->layers; ++l) {
        for (int32_t i = 0; i < x->len[c]; ++i) {
            const uint16_t *s = x->pool + ((int64_t)l * x->pool_rows + x->src_row[c] + i) * 576;
            uint16_t *d = x->out + ((int64_t)l * x->out_rows + x->dst_row[c] + i) * 576;
            memcpy(d, s, 512 * 2);
            for (int j = 0; j < 32; ++j) {
                int ilo = x->interleaved ? 2 * j : j, ihi = x->interleaved ? 2 * j + 1 : j + 32;
                float lo = bf2f(s[512 + ilo]), hi = bf2f(s[512 + ihi]);
                d[512 + ilo] = f2bf(lo * cs[j] - hi * sn[j]);
                d[512 + ihi] = f2bf(lo * sn[j] + hi * cs[j]);
            }
        }
    }
}
void oracle_rotate_gather_bf16(const uint16_t *pool, int64_t pool_rows, uint16_t *out,
                               int64_t out_rows, int32_t layers, const int64_t *src_row,
                               const int64_t *dst_row, const int32_t *len, const int64_t *delta,
                               int64_t n_chunks, const double *inv_freq, int32_t interleaved,
                               int32_t n_threads) {
    rot_ctx ctx = {pool, pool_rows, out, out_rows, layers, src_row, dst_row, len, delta,
                   inv_freq, interleaved};
    par_for(n_chunks, n_threads, rot_body, &ctx);
}

int32_t oracle_max_threads(void) { return (int32_t)sysconf(_SC_NPROCESSORS_ONLN); }
