// K0: batched exact-prefix index on the device (phase 1 of the serve path).
//
// Replaces RadixTree.insert / match_prefix (reference radix.py:31-89, called
// by engine.serve at engine.py:170 and :228) for a batch of operations. The
// reference walks a compressed radix tree per request; here every prefix of
// every inserted sequence is one key of an open-addressing table:
//
//   key(s, d) = fmix64(H(s[0:d]) + d * phi),  H = polynomial hash mod 2^61 - 1
//   slot value = the smallest insert epoch whose sequence has that prefix
//
// "some sequence inserted before epoch e shares the first d tokens of q" is
// then one lookup (slot epoch < e), and it is monotone in d (a sequence that
// shares d tokens shares every shorter prefix), so the longest match is a
// binary search over d. The earliest-inserted witness at that depth is the
// slot's epoch (radix.py:85-89 keeps the earliest handle on every node).
// All prefix hashes of a batch come from one segmented scan of affine maps
// x -> B x + (t + 1) (mod 2^61 - 1), so the work is O(tokens) and parallel.
//
// The hash is keyed per index (irm_prefix_view.hash_key: the polynomial base
// and the key mixing both derive from it; the Python index draws it from
// os.urandom), so colliding token sequences cannot be prepared offline.
//
// Exactness: a hash collision could only make a prefix look present. The
// final answer of every query is verified token by token against the
// witness's stored tokens; on a mismatch the query is answered again by an
// exact scan of every sequence inserted before it (longest common prefix,
// earliest epoch on ties, radix.py:60-89) and flag 4 records that a collision
// was resolved. A colliding slot therefore costs a scan, never a wrong answer
// and never an error. Deeper-prefix false negatives cannot happen.
#include "common.cuh"

namespace irm {
namespace prefix {

constexpr uint64_t P61 = (1ULL << 61) - 1;
constexpr int CH = 1024;       // tokens per chunk (one CTA)
constexpr int PT = 256;        // threads per CTA
constexpr int TPT = CH / PT;   // tokens per thread
enum : int64_t { ERR_TABLE_FULL = 1, ERR_VERIFY = 2, COLLISION_RESOLVED = 4 };
constexpr uint64_t DEGENERATE_KEY = 1;  // test hook: every prefix of one length collides

struct Aff {  // x -> a x + b (mod p)
    uint64_t a, b;
};

__device__ __forceinline__ uint64_t mulmod(uint64_t x, uint64_t y) {
    const uint64_t lo = x * y, hi = __umul64hi(x, y);
    uint64_t r = (lo & P61) + ((lo >> 61) | (hi << 3));
    r = (r & P61) + (r >> 61);
    return r >= P61 ? r - P61 : r;
}
__device__ __forceinline__ uint64_t addmod(uint64_t x, uint64_t y) {
    const uint64_t r = x + y;
    return r >= P61 ? r - P61 : r;
}
// f then g
__device__ __forceinline__ Aff compose(Aff f, Aff g) { return {mulmod(f.a, g.a), addmod(mulmod(g.a, f.b), g.b)}; }
__device__ __forceinline__ Aff tok_aff(uint32_t t, uint64_t base) { return {base, (uint64_t)t + 1}; }

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
// the polynomial base of this index, in [2, p - 1)
__device__ __forceinline__ uint64_t key_base(uint64_t hash_key) { return 2 + splitmix(hash_key) % (P61 - 3); }

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDULL;
    k ^= k >> 33;
    k *= 0xC4CEB9FE1A85EC53ULL;
    k ^= k >> 33;
    return k;
}
__device__ __forceinline__ uint64_t prefix_key(uint64_t h, int64_t d, uint64_t hash_key) {
    if (hash_key == DEGENERATE_KEY) h = 0;
    const uint64_t k = fmix64((h ^ splitmix(hash_key ^ 0x5851F42D4C957F2DULL)) + (uint64_t)d * 0x9E3779B97F4A7C15ULL);
    return k == IRM_EMPTY_KEY ? k - 1 : k;
}

__device__ __forceinline__ uint64_t *slot_key(const irm_prefix_view &ix, uint64_t i) { return ix.slots + 2 * i; }
__device__ __forceinline__ long long *slot_epoch(const irm_prefix_view &ix, uint64_t i) {
    return reinterpret_cast<long long *>(ix.slots + 2 * i + 1);
}

// Slot placement. The keys of depths 64b + 1 .. 64b + 64 of a sequence share the home
// region of the key of its prefix of length 64b (a constant for b = 0): home(d) = region +
// (d - 1) % 64, a 1 KB run of slots, so inserting a sequence writes consecutive slots (DRAM
// rows, not one random sector per token) and a query's binary search lands in the same runs.
// Probe sequence of a key: its home slot, then the same offset in a second region chosen by
// the region key (another block that took the home region: the block's keys move on together
// and stay contiguous), then double hashing by the key itself (sequences diverging inside
// one block -- e.g. every request after a shared header -- scatter instead of queueing behind
// each other). The sequence is fixed by (region key, depth, key), so lookups follow the
// inserts exactly; the first empty slot ends a search (there are no deletions).
constexpr int REGION = 64;
__device__ __forceinline__ uint64_t region_base0(uint64_t hash_key) { return splitmix(hash_key ^ 0xD1B54A32D192ED03ULL); }
__device__ __forceinline__ uint64_t home_slot(const irm_prefix_view &ix, uint64_t base_key, int64_t d) {
    const uint64_t m = (uint64_t)ix.n_slots - 1;
    const uint64_t region = (fmix64(base_key) & m) & ~(uint64_t)(REGION - 1);
    return (region + (uint64_t)((d - 1) & (REGION - 1))) & m;
}
// offset of the second probe: an odd number of regions
__device__ __forceinline__ uint64_t region_step(uint64_t base_key) {
    return ((fmix64(base_key ^ 0x9E3779B97F4A7C15ULL) >> 20) | 1) * REGION;
}
struct Probe {  // probe i of a key: home, home + rstep, then + kstep per further probe
    uint64_t idx, kstep, m;
    __device__ __forceinline__ Probe(const irm_prefix_view &ix, uint64_t home, uint64_t base_key, uint64_t key)
        : idx(home), kstep((key >> 7) | 1), m((uint64_t)ix.n_slots - 1) {
        rstep = region_step(base_key);
    }
    uint64_t rstep;
    __device__ __forceinline__ void next(int64_t i) {  // from probe i to i + 1
        idx = (idx + (i == 0 ? rstep : kstep)) & m;
    }
};

__device__ __forceinline__ int64_t find(const irm_prefix_view &ix, uint64_t key, uint64_t home, uint64_t base_key) {
    Probe p(ix, home, base_key, key);
    for (int64_t probe = 0; probe < ix.n_slots; p.next(probe++)) {
        const uint64_t k = *(volatile uint64_t *)slot_key(ix, p.idx);
        if (k == key) return (int64_t)p.idx;
        if (k == IRM_EMPTY_KEY) return -1;
    }
    return -1;
}

// from the second probe on (the caller tried the home slot itself)
__device__ __forceinline__ void insert_probe(const irm_prefix_view &ix, uint64_t key, uint64_t home,
                                             uint64_t base_key, int64_t epoch) {
    Probe p(ix, home, base_key, key);
    p.next(0);
    for (int64_t probe = 1; probe < ix.n_slots; p.next(probe++)) {
        uint64_t k = *(volatile uint64_t *)slot_key(ix, p.idx);
        if (k == IRM_EMPTY_KEY) {
            k = atomicCAS((unsigned long long *)slot_key(ix, p.idx), (unsigned long long)IRM_EMPTY_KEY,
                          (unsigned long long)key);
            if (k == IRM_EMPTY_KEY) {
                atomicAdd((unsigned long long *)&ix.counters[0], 1ULL);
                k = key;
            }
        }
        if (k == key) {
            atomicMin(slot_epoch(ix, p.idx), (long long)epoch);
            return;
        }
    }
    atomicOr((unsigned long long *)&ix.counters[1], (unsigned long long)ERR_TABLE_FULL);
}

__global__ void reset_kernel(irm_prefix_view ix) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ix.n_slots) {
        *slot_key(ix, i) = IRM_EMPTY_KEY;
        *slot_epoch(ix, i) = INT64_MAX;
    }
    if (i < 2) ix.counters[i] = 0;
}

// chunk_off[i] = exclusive scan of ceil(len_i / CH) (one CTA, tiles of PT sequences)
__global__ void __launch_bounds__(PT) chunk_plan_kernel(const int64_t *__restrict__ seq_off, int32_t n_seq,
                                                         int64_t *__restrict__ chunk_off) {
    __shared__ int64_t carry, sm[PT / 32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n_seq; base += PT) {
        const int i = base + threadIdx.x;
        const int64_t c = i < n_seq ? (seq_off[i + 1] - seq_off[i] + CH - 1) / CH : 0;
        int64_t total;
        const int64_t ex = block_exclusive_scan<PT>(c, &total, sm);
        if (i < n_seq) chunk_off[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) chunk_off[n_seq] = carry;
}

// which (sequence, chunk) this CTA owns; false past the last chunk
__device__ __forceinline__ bool locate(const int64_t *chunk_off, int32_t n_seq, int64_t c, int &seq, int64_t &j) {
    if (c >= chunk_off[n_seq]) return false;
    int lo = 0, hi = n_seq - 1;  // last seq with chunk_off[seq] <= c
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (chunk_off[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    seq = lo;
    j = c - chunk_off[lo];
    return true;
}

// block-wide exclusive scan of per-thread affine maps; returns this thread's exclusive
// prefix and writes the block aggregate
__device__ __forceinline__ Aff block_scan_aff(Aff v, Aff *agg) {
    __shared__ Aff warp_tot[PT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    Aff inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Aff o;
        o.a = __shfl_up_sync(0xffffffffu, inc.a, off);
        o.b = __shfl_up_sync(0xffffffffu, inc.b, off);
        if (lane >= off) inc = compose(o, inc);
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    Aff wpre = {1, 0};
    for (int k = 0; k < w; ++k) wpre = compose(wpre, warp_tot[k]);
    Aff tot = {1, 0};
    for (int k = 0; k < PT / 32; ++k) tot = compose(tot, warp_tot[k]);
    Aff ex;
    ex.a = __shfl_up_sync(0xffffffffu, inc.a, 1);
    ex.b = __shfl_up_sync(0xffffffffu, inc.b, 1);
    if (lane == 0) ex = {1, 0};
    *agg = tot;
    __syncthreads();
    return compose(wpre, ex);
}

__device__ __forceinline__ Aff thread_aff(const uint32_t *tok, int64_t s0, int64_t len, int64_t j, uint32_t t[TPT],
                                          uint64_t base) {
    Aff a = {1, 0};
    const int64_t d0 = j * CH + (int64_t)threadIdx.x * TPT;
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        const int64_t d = d0 + q;
        t[q] = d < len ? tok[s0 + d] : 0;
        if (d < len) a = compose(a, tok_aff(t[q], base));
    }
    return a;
}

__global__ void __launch_bounds__(PT) aggregate_kernel(const uint32_t *__restrict__ tok,
                                                        const int64_t *__restrict__ seq_off, int32_t n_seq,
                                                        const int64_t *__restrict__ chunk_off, Aff *__restrict__ agg,
                                                        uint64_t base) {
    int seq;
    int64_t j;
    if (!locate(chunk_off, n_seq, blockIdx.x, seq, j)) return;
    const int64_t s0 = seq_off[seq], len = seq_off[seq + 1] - s0;
    uint32_t t[TPT];
    Aff a = thread_aff(tok, s0, len, j, t, base), tot;
    block_scan_aff(a, &tot);
    if (threadIdx.x == 0) agg[blockIdx.x] = tot;
}

// per sequence: exclusive prefix of its chunk aggregates (sequential; ~len/1024 steps)
__global__ void carry_kernel(const int64_t *__restrict__ chunk_off, int32_t n_seq, const Aff *__restrict__ agg,
                             Aff *__restrict__ carry) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_seq) return;
    Aff c = {1, 0};
    for (int64_t k = chunk_off[i]; k < chunk_off[i + 1]; ++k) {
        carry[k] = c;
        c = compose(c, agg[k]);
    }
}

// keys of every depth (key[seq_off[s] + d - 1] = key of prefix length d), inserted
// with the sequence's epoch when op_insert
__global__ void __launch_bounds__(PT) keys_kernel(irm_prefix_view ix, const uint32_t *__restrict__ tok,
                                                   const int64_t *__restrict__ seq_off, int32_t n_seq,
                                                   const int64_t *__restrict__ chunk_off, const Aff *__restrict__ carry,
                                                   const int64_t *__restrict__ op_epoch,
                                                   const uint8_t *__restrict__ op_insert, uint64_t *__restrict__ key) {
    int seq;
    int64_t j;
    if (!locate(chunk_off, n_seq, blockIdx.x, seq, j)) return;
    const int64_t s0 = seq_off[seq], len = seq_off[seq + 1] - s0;
    const uint64_t base = key_base(ix.hash_key);
    uint32_t t[TPT];
    Aff a = thread_aff(tok, s0, len, j, t, base), tot;
    Aff h = compose(carry[blockIdx.x], block_scan_aff(a, &tot));  // maps H(empty) = 0 to H before my tokens
    const int64_t ep = op_epoch[seq];
    const bool ins = op_insert && op_insert[seq] && ep >= 0;  // epoch -1: a wave that did not fit
    const int64_t d0 = j * CH + (int64_t)threadIdx.x * TPT;
    uint64_t H = h.b;  // hash of the prefix before my first token (applied to x = 0)
    uint64_t k[TPT];
    int nk = 0;
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        const int64_t d = d0 + q;
        if (d < len) {
            H = addmod(mulmod(H, base), (uint64_t)t[q] + 1);
            k[q] = prefix_key(H, d + 1, ix.hash_key);
            key[s0 + d] = k[q];
            nk = q + 1;
        }
    }
    if (!ins) return;
    // the region key of each 64-depth block of the chunk: the key of the prefix ending just
    // before it (the previous chunk's last depth for the first block, from the carry)
    static_assert(CH % REGION == 0 && REGION % TPT == 0, "blocks align with chunks and threads");
    __shared__ uint64_t sbase[CH / REGION];
    constexpr int TPB = REGION / TPT;  // threads per block
    if (threadIdx.x == 0)
        sbase[0] = j == 0 ? region_base0(ix.hash_key) : prefix_key(carry[blockIdx.x].b, j * CH, ix.hash_key);
    if ((threadIdx.x + 1) % TPB == 0 && (threadIdx.x + 1) / TPB < CH / REGION && nk == TPT)
        sbase[(threadIdx.x + 1) / TPB] = k[TPT - 1];
    __syncthreads();
    const uint64_t bkey = sbase[threadIdx.x / TPB];
    // inserts: the home probe of every key in flight at once (claim by CAS), then every epoch
    // min at once; a key whose home slot holds another key goes on to its probe sequence
    uint64_t home[TPT];
    int64_t slot[TPT];
    unsigned claimed = 0;
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        slot[q] = -1;
        if (q < nk) {
            home[q] = home_slot(ix, bkey, d0 + q + 1);
            const unsigned long long old = atomicCAS((unsigned long long *)slot_key(ix, home[q]),
                                                     (unsigned long long)IRM_EMPTY_KEY, (unsigned long long)k[q]);
            if (old == IRM_EMPTY_KEY) claimed++;
            if (old == IRM_EMPTY_KEY || old == k[q]) slot[q] = (int64_t)home[q];
        }
    }
#pragma unroll
    for (int q = 0; q < TPT; ++q) {
        if (q >= nk) continue;
        if (slot[q] >= 0) atomicMin(slot_epoch(ix, slot[q]), (long long)ep);
        else insert_probe(ix, k[q], home[q], bkey, ep);  // home slot taken: the probe sequence
    }
    // slots used: one atomic per warp
    unsigned c = claimed;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long *)&ix.counters[0], (unsigned long long)c);
}

__global__ void query_kernel(irm_prefix_view ix, const int64_t *__restrict__ seq_off, int32_t n_seq,
                             const int64_t *__restrict__ op_epoch, const uint8_t *__restrict__ op_query,
                             const uint64_t *__restrict__ key, int64_t *__restrict__ m_out,
                             int64_t *__restrict__ wit_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_seq) return;
    if (op_query && !op_query[i]) {
        m_out[i] = 0;
        wit_out[i] = -1;
        return;
    }
    const int64_t s0 = seq_off[i], len = seq_off[i + 1] - s0, e = op_epoch[i];
    int64_t lo = 0, hi = len, wit = -1;
    while (lo < hi) {  // largest d with a prefix of length d inserted before epoch e
        const int64_t mid = (lo + hi + 1) >> 1;
        const int64_t blk = (mid - 1) / REGION * REGION;  // prefix length of the region key
        const uint64_t bkey = blk == 0 ? region_base0(ix.hash_key) : key[s0 + blk - 1];
        const int64_t s = find(ix, key[s0 + mid - 1], home_slot(ix, bkey, mid), bkey);
        const int64_t ep = s >= 0 ? *(volatile int64_t *)slot_epoch(ix, s) : INT64_MAX;
        if (ep < e) {
            lo = mid;
            wit = ep;
        } else {
            hi = mid - 1;
        }
    }
    m_out[i] = lo;
    wit_out[i] = lo > 0 ? wit : -1;
}

// token-by-token check of every answer against the witness's stored tokens; a
// mismatch (a hash collision) is answered again by an exact scan of every sequence
// inserted before the query: the longest common prefix, the earliest epoch on ties
__global__ void verify_kernel(irm_prefix_view ix, const uint32_t *__restrict__ tok, const int64_t *__restrict__ seq_off,
                              int32_t n_seq, const int64_t *__restrict__ op_epoch, const uint8_t *__restrict__ op_query,
                              const uint32_t *__restrict__ arena, const int64_t *__restrict__ wit_off,
                              const int64_t *__restrict__ wit_len, int64_t *__restrict__ m,
                              int64_t *__restrict__ wit) {
    __shared__ unsigned long long first_diff;
    const int i = blockIdx.x;
    if (i >= n_seq || (op_query && !op_query[i])) return;
    const int64_t mi = m[i];
    const int64_t w = wit[i];
    const int64_t s0 = seq_off[i], len = seq_off[i + 1] - s0;
    const uint32_t *a = tok + s0;
    bool bad = mi > 0 && (w < 0 || wit_len[w] < mi);
    if (mi > 0 && !bad) {
        const uint32_t *b = arena + wit_off[w];
        for (int64_t d = threadIdx.x; d < mi; d += blockDim.x) bad |= a[d] != b[d];
    }
    if (!__syncthreads_or(bad)) return;
    int64_t best = 0, best_w = -1;
    const int64_t e = op_epoch[i];
    for (int64_t v = 0; v < e; ++v) {
        const int64_t L = min(len, wit_len[v]);
        if (L <= best) continue;  // cannot beat the current answer (uniform: same values in every thread)
        if (threadIdx.x == 0) first_diff = (unsigned long long)L;
        __syncthreads();
        const uint32_t *b = arena + wit_off[v];
        for (int64_t d = threadIdx.x; d < L; d += blockDim.x)
            if (a[d] != b[d]) {
                atomicMin(&first_diff, (unsigned long long)d);
                break;
            }
        __syncthreads();
        const int64_t lcp = (int64_t)first_diff;
        __syncthreads();
        if (lcp > best) {
            best = lcp;
            best_w = v;
        }
    }
    if (threadIdx.x == 0) {
        m[i] = best;
        wit[i] = best > 0 ? best_w : -1;
        atomicOr((unsigned long long *)&ix.counters[1], (unsigned long long)COLLISION_RESOLVED);
    }
}

// Graph-capturable wave form (the serve pipeline's phase 1): append the wave's
// sequences to the token arena at the device-side fill level, give sequence r
// the insert epoch epoch_next + r, then bump both counters. No host involvement.
__global__ void wave_arena_kernel(uint32_t *__restrict__ arena, int64_t arena_cap,
                                  const int64_t *__restrict__ arena_used, int64_t *__restrict__ wit_off,
                                  int64_t *__restrict__ wit_len, int64_t wit_cap,
                                  const int64_t *__restrict__ epoch_next, const uint32_t *__restrict__ tok,
                                  const int64_t *__restrict__ seq_off, int32_t n_seq, int64_t *__restrict__ op_epoch,
                                  int64_t *__restrict__ counters) {
    const int64_t used = *arena_used, e0 = *epoch_next;
    const int64_t n_tok = seq_off[n_seq] - seq_off[0];
    const bool fits = used + n_tok <= arena_cap && e0 + n_seq <= wit_cap;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (!fits) {
        if (g == 0) atomicOr((unsigned long long *)&counters[1], (unsigned long long)ERR_TABLE_FULL);
        for (int64_t r = g; r < n_seq; r += stride) op_epoch[r] = -1;  // nothing inserted or matched
        return;
    }
    for (int64_t r = g; r < n_seq; r += stride) {
        op_epoch[r] = e0 + r;
        wit_off[e0 + r] = used + seq_off[r] - seq_off[0];
        wit_len[e0 + r] = seq_off[r + 1] - seq_off[r];
    }
    for (int64_t i = g; i < n_tok; i += stride) arena[used + i] = tok[seq_off[0] + i];
}

__global__ void wave_bump_kernel(int64_t arena_cap, int64_t *__restrict__ arena_used, int64_t wit_cap,
                                 int64_t *__restrict__ epoch_next, const int64_t *__restrict__ seq_off,
                                 int32_t n_seq) {
    const int64_t n_tok = seq_off[n_seq] - seq_off[0];
    if (*arena_used + n_tok <= arena_cap && *epoch_next + n_seq <= wit_cap) {
        *arena_used += n_tok;
        *epoch_next += n_seq;
    }
}

}  // namespace prefix
}  // namespace irm

namespace irm {
namespace prefix {
// host copy of key_base (the aggregate kernel takes the base as an argument)
static uint64_t key_base_host(uint64_t hash_key) {
    uint64_t x = hash_key + 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    x ^= x >> 31;
    return 2 + x % (P61 - 3);
}
}  // namespace prefix
}  // namespace irm

using namespace irm;
using prefix::Aff;

extern "C" int irm_prefix_reset(const irm_prefix_view *ix, irm_stream_t stream) {
    IRM_REQUIRE(ix && ix->slots && ix->counters, "null pointer");
    IRM_REQUIRE(ix->n_slots >= 2 && (ix->n_slots & (ix->n_slots - 1)) == 0, "n_slots must be a power of two");
    const int64_t n = ix->n_slots;
    prefix::reset_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*ix);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

static int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

extern "C" int64_t irm_prefix_workspace_bytes(int64_t n_tokens, int32_t n_seq) {
    const int64_t n_chunks = n_tokens / prefix::CH + n_seq + 1;
    return align256((int64_t)(n_seq + 1) * 8) + 2 * align256(n_chunks * (int64_t)sizeof(Aff)) +
           align256(n_tokens * 8);
}

extern "C" int irm_prefix_match_insert(const irm_prefix_view *ix, const uint32_t *tok, const int64_t *seq_off,
                                       int32_t n_seq, int64_t n_tokens, const int64_t *op_epoch,
                                       const uint8_t *op_insert, const uint8_t *op_query, const uint32_t *arena,
                                       const int64_t *wit_off, const int64_t *wit_len, int64_t *m, int64_t *wit,
                                       void *ws, int64_t ws_bytes, irm_stream_t stream) {
    IRM_REQUIRE(ix && ix->slots && ix->counters, "null index");
    IRM_REQUIRE(n_seq >= 0 && n_tokens >= 0, "bad sizes");
    if (n_seq == 0) return IRM_OK;
    IRM_REQUIRE(seq_off && op_epoch && m && wit && ws, "null pointer");
    IRM_REQUIRE(n_tokens == 0 || tok, "null tokens");
    IRM_REQUIRE(arena && wit_off && wit_len, "queries are verified against the arena: arena/wit_off/wit_len required");
    IRM_REQUIRE(ws_bytes >= irm_prefix_workspace_bytes(n_tokens, n_seq), "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n_chunks_cap = n_tokens / prefix::CH + n_seq + 1;
    uint8_t *w = (uint8_t *)ws;
    int64_t *chunk_off = (int64_t *)w;
    w += align256((int64_t)(n_seq + 1) * 8);
    Aff *agg = (Aff *)w;
    w += align256(n_chunks_cap * (int64_t)sizeof(Aff));
    Aff *carry = (Aff *)w;
    w += align256(n_chunks_cap * (int64_t)sizeof(Aff));
    uint64_t *key = (uint64_t *)w;
    prefix::chunk_plan_kernel<<<1, prefix::PT, 0, s>>>(seq_off, n_seq, chunk_off);
    IRM_LAUNCH_CHECK();
    // grid = an upper bound on the chunk count; CTAs past the real count exit
    const unsigned grid = (unsigned)n_chunks_cap;
    prefix::aggregate_kernel<<<grid, prefix::PT, 0, s>>>(tok, seq_off, n_seq, chunk_off, agg,
                                                          prefix::key_base_host(ix->hash_key));
    IRM_LAUNCH_CHECK();
    prefix::carry_kernel<<<(n_seq + 127) / 128, 128, 0, s>>>(chunk_off, n_seq, agg, carry);
    IRM_LAUNCH_CHECK();
    prefix::keys_kernel<<<grid, prefix::PT, 0, s>>>(*ix, tok, seq_off, n_seq, chunk_off, carry, op_epoch, op_insert,
                                                     key);
    IRM_LAUNCH_CHECK();
    prefix::query_kernel<<<(n_seq + 127) / 128, 128, 0, s>>>(*ix, seq_off, n_seq, op_epoch, op_query, key, m, wit);
    IRM_LAUNCH_CHECK();
    prefix::verify_kernel<<<n_seq, 256, 0, s>>>(*ix, tok, seq_off, n_seq, op_epoch, op_query, arena, wit_off, wit_len,
                                                 m, wit);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_prefix_wave_prepare(const irm_prefix_view *ix, uint32_t *arena, int64_t arena_cap,
                                       int64_t *arena_used, int64_t *wit_off, int64_t *wit_len, int64_t wit_cap,
                                       int64_t *epoch_next, const uint32_t *tok, const int64_t *seq_off,
                                       int32_t n_seq, int64_t *op_epoch, irm_stream_t stream) {
    IRM_REQUIRE(ix && ix->counters, "null index");
    IRM_REQUIRE(n_seq >= 0 && arena_cap >= 0 && wit_cap >= 0, "bad sizes");
    if (n_seq == 0) return IRM_OK;
    IRM_REQUIRE(arena && arena_used && wit_off && wit_len && epoch_next && tok && seq_off && op_epoch,
                "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = irm::sm_count() * 4;
    prefix::wave_arena_kernel<<<grid, 256, 0, s>>>(arena, arena_cap, arena_used, wit_off, wit_len, wit_cap,
                                                    epoch_next, tok, seq_off, n_seq, op_epoch, ix->counters);
    IRM_LAUNCH_CHECK();
    prefix::wave_bump_kernel<<<1, 1, 0, s>>>(arena_cap, arena_used, wit_cap, epoch_next, seq_off, n_seq);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}
