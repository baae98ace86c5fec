// K1 (CDC + xxh64) and K2 (batched xxh64 spans) for sm_100a.
//
// Replaces chunking.cdc_chunk (reference chunking.py:89-133) and
// fingerprint.fingerprint (fingerprint.py:28-30) with one batched,
// bit-exact device pass.
//
// The Gear recurrence h_t = rotl64(h_{t-1}, 1) + g_t (chunking.py:114) has no
// window, so it is not a plain scan. Writing rotl(h) = 2h + msb(h) (mod 2^64)
// gives the exact decomposition
//     h_t = G_t + B_t  (mod 2^64),
//     G_t = sum_{k<64} g_{t-k} << k          (windowed, warp-scannable)
//     B_t = sum_{k<64} m_{t-1-k} << k,  m_t = msb(h_t)
// so the only sequential dependency is ONE BIT per token. A warp handles 32
// tokens per step: lane j knows B up to the 2^j-1 contribution of lanes < j,
// so msb(h) is determined when msb(lo) == msb(lo + 2^j - 1); otherwise
// (≈2^-32 per lane on random input) the lane is resolved exactly, in lane
// order. Then B advances by (B << 32) | brev(ballot(m)).
//
// Marker pins reset h (chunking.py:116-118), so the stream splits into
// independent regions; one CTA scans one region (producer / chain / walker
// warps, see cdc_region_kernel), walks the boundary rule with ballot/ffs over
// the candidate words, then hashes its chunks (XXH64 from L2-resident tokens).
// That is the fused form; the split form (further below) computes G on every
// SM first and hashes on every SM after, for batches of few long regions.
#include "common.cuh"
#include "tma.cuh"
#include <stdlib.h>
#include <string.h>
#include <algorithm>

namespace irm {

struct Region {
    int64_t tok_begin;     // absolute index into tok[] of the region's first token
    int64_t stream_begin;  // absolute index of the owning stream's first token
    int64_t cap_off;       // staging slot of the region's first chunk
    int32_t len;           // tokens (>= 1)
    int32_t ends_pin;      // last token carries a marker pin
};

// gear[i] = splitmix64 output i + 1 of `seed` (rng.py:17-24: state_i = seed + (i+1) * gamma,
// then mix; chunking.py:64-66). A closed form of the index, so the K1 kernels can
// compute it instead of looking it up: ~20 integer instructions against a random
// 8-byte L1/L2 read per token (one L1 wavefront per lane).
__device__ __forceinline__ uint64_t gear_splitmix(uint64_t seed, uint32_t i) {
    uint64_t z = seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void gear_table_kernel(uint64_t seed, uint64_t *out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 65536) return;
    out[i] = gear_splitmix(seed, (uint32_t)i);
}

// where K1 takes g_t from: the caller's 65,536-entry table, or (SEEDED) the
// table's generating seed
struct GearSrc {
    const uint64_t *table;
    uint64_t seed;
};

template <bool SEEDED>
__device__ __forceinline__ uint64_t gear_of(const GearSrc &gs, uint32_t tok) {
    if constexpr (SEEDED) return gear_splitmix(gs.seed, tok & 0xFFFFu);
    else return __ldg(gs.table + (tok & 0xFFFFu));
}

// Walk one stream's sorted pins: calls emit(start, last, ends_pin) per region.
template <typename F>
__device__ __forceinline__ int64_t for_each_region(int64_t n, const int64_t *pins, int64_t np,
                                                   F emit) {
    int64_t rs = 0, prev = -1, cnt = 0;
    for (int64_t i = 0; i < np; ++i) {
        int64_t p = pins[i];
        if (p < 0 || p >= n || p == prev) continue;
        prev = p;
        emit(rs, p, 1, cnt);
        ++cnt;
        rs = p + 1;
    }
    if (rs < n) {
        emit(rs, n - 1, 0, cnt);
        ++cnt;
    }
    return cnt;
}

constexpr int PLAN_BLOCK = 1024;

struct PlanArgs {
    const int64_t *stream_off;
    int32_t n_streams;
    const int64_t *pin_off, *pins;
    int32_t use_pins, min_size;
    Region *regions;
    int64_t *r_first, *n_regions;
};

// the region plan of a batch (one CTA of BLOCK threads): regions per stream, their
// exclusive scan, then one Region record per pin-delimited region
template <int BLOCK>
__device__ __forceinline__ void plan_regions(const PlanArgs &a) {
    const int64_t *__restrict__ stream_off = a.stream_off;
    const int32_t n_streams = a.n_streams;
    const int64_t *__restrict__ pin_off = a.pin_off;
    const int64_t *__restrict__ pins = a.pins;
    const int32_t use_pins = a.use_pins, min_size = a.min_size;
    Region *__restrict__ regions = a.regions;
    int64_t *__restrict__ r_first = a.r_first;
    __shared__ int64_t sm[BLOCK / 32];
    int64_t carry = 0;
    for (int32_t s0 = 0; s0 < n_streams; s0 += BLOCK) {
        const int32_t s = s0 + threadIdx.x;
        int64_t cnt = 0, n = 0, p0 = 0, np = 0, sb = 0;
        if (s < n_streams) {
            sb = stream_off[s];
            n = stream_off[s + 1] - sb;
            if (use_pins) {
                p0 = pin_off[s];
                np = pin_off[s + 1] - p0;
            }
            cnt = for_each_region(n, pins + p0, np, [](int64_t, int64_t, int, int64_t) {});
        }
        int64_t tot;
        const int64_t ex = block_exclusive_scan<BLOCK>(cnt, &tot, sm);
        if (s < n_streams) {
            const int64_t rbase = carry + ex;
            r_first[s] = rbase;
            for_each_region(n, pins + p0, np, [&](int64_t rs, int64_t last, int pin, int64_t i) {
                Region R;
                R.tok_begin = sb + rs;
                R.stream_begin = sb;
                R.len = (int32_t)(last - rs + 1);
                R.ends_pin = pin;
                R.cap_off = (sb + rs) / min_size + (rbase + i);
                regions[rbase + i] = R;
            });
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        r_first[n_streams] = carry;
        *a.n_regions = carry;
    }
}

__global__ void __launch_bounds__(PLAN_BLOCK) cdc_plan_kernel(PlanArgs a) { plan_regions<PLAN_BLOCK>(a); }

// One CTA per region, four warp roles pipelined over 1024-token tiles:
//   producers (warps 0..7):  windowed G_t of tile i (lane-serial over 4 tokens per
//                            thread + a 4-round warp scan; tokens loaded two tiles
//                            ahead, Gear values computed from the seed or looked up
//                            one tile ahead)
//   chain     (warp 0):      the sequential MSB recurrence over tile i-1 -- ONLY
//                            m_t, ~6 dependent instructions per 32 tokens
//   cand      (warp 1):      h_t and the mask candidates of tile i-2 (parallel
//                            over steps: B at every step is known from the m's)
//   walker    (warp 2):      the boundary rule over the candidate words of tile i-3
// msb(h) is decided on the high 32-bit words alone (the low words carry at
// most 2 into them); the rare ambiguous lanes are resolved exactly in lane order.
#ifndef IRM_CDC_PRODUCE
#define IRM_CDC_PRODUCE 1  // fused-form producers: 1 = lane-serial G (4 tokens per thread), 0 = Kogge-Stone
#endif
#ifndef IRM_CDC_NPROD
#define IRM_CDC_NPROD 8  // producer warps of the lane-serial form
#endif
#ifndef IRM_CDC_HASHERS
// warps fingerprinting, inside the tile loop, the chunks the walker emitted one tile earlier.
// 0 (default): measured slower at 1, 2 and 4 (296 x 32K: 97 -> 150-207 us) -- a quad's XXH64
// walks its chunk by dependent L2 round trips, which stretch the lock-step tile period; the
// tail after the loop hashes every chunk of the region with all warps at once instead
#define IRM_CDC_HASHERS 0
#endif
constexpr int RG_HASHERS = IRM_CDC_PRODUCE ? IRM_CDC_HASHERS : 0;
constexpr int RG_THREADS = IRM_CDC_PRODUCE ? (IRM_CDC_NPROD + 4 + RG_HASHERS) * 32 : 512;
constexpr int RG_TILE = 1024;                 // tokens per pipeline tile
constexpr int RG_SUB = RG_TILE / 32;          // 32-token sub-blocks (chain steps) per tile
constexpr int RG_PRODUCERS = RG_THREADS / 32 - 4 - RG_HASHERS;  // warps 0 .. RG_PRODUCERS - 1
constexpr int W_WALK = RG_PRODUCERS, W_CAND0 = RG_PRODUCERS + 1, W_CAND1 = RG_PRODUCERS + 2,
              W_CHAIN = RG_PRODUCERS + 3, W_HASH = RG_PRODUCERS + 4;
constexpr int RG_PER = (RG_SUB + RG_PRODUCERS - 1) / RG_PRODUCERS;

__device__ __forceinline__ void producer_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(RG_PRODUCERS * 32) : "memory");
}

// stage tile `tile` tokens into sTok with 4-byte cp.async (regions are not 16-B aligned)
__device__ __forceinline__ void stage_tokens(const uint32_t *__restrict__ rt, int32_t len, int32_t tile,
                                             uint32_t *sTok, int ptid) {
    const int32_t base = tile * RG_TILE;
    for (int i = ptid; i < RG_TILE; i += RG_PRODUCERS * 32) {
        if (base + i < len) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sTok + i)),
                         "l"(rt + base + i)
                         : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// gear values g_t of this producer thread's tokens of a tile (the L2 lookups are issued one
// tile ahead of their use, so their latency hides under the previous tile's scan)
template <bool SEEDED>
__device__ __forceinline__ void load_gear(const uint32_t *sTok, int32_t len, int32_t tile_start,
                                          const GearSrc &gear, int pw, int lane,
                                          uint64_t (&g)[RG_PER]) {
#pragma unroll
    for (int q = 0; q < RG_PER; ++q) {
        const int c = pw + q * RG_PRODUCERS;
        const int32_t t = tile_start + c * 32 + lane;
        g[q] = (c < RG_SUB && t < len) ? gear_of<SEEDED>(gear, sTok[c * 32 + lane]) : 0ULL;
    }
}

// G_t for tokens [tile_start, tile_start + RG_TILE) of a region into sGdst, from the tile's
// gear values g (load_gear).
__device__ __forceinline__ void produce_tile(uint64_t (&g)[RG_PER], int32_t len, int32_t tile_start,
                                             uint64_t *sGdst, const uint64_t *sGprev, uint64_t *sS31, int pw,
                                             int lane) {
    // in-block windowed scan S_j = sum_{i<=j} g_i << (j-i), Kogge-Stone through
    // shared memory: the warp-shuffle unit is left to the chain/cand warps'
    // votes, which sit on the CTA's critical path
#pragma unroll
    for (int q = 0; q < RG_PER; ++q) {
        const int c = pw + q * RG_PRODUCERS;
        if (c < RG_SUB) sGdst[c * 32 + lane] = g[q];
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        __syncwarp();
        uint64_t y[RG_PER];
#pragma unroll
        for (int q = 0; q < RG_PER; ++q) {
            const int c = pw + q * RG_PRODUCERS;
            y[q] = (c < RG_SUB && lane >= d) ? sGdst[c * 32 + lane - d] : 0ULL;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < RG_PER; ++q) {
            const int c = pw + q * RG_PRODUCERS;
            g[q] += y[q] << d;
            if (c < RG_SUB) sGdst[c * 32 + lane] = g[q];
        }
    }
#pragma unroll
    for (int q = 0; q < RG_PER; ++q) {
        const int c = pw + q * RG_PRODUCERS;
        if (c < RG_SUB && lane == 31) sS31[c] = g[q];
    }
    producer_bar();
    // carry-in G_{base-1} = G of the previous sub-block's last token:
    // G_last(c) = S31(c) + (G_last(c-1) << 32), so two sub-blocks suffice
    const uint64_t prevG = sGprev ? sGprev[RG_TILE - 1] : 0ULL;
#pragma unroll
    for (int q = 0; q < RG_PER; ++q) {
        const int c = pw + q * RG_PRODUCERS;
        if (c >= RG_SUB) break;
        const uint64_t gb = c == 0 ? prevG
                          : c == 1 ? sS31[0] + (prevG << 32)
                                   : sS31[c - 1] + (sS31[c - 2] << 32);
        sGdst[c * 32 + lane] += gb << (lane + 1);
    }
}

// producers, lane-serial form (IRM_CDC_PRODUCE=1): thread p of the RG_PRODUCERS warps owns
// tokens PT*p .. PT*p+PT-1 of a tile. Its local G over those tokens is a serial shift-add
// (L_j = 2 L_{j-1} + g_j); the warp then scans the per-thread ends e with
// x_i = e_i + (x_{i-1} << PT) in four shuffle rounds -- 16 threads span 64 tokens, so lane
// 31's x is complete without any carry-in, and lanes < 15 add the carry C (G at the token
// before the warp) shifted by their distance. About 40 integer instructions per token
// against ~115 for a Kogge-Stone over 64-bit values in shared memory.
constexpr int PT = RG_TILE / (RG_PRODUCERS * 32);
static_assert(!IRM_CDC_PRODUCE || (PT * RG_PRODUCERS * 32 == RG_TILE && PT % 2 == 0), "tile split");

__device__ __forceinline__ void load_tok_pt(const uint32_t *__restrict__ rt, int32_t len, int32_t tile,
                                            int ptid, uint32_t (&tk)[PT]) {
    const int32_t t0 = tile * RG_TILE + PT * ptid;
#pragma unroll
    for (int j = 0; j < PT; ++j) tk[j] = t0 + j < len ? __ldg(rt + t0 + j) : 0u;
}

template <bool SEEDED>
__device__ __forceinline__ void gear_pt(const GearSrc &gear, const uint32_t (&tk)[PT], uint64_t (&g)[PT]) {
#pragma unroll
    for (int j = 0; j < PT; ++j) g[j] = gear_of<SEEDED>(gear, tk[j]);
}

// sX[2][RG_PRODUCERS]: each warp's complete G at its last token, by tile parity
__device__ __forceinline__ void produce_tile_serial(const uint64_t (&g)[PT], int32_t tile, uint64_t *sGdst,
                                                    uint64_t *sX, int pw, int lane, int ptid) {
    uint64_t L[PT];
    uint64_t acc = 0;
#pragma unroll
    for (int j = 0; j < PT; ++j) {
        acc = (acc << 1) + g[j];
        L[j] = acc;
    }
    uint64_t x = acc;
#pragma unroll
    for (int d = 1; d * PT < 64; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y << (PT * d);
    }
    if (lane == 31) sX[(tile & 1) * RG_PRODUCERS + pw] = x;
    producer_bar();
    const uint64_t C = pw > 0 ? sX[(tile & 1) * RG_PRODUCERS + pw - 1]
                     : tile > 0 ? sX[((tile - 1) & 1) * RG_PRODUCERS + RG_PRODUCERS - 1] : 0ULL;
    if (PT * (lane + 1) < 64) x += C << (PT * (lane + 1));
    uint64_t gp = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) gp = C;
    ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(sGdst + PT * ptid);
#pragma unroll
    for (int j = 0; j < PT; j += 2)
        dst[j / 2] = make_ulonglong2(L[j] + (gp << (j + 1)), L[j + 1] + (gp << (j + 2)));
}

#ifndef IRM_CDC_CHAIN_LEAN
#define IRM_CDC_CHAIN_LEAN 1
#endif

// chain warp: sBm[s] = W_s, the low word of B after step s of one tile
// (bit 31-i = m_i of the step's token i). Lane L handles token j = 31 - L, so
// the ballot itself is the bit-reversed word and the loop-carried path is
// funnel-shift -> add -> vote (~30 cycles per 32 tokens, microbenchmarked:
// a BREV or an ambiguity branch on the path costs ~20-25 cycles each).
// Ambiguous lanes (high word at a carry boundary, ~2^-30 per token) are only
// accumulated; a tile that saw one is recomputed exactly (64-bit, lane order).
__device__ __forceinline__ void chain_tile(const uint64_t *sG, uint32_t *sBm, int32_t tile_start,
                                           int32_t len, uint32_t &Blo, uint32_t &Bhi, int lane) {
    const int nsteps = min(RG_SUB, (len - tile_start + 31) / 32);
    const int j = 31 - lane;
    const uint32_t Blo0 = Blo, Bhi0 = Bhi;
    uint32_t myW = 0;  // lane s keeps W_s
    bool amb = false;  // per lane: some step's high word sat at a carry boundary
    // G's high words are read CH_AHEAD steps ahead: the producers keep shared memory busy,
    // so one step of lead does not cover the load latency
    constexpr int CH_AHEAD = 4;
#if IRM_CDC_CHAIN_LEAN
    // lean step (~9 issue slots): 32-bit loads of G's high word only; ambiguity as bit 31 of
    // an OR of (hs + 2) ^ hs -- adding the pending carry (<= 2) flips bit 31 exactly at a carry
    // boundary; lane 0 stores W_s (no per-step select)
    const uint32_t *sGhi = reinterpret_cast<const uint32_t *>(sG) + 1;
    uint32_t amb_acc = 0;
    uint32_t Gq[CH_AHEAD];
#pragma unroll
    for (int a = 0; a < CH_AHEAD; ++a) Gq[a] = a < nsteps ? sGhi[2 * (a * 32 + j)] : 0u;
#pragma unroll CH_AHEAD
    for (int s = 0; s < nsteps; ++s) {
        const uint32_t Ghi = Gq[0];
#pragma unroll
        for (int a = 0; a + 1 < CH_AHEAD; ++a) Gq[a] = Gq[a + 1];
        Gq[CH_AHEAD - 1] = s + CH_AHEAD < nsteps ? sGhi[2 * ((s + CH_AHEAD) * 32 + j)] : 0u;
        const uint32_t hs = Ghi + __funnelshift_l(Blo, Bhi, j);  // high word of h, carry c in {0,1,2} pending
        const unsigned W = __ballot_sync(0xffffffffu, (int32_t)hs < 0);
        amb_acc |= (hs + 2u) ^ hs;  // (past-the-end lanes may trigger a harmless redo)
        if (lane == 0) sBm[s] = W;
        Bhi = Blo;
        Blo = W;
    }
    amb = (int32_t)amb_acc < 0;
#else
    uint32_t Gq[CH_AHEAD];
#pragma unroll
    for (int a = 0; a < CH_AHEAD; ++a) Gq[a] = a < nsteps ? (uint32_t)(sG[a * 32 + j] >> 32) : 0u;
#pragma unroll CH_AHEAD
    for (int s = 0; s < nsteps; ++s) {
        const uint32_t Ghi = Gq[0];
#pragma unroll
        for (int a = 0; a + 1 < CH_AHEAD; ++a) Gq[a] = Gq[a + 1];
        Gq[CH_AHEAD - 1] = s + CH_AHEAD < nsteps ? (uint32_t)(sG[(s + CH_AHEAD) * 32 + j] >> 32) : 0u;
        const uint32_t hs = Ghi + __funnelshift_l(Blo, Bhi, j);  // high word of h, carry c in {0,1,2} pending
        const unsigned W = __ballot_sync(0xffffffffu, hs >> 31);
        amb |= (hs & 0x7FFFFFFEu) == 0x7FFFFFFEu;  // (past-the-end lanes may trigger a harmless redo)
        myW = lane == s ? W : myW;
        Bhi = Blo;
        Blo = W;
    }
#endif
    if (__any_sync(0xffffffffu, amb)) {  // rare: redo the tile with exact 64-bit arithmetic, lanes in token order
        Blo = Blo0;
        Bhi = Bhi0;
        for (int s = 0; s < nsteps; ++s) {
            const bool valid = tile_start + 32 * s + lane < len;
            const uint64_t lo = sG[s * 32 + lane] + ((((uint64_t)Bhi << 32) | Blo) << lane);
            const uint64_t hi = lo + ((1ULL << lane) - 1);
            unsigned M = __ballot_sync(0xffffffffu, (unsigned)(lo >> 63));
            unsigned u2 = __ballot_sync(0xffffffffu, valid && ((lo ^ hi) >> 63));
            while (u2) {
                const int jj = __ffs(u2) - 1;
                unsigned mb = 0;
                if (lane == jj) {
                    const uint64_t u = (uint64_t)((__brev(M) >> (31 - jj)) >> 1);
                    mb = (unsigned)((lo + u) >> 63);
                }
                mb = __shfl_sync(0xffffffffu, mb, jj);
                M = (M & ~(1u << jj)) | (mb << jj);
                u2 &= u2 - 1;
            }
            const uint32_t W = __brev(M);
            myW = lane == s ? W : myW;
            Bhi = Blo;
            Blo = W;
        }
#if IRM_CDC_CHAIN_LEAN
        __syncwarp();
        if (lane < nsteps) sBm[lane] = myW;
#endif
    }
#if !IRM_CDC_CHAIN_LEAN
    sBm[lane] = myW;
#endif
}

// cand warp: candidate words ((h & mask) == 0, chunking.py:121) of one tile.
// Step s needs B before it: low word sBm[s-1], high word sBm[s-2] (previous
// tile's last words in Bprev0/Bprev1 at s = 0, 1).
// Two cand warps split the steps by parity; only B's low word matters for
// (h & mask) with mask < 2^32.
__device__ __forceinline__ void cand_tile(const uint64_t *sG, const uint32_t *sBm, unsigned *sCand,
                                          int32_t tile_start, int32_t len, uint32_t mask,
                                          uint32_t &Bprev_lo, int parity, int lane) {
    const int nsteps = min(RG_SUB, (len - tile_start + 31) / 32);
    unsigned my_cand = 0;
#pragma unroll 4
    for (int s = parity; s < nsteps; s += 2) {
        const uint32_t b_lo = s >= 1 ? sBm[s - 1] : Bprev_lo;  // B before step s (low word)
        const uint32_t mnew = sBm[s];                          // W_s: bit 31-i = m_i
        const uint32_t Glo = (uint32_t)sG[s * 32 + lane];
        const uint32_t hlo = Glo + (b_lo << lane) + ((mnew >> (31 - lane)) >> 1);
        const bool valid = tile_start + 32 * s + lane < len;
        const unsigned cand = __ballot_sync(0xffffffffu, valid && (hlo & mask) == 0);
        my_cand = lane == s ? cand : my_cand;
    }
    if ((lane & 1) == parity) sCand[lane] = lane < nsteps ? my_cand : 0u;
    if (nsteps >= 1) Bprev_lo = sBm[nsteps - 1];
}

struct ChunkSink {
    int32_t *st_start, *st_len;
    uint8_t *st_forced;
    int64_t cap;
    int32_t rel0;
    __device__ __forceinline__ void emit(int lane, int32_t n, int32_t start, int32_t len, uint8_t f) const {
        if (lane == 0) {
            st_start[cap + n] = rel0 + start;
            st_len[cap + n] = len;
            st_forced[cap + n] = f;
        }
    }
};

// walker warp: boundary rule over one tile (chunking.py:116-124:
// marker > max_clamp > mask hit); lane w holds the candidate word of sub-block w
__device__ __forceinline__ void walk_tile(const unsigned *sCand, int32_t tile_start, int32_t len,
                                          int32_t min_size, int32_t max_size, int32_t t_pin,
                                          int32_t &start, int32_t &nch, const ChunkSink &sink,
                                          int lane) {
    const unsigned my_cand = sCand[lane];
    const int32_t tile_end = min(tile_start + RG_TILE, len);
    const int32_t word_lo = tile_start + 32 * lane;
    while (true) {
        const int32_t t_max = start + max_size - 1;
        const int32_t lo_c = max(tile_start, start + min_size - 1);
        unsigned mw = 0;
        if (lo_c < word_lo + 32) mw = lo_c <= word_lo ? my_cand : my_cand & (0xffffffffu << (lo_c - word_lo));
        const unsigned found = __ballot_sync(0xffffffffu, mw != 0);
        int32_t t_cand = INT32_MAX;
        if (found) {
            const int w = __ffs(found) - 1;
            const unsigned fw = __shfl_sync(0xffffffffu, mw, w);
            t_cand = tile_start + 32 * w + __ffs(fw) - 1;
        }
        // the pin (region end) counts only while the open chunk can reach it
        const int32_t nxt = min(t_max, min(t_pin >= start ? t_pin : INT32_MAX, t_cand));
        if (nxt >= tile_end) break;
        sink.emit(lane, nch, start, nxt - start + 1,
                  nxt == t_pin ? IRM_FORCED_MARKER : nxt == t_max ? IRM_FORCED_MAX_CLAMP : IRM_FORCED_NONE);
        ++nch;
        start = nxt + 1;
    }
}

// walker, scalar form (split K1): the warp builds next-candidate words once per tile
// (suffix min over lanes), then lane 0 alone walks the boundary rule with two shared
// loads per chunk: no vote / shuffle on the per-chunk dependency chain. Same rule as
// walk_tile; walker state (start, nch) lives in lane 0.
__device__ __forceinline__ void walk_tile_scalar(const unsigned *sCand, int32_t *sNext, int32_t tile_start,
                                                 int32_t len, int32_t min_size, int32_t max_size, int32_t t_pin,
                                                 int32_t &start, int32_t &nch, const ChunkSink &sink, int lane) {
    const unsigned my_cand = sCand[lane];
    int32_t nc = my_cand ? tile_start + 32 * lane + __ffs(my_cand) - 1 : INT32_MAX;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_down_sync(0xffffffffu, nc, d);
        if (lane + d < 32) nc = min(nc, y);
    }
    sNext[lane] = nc;  // first candidate at or after word `lane`
    if (lane == 0) sNext[32] = INT32_MAX;
    __syncwarp();
    if (lane != 0) return;
    const int32_t tile_end = min(tile_start + RG_TILE, len);
    while (true) {
        const int32_t t_max = start + max_size - 1;
        const int32_t rel = max(0, start + min_size - 1 - tile_start);
        int32_t t_cand = INT32_MAX;
        if (rel < RG_TILE) {
            const int w = rel >> 5;
            const unsigned cw = sCand[w] & (0xffffffffu << (rel & 31));
            const int32_t nx = sNext[w + 1];
            t_cand = cw ? tile_start + 32 * w + __ffs(cw) - 1 : nx;
        }
        const int32_t nxt = min(t_max, min(t_pin >= start ? t_pin : INT32_MAX, t_cand));
        if (nxt >= tile_end) break;
        sink.emit(0, nch, start, nxt - start + 1,
                  nxt == t_pin ? IRM_FORCED_MARKER : nxt == t_max ? IRM_FORCED_MAX_CLAMP : IRM_FORCED_NONE);
        ++nch;
        start = nxt + 1;
    }
}

#ifndef IRM_CDC_FUSED_WALK
#define IRM_CDC_FUSED_WALK 1  // fused-form walker: 1 = lane-0 scalar (walk_tile_scalar), 0 = warp vote per chunk
#endif

template <bool SEEDED>
__global__ void __launch_bounds__(RG_THREADS)
cdc_region_kernel(const uint32_t *__restrict__ tok, const Region *__restrict__ regions,
                  const int64_t *__restrict__ n_regions_p, const GearSrc gear,
                  int32_t k, int32_t min_size, int32_t max_size, int32_t *__restrict__ st_start,
                  int32_t *__restrict__ st_len, uint8_t *__restrict__ st_forced,
                  uint64_t *__restrict__ st_fp, int32_t *__restrict__ r_count, int dbg) {
    __shared__ __align__(16) uint64_t sG[3][RG_TILE];
#if IRM_CDC_PRODUCE
    __shared__ uint64_t sX[2 * RG_PRODUCERS];
#else
    __shared__ uint32_t sTok[3][RG_TILE];
    __shared__ uint64_t sS31[RG_SUB];
#endif
    __shared__ uint32_t sBm[2][RG_SUB];
    __shared__ unsigned sCand[2][RG_SUB];
    __shared__ int32_t sNext[RG_SUB + 1];
    __shared__ int32_t sEmit[2];  // chunks emitted by the walker up to iteration i (by parity)
    __shared__ int32_t sCount;
    const int64_t r = blockIdx.x;
    if (r >= *n_regions_p) return;  // uniform per CTA
    const Region R = regions[r];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t *__restrict__ rt = tok + R.tok_begin;
    const uint32_t mask = (1u << k) - 1;  // k <= 20: the low word of h decides
    const int32_t t_pin = R.ends_pin ? R.len - 1 : INT32_MAX;
    const ChunkSink sink{st_start, st_len, st_forced, R.cap_off, (int32_t)(R.tok_begin - R.stream_begin)};
    const int ntiles = (R.len + RG_TILE - 1) / RG_TILE;

    uint32_t Blo = 0, Bhi = 0;  // chain: the previous 64 MSBs
    uint32_t Cprev_lo = 0;      // cand: B low word at the end of the previous tile
    int32_t start = 0, nch = 0; // walker
    // role warps take the highest warp ids
    const bool producer = warp < RG_PRODUCERS;
    const int pw = warp, ptid = threadIdx.x;
    int32_t hashed = 0;  // hashers: chunks [0, hashed) fingerprinted
    if (threadIdx.x == 0) sEmit[0] = sEmit[1] = 0;
    __syncthreads();
#if IRM_CDC_PRODUCE
    // producers: gear values of tile i (gcur), of tile i + 1 in flight, tokens of tile i + 2 in flight
    uint64_t gcur[PT];
    uint32_t tk1[PT];
    if (producer) {
        uint32_t tk0[PT];
        load_tok_pt(rt, R.len, 0, ptid, tk0);
        load_tok_pt(rt, R.len, 1, ptid, tk1);
        gear_pt<SEEDED>(gear, tk0, gcur);
    }
#else
    uint64_t gcur[RG_PER];  // producers: gear values of the tile being scanned
    if (producer) {
        stage_tokens(rt, R.len, 0, sTok[0], ptid);
        stage_tokens(rt, R.len, 1, sTok[1], ptid);
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // tile 0's tokens landed
        producer_bar();
        load_gear<SEEDED>(sTok[0], R.len, 0, gear, pw, lane, gcur);
    }
#endif
    long long t_work = 0, t_all = clock64();
    for (int i = 0; i <= ntiles + 2; ++i) {
        const long long t0 = clock64();
        if (warp == W_CHAIN) {
            if (i >= 1 && i <= ntiles && !(dbg & 4))
                chain_tile(sG[(i - 1) % 3], sBm[(i - 1) & 1], (i - 1) * RG_TILE, R.len, Blo, Bhi, lane);
        } else if (warp == W_CAND0 || warp == W_CAND1) {
            if (i >= 2 && i <= ntiles + 1)
                cand_tile(sG[(i - 2) % 3], sBm[i & 1], sCand[i & 1], (i - 2) * RG_TILE, R.len, mask,
                          Cprev_lo, warp == W_CAND1, lane);
        } else if (warp == W_WALK) {
            if (i >= 3) {
#if IRM_CDC_FUSED_WALK
                walk_tile_scalar(sCand[(i - 3) & 1], sNext, (i - 3) * RG_TILE, R.len, min_size, max_size, t_pin,
                                 start, nch, sink, lane);
#else
                walk_tile(sCand[(i - 3) & 1], (i - 3) * RG_TILE, R.len, min_size, max_size, t_pin, start,
                          nch, sink, lane);
#endif
                if (lane == 0) sEmit[i & 1] = nch;
            }
        } else if (warp >= W_HASH) {
            // the chunks emitted up to iteration i - 1 (their (start, len) were stored before the
            // barrier that closed it); tokens from L2, a quad of lanes per chunk
            const int32_t upto = sEmit[(i - 1) & 1];
            const uint32_t *__restrict__ sbase = tok + R.stream_begin;
            for (int c0 = hashed + (warp - W_HASH) * 8; c0 < upto; c0 += RG_HASHERS * 8) {  // warp-uniform
                const int c = c0 + (lane >> 2);
                const bool ok = c < upto;
                const uint64_t h = xxh64_words_quad(sbase + (ok ? st_start[R.cap_off + c] : 0),
                                                    ok ? st_len[R.cap_off + c] : 0, 0, lane);
                if (ok && (lane & 3) == 0) st_fp[R.cap_off + c] = h;
            }
            hashed = upto;
        } else if (i < ntiles && !(dbg & 2)) {
#if IRM_CDC_PRODUCE
            uint64_t gnext[PT];
            gear_pt<SEEDED>(gear, tk1, gnext);           // tile i + 1 (table form: lookups in flight)
            load_tok_pt(rt, R.len, i + 2, ptid, tk1);    // tile i + 2
            produce_tile_serial(gcur, i, sG[i % 3], sX, pw, lane, ptid);
#pragma unroll
            for (int q = 0; q < PT; ++q) gcur[q] = gnext[q];
#else
            stage_tokens(rt, R.len, i + 2, sTok[(i + 2) % 3], ptid);  // empty group past the end
            asm volatile("cp.async.wait_group 1;" ::: "memory");       // tile i + 1's tokens landed
            producer_bar();
            uint64_t gnext[RG_PER];
            load_gear<SEEDED>(sTok[(i + 1) % 3], R.len, (i + 1) * RG_TILE, gear, pw, lane, gnext);  // in flight
            produce_tile(gcur, R.len, i * RG_TILE, sG[i % 3], i ? sG[(i - 1) % 3] : nullptr, sS31, pw, lane);
#pragma unroll
            for (int q = 0; q < RG_PER; ++q) gcur[q] = gnext[q];
#endif
        }
        t_work += clock64() - t0;
        __syncthreads();
    }
    const long long t_loop = clock64() - t_all;
    if (warp == W_WALK) {
        if (start < R.len) {  // only when the region ends at the stream end
            sink.emit(lane, nch, start, R.len - start, IRM_FORCED_STREAM_END);
            ++nch;
        }
        if (lane == 0) {
            sCount = nch;
            r_count[r] = nch;
        }
    }
    __syncthreads();
    // fingerprints (fingerprint.py:28-30) of the chunks the hashers have not taken: a quad of
    // lanes per chunk, tokens from L2
    const uint32_t *__restrict__ sbase = tok + R.stream_begin;
    const int64_t cap = R.cap_off;
    const int n_chunks = sCount;
    const int first = RG_HASHERS ? sEmit[(ntiles + 1) & 1] : 0;
    for (int c0 = first + warp * 8; c0 < n_chunks; c0 += RG_THREADS / 4) {  // warp-uniform trip count
        const int c = c0 + (lane >> 2);
        const bool ok = c < n_chunks;
        const uint64_t h = xxh64_words_quad(sbase + (ok ? st_start[cap + c] : 0), ok ? st_len[cap + c] : 0,
                                            0, lane);
        if (ok && (lane & 3) == 0) st_fp[cap + c] = h;
    }
    if (dbg && (threadIdx.x & 31) == 0 && (!producer || pw == 0 || pw == 3) && R.len > 10000)  // IRM_CDC_DEBUG=1
        printf("region %lld warp %d work %lld loop %lld with-hash %lld tiles %d\n", (long long)r, warp,
               t_work, t_loop, clock64() - t_all, ntiles);
}

// ---------------------------------------------------------------- K1 split form
// G_t is windowed (64 tokens), so it need not sit on the per-region critical path:
// gear_window_kernel computes it for the whole flat token array on every SM
// (G over the flat array, ignoring region starts), and cdc_region_split_kernel only
// stages it, corrects the first 63 tokens of its region
//     G_local_t = G_flat_t - (G_flat_{rs-1} << (t - rs + 1))      (mod 2^64)
// and runs the chain / cand / walker roles. Its tile time is the roles' own.
constexpr int GW_THREADS = 256;
constexpr int GW_PER = 8;                              // sub-blocks per warp, loads batched
constexpr int GW_SUB = GW_THREADS / 32 * GW_PER - 2;   // output sub-blocks per CTA (+2 halo in front)

// (its last CTA plans the regions meanwhile: one launch instead of two)
template <bool SEEDED>
__global__ void __launch_bounds__(GW_THREADS)
gear_window_kernel(const uint32_t *__restrict__ tok, int64_t n, const GearSrc gear,
                   uint64_t *__restrict__ G, PlanArgs plan) {
    if (blockIdx.x == gridDim.x - 1) {
        plan_regions<GW_THREADS>(plan);
        return;
    }
    __shared__ uint64_t sS[(GW_SUB + 2) * 32];
    __shared__ uint64_t sS31[GW_SUB + 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nblk = gridDim.x - 1;
    for (int64_t base = (int64_t)blockIdx.x * GW_SUB * 32; base < n; base += nblk * GW_SUB * 32) {
        // in-sub-block scans S_j(l) = sum_{i<=l} g_i << (l - i); sub-block j covers base + 32 (j - 2) ..
        // (all token loads of the warp in flight, then all gear lookups, then the scans)
        uint32_t tk[GW_PER];
        uint64_t g[GW_PER];
#pragma unroll
        for (int u = 0; u < GW_PER; ++u) {
            const int64_t t = base + 32 * (warp * GW_PER + u - 2) + lane;
            tk[u] = (t >= 0 && t < n) ? __ldg(tok + t) : 0u;
        }
#pragma unroll
        for (int u = 0; u < GW_PER; ++u) {
            const int64_t t = base + 32 * (warp * GW_PER + u - 2) + lane;
            g[u] = (t >= 0 && t < n) ? gear_of<SEEDED>(gear, tk[u]) : 0ULL;
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int u = 0; u < GW_PER; ++u) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, g[u], d);
                if (lane >= d) g[u] += y << d;
            }
        }
#pragma unroll
        for (int u = 0; u < GW_PER; ++u) {
            const int j = warp * GW_PER + u;
            sS[j * 32 + lane] = g[u];
            if (lane == 31) sS31[j] = g[u];
        }
        __syncthreads();
        for (int j = 2 + warp; j < GW_SUB + 2; j += GW_THREADS / 32) {
            const int64_t t = base + 32 * (j - 2) + lane;
            // carry-in G_{first-1} = S31(j-1) + (S31(j-2) << 32)
            const uint64_t gb = sS31[j - 1] + (sS31[j - 2] << 32);
            if (t < n) G[t] = sS[j * 32 + lane] + (gb << (lane + 1));
        }
        __syncthreads();
    }
}

#ifndef IRM_CDC2_THREADS
#define IRM_CDC2_THREADS 256
#endif
constexpr int RG2_THREADS = IRM_CDC2_THREADS;
constexpr int RG2_LOADERS = RG2_THREADS / 32 - 4;
constexpr int W2_WALK = RG2_LOADERS, W2_CAND = RG2_LOADERS + 1, W2_CHAIN = RG2_LOADERS + 3;

// G of tile `tile` into sGdst with 8-byte cp.async (zero-filled past the region end)
__device__ __forceinline__ void stage_G(const uint64_t *__restrict__ rG, int32_t len, int32_t tile,
                                        uint64_t *sGdst, int ptid) {
    const int32_t base = tile * RG_TILE;
    for (int i = ptid; i < RG_TILE; i += RG2_LOADERS * 32) {
        const bool in = base + i < len;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(sGdst + i)),
                     "l"(rG + (in ? base + i : 0)), "r"(in ? 8 : 0)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(RG2_THREADS)
cdc_region_split_kernel(const uint32_t *__restrict__ tok, const uint64_t *__restrict__ Gflat,
                   const Region *__restrict__ regions, const int64_t *__restrict__ n_regions_p, int32_t k,
                   int32_t min_size, int32_t max_size, int32_t *__restrict__ st_start,
                   int32_t *__restrict__ st_len, uint8_t *__restrict__ st_forced,
                   uint64_t *__restrict__ st_fp, int32_t *__restrict__ r_count, int dbg) {
    __shared__ uint64_t sG[4][RG_TILE];
    __shared__ uint32_t sBm[2][RG_SUB];
    __shared__ unsigned sCand[2][RG_SUB];
    __shared__ int32_t sNext[RG_SUB + 1];

    const int64_t r = blockIdx.x;
    if (r >= *n_regions_p) return;  // uniform per CTA
    const Region R = regions[r];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t *__restrict__ rG = Gflat + R.tok_begin;
    const uint32_t mask = (1u << k) - 1;
    const int32_t t_pin = R.ends_pin ? R.len - 1 : INT32_MAX;
    const ChunkSink sink{st_start, st_len, st_forced, R.cap_off, (int32_t)(R.tok_begin - R.stream_begin)};
    const int ntiles = (R.len + RG_TILE - 1) / RG_TILE;

    uint32_t Blo = 0, Bhi = 0;
    uint32_t Cprev_lo = 0;
    int32_t start = 0, nch = 0;
    const int ptid = threadIdx.x;
    const uint64_t Gcut = R.tok_begin > 0 ? Gflat[R.tok_begin - 1] : 0ULL;  // G_flat_{rs-1}
    if (warp < W2_WALK) stage_G(rG, R.len, 0, sG[0], ptid);
    long long t_work = 0, t_all = clock64();
    for (int i = 0; i <= ntiles + 2; ++i) {
        const long long t0 = clock64();
        if (warp == W2_CHAIN) {
            if (i >= 1 && i <= ntiles && !(dbg & 4))
                chain_tile(sG[(i - 1) & 3], sBm[(i - 1) & 1], (i - 1) * RG_TILE, R.len, Blo, Bhi, lane);
        } else if (warp == W2_CAND || warp == W2_CAND + 1) {
            if (i >= 2 && i <= ntiles + 1)
                cand_tile(sG[(i - 2) & 3], sBm[i & 1], sCand[i & 1], (i - 2) * RG_TILE, R.len, mask,
                          Cprev_lo, warp - W2_CAND, lane);
        } else if (warp == W2_WALK) {
            if (i >= 3)
                walk_tile_scalar(sCand[(i - 3) & 1], sNext, (i - 3) * RG_TILE, R.len, min_size, max_size, t_pin,
                                 start, nch, sink, lane);
        } else {
            if (i < ntiles) {
                if (i + 1 < ntiles) stage_G(rG, R.len, i + 1, sG[(i + 1) & 3], ptid);
                else asm volatile("cp.async.commit_group;" ::: "memory");
                asm volatile("cp.async.wait_group 1;" ::: "memory");  // this thread's part of tile i landed
                // the region's first 63 tokens: drop the window's part before the region start
                // (each thread fixes the elements it staged itself)
                if (i == 0 && Gcut)
                    for (int t = ptid; t < 63 && t < R.len; t += RG2_LOADERS * 32) sG[0][t] -= Gcut << (t + 1);
            }
        }
        t_work += clock64() - t0;
        __syncthreads();
    }
    const long long t_loop = clock64() - t_all;
    if (warp == W2_WALK) {
        if (start < R.len) {
            sink.emit(lane, nch, start, R.len - start, IRM_FORCED_STREAM_END);
            ++nch;
        }
        if (lane == 0) r_count[r] = nch;
    }
    if (dbg && (threadIdx.x & 31) == 0 && (warp >= W2_WALK || warp == 0) && R.len > 10000)
        printf("region-split %lld warp %d work %lld loop %lld tiles %d\n", (long long)r, warp, t_work, t_loop, ntiles);
}

// fingerprints + compaction (split K1), over every chunk of the batch on every SM: a quad
// of lanes per chunk (fingerprint.py:28-30), the chunk's region found by binary search
// over the regions' output offsets. The split form runs only for batches of at most
// HC_THREADS regions, so every CTA scans the region chunk counts itself (the offsets pass
// folded in; CTA 0 publishes chunk_off).
constexpr int HC_THREADS = 256;

// r_out_g == nullptr: at most HC_THREADS regions, every CTA scans their counts itself;
// otherwise the region offsets come from cdc_offsets_kernel (r_out_g, chunk_off written).
__global__ void __launch_bounds__(HC_THREADS)
cdc_hash_compact_kernel(const uint32_t *__restrict__ tok, const int64_t *__restrict__ n_regions_p,
                        const Region *__restrict__ regions, const int32_t *__restrict__ r_count,
                        const int64_t *__restrict__ r_first, int32_t n_streams, int64_t *__restrict__ chunk_off,
                        const int32_t *__restrict__ st_start, const int32_t *__restrict__ st_len,
                        const uint8_t *__restrict__ st_forced, int32_t *__restrict__ c_start,
                        int32_t *__restrict__ c_len, uint64_t *__restrict__ c_fp, uint8_t *__restrict__ c_forced,
                        const int64_t *__restrict__ r_out_g) {
    __shared__ int64_t sScan[HC_THREADS / 32];
    __shared__ int64_t r_out_s[HC_THREADS + 1];
    const int64_t nr = *n_regions_p;
    const int64_t *r_out = r_out_g ? r_out_g : r_out_s;
    if (!r_out_g) {  // nr <= HC_THREADS (host-checked bound)
        const int64_t c = threadIdx.x < nr ? r_count[threadIdx.x] : 0;
        int64_t tot;
        const int64_t ex = block_exclusive_scan<HC_THREADS>(c, &tot, sScan);
        if (threadIdx.x < nr) r_out_s[threadIdx.x] = ex;
        if (threadIdx.x == 0) r_out_s[nr] = tot;
        __syncthreads();
        if (blockIdx.x == 0)
            for (int32_t s = threadIdx.x; s <= n_streams; s += HC_THREADS) chunk_off[s] = r_out_s[r_first[s]];
    }
    const int64_t total = r_out[nr];
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * 64;
    for (int64_t q0 = (int64_t)blockIdx.x * 64 + (threadIdx.x >> 5) * 8; q0 < total; q0 += stride) {
        const int64_t q = q0 + (lane >> 2);
        const bool ok = q < total;
        int64_t lo = 0, hi = nr - 1;  // last region with r_out[r] <= q
        while (ok && lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (r_out[mid] <= q) lo = mid;
            else hi = mid - 1;
        }
        const int64_t src = ok ? regions[lo].cap_off + (q - r_out[lo]) : 0;
        const int32_t st = ok ? st_start[src] : 0, ln = ok ? st_len[src] : 0;
        const uint64_t h = xxh64_words_quad(tok + (ok ? regions[lo].stream_begin : 0) + st, ln, 0, lane);
        if (ok && (lane & 3) == 0) {
            c_start[q] = st;
            c_len[q] = ln;
            c_fp[q] = h;
            c_forced[q] = st_forced[src];
        }
    }
}

__global__ void __launch_bounds__(PLAN_BLOCK)
cdc_offsets_kernel(const int64_t *__restrict__ n_regions_p, const int32_t *__restrict__ r_count,
                   int64_t *__restrict__ r_out, const int64_t *__restrict__ r_first,
                   int32_t n_streams, int64_t *__restrict__ chunk_off) {
    __shared__ int64_t sm[PLAN_BLOCK / 32];
    const int64_t nr = *n_regions_p;
    int64_t carry = 0;
    for (int64_t r0 = 0; r0 < nr; r0 += PLAN_BLOCK) {
        const int64_t r = r0 + threadIdx.x;
        const int64_t c = r < nr ? r_count[r] : 0;
        int64_t tot;
        const int64_t ex = block_exclusive_scan<PLAN_BLOCK>(c, &tot, sm);
        if (r < nr) r_out[r] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) r_out[nr] = carry;
    __syncthreads();
    for (int32_t s = threadIdx.x; s <= n_streams; s += PLAN_BLOCK) chunk_off[s] = r_out[r_first[s]];
}

__global__ void __launch_bounds__(128)
cdc_compact_kernel(const int64_t *__restrict__ n_regions_p, const Region *__restrict__ regions,
                   const int32_t *__restrict__ r_count, const int64_t *__restrict__ r_out,
                   const int32_t *__restrict__ st_start, const int32_t *__restrict__ st_len,
                   const uint8_t *__restrict__ st_forced, const uint64_t *__restrict__ st_fp,
                   int32_t *__restrict__ c_start, int32_t *__restrict__ c_len,
                   uint64_t *__restrict__ c_fp, uint8_t *__restrict__ c_forced) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= *n_regions_p) return;
    const int64_t src = regions[r].cap_off, dst = r_out[r];
    const int32_t n = r_count[r];
    for (int32_t i = lane; i < n; i += 32) {
        c_start[dst + i] = st_start[src + i];
        c_len[dst + i] = st_len[src + i];
        c_fp[dst + i] = st_fp[src + i];
        c_forced[dst + i] = st_forced[src + i];
    }
}

__global__ void xxh64_spans_kernel(const uint8_t *__restrict__ base, const int64_t *__restrict__ off,
                                   const int64_t *__restrict__ len, int64_t n, uint64_t seed,
                                   uint64_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t o = off[i], l = len[i];
    // token spans (4-byte aligned, whole words) take the word path
    if (((o | l) & 3) == 0 && (((uintptr_t)base) & 3) == 0)
        out[i] = xxh64_words(reinterpret_cast<const uint32_t *>(base + o), l / 4, seed);
    else
        out[i] = xxh64_bytes(base + o, l, seed);
}

// ------------------------------------------------------------- workspace
struct CdcWs {
    Region *regions;
    int64_t *r_first, *n_regions, *r_out;
    int32_t *r_count, *st_start, *st_len;
    uint8_t *st_forced;
    uint64_t *st_fp;
    uint64_t *G;
    int64_t bytes;
};

static inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

static CdcWs carve_cdc_ws(void *ws, int64_t n_tokens, int32_t n_streams, int64_t n_pins,
                          int32_t min_size) {
    const int64_t rmax = (int64_t)n_streams + n_pins + 1;
    const int64_t smax = n_tokens / min_size + rmax + 1;
    CdcWs w{};
    char *p = (char *)ws;
    int64_t o = 0;
    auto take = [&](int64_t bytes) {
        char *q = p ? p + o : nullptr;
        o = align_up(o + bytes, 256);
        return q;
    };
    w.regions = (Region *)take(rmax * sizeof(Region));
    w.r_first = (int64_t *)take((n_streams + 1) * sizeof(int64_t));
    w.n_regions = (int64_t *)take(sizeof(int64_t));
    w.r_out = (int64_t *)take((rmax + 1) * sizeof(int64_t));
    w.r_count = (int32_t *)take(rmax * sizeof(int32_t));
    w.st_start = (int32_t *)take(smax * sizeof(int32_t));
    w.st_len = (int32_t *)take(smax * sizeof(int32_t));
    w.st_fp = (uint64_t *)take(smax * sizeof(uint64_t));
    w.st_forced = (uint8_t *)take(smax);
    w.G = (uint64_t *)take(n_tokens * sizeof(uint64_t));
    w.bytes = o;
    return w;
}

}  // namespace irm

using namespace irm;

extern "C" int irm_gear_table(uint64_t seed, uint64_t *out, irm_stream_t stream) {
    IRM_REQUIRE(out != nullptr, "irm_gear_table: out is null");
    gear_table_kernel<<<65536 / 256, 256, 0, (cudaStream_t)stream>>>(seed, out);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int64_t irm_cdc_chunk_bound(int64_t n_tokens, int32_t n_streams, int64_t n_pins,
                                       int32_t min_size) {
    if (min_size < 1) return -1;
    return n_tokens / min_size + (int64_t)n_streams + n_pins + 1;
}

extern "C" int64_t irm_cdc_workspace_bytes(int64_t n_tokens, int32_t n_streams, int64_t n_pins,
                                           int32_t min_size) {
    if (min_size < 1 || n_streams < 0 || n_tokens < 0 || n_pins < 0) return -1;
    return carve_cdc_ws(nullptr, n_tokens, n_streams, n_pins, min_size).bytes;
}

static int cdc_xxh64_impl(const uint32_t *tok, int64_t n_tokens, const int64_t *stream_off,
                          int32_t n_streams, const int64_t *pin_off, const int64_t *pins,
                          int64_t n_pins, int32_t mask_exponent, int32_t min_size,
                          int32_t max_size, int32_t marker_pinned, const GearSrc gear, bool seeded,
                          int32_t *c_start, int32_t *c_len, uint64_t *c_fp, uint8_t *c_forced,
                          int64_t *chunk_off, int64_t cap, void *ws, int64_t ws_bytes,
                          irm_stream_t stream) {
    // ChunkerParams validation, chunking.py:45-49
    IRM_REQUIRE(mask_exponent >= 1 && mask_exponent <= 20, "mask_exponent must be in [1, 20]");
    IRM_REQUIRE(min_size >= 1 && min_size < max_size, "need 1 <= min_size < max_size");
    IRM_REQUIRE(n_streams >= 0 && n_tokens >= 0 && n_pins >= 0, "negative sizes");
    IRM_REQUIRE(n_tokens < (int64_t)1 << 40, "n_tokens too large");
    IRM_REQUIRE(stream_off && chunk_off, "null stream_off/chunk_off");
    IRM_REQUIRE(n_tokens == 0 || (tok && (seeded || gear.table)), "null tok/gear");
    if (marker_pinned && n_pins > 0) IRM_REQUIRE(pin_off && pins, "null pins");
    const int64_t bound = irm_cdc_chunk_bound(n_tokens, n_streams, marker_pinned ? n_pins : 0,
                                              min_size);
    if (cap < bound) {
        set_error("chunk capacity %lld < bound %lld", (long long)cap, (long long)bound);
        return IRM_ECAPACITY;
    }
    const int64_t np = marker_pinned ? n_pins : 0;
    CdcWs w = carve_cdc_ws(ws, n_tokens, n_streams, np, min_size);
    if (ws_bytes < w.bytes || ws == nullptr) {
        set_error("workspace %lld < %lld bytes", (long long)ws_bytes, (long long)w.bytes);
        return IRM_ECAPACITY;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (n_streams == 0) {
        IRM_CUDA_CHECK(cudaMemsetAsync(chunk_off, 0, sizeof(int64_t), st));
        return IRM_OK;
    }
    const int32_t use_pins = marker_pinned && n_pins > 0;
    const PlanArgs plan{stream_off, n_streams, pin_off, pins, use_pins, min_size, w.regions, w.r_first, w.n_regions};
    const int64_t rmax = (int64_t)n_streams + np;
    const int dbg = getenv("IRM_CDC_DEBUG") ? atoi(getenv("IRM_CDC_DEBUG")) : 0;
    // two forms, same results: "fused" (G computed inside the region kernel; many regions in
    // flight hide its latency) and "split" (G on every SM first, hashing on every SM after;
    // shortest critical path when a few long regions leave most SMs idle)
    const char *form = getenv("IRM_CDC_FORM");
    const bool v1 = form ? strcmp(form, "fused") == 0 : rmax >= sm_count();
    if (v1) {
        cdc_plan_kernel<<<1, PLAN_BLOCK, 0, st>>>(plan);
        IRM_LAUNCH_CHECK();
        (seeded ? cdc_region_kernel<true> : cdc_region_kernel<false>)<<<(unsigned)rmax, RG_THREADS, 0, st>>>(
            tok, w.regions, w.n_regions, gear, mask_exponent, min_size, max_size, w.st_start, w.st_len,
            w.st_forced, w.st_fp, w.r_count, dbg);
    } else {
        const int64_t gw_tiles = (n_tokens + GW_SUB * 32 - 1) / (GW_SUB * 32);
        (seeded ? gear_window_kernel<true> : gear_window_kernel<false>)
            <<<(unsigned)(std::max<int64_t>(1, std::min<int64_t>(gw_tiles, (int64_t)sm_count() * 8)) + 1),
               GW_THREADS, 0, st>>>(tok, n_tokens, gear, w.G, plan);
        IRM_LAUNCH_CHECK();
        cdc_region_split_kernel<<<(unsigned)rmax, RG2_THREADS, 0, st>>>(
            tok, w.G, w.regions, w.n_regions, mask_exponent, min_size, max_size, w.st_start, w.st_len,
            w.st_forced, w.st_fp, w.r_count, dbg);
    }
    IRM_LAUNCH_CHECK();
    if (v1) {
        cdc_offsets_kernel<<<1, PLAN_BLOCK, 0, st>>>(w.n_regions, w.r_count, w.r_out, w.r_first,
                                                     n_streams, chunk_off);
        IRM_LAUNCH_CHECK();
        cdc_compact_kernel<<<(unsigned)((rmax + 3) / 4), 128, 0, st>>>(
            w.n_regions, w.regions, w.r_count, w.r_out, w.st_start, w.st_len, w.st_forced, w.st_fp,
            c_start, c_len, c_fp, c_forced);
    } else {
        const bool many = rmax > HC_THREADS;
        if (many) {
            cdc_offsets_kernel<<<1, PLAN_BLOCK, 0, st>>>(w.n_regions, w.r_count, w.r_out, w.r_first, n_streams,
                                                         chunk_off);
            IRM_LAUNCH_CHECK();
        }
        const int64_t blocks = std::min<int64_t>((bound + 63) / 64, (int64_t)sm_count() * 8);
        cdc_hash_compact_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), HC_THREADS, 0, st>>>(
            tok, w.n_regions, w.regions, w.r_count, w.r_first, n_streams, chunk_off, w.st_start, w.st_len,
            w.st_forced, c_start, c_len, c_fp, c_forced, many ? w.r_out : nullptr);
    }
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}

extern "C" int irm_cdc_xxh64(const uint32_t *tok, int64_t n_tokens, const int64_t *stream_off,
                             int32_t n_streams, const int64_t *pin_off, const int64_t *pins,
                             int64_t n_pins, int32_t mask_exponent, int32_t min_size,
                             int32_t max_size, int32_t marker_pinned, const uint64_t *gear,
                             int32_t *c_start, int32_t *c_len, uint64_t *c_fp, uint8_t *c_forced,
                             int64_t *chunk_off, int64_t cap, void *ws, int64_t ws_bytes,
                             irm_stream_t stream) {
    return cdc_xxh64_impl(tok, n_tokens, stream_off, n_streams, pin_off, pins, n_pins, mask_exponent, min_size,
                          max_size, marker_pinned, GearSrc{gear, 0}, false, c_start, c_len, c_fp, c_forced,
                          chunk_off, cap, ws, ws_bytes, stream);
}

extern "C" int irm_cdc_xxh64_seeded(const uint32_t *tok, int64_t n_tokens, const int64_t *stream_off,
                                    int32_t n_streams, const int64_t *pin_off, const int64_t *pins,
                                    int64_t n_pins, int32_t mask_exponent, int32_t min_size,
                                    int32_t max_size, int32_t marker_pinned, uint64_t gear_seed,
                                    int32_t *c_start, int32_t *c_len, uint64_t *c_fp, uint8_t *c_forced,
                                    int64_t *chunk_off, int64_t cap, void *ws, int64_t ws_bytes,
                                    irm_stream_t stream) {
    return cdc_xxh64_impl(tok, n_tokens, stream_off, n_streams, pin_off, pins, n_pins, mask_exponent, min_size,
                          max_size, marker_pinned, GearSrc{nullptr, gear_seed}, true, c_start, c_len, c_fp,
                          c_forced, chunk_off, cap, ws, ws_bytes, stream);
}

extern "C" int irm_xxh64_spans(const uint8_t *base, const int64_t *off, const int64_t *len,
                               int64_t n, uint64_t seed, uint64_t *out, irm_stream_t stream) {
    IRM_REQUIRE(n >= 0, "n must be >= 0");
    if (n == 0) return IRM_OK;
    IRM_REQUIRE(off && len && out, "null pointer");
    xxh64_spans_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        base, off, len, n, seed, out);
    IRM_LAUNCH_CHECK();
    return IRM_OK;
}
