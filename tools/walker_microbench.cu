// Microbenchmark of the K1 walker (boundary rule over candidate words, chunking.py:116-124):
// one warp walks NT tiles of 1024 tokens whose candidate words are random with density 1/128
// (mask_exponent 7), min 32, max 512. Variants: the scalar walker of cdc.cu, the same without
// the chunk stores, and a register form (candidate words and next-word table in lanes, read by
// shuffles). nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/walker_mb tools/walker_microbench.cu
#include <cstdio>
#include <cstdint>
#include <climits>
#include <cstdlib>

constexpr int TILE = 1024;

template <int VAR>
__global__ void walk(const unsigned *cand_g, int nt, int min_size, int max_size, int *out_start, int *out_len,
                     long long *cyc, int *nch_out) {
    __shared__ unsigned sCand[32];
    __shared__ int sNext[33];
    __shared__ unsigned sAll[64 * 32];  // every tile's candidate words, staged before the clock starts
    const int lane = threadIdx.x;
    for (int i = lane; i < nt * 32; i += 32) sAll[i] = cand_g[i];
    __syncwarp();
    int start = 0, nch = 0;
    long long t0 = clock64();
    for (int tile = 0; tile < nt; ++tile) {
        const int tile_start = tile * TILE;
        const unsigned my_cand = sAll[tile * 32 + lane];
        int nc = my_cand ? tile_start + 32 * lane + __ffs(my_cand) - 1 : INT_MAX;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_down_sync(0xffffffffu, nc, d);
            if (lane + d < 32) nc = min(nc, y);
        }
        if (VAR == 5) {
            // per-position jump table, transposed build: lane L fills offsets 32 w + L of every word w
            // (conflict-free u16 stores); the word's bits at or above L, else the next word's first
            __shared__ unsigned short jt5[TILE];
            __shared__ unsigned sC[32];
            __shared__ int sN[33];
            sC[lane] = my_cand;
            sN[lane] = nc == INT_MAX ? 0xFFFF : nc - tile_start;  // first candidate at or after word lane
            if (lane == 0) sN[32] = 0xFFFF;
            __syncwarp();
            const unsigned above = 0xffffffffu << lane;
#pragma unroll 8
            for (int w = 0; w < 32; ++w) {
                const unsigned m = sC[w] & above;
                jt5[32 * w + lane] = (unsigned short)(m ? 32 * w + __ffs(m) - 1 : sN[w + 1]);
            }
            __syncwarp();
            if (lane == 0) {
                const int tile_end = tile_start + TILE;
                while (true) {
                    const int t_max = start + max_size - 1;
                    const int rel = max(0, start + min_size - 1 - tile_start);
                    const int j = rel < TILE ? jt5[rel] : 0xFFFF;
                    const int t_cand = j == 0xFFFF ? INT_MAX : tile_start + j;
                    const int nxt = min(t_max, t_cand);
                    if (nxt >= tile_end) break;
                    out_start[nch] = start;
                    out_len[nch] = nxt - start + 1;
                    ++nch;
                    start = nxt + 1;
                }
            }
            __syncwarp();
        } else if (VAR == 4) {
            // per-position jump table: jt[r] = first candidate at or after tile offset r (0xFFFF: none
            // in this tile), built by the warp; lane 0 then needs ONE shared load per chunk
            __shared__ unsigned short jt[TILE];
            int nx = __shfl_down_sync(0xffffffffu, nc, 1);
            nx = (lane == 31 || nx == INT_MAX) ? 0xFFFF : nx - tile_start;
#pragma unroll
            for (int b = 31; b >= 0; --b) {
                if ((my_cand >> b) & 1u) nx = 32 * lane + b;
                jt[32 * lane + b] = (unsigned short)nx;
            }
            __syncwarp();
            if (lane == 0) {
                const int tile_end = tile_start + TILE;
                while (true) {
                    const int t_max = start + max_size - 1;
                    const int rel = max(0, start + min_size - 1 - tile_start);
                    const int j = rel < TILE ? jt[rel] : 0xFFFF;
                    const int t_cand = j == 0xFFFF ? INT_MAX : tile_start + j;
                    const int nxt = min(t_max, t_cand);
                    if (nxt >= tile_end) break;
                    out_start[nch] = start;
                    out_len[nch] = nxt - start + 1;
                    ++nch;
                    start = nxt + 1;
                }
            }
            __syncwarp();
        } else if (VAR == 3) {
            // branch-free step: clamped word index, both loads unconditional, selects
            sCand[lane] = my_cand;
            sNext[lane] = nc;
            if (lane == 0) sNext[32] = INT_MAX;
            __syncwarp();
            if (lane == 0) {
                const int tile_end = tile_start + TILE;
                while (true) {
                    const int t_max = start + max_size - 1;
                    const int rel = max(0, start + min_size - 1 - tile_start);
                    const int w = min(rel >> 5, 31);
                    const unsigned m = rel < TILE ? (0xffffffffu << (rel & 31)) : 0u;
                    const unsigned cw = sCand[w] & m;
                    const int nx = rel < TILE ? sNext[w + 1] : INT_MAX;
                    const int hitp = tile_start + 32 * w + __ffs(cw) - 1;
                    const int t_cand = cw ? hitp : nx;
                    const int nxt = min(t_max, t_cand);
                    if (nxt >= tile_end) break;
                    out_start[nch] = start;
                    out_len[nch] = nxt - start + 1;
                    ++nch;
                    start = nxt + 1;
                }
            }
            __syncwarp();
        } else if (VAR <= 1) {
            sCand[lane] = my_cand;
            sNext[lane] = nc;
            if (lane == 0) sNext[32] = INT_MAX;
            __syncwarp();
            if (lane == 0) {
                const int tile_end = tile_start + TILE;
                while (true) {
                    const int t_max = start + max_size - 1;
                    const int rel = max(0, start + min_size - 1 - tile_start);
                    int t_cand = INT_MAX;
                    if (rel < TILE) {
                        const int w = rel >> 5;
                        const unsigned cw = sCand[w] & (0xffffffffu << (rel & 31));
                        const int nx = sNext[w + 1];
                        t_cand = cw ? tile_start + 32 * w + __ffs(cw) - 1 : nx;
                    }
                    const int nxt = min(t_max, t_cand);
                    if (nxt >= tile_end) break;
                    if (VAR == 0) {
                        out_start[nch] = start;
                        out_len[nch] = nxt - start + 1;
                    }
                    ++nch;
                    start = nxt + 1;
                }
            }
            __syncwarp();
        } else {
            // VAR 2: the whole warp walks; candidate words and next table stay in lanes (shuffles)
            const int tile_end = tile_start + TILE;
            int nxw = __shfl_down_sync(0xffffffffu, nc, 1);
            if (lane == 31) nxw = INT_MAX;  // first candidate at or after word lane + 1
            while (true) {
                const int t_max = start + max_size - 1;
                const int rel = max(0, start + min_size - 1 - tile_start);
                const int w = min(rel >> 5, 31);
                const unsigned cw = __shfl_sync(0xffffffffu, my_cand, w) & (rel < TILE ? (0xffffffffu << (rel & 31)) : 0u);
                const int nx = __shfl_sync(0xffffffffu, nxw, w);
                const int t_cand = rel < TILE ? (cw ? tile_start + 32 * w + __ffs(cw) - 1 : nx) : INT_MAX;
                const int nxt = min(t_max, t_cand);
                if (nxt >= tile_end) break;
                if (lane == 0) {
                    out_start[nch] = start;
                    out_len[nch] = nxt - start + 1;
                }
                ++nch;
                start = nxt + 1;
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) {
        cyc[VAR] = t1 - t0;
        nch_out[VAR] = nch;
    }
}

int main() {
    const int nt = 64;
    unsigned *h = (unsigned *)malloc(nt * 32 * 4);
    srand(3);
    for (int i = 0; i < nt * 32; ++i) {
        unsigned w = 0;
        for (int b = 0; b < 32; ++b)
            if (rand() % 128 == 0) w |= 1u << b;
        h[i] = w;
    }
    unsigned *cand;
    int *os, *ol, *nch;
    long long *cyc;
    cudaMalloc(&cand, nt * 32 * 4);
    cudaMalloc(&os, 1 << 20);
    cudaMalloc(&ol, 1 << 20);
    cudaMalloc(&cyc, 64);
    cudaMalloc(&nch, 64);
    cudaMemcpy(cand, h, nt * 32 * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
        walk<0><<<1, 32>>>(cand, nt, 32, 512, os, ol, cyc, nch);
        walk<1><<<1, 32>>>(cand, nt, 32, 512, os, ol, cyc, nch);
        walk<2><<<1, 32>>>(cand, nt, 32, 512, os, ol, cyc, nch);
        walk<3><<<1, 32>>>(cand, nt, 32, 512, os, ol, cyc, nch);
        walk<4><<<1, 32>>>(cand, nt, 32, 512, os, ol, cyc, nch);
        walk<5><<<1, 32>>>(cand, nt, 32, 512, os, ol, cyc, nch);
    }
    long long c[6];
    int n[6];
    cudaMemcpy(c, cyc, 48, cudaMemcpyDeviceToHost);
    cudaMemcpy(n, nch, 24, cudaMemcpyDeviceToHost);
    const char *names[] = {"scalar lane 0 (cdc.cu)", "scalar, no stores", "warp + shuffles", "scalar, branch-free",
                           "per-position jump table", "jump table, transposed build"};
    for (int i = 0; i < 6; ++i)
        printf("%-24s %lld cycles, %d chunks: %.1f cycles/chunk, %.0f cycles/tile\n", names[i], c[i], n[i],
               (double)c[i] / n[i], (double)c[i] / nt);
    return 0;
}
