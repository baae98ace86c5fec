// Microbenchmark of the CDC chain-warp step variants (one warp, clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_mb tools/chain_microbench.cu
#include <cstdio>
#include <cstdint>

__global__ void bench(const uint64_t *G, uint32_t *out, long long *cyc, int steps) {
    __shared__ uint64_t sG[1024];
    __shared__ uint32_t sBm[1024];
    const int lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sG[i] = G[i];
    __syncwarp();
    uint32_t Blo = 0, Bhi = 0;
    long long t0, t1;
    // variant 0: ballot + brev only (the loop-carried core)
    t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const uint32_t Ghi = (uint32_t)(sG[(s & 31) * 32 + lane] >> 32);
        const uint32_t hs = Ghi + __funnelshift_l(Blo, Bhi, lane);
        const unsigned M = __ballot_sync(0xffffffffu, hs >> 31);
        Bhi = Blo;
        Blo = __brev(M);
    }
    t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    out[lane] = Blo ^ Bhi;
    // variant 1: + und ballot + branch
    Blo = Bhi = 0;
    t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const uint32_t Ghi = (uint32_t)(sG[(s & 31) * 32 + lane] >> 32);
        const uint32_t hs = Ghi + __funnelshift_l(Blo, Bhi, lane);
        unsigned M = __ballot_sync(0xffffffffu, hs >> 31);
        const unsigned und = __ballot_sync(0xffffffffu, (hs & 0x7FFFFFFEu) == 0x7FFFFFFEu);
        if (__builtin_expect(und != 0, 0)) M ^= und;
        Bhi = Blo;
        Blo = __brev(M);
    }
    t1 = clock64();
    if (lane == 0) cyc[1] = t1 - t0;
    out[32 + lane] = Blo ^ Bhi;
    // variant 2: + store of B word every step (all lanes, same address)
    Blo = Bhi = 0;
    t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const uint32_t Ghi = (uint32_t)(sG[(s & 31) * 32 + lane] >> 32);
        const uint32_t hs = Ghi + __funnelshift_l(Blo, Bhi, lane);
        unsigned M = __ballot_sync(0xffffffffu, hs >> 31);
        const unsigned und = __ballot_sync(0xffffffffu, (hs & 0x7FFFFFFEu) == 0x7FFFFFFEu);
        if (__builtin_expect(und != 0, 0)) M ^= und;
        Bhi = Blo;
        Blo = __brev(M);
        sBm[s & 1023] = Blo;
    }
    t1 = clock64();
    if (lane == 0) cyc[2] = t1 - t0;
    out[64 + lane] = Blo ^ Bhi;
    // variant 3: + lane-0 divergent store
    Blo = Bhi = 0;
    t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const uint32_t Ghi = (uint32_t)(sG[(s & 31) * 32 + lane] >> 32);
        const uint32_t hs = Ghi + __funnelshift_l(Blo, Bhi, lane);
        unsigned M = __ballot_sync(0xffffffffu, hs >> 31);
        const unsigned und = __ballot_sync(0xffffffffu, (hs & 0x7FFFFFFEu) == 0x7FFFFFFEu);
        if (__builtin_expect(und != 0, 0)) M ^= und;
        Bhi = Blo;
        Blo = __brev(M);
        if (lane == 0) sBm[s & 1023] = Blo;
    }
    t1 = clock64();
    if (lane == 0) cyc[3] = t1 - t0;
    out[96 + lane] = Blo ^ Bhi ^ sBm[lane];
    // variant 4: match.any-free: ballot via __any? use redux instead of brev: vote only
    Blo = Bhi = 0;
    t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const uint32_t hs = Blo + lane;
        Blo = __ballot_sync(0xffffffffu, hs >> 31);
    }
    t1 = clock64();
    if (lane == 0) cyc[4] = t1 - t0;
    out[128 + lane] = Blo;
    // variant 5: brev only chain
    Blo = lane;
    t0 = clock64();
    for (int s = 0; s < steps; ++s) Blo = __brev(Blo + 1);
    t1 = clock64();
    if (lane == 0) cyc[5] = t1 - t0;
    out[160 + lane] = Blo;
    // variant 6: shfl-broadcast chain (alternative to ballot)
    Blo = lane;
    t0 = clock64();
    for (int s = 0; s < steps; ++s) Blo = __shfl_sync(0xffffffffu, Blo + 1, 3);
    t1 = clock64();
    if (lane == 0) cyc[6] = t1 - t0;
    out[192 + lane] = Blo;
    // variant 7: the shipped chain step (cdc.cu chain_tile, IRM_CDC_CHAIN_LEAN): lane j = 31 - lane so
    // the ballot is already bit-reversed, G's high word by a 32-bit load 4 steps ahead, carry-boundary
    // test OR-accumulated, lane 0 stores W
    {
        const int j = 31 - lane;
        const uint32_t *sGhi = reinterpret_cast<const uint32_t *>(sG) + 1;
        uint32_t Blo7 = 0, Bhi7 = 0, acc = 0;
        uint32_t Gq[4];
        for (int a = 0; a < 4; ++a) Gq[a] = sGhi[2 * (a * 32 + j)];
        t0 = clock64();
#pragma unroll 4
        for (int s = 0; s < steps; ++s) {
            const uint32_t Ghi = Gq[0];
            Gq[0] = Gq[1];
            Gq[1] = Gq[2];
            Gq[2] = Gq[3];
            Gq[3] = sGhi[2 * (((s + 4) & 31) * 32 + j)];
            const uint32_t hs = Ghi + __funnelshift_l(Blo7, Bhi7, j);
            const unsigned W = __ballot_sync(0xffffffffu, (int32_t)hs < 0);
            acc |= (hs + 2u) ^ hs;
            if (lane == 0) sBm[s & 1023] = W;
            Bhi7 = Blo7;
            Blo7 = W;
        }
        t1 = clock64();
        if (lane == 0) cyc[7] = t1 - t0;
        out[224 + lane] = Blo7 ^ acc;
    }
}

int main() {
    uint64_t *G;
    uint32_t *out;
    long long *cyc;
    cudaMalloc(&G, 8192);
    cudaMalloc(&out, 4096);
    cudaMalloc(&cyc, 64);
    cudaMemset(G, 0x5a, 8192);
    const int steps = 4096;
    for (int rep = 0; rep < 2; ++rep) bench<<<1, 32>>>(G, out, cyc, steps);
    long long h[8];
    cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
    const char *names[] = {"ballot+brev core", "+und ballot+branch", "+all-lane STS", "+lane0 STS",
                           "ballot-only chain", "brev-only chain", "shfl-only chain", "shipped lean step"};
    for (int i = 0; i < 8; ++i) printf("%-22s %.1f cycles/step\n", names[i], (double)h[i] / steps);
    return 0;
}
