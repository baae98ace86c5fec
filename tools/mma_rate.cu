// Microbenchmark: tensor-pipe cycles per K5 tile for the MMA shapes K5 issues (cta_group::2,
// M = 128, bf16, K = 16 per instruction), operands in smem (SS) or A in TMEM (TS).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_05696_b200/csrc \
//        -o tools/mma_rate tools/mma_rate.cu && tools/mma_rate
// One elected thread of the leader CTA issues `iters` tiles of a pattern back to back (no data
// dependencies, no waits), commits once and waits; cycles / tile vs the floor 128 N / 512 per
// instruction (B300_MICROARCH.md "tcgen05 floor").
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "cluster.cuh"
#include "tcgen05.cuh"

using namespace irm;

struct Pat {
    const char *name;
    int n;        // MMA N
    int ts;       // instructions with A from TMEM
    int ss;       // instructions with A from smem
    int pv;       // extra N = 256 SS instructions (PV)
    int chains;   // independent accumulators the QK instructions rotate over (1 = one dependent chain)
    int inter;    // 1: PV instructions interleaved evenly between the QK ones instead of after them
};

template <int PN, int PTS, int PSS, int PPV, int PCH, int PINT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) rate_kernel(int iters, long long *out) {
    constexpr Pat pat{"", PN, PTS, PSS, PPV, PCH, PINT};
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase_s;
    const uint32_t rank = cl::cta_rank();
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tc2::tmem_alloc(&tbase_s, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    cl::cluster_sync();
    tc::fence_after();
    const uint32_t tb = tbase_s;
    if (rank == 0 && warp == 1) {
        const uint32_t id_n = tc::idesc_bf16(128, pat.n, false, false);
        const uint32_t id_pv = tc::idesc_bf16(128, 256, false, true);
        const uint64_t a = tc::smem_desc_sw128(smem_u32(smem), 16, 1024);
        const uint64_t b = tc::smem_desc_sw128(smem_u32(smem + 64 * 1024), 16, 1024);
        const uint64_t v = tc::smem_desc_sw128(smem_u32(smem + 96 * 1024), 4096, 1024);
        const uint32_t a_lo = (uint32_t)a, a_hi = (uint32_t)(a >> 32), b_lo = (uint32_t)b, b_hi = (uint32_t)(b >> 32);
        const uint32_t v_lo = (uint32_t)v, v_hi = (uint32_t)(v >> 32);
        long long t0 = clock64();
        if (tc::elect_one()) {
            for (int it = 0; it < iters; ++it) {
                const uint32_t d0 = tb + (it & 1) * (pat.n / 2) * pat.chains;
                constexpr int nq = pat.ts + pat.ss, every = pat.pv ? (nq + pat.pv - 1) / pat.pv : 1 << 30;
                int pv_done = 0;
#pragma unroll
                for (int i = 0; i < nq; ++i) {
                    const uint32_t d = d0 + (i % pat.chains) * (pat.n / 2);
                    if (i < pat.ts)
                        tc2::mma_bf16_ts_w(d, tb + 320 + 8 * (i & 7), b_lo + 2 * (i & 3), b_hi, id_n, i >= pat.chains);
                    else
                        tc2::mma_bf16_ss_w(d, a_lo + 2 * (i & 3), a_hi, b_lo + 2 * (i & 3), b_hi, id_n, 1);
                    if (pat.inter && pv_done < pat.pv && (i + 1) % every == 0) {
                        tc2::mma_bf16_ss_w(tb + 384, a_lo + 2 * (pv_done & 3), a_hi, v_lo + 128 * (pv_done & 3), v_hi,
                                           id_pv, 1);
                        ++pv_done;
                    }
                }
#pragma unroll
                for (int j = 0; j < pat.pv; ++j) {
                    if (j < pv_done) continue;
                    tc2::mma_bf16_ss_w(tb + 384, a_lo + 2 * (j & 3), a_hi, v_lo + 128 * (j & 3), v_hi, id_pv, 1);
                }
            }
            tc2::commit_both(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = t1 - t0;
    } else if (rank == 1 && warp == 1) {
        mbar_wait(&bar, 0);
    }
    tc::fence_before();
    cl::cluster_sync();
    tc::fence_after();
    if (warp == 0) tc2::tmem_dealloc(tb, 512);
}

template <int PN, int PTS, int PSS, int PPV, int PCH, int PINT>
void run(const char *name, long long *d_out) {
    const int smem = 160 * 1024 + 1024;
    auto k = rate_kernel<PN, PTS, PSS, PPV, PCH, PINT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    long long cyc = 0;
    for (int rep = 0; rep < 3; ++rep) {
        k<<<2, 128, smem>>>(iters, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            exit(1);
        }
        cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    }
    const int n_inst = PTS + PSS;
    const double floor = n_inst * 128.0 * PN / 512 + PPV * 64.0;
    printf("  %-36s %8.1f cycles/tile  floor %6.0f  ratio %.3f  (%.1f cyc/inst)\n", name, (double)cyc / iters, floor,
           (double)cyc / iters / floor, (double)cyc / iters / (n_inst + PPV));
}

int main() {
    long long *d_out;
    cudaMalloc(&d_out, 8);
    // per K5 64-key tile: QK = 9 pieces x 4 (N = 64; 5 pieces TS, 4 SS), PV = 2 key halves x 2 dim
    // halves x 2 k-steps (N = 256)
    run<64, 20, 16, 0, 1, 0>("QK as K5 (N64: 20 TS + 16 SS)", d_out);
    run<64, 0, 36, 0, 1, 0>("QK all SS (N64 x 36)", d_out);
    run<64, 0, 36, 0, 2, 0>("QK all SS, 2 chains", d_out);
    run<64, 0, 36, 0, 4, 0>("QK all SS, 4 chains", d_out);
    run<64, 36, 0, 0, 1, 0>("QK all TS (N64 x 36)", d_out);
    run<64, 36, 0, 0, 2, 0>("QK all TS, 2 chains", d_out);
    run<64, 20, 16, 0, 2, 0>("QK as K5, 2 chains", d_out);
    run<64, 0, 0, 8, 1, 0>("PV only (N256 SS x 8)", d_out);
    run<64, 20, 16, 8, 1, 0>("K5 tile (QK as K5 + PV after)", d_out);
    run<64, 20, 16, 8, 1, 1>("K5 tile, PV interleaved", d_out);
    run<64, 20, 16, 8, 2, 1>("K5 tile, 2 chains, PV interleaved", d_out);
    run<64, 20, 16, 8, 2, 0>("K5 tile, 2 chains, PV after", d_out);
    run<128, 0, 18, 0, 1, 0>("QK N128 all SS (x 18)", d_out);
    run<128, 0, 18, 0, 2, 0>("QK N128 all SS, 2 chains", d_out);
    run<128, 9, 9, 8, 1, 0>("QK N128 9 TS + 9 SS + PV", d_out);
    run<256, 0, 9, 0, 1, 0>("QK N256 all SS (x 9)", d_out);
    return 0;
}
