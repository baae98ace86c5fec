// Probe: shared-memory address layout in a 4-CTA cluster and the mbarrier a
// .cta_group::2 .multicast::cluster TMA completes on (which CTA of each destination pair).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mc_probe tools/mc_probe.cu -lcuda && ./mc_probe
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__device__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ bool try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}

__global__ void __cluster_dims__(4, 1, 1) probe(const __grid_constant__ CUtensorMap tm, int mode, int *res) {
    __shared__ __align__(1024) uint8_t buf[4096];
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        for (int i = 0; i < 4096; ++i) buf[i] = 0;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0 && mode == 0)
        printf("rank %u: smem_u32(bar)=%08x mapa0=%08x mapa1=%08x mapa2=%08x mapa3=%08x\n", rank, smem_u32(&bar),
               mapa(smem_u32(&bar), 0), mapa(smem_u32(&bar), 1), mapa(smem_u32(&bar), 2), mapa(smem_u32(&bar), 3));
    if (threadIdx.x == 0) {
        if ((rank & 1) == 0)  // pair leaders expect both pair CTAs' bytes
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(8192));
        if (rank < 2) {  // CTA r multicasts rows [32 r, +32) to {r, r + 2}
            const uint16_t mask = (uint16_t)((1u << rank) | (1u << (rank + 2)));
            uint32_t b = mode == 1 ? (smem_u32(&bar) & 0xFEFFFFFFu) : mapa(smem_u32(&bar), 0);
            asm volatile(
                "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(buf)),
                "l"(&tm), "r"(0), "r"(32 * (int)rank), "r"(b), "h"(mask)
                : "memory");
        }
        int ok = 1;
        if ((rank & 1) == 0) {
            long spins = 0;
            while (!try_wait(&bar, 0) && ++spins < 20000000) {
            }
            ok = spins < 20000000;
        }
        res[mode * 8 + rank] = ok;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) res[mode * 8 + 4 + rank] = buf[0] + 256 * buf[2 * 64];  // first bytes of row 0 / 1
}

int main() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    uint8_t *g;
    cudaMalloc(&g, 64 * 64 * 2);
    uint8_t h[64 * 128];
    for (int r = 0; r < 64; ++r)
        for (int c = 0; c < 128; ++c) h[r * 128 + c] = (uint8_t)(r + 1);
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, 64}, strides[1] = {128};
    cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
    encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int *res;
    cudaMallocManaged(&res, 64 * sizeof(int));
    for (int mode = 0; mode < 2; ++mode) {
        probe<<<4, 32>>>(tm, mode, res);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d (%s): %s | leader0 ok %d leader2 ok %d | data rank0..3 = %d %d %d %d\n", mode,
               mode == 0 ? "barrier = mapa(bar, 0)" : "barrier = local & ~peer bit", cudaGetErrorString(e),
               res[mode * 8 + 0], res[mode * 8 + 2], res[mode * 8 + 4], res[mode * 8 + 5], res[mode * 8 + 6],
               res[mode * 8 + 7]);
    }
    return 0;
}
