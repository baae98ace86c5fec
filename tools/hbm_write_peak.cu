// HBM write-bandwidth probe (B200): what a write-dominated kernel can reach.
//   bulk   : persistent CTAs (1/SM), each streams 36 KB shared-memory tiles to
//            consecutive global ranges with cp.async.bulk stores, D in flight
//   vec    : grid-stride 16-byte st.global from registers
//   copy   : 1:1 read + write with 16-byte loads/stores (the MEASURED_PEAKS kind)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_write_peak tools/hbm_write_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_05696_b200/csrc/tma.cuh"

using namespace irm;
constexpr int TILE = 36864, STAGES = 6;

template <int D>
__global__ void __launch_bounds__(128) bulk_write(char *out, int64_t tiles, int64_t scatter) {
    extern __shared__ __align__(128) uint8_t smem[];
    for (int i = threadIdx.x; i < STAGES * TILE / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(i, blockIdx.x, 7, 9);
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x) return;
    int64_t k = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
        // scatter != 0: tile t goes to position (t * scatter) mod tiles (a scattered write pattern)
        const int64_t pos = scatter ? (t * scatter) % tiles : t;
        bulk_s2g(out + pos * TILE, smem + (k % STAGES) * TILE, TILE);
        bulk_commit();
        bulk_wait_read<D>();
    }
    bulk_wait<0>();
}

// 8 bulk stores per bulk load (the K4 fan-out's write:read mix on the config-2 wave)
__global__ void __launch_bounds__(128) bulk_mix(char *out, const char *in, int64_t tiles, int ratio) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x) return;
    int64_t k = 0;
    uint32_t phase = 0;
    bool pending = false;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
        if (k % ratio == 0) {
            if (pending) {
                mbar_wait(&bar, phase);
                phase ^= 1;
            }
            mbar_arrive_expect_tx(&bar, TILE);
            bulk_g2s(smem + (STAGES - 1) * TILE, in + ((t / ratio) % tiles) * TILE, TILE, &bar);
            pending = true;
        }
        bulk_s2g(out + t * TILE, smem + (k % (STAGES - 1)) * TILE, TILE);
        bulk_commit();
        bulk_wait_read<3>();
    }
    if (pending) mbar_wait(&bar, phase);
    bulk_wait<0>();
}

// every store preceded by a bulk load of its tile; 8 consecutive stores of a CTA share one source tile
// (the first load of a group misses to HBM, the rest hit L2): the K4 fan-out reload pattern, no math
__global__ void __launch_bounds__(128) bulk_reload(char *out, const char *in, int64_t tiles, int group) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[STAGES];
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x) return;
    const int64_t mine = (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    auto src_of = [&](int64_t k) { return in + (((blockIdx.x + k * gridDim.x) / group) % tiles) * (int64_t)TILE; };
    constexpr int AHEAD = 3;  // loads in flight; STAGES - AHEAD stores in flight
    for (int64_t k = 0; k < AHEAD && k < mine; ++k) {
        mbar_arrive_expect_tx(&bar[k % STAGES], TILE);
        bulk_g2s(smem + (k % STAGES) * TILE, src_of(k), TILE, &bar[k % STAGES]);
    }
    for (int64_t k = 0; k < mine; ++k) {
        const int s = (int)(k % STAGES);
        mbar_wait(&bar[s], (uint32_t)((k / STAGES) & 1));
        bulk_s2g(out + (blockIdx.x + k * gridDim.x) * (int64_t)TILE, smem + s * TILE, TILE);
        bulk_commit();
        const int64_t nk = k + AHEAD;
        if (nk < mine) {
            bulk_wait_read<STAGES - AHEAD - 1>();  // store nk - STAGES has left stage nk % STAGES
            mbar_arrive_expect_tx(&bar[nk % STAGES], TILE);
            bulk_g2s(smem + (nk % STAGES) * TILE, src_of(nk), TILE, &bar[nk % STAGES]);
        }
    }
    bulk_wait<0>();
}

__global__ void vec_write(uint4 *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

__global__ void vec_copy(const uint4 *in, uint4 *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

template <typename F>
static float time_ms(F f, int reps = 10) {
    f();
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    const int64_t bytes = (int64_t)8 << 30;
    const int64_t tiles = bytes / TILE;
    char *buf, *src;
    cudaMalloc(&buf, tiles * TILE);
    cudaMalloc(&src, tiles * TILE);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = STAGES * TILE;
    cudaFuncSetAttribute(bulk_write<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bulk_write<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bulk_write<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const double gb = tiles * (double)TILE / 1e9;
    float ms = time_ms([&] { bulk_write<1><<<sms, 128, smem>>>(buf, tiles, 0); });
    printf("bulk  D=2 in flight : %.0f GB/s write\n", gb / ms * 1e3);
    ms = time_ms([&] { bulk_write<3><<<sms, 128, smem>>>(buf, tiles, 0); });
    printf("bulk  D=4 in flight : %.0f GB/s write\n", gb / ms * 1e3);
    ms = time_ms([&] { bulk_write<5><<<sms, 128, smem>>>(buf, tiles, 0); });
    printf("bulk  D=6 in flight : %.0f GB/s write\n", gb / ms * 1e3);
    for (int64_t sc : {7919LL, 1000003LL, 27LL, 8LL * 27 + 1}) {
        ms = time_ms([&] { bulk_write<3><<<sms, 128, smem>>>(buf, tiles, sc); });
        printf("bulk  D=4 scatter %lld : %.0f GB/s write\n", (long long)sc, gb / ms * 1e3);
    }
    cudaFuncSetAttribute(bulk_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int ratio : {8, 4, 2, 1}) {
        ms = time_ms([&] { bulk_mix<<<sms, 128, smem>>>(buf, src, tiles, ratio); });
        printf("bulk  %d stores : 1 load : %.0f GB/s write + %.0f GB/s read\n", ratio, gb / ms * 1e3,
               gb / ratio / ms * 1e3);
    }
    cudaFuncSetAttribute(bulk_reload, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int group : {8, 1}) {
        ms = time_ms([&] { bulk_reload<<<sms, 128, smem>>>(buf, src, tiles, group); });
        printf("bulk  load+store per tile, %d stores per source tile : %.0f GB/s write (+%.0f GB/s HBM read)\n",
               group, gb / ms * 1e3, gb / group / ms * 1e3);
    }
    const int64_t n16 = tiles * TILE / 16;
    ms = time_ms([&] { vec_write<<<sms * 8, 512>>>((uint4 *)buf, n16); });
    printf("vec   st.global.v4  : %.0f GB/s write\n", gb / ms * 1e3);
    ms = time_ms([&] { vec_copy<<<sms * 8, 512>>>((const uint4 *)src, (uint4 *)buf, n16); });
    printf("copy  ld+st v4      : %.0f GB/s read+write\n", 2 * gb / ms * 1e3);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
