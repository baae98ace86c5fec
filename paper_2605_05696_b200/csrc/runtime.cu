// ABI plumbing: error strings, version, device queries.
#include "common.cuh"
#include <atomic>

namespace irm {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static std::atomic<int64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return n;
}

}  // namespace irm

extern "C" int irm_abi_version(void) { return 1; }
extern "C" const char *irm_last_error(void) { return irm::g_err; }
extern "C" int irm_device_sm_count(void) { return irm::sm_count(); }
extern "C" int64_t irm_launch_count(void) { return irm::g_launches.load(std::memory_order_relaxed); }
