// C-ABI plumbing shared by all entry points: error text, per-device setup,
// launch accounting, and an fp64 FMA throughput probe (roofline denominator
// for the exact-mode policy kernels; MEASURED_PEAKS.json has no fp64 figure).
#include <atomic>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

namespace dp {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Raise a kernel's dynamic shared-memory cap once per (kernel, device) to the
// device opt-in maximum minus its static shared memory.  (Setting it to the
// size of one launch would LOWER the cap for later, larger launches.)
cudaError_t allow_big_smem(const void *func, size_t bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(func, dev);
    if (done.count(key)) return cudaSuccess;
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, func);
    if (e != cudaSuccess) return e;
    const int cap = optin - (int)fa.sharedSizeBytes;
    if ((size_t)cap < bytes) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

// 8 independent DFMA chains per thread; x stays bounded (a*x+b with |a|<1).
__global__ void fp64_fma_probe_kernel(int iters, double a, double b, double *out) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fma(a, x[i], b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

}  // namespace dp

extern "C" const char *dp_last_error(void) { return dp::g_last_error.c_str(); }

extern "C" int64_t dp_launch_count(void) { return dp::g_launches.load(); }

extern "C" int dp_fp64_fma_probe(int32_t blocks, int32_t threads, int32_t iters, double *scratch, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(blocks > 0 && threads > 0 && iters > 0 && scratch, "dp_fp64_fma_probe: bad arguments");
    dp::fp64_fma_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, 0.999999, 1e-7, scratch);
    DP_LAUNCH_CHECK();
    return DP_OK;
}
