// C-ABI plumbing shared by all entry points: error text, per-device setup.
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

namespace dp {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

cudaError_t allow_big_smem(const void *func, size_t bytes) {
    static std::mutex mu;
    static std::set<std::pair<std::pair<const void *, int>, size_t>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(std::make_pair(func, dev), bytes);
    if (done.count(key)) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

}  // namespace dp

extern "C" const char *dp_last_error(void) { return dp::g_last_error.c_str(); }
