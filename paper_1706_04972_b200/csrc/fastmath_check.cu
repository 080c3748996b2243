// Accuracy check of fastmath.cuh against the CUDA libm (correctly rounded
// division, <= 1-2 ulp exp/expm1) over the argument ranges the kernels use:
// max ulp distance per function, for tests/test_fastmath_gpu.py.
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "fastmath.cuh"

namespace dp {
namespace {

__device__ unsigned long long ulp_dist(double a, double b) {
    if (a == b) return 0;
    const long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
    if ((ia < 0) != (ib < 0)) return 1ull << 62;
    const long long d = ia - ib;
    return (unsigned long long)(d < 0 ? -d : d);
}

__device__ double ref_act(double x, bool t) {
    const double e = expm1(t ? -2.0 * fabs(x) : -x);
    const double r = (t ? -e : 1.0) / (2.0 + e);
    return t ? copysign(r, x) : r;
}

// out: [sigmoid, tanh, exp, expm1, div] max ulps
__global__ void fastmath_err_kernel(long long n, unsigned long long *out) {
    unsigned long long m[5] = {0, 0, 0, 0, 0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double u = (double)i / (double)n;      // [0, 1)
        const double x = -60.0 + 120.0 * u;          // activations
        m[0] = max(m[0], ulp_dist(fm_gate_act(x, false), ref_act(x, false)));
        m[1] = max(m[1], ulp_dist(fm_gate_act(x, true), ref_act(x, true)));
        const double y = -700.0 + 1400.0 * u;        // softmax exponents
        m[2] = max(m[2], ulp_dist(fm_exp(y), exp(y)));
        const double z = -2.0 + 4.0 * u;
        m[3] = max(m[3], ulp_dist(fm_expm1(z), expm1(z)));
        const double b = 1.0 + 1e6 * u * u, a = 3.0 * u - 1.5;  // divisors >= 1
        m[4] = max(m[4], ulp_dist(fm_div(a, b), a / b));
    }
    for (int k = 0; k < 5; k++) atomicMax(out + k, m[k]);
}

}  // namespace
}  // namespace dp

using namespace dp;

extern "C" int dp_debug_fastmath_error(int64_t n, uint64_t *h_max_ulps) {
    DP_ENTRY();
    DP_REQUIRE(n >= 1 && h_max_ulps, "dp_debug_fastmath_error: bad arguments");
    unsigned long long *d = nullptr;
    DP_CUDA_TRY(cudaMalloc(&d, 5 * sizeof(unsigned long long)));
    cudaMemset(d, 0, 5 * sizeof(unsigned long long));
    fastmath_err_kernel<<<2 * kNumSMs, 256>>>(n, d);
    const cudaError_t e = cudaMemcpy(h_max_ulps, d, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    DP_CUDA_TRY(e);
    return DP_OK;
}
