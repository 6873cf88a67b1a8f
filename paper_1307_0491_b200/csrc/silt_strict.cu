// silt_strict.cu — STRICT numerical variant: the reference's operation order;
// this TU is compiled with -fmad=false (no FMA contraction) so every
// arithmetic result matches the CPU reference bit for bit.
#include "silt_kernels.cuh"
#include "silt_launch.h"

SILT_DEFINE_LAUNCHERS(true, silt_strict)

namespace {
__global__ void selftest_math_kernel(const double* x, const double* y, long long n, double* out) {
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    out[4 * k + 0] = silt_dev::rcp(x[k]);
    out[4 * k + 1] = __drcp_rn(x[k]);
    out[4 * k + 2] = silt_dev::hypot_glibc(x[k], y[k]);
    out[4 * k + 3] = silt_dev::fsqrt(x[k]);
}
}  // namespace

void silt_selftest_math_launch(const double* x, const double* y, long long n, double* out) {
    selftest_math_kernel<<<(unsigned)((n + 127) / 128), 128>>>(x, y, n, out);
}
