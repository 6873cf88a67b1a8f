// silt_fast.cu — FAST numerical variant of the fused step (FMA contraction on).
#include "silt_kernels.cuh"
#include "silt_launch.h"

SILT_DEFINE_LAUNCHERS(false, silt_fast)


#ifdef SILT_STATS
// diagnostics build only: read and reset the solver counters
extern "C" int silt_debug_stats(unsigned long long* out, int n) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, silt_dev::g_stats, sizeof(unsigned long long) * (n < 8 ? n : 8));
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(silt_dev::g_stats, z, sizeof z);
    return 0;
}
#endif

#ifdef SILT_TRACE
extern "C" int silt_debug_trace(unsigned long long* dev_buf) {
    return (int)cudaMemcpyToSymbol(silt_dev::g_trace, &dev_buf, sizeof dev_buf);
}
#endif
