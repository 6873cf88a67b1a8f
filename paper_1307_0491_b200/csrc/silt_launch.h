// silt_launch.h — launchers exported by the two numerical-variant TUs.
#pragma once
#include <cuda_runtime.h>

#include "silt_layout.h"

#define SILT_DECLARE_LAUNCHERS(NAME)                                                         \
    void NAME##_step(const StepArgs& A, int li, dim3 grid, cudaStream_t st);                 \
    int NAME##_step1d_coop(const StepArgs& A, int li0, int n, dim3 grid, cudaStream_t st);   \
    int NAME##_step1d_coop_blocks(int shields);                                              \
    int NAME##_step2d_ctas_per_sm(int shields);                                              \
    int NAME##_debug_checks(unsigned long long* out);                                        \
    int NAME##_step1d_cluster(const StepArgs& A, int li0, int n, int ctas, cudaStream_t st); \
    void NAME##_reduce(const StepArgs& A, int li, int blocks, cudaStream_t st);              \
    void NAME##_faces(const silt_dev::Params& P, const double* L, const double* R,           \
                      long long n, int axis, double* out, unsigned* err, cudaStream_t st);   \
    void NAME##_law(const silt_dev::Params& P, const double* X, long long n, double* out,    \
                    cudaStream_t st);

SILT_DECLARE_LAUNCHERS(silt_fast)
SILT_DECLARE_LAUNCHERS(silt_strict)

void silt_selftest_math_launch(const double* x, const double* y, long long n, double* out);
