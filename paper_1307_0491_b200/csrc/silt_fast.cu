// silt_fast.cu — FAST numerical variant of the fused step (FMA contraction on).
#include "silt_kernels.cuh"
#include "silt_launch.h"

SILT_DEFINE_LAUNCHERS(false, silt_fast)

