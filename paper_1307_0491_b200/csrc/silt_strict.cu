// silt_strict.cu — STRICT numerical variant: the reference's operation order;
// this TU is compiled with -fmad=false (no FMA contraction) so every
// arithmetic result matches the CPU reference bit for bit.
#include "silt_kernels.cuh"
#include "silt_launch.h"

SILT_DEFINE_LAUNCHERS(true, silt_strict)
