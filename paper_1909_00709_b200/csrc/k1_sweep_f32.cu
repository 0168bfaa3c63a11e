// K1 instantiations for fp32 fields (see sweep.cuh).
#include "launch.h"
#include "sweep.cuh"
#define K1_T float
#define K1_LAUNCH launch_k1_f32
#include "k1_dispatch.inc"
