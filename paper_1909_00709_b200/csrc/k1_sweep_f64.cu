// K1 instantiations for fp64 fields (see sweep.cuh).
#include "launch.h"
#include "sweep.cuh"
#define K1_T double
#define K1_LAUNCH launch_k1_f64
#include "k1_dispatch.inc"
