// y-march K1 instantiations for float fields (see sweep_y.cuh).
#include "launch.h"
#include "sweep_y.cuh"
#define K1_T float
#define K1Y_LAUNCH launch_k1y_f32
#define K1Y_OCC k1y_occ_f32
#include "k1y_dispatch.inc"
