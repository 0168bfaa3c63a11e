// y-march K1 instantiations for double fields (see sweep_y.cuh).
#include "launch.h"
#include "sweep_y.cuh"
#define K1_T double
#define K1Y_LAUNCH launch_k1y_f64
#define K1Y_OCC k1y_occ_f64
#include "k1y_dispatch.inc"
