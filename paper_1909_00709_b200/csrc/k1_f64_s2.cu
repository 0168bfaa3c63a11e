// z-march K1 for double fields, shape SHAPE_HOTSPOT7 (see sweep.cuh, k1_shape.inc).
#define K1_T double
#define K1_S SHAPE_HOTSPOT7
#define K1_FN launch_k1_f64_s2
#include "k1_shape.inc"
