// z-march K1 for float fields, shape SHAPE_GENERIC (see sweep.cuh, k1_shape.inc).
#define K1_T float
#define K1_S SHAPE_GENERIC
#define K1_FN launch_k1_f32_s0
#include "k1_shape.inc"
