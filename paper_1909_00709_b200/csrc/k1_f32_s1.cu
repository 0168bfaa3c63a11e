// z-march K1 for float fields, shape SHAPE_FIG2_5PT (see sweep.cuh, k1_shape.inc).
#define K1_T float
#define K1_S SHAPE_FIG2_5PT
#define K1_FN launch_k1_f32_s1
#include "k1_shape.inc"
