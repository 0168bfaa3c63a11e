// z-march K1 for double fields, shape SHAPE_FIG2_5PT (see sweep.cuh, k1_shape.inc).
#define K1_T double
#define K1_S SHAPE_FIG2_5PT
#define K1_FN launch_k1_f64_s1
#include "k1_shape.inc"
