// z-march K1 for double fields, shape SHAPE_BOX27 (see sweep.cuh, k1_shape.inc).
#define K1_T double
#define K1_S SHAPE_BOX27
#define K1_FN launch_k1_f64_s3
#include "k1_shape.inc"
