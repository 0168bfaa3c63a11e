// z-march K1 for double fields, shape SHAPE_BOX27, checksum variant K1_CK_NONE only
// (the 27-point box is the slowest to compile: one unit per variant, built in parallel).
#define K1_T double
#define K1_S SHAPE_BOX27
#define K1_CHK K1_CK_NONE
#define K1_FN launch_k1_f64_s3_ck0
#include "k1_shape.inc"
