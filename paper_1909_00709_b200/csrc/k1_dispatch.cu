// Shape dispatch of the z-march K1 (one translation unit per dtype x shape).
#include "launch.h"

namespace abft {

cudaError_t launch_k1_f32(int shape, int chk, int var, dim3 grid, cudaStream_t s, const CUtensorMap& tu,
                          const SweepParams& p) {
  switch (shape) {
    case SHAPE_FIG2_5PT: return launch_k1_f32_s1(chk, var, grid, s, tu, p);
    case SHAPE_HOTSPOT7: return launch_k1_f32_s2(chk, var, grid, s, tu, p);
    case SHAPE_BOX27:
      return chk == K1_CK_AB ? launch_k1_f32_s3_ck1(chk, var, grid, s, tu, p)
           : chk == K1_CK_B  ? launch_k1_f32_s3_ck2(chk, var, grid, s, tu, p)
                             : launch_k1_f32_s3_ck0(chk, var, grid, s, tu, p);
    case SHAPE_HOTSPOT7_FS: return launch_k1_f32_s4(chk, var, grid, s, tu, p);
    default: return launch_k1_f32_s0(chk, var, grid, s, tu, p);
  }
}

cudaError_t launch_k1_f64(int shape, int chk, int var, dim3 grid, cudaStream_t s, const CUtensorMap& tu,
                          const SweepParams& p) {
  switch (shape) {
    case SHAPE_FIG2_5PT: return launch_k1_f64_s1(chk, var, grid, s, tu, p);
    case SHAPE_HOTSPOT7: return launch_k1_f64_s2(chk, var, grid, s, tu, p);
    case SHAPE_BOX27:
      return chk == K1_CK_AB ? launch_k1_f64_s3_ck1(chk, var, grid, s, tu, p)
           : chk == K1_CK_B  ? launch_k1_f64_s3_ck2(chk, var, grid, s, tu, p)
                             : launch_k1_f64_s3_ck0(chk, var, grid, s, tu, p);
    case SHAPE_HOTSPOT7_FS: return launch_k1_f64_s4(chk, var, grid, s, tu, p);
    default: return launch_k1_f64_s0(chk, var, grid, s, tu, p);
  }
}

}  // namespace abft
