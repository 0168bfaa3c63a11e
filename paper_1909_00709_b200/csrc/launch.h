// launch.h -- host-side launchers of the sm_100a kernels (one translation unit
// per dtype for K1 so the template instantiations compile in parallel).
#pragma once

#include <utility>

#include "common.cuh"

namespace abft {

// launch with programmatic stream serialization (PDL): the grid may be
// scheduled while the previous kernel on the stream drains; the kernel calls
// grid_dependency_wait() before it reads that kernel's results
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  return launch_ex(kern, grid, block, smem, s, true, std::forward<Args>(args)...);
}

// K1 `var` flag: launch without programmatic serialization (the pipelined
// schedule lets the checks' CTAs in first)
constexpr int K1_NO_PDL = 8;

struct K1Geometry {
  int tile_x, tile_y, smem, threads;
};
K1Geometry k1_geometry(int dtype);


cudaError_t launch_k1_f32(int shape, int chk, int var, dim3 grid, cudaStream_t s,
                          const CUtensorMap& tu, const SweepParams& p);
cudaError_t launch_k1_f64(int shape, int chk, int var, dim3 grid, cudaStream_t s,
                          const CUtensorMap& tu, const SweepParams& p);
// per (dtype, shape) translation units (k1_<dtype>_s<shape>.cu)
#define ABFT_K1_DECL(name) \
  cudaError_t name(int chk, int var, dim3 grid, cudaStream_t s, const CUtensorMap& tu, const SweepParams& p);
ABFT_K1_DECL(launch_k1_f32_s0) ABFT_K1_DECL(launch_k1_f32_s1) ABFT_K1_DECL(launch_k1_f32_s2)
ABFT_K1_DECL(launch_k1_f32_s4)
ABFT_K1_DECL(launch_k1_f64_s0) ABFT_K1_DECL(launch_k1_f64_s1) ABFT_K1_DECL(launch_k1_f64_s2)
ABFT_K1_DECL(launch_k1_f64_s4)
// the 27-point box compiles slowest: one translation unit per checksum variant
ABFT_K1_DECL(launch_k1_f32_s3_ck0) ABFT_K1_DECL(launch_k1_f32_s3_ck1) ABFT_K1_DECL(launch_k1_f32_s3_ck2)
ABFT_K1_DECL(launch_k1_f64_s3_ck0) ABFT_K1_DECL(launch_k1_f64_s3_ck1) ABFT_K1_DECL(launch_k1_f64_s3_ck2)
#undef ABFT_K1_DECL
// K2 over the layers [p.zr0, p.zr1)
cudaError_t launch_k2(int dtype, int shape, cudaStream_t s, const CheckParams& p);
// fill n elements of a field buffer with v (constant ghost layers)
cudaError_t launch_fill(int dtype, void* ptr, int64_t n, double v, cudaStream_t s);
// load the check kernels of (dtype, shape, bc) now (CUDA lazy module loading)
cudaError_t prime_checks(int dtype, int shape, int bc);
// K3 (lazy checksum policy)
cudaError_t launch_k3(int dtype, int shape, cudaStream_t s, const CheckParams& p);
// K0: A[z + off][x] / B[z + off][y] sums of the field buffer `u`
cudaError_t launch_k0_field(int dtype, const void* u, int64_t px, int64_t plane, int nx, int ny,
                            int zc, double* A, double* B, int off, cudaStream_t s);
// K0: c_x / c_y of the constant term
cudaError_t launch_k0_const(int dtype, const void* field, int64_t fpx, int nx, int ny, int zc,
                            int nsources, int field_src, const double* coef, const double* scalar,
                            double* cA, double* cB, cudaStream_t s);

}  // namespace abft
