// sweep.cuh -- K1: the fused stencil sweep + actual checksums (steps (1) of
// include/abft_stencil.h), hand-written for sm_100a.
//
// Eq. 1 over one z-slab, fused with Eqs. 2-3
// as the paper prescribes for its fig.sweep listing ("adding a
// single addition operation to the kernel").  B200 design:
//  * one CTA owns a TX x TY tile of every layer of a z-chunk and marches up
//    z; the input layers z-1, z, z+1 (incl. a 1-row / 16-byte x halo) are
//    staged in shared memory by TMA (cp.async.bulk.tensor.3d) through an
//    NS-deep mbarrier ring, the source field C (HotSpot power) through its own
//    ring, so every HBM byte is read once per sweep by the tile that needs it;
//  * each thread register-blocks V (one 16-byte vector) x RY cells, evaluates
//    the canonical FMA chain of the stencil (points in the caller's order),
//    stores with 128-bit coalesced stores;
//  * the row sums b_y (over x) are reduced across the warp with a transposed
//    shuffle reduction in fp64, the column sums a_x (over y) across the warps
//    in shared memory, then one fp64 RED per (tile, row) and (tile, column)
//    into the L2-resident checksum generation -- no extra HBM traffic;
//  * fault injection flips the value after the update and before the
//    store, so the checksums see the corrupted value (template INJ).
#pragma once

#include "common.cuh"

namespace abft {

template <typename T> struct Tile {
  static constexpr int V = 16 / (int)sizeof(T);   // elements per 16-byte vector
  static constexpr int TX = 32 * V;               // tile width: one vector per lane
  static constexpr int HV = V;                    // x halo per side (keeps 16 B alignment)
  static constexpr int HX = TX + 2 * HV;          // staged row length
  static constexpr int WARPS = 8;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int RY = sizeof(T) == 4 ? 4 : 2;  // output rows per thread
  static constexpr int TY = WARPS * RY;
  static constexpr int ROWS = TY + 2;
  static constexpr int T_BYTES = ROWS * HX * (int)sizeof(T);
  static constexpr int T_STRIDE = (T_BYTES + 127) / 128 * 128;
  static constexpr int P_BYTES = TX * TY * (int)sizeof(T);
  static constexpr int P_STRIDE = (P_BYTES + 127) / 128 * 128;
  static constexpr int NS = 4;    // field-layer ring: z-1, z, z+1 + 1 prefetch
  static constexpr int NSP = 2;   // source-layer ring
  static constexpr int PART_BYTES = WARPS * TX * 8;
  static constexpr int BAR_BYTES = 128;
  static constexpr int SMEM = NS * T_STRIDE + NSP * P_STRIDE + PART_BYTES + BAR_BYTES + 128;
};

template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; };
template <> struct Vec<double> { using type = double2; };

template <typename T, int V> __device__ __forceinline__ void ld_vec(T (&dst)[V], const T* src) {
  using VT = typename Vec<T>::type;
  VT v = *reinterpret_cast<const VT*>(src);
  const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int k = 0; k < V; ++k) dst[k] = e[k];
}

// transposed warp reduction of RY per-lane row sums: on return lane l holds the
// full sum of row row_of_lane<RY>(l); lanes with final_lane<RY>(l) own it.
template <int RY> __device__ __forceinline__ double row_reduce(const double (&s)[RY], int lane);
template <> __device__ __forceinline__ double row_reduce<4>(const double (&s)[4], int lane) {
  const bool hi = lane & 16;
  double a0 = hi ? s[2] : s[0], a1 = hi ? s[3] : s[1];
  double b0 = hi ? s[0] : s[2], b1 = hi ? s[1] : s[3];
  a0 += __shfl_xor_sync(0xffffffffu, b0, 16);
  a1 += __shfl_xor_sync(0xffffffffu, b1, 16);
  const bool m = lane & 8;
  double c = m ? a1 : a0, d = m ? a0 : a1;
  c += __shfl_xor_sync(0xffffffffu, d, 8);
  c += __shfl_xor_sync(0xffffffffu, c, 4);
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;
}
template <> __device__ __forceinline__ double row_reduce<2>(const double (&s)[2], int lane) {
  const bool hi = lane & 16;
  double c = hi ? s[1] : s[0], d = hi ? s[0] : s[1];
  c += __shfl_xor_sync(0xffffffffu, d, 16);
  c += __shfl_xor_sync(0xffffffffu, c, 8);
  c += __shfl_xor_sync(0xffffffffu, c, 4);
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;
}
template <int RY> __device__ __forceinline__ int row_of_lane(int l);
template <> __device__ __forceinline__ int row_of_lane<4>(int l) { return ((l >> 4) << 1) | ((l >> 3) & 1); }
template <> __device__ __forceinline__ int row_of_lane<2>(int l) { return l >> 4; }
template <int RY> __device__ __forceinline__ bool final_lane(int l);
template <> __device__ __forceinline__ bool final_lane<4>(int l) { return (l & 7) == 0; }
template <> __device__ __forceinline__ bool final_lane<2>(int l) { return (l & 15) == 0; }

// K1.  S: ShapeId (SHAPE_GENERIC = runtime point list).  CHK: accumulate the
// actual checksums.  INJ: apply this launch's scheduled bit-flips.
template <typename T, int S, bool CHK, bool INJ>
__global__ void __launch_bounds__(Tile<T>::THREADS, 1)
    k1_sweep(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_src,
             const __grid_constant__ SweepParams p) {
  using TL = Tile<T>;
  constexpr int V = TL::V, TX = TL::TX, HV = TL::HV, HX = TL::HX, RY = TL::RY, TY = TL::TY;
  constexpr int NS = TL::NS, NSP = TL::NSP, WARPS = TL::WARPS;
  constexpr bool GEN = (S == SHAPE_GENERIC);
  constexpr bool NZ = GEN ? true : shape_needs_z<GEN ? SHAPE_HOTSPOT7 : S>();

  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  T* sT = reinterpret_cast<T*>(base);
  T* sP = reinterpret_cast<T*>(base + NS * TL::T_STRIDE);
  double* sPart = reinterpret_cast<double*>(base + NS * TL::T_STRIDE + NSP * TL::P_STRIDE);
  uint64_t* barT = reinterpret_cast<uint64_t*>(base + NS * TL::T_STRIDE + NSP * TL::P_STRIDE +
                                               TL::PART_BYTES);
  uint64_t* barP = barT + NS;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = p.nx, ny = p.ny, zc = p.zc;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int zs = blockIdx.z * p.zchunk, ze = min(zs + p.zchunk, zc);
  const int q0 = NZ ? zs - 1 : zs;
  const int nT = (NZ ? ze + 1 : ze) - q0;
  const int nZ = ze - zs;
  const bool hasP = p.field_src >= 0;

  if (tid == 0) {
    prefetch_tmap(&tm_u);
    if (hasP) prefetch_tmap(&tm_src);
    for (int i = 0; i < NS; ++i) mbar_init(&barT[i], 1);
    for (int i = 0; i < NSP; ++i) mbar_init(&barP[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue_T = [&](int i) {
    const int st = i % NS;
    mbar_arrive_expect_tx(&barT[st], TL::T_BYTES);
    tma_load_3d(sT + st * (TL::T_STRIDE / (int)sizeof(T)), &tm_u, &barT[st], x0 - HV, y0 - 1,
                zmap(q0 + i, zc, p.has_lo, p.has_hi));
  };
  auto issue_P = [&](int i) {
    const int st = i % NSP;
    mbar_arrive_expect_tx(&barP[st], TL::P_BYTES);
    tma_load_3d(sP + st * (TL::P_STRIDE / (int)sizeof(T)), &tm_src, &barP[st], x0, y0, zs + i);
  };
  if (tid == 0) {
    for (int i = 0; i < NS && i < nT; ++i) issue_T(i);
    if (hasP)
      for (int i = 0; i < NSP && i < nZ; ++i) issue_P(i);
  }

  // per-thread geometry
  const int gx0 = x0 + lane * V;
  const int ry0 = warp * RY;
  const int gyb = y0 + ry0;
  int srow[RY + 2];  // staged row of input row gyb - 1 + t, clamped
#pragma unroll
  for (int t = 0; t < RY + 2; ++t) srow[t] = max(0, min(gyb - 1 + t, ny - 1)) - y0 + 1;

  for (int z = zs; z < ze; ++z) {
    const int it = z - zs;
    const T* pl[3];
    if (NZ) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int i = it + d;
        mbar_wait(&barT[i % NS], (i / NS) & 1);
        pl[d] = sT + (i % NS) * (TL::T_STRIDE / (int)sizeof(T));
      }
    } else {
      mbar_wait(&barT[it % NS], (it / NS) & 1);
      pl[0] = pl[2] = nullptr;
      pl[1] = sT + (it % NS) * (TL::T_STRIDE / (int)sizeof(T));
    }
    const T* ps = sP + (it % NSP) * (TL::P_STRIDE / (int)sizeof(T));
    if (hasP) mbar_wait(&barP[it % NSP], (it / NSP) & 1);

    T out[RY][V];
    if constexpr (!GEN) {
      constexpr int NP = Shape<S>::NP;
      T W[3][RY + 2][V + 2];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int dk = d - 1;
        if (!NZ && dk != 0) continue;
#pragma unroll
        for (int t = 0; t < RY + 2; ++t) {
          bool need = false;
#pragma unroll
          for (int dj = -1; dj <= 1; ++dj)
            if (shape_uses<S>(dk, dj) && t - 1 - dj >= 0 && t - 1 - dj < RY) need = true;
          if (!need) continue;
          const T* row = pl[d] + srow[t] * HX;
          T c[V];
          ld_vec<T, V>(c, row + HV + lane * V);
#pragma unroll
          for (int k = 0; k < V; ++k) W[d][t][k + 1] = c[k];
          if (shape_uses_x_halo<S>(dk)) {
            T left = __shfl_up_sync(0xffffffffu, c[V - 1], 1);
            T right = __shfl_down_sync(0xffffffffu, c[0], 1);
            if (lane == 0) left = row[HV - 1];
            if (lane == 31) right = row[HV + TX];
            W[d][t][0] = left;
            W[d][t][V + 1] = right;
            if (gx0 == 0) W[d][t][0] = W[d][t][1];
            if (gx0 + V >= nx) {
#pragma unroll
              for (int c2 = 1; c2 < V + 2; ++c2)
                if (gx0 - 1 + c2 >= nx) W[d][t][c2] = W[d][t][c2 - 1];
            }
          }
        }
      }
      T wr[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) wr[q] = (T)p.w[q];
#pragma unroll
      for (int r = 0; r < RY; ++r) {
#pragma unroll
        for (int k = 0; k < V; ++k) {
          T acc;
#pragma unroll
          for (int q = 0; q < NP; ++q) {
            const int di = Shape<S>::off(q, 0), dj = Shape<S>::off(q, 1), dk = Shape<S>::off(q, 2);
            const T v = W[dk + 1][r + 1 + dj][k + 1 + di];
            acc = (q == 0) ? mul_rn(wr[q], v) : fma_rn(wr[q], v, acc);
          }
          out[r][k] = acc;
        }
      }
    } else {
      // generic radius-1 point list: runtime offsets, identical FMA chain
#pragma unroll
      for (int r = 0; r < RY; ++r) {
#pragma unroll
        for (int k = 0; k < V; ++k) {
          T acc = T(0);
          for (int q = 0; q < p.npoints; ++q) {
            const int di = p.di[q], dj = p.dj[q], dk = p.dk[q];
            const T* pp = dk < 0 ? pl[0] : (dk > 0 ? pl[2] : pl[1]);
            const int sr = max(0, min(gyb + r + dj, ny - 1)) - y0 + 1;
            const int sc = max(0, min(gx0 + k + di, nx - 1)) - x0 + HV;
            const T v = pp[sr * HX + sc];
            const T w = (T)p.w[q];
            acc = (q == 0) ? mul_rn(w, v) : fma_rn(w, v, acc);
          }
          out[r][k] = acc;
        }
      }
    }
    // constant term C of Eq. 1: sources in order
    for (int q = 0; q < p.nsources; ++q) {
      const T cf = (T)p.coef[q];
      if (q == p.field_src) {
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          T pv[V];
          ld_vec<T, V>(pv, ps + (ry0 + r) * TX + lane * V);
#pragma unroll
          for (int k = 0; k < V; ++k) out[r][k] = fma_rn(cf, pv[k], out[r][k]);
        }
      } else {
        const T sv = (T)p.scalar[q];
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int k = 0; k < V; ++k) out[r][k] = fma_rn(cf, sv, out[r][k]);
      }
    }
    if constexpr (INJ) {  // after the update, before the store
      for (int f = 0; f < p.nfaults; ++f) {
        const LocalFault F = p.faults[f];
        if (F.z != z) continue;
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (F.y == gyb + r && F.x == gx0 + k) out[r][k] = flip_bit(out[r][k], F.bit);
      }
    }
    // store (128-bit where the vector is whole)
    T* obase = reinterpret_cast<T*>(p.out) + (size_t)(z + 1) * p.plane;
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int gy = gyb + r;
      if (gy < ny) {
        T* o = obase + (size_t)gy * p.px + gx0;
        if (gx0 + V <= nx) {
          using VT = typename Vec<T>::type;
          VT v;
          T* e = reinterpret_cast<T*>(&v);
#pragma unroll
          for (int k = 0; k < V; ++k) e[k] = out[r][k];
          *reinterpret_cast<VT*>(o) = v;
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (gx0 + k < nx) o[k] = out[r][k];
        }
      }
    }
    double cs[V];
    if constexpr (CHK) {
      double rs[RY];
#pragma unroll
      for (int k = 0; k < V; ++k) cs[k] = 0.0;
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        rs[r] = 0.0;
        const bool vy = gyb + r < ny;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const double d = (vy && gx0 + k < nx) ? (double)out[r][k] : 0.0;
          rs[r] += d;
          cs[k] += d;
        }
      }
      // b^s_y += sum over this tile's columns (Eq. 3)
      const double tot = row_reduce<RY>(rs, lane);
      const int gy = gyb + row_of_lane<RY>(lane);
      if (final_lane<RY>(lane) && gy < ny) atomicAdd(&p.B[(size_t)(z + 1) * ny + gy], tot);
      __syncthreads();  // the previous layer's column partials have been consumed
#pragma unroll
      for (int k = 0; k < V; ++k) sPart[warp * TX + lane * V + k] = cs[k];
    }
    __syncthreads();  // every read of the lowest staged layer and of the source layer is done
    if (tid == 0) {
      fence_proxy_async();
      if (it + NS < nT) issue_T(it + NS);
      if (hasP && it + NSP < nZ) issue_P(it + NSP);
    }
    if constexpr (CHK) {
      // a^s_x += sum over this tile's rows (Eq. 2)
      if (tid < TX) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) s += sPart[w * TX + tid];
        if (x0 + tid < nx) atomicAdd(&p.A[(size_t)(z + 1) * nx + x0 + tid], s);
      }
    }
  }
}

}  // namespace abft
