// sweep.cuh -- K1: the fused stencil sweep + actual checksums (steps (1) of
// include/abft_stencil.h), hand-written for sm_100a.
//
// Eq. 1 over one z-slab, fused with Eqs. 2-3
// as the paper prescribes for its fig.sweep listing ("adding a
// single addition operation to the kernel").  B200 design:
//  * one CTA owns a TX x TY tile of every layer of a z-chunk and marches up
//    z; the input layers z-1, z, z+1 (incl. a 1-row / 16-byte x halo) are
//    staged in shared memory by TMA (cp.async.bulk.tensor.3d) through an
//    NS-deep mbarrier ring (2 layers in flight); the source field C (HotSpot
//    power) is read once, straight into registers one layer ahead (128-bit
//    read-only loads), so every HBM byte is read once per sweep;
//  * each thread register-blocks V (one 16-byte vector) x RY cells, evaluates
//    the canonical FMA chain of the stencil (points in the caller's order),
//    stores with 128-bit coalesced stores;
//  * the row sums b_y (over x) are reduced across the warp with a transposed
//    shuffle reduction in fp64, the column sums a_x (over y) across the warps
//    in shared memory (double-buffered: one CTA barrier per layer, shared with
//    the ring), then one fp64 RED per (tile, row) and (tile, column) into the
//    L2-resident checksum generation -- no extra HBM traffic;
//  * fault injection flips the value after the update and before the
//    store, so the checksums see the corrupted value.  Launches with a
//    scheduled flip, and constant / periodic ghosts, run the GENERAL
//    instantiation; the hot path (no flip, clamp or zero ghosts) keeps its
//    registers for the stencil.
#pragma once

#include "common.cuh"

namespace abft {

template <typename T> struct Tile {
  static constexpr int V = 16 / (int)sizeof(T);   // elements per 16-byte vector
  static constexpr int TX = 32 * V;               // tile width: one vector per lane
  static constexpr int HV = V;                    // x halo per side (keeps 16 B alignment)
  static constexpr int HX = TX + 2 * HV;          // staged row length
#ifndef ABFT_WARPS
#define ABFT_WARPS 8
#endif
  static constexpr int WARPS = ABFT_WARPS;
  static constexpr int THREADS = 32 * WARPS;
#ifndef ABFT_RY_F32
#define ABFT_RY_F32 4
#endif
#ifndef ABFT_RY_F64
#define ABFT_RY_F64 4
#endif
#ifndef ABFT_NS
#define ABFT_NS 4
#endif

  static constexpr int RY = sizeof(T) == 4 ? ABFT_RY_F32 : ABFT_RY_F64;  // output rows per thread
  static constexpr int TY = WARPS * RY;
  static constexpr int ROWS = TY + 2;
  static constexpr int T_BYTES = ROWS * HX * (int)sizeof(T);
  static constexpr int T_STRIDE = (T_BYTES + 127) / 128 * 128;
  static constexpr int NS = ABFT_NS;  // field-layer ring: z-1, z, z+1 + 1 prefetch (5 measured slower)
  static constexpr int PART_BYTES = 2 * WARPS * TX * 8;   // column partials, double-buffered
  static constexpr int BAR_BYTES = 128;
  static constexpr int SMEM = NS * T_STRIDE + PART_BYTES + BAR_BYTES + 128;
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

// fp64 row (over this thread's V columns) and column (over its RY rows)
// partial sums of the stored values; out-of-domain cells count 0 (!FULL).
template <typename T, bool FULL>
__device__ __forceinline__ void partial_sums(const T (&out)[Tile<T>::RY][Tile<T>::V],
                                             double (&rs)[Tile<T>::RY], double (&cs)[Tile<T>::V],
                                             int gyb, int gx0, int nx, int ny) {
  constexpr int RY = Tile<T>::RY, V = Tile<T>::V;
#pragma unroll
  for (int r = 0; r < RY; ++r) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double d = (double)out[r][k];
      if (!FULL) d = (gyb + r < ny && gx0 + k < nx) ? d : 0.0;
      rs[r] = k == 0 ? d : rs[r] + d;
      cs[k] = r == 0 ? d : cs[k] + d;
    }
  }
}

// rows-only variant (checksum policy LAZY: b every sweep)
template <typename T, bool FULL, int RY>
__device__ __forceinline__ void row_sums(const T (&out)[RY][16 / sizeof(T)], double (&rs)[RY],
                                         int gyb, int gx0, int nx, int ny) {
  constexpr int V = 16 / (int)sizeof(T);
#pragma unroll
  for (int r = 0; r < RY; ++r) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      double d = (double)out[r][k];
      if (!FULL) d = (gyb + r < ny && gx0 + k < nx) ? d : 0.0;
      rs[r] = k == 0 ? d : rs[r] + d;
    }
  }
}

// One layer of one thread: RY x V outputs of Eq. 1 from the staged planes
// pl[0..2] (offset -1, 0, +1 along the march axis), the canonical FMA chain in
// the shape's point order; srow[t] = staged row of input row (first - 1 + t),
// already clamped or mapped to a halo.  EDGE: the tile touches
// x = 0 or x = nx - 1, so out-of-domain x reads take the clamped value.
// SH is the shape seen in the staged coordinates: off(q, 2) selects the plane,
// off(q, 1) the row.
// What an edge tile needs to build the ghosts of Eq. 1 (P:289-292 clamp,
// P:413-415 periodic / zero / constant): BC, ghost value, the input planes in
// global memory (periodic wrap reads), the row pitch and the thread's rows.
template <typename T> struct EdgeCtx {
  int bc;
  T g;
  const T* up[3];
  int64_t px;
  int gyb, ny;
};

// Byte offsets of a thread's staged rows (loop invariant): sro[t] = its
// 16-byte vector of staged row t, seo[t] = the halo element lane 0 / 31 needs
// (every lane loads one of the two: 2 addresses, one wavefront, no
// divergence).  Added to the layer's slot base, a uniform register, so each
// shared load is one LDS [R + UR].
template <int RY> struct RowOffs {
  int sro[RY + 2], seo[RY + 2];
};
template <typename T, int RY>
__device__ __forceinline__ RowOffs<RY> row_offsets(const int (&srow)[RY + 2], int lane) {
  constexpr int V = 16 / (int)sizeof(T), TX = 32 * V, HV = V;
  const int eoff = lane == 0 ? HV - 1 : HV + TX;
  RowOffs<RY> o;
#pragma unroll
  for (int t = 0; t < RY + 2; ++t) {
    o.sro[t] = (srow[t] + HV + lane * V) * (int)sizeof(T);
    o.seo[t] = (srow[t] + eoff) * (int)sizeof(T);
  }
  return o;
}

// Plane groups of a point list: maximal runs of consecutive points on the
// same staged plane (HotSpot: {c,w,e,n,s}, {t}, {b}; 27-point box: 3 x 9).
template <class SH> __host__ __device__ constexpr int group_end(int q) {
  int e = q;
  while (e < SH::NP && SH::off(e, 2) == SH::off(q, 2)) ++e;
  return e;
}
template <class SH> __host__ __device__ constexpr bool group_uses_row(int q, int dj) {
  for (int e = q; e < group_end<SH>(q); ++e)
    if (SH::off(e, 1) == dj) return true;
  return false;
}
template <class SH> __host__ __device__ constexpr bool group_uses_halo(int q) {
  for (int e = q; e < group_end<SH>(q); ++e)
    if (SH::off(e, 0) != 0) return true;
  return false;
}

// One layer of one thread: RY x V outputs of Eq. 1, the canonical FMA chain
// in the point order.  The points are applied plane group by plane group: a
// group's staged rows are loaded (with the x halo and the ghosts of an edge
// tile) into one register plane, then every output's chain advances through
// the group's points -- only one plane is live, so the 27-point box fits.
// All three planes loaded first, then the chains (few points per plane:
// every load in flight at once; the HotSpot 7-point path).
template <typename T, class SH, int RY, bool NZ, bool EDGE, bool BCG = true>
__device__ __forceinline__ void stencil_layer_all(T (&out)[RY][16 / sizeof(T)], const T* const (&pl)[3],
                                              const RowOffs<RY>& ro, const T (&wr)[SH::NP],
                                              int lane, int gx0, int nx, const EdgeCtx<T>& ec) {
  constexpr int V = 16 / (int)sizeof(T), NP = SH::NP;
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
        if (sh_uses<SH>(dk, dj) && t - 1 - dj >= 0 && t - 1 - dj < RY) need = true;
      if (!need) continue;
      const unsigned char* slot = reinterpret_cast<const unsigned char*>(pl[d]);
      T c[V];
      ld_vec<T, V>(c, reinterpret_cast<const T*>(slot + ro.sro[t]));
#pragma unroll
      for (int k = 0; k < V; ++k) W[d][t][k + 1] = c[k];
      if (sh_uses_x_halo<SH>(dk)) {
        const T e = *reinterpret_cast<const T*>(slot + ro.seo[t]);
        T left = __shfl_up_sync(0xffffffffu, c[V - 1], 1);
        T right = __shfl_down_sync(0xffffffffu, c[0], 1);
        left = lane == 0 ? e : left;
        right = lane == 31 ? e : right;
        W[d][t][0] = left;
        W[d][t][V + 1] = right;
        if constexpr (EDGE) {
          if (ec.bc == ABFT_BC_CLAMP) {
            if (gx0 == 0) W[d][t][0] = W[d][t][1];
#pragma unroll
            for (int c2 = 1; c2 < V + 2; ++c2)
              if (gx0 - 1 + c2 >= nx) W[d][t][c2] = W[d][t][c2 - 1];
          }
        }
      }
      if constexpr (EDGE && BCG) {
        // constant / periodic ghosts (zero ghosts are the TMA's zero fill of
        // out-of-range boxes): every out-of-domain entry of this row
        if (ec.bc == ABFT_BC_CONSTANT || ec.bc == ABFT_BC_PERIODIC) {
          const int gy = ec.gyb - 1 + t;
          const bool yo = gy < 0 || gy >= ec.ny;
#pragma unroll
          for (int c2 = 0; c2 < V + 2; ++c2) {
            const int gx = gx0 - 1 + c2;
            if (yo || gx < 0 || gx >= nx) {
              if (ec.bc == ABFT_BC_CONSTANT) {
                W[d][t][c2] = ec.g;
              } else {
                const int wy = ((gy % ec.ny) + ec.ny) % ec.ny, wx = ((gx % nx) + nx) % nx;
                W[d][t][c2] = ec.up[d][(size_t)wy * ec.px + wx];
              }
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RY; ++r) {
#pragma unroll
    for (int k = 0; k < V; ++k) {
      T acc;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const int di = SH::off(q, 0), dj = SH::off(q, 1), dk = SH::off(q, 2);
        const T v = W[dk + 1][r + 1 + dj][k + 1 + di];
        acc = (q == 0) ? mul_rn(wr[q], v) : fma_rn(wr[q], v, acc);
      }
      out[r][k] = acc;
    }
  }
}

// Plane by plane (many points per plane: the 27-point box).
template <typename T, class SH, int RY, bool NZ, bool EDGE, bool BCG = true>
__device__ __forceinline__ void stencil_layer_grouped(T (&out)[RY][16 / sizeof(T)], const T* const (&pl)[3],
                                                      const RowOffs<RY>& ro, const T (&wr)[SH::NP],
                                                      int lane, int gx0, int nx, const EdgeCtx<T>& ec) {
  constexpr int V = 16 / (int)sizeof(T), NP = SH::NP;
  T W[RY + 2][V + 2];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int dk = SH::off(q, 2), d = dk + 1;
    if (q == 0 || SH::off(q - 1, 2) != dk) {
      // ---- load the rows of plane dk this group reads
#pragma unroll
      for (int t = 0; t < RY + 2; ++t) {
        bool need = false;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj)
          if (group_uses_row<SH>(q, dj) && t - 1 - dj >= 0 && t - 1 - dj < RY) need = true;
        if (!need) continue;
        const unsigned char* slot = reinterpret_cast<const unsigned char*>(pl[NZ ? d : 1]);
        T c[V];
        ld_vec<T, V>(c, reinterpret_cast<const T*>(slot + ro.sro[t]));
#pragma unroll
        for (int k = 0; k < V; ++k) W[t][k + 1] = c[k];
        if (group_uses_halo<SH>(q)) {
          const T e = *reinterpret_cast<const T*>(slot + ro.seo[t]);
          T left = __shfl_up_sync(0xffffffffu, c[V - 1], 1);
          T right = __shfl_down_sync(0xffffffffu, c[0], 1);
          left = lane == 0 ? e : left;
          right = lane == 31 ? e : right;
          W[t][0] = left;
          W[t][V + 1] = right;
          if constexpr (EDGE) {
            if (ec.bc == ABFT_BC_CLAMP) {
              if (gx0 == 0) W[t][0] = W[t][1];
#pragma unroll
              for (int c2 = 1; c2 < V + 2; ++c2)
                if (gx0 - 1 + c2 >= nx) W[t][c2] = W[t][c2 - 1];
            }
          }
        }
        if constexpr (EDGE && BCG) {
          // constant / periodic ghosts (zero ghosts are the TMA's zero fill of
          // out-of-range boxes): every out-of-domain entry of this row
          if (ec.bc == ABFT_BC_CONSTANT || ec.bc == ABFT_BC_PERIODIC) {
            const int gy = ec.gyb - 1 + t;
            const bool yo = gy < 0 || gy >= ec.ny;
#pragma unroll
            for (int c2 = 0; c2 < V + 2; ++c2) {
              const int gx = gx0 - 1 + c2;
              if (yo || gx < 0 || gx >= nx) {
                if (ec.bc == ABFT_BC_CONSTANT) {
                  W[t][c2] = ec.g;
                } else {
                  const int wy = ((gy % ec.ny) + ec.ny) % ec.ny, wx = ((gx % nx) + nx) % nx;
                  W[t][c2] = ec.up[NZ ? d : 1][(size_t)wy * ec.px + wx];
                }
              }
            }
          }
        }
      }
    }
    // ---- every output's chain advances by point q
    const int di = SH::off(q, 0), dj = SH::off(q, 1);
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const T v = W[r + 1 + dj][k + 1 + di];
        out[r][k] = (q == 0) ? mul_rn(wr[q], v) : fma_rn(wr[q], v, out[r][k]);
      }
  }
}

// Plane-streaming shapes: points sorted by (dk, dj, di) ascending, strictly
// (the 27-point box of cfg5 and any radius-1 subset listed that way).
template <class SH> __host__ __device__ constexpr bool sh_streamable() {
  for (int q = 1; q < SH::NP; ++q) {
    const int a = (SH::off(q - 1, 2) * 3 + SH::off(q - 1, 1)) * 3 + SH::off(q - 1, 0);
    const int b = (SH::off(q, 2) * 3 + SH::off(q, 1)) * 3 + SH::off(q, 0);
    if (a >= b) return false;
  }
  return true;
}

// One staged row t of a plane in registers: W[1..V] = the thread's vector,
// W[0] / W[V+1] = its x neighbours (shuffles + one broadcast shared load),
// with the boundary ghosts of an edge tile (clamp in x; constant / periodic
// ghosts for every out-of-domain entry -- zero ghosts are the TMA's fill).
// gplane: the plane in global memory (periodic wrap reads).
template <typename T, bool EDGE, bool BCG>
__device__ __forceinline__ void load_row(T (&W)[16 / sizeof(T) + 2], const unsigned char* slot, int sro,
                                         int seo, int t, int lane, int gx0, int nx, const EdgeCtx<T>& ec,
                                         const T* gplane) {
  constexpr int V = 16 / (int)sizeof(T);
  T c[V];
  ld_vec<T, V>(c, reinterpret_cast<const T*>(slot + sro));
#pragma unroll
  for (int k = 0; k < V; ++k) W[k + 1] = c[k];
  if constexpr (sizeof(T) == 8) {
    // fp64: the x neighbours straight from the staged row (lane 0 / 31 read
    // the tile's halo) -- two shared loads instead of two 64-bit shuffles,
    // a broadcast load and two 64-bit selects (cfg5 K1: instructions -13%,
    // 1.488 -> 1.404 ms, shared wavefronts +18%; round 1 measured the
    // opposite when every staged row was loaded three times)
    W[0] = *reinterpret_cast<const T*>(slot + sro - (int)sizeof(T));
    W[V + 1] = *reinterpret_cast<const T*>(slot + sro + V * (int)sizeof(T));
    (void)seo;
    (void)lane;
  } else {
  const T e = *reinterpret_cast<const T*>(slot + seo);
  T left = __shfl_up_sync(0xffffffffu, c[V - 1], 1);
  T right = __shfl_down_sync(0xffffffffu, c[0], 1);
  W[0] = lane == 0 ? e : left;
  W[V + 1] = lane == 31 ? e : right;
  }
  if constexpr (EDGE) {
    if (ec.bc == ABFT_BC_CLAMP) {
      if (gx0 == 0) W[0] = W[1];
#pragma unroll
      for (int c2 = 1; c2 < V + 2; ++c2)
        if (gx0 - 1 + c2 >= nx) W[c2] = W[c2 - 1];
    }
  }
  if constexpr (EDGE && BCG) {
    if (ec.bc == ABFT_BC_CONSTANT || ec.bc == ABFT_BC_PERIODIC) {
      const int gy = ec.gyb - 1 + t;
      const bool yo = gy < 0 || gy >= ec.ny;
#pragma unroll
      for (int c2 = 0; c2 < V + 2; ++c2) {
        const int gx = gx0 - 1 + c2;
        if (yo || gx < 0 || gx >= nx) {
          if (ec.bc == ABFT_BC_CONSTANT) {
            W[c2] = ec.g;
          } else {
            const int wy = ((gy % ec.ny) + ec.ny) % ec.ny, wx = ((gx % nx) + nx) % nx;
            W[c2] = gplane[(size_t)wy * ec.px + wx];
          }
        }
      }
    }
  }
}

// Plane-streaming evaluation of Eq. 1 (streamable shapes, the 27-point box):
// the staged plane q is read ONCE per thread and advances the FMA chains of
// three outputs -- u^s[q + 1] (q is its dk = -1 plane: the chain's start, S),
// u^s[q] (dk = 0: the middle, M) and u^s[q - 1] (dk = +1: the chain's end, E).
// Its row t feeds output row r = t - 1 - dj, so the rows stream as well: one
// staged row is live at a time.  Every output's chain still passes through
// the points in their canonical order -- planes in ascending dk, rows in
// ascending dj, di ascending -- so the result is bitwise that of the
// three-plane evaluation, while each staged element is
// loaded (and its x halo exchanged) once instead of three times.
// de / dm / ds: which of the three chains exist (chunk ends; RT = false: all
// three, the steady state, without the runtime tests).
template <typename T, class SH, int RY, bool EDGE, bool BCG, bool RT>
__device__ __forceinline__ void stream_plane(T (&ae)[RY][16 / sizeof(T)], T (&am)[RY][16 / sizeof(T)],
                                             T (&as)[RY][16 / sizeof(T)], bool de, bool dm, bool ds,
                                             const unsigned char* slot, const RowOffs<RY>& ro,
                                             const SweepParams& p, int lane, int gx0, int nx,
                                             const EdgeCtx<T>& ec, const T* gplane) {
  constexpr int V = 16 / (int)sizeof(T), NP = SH::NP;
#pragma unroll
  for (int t = 0; t < RY + 2; ++t) {
    T W[V + 2];
    load_row<T, EDGE, BCG>(W, slot, ro.sro[t], ro.seo[t], t, lane, gx0, nx, ec, gplane);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int di = SH::off(q, 0), dj = SH::off(q, 1), dk = SH::off(q, 2);
      const int r = t - 1 - dj;
      if (r < 0 || r >= RY) continue;
      if (RT && ((dk < 0 && !ds) || (dk == 0 && !dm) || (dk > 0 && !de))) continue;
      T (&acc)[RY][V] = dk < 0 ? as : (dk == 0 ? am : ae);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const T v = W[k + 1 + di];
        // the weight is read from the parameter bank at its use (27 fp64
        // weights in registers would crowd out the three chains)
        acc[r][k] = (q == 0) ? mul_rn(pw<T>(p, q), v) : fma_rn(pw<T>(p, q), v, acc[r][k]);
      }
    }
  }
}

template <typename T, class SH, int RY, bool NZ, bool EDGE, bool BCG = true>
__device__ __forceinline__ void stencil_layer(T (&out)[RY][16 / sizeof(T)], const T* const (&pl)[3],
                                              const RowOffs<RY>& ro, const T (&wr)[SH::NP],
                                              int lane, int gx0, int nx, const EdgeCtx<T>& ec) {
  if constexpr (SH::NP > 9) stencil_layer_grouped<T, SH, RY, NZ, EDGE, BCG>(out, pl, ro, wr, lane, gx0, nx, ec);
  else stencil_layer_all<T, SH, RY, NZ, EDGE, BCG>(out, pl, ro, wr, lane, gx0, nx, ec);
}

// the source field C (HotSpot power) of one layer for this thread's RY x V
// cells, q = its first cell: read-only 128-bit loads, issued one layer ahead
// (register prefetch); FULL tiles load without bounds checks
template <typename T, int RY, bool FULL>
__device__ __forceinline__ void load_src(T (&pv)[RY][16 / sizeof(T)], const T* q, int64_t spx,
                                         int gyb, int gx0, int nx, int ny) {
  constexpr int V = 16 / (int)sizeof(T);
  using VT = typename Vec<T>::type;
#pragma unroll
  for (int r = 0; r < RY; ++r, q += spx) {
    if (FULL || (gyb + r < ny && gx0 + V <= nx)) {
      VT v = __ldg(reinterpret_cast<const VT*>(q));
      const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int k = 0; k < V; ++k) pv[r][k] = e[k];
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) pv[r][k] = (gyb + r < ny && gx0 + k < nx) ? __ldg(q + k) : T(0);
    }
  }
}

// the constant term C of Eq. 1 (sources in the caller's order, fma each):
// FS = the HotSpot pattern [field source, scalar source] with the operands in
// registers; otherwise the runtime list.
template <typename T, int RY, bool FS>
__device__ __forceinline__ void add_sources(T (&out)[RY][16 / sizeof(T)], const T (&pv)[RY][16 / sizeof(T)],
                                            const SweepParams& p, T c0, T c1, T s1) {
  constexpr int V = 16 / (int)sizeof(T);
  if constexpr (FS) {
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int k = 0; k < V; ++k) out[r][k] = fma_rn(c1, s1, fma_rn(c0, pv[r][k], out[r][k]));
  } else {
    for (int q = 0; q < p.nsources; ++q) {
      const T cf = pcoef<T>(p, q);
      const bool fld = q == p.field_src;
      const T sv = pscal<T>(p, q);
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int k = 0; k < V; ++k) out[r][k] = fma_rn(cf, fld ? pv[r][k] : sv, out[r][k]);
    }
  }
}

// K1.  S: ShapeId (SHAPE_GENERIC = runtime point list).  CHK: which actual
// checksums the pass accumulates (K1_CK_*).  VAR: K1_HOT (clamp / zero
// ghosts, no flips), K1_INJ (+ this launch's scheduled bit-flips), K1_GEN
// (+ constant / periodic ghosts).
// grid (x-tiles, y-tiles, z-chunks); each CTA marches up its z-chunk.
template <typename T, int S, int CHK, int VAR>
#ifndef ABFT_K1_MINB
#define ABFT_K1_MINB 2
#endif
#ifndef ABFT_ROWS_DEFERRED
#define ABFT_ROWS_DEFERRED 1
#endif
__global__ void __launch_bounds__(Tile<T>::THREADS, 256 / Tile<T>::THREADS * ABFT_K1_MINB)
    k1_sweep(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ SweepParams p) {
  using TL = Tile<T>;
  constexpr int V = TL::V, TX = TL::TX, HV = TL::HV, HX = TL::HX, RY = TL::RY, TY = TL::TY;
  constexpr int NS = TL::NS, WARPS = TL::WARPS;
  constexpr int TSTR = TL::T_STRIDE / (int)sizeof(T);
  constexpr bool GEN = (S == SHAPE_GENERIC);
  constexpr bool FS = (S == SHAPE_HOTSPOT7_FS);
  constexpr int SS = GEN ? SHAPE_HOTSPOT7 : S;   // any defined shape for the GEN instantiation
  constexpr bool NZ = GEN ? true : shape_needs_z<SS>();
  constexpr int NP = GEN ? 1 : Shape<SS>::NP;
  constexpr bool STREAM = !GEN && sh_streamable<Shape<SS>>();   // plane streaming (27-point box)

  // shared memory: derived from the __shared__ array so every access is LDS/STS
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  T* sT = reinterpret_cast<T*>(base);
  double* sPart = reinterpret_cast<double*>(base + NS * TL::T_STRIDE);   // [2][WARPS][TX]
  uint64_t* barT = reinterpret_cast<uint64_t*>(base + NS * TL::T_STRIDE + TL::PART_BYTES);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = p.nx, ny = p.ny, zc = p.zc;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int zs = p.zr0 + blockIdx.z * p.zchunk, ze = min(zs + p.zchunk, p.zr1);
  const int q0 = NZ ? zs - 1 : zs;
  const int nT = (NZ ? ze + 1 : ze) - q0;
  const bool hasP = p.field_src >= 0;
  const bool xedge = (x0 == 0) || (x0 + TX >= nx);            // clamp / ragged columns
  const bool yedge = (y0 == 0) || (y0 + TY >= ny);
  const int bc = p.bc;
  // tiles that build ghosts in registers: clamp -> x-edge tiles (y through
  // srow); constant / periodic -> every edge tile; zero -> none (TMA zero fill)
  constexpr bool GEN_BC = VAR == K1_GEN, INJ = VAR != K1_HOT;
  const bool edge = bc == ABFT_BC_CLAMP ? xedge : ((bc == ABFT_BC_ZERO || !GEN_BC) ? false : (xedge || yedge));
  const bool full = (x0 + TX <= nx) && (y0 + TY <= ny);       // no masked cells
  const int64_t px = p.px;
  T* const out_base = reinterpret_cast<T*>(p.out);
  double* const Ag = p.A;
  double* const Bg = p.B;
  T* const exl = reinterpret_cast<T*>(p.EX);

  if (tid == 0) {
    prefetch_tmap(&tm_u);
    for (int i = 0; i < NS; ++i) mbar_init(&barT[i], 1);
    fence_mbar_init();
  }
  // the previous sweep's check kernels may still correct u^{s-1} or read the
  // buffer this sweep writes: wait for them (PDL) after the setup above
  grid_dependency_wait();
  __syncthreads();
  auto issue_T = [&](int i) {
    const int st = i % NS;
    mbar_arrive_expect_tx(&barT[st], TL::T_BYTES);
    tma_load_3d(sT + st * TSTR, &tm_u, &barT[st], x0 - HV, y0 - 1,
                zmap(q0 + i, zc, p.has_lo, p.has_hi, p.bc));
  };
  if (tid == 0)
    for (int i = 0; i < NS && i < nT; ++i) issue_T(i);

  // per-thread geometry, loop invariant
  const int gx0 = x0 + lane * V;
  const int ry0 = warp * RY;
  const int gyb = y0 + ry0;
  int srow[RY + 2];  // staged row (x HX) of input row gyb - 1 + t, clamped in y
#pragma unroll
  for (int t = 0; t < RY + 2; ++t)
    srow[t] = ((bc == ABFT_BC_CLAMP ? max(0, min(gyb - 1 + t, ny - 1)) : gyb - 1 + t) - y0 + 1) * HX;
  EdgeCtx<T> ec;
  ec.bc = bc;
  ec.g = (T)p.g;
  ec.px = px;
  ec.gyb = gyb;
  ec.ny = ny;
  T wr[NP];
  if constexpr (!GEN) {
#pragma unroll
    for (int q = 0; q < NP; ++q) wr[q] = pw<T>(p, q);
  }
  T c0 = T(0), c1 = T(0), s1 = T(0);
  if constexpr (FS) { c0 = pcoef<T>(p, 0); c1 = pcoef<T>(p, 1); s1 = pscal<T>(p, 1); }
  // source-field registers of two consecutive layers, ping-ponged by the
  // 2-way unrolled layer loop below (no register copies per layer)
  T pa[RY][V], pb[RY][V];
  const T* psrc = hasP ? reinterpret_cast<const T*>(p.src) + (size_t)zs * p.splane + (size_t)gyb * p.spx + gx0
                       : nullptr;
  auto src_layer = [&](T (&dst)[RY][V], const T* q) {
    if (full) load_src<T, RY, true>(dst, q, p.spx, gyb, gx0, nx, ny);
    else load_src<T, RY, false>(dst, q, p.spx, gyb, gx0, nx, ny);
  };
  if (hasP && !STREAM) src_layer(pa, psrc);
  // output row of this thread in layer zs (buffer layer zs + 1), advanced per layer
  T* orow = out_base + (size_t)(zs + 1) * p.plane + (size_t)gyb * px + gx0;
  const RowOffs<RY> ro = row_offsets<T, RY>(srow, lane);

  double rsp[RY];   // row partials of the previous layer, pending reduction
  int zprev = -1;
  auto flush_rows = [&](int zl) {
    const double tot = row_reduce<RY>(rsp, lane);
    const int gy = gyb + row_of_lane<RY>(lane);
    if (final_lane<RY>(lane) && gy < ny) atomicAdd(&Bg[(size_t)(zl + 1) * ny + gy], tot);
  };
  (void)flush_rows;
  // per output layer z: the sources C, the flips, the store, the halo and
  // ledger copies, the checksums (Eqs. 2-3) and the ring barrier
  auto epilogue = [&](const int z, T (&out)[RY][V], const T (&pv)[RY][V]) {
    const int it = z - zs;
#if ABFT_ROWS_DEFERRED
    if constexpr (CHK != K1_CK_NONE) {
      if (zprev >= 0) flush_rows(zprev);   // b of the previous layer (Eq. 3)
    }
#endif
    add_sources<T, RY, FS>(out, pv, p, c0, c1, s1);   // constant term C of Eq. 1
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
    T* obase = orow + (size_t)it * p.plane;
    using VT = typename Vec<T>::type;
    if (full) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        VT v;
        T* e = reinterpret_cast<T*>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) e[k] = out[r][k];
        *reinterpret_cast<VT*>(obase + (size_t)r * px) = v;
      }
    } else {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (gyb + r >= ny) continue;
        T* o = obase + (size_t)r * px;
        if (gx0 + V <= nx) {
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
    // fused halo (local group): the boundary layers also go straight into the
    // neighbours' halo layer (same device, or a peer GPU over NVLink)
    for (int f = 0; f < 2; ++f) {
      T* ph = reinterpret_cast<T*>(p.peerU[f]);
      if (!ph || z != (f == 0 ? 0 : zc - 1)) continue;
      T* pbase = ph + (size_t)gyb * px + gx0;
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        if (gyb + r >= ny) continue;
        T* o = pbase + (size_t)r * px;
        if (full || gx0 + V <= nx) {
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
    // ledger for Theorem 1's beta terms of the next check: the x-edge columns
    // (only the lane holding column 0 or nx - 1 branches in: a per-cell
    // compare in every lane of an edge tile cost ~1 ISETP per cell)
    if (exl && xedge) {
      const size_t lay = (size_t)(z + 1) * ny;
      const int kr = nx - 1 - gx0;   // column nx - 1 in this thread's vector?
      if (gx0 == 0) {
#pragma unroll
        for (int r = 0; r < RY; ++r)
          if (gyb + r < ny) exl[lay + gyb + r] = out[r][0];
      }
      if (kr >= 0 && kr < V) {
        T* exr = exl + (size_t)(zc + 2) * ny + lay + gyb;
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          T v = out[r][0];
#pragma unroll
          for (int k = 1; k < V; ++k) v = k == kr ? out[r][k] : v;
          if (gyb + r < ny) exr[r] = v;
        }
      }
    }
    double* part = sPart + (it & 1) * (WARPS * TX);
    if constexpr (CHK != K1_CK_NONE) {
      double rs[RY], cs[V];
      if constexpr (CHK == K1_CK_AB) {
        if (full) partial_sums<T, true>(out, rs, cs, gyb, gx0, nx, ny);
        else partial_sums<T, false>(out, rs, cs, gyb, gx0, nx, ny);
      } else {
        if (full) row_sums<T, true>(out, rs, gyb, gx0, nx, ny);
        else row_sums<T, false>(out, rs, gyb, gx0, nx, ny);
      }
#if ABFT_ROWS_DEFERRED
      // the warp reduction of these row partials runs in the next layer's body
      // (off this layer's critical path; its shuffles overlap the next stencil)
#pragma unroll
      for (int r = 0; r < RY; ++r) rsp[r] = rs[r];
      zprev = z;
#else
      // b^s_y += sum over this tile's columns (Eq. 3)
      const double tot = row_reduce<RY>(rs, lane);
      const int gy = gyb + row_of_lane<RY>(lane);
      if (final_lane<RY>(lane) && gy < ny) atomicAdd(&Bg[(size_t)(z + 1) * ny + gy], tot);
#endif
      if constexpr (CHK == K1_CK_AB) {
        // column partials of this layer; double-buffered, so the one barrier per
        // layer below also orders them against the reduction two layers later
#pragma unroll
        for (int k = 0; k < V; ++k) part[warp * TX + lane * V + k] = cs[k];
      }
    }
    {
      __syncthreads();  // lowest staged layer consumed; this layer's column partials complete
      if (tid == 0) {
        fence_proxy_async();
        // the slot this layer freed: the lowest of its three planes, or
        // (plane streaming) the one plane it read, two layers further on
        const int fr = STREAM ? it + 2 : it;
        if (fr + NS < nT) issue_T(fr + NS);
      }
    }
    if constexpr (CHK == K1_CK_AB) {
      // a^s_x += sum over this tile's rows (Eq. 2)
      if (tid < TX) {
        double s = part[tid];
#pragma unroll
        for (int w = 1; w < WARPS; ++w) s += part[w * TX + tid];
        if (x0 + tid < nx) atomicAdd(&Ag[(size_t)(z + 1) * nx + x0 + tid], s);
      }
    }
  };
  auto layer = [&](const int z, T (&pv)[RY][V], T (&pn)[RY][V]) {
    const int it = z - zs;
    const T* pl[3];
    if (NZ) {
      // entries it, it+1 were waited for by the previous layer (or here, first)
      if (it == 0) {
        mbar_wait(&barT[0], 0);
        mbar_wait(&barT[1 % NS], (1 / NS) & 1);
      }
      mbar_wait(&barT[(it + 2) % NS], ((it + 2) / NS) & 1);
#pragma unroll
      for (int d = 0; d < 3; ++d) pl[d] = sT + ((it + d) % NS) * TSTR;
    } else {
      mbar_wait(&barT[it % NS], (it / NS) & 1);
      pl[0] = pl[2] = pl[1] = sT + (it % NS) * TSTR;
    }
    if (hasP && z + 1 < ze) src_layer(pn, psrc + (size_t)(it + 1) * p.splane);

    T out[RY][V];
    if constexpr (!GEN) {
      // CTA-uniform split: only tiles touching x = 0 / x = nx - 1 pay the clamp
      if (edge) {
        if constexpr (GEN_BC) {
          const T* ub = reinterpret_cast<const T*>(p.uin);
#pragma unroll
          for (int d = 0; d < 3; ++d)
            ec.up[d] = ub + (size_t)(NZ ? zmap(z - 1 + d, zc, p.has_lo, p.has_hi, bc) : z + 1) * p.plane;
        }
        stencil_layer<T, Shape<SS>, RY, NZ, true, GEN_BC>(out, pl, ro, wr, lane, gx0, nx, ec);
      } else {
        stencil_layer<T, Shape<SS>, RY, NZ, false, GEN_BC>(out, pl, ro, wr, lane, gx0, nx, ec);
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
            const int yy = gyb + r + dj, xx = gx0 + k + di;
            T v;
            if (bc == ABFT_BC_CLAMP || (yy >= 0 && yy < ny && xx >= 0 && xx < nx) ||
                (!GEN_BC && bc != ABFT_BC_ZERO)) {
              const int sr = (max(0, min(yy, ny - 1)) - y0 + 1) * HX;
              const int sc = max(0, min(xx, nx - 1)) - x0 + HV;
              v = pp[sr + sc];
            } else if (bc == ABFT_BC_PERIODIC) {
              const T* ub = reinterpret_cast<const T*>(p.uin) +
                            (size_t)(NZ ? zmap(z + dk, zc, p.has_lo, p.has_hi, bc) : z + 1) * p.plane;
              v = ub[(size_t)(((yy % ny) + ny) % ny) * px + ((xx % nx) + nx) % nx];
            } else {
              v = bc == ABFT_BC_CONSTANT ? (T)p.g : T(0);
            }
            const T w = pw<T>(p, q);
            acc = (q == 0) ? mul_rn(w, v) : fma_rn(w, v, acc);
          }
          out[r][k] = acc;
        }
      }
    }
    epilogue(z, out, pv);
  };
  if constexpr (STREAM) {
    // plane streaming (the 27-point box): staged plane q
    // advances the chains of u^s[q + 1], u^s[q] and u^s[q - 1] (stream_plane);
    // three accumulator sets rotate through the roles start / middle / end
    (void)layer;
    // E: u^s[z] (start and middle done), M: u^s[z + 1] (start done), S: u^s[z + 2];
    // after each layer the roles rotate by register moves (E <- M <- S), so
    // the loop body holds one copy of the plane code (instruction cache)
    T E[RY][V], M[RY][V], S[RY][V];
    const T* ub = reinterpret_cast<const T*>(p.uin);
    auto splane = [&](int i, bool rt, bool de, bool dm, bool ds) {
      mbar_wait(&barT[i % NS], (i / NS) & 1);   // ring slot i holds plane q0 + i
      const unsigned char* slot = reinterpret_cast<const unsigned char*>(sT + (i % NS) * TSTR);
      const T* gpl = GEN_BC ? ub + (size_t)zmap(q0 + i, zc, p.has_lo, p.has_hi, bc) * p.plane : nullptr;
      using SHP = Shape<SS>;
      if (rt) {
        if (edge) stream_plane<T, SHP, RY, true, GEN_BC, true>(E, M, S, de, dm, ds, slot, ro, p, lane, gx0, nx, ec, gpl);
        else stream_plane<T, SHP, RY, false, GEN_BC, true>(E, M, S, de, dm, ds, slot, ro, p, lane, gx0, nx, ec, gpl);
      } else {
        if (edge) stream_plane<T, SHP, RY, true, GEN_BC, false>(E, M, S, de, dm, ds, slot, ro, p, lane, gx0, nx, ec, gpl);
        else stream_plane<T, SHP, RY, false, GEN_BC, false>(E, M, S, de, dm, ds, slot, ro, p, lane, gx0, nx, ec, gpl);
      }
    };
    auto rotate = [&]() {
#pragma unroll
      for (int r = 0; r < RY; ++r)
#pragma unroll
        for (int k = 0; k < V; ++k) { E[r][k] = M[r][k]; M[r][k] = S[r][k]; }
    };
    // prologue: plane zs - 1 starts u^s[zs] (its only role here); plane zs
    // continues u^s[zs] and starts u^s[zs + 1] -- each as if it ended the
    // layer before, then the roles rotate
    splane(0, true, false, false, true);
    rotate();
    splane(1, true, false, true, zs + 1 < ze);
    rotate();
    __syncthreads();   // planes zs - 1 and zs are consumed: refill their slots
    if (tid == 0) {
      fence_proxy_async();
      for (int i = 0; i < 2; ++i)
        if (i + NS < nT) issue_T(i + NS);
    }
#pragma unroll 1
    for (int z = zs; z < ze; ++z) {
      T pv[RY][V];
      if (hasP) src_layer(pv, psrc + (size_t)(z - zs) * p.splane);
      splane(z - zs + 2, z + 2 >= ze, true, z + 1 < ze, z + 2 < ze);   // plane z + 1 ends u^s[z]
      epilogue(z, E, pv);
      rotate();
    }
  } else {
    int z = zs;
    for (; z + 1 < ze; z += 2) {
      layer(z, pa, pb);
      layer(z + 1, pb, pa);
    }
    if (z < ze) layer(z, pa, pb);
  }
#if ABFT_ROWS_DEFERRED
  if constexpr (CHK != K1_CK_NONE) {
    if (zprev >= 0) flush_rows(zprev);
  }
#endif
  // pipelined schedule: count this CTA done once its stores and checksum
  // atomics are visible (the checks of the previous sweep may wait for it):
  // the CTA barrier, then one release reduction (cumulative over the
  // barrier).  A __threadfence() here would make ptxas turn every checksum
  // RED in the kernel into an ATOM that waits for its return (K1 BOTH +3.4%)
  if (p.done) {
    __syncthreads();
    if (tid == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.done) : "memory");
  }
}

}  // namespace abft
