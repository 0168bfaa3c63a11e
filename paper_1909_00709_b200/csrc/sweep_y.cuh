// sweep_y.cuh -- K1 for 3D stencils: the y-march.  Same numeric contract as
// the z-march of sweep.cuh (Eq. 1 as the canonical FMA chain, PAPER.md:250-254;
// the actual checksums Eqs. 2-3, in the same pass), different
// traversal, chosen for where the checksums live:
//
//  * a CTA owns an x-tile of TX columns and a z-tile of TZ layers and slides
//    along y.  Each step stages the (x, z) slice at one y -- TZ + 2 layers with
//    the 1-layer z halo and a 16-byte x halo -- by TMA into an NS-deep ring;
//    the stencil reads slices y-1, y, y+1 (the point list with y and z
//    exchanged, SwapYZ);
//  * a_x of layer z (Eq. 2, the sum over y) is exactly what a thread
//    accumulates while it slides: fp64 registers, one RED per cell of the
//    tile per segment instead of one per tile-row and step -- no shared
//    memory, no barrier;
//  * b_y of layer z (Eq. 3, the sum over x) is a warp reduction (transposed
//    shuffles) and one fp64 RED per (x-tile, layer, y) into the L2-resident
//    generation;
//  * full/empty mbarrier pairs per ring slot, no CTA barrier in the loop:
//    lane 0 of warp 0 also produces (issues the TMA loads LA slices ahead of
//    its own step, blocking only when it runs 2 steps ahead of the slowest
//    warp), so all 16 warps compute with 128 registers each;
//  * persistent: one CTA per SM, each takes an equal contiguous share of the
//    (tile, y) rows (segments restart the ring, flush a_x), so the grid has no
//    tail wave.
// Fault injection and the x-edge ledger for Theorem 1's beta terms are
// as in the z-march.
#pragma once

#include "sweep.cuh"

namespace abft {

template <typename T> struct YTile {
  static constexpr int V = 16 / (int)sizeof(T);
  static constexpr int TX = 32 * V;
  static constexpr int HV = V;
  static constexpr int HX = TX + 2 * HV;
  static constexpr int CW = 16;                 // warps
  static constexpr int RZ = 2;                  // z-rows per thread
  static constexpr int TZ = CW * RZ;            // layers per tile
  static constexpr int ROWS = TZ + 2;
  static constexpr int THREADS = 32 * CW;
  static constexpr int S_BYTES = ROWS * HX * (int)sizeof(T);
  static constexpr int S_STRIDE = (S_BYTES + 127) / 128 * 128;
  static constexpr int P_BYTES = TX * TZ * (int)sizeof(T);
  static constexpr int P_STRIDE = (P_BYTES + 127) / 128 * 128;
  static constexpr int NS = 7;    // slices y-1, y, y+1 in use + LA in flight + 2 slack
  static constexpr int NSP = 4;   // source slices
  static constexpr int LA = NS - 4;    // slices issued beyond y+1
  static constexpr int LAP = NSP - 2;  // source slices issued beyond y
  static constexpr int BAR_BYTES = 2 * (NS + NSP) * 8;
  static constexpr int SMEM = NS * S_STRIDE + NSP * P_STRIDE + BAR_BYTES + 128;
};

// K1, y-march.  S: ShapeId (SHAPE_GENERIC = runtime point list).  CHK: the
// actual checksums.  INJ: this launch's scheduled bit-flips.  grid = (G),
// G = resident CTAs; p.ntx x p.ntz tiles of ny rows each are split evenly.
template <typename T, int S, bool CHK, bool INJ>
__global__ void __launch_bounds__(YTile<T>::THREADS, 1)
    k1_ymarch(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_src,
              const __grid_constant__ SweepParams p) {
  using TL = YTile<T>;
  constexpr int V = TL::V, TX = TL::TX, HV = TL::HV, HX = TL::HX, RZ = TL::RZ, TZ = TL::TZ;
  constexpr int NS = TL::NS, NSP = TL::NSP, CW = TL::CW;
  constexpr int SSTR = TL::S_STRIDE / (int)sizeof(T), PSTR = TL::P_STRIDE / (int)sizeof(T);
  constexpr bool GEN = (S == SHAPE_GENERIC);
  constexpr int SS = GEN ? SHAPE_HOTSPOT7 : S;
  constexpr int NP = GEN ? 1 : Shape<SS>::NP;
  using SH = SwapYZ<SS>;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  T* sT = reinterpret_cast<T*>(base);
  T* sP = reinterpret_cast<T*>(base + NS * TL::S_STRIDE);
  uint64_t* fullT = reinterpret_cast<uint64_t*>(base + NS * TL::S_STRIDE + NSP * TL::P_STRIDE);
  uint64_t* emptyT = fullT + NS;
  uint64_t* fullP = emptyT + NS;
  uint64_t* emptyP = fullP + NSP;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = p.nx, ny = p.ny, zc = p.zc, ntx = p.ntx;
  const bool hasP = p.field_src >= 0;
  const int64_t total = (int64_t)p.ntx * p.ntz * ny;
  const int64_t beg = total * blockIdx.x / gridDim.x, end = total * (blockIdx.x + 1) / gridDim.x;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&fullT[i], 1); mbar_init(&emptyT[i], CW); }
    for (int i = 0; i < NSP; ++i) { mbar_init(&fullP[i], 1); mbar_init(&emptyP[i], CW); }
    fence_mbar_init();
  }
  __syncthreads();

  // ---- producer state (lane 0 of warp 0): issued entries and segment cursors.
  // Field entries: per segment the slices ya-1 .. yb (clamped in y);
  // source entries: per segment the slices ya .. yb-1.
  uint32_t pT = 0, pP = 0;
  int64_t tIdx = beg, qIdx = beg;
  int tI = 0, qI = 0;
  auto seg = [&](int64_t i0, int& x0s, int& zt0s, int& yas, int& ns) {
    const int64_t tile = i0 / ny;
    yas = (int)(i0 % ny);
    ns = (int)min((int64_t)ny - yas, end - i0);
    x0s = (int)(tile % ntx) * TX;
    zt0s = (int)(tile / ntx) * TZ;
  };
  auto produce = [&](uint32_t wantT, uint32_t wantP) {
    int x0s, zt0s, yas, ns;
    while (pT < wantT && tIdx < end) {
      seg(tIdx, x0s, zt0s, yas, ns);
      const int st = pT % NS;
      if (pT >= NS) mbar_wait(&emptyT[st], ((pT / NS) - 1) & 1);
      mbar_arrive_expect_tx(&fullT[st], TL::S_BYTES);
      tma_load_3d(sT + st * SSTR, &tm_u, &fullT[st], x0s - HV, max(0, min(yas - 1 + tI, ny - 1)), zt0s);
      ++pT;
      if (++tI == ns + 2) { tI = 0; tIdx += ns; }
    }
    while (hasP && pP < wantP && qIdx < end) {
      seg(qIdx, x0s, zt0s, yas, ns);
      const int st = pP % NSP;
      if (pP >= NSP) mbar_wait(&emptyP[st], ((pP / NSP) - 1) & 1);
      mbar_arrive_expect_tx(&fullP[st], TL::P_BYTES);
      tma_load_3d(sP + st * PSTR, &tm_src, &fullP[st], x0s, yas + qI, zt0s);
      ++pP;
      if (++qI == ns) { qI = 0; qIdx += ns; }
    }
  };
  if (tid == 0) {
    prefetch_tmap(&tm_u);
    if (hasP) prefetch_tmap(&tm_src);
  }

  uint32_t gT = 0, gP = 0;
  T wr[NP];
  if constexpr (!GEN) {
#pragma unroll
    for (int q = 0; q < NP; ++q) wr[q] = pw<T>(p, q);
  }
  T* const out_base = reinterpret_cast<T*>(p.out);
  T* const exl = reinterpret_cast<T*>(p.EX);
  const size_t side = (size_t)(zc + 2) * ny;

  for (int64_t idx = beg; idx < end;) {
    const int64_t tile = idx / ny;
    const int ya = (int)(idx % ny);
    const int yb = (int)min((int64_t)ny, (int64_t)ya + (end - idx));
    const int x0 = (int)(tile % ntx) * TX, zt0 = (int)(tile / ntx) * TZ;
    const int gx0 = x0 + lane * V;
    const int zq0 = zt0 + warp * RZ;     // first output layer of this thread
    const bool xedge = (x0 == 0) || (x0 + TX >= nx);
    const bool wfull = (x0 + TX <= nx) && (zq0 + RZ <= zc);
    int srow[RZ + 2];   // staged row of layer zq0 - 1 + t: clamp / halo via zmap
#pragma unroll
    for (int t = 0; t < RZ + 2; ++t) srow[t] = (zmap(zq0 - 1 + t, zc, p.has_lo, p.has_hi) - zt0) * HX;
    double accA[RZ][V];
#pragma unroll
    for (int r = 0; r < RZ; ++r)
#pragma unroll
      for (int k = 0; k < V; ++k) accA[r][k] = 0.0;

    if (warp == 0) {
      if (lane == 0) produce(gT + 2, gP);
      __syncwarp();
    }
    mbar_wait(&fullT[gT % NS], (gT / NS) & 1);
    mbar_wait(&fullT[(gT + 1) % NS], ((gT + 1) / NS) & 1);
    for (int y = ya; y < yb; ++y) {
      if (warp == 0) {
        if (lane == 0) produce(gT + 3 + TL::LA, gP + 1 + TL::LAP);
        __syncwarp();
      }
      mbar_wait(&fullT[(gT + 2) % NS], ((gT + 2) / NS) & 1);
      const T* pl[3] = {sT + (gT % NS) * SSTR, sT + ((gT + 1) % NS) * SSTR, sT + ((gT + 2) % NS) * SSTR};
      const T* ps = sP + (gP % NSP) * PSTR;
      if (hasP) mbar_wait(&fullP[gP % NSP], (gP / NSP) & 1);

      T out[RZ][V];
      if constexpr (!GEN) {
        EdgeCtx<T> ec{};          // the y-march runs clamp only
        ec.bc = ABFT_BC_CLAMP;
        const RowOffs<RZ> ro = row_offsets<T, RZ>(srow, lane);
        if (xedge) stencil_layer<T, SH, RZ, true, true>(out, pl, ro, wr, lane, gx0, nx, ec);
        else stencil_layer<T, SH, RZ, true, false>(out, pl, ro, wr, lane, gx0, nx, ec);
      } else {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
#pragma unroll
          for (int k = 0; k < V; ++k) {
            T acc = T(0);
            for (int q = 0; q < p.npoints; ++q) {
              const int di = p.di[q], dj = p.dj[q], dk = p.dk[q];
              const T* pp = dj < 0 ? pl[0] : (dj > 0 ? pl[2] : pl[1]);
              const int sr = (zmap(zq0 + r + dk, zc, p.has_lo, p.has_hi) - zt0) * HX;
              const int sc = max(0, min(gx0 + k + di, nx - 1)) - x0 + HV;
              const T v = pp[sr + sc];
              const T w = pw<T>(p, q);
              acc = (q == 0) ? mul_rn(w, v) : fma_rn(w, v, acc);
            }
            out[r][k] = acc;
          }
        }
      }
      // constant term C of Eq. 1: sources in order
      for (int q = 0; q < p.nsources; ++q) {
        const T cf = pcoef<T>(p, q);
        if (q == p.field_src) {
#pragma unroll
          for (int r = 0; r < RZ; ++r) {
            T pv[V];
            ld_vec<T, V>(pv, ps + (warp * RZ + r) * TX + lane * V);
#pragma unroll
            for (int k = 0; k < V; ++k) out[r][k] = fma_rn(cf, pv[k], out[r][k]);
          }
        } else {
          const T sv = pscal<T>(p, q);
#pragma unroll
          for (int r = 0; r < RZ; ++r)
#pragma unroll
            for (int k = 0; k < V; ++k) out[r][k] = fma_rn(cf, sv, out[r][k]);
        }
      }
      // every read of slice y-1 and of the source slice is done
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&emptyT[gT % NS]);
        if (hasP) mbar_arrive(&emptyP[gP % NSP]);
      }
      ++gT;
      if (hasP) ++gP;

      if constexpr (INJ) {  // after the update, before the store
        for (int f = 0; f < p.nfaults; ++f) {
          const LocalFault F = p.faults[f];
          if (F.y != y) continue;
#pragma unroll
          for (int r = 0; r < RZ; ++r)
#pragma unroll
            for (int k = 0; k < V; ++k)
              if (F.z == zq0 + r && F.x == gx0 + k) out[r][k] = flip_bit(out[r][k], F.bit);
        }
      }
      // store: one 16-byte vector per layer row
      using VT = typename Vec<T>::type;
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        T* o = out_base + (size_t)(zq0 + r + 1) * p.plane + (size_t)y * p.px + gx0;
        if (wfull || (zq0 + r < zc && gx0 + V <= nx)) {
          VT v;
          T* e = reinterpret_cast<T*>(&v);
#pragma unroll
          for (int k = 0; k < V; ++k) e[k] = out[r][k];
          *reinterpret_cast<VT*>(o) = v;
        } else if (zq0 + r < zc) {
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (gx0 + k < nx) o[k] = out[r][k];
        }
      }
      // ledger for Theorem 1's beta terms of the next check: the x-edge columns
      if (exl && xedge) {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          if (zq0 + r >= zc) continue;
          const size_t lay = (size_t)(zq0 + r + 1) * ny + y;
#pragma unroll
          for (int k = 0; k < V; ++k) {
            if (gx0 + k == 0) exl[lay] = out[r][k];
            if (gx0 + k == nx - 1) exl[side + lay] = out[r][k];
          }
        }
      }
      if constexpr (CHK) {
        double rs[RZ];
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
#pragma unroll
          for (int k = 0; k < V; ++k) {
            double d = (double)out[r][k];
            if (!wfull) d = (zq0 + r < zc && gx0 + k < nx) ? d : 0.0;
            rs[r] = k == 0 ? d : rs[r] + d;
            accA[r][k] += d;                       // a_x: sum over y (Eq. 2)
          }
        }
        // b_y += sum over this tile's columns (Eq. 3)
        const double tot = row_reduce<RZ>(rs, lane);
        const int gz = zq0 + row_of_lane<RZ>(lane);
        if (final_lane<RZ>(lane) && gz < zc) atomicAdd(&p.B[(size_t)(gz + 1) * ny + y], tot);
      }
    }
    // release the last two slices of the segment
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&emptyT[gT % NS]);
      mbar_arrive(&emptyT[(gT + 1) % NS]);
    }
    gT += 2;
    if constexpr (CHK) {
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        if (zq0 + r >= zc) continue;
#pragma unroll
        for (int k = 0; k < V; ++k)
          if (gx0 + k < nx) atomicAdd(&p.A[(size_t)(zq0 + r + 1) * nx + gx0 + k], accA[r][k]);
      }
    }
    idx += yb - ya;
  }
}

}  // namespace abft
