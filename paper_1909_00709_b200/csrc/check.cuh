// check.cuh -- K2: per-layer prediction / compare / locate / correct
// (steps (2)-(5) of include/abft_stencil.h) and K0: the initial checksums.
//
// One CTA per z-layer.  The predicted checksums follow Theorem 1 (PAPER.md:
// 314-336) point by point in the caller's order, in fp64 with separately
// rounded products and sums, the vertical points reading the neighbour
// layer's checksum vector, alpha/beta from the edge rows /
// columns of u^{s-1} under clamp (Q3).  The compare is fig.detect
// in fp64; the locate is the intersection of the flagged row and
// column; the correction is Eq. 8 averaged over both checksums
// (fig.correction), with (a - u) evaluated as the sum of the other
// cells of the column (Q11) and the checksums repaired exactly (Q12).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace abft {

__device__ __forceinline__ int flag_rel(double pred, double act, double eps) {
  // fig.detect: rel = |pred / act - 1|; flagged iff !(rel <= eps); equal never flagged
  if (pred == act) return 0;
  const double rel = fabs(__dadd_rn(__ddiv_rn(pred, act), -1.0));
  return !(rel <= eps);
}

template <int NT> __device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < NT / 32; ++w) s += red[w];
  return s;  // valid on thread 0
}

__device__ __forceinline__ void push_record(DevState* st, const abft_record& r) {
  const unsigned long long i = atomicAdd(&st->nrec, 1ull);
  if (i < (unsigned long long)kRecordCap) st->rec[i] = r;
}
__device__ __forceinline__ void bump(DevState* st, int k, long long v = 1) {
  atomicAdd(reinterpret_cast<unsigned long long*>(&st->cnt[k]), (unsigned long long)v);
}

#ifndef ABFT_CHECK_THREADS
#define ABFT_CHECK_THREADS 128
#endif
constexpr int kCheckThreads = ABFT_CHECK_THREADS;   // 9+ CTAs per SM: a 1024-layer slab in one wave

// one entry of a'_x (A == true) or b'_y of layer z, Theorem 1 (Eqs. 4-5):
//   a'_x = c_x + sum_S w (a_{zeta(z+k)}[x+i] + alpha_{x+i, j})
//   b'_y = c_y + sum_S w (b_{zeta(z+k)}[y+j] + beta_{i, y+j})
// points in the caller's order, fp64, separately rounded; all loads issued first.
template <typename T, int S, bool A, bool BCG>
__device__ __forceinline__ double predict_entry(const CheckParams& p, int z, int e) {
  constexpr bool GEN = S == SHAPE_GENERIC;
  constexpr int NPM = GEN ? kMaxPoints : Shape<(GEN ? SHAPE_HOTSPOT7 : S)>::NP;
  const int nx = p.nx, ny = p.ny, zc = p.zc;
  const int np = GEN ? p.npoints : NPM;
  const T* up = reinterpret_cast<const T*>(p.uprev);
  const T* ex = reinterpret_cast<const T*>(p.EXp);
  const size_t side = (size_t)(zc + 2) * ny;
  double Sv[NPM];
#pragma unroll
  for (int q = 0; q < NPM; ++q) {
    if (q >= np) break;
    int di, dj, dk;
    if constexpr (GEN) { di = p.di[q]; dj = p.dj[q]; dk = p.dk[q]; }
    else { di = Shape<S>::off(q, 0); dj = Shape<S>::off(q, 1); dk = Shape<S>::off(q, 2); }
    const int bc = BCG ? p.bc : ABFT_BC_CLAMP;   // BCG: periodic / zero / constant ghosts
    const bool ghostv = bc == ABFT_BC_ZERO || bc == ABFT_BC_CONSTANT;
    const double g = bc == ABFT_BC_CONSTANT ? p.g : 0.0;
    const int zq = zmap(z + dk, zc, p.has_lo, p.has_hi, bc);
    const bool zg = zghost(z + dk, zc, p.has_lo, p.has_hi, bc);
    if (A) {
      const int xs = e + di;
      const bool xg = ghostv && (xs < 0 || xs >= nx);
      if (zg || xg) {          // the shifted column lies in the ghost region
        Sv[q] = __dmul_rn((double)ny, g);
        continue;
      }
      const int xr = (xs >= 0 && xs < nx) ? xs : (bc == ABFT_BC_PERIODIC ? wrap(xs, nx) : max(0, min(xs, nx - 1)));
      double s = p.Ap[(size_t)zq * nx + xr];
      if (dj != 0) {   // alpha at the shifted column (Q3): ghost row minus the far edge row
        const T* col = up + (size_t)zq * p.plane + xr;
        const double top = (double)col[0], bot = (double)col[(size_t)(ny - 1) * p.px];
        // value of row -1 / row ny: clamp top / bot, periodic bot / top, zero 0, constant g
        const double gt = bc == ABFT_BC_CLAMP ? top : (bc == ABFT_BC_PERIODIC ? bot : g);
        const double gb = bc == ABFT_BC_CLAMP ? bot : (bc == ABFT_BC_PERIODIC ? top : g);
        s = __dadd_rn(s, dj < 0 ? __dsub_rn(gt, bot) : __dsub_rn(gb, top));
      }
      Sv[q] = s;
    } else {
      const int ys = e + dj;
      const bool yg = ghostv && (ys < 0 || ys >= ny);
      if (zg || yg) {
        Sv[q] = __dmul_rn((double)nx, g);
        continue;
      }
      const int yr = (ys >= 0 && ys < ny) ? ys : (bc == ABFT_BC_PERIODIC ? wrap(ys, ny) : max(0, min(ys, ny - 1)));
      double s = p.Bp[(size_t)zq * ny + yr];
      if (di != 0) {   // beta: the x-edge columns of u^{s-1} (ledger, or the halo layer itself)
        double lft, rgt;
        if (ex && zq >= 1 && zq <= zc) {
          lft = (double)ex[(size_t)zq * ny + yr];
          rgt = (double)ex[side + (size_t)zq * ny + yr];
        } else {
          const T* row = up + (size_t)zq * p.plane + (size_t)yr * p.px;
          lft = (double)row[0];
          rgt = (double)row[nx - 1];
        }
        const double gl = bc == ABFT_BC_CLAMP ? lft : (bc == ABFT_BC_PERIODIC ? rgt : g);
        const double gr = bc == ABFT_BC_CLAMP ? rgt : (bc == ABFT_BC_PERIODIC ? lft : g);
        s = __dadd_rn(s, di < 0 ? __dsub_rn(gl, rgt) : __dsub_rn(gr, lft));
      }
      Sv[q] = s;
    }
  }
  double acc = A ? p.cA[(size_t)z * nx + e] : p.cB[(size_t)z * ny + e];
#pragma unroll
  for (int q = 0; q < NPM; ++q) {
    if (q >= np) break;
    acc = __dadd_rn(acc, __dmul_rn(p.w[q], Sv[q]));
  }
  return acc;
}

// The layer-uniform part of the prediction of layer z (the same for every
// entry a CTA predicts, computed once per CTA instead of once per point and
// entry): per plane offset dk = d - 1 the predictor row of layer zeta(z + dk),
// whether that layer is a zero / constant ghost, the layer of u^{s-1} (alpha:
// its top / bottom rows; beta without a ledger: its edge columns) and the
// x-edge ledger rows of u^{s-1} (beta).
template <typename T, bool A>
struct PredLayer {
  const double* prow[3];
  const T* lay[3];
  const T* exl[3];
  const T* exr[3];
  bool zg[3];
  const double* crow;
};
template <typename T, bool A, bool BCG>
__device__ __forceinline__ PredLayer<T, A> pred_layer(const CheckParams& p, int z) {
  PredLayer<T, A> L;
  const int bc = BCG ? p.bc : ABFT_BC_CLAMP;
  const T* up = reinterpret_cast<const T*>(p.uprev);
  const T* ex = reinterpret_cast<const T*>(p.EXp);
  const size_t side = (size_t)(p.zc + 2) * p.ny;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int zq = zmap(z + d - 1, p.zc, p.has_lo, p.has_hi, bc);
    L.zg[d] = zghost(z + d - 1, p.zc, p.has_lo, p.has_hi, bc);
    L.prow[d] = A ? p.Ap + (size_t)zq * p.nx : p.Bp + (size_t)zq * p.ny;
    L.lay[d] = up + (size_t)zq * p.plane;
    const bool led = !A && ex && zq >= 1 && zq <= p.zc;
    L.exl[d] = led ? ex + (size_t)zq * p.ny : nullptr;
    L.exr[d] = led ? ex + side + (size_t)zq * p.ny : nullptr;
  }
  L.crow = A ? p.cA + (size_t)z * p.nx : p.cB + (size_t)z * p.ny;
  return L;
}
// predict_entry for a compile-time point list with the layer part hoisted:
// the same operations in the same order, so the same bits
template <typename T, int S, bool A, bool BCG>
__device__ __forceinline__ double predict_entry_l(const CheckParams& p, const PredLayer<T, A>& L, int e) {
  using SH = Shape<S>;
  constexpr int NP = SH::NP;
  const int nx = p.nx, ny = p.ny;
  const int bc = BCG ? p.bc : ABFT_BC_CLAMP;
  const bool ghostv = bc == ABFT_BC_ZERO || bc == ABFT_BC_CONSTANT;
  const double g = bc == ABFT_BC_CONSTANT ? p.g : 0.0;
  double Sv[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int di = SH::off(q, 0), dj = SH::off(q, 1), d = SH::off(q, 2) + 1;
    if (A) {
      const int xs = e + di;
      const bool xg = ghostv && (xs < 0 || xs >= nx);
      if (L.zg[d] || xg) {
        Sv[q] = __dmul_rn((double)ny, g);
        continue;
      }
      const int xr = (xs >= 0 && xs < nx) ? xs : (bc == ABFT_BC_PERIODIC ? wrap(xs, nx) : max(0, min(xs, nx - 1)));
      double s = L.prow[d][xr];
      if (dj != 0) {   // alpha at the shifted column (Q3)
        const T* col = L.lay[d] + xr;
        const double top = (double)col[0], bot = (double)col[(size_t)(ny - 1) * p.px];
        const double gt = bc == ABFT_BC_CLAMP ? top : (bc == ABFT_BC_PERIODIC ? bot : g);
        const double gb = bc == ABFT_BC_CLAMP ? bot : (bc == ABFT_BC_PERIODIC ? top : g);
        s = __dadd_rn(s, dj < 0 ? __dsub_rn(gt, bot) : __dsub_rn(gb, top));
      }
      Sv[q] = s;
    } else {
      const int ys = e + dj;
      const bool yg = ghostv && (ys < 0 || ys >= ny);
      if (L.zg[d] || yg) {
        Sv[q] = __dmul_rn((double)nx, g);
        continue;
      }
      const int yr = (ys >= 0 && ys < ny) ? ys : (bc == ABFT_BC_PERIODIC ? wrap(ys, ny) : max(0, min(ys, ny - 1)));
      double s = L.prow[d][yr];
      if (di != 0) {   // beta: the x-edge columns of u^{s-1} (ledger, or the halo layer itself)
        double lft, rgt;
        if (L.exl[d]) {
          lft = (double)L.exl[d][yr];
          rgt = (double)L.exr[d][yr];
        } else {
          const T* row = L.lay[d] + (size_t)yr * p.px;
          lft = (double)row[0];
          rgt = (double)row[nx - 1];
        }
        const double gl = bc == ABFT_BC_CLAMP ? lft : (bc == ABFT_BC_PERIODIC ? rgt : g);
        const double gr = bc == ABFT_BC_CLAMP ? rgt : (bc == ABFT_BC_PERIODIC ? lft : g);
        s = __dadd_rn(s, di < 0 ? __dsub_rn(gl, rgt) : __dsub_rn(gr, lft));
      }
      Sv[q] = s;
    }
  }
  double acc = L.crow[e];
#pragma unroll
  for (int q = 0; q < NP; ++q) acc = __dadd_rn(acc, __dmul_rn(p.w[q], Sv[q]));
  return acc;
}

// Eq. 1 for the one cell (z, y, x) of u^s from u^{s-1} (p.uprev), with the
// ghosts of the boundary condition: the same canonical FMA chain as K1
// (points in order, then the sources).  correction_form 2.
template <typename T, bool CG = false>
__device__ T cell_update(const CheckParams& p, int z, int y, int x, const void* in = nullptr) {
  const T* up = reinterpret_cast<const T*>(in ? in : p.uprev);
  const int nx = p.nx, ny = p.ny, zc = p.zc, bc = p.bc;
  const T g = bc == ABFT_BC_CONSTANT ? (T)p.g : T(0);
  T acc = T(0);
  for (int q = 0; q < p.npoints; ++q) {
    const int zz = z + p.dk[q], yy = y + p.dj[q], xx = x + p.di[q];
    T v;
    const bool yo = yy < 0 || yy >= ny, xo = xx < 0 || xx >= nx;
    if (zghost(zz, zc, p.has_lo, p.has_hi, bc) ||
        ((bc == ABFT_BC_ZERO || bc == ABFT_BC_CONSTANT) && (yo || xo))) {
      v = g;
    } else {
      const int bl = zmap(zz, zc, p.has_lo, p.has_hi, bc);
      const int yr = !yo ? yy : (bc == ABFT_BC_PERIODIC ? wrap(yy, ny) : max(0, min(yy, ny - 1)));
      const int xr = !xo ? xx : (bc == ABFT_BC_PERIODIC ? wrap(xx, nx) : max(0, min(xx, nx - 1)));
      const T* a = up + (size_t)bl * p.plane + (size_t)yr * p.px + xr;
      v = CG ? __ldcg(a) : *a;
    }
    const T w = (T)p.w[q];
    acc = (q == 0) ? mul_rn(w, v) : fma_rn(w, v, acc);
  }
  for (int q = 0; q < p.nsources; ++q) {
    const T sv = q == p.field_src
                     ? reinterpret_cast<const T*>(p.src)[(size_t)z * p.splane + (size_t)y * p.spx + x]
                     : (T)p.scalar[q];
    acc = fma_rn((T)p.coef[q], sv, acc);
  }
  return acc;
}

__device__ __forceinline__ bool same_bits(float a, float b) { return __float_as_uint(a) == __float_as_uint(b); }
__device__ __forceinline__ bool same_bits(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

// ---------------------------------------------------------------- pipelined
// Pipelined online schedule ("K2/K3 beside the next sweep"):
// the checks of sweep s run while K1 of sweep s + 1 already reads u^s, so a
// cell the checks rewrite may have been read before or after its repair.
// Every rewrite is listed here; the CTA that finishes the check then waits for
// that K1 and recomputes the cells of u^{s+1} whose stencil reads a rewritten
// cell (fix_next), so u^{s+1} and its checksums end bitwise as if the checks
// had run first -- the paper's order (fig.abft caption).
__device__ __forceinline__ void note_change(const CheckParams& p, int z, int y, int x) {
  if (!p.fix) return;
  const int i = atomicAdd(&p.st->nchg, 1);
  if (i < kChgCap) { p.st->chg[i][0] = z; p.st->chg[i][1] = y; p.st->chg[i][2] = x; }
  atomicMax(&p.st->chg_zlo, 0x7fffffff - z);
  atomicMax(&p.st->chg_zhi, z + 1);
}

// candidate d (0..26: offsets in {-1,0,1}^3) of rewritten cell c: the cell of
// u^{s+1} at c + offset (periodic: wrapped; else outside -> false)
__device__ __forceinline__ bool fix_cand(const CheckParams& p, const int* c, int d, int* o) {
  const int off[3] = {d / 9 - 1, (d / 3) % 3 - 1, d % 3 - 1};
  const int n[3] = {p.zc, p.ny, p.nx};
  const bool per = p.bc == ABFT_BC_PERIODIC;
  for (int a = 0; a < 3; ++a) {
    int v = c[a] + off[a];
    if (v < 0 || v >= n[a]) {
      if (!per || (a == 0 && (p.has_lo || p.has_hi))) return false;
      v = wrap(v, n[a]);
    }
    o[a] = v;
  }
  return true;
}
__device__ __forceinline__ bool near1(int a, int b, int n, bool per) {
  const int d = abs(a - b);
  return d <= 1 || (per && n - d <= 1);
}

// u^{s+1} at (z, y, x) recomputed from the repaired u^s (Eq. 1, the sweep's
// FMA chain) with sweep s + 1's scheduled flips re-applied; stored and
// the ledger patched if it differs.  Returns whether it changed.
template <typename T>
__device__ __forceinline__ bool fix_cell(const CheckParams& p, int z, int y, int x) {
  T v = cell_update<T, true>(p, z, y, x, p.ucur);
  for (int f = 0; f < p.nfn; ++f)
    if (p.fn[f].z == z && p.fn[f].y == y && p.fn[f].x == x) v = flip_bit(v, p.fn[f].bit);
  T* cell = reinterpret_cast<T*>(p.unext) + (size_t)(z + 1) * p.plane + (size_t)y * p.px + x;
  if (same_bits(v, __ldcg(cell))) return false;
  *cell = v;
  if (p.EXnext) {
    T* ex = reinterpret_cast<T*>(p.EXnext);
    if (x == 0) ex[(size_t)(z + 1) * p.ny + y] = v;
    if (x == p.nx - 1) ex[(size_t)(p.zc + 2) * p.ny + (size_t)(z + 1) * p.ny + y] = v;
  }
  return true;
}
// b^{s+1}[z][y] (and a^{s+1}[z][x]) re-summed from the fixed field: a sum over
// values that now include no corrupted one is exact for fp32 data, so it
// equals the atomic accumulation K1 would have made
template <typename T>
__device__ __forceinline__ void fix_row(const CheckParams& p, int z, int y) {
  const T* row = reinterpret_cast<const T*>(p.unext) + (size_t)(z + 1) * p.plane + (size_t)y * p.px;
  double b = 0.0;
  for (int x = 0; x < p.nx; ++x) b += (double)__ldcg(row + x);
  p.Bnext[(size_t)(z + 1) * p.ny + y] = b;
}
template <typename T>
__device__ __forceinline__ void fix_col(const CheckParams& p, int z, int x) {
  const T* col = reinterpret_cast<const T*>(p.unext) + (size_t)(z + 1) * p.plane + x;
  double a = 0.0;
  for (int y = 0; y < p.ny; ++y) a += (double)__ldcg(col + (size_t)y * p.px);
  p.Anext[(size_t)(z + 1) * p.nx + x] = a;
}

// Run by every thread of the one CTA that finishes a pipelined check.
template <typename T>
__device__ __noinline__ void fix_next(const CheckParams& p) {
  __shared__ int s_n, s_ok;
  __shared__ unsigned s_chg[(kChgCap * 27 + 31) / 32];
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_n = *(volatile int*)&p.st->nchg;
    s_ok = 1;
    if (s_n > 0 && p.fix) {   // wait for K1 of s + 1 (launched before this check could finish)
      unsigned long long t0, t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while (*(volatile unsigned*)&p.st->k1_cnt[(p.sweep + 1) & 1] < p.k1_target) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 4000000000ull) { s_ok = 0; break; }
        __nanosleep(256);
      }
      __threadfence();
    }
  }
  for (int i = tid; i < (kChgCap * 27 + 31) / 32; i += blockDim.x) s_chg[i] = 0u;
  __syncthreads();
  const int n = s_n;
  if (n == 0) return;
  const bool per = p.bc == ABFT_BC_PERIODIC;
  if (!s_ok || !p.fix) {
    if (tid == 0 && !s_ok) atomicMax(&p.st->worst, 3);   // K1 never finished: state unknown
  } else if (n <= kChgCap) {
    // the unique candidates: (i, d) is skipped when an earlier rewritten cell's
    // neighbourhood or an earlier offset of the same cell reaches the same cell
    const int m = n * 27;
    for (int k = tid; k < m; k += blockDim.x) {
      const int i = k / 27, d = k % 27;
      const int* c = p.st->chg[i];
      int o[3];
      if (!fix_cand(p, c, d, o)) continue;
      bool dup = false;
      for (int j = 0; j < i && !dup; ++j)
        dup = near1(o[0], p.st->chg[j][0], p.zc, per) && near1(o[1], p.st->chg[j][1], p.ny, per) &&
              near1(o[2], p.st->chg[j][2], p.nx, per);
      for (int e = 0; e < d && !dup; ++e) {
        int q[3];
        dup = fix_cand(p, c, e, q) && q[0] == o[0] && q[1] == o[1] && q[2] == o[2];
      }
      if (!dup && fix_cell<T>(p, o[0], o[1], o[2])) atomicOr(&s_chg[k / 32], 1u << (k % 32));
    }
    __syncthreads();
    __threadfence_block();
    // each row / column holding a changed cell, re-summed once (by its first changed candidate)
    for (int k = tid; k < m; k += blockDim.x) {
      if (!((s_chg[k / 32] >> (k % 32)) & 1u)) continue;
      int o[3];
      fix_cand(p, p.st->chg[k / 27], k % 27, o);
      bool row_first = true, col_first = true;
      for (int j = 0; j < k && (row_first || col_first); ++j) {
        if (!((s_chg[j / 32] >> (j % 32)) & 1u)) continue;
        int q[3];
        fix_cand(p, p.st->chg[j / 27], j % 27, q);
        if (q[0] == o[0] && q[1] == o[1]) row_first = false;
        if (q[0] == o[0] && q[2] == o[2]) col_first = false;
      }
      if (row_first) fix_row<T>(p, o[0], o[1]);
      if (col_first && p.Anext) fix_col<T>(p, o[0], o[2]);
    }
  } else {
    // many rewrites (a layer recompute, Q27): every cell of the layers within
    // one of a rewritten layer, then all their rows and columns.  Rare, slow.
    const int zlo = 0x7fffffff - *(volatile int*)&p.st->chg_zlo, zhi = *(volatile int*)&p.st->chg_zhi - 1;
    auto member = [&](int z) {
      if (z >= zlo - 1 && z <= zhi + 1) return true;
      if (!per || p.has_lo || p.has_hi) return false;
      return (zlo == 0 && z == p.zc - 1) || (zhi == p.zc - 1 && z == 0);
    };
    const int64_t lay = (int64_t)p.ny * p.nx;
    for (int z = 0; z < p.zc; ++z) {
      if (!member(z)) continue;
      for (int64_t e = tid; e < lay; e += blockDim.x) fix_cell<T>(p, z, (int)(e / p.nx), (int)(e % p.nx));
    }
    __syncthreads();
    __threadfence_block();
    for (int z = 0; z < p.zc; ++z) {
      if (!member(z)) continue;
      for (int y = tid; y < p.ny; y += blockDim.x) fix_row<T>(p, z, y);
      if (p.Anext)
        for (int x = tid; x < p.nx; x += blockDim.x) fix_col<T>(p, z, x);
    }
  }
  __syncthreads();
  if (tid == 0) { p.st->nchg = 0; p.st->chg_zlo = 0; p.st->chg_zhi = 0; }
}

// correction_form 2 when the flags of layer z do not intersect in one cell
// (Q27; locality): every cell of the layer is
// recomputed from the intact u^{s-1} (Eq. 1, the sweep's own FMA chain, so an
// intact cell reproduces its stored bits), the differing cells are rewritten
// and recorded, then a[z] (one thread per column) and b[z] (one thread per
// row) are re-summed from the repaired layer in ascending index order.  Rare
// (a detection that Eq. 8 cannot resolve), so one CTA does the layer.
template <typename T>
__device__ __noinline__ void recompute_layer(const CheckParams& p, int z, abft_record r) {
  __shared__ int s_changed;
  const int tid = threadIdx.x, bz = z + 1, nx = p.nx, ny = p.ny, zc = p.zc;
  T* lay = reinterpret_cast<T*>(p.ucur) + (size_t)bz * p.plane;
  if (tid == 0) s_changed = 0;
  __syncthreads();
  for (int x = tid; x < nx; x += kCheckThreads) {
    double a = 0.0;
    for (int y = 0; y < ny; ++y) {
      T* cell = lay + (size_t)y * p.px + x;
      const T v = cell_update<T>(p, z, y, x), uo = *cell;
      if (!same_bits(v, uo)) {
        *cell = v;
        note_change(p, z, y, x);
        for (int f = 0; f < 2; ++f)   // fused halo: the neighbour's copy
          if (z == (f == 0 ? 0 : zc - 1) && p.peerU[f])
            reinterpret_cast<T*>(p.peerU[f])[(size_t)y * p.px + x] = v;
        if (p.EXc) {
          T* exc = reinterpret_cast<T*>(p.EXc);
          if (x == 0) exc[(size_t)bz * ny + y] = v;
          if (x == nx - 1) exc[(size_t)(zc + 2) * ny + (size_t)bz * ny + y] = v;
        }
        abft_record rc = r;
        rc.y = y; rc.x = x;
        rc.observed = (double)uo; rc.corrected = (double)v;
        rc.status = ABFT_REC_RECOMPUTED;
        push_record(p.st, rc);
        bump(p.st, ST_LOCATED); bump(p.st, ST_CORRECTED);
        atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->ncorr), 1ull);
        atomicAdd(&s_changed, 1);
      }
      a += (double)v;
    }
    p.Ac[(size_t)bz * nx + x] = a;
    for (int f = 0; f < 2; ++f)
      if (z == (f == 0 ? 0 : zc - 1) && p.fwdA[f]) p.fwdA[f][x] = a;
  }
  __syncthreads();   // the repaired layer is in place
  for (int y = tid; y < ny; y += kCheckThreads) {
    const T* row = lay + (size_t)y * p.px;
    double b = 0.0;
    for (int x = 0; x < nx; ++x) b += (double)row[x];
    p.Bc[(size_t)bz * ny + y] = b;
    for (int f = 0; f < 2; ++f)
      if (z == (f == 0 ? 0 : zc - 1) && p.fwdB[f]) p.fwdB[f][y] = b;
  }
  if (tid == 0) {
    bump(p.st, ST_DETECT);
    if (s_changed == 0) {
      r.status = ABFT_REC_VERIFIED;
      push_record(p.st, r);
    }
  }
}

// Steps (4)-(5) for layer z once its compare is complete (na / nb flagged
// entries, x0 / y0 the first flagged index, pa / pb their predictions); run by
// every thread of one CTA of kCheckThreads threads (block-uniform arguments).
template <typename T>
__device__ __forceinline__ void finish_layer(const CheckParams& p, int z, int na, int nb, int x0,
                                             int y0, double pa, double pb, double* red) {
  const int tid = threadIdx.x, bz = z + 1, nx = p.nx, ny = p.ny, zc = p.zc;
  if ((na | nb) == 0) return;
  abft_record r;
  r.sweep = p.sweep + *(volatile int*)&p.st->sweep_off; r.z = p.z_begin + z; r.y = y0; r.x = x0;
  r.observed = 0.0; r.corrected = 0.0; r.vx = 0.0; r.vy = 0.0;
  r.nflag_a = na; r.nflag_b = nb; r.pad = 0;
  if (p.flags & CK_OFFLINE_END) {
    if (tid == 0) {
      r.status = (p.flags & CK_PERSIST) ? ABFT_REC_PERSISTENT : ABFT_REC_WINDOW_DIRTY;
      push_record(p.st, r);
      bump(p.st, ST_DETECT);
      atomicAdd(&p.st->dirty, 1);
      // the flagged layers' extent (partial re-execution, Q28)
      atomicMax(&p.st->zext[0], (int)(0x7fffffffLL - r.z));
      atomicMax(&p.st->zext[1], (int)(r.z + 1));
      p.zflag[r.z] = 1;
    }
    return;
  }
  if (!(p.flags & CK_CORRECT)) return;
  if (na == 1 && nb == 1) {
    // ---- locate and correct (Eq. 8, fig.correction)
    T* lay = reinterpret_cast<T*>(p.ucur) + (size_t)bz * p.plane;
    double sx = 0.0, sy = 0.0;
    if (p.form != 1) {   // (a - u) as the sum of the other cells (Q11)
      for (int y = tid; y < ny; y += kCheckThreads)
        if (y != y0) sx += (double)lay[(size_t)y * p.px + x0];
      for (int x = tid; x < nx; x += kCheckThreads)
        if (x != x0) sy += (double)lay[(size_t)y0 * p.px + x];
    }
    sx = block_sum<kCheckThreads>(sx, red);
    sy = block_sum<kCheckThreads>(sy, red);
    if (tid == 0) {
      T* cell = lay + (size_t)y0 * p.px + x0;
      const double uo = (double)*cell;
      double* ax = &p.Ac[(size_t)bz * nx + x0];
      double* by = &p.Bc[(size_t)bz * ny + y0];
      double vx, vy;
      T cor;
      if (p.form != 1) {
        vx = pa - sx;
        vy = pb - sy;
        // form 2: stencil locality -- u^{s-1} is intact,
        // the located cell is recomputed with Eq. 1, exactly
        cor = p.form == 2 ? cell_update<T>(p, z, y0, x0) : (T)((vx + vy) / 2.0);
        *ax = sx + (double)cor;   // exact repair (Q12)
        *by = sy + (double)cor;
      } else {                    // literal listing
        vx = pa - (*ax - uo);
        vy = pb - (*by - uo);
        cor = (T)((vx + vy) / 2.0);
        *ax += (double)cor - uo;
        *by += (double)cor - uo;
      }
      *cell = cor;
      note_change(p, z, y0, x0);
      for (int f = 0; f < 2; ++f) {   // fused halo: the neighbours' copies
        if (z != (f == 0 ? 0 : zc - 1)) continue;
        if (p.peerU[f]) reinterpret_cast<T*>(p.peerU[f])[(size_t)y0 * p.px + x0] = cor;
        if (p.fwdA[f]) p.fwdA[f][x0] = *ax;
        if (p.fwdB[f]) p.fwdB[f][y0] = *by;
      }
      if (p.EXc) {   // keep the edge ledger of u^s in step with the field
        T* exc = reinterpret_cast<T*>(p.EXc);
        if (x0 == 0) exc[(size_t)bz * ny + y0] = cor;
        if (x0 == nx - 1) exc[(size_t)(zc + 2) * ny + (size_t)bz * ny + y0] = cor;
      }
      r.observed = uo; r.corrected = (double)cor; r.vx = vx; r.vy = vy;
      r.status = ABFT_REC_CORRECTED;
      push_record(p.st, r);
      bump(p.st, ST_DETECT); bump(p.st, ST_LOCATED); bump(p.st, ST_CORRECTED);
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->ncorr), 1ull);
    }
  } else if (p.form == 2) {
    recompute_layer<T>(p, z, r);
  } else if (tid == 0) {
    r.status = (na == 0 || nb == 0) ? ABFT_REC_UNLOCATED : ABFT_REC_UNCORRECTABLE;
    push_record(p.st, r);
    bump(p.st, ST_DETECT);
    bump(p.st, r.status == ABFT_REC_UNLOCATED ? ST_UNLOCATED : ST_UNCORR);
    atomicMax(&p.st->worst, 1);
  }
}

// K2.  One CTA per z-layer (grid = zc): every thread predicts / compares
// KU entries of a' and b' per round with all their loads in flight; the
// layer's flags meet in shared memory, so the same CTA then locates, corrects
// and records (Eq. 8, fig.correction) -- no cross-CTA handshake.
#ifndef ABFT_KU
#define ABFT_KU 4
#endif
constexpr int kCheckUnroll = ABFT_KU;
// entries per thread in flight: the K2 round is memory-latency bound, so
// few-point shapes take more entries per round; the 27-point prediction keeps
// 27 terms per entry live and takes fewer (registers, occupancy)
#ifndef ABFT_KU_FEW
#define ABFT_KU_FEW 4
#endif
#ifndef ABFT_KU_MANY
#define ABFT_KU_MANY 1
#endif
template <int S> constexpr int check_unroll() {
  return (S == SHAPE_BOX27 || S == SHAPE_GENERIC) ? ABFT_KU_MANY : ABFT_KU_FEW;
}

// one vector (a' over x if A, else b' over y) of layer z: predict, store the
// prediction (offline P / explicit check), compare with the actual checksum,
// clear the generation of sweep s + 2; flags meet in shared memory.
template <typename T, int S, bool A, bool BCG>
__device__ __forceinline__ void check_vec(const CheckParams& p, int z, int* s_n, int* s_k, double* s_pred,
                                          int part = 0, int nparts = 1) {
  const int nn = A ? p.nx : p.ny, bz = z + 1;
  const int lo = (int)((int64_t)nn * part / nparts), n = (int)((int64_t)nn * (part + 1) / nparts);
  const double* act = A ? p.Ac : p.Bc;
  double* pout = A ? p.PAo : p.PBo;
  double* zero = A ? p.zA : p.zB;
  const bool cmp = p.flags & CK_COMPARE;
  // fused halo: this layer's rows the neighbours need (predictions when they
  // are stored, else the actual checksums)
  double* fwd0 = z == 0 ? (A ? p.fwdA[0] : p.fwdB[0]) : nullptr;
  double* fwd1 = z == p.zc - 1 ? (A ? p.fwdA[1] : p.fwdB[1]) : nullptr;
  const bool fwd_pred = p.flags & CK_STORE_PRED;
  constexpr int KU = check_unroll<S>();
  constexpr bool GEN = S == SHAPE_GENERIC;
  const PredLayer<T, A> PL = pred_layer<T, A, BCG>(p, z);   // (unused by the generic list)
  (void)PL;
  for (int e0 = lo + threadIdx.x; e0 < n; e0 += kCheckThreads * KU) {
    double pr[KU], ac[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int e = e0 + u * kCheckThreads;
      const bool in = e < n;
      if constexpr (GEN) pr[u] = in ? predict_entry<T, S, A, BCG>(p, z, e) : 0.0;
      else pr[u] = in ? predict_entry_l<T, (GEN ? SHAPE_HOTSPOT7 : S), A, BCG>(p, PL, e) : 0.0;
      ac[u] = (in && cmp) ? act[(size_t)bz * nn + e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int e = e0 + u * kCheckThreads;
      if (e >= n) break;
      if (p.flags & CK_STORE_PRED) pout[(size_t)bz * nn + e] = pr[u];
      if (cmp && flag_rel(pr[u], ac[u], p.eps)) {
        atomicAdd(s_n, 1);
        atomicMax(s_k, 0x7fffffff - e);
        *s_pred = pr[u];
      }
      if (zero) zero[(size_t)bz * nn + e] = 0.0;
      if (fwd0 || fwd1) {
        const double v = fwd_pred ? pr[u] : act[(size_t)bz * nn + e];
        if (fwd0) fwd0[e] = v;
        if (fwd1) fwd1[e] = v;
      }
    }
  }
}
template <typename T, int S, bool BCG>
__device__ __forceinline__ void k2_layer(const CheckParams& p) {
  const int z = p.zr0 + blockIdx.x, bz = z + 1;
  const int tid = threadIdx.x, part = blockIdx.y, nparts = gridDim.y;
  LayerSummary* L = &p.summ[z];
  __shared__ int s_na, s_nb, s_xk, s_yk, s_last;
  __shared__ double s_pa, s_pb;
  __shared__ double red[kCheckThreads / 32];
  int na, nb, xk, yk;
  double pa, pb;
  (void)bz;
  grid_dependency_wait();   // K1's checksums and field (PDL)
  if (p.k1_reset && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) p.st->k1_cnt[p.sweep & 1] = 0u;
  if (!(p.flags & CK_FROM_SUMMARY)) {
    if (tid == 0) { s_na = 0; s_nb = 0; s_xk = 0; s_yk = 0; s_pa = 0.0; s_pb = 0.0; }
    __syncthreads();
    // a' (entries x) then b' (entries y): no divergent entry kinds inside a
    // round, so the loads of all kCheckUnroll entries are in flight together.
    // Lazy policy: b' only; a is computed by K3 for the
    // layers whose b flags.  nparts > 1 (few layers): this CTA's share.
    // Offline under LAZY (CK_BONLY, Q29): b' only, and no K3 -- a window
    // is rolled back, never corrected, so a is never needed.
    if (!(p.flags & (CK_LAZY | CK_BONLY))) check_vec<T, S, true, BCG>(p, z, &s_na, &s_xk, &s_pa, part, nparts);
    check_vec<T, S, false, BCG>(p, z, &s_nb, &s_yk, &s_pb, part, nparts);
    if (!(p.flags & CK_COMPARE)) return;
    __syncthreads();
    if (nparts > 1) {
      // merge this share into the layer summary; the CTA that completes the
      // layer continues with the layer's totals
      if (tid == 0) {
        if (s_na) { atomicAdd(&L->na, s_na); atomicMax(&L->xk, s_xk); L->pa = s_pa; }
        if (s_nb) { atomicAdd(&L->nb, s_nb); atomicMax(&L->yk, s_yk); L->pb = s_pb; }
        __threadfence();
        s_last = atomicAdd(&L->cnt2, 1) == nparts - 1;
      }
      __syncthreads();
      if (!s_last) return;
      __threadfence();
      na = *(volatile int*)&L->na; nb = *(volatile int*)&L->nb;
      xk = *(volatile int*)&L->xk; yk = *(volatile int*)&L->yk;
      pa = *(volatile double*)&L->pa; pb = *(volatile double*)&L->pb;
      __syncthreads();
      if (tid == 0) {
        L->cnt2 = 0;
        if (!(p.flags & (CK_LAZY | CK_SUMMARY))) { L->na = 0; L->nb = 0; L->xk = 0; L->yk = 0; }
        if (p.flags & CK_LAZY) { L->na = 0; L->xk = 0; }
      }
    } else {
      na = s_na; nb = s_nb; xk = s_xk; yk = s_yk; pa = s_pa; pb = s_pb;
    }
    if (p.flags & CK_LAZY) {      // hand the flagged layer to K3
      if (nb) {
        // the rows of a this layer's check reads: a^{s-1} of zeta(z-1), z,
        // zeta(z+1) and a^s of z -- each marked once (a neighbour layer may
        // need the same row), zeroed for K3's partial sums, listed
        __shared__ int s_new[4], s_row[4];
        if (tid == 0) {
          L->nb = nb; L->yk = yk; L->pb = pb;
          p.lazy_list[atomicAdd(&p.st->lazy_n[p.sweep & 1], 1)] = z;
          for (int k = 0; k < 4; ++k) {
            const int sel = k == 3, bl = sel ? z + 1 : zmap(z + k - 1, p.zc, p.has_lo, p.has_hi, p.bc);
            s_row[k] = (sel << 30) | bl;
            s_new[k] = atomicCAS(&p.lazy_mark[sel * (p.zc + 2) + bl], 0, 1) == 0;
            if (s_new[k]) p.lazy_rowlist[atomicAdd(&p.st->lazy_rows[p.sweep & 1], 1)] = s_row[k];
          }
        }
        __syncthreads();
        for (int k = 0; k < 4; ++k) {
          if (!s_new[k]) continue;
          double* row = ((s_row[k] >> 30) ? p.Ac : p.Aw) + (size_t)(s_row[k] & 0x3fffffff) * p.nx;
          for (int x = tid; x < p.nx; x += kCheckThreads) row[x] = 0.0;
        }
      }
      return;
    }
    if (p.flags & CK_SUMMARY) {   // explicit check(): keep the summary for correct()
      if (tid == 0) {
        L->na = na; L->nb = nb; L->xk = xk; L->yk = yk; L->pa = pa; L->pb = pb;
        if (na) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->flag_a), (unsigned long long)na);
        if (nb) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->flag_b), (unsigned long long)nb);
      }
      return;
    }
  } else {
    na = L->na; nb = L->nb; xk = L->xk; yk = L->yk; pa = L->pa; pb = L->pb;
    __syncthreads();
    if (tid == 0) { L->na = 0; L->nb = 0; L->xk = 0; L->yk = 0; }
  }
  const int x0 = na ? 0x7fffffff - xk : -1;
  const int y0 = nb ? 0x7fffffff - yk : -1;
  finish_layer<T>(p, z, na, nb, x0, y0, pa, pb, red);
}
template <typename T, int S, bool BCG>
__global__ void __launch_bounds__(kCheckThreads) k2_check(const __grid_constant__ CheckParams p) {
  k2_layer<T, S, BCG>(p);
  if (p.fix && !(p.flags & CK_LAZY)) {
    // pipelined schedule, policy BOTH: the CTA that finishes K2 last repairs
    // u^{s+1} where K1 of s + 1 read a cell this check rewrote
    __shared__ int s_fin;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_fin = atomicAdd(&p.st->k2_done, 1) == (int)(gridDim.x * gridDim.y) - 1;
    __syncthreads();
    if (s_fin) {
      __threadfence();
      fix_next<T>(p);
      if (threadIdx.x == 0) p.st->k2_done = 0;
    }
  }
}

// K3 (lazy checksum policy): for the layers whose b flagged in K2, the
// second checksum vector "only in case of error, to enable correction"
// (P:271-273): a^{s-1} of the layers the prediction reads
// (zeta(z-1), z, zeta(z+1): column sums of u^{s-1}, halo layers included) and
// a^s of z (of u^s).  K2 marked each needed row once, zeroed it and listed it;
// here every CTA (x-tile, row chunk) adds its chunk's column partials into the
// listed rows (fp64 RED: exact for fp32 data, like the z-march), and the CTA
// that finishes last predicts a' (Theorem 1), compares, locates and corrects
// each flagged layer as K2 does for policy BOTH, then clears the marks.
// Exits at once when no layer flagged.  Lists alternate by sweep parity: K3 of
// sweep s clears the counts of sweep s + 1 before K2 of s + 1 appends.
template <typename T, int S, bool BCG>
__global__ void __launch_bounds__(kCheckThreads) k3_lazy(const __grid_constant__ CheckParams p) {
  __shared__ int s_na, s_xk, s_last;
  __shared__ double s_pa;
  __shared__ double red[kCheckThreads / 32];
  const int tid = threadIdx.x, nx = p.nx, ny = p.ny, zc = p.zc;
  grid_dependency_wait();   // K2's lists (PDL)
  const int par = p.sweep & 1;
  const int n = *(volatile int*)&p.st->lazy_n[par];
  const int nrows = *(volatile int*)&p.st->lazy_rows[par];
  // the next sweep's K2 counts into the other slot: clear it (nobody reads it now)
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
    p.st->lazy_n[par ^ 1] = 0;
    p.st->lazy_rows[par ^ 1] = 0;
  }
  if (n == 0) return;
  // ---- column partials of this CTA's x-tile and row chunk, every listed row
  const int x = blockIdx.x * kCheckThreads + tid;
  const int chunk = (ny + gridDim.y - 1) / gridDim.y;
  const int y0c = blockIdx.y * chunk, y1c = min(ny, y0c + chunk);
  if (x < nx) {
    // four listed rows at a time, their 4 x 8 loads in flight together (one
    // flagged layer lists four rows: one memory round trip per 8 rows of the
    // chunk instead of four); each row's partial still adds in ascending y
    constexpr int NR = 4;
    for (int i0 = 0; i0 < nrows; i0 += NR) {
      const int m = min(NR, nrows - i0);
      const T* col[NR];
      double* dst[NR];
      double part[NR];
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const int e = p.lazy_rowlist[i0 + (j < m ? j : 0)];   // j >= m: a harmless repeat
        const int sel = e >> 30, bl = e & 0x3fffffff;   // sel 0: a^{s-1} (u^{s-1}), 1: a^s (u^s)
        col[j] = reinterpret_cast<const T*>(sel ? p.ucur : p.uprev) + (size_t)bl * p.plane + x;
        dst[j] = (sel ? p.Ac : p.Aw) + (size_t)bl * nx + x;
        part[j] = 0.0;
      }
      int y = y0c;
      for (; y + 8 <= y1c; y += 8) {
        T v[NR][8];
#pragma unroll
        for (int j = 0; j < NR; ++j)
#pragma unroll
          for (int k = 0; k < 8; ++k) v[j][k] = col[j][(size_t)(y + k) * p.px];
#pragma unroll
        for (int j = 0; j < NR; ++j)
#pragma unroll
          for (int k = 0; k < 8; ++k) part[j] += (double)v[j][k];
      }
      for (; y < y1c; ++y) {
#pragma unroll
        for (int j = 0; j < NR; ++j) part[j] += (double)col[j][(size_t)y * p.px];
      }
      if (y1c > y0c) {
#pragma unroll
        for (int j = 0; j < NR; ++j)
          if (j < m) atomicAdd(dst[j], part[j]);
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&p.st->lazy_done, 1) == (int)(gridDim.x * gridDim.y) - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // ---- the last CTA: steps (2)-(5) for a of every flagged layer
  for (int i = 0; i < n; ++i) {
    const int z = p.lazy_list[i];
    LayerSummary* L = &p.summ[z];
    if (tid == 0) { s_na = 0; s_xk = 0; s_pa = 0.0; }
    __syncthreads();
    CheckParams q = p;
    q.flags = CK_COMPARE;
    q.Ap = p.Aw;
    q.PAo = nullptr;
    q.zA = nullptr;
    check_vec<T, S, true, BCG>(q, z, &s_na, &s_xk, &s_pa);
    __syncthreads();
    const int na = s_na, nb = L->nb;
    const int x0 = na ? 0x7fffffff - s_xk : -1, y0 = 0x7fffffff - L->yk;
    const double pa = s_pa, pb = L->pb;
    __syncthreads();
    if (tid == 0) { L->nb = 0; L->yk = 0; }
    finish_layer<T>(p, z, na, nb, x0, y0, pa, pb, red);
    __syncthreads();
  }
  for (int i = tid; i < nrows; i += kCheckThreads) {   // marks of this sweep's rows
    const int e = p.lazy_rowlist[i];
    p.lazy_mark[(e >> 30) * (zc + 2) + (e & 0x3fffffff)] = 0;
  }
  if (tid == 0) p.st->lazy_done = 0;
  if (p.fix) fix_next<T>(p);   // pipelined schedule (see fix_next)
}

// ---------------------------------------------------------------- K0
// Initial checksums a^0, b^0 of the trusted input (Eqs. 2-3) and c_x, c_y of
// the constant term (Theorem 1, "pre-computed" P:392).  Each sum is
// taken sequentially in ascending index order by one thread -- the
// definition's order, so sums of fp64 terms (c_x, c_y; fp64 data) are
// reproducible bitwise -- with many loads in flight ahead of the dependent
// additions: 8 rows per column thread (k0_colsum); rows staged through shared
// memory for the row sums (k0_rowsum).
struct FieldVal {   // u of field buffer layer z (layer pitch `plane`, halo offset 1)
  const void* u;
  int64_t px, plane;
  int dtype;
  __device__ __forceinline__ const char* row(int z, int y) const {
    return static_cast<const char*>(u) + ((size_t)(z + 1) * plane + (size_t)y * px) * (dtype == ABFT_F32 ? 4 : 8);
  }
};
struct ConstVal {   // C_{x,y} = sum_q coef_q * src_q (fp64, dtype-rounded operands)
  const void* field;
  int64_t fpx, fplane;
  int dtype, nsources, field_src;
  double coef[kMaxSources], scalar[kMaxSources];
  __device__ __forceinline__ const char* row(int z, int y) const {
    return field ? static_cast<const char*>(field) + ((size_t)z * fplane + (size_t)y * fpx) * (dtype == ABFT_F32 ? 4 : 8)
                 : nullptr;
  }
};
// ConstVal's per-cell sum, the same operations in the same order as
//   s = t_0; s = s + t_q (q = 1 ..), t_q = coef_q * (q == field_src ? P : scalar_q)
// with every term that does not read the field (and the partial sum before
// the field term) evaluated once per thread instead of once per cell; NPOST =
// constant terms after the field term (HotSpot: 1).
template <int NPOST> struct ConstEval {
  double pre, cf, post[NPOST > 0 ? NPOST : 1], all;
  int fs;
  __device__ __forceinline__ explicit ConstEval(const ConstVal& c) {
    // compile-time indices only (a runtime index would put the terms on the stack)
    fs = c.field_src;
    pre = 0.0;
    cf = 0.0;
    double t[kMaxSources];
#pragma unroll
    for (int q = 0; q < kMaxSources; ++q) {
      t[q] = __dmul_rn(c.coef[q], c.scalar[q]);
      if (q < c.nsources && (fs < 0 || q < fs)) pre = (q == 0) ? t[q] : __dadd_rn(pre, t[q]);
      if (q == fs) cf = c.coef[q];
    }
#pragma unroll
    for (int j = 0; j < (NPOST > 0 ? NPOST : 1); ++j) {
      post[j] = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxSources; ++q)
        if (q == fs + 1 + j) post[j] = t[q];
    }
    all = fs < 0 ? pre : 0.0;
  }
  __device__ __forceinline__ double val(double fv, int) const {
    if (fs < 0) return all;                 // no field source: C is one constant
    const double t = __dmul_rn(cf, fv);
    double s = fs == 0 ? t : __dadd_rn(pre, t);
#pragma unroll
    for (int j = 0; j < NPOST; ++j) s = __dadd_rn(s, post[j]);
    return s;
  }
};
struct FieldEval {
  __device__ __forceinline__ explicit FieldEval(const FieldVal&) {}
  __device__ __forceinline__ double val(double v, int) const { return v; }
};
// A[z][x] = sum_y f(z, y, x); 1D grid of zc x ceil(nx / (256 V)) CTAs, a
// thread owns V consecutive columns (one 16-byte vector: V = 4 fp32, 2 fp64;
// element loads on a ragged row end); out row stride nx, layer offset `off`
template <typename F, typename E, typename T>
__global__ void __launch_bounds__(256) k0_colsum(const __grid_constant__ F f, int nx, int ny, double* A, int off) {
  const E ev(f);
  constexpr int V = 16 / (int)sizeof(T), U = 8;
  using VT = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const int64_t nxb = (nx + 256 * V - 1) / (256 * V);
  const int z = (int)(blockIdx.x / nxb), x0 = ((int)(blockIdx.x % nxb) * 256 + threadIdx.x) * V;
  if (x0 >= nx) return;
  const bool whole = x0 + V <= nx;
  double s[V];
#pragma unroll
  for (int k = 0; k < V; ++k) s[k] = 0.0;
  auto load = [&](int y, T (&v)[V]) {
    const char* row = f.row(z, y);
    if (!row) {
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = T(0);
    } else if (whole) {
      const VT w = __ldg(reinterpret_cast<const VT*>(reinterpret_cast<const T*>(row) + x0));
      const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = e[k];
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = x0 + k < nx ? __ldg(reinterpret_cast<const T*>(row) + x0 + k) : T(0);
    }
  };
  int y = 0;
  for (; y + U <= ny; y += U) {
    T v[U][V];
#pragma unroll
    for (int j = 0; j < U; ++j) load(y + j, v[j]);
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) s[k] = __dadd_rn(s[k], ev.val((double)v[j][k], x0 + k));
  }
  for (; y < ny; ++y) {
    T v[V];
    load(y, v);
#pragma unroll
    for (int k = 0; k < V; ++k) s[k] = __dadd_rn(s[k], ev.val((double)v[k], x0 + k));
  }
#pragma unroll
  for (int k = 0; k < V; ++k)
    if (x0 + k < nx) A[(size_t)(z + off) * nx + x0 + k] = s[k];
}

// B[z][y] = sum_x f(z, y, x), ascending x by the row's own lane.  A warp owns
// 32 consecutive rows and walks x in 128-byte chunks: the chunk of all 32
// rows is loaded coalesced (each load instruction: 4 rows x 128 B) one chunk
// ahead, staged through shared memory, and lane r then adds row r's elements
// in order (padded rows: no bank conflicts).  Round 1's one-row-per-thread
// reads (32 rows 4 KiB apart per warp load) ran at ~4.4 TB/s.
template <typename F, typename E, typename T>
__global__ void __launch_bounds__(256) k0_rowsum(const __grid_constant__ F f, int nx, int ny, int zc, double* B, int off) {
  constexpr int V = 16 / (int)sizeof(T), CH = 128 / (int)sizeof(T);
  using VT = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  __shared__ T tile[8][32][CH + 1];
  const E ev(f);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t rows = (int64_t)zc * ny;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + w) * 32;
  if (r0 >= rows) return;   // warp-uniform
  const int64_t my = r0 + lane;
  const bool mine = my < rows;
  // the rows whose 16-byte segment (lane & 7) this lane loads: r0 + 4 j + lane / 8
  const T* lrow[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t rr = r0 + 4 * j + (lane >> 3);
    lrow[j] = rr < rows ? reinterpret_cast<const T*>(f.row((int)(rr / ny), (int)(rr % ny))) : nullptr;
  }
  const int seg = (lane & 7) * V;
  auto load = [&](int x, VT (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (lrow[j]) v[j] = __ldg(reinterpret_cast<const VT*>(lrow[j] + x + seg));
      else v[j] = VT{};
    }
  };
  double s = 0.0;
  const int nfull = nx / CH * CH;
  VT cur[8];
  if (nfull > 0) load(0, cur);
  for (int x = 0; x < nfull; x += CH) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const T* e = reinterpret_cast<const T*>(&cur[j]);
#pragma unroll
      for (int k = 0; k < V; ++k) tile[w][4 * j + (lane >> 3)][seg + k] = e[k];
    }
    if (x + CH < nfull) load(x + CH, cur);   // next chunk in flight during the sums
    __syncwarp();
    if (mine) {
#pragma unroll 8
      for (int k = 0; k < CH; ++k) s = __dadd_rn(s, ev.val((double)tile[w][lane][k], x + k));
    }
    __syncwarp();
  }
  if (!mine) return;
  const int z = (int)(my / ny), y = (int)(my % ny);
  const T* row = reinterpret_cast<const T*>(f.row(z, y));
  for (int x = nfull; x < nx; ++x) s = __dadd_rn(s, ev.val(row ? (double)__ldg(row + x) : 0.0, x));
  B[(size_t)(z + off) * ny + y] = s;
}

}  // namespace abft
