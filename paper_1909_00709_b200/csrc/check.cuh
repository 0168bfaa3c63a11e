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

constexpr int kCheckThreads = 512;

template <typename T>
__global__ void __launch_bounds__(kCheckThreads) k2_check(const __grid_constant__ CheckParams p) {
  const int z = blockIdx.x, bz = z + 1;
  const int nx = p.nx, ny = p.ny, zc = p.zc;
  const int tid = threadIdx.x;
  __shared__ int s_na, s_nb, s_x0, s_y0;
  __shared__ double s_pa, s_pb;
  __shared__ double red[kCheckThreads / 32];
  const T* up = reinterpret_cast<const T*>(p.uprev);
  T* uc = reinterpret_cast<T*>(p.ucur);
  if (tid == 0) {
    s_na = 0; s_nb = 0; s_x0 = 0x7fffffff; s_y0 = 0x7fffffff; s_pa = 0.0; s_pb = 0.0;
    if (p.flags & CK_FROM_SUMMARY) {
      const LayerSummary L = p.summ[z];
      s_na = L.na; s_nb = L.nb; s_x0 = L.x0; s_y0 = L.y0; s_pa = L.pa; s_pb = L.pb;
    }
  }
  __syncthreads();
  if (!(p.flags & CK_FROM_SUMMARY)) {
    // ---- a'_x, Theorem 1 (Eq. 4): c_x + sum_S w (a_{x+i} + alpha_{x+i,j})
    for (int x = tid; x < nx; x += kCheckThreads) {
      double pa = p.cA[(size_t)z * nx + x];
      for (int q = 0; q < p.npoints; ++q) {
        const int zq = zmap(z + p.dk[q], zc, p.has_lo, p.has_hi);
        const int xr = max(0, min(x + p.di[q], nx - 1));
        double S = p.Ap[(size_t)zq * nx + xr];
        if (p.dj[q] != 0) {
          const T* col = up + (size_t)zq * p.plane + xr;
          const double top = (double)col[0], bot = (double)col[(size_t)(ny - 1) * p.px];
          S = __dadd_rn(S, p.dj[q] < 0 ? __dsub_rn(top, bot) : __dsub_rn(bot, top));
        }
        pa = __dadd_rn(pa, __dmul_rn(p.w[q], S));
      }
      if (p.flags & CK_STORE_PRED) p.PAo[(size_t)bz * nx + x] = pa;
      if ((p.flags & CK_COMPARE) && flag_rel(pa, p.Ac[(size_t)bz * nx + x], p.eps)) {
        atomicAdd(&s_na, 1);
        atomicMin(&s_x0, x);
        s_pa = pa;
      }
    }
    // ---- b'_y, Theorem 1 (Eq. 5): c_y + sum_S w (b_{y+j} + beta_{i,y+j})
    for (int y = tid; y < ny; y += kCheckThreads) {
      double pb = p.cB[(size_t)z * ny + y];
      for (int q = 0; q < p.npoints; ++q) {
        const int zq = zmap(z + p.dk[q], zc, p.has_lo, p.has_hi);
        const int yr = max(0, min(y + p.dj[q], ny - 1));
        double S = p.Bp[(size_t)zq * ny + yr];
        if (p.di[q] != 0) {
          const T* row = up + (size_t)zq * p.plane + (size_t)yr * p.px;
          const double lft = (double)row[0], rgt = (double)row[nx - 1];
          S = __dadd_rn(S, p.di[q] < 0 ? __dsub_rn(lft, rgt) : __dsub_rn(rgt, lft));
        }
        pb = __dadd_rn(pb, __dmul_rn(p.w[q], S));
      }
      if (p.flags & CK_STORE_PRED) p.PBo[(size_t)bz * ny + y] = pb;
      if ((p.flags & CK_COMPARE) && flag_rel(pb, p.Bc[(size_t)bz * ny + y], p.eps)) {
        atomicAdd(&s_nb, 1);
        atomicMin(&s_y0, y);
        s_pb = pb;
      }
    }
  }
  __syncthreads();
  const int na = s_na, nb = s_nb;
  if (p.flags & CK_SUMMARY) {
    if (tid == 0) {
      LayerSummary L;
      L.na = na; L.nb = nb; L.x0 = na ? s_x0 : -1; L.y0 = nb ? s_y0 : -1; L.pa = s_pa; L.pb = s_pb;
      p.summ[z] = L;
      if (na) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->flag_a), (unsigned long long)na);
      if (nb) atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->flag_b), (unsigned long long)nb);
    }
  } else if ((p.flags & (CK_COMPARE | CK_FROM_SUMMARY)) && (na | nb)) {
    abft_record r;
    r.sweep = p.sweep; r.z = p.z_begin + z;
    r.y = nb ? s_y0 : -1; r.x = na ? s_x0 : -1;
    r.observed = 0.0; r.corrected = 0.0; r.vx = 0.0; r.vy = 0.0;
    r.nflag_a = na; r.nflag_b = nb; r.pad = 0;
    if (p.flags & CK_OFFLINE_END) {
      if (tid == 0) {
        r.status = (p.flags & CK_PERSIST) ? ABFT_REC_PERSISTENT : ABFT_REC_WINDOW_DIRTY;
        push_record(p.st, r);
        bump(p.st, ST_DETECT);
        atomicAdd(&p.st->dirty, 1);
      }
    } else if (p.flags & CK_CORRECT) {
      if (na == 1 && nb == 1) {
        // ---- locate and correct (Eq. 8, fig.correction)
        const int x0 = s_x0, y0 = s_y0;
        T* lay = uc + (size_t)bz * p.plane;
        double sx = 0.0, sy = 0.0;
        if (p.form == 0) {
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
          if (p.form == 0) {
            vx = s_pa - sx;
            vy = s_pb - sy;
            cor = (T)((vx + vy) / 2.0);
            *ax = sx + (double)cor;
            *by = sy + (double)cor;
          } else {
            vx = s_pa - (*ax - uo);
            vy = s_pb - (*by - uo);
            cor = (T)((vx + vy) / 2.0);
            *ax += (double)cor - uo;
            *by += (double)cor - uo;
          }
          *cell = cor;
          r.observed = uo; r.corrected = (double)cor; r.vx = vx; r.vy = vy;
          r.status = ABFT_REC_CORRECTED;
          push_record(p.st, r);
          bump(p.st, ST_DETECT); bump(p.st, ST_LOCATED); bump(p.st, ST_CORRECTED);
          atomicAdd(reinterpret_cast<unsigned long long*>(&p.st->ncorr), 1ull);
        }
      } else if (tid == 0) {
        r.status = (na == 0 || nb == 0) ? ABFT_REC_UNLOCATED : ABFT_REC_UNCORRECTABLE;
        push_record(p.st, r);
        bump(p.st, ST_DETECT);
        bump(p.st, r.status == ABFT_REC_UNLOCATED ? ST_UNLOCATED : ST_UNCORR);
        atomicMax(&p.st->worst, 1);
      }
    }
  }
  // clear the checksum generation the next sweep accumulates into
  if (p.zA)
    for (int x = tid; x < nx; x += kCheckThreads) p.zA[(size_t)bz * nx + x] = 0.0;
  if (p.zB)
    for (int y = tid; y < ny; y += kCheckThreads) p.zB[(size_t)bz * ny + y] = 0.0;
}

// ---------------------------------------------------------------- K0
// Initial checksums a^0, b^0 of the trusted input (Eqs. 2-3) and c_x, c_y of
// the constant term (Theorem 1, "pre-computed" P:392).  Each sum is
// taken sequentially in ascending index order by one thread (coalesced
// through a shared-memory transpose for the row sums), i.e. the same order as
// the definition, so fp64-data results are reproducible.
struct FieldVal {   // u of field buffer layer z (layer pitch `plane`, halo offset 1)
  const void* u;
  int64_t px, plane;
  int dtype;
  __device__ __forceinline__ double operator()(int z, int y, int x) const {
    const size_t i = (size_t)(z + 1) * plane + (size_t)y * px + x;
    return dtype == ABFT_F32 ? (double)reinterpret_cast<const float*>(u)[i]
                             : reinterpret_cast<const double*>(u)[i];
  }
};
struct ConstVal {   // C_{x,y} = sum_q coef_q * src_q (fp64, dtype-rounded operands)
  const void* field;
  int64_t fpx, fplane;
  int dtype, nsources, field_src;
  double coef[kMaxSources], scalar[kMaxSources];
  __device__ __forceinline__ double operator()(int z, int y, int x) const {
    double s = 0.0;
    for (int q = 0; q < nsources; ++q) {
      double sv;
      if (q == field_src) {
        const size_t i = (size_t)z * fplane + (size_t)y * fpx + x;
        sv = dtype == ABFT_F32 ? (double)reinterpret_cast<const float*>(field)[i]
                               : reinterpret_cast<const double*>(field)[i];
      } else {
        sv = scalar[q];
      }
      const double t = __dmul_rn(coef[q], sv);
      s = (q == 0) ? t : __dadd_rn(s, t);
    }
    return s;
  }
};

// A[z][x] = sum_y f(z, y, x); grid (zc, ceil(nx / 256)); out row stride nx, layer offset `off`
template <typename F>
__global__ void __launch_bounds__(256) k0_colsum(F f, int nx, int ny, double* A, int off) {
  const int z = blockIdx.x, x = blockIdx.y * 256 + threadIdx.x;
  if (x >= nx) return;
  double s = 0.0;
  for (int y = 0; y < ny; ++y) s = __dadd_rn(s, f(z, y, x));
  A[(size_t)(z + off) * nx + x] = s;
}
// B[z][y] = sum_x f(z, y, x); grid (zc, ceil(ny / 128)), 128 threads, one row per thread
template <typename F>
__global__ void __launch_bounds__(128) k0_rowsum(F f, int nx, int ny, double* B, int off) {
  __shared__ double tile[128][33];
  const int z = blockIdx.x, yb = blockIdx.y * 128;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s = 0.0;
  for (int xc = 0; xc < nx; xc += 32) {
    for (int rr = warp; rr < 128; rr += 4) {
      const int y = yb + rr, x = xc + lane;
      tile[rr][lane] = (y < ny && x < nx) ? f(z, y, x) : 0.0;
    }
    __syncthreads();
    const int m = min(32, nx - xc);
    for (int c = 0; c < m; ++c) s = __dadd_rn(s, tile[threadIdx.x][c]);
    __syncthreads();
  }
  const int y = yb + threadIdx.x;
  if (y < ny) B[(size_t)(z + off) * ny + y] = s;
}

}  // namespace abft
