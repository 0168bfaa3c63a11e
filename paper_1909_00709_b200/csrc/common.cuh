// common.cuh -- shared device definitions of the B200 (sm_100a) ABFT stencil path.
// PTX wrappers for mbarrier + TMA (cp.async.bulk.tensor), the stencil shapes,
// and the parameter blocks passed from the host library to the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "abft_stencil.h"

namespace abft {

constexpr int kMaxPoints = 27;   // radius-1 stencils in 3D
constexpr int kMaxSources = 4;
constexpr int kMaxFaultsPerLaunch = 64;   // scheduled flips per sweep and slab (set_faults checks)
constexpr int kRecordCap = 4096;
constexpr int kMaxDevices = 64;          // per-device launch attributes
constexpr int kGens = 4;                 // rotating checksum generations (pipelined schedule: 4)
constexpr int kChgCap = 32;              // pipelined schedule: changed cells listed per sweep

// ------------------------------------------------------------------ shapes
// The sweep evaluates the points of S in the caller's order (the FMA chain is
// part of the numeric contract).  Shapes whose point ORDER is known at compile
// time get a register-blocked kernel; any other radius-1 list runs the generic
// kernel (runtime offsets, same arithmetic).
enum ShapeId { SHAPE_GENERIC = 0, SHAPE_FIG2_5PT = 1, SHAPE_HOTSPOT7 = 2, SHAPE_BOX27 = 3,
               SHAPE_HOTSPOT7_FS = 4 /* HotSpot points + sources [field, scalar] */ };

template <int S> struct Shape;
// fig.sweep: c, w(x-1), e(x+1), s(y+1), n(y-1)
template <> struct Shape<SHAPE_FIG2_5PT> {
  static constexpr int NP = 5;
  __host__ __device__ static constexpr int off(int p, int a) {
    constexpr int t[5][3] = {{0, 0, 0}, {-1, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, -1, 0}};
    return t[p][a];
  }
};
// HotSpot3D-like (BASELINE.json configs[1]): c, w, e, n(y-1), s(y+1), t(z+1), b(z-1)
template <> struct Shape<SHAPE_HOTSPOT7> {
  static constexpr int NP = 7;
  __host__ __device__ static constexpr int off(int p, int a) {
    constexpr int t[7][3] = {{0, 0, 0},  {-1, 0, 0}, {1, 0, 0}, {0, -1, 0},
                             {0, 1, 0},  {0, 0, 1},  {0, 0, -1}};
    return t[p][a];
  }
};
template <> struct Shape<SHAPE_HOTSPOT7_FS> : Shape<SHAPE_HOTSPOT7> {};
// 27-point box, dk outer, dj middle, di inner, ascending (BASELINE.json configs[4])
template <> struct Shape<SHAPE_BOX27> {
  static constexpr int NP = 27;
  __host__ __device__ static constexpr int off(int p, int a) {
    return a == 0 ? (p % 3) - 1 : (a == 1 ? (p / 3) % 3 - 1 : p / 9 - 1);
  }
};

// The helpers take the shape as a type (a point list seen in staged
// coordinates).
template <class SH> __host__ __device__ constexpr bool sh_needs_z() {
  for (int p = 0; p < SH::NP; ++p)
    if (SH::off(p, 2) != 0) return true;
  return false;
}
// does staged plane dk need input row offset dj (relative to an output row)?
template <class SH> __host__ __device__ constexpr bool sh_uses(int dk, int dj) {
  for (int p = 0; p < SH::NP; ++p)
    if (SH::off(p, 2) == dk && SH::off(p, 1) == dj) return true;
  return false;
}
template <class SH> __host__ __device__ constexpr bool sh_uses_x_halo(int dk) {
  for (int p = 0; p < SH::NP; ++p)
    if (SH::off(p, 2) == dk && SH::off(p, 0) != 0) return true;
  return false;
}
template <int S> __host__ __device__ constexpr bool shape_needs_z() { return sh_needs_z<Shape<S>>(); }


// K1 instantiation variants: hot path, with scheduled bit-flips, general
enum K1Variant { K1_HOT = 0, K1_INJ = 1, K1_GEN = 2 };

// which actual checksums K1 accumulates in its pass
enum K1Checksums { K1_CK_NONE = 0, K1_CK_AB = 1 /* a and b */, K1_CK_B = 2 /* b only (lazy a) */ };

// ------------------------------------------------------------ param blocks
struct LocalFault { int z, y, x, bit; };  // slab-local layer, row, column



// per-handle device state (lives in the aux workspace)
struct DevState {
  unsigned long long nrec;
  long long cnt[9];        // mirrors abft_stats order
  int worst;               // 0 / 1 / 3
  int dirty;               // offline: flagged layers in the last window check
  int zext[2];             // offline: INT_MAX - lowest and 1 + highest flagged global layer (0: none)
  long long flag_a, flag_b;  // explicit check(): flagged entries
  long long ncorr;           // explicit correct(): corrections
  int lazy_n[2];             // lazy checksum policy: layers whose b flagged, by sweep parity
  int lazy_rows[2];          // lazy policy: a rows to compute, by sweep parity
  int lazy_done;             // lazy policy: K3 CTAs finished
  // pipelined online schedule (K2/K3 of sweep s beside K1 of sweep s + 1):
  // the cells of u^s the checks rewrote (the first kChgCap of nchg), the
  // extent of their layers, K1 CTAs completed (monotonic), K2 CTAs done
  int nchg, chg_zlo, chg_zhi, k2_done;
  unsigned k1_cnt[2];        // K1 CTAs finished, by sweep parity (K2 of that sweep resets it)
  int sweep_off;             // added to the recorded sweep (a cached graph replayed later)
  int pad_;
  int chg[kChgCap][3];       // (z, y, x), slab-local
  abft_record rec[kRecordCap];
};
enum { ST_SWEEPS = 0, ST_DETECT, ST_LOCATED, ST_CORRECTED, ST_UNLOCATED, ST_UNCORR,
       ST_ROLLBACKS, ST_WINDOWS, ST_PERSIST };

// per-layer summary written by check() and consumed by correct()
// Written by an explicit check(), consumed and reset by correct().
struct LayerSummary {
  int na, nb;      // flagged entries of a (over x) and b (over y)
  int xk, yk;      // max of (INT_MAX - index) over flagged entries: the first flagged index
  int cnt;         // spare
  int cnt2;        // K2 CTAs of this layer done (split layers, gridDim.y > 1)
  double pa, pb;   // predicted a'_{x0}, b'_{y0} (meaningful when na == 1 / nb == 1)
};

enum CheckFlags {
  CK_STORE_PRED = 1,     // write the predicted vectors (offline P, explicit check)
  CK_COMPARE = 2,        // compare against the actual checksums
  CK_CORRECT = 4,        // locate + correct (online)
  CK_OFFLINE_END = 8,    // window end: records are WINDOW_DIRTY / PERSISTENT, no correction
  CK_PERSIST = 16,       // second attempt of a window
  CK_SUMMARY = 32,       // write LayerSummary (explicit check())
  CK_FROM_SUMMARY = 64,  // correct() from a stored summary, no prediction
  CK_LAZY = 128,         // checksum policy LAZY: compare b only; flagged layers -> K3
  CK_BONLY = 256,        // offline, policy LAZY: predict / compare b only (Q29)
};

struct CheckParams {
  int nx, ny, zc;
  int64_t px, plane;
  int has_lo, has_hi;
  int bc;              // abft_bc
  double g;            // ghost value (ABFT_BC_CONSTANT), rounded to the dtype
  const void* uprev;   // field buffer read by the sweep (ledger for alpha / beta)
  void* ucur;          // field buffer written by the sweep (corrected in place)
  const double* Ap;    // predictor input a^{s-1} (or offline P^{s-1}), [(zc+2)][nx]
  const double* Bp;
  double* Ac;          // actual a^s, repaired by the correction
  double* Bc;
  double* PAo;         // predicted output (CK_STORE_PRED), [(zc+2)][nx]
  double* PBo;
  const double* cA;    // c_x [zc][nx]
  const double* cB;    // c_y [zc][ny]
  double* zA;          // generation to clear for the next sweep (or null)
  double* zB;
  const void* EXp;     // edge columns x = 0 / nx-1 of uprev, [2][zc+2][ny] (interior layers)
  void* EXc;           // edge columns of ucur (patched by a correction)
  LayerSummary* summ;  // [zc]
  DevState* st;
  int* zflag;          // offline window end: [nz_global], 1 for a flagged global layer (Q28)
  double* Aw;          // lazy policy: a^{s-1} written by K3 (the predictor input generation)
  void* peerU[2];      // fused halo: neighbours' halo layer of ucur (corrections), or null
  double* fwdA[2];     // fused halo: neighbours' halo row of the checksums / predictions
  double* fwdB[2];     //   this kernel produces for layer 0 ([0]) and zc-1 ([1]), or null
  int* lazy_list;      // lazy policy: flagged layers of this sweep, [zc]
  int* lazy_rowlist;   // lazy policy: (sel << 30 | buffer layer) of the a rows K3 sums, [2 (zc+2)]
  int* lazy_mark;      // lazy policy: row already listed this sweep, [2][zc+2]
  int npoints;
  int di[kMaxPoints], dj[kMaxPoints], dk[kMaxPoints];
  double w[kMaxPoints];
  int nsources, field_src;       // the constant term C of Eq. 1 (correction_form 2)
  double coef[kMaxSources], scalar[kMaxSources];   // rounded to the dtype
  const void* src;
  int64_t spx, splane;
  double eps;
  int flags, form;
  long long sweep, z_begin;
  int zr0, zr1;        // slab-local layers of this launch, [zr0, zr1) (K2: one per grid.x)
  // pipelined schedule: K1 of sweep s + 1 ran beside this check reading u^s
  // (ucur) while it was corrected; the kernel that finishes the check (K2
  // under BOTH, K3 under LAZY) waits for it (k1_cnt[(s + 1) & 1] == k1_target) and
  // recomputes the cells of u^{s+1} that read a rewritten cell (fix_next)
  int fix;             // 1: K1 of s + 1 is in flight; 0: only list / clear
  int nfn;             // flips of sweep s + 1 in this slab (re-applied by the fix)
  unsigned k1_target;  // CTAs of K1 of s + 1 (DevState::k1_cnt[(s + 1) & 1] when it is done)
  int k1_reset;        // pipelined: K2 clears DevState::k1_cnt[s & 1] (K1 of s is done)
  void* unext;         // u^{s+1} buffer
  double* Anext;       // a^{s+1} (null under LAZY), b^{s+1}
  double* Bnext;
  void* EXnext;        // edge columns of u^{s+1}
  LocalFault fn[kMaxFaultsPerLaunch];
};

struct SweepParams {
  int nx, ny, zc, zchunk;
  int zr0, zr1;        // slab-local layers this launch computes, [zr0, zr1) (partial re-execution)
  int64_t px;          // row pitch of the field buffers (elements)
  int64_t plane;       // layer pitch = px * ny
  int has_lo, has_hi;  // neighbour rank below / above (halo layers valid)
  int bc;              // abft_bc of Eq. 1's ghosts
  double g;            // ghost value (ABFT_BC_CONSTANT), rounded to the dtype
  const void* uin;     // input field buffer (periodic wrap reads at tile edges)
  void* peerU[2];      // fused halo: the lower / upper neighbour's halo layer in its
                       // copy of `out` (local group, same or peer GPU), or null
  void* out;           // output field buffer (layer 0 = lower halo)
  double* A;           // checksum generation accumulated by this sweep, [(zc+2)][nx]
  double* B;           // [(zc+2)][ny]
  int npoints, nsources;
  int di[kMaxPoints], dj[kMaxPoints], dk[kMaxPoints];
  double w[kMaxPoints];          // already rounded to the dtype
  double coef[kMaxSources];      // already rounded to the dtype
  double scalar[kMaxSources];    // already rounded to the dtype
  float wf[kMaxPoints];          // the same values as float (fp32 fields; exact)
  float coeff[kMaxSources];
  float scalarf[kMaxSources];
  int field_src;                 // index of the source with a field, -1 if none
  const void* src;               // that field, [zc][ny][spx] (16-byte aligned rows)
  int64_t spx, splane;
  void* EX;            // edge columns of the output: [2][zc+2][ny] (x = 0, x = nx-1), or null
  unsigned* done;      // pipelined schedule: +1 per finished CTA (DevState::k1_cnt), or null
  int nfaults;
  LocalFault faults[kMaxFaultsPerLaunch];
};

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 3D tiled TMA load of one box into shared memory, completion on `bar`
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// Programmatic dependent launch: the kernels are launched with programmatic
// stream serialization, so a grid may be scheduled while the previous one
// drains; every kernel waits here before it touches memory the previous grid
// wrote (no-op when launched without the attribute).
__device__ __forceinline__ void grid_dependency_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// exact-arithmetic helpers: no contraction anywhere the numeric contract matters
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// parameter-space weights in the field dtype (no per-use conversion)
template <typename T> __device__ __forceinline__ T pw(const SweepParams& p, int q);
template <> __device__ __forceinline__ float pw<float>(const SweepParams& p, int q) { return p.wf[q]; }
template <> __device__ __forceinline__ double pw<double>(const SweepParams& p, int q) { return p.w[q]; }
template <typename T> __device__ __forceinline__ T pcoef(const SweepParams& p, int q);
template <> __device__ __forceinline__ float pcoef<float>(const SweepParams& p, int q) { return p.coeff[q]; }
template <> __device__ __forceinline__ double pcoef<double>(const SweepParams& p, int q) { return p.coef[q]; }
template <typename T> __device__ __forceinline__ T pscal(const SweepParams& p, int q);
template <> __device__ __forceinline__ float pscal<float>(const SweepParams& p, int q) { return p.scalarf[q]; }
template <> __device__ __forceinline__ double pscal<double>(const SweepParams& p, int q) { return p.scalar[q]; }

__device__ __forceinline__ float flip_bit(float v, int bit) {
  return __uint_as_float(__float_as_uint(v) ^ (1u << bit));
}
__device__ __forceinline__ double flip_bit(double v, int bit) {
  return __longlong_as_double(__double_as_longlong(v) ^ (1ll << bit));
}

// buffer layer index of slab-local layer q in [-1, zc] (layer 0 = lower halo):
// interior q -> q + 1; beyond a neighbour -> its halo layer; beyond the global
// domain edge -> clamp (P:289-292 bounce-back extended to z).
// Zero / constant ghosts: the buffer layers 0 / zc+1 that no
// neighbour owns are filled with the ghost value at init, so they are the
// ghost layer.  Periodic (single slab): wrap.
__host__ __device__ __forceinline__ int zmap(int q, int zc, int has_lo, int has_hi, int bc = ABFT_BC_CLAMP) {
  if (q < 0) {
    if (has_lo) return 0;
    return bc == ABFT_BC_CLAMP ? 1 : (bc == ABFT_BC_PERIODIC ? zc : 0);
  }
  if (q >= zc) {
    if (has_hi) return zc + 1;
    return bc == ABFT_BC_CLAMP ? zc : (bc == ABFT_BC_PERIODIC ? 1 : zc + 1);
  }
  return q + 1;
}
// global layer index q beyond a global face with zero / constant ghosts?
__host__ __device__ __forceinline__ bool zghost(int q, int zc, int has_lo, int has_hi, int bc) {
  return (bc == ABFT_BC_ZERO || bc == ABFT_BC_CONSTANT) && ((q < 0 && !has_lo) || (q >= zc && !has_hi));
}
__host__ __device__ __forceinline__ int wrap(int c, int n) { return c < 0 ? c + n : (c >= n ? c - n : c); }

}  // namespace abft
