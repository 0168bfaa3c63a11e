/*
 * abft_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, scalar CPU oracle of the ABFT-protected stencil method of
 * Cavelan & Ciorba, "Algorithm-Based Fault Tolerance for Parallel Stencil
 * Computations" (arXiv 1909.00709; /root/reference/PAPER.md, cited P:<line>).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load, link or execute this code.  It shares no code, header, table
 * or constant with the CUDA path (paper_1909_00709_b200/), and the CUDA path
 * never calls it.  Parity status of every function is in DESIGN.md §Oracle.
 *
 * Layout: fields are u[z][y][x] (x contiguous), dtype float (OR_F32) or
 * double (OR_F64).  Checksums are fp64: A[z][x] = sum_y u (the paper's row
 * checksum a_x, Eq. 2) and B[z][y] = sum_x u (column checksum b_y, Eq. 3).
 */
#ifndef ABFT_ORACLE_H
#define ABFT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_F32 = 0, OR_F64 = 1 };
enum { OR_BC_CLAMP = 0, OR_BC_PERIODIC = 1, OR_BC_ZERO = 2, OR_BC_CONSTANT = 3 };
enum { OR_MODE_NONE = 0, OR_MODE_ONLINE = 1, OR_MODE_OFFLINE = 2 };
enum {
  OR_REC_CORRECTED = 1,      /* located by intersection and corrected (Eq. 8)   */
  OR_REC_UNLOCATED = 2,      /* only one checksum vector flagged        */
  OR_REC_UNCORRECTABLE = 3,  /* >= 2 flags in a vector of one plane (Q13)       */
  OR_REC_WINDOW_DIRTY = 4,   /* offline: plane flagged at window end    */
  OR_REC_PERSISTENT = 5,     /* offline: still flagged after rollback           */
  OR_REC_RECOMPUTED = 6,     /* form 2, no single intersection: the layer was
                                recomputed from u^(t) and this cell differed  */
  OR_REC_VERIFIED = 7        /* form 2, no single intersection: the layer was
                                recomputed and no cell differed               */
};

typedef struct { int32_t di, dj, dk, pad; double w; } or_point;
typedef struct { double coef; const void* field; double scalar; } or_source;
typedef struct { int64_t sweep, z, y, x; int32_t bit, armed; } or_fault;
typedef struct {
  int64_t sweep, z, y, x;
  double observed, corrected, vx, vy;
  int32_t status, nflag_a, nflag_b, pad;
} or_record;
typedef struct {
  int64_t sweeps, detections, located, corrected, unlocated, uncorrectable,
      rollbacks, windows, persistent;
} or_stats;

typedef struct {
  int64_t nx, ny, nz;
  int32_t dtype, bc;
  double bc_value;
  int32_t npoints, nsources;
  const or_point* points;
  const or_source* sources;
  double eps;
  int32_t mode, delta;
  int32_t correction_form; /* online: 0 Eq. 8 re-summed (Q11), 1 literal fig.correction,
                              2 recompute the located cell from u^(t) */
  int32_t checksums;   /* online: 0 = a and b every sweep (SURVEY Q8 reading);
                          1 = b every sweep, a only for layers whose b flags
                          (the paper's recommendation);
                          offline: 0 = a and b compared at each window end,
                          1 = b only (offline never corrects, so the second
                          vector the paper computes "to enable correction" is
                          never needed; Q29) */
  int32_t recovery;    /* offline, dirty window: 0 = roll back to the window's
                          checkpoint and re-execute it;
                          1 = re-execute only the layers an error detected in
                          the window can have reached: those within 2 (L - 1)
                          of a flagged layer (stencil locality, P:107-108,
                          P:743-745; Q28) */
} or_problem;

/* flip bit `bit` of cell idx */
void or_flip(void* u, int64_t idx, int32_t dtype, int32_t bit);
/* one Jacobi sweep, Eq. 1; faults of this sweep flipped before the store */
void or_sweep(const or_problem* p, const void* uin, void* uout, int64_t sweep,
              or_fault* faults, int64_t nfaults);
/* actual checksums, Eqs. 2-3 */
void or_checksums(const or_problem* p, const void* u, double* A, double* B);
/* c_x, c_y of Theorem 1 */
void or_constant_sums(const or_problem* p, double* cA, double* cB);
/* predicted checksums, Theorem 1 (Eqs. 4-5) incl. alpha/beta */
void or_predict(const or_problem* p, const double* A, const double* B,
                const void* uprev, const double* cA, const double* cB,
                double* PA, double* PB);
/* detection rule, relative error vs threshold (fig.detect) */
int32_t or_flag(double pred, double act, double eps);
/* full protected run of nsweeps sweeps starting after sweep `sweep0`;
   u: in u^{sweep0}, out final field; A/B: in trusted checksums of u (or NULL
   to compute them), out final checksums.  Returns the worst status
   (0 ok, 1 detected-uncorrectable, 3 persistent error). */
int32_t or_run(const or_problem* p, void* u, double* A, double* B,
               int64_t sweep0, int64_t nsweeps, or_fault* faults, int64_t nfaults,
               or_record* recs, int64_t cap, int64_t* nrec, or_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
