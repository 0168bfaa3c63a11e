/*
 * abft_oracle.c -- TEST INFRASTRUCTURE ONLY (see abft_oracle.h).
 *
 * Plain scalar C, fp64 for every checksum quantity, the field in the dtype
 * the problem states (the paper's experiments are fp32).  Each
 * function follows one passage of PAPER.md, cited as P:<line>; readings of
 * ambiguous passages are SURVEY.md §8(c) Q<n>, restated in DESIGN.md.
 * Build: gcc -O2 -fopenmp -ffp-contract=off (no FMA contraction: the only
 * fused multiply-adds are the explicit fmaf()/fma() of the sweep chain).
 * OpenMP only distributes independent cells / planes (the paper's own
 * decomposition, one thread per layer); results do not depend on the
 * thread count.
 */
#include "abft_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- helpers */

static double ld(const void* u, int64_t i, int32_t dt) {
  return dt == OR_F32 ? (double)((const float*)u)[i] : ((const double*)u)[i];
}

/* store v rounded to the dtype (IEEE round-to-nearest-even, Q23) */
static void st(void* u, int64_t i, int32_t dt, double v) {
  if (dt == OR_F32) ((float*)u)[i] = (float)v;
  else ((double*)u)[i] = v;
}

static double rnd(int32_t dt, double v) { return dt == OR_F32 ? (double)(float)v : v; }

static size_t esz(int32_t dt) { return dt == OR_F32 ? sizeof(float) : sizeof(double); }

/* Boundary resolution of one coordinate c of an axis of extent n.
 * Clamp is the "bounce-back" of fig.sweep (Q4): out-of-range reads
 * the nearest in-domain index.  Periodic wraps.  Zero / constant ghosts
 * return -1: the read yields the ghost value. */
static int64_t res(int64_t c, int64_t n, int32_t bc) {
  if (c >= 0 && c < n) return c;
  if (bc == OR_BC_CLAMP) return c < 0 ? 0 : n - 1;
  if (bc == OR_BC_PERIODIC) return ((c % n) + n) % n;
  return -1;
}

static double ghost(const or_problem* p) {
  return p->bc == OR_BC_CONSTANT ? rnd(p->dtype, p->bc_value) : 0.0;
}

/* u^(t) at (z, y, x) including ghosts (the operand of Eq. 1) */
static double val(const or_problem* p, const void* u, int64_t z, int64_t y, int64_t x) {
  int64_t zr = res(z, p->nz, p->bc), yr = res(y, p->ny, p->bc), xr = res(x, p->nx, p->bc);
  if (zr < 0 || yr < 0 || xr < 0) return ghost(p);
  return ld(u, (zr * p->ny + yr) * p->nx + xr, p->dtype);
}

/* ------------------------------------------------------------ fault hook */

/* Single bit-flip: flip bit `bit` of the IEEE representation. */
void or_flip(void* u, int64_t idx, int32_t dtype, int32_t bit) {
  if (dtype == OR_F32) {
    uint32_t b;
    memcpy(&b, (float*)u + idx, 4);
    b ^= (uint32_t)1u << bit;
    memcpy((float*)u + idx, &b, 4);
  } else {
    uint64_t b;
    memcpy(&b, (double*)u + idx, 8);
    b ^= (uint64_t)1u << bit;
    memcpy((double*)u + idx, &b, 8);
  }
}

/* ------------------------------------------------------------ Eq. 1 sweep */

/* u^(t+1)_{x,y} = C_{x,y} + sum_{(i,j,w) in S} w * u^(t)_{x+i,y+j}   (Eq. 1)
 * extended by dk for 3D.  Canonical evaluation:
 * acc = w_0 * v_0 (rounded); acc = fma(w_p, v_p, acc) for the remaining points
 * in the stated order; then acc = fma(coef_q, src_q, acc) for each term of C.
 * Weights, coefficients and scalars are first rounded to the dtype.
 * Fault injection: the flip is applied after the point is updated and
 * before it is stored; since a Jacobi sweep never reads its own output, the
 * flips are applied to the stored values right after the update loop. */
/* Eq. 1 for one cell (z, y, x) of u^{(t+1)} from u^{(t)} = uin, the
 * canonical FMA chain (Q23): acc = w0 v0, acc = fma(w_p, v_p, acc) over the
 * points in order, then acc = fma(coef_q, src_q, acc) over the sources. */
static double cell_update(const or_problem* p, const void* uin, int64_t z, int64_t y, int64_t x) {
  const int64_t c = (z * p->ny + y) * p->nx + x;
  if (p->dtype == OR_F32) {
    float acc = 0.0f;
    for (int32_t k = 0; k < p->npoints; k++) {
      const or_point* q = &p->points[k];
      float w = (float)q->w;
      float v = (float)val(p, uin, z + q->dk, y + q->dj, x + q->di);
      acc = (k == 0) ? w * v : fmaf(w, v, acc);
    }
    for (int32_t k = 0; k < p->nsources; k++) {
      const or_source* s = &p->sources[k];
      float cf = (float)s->coef;
      float sv = s->field ? ((const float*)s->field)[c] : (float)s->scalar;
      acc = fmaf(cf, sv, acc);
    }
    return acc;
  }
  double acc = 0.0;
  for (int32_t k = 0; k < p->npoints; k++) {
    const or_point* q = &p->points[k];
    double v = val(p, uin, z + q->dk, y + q->dj, x + q->di);
    acc = (k == 0) ? q->w * v : fma(q->w, v, acc);
  }
  for (int32_t k = 0; k < p->nsources; k++) {
    const or_source* s = &p->sources[k];
    double sv = s->field ? ((const double*)s->field)[c] : s->scalar;
    acc = fma(s->coef, sv, acc);
  }
  return acc;
}

void or_sweep(const or_problem* p, const void* uin, void* uout, int64_t sweep,
              or_fault* faults, int64_t nfaults) {
  const int64_t nx = p->nx, ny = p->ny, nz = p->nz;
  const int32_t dt = p->dtype;
#pragma omp parallel for schedule(static)
  for (int64_t zy = 0; zy < nz * ny; zy++) {
    const int64_t z = zy / ny, y = zy % ny;
    for (int64_t x = 0; x < nx; x++) st(uout, (z * ny + y) * nx + x, dt, cell_update(p, uin, z, y, x));
  }
  for (int64_t f = 0; f < nfaults; f++) {
    or_fault* F = &faults[f];
    if (!F->armed || F->sweep != sweep) continue;
    /* each fault fires once (transient fault model, Q18); at most one fault
       per cell per execution of a sweep -- a second scheduled copy fires on
       the re-execution of that sweep after a rollback */
    int64_t dup = 0;
    for (int64_t g = 0; g < f; g++)
      if (faults[g].sweep == sweep && faults[g].z == F->z && faults[g].y == F->y &&
          faults[g].x == F->x && faults[g].armed == -1) dup = 1;
    if (dup) continue;
    or_flip(uout, (F->z * ny + F->y) * nx + F->x, dt, F->bit);
    F->armed = -1;
  }
  for (int64_t f = 0; f < nfaults; f++)
    if (faults[f].armed == -1) faults[f].armed = 0;
}

/* -------------------------------------------------------- Eqs. 2-3 sums */

/* a_x = sum_y u_{x,y} (Eq. 2), b_y = sum_x u_{x,y} (Eq. 3), per z-layer,
 * fp64, ascending index order; sums run over 0..n-1 (Q1). */
void or_checksums(const or_problem* p, const void* u, double* A, double* B) {
  const int64_t nx = p->nx, ny = p->ny, nz = p->nz;
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < nz; z++) {
    for (int64_t x = 0; x < nx; x++) {
      double s = 0.0;
      for (int64_t y = 0; y < ny; y++) s += ld(u, (z * ny + y) * nx + x, p->dtype);
      A[z * nx + x] = s;
    }
    for (int64_t y = 0; y < ny; y++) {
      double s = 0.0;
      for (int64_t x = 0; x < nx; x++) s += ld(u, (z * ny + y) * nx + x, p->dtype);
      B[z * ny + y] = s;
    }
  }
}

/* C_{x,y} of Eq. 1 as the exact-intent value sum_q coef_q * src_q (fp64,
 * dtype-rounded operands), then c_x = sum_y C_{x,y}, c_y = sum_x C_{x,y}
 * (Theorem 1; "pre-computed"). */
static double cval(const or_problem* p, int64_t c) {
  double s = 0.0;
  for (int32_t k = 0; k < p->nsources; k++) {
    const or_source* q = &p->sources[k];
    double cf = rnd(p->dtype, q->coef);
    double sv = q->field ? ld(q->field, c, p->dtype) : rnd(p->dtype, q->scalar);
    double t = cf * sv;
    s = (k == 0) ? t : s + t;
  }
  return s;
}

void or_constant_sums(const or_problem* p, double* cA, double* cB) {
  const int64_t nx = p->nx, ny = p->ny, nz = p->nz;
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < nz; z++) {
    for (int64_t x = 0; x < nx; x++) {
      double s = 0.0;
      for (int64_t y = 0; y < ny; y++) s += cval(p, (z * ny + y) * nx + x);
      cA[z * nx + x] = s;
    }
    for (int64_t y = 0; y < ny; y++) {
      double s = 0.0;
      for (int64_t x = 0; x < nx; x++) s += cval(p, (z * ny + y) * nx + x);
      cB[z * ny + y] = s;
    }
  }
}

/* ------------------------------------------------- Theorem 1 prediction */

/* alpha_{x,j} of Theorem 1, evaluated at the shifted column x
 * (the proof's u_{x+i,.}, Q3) of layer z; j != 0:
 *   j < 0: sum_{y=j}^{-1} u_{x,y} - sum_{y=ny+j}^{ny-1} u_{x,y}
 *   j > 0: sum_{y=ny}^{ny+j-1} u_{x,y} - sum_{y=0}^{j-1} u_{x,y}
 * (bounds read as 0..n-1, Q1); out-of-domain u are the BC's ghosts. */
static double alpha(const or_problem* p, const void* u, int64_t z, int64_t x, int32_t j) {
  const int64_t ny = p->ny;
  double s1 = 0.0, s2 = 0.0;
  if (j < 0) {
    for (int64_t y = j; y <= -1; y++) s1 += val(p, u, z, y, x);
    for (int64_t y = ny + j; y <= ny - 1; y++) s2 += val(p, u, z, y, x);
  } else {
    for (int64_t y = ny; y <= ny + j - 1; y++) s1 += val(p, u, z, y, x);
    for (int64_t y = 0; y <= j - 1; y++) s2 += val(p, u, z, y, x);
  }
  return s1 - s2;
}

/* beta_{i,y} of Theorem 1, layer z, row y; i != 0 */
static double beta(const or_problem* p, const void* u, int64_t z, int64_t y, int32_t i) {
  const int64_t nx = p->nx;
  double s1 = 0.0, s2 = 0.0;
  if (i < 0) {
    for (int64_t x = i; x <= -1; x++) s1 += val(p, u, z, y, x);
    for (int64_t x = nx + i; x <= nx - 1; x++) s2 += val(p, u, z, y, x);
  } else {
    for (int64_t x = nx; x <= nx + i - 1; x++) s1 += val(p, u, z, y, x);
    for (int64_t x = 0; x <= i - 1; x++) s2 += val(p, u, z, y, x);
  }
  return s1 - s2;
}

/* Theorem 1 (Eqs. 4-5), per z-layer with the vertical
 * neighbours read from the neighbour layer's checksum vector (Q6):
 *   a'_x = c_x + sum_{(i,j,k,w) in S} w * (a^{(t)}_{zeta(z+k)}[x+i] + alpha_{x+i,j})
 *   b'_y = c_y + sum_{(i,j,k,w) in S} w * (b^{(t)}_{zeta(z+k)}[y+j] + beta_{i,y+j})
 * Evaluated in fp64, each product and sum separately rounded, points in the
 * stated order.  If the shifted line lies wholly in a zero/constant ghost
 * region its sum is n * ghost. */
void or_predict(const or_problem* p, const double* A, const double* B,
                const void* u, const double* cA, const double* cB,
                double* PA, double* PB) {
  const int64_t nx = p->nx, ny = p->ny, nz = p->nz;
  const double g = ghost(p);
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < nz; z++) {
    for (int64_t x = 0; x < nx; x++) {
      double acc = cA[z * nx + x];
      for (int32_t k = 0; k < p->npoints; k++) {
        const or_point* q = &p->points[k];
        double w = rnd(p->dtype, q->w);
        int64_t zr = res(z + q->dk, nz, p->bc), xr = res(x + q->di, nx, p->bc);
        double S;
        if (zr < 0 || xr < 0) {
          S = (double)ny * g;
        } else {
          S = A[zr * nx + xr];
          if (q->dj != 0) S = S + alpha(p, u, zr, xr, q->dj);
        }
        acc = acc + w * S;
      }
      PA[z * nx + x] = acc;
    }
    for (int64_t y = 0; y < ny; y++) {
      double acc = cB[z * ny + y];
      for (int32_t k = 0; k < p->npoints; k++) {
        const or_point* q = &p->points[k];
        double w = rnd(p->dtype, q->w);
        int64_t zr = res(z + q->dk, nz, p->bc), yr = res(y + q->dj, ny, p->bc);
        double S;
        if (zr < 0 || yr < 0) {
          S = (double)nx * g;
        } else {
          S = B[zr * ny + yr];
          if (q->di != 0) S = S + beta(p, u, zr, yr, q->di);
        }
        acc = acc + w * S;
      }
      PB[z * ny + y] = acc;
    }
  }
}

/* --------------------------------------------------- Detection (Thm 2) */

/* fig.detect: rel = |pred/act - 1|, flagged if rel > EPSILON.
 * fp64 instead of float (Q7); NaN-safe: flagged unless rel <= eps; equal
 * values (incl. 0 == 0) are never flagged (Q24). */
int32_t or_flag(double pred, double act, double eps) {
  if (pred == act) return 0;
  double rel = fabs(pred / act - 1.0);
  return !(rel <= eps);
}

/* ------------------------------------- locate + correct (Eq. 8, fig.correction) */

static void push(or_record* recs, int64_t cap, int64_t* nrec, const or_record* r) {
  if (*nrec < cap) recs[*nrec] = *r;
  (*nrec)++;
}

/* One layer z of sweep s: compare, locate by intersection of the
 * flagged row and column, correct with Eq. 8 averaged over
 * both checksums (fig.correction) and repair the
 * checksums.  Returns 1 if detected but not corrected. */
static int32_t check_layer(const or_problem* p, int64_t s, int64_t z, void* u, const void* uprev,
                           double* A, double* B, const double* PA, const double* PB,
                           or_record* recs, int64_t cap, int64_t* nrec, or_stats* st_) {
  const int64_t nx = p->nx, ny = p->ny;
  int64_t na = 0, nb = 0, x0 = -1, y0 = -1;
  for (int64_t y = 0; y < ny; y++)
    if (or_flag(PB[z * ny + y], B[z * ny + y], p->eps)) { if (y0 < 0) y0 = y; nb++; }
  /* "it is only necessary to perform the detection on one of the two
     checksums.  If one or more errors are detected, only then ... interpolate
     the other checksum and ... perform detection" (checksums == 1) */
  if (p->checksums == 1 && nb == 0) return 0;
  for (int64_t x = 0; x < nx; x++)
    if (or_flag(PA[z * nx + x], A[z * nx + x], p->eps)) { if (x0 < 0) x0 = x; na++; }
  if (na == 0 && nb == 0) return 0;
  st_->detections++;
  or_record r;
  memset(&r, 0, sizeof r);
  r.sweep = s; r.z = z; r.y = y0; r.x = x0;
  r.nflag_a = (int32_t)na; r.nflag_b = (int32_t)nb;
  if (na == 1 && nb == 1) {
    const int64_t c = (z * ny + y0) * nx + x0;
    const double uo = ld(u, c, p->dtype);
    double vx, vy, cor;
    if (p->correction_form == 0 || p->correction_form == 2) {
      /* Eq. 8 with (a - u) evaluated as the sum of the other cells (Q11, Q12) */
      double sx = 0.0, sy = 0.0;
      for (int64_t y = 0; y < ny; y++) if (y != y0) sx += ld(u, (z * ny + y) * nx + x0, p->dtype);
      for (int64_t x = 0; x < nx; x++) if (x != x0) sy += ld(u, (z * ny + y0) * nx + x, p->dtype);
      vx = PA[z * nx + x0] - sx;
      vy = PB[z * ny + y0] - sy;
      /* form 2: stencil locality -- u^(t) is intact, so
         the located cell is recomputed from it (Eq. 1), exactly */
      cor = p->correction_form == 2 ? cell_update(p, uprev, z, y0, x0) : rnd(p->dtype, (vx + vy) / 2.0);
      A[z * nx + x0] = sx + cor;
      B[z * ny + y0] = sy + cor;
    } else {
      /* literal fig.correction listing */
      vx = PA[z * nx + x0] - (A[z * nx + x0] - uo);
      vy = PB[z * ny + y0] - (B[z * ny + y0] - uo);
      cor = rnd(p->dtype, (vx + vy) / 2.0);
      A[z * nx + x0] += cor - uo;
      B[z * ny + y0] += cor - uo;
    }
    st(u, c, p->dtype, cor);
    r.observed = uo; r.corrected = cor; r.vx = vx; r.vy = vy;
    r.status = OR_REC_CORRECTED;
    st_->located++;
    st_->corrected++;
    push(recs, cap, nrec, &r);
    return 0;
  }
  if (p->correction_form == 2) {
    /* form 2 when the flags do not intersect in one cell (several flagged
       entries, or only one vector flagged): stencil locality (P:107-108,
       P:743-745) -- u^(t) is intact, so every cell of layer z is recomputed
       from it with Eq. 1 and the cells whose stored value differs (bitwise)
       are the errors; they are rewritten, and a[z], b[z] are re-summed from
       the repaired layer (Eqs. 2-3, ascending index order).  Reading Q27. */
    int64_t changed = 0;
    for (int64_t y = 0; y < ny; y++)
      for (int64_t x = 0; x < nx; x++) {
        const int64_t c = (z * ny + y) * nx + x;
        const double v = cell_update(p, uprev, z, y, x);
        int differs;
        if (p->dtype == OR_F32) {
          const float fv = (float)v;
          differs = memcmp(&fv, (const float*)u + c, sizeof fv) != 0;
        } else {
          differs = memcmp(&v, (const double*)u + c, sizeof v) != 0;
        }
        if (!differs) continue;
        or_record rc = r;
        rc.y = y; rc.x = x;
        rc.observed = ld(u, c, p->dtype); rc.corrected = v;
        rc.status = OR_REC_RECOMPUTED;
        st(u, c, p->dtype, v);
        st_->located++;
        st_->corrected++;
        push(recs, cap, nrec, &rc);
        changed++;
      }
    for (int64_t x = 0; x < nx; x++) {
      double a = 0.0;
      for (int64_t y = 0; y < ny; y++) a += ld(u, (z * ny + y) * nx + x, p->dtype);
      A[z * nx + x] = a;
    }
    for (int64_t y = 0; y < ny; y++) {
      double b = 0.0;
      for (int64_t x = 0; x < nx; x++) b += ld(u, (z * ny + y) * nx + x, p->dtype);
      B[z * ny + y] = b;
    }
    if (changed == 0) {
      r.status = OR_REC_VERIFIED;
      push(recs, cap, nrec, &r);
    }
    return 0;
  }
  if (na == 0 || nb == 0) {
    r.status = OR_REC_UNLOCATED;         /* fig.abft.error scenario 2, Q14 */
    st_->unlocated++;
  } else {
    r.status = OR_REC_UNCORRECTABLE;     /* Q13 */
    st_->uncorrectable++;
  }
  push(recs, cap, nrec, &r);
  return 1;
}

/* -------------------------------------------------------------- driver */

int32_t or_run(const or_problem* p, void* u, double* Aout, double* Bout,
               int64_t sweep0, int64_t nsweeps, or_fault* faults, int64_t nfaults,
               or_record* recs, int64_t cap, int64_t* nrec, or_stats* stats) {
  const int64_t nx = p->nx, ny = p->ny, nz = p->nz, n = nx * ny * nz;
  const size_t fb = (size_t)n * esz(p->dtype);
  int32_t worst = 0;
  void* tmp = malloc(fb);
  void* cur = u;
  void* nxt = tmp;
  double* Ap = malloc(sizeof(double) * nz * nx);
  double* Bp = malloc(sizeof(double) * nz * ny);
  double* An = malloc(sizeof(double) * nz * nx);
  double* Bn = malloc(sizeof(double) * nz * ny);
  double* PA = malloc(sizeof(double) * nz * nx);
  double* PB = malloc(sizeof(double) * nz * ny);
  double* QA = malloc(sizeof(double) * nz * nx);
  double* QB = malloc(sizeof(double) * nz * ny);
  double* cA = malloc(sizeof(double) * nz * nx);
  double* cB = malloc(sizeof(double) * nz * ny);
  *nrec = 0;
  memset(stats, 0, sizeof *stats);
  /* trusted initial checksums of u^(sweep0) (Theorem 2 proof: "initial
     checksum is also correct") and the pre-computed c_x, c_y */
  or_checksums(p, cur, Ap, Bp);
  or_constant_sums(p, cA, cB);

  if (p->mode != OR_MODE_OFFLINE) {
    for (int64_t s = sweep0 + 1; s <= sweep0 + nsweeps; s++) {
      or_sweep(p, cur, nxt, s, faults, nfaults);
      if (p->mode == OR_MODE_ONLINE) {
        or_checksums(p, nxt, An, Bn);                    /* step 1, fig.abft */
        if (p->checksums == 1) {
          /* a is not carried from sweep to sweep: a^{s-1} is the column sum
             of u^{s-1} as it stands (computed only when needed;
             its values enter only layers whose b flags, check_layer) */
          double* Bt = malloc(sizeof(double) * nz * ny);
          or_checksums(p, cur, Ap, Bt);
          free(Bt);
        }
        or_predict(p, Ap, Bp, cur, cA, cB, PA, PB);      /* step 2 */
        for (int64_t z = 0; z < nz; z++)                 /* step 3 + correction */
          if (check_layer(p, s, z, nxt, cur, An, Bn, PA, PB, recs, cap, nrec, stats)) worst = 1;
        double* t;
        t = Ap; Ap = An; An = t;
        t = Bp; Bp = Bn; Bn = t;
      }
      void* tv = cur; cur = nxt; nxt = tv;
      stats->sweeps++;
    }
    if (p->mode == OR_MODE_NONE) or_checksums(p, cur, Ap, Bp);
  } else {
    /* Offline ABFT (Section IV): the checksums of the last verified
       state are interpolated once per sweep (algo.offline.inteprolation, P:713-726,
       applied incrementally, Q17), compared at the end of each window of delta
       sweeps; on mismatch the window is recomputed from the checkpoint taken
       at its start. */
    void* ckpt = malloc(fb);
    void* first = p->recovery == 1 ? malloc(fb) : NULL;
    char* redo = malloc((size_t)nz);      /* layers the re-execution replaces */
    char* flagged = malloc((size_t)nz);   /* layers the last window check flagged */
    int64_t s = sweep0;
    const int64_t end = sweep0 + nsweeps;
    while (s < end) {
      const int64_t wend = (s + p->delta < end) ? s + p->delta : end;
      memcpy(ckpt, cur, fb);                         /* in-memory checkpoint */
      /* layers the window check covers: all, and after a partial
         re-execution only the re-executed ones (Q28) */
      memset(redo, 1, (size_t)nz);
      for (int32_t attempt = 0; attempt < 2; attempt++) {
        memcpy(PA, Ap, sizeof(double) * nz * nx);    /* interpolation starts from */
        memcpy(PB, Bp, sizeof(double) * nz * ny);    /* the checkpoint's checksums */
        for (int64_t t = s + 1; t <= wend; t++) {
          or_sweep(p, cur, nxt, t, faults, nfaults);
          or_predict(p, PA, PB, cur, cA, cB, QA, QB);
          double* tp;
          tp = PA; PA = QA; QA = tp;
          tp = PB; PB = QB; QB = tp;
          void* tv = cur; cur = nxt; nxt = tv;
          stats->sweeps++;
        }
        if (attempt == 1 && p->recovery == 1) {
          /* partial re-execution (Q28): only the layers marked in redo come
             from the re-execution; every other layer keeps the first
             execution's values (no detected error reached it) */
          const size_t lb = (size_t)nx * ny * esz(p->dtype);
          for (int64_t z = 0; z < nz; z++)
            if (!redo[z]) memcpy((char*)cur + z * lb, (const char*)first + z * lb, lb);
        }
        or_checksums(p, cur, An, Bn);
        stats->windows++;
        int64_t dirty = 0;
        memset(flagged, 0, (size_t)nz);
        for (int64_t z = 0; z < nz; z++) {
          if (!redo[z]) continue;
          int64_t na = 0, nb = 0, x0 = -1, y0 = -1;
          /* checksums 1 (Q29): detection by b alone -- a is never compared */
          if (p->checksums != 1)
            for (int64_t x = 0; x < nx; x++)
              if (or_flag(PA[z * nx + x], An[z * nx + x], p->eps)) { if (x0 < 0) x0 = x; na++; }
          for (int64_t y = 0; y < ny; y++)
            if (or_flag(PB[z * ny + y], Bn[z * ny + y], p->eps)) { if (y0 < 0) y0 = y; nb++; }
          if (na + nb == 0) continue;
          dirty++;
          flagged[z] = 1;
          stats->detections++;
          or_record r;
          memset(&r, 0, sizeof r);
          r.sweep = wend; r.z = z; r.y = y0; r.x = x0;
          r.nflag_a = (int32_t)na; r.nflag_b = (int32_t)nb;
          r.status = attempt == 0 ? OR_REC_WINDOW_DIRTY : OR_REC_PERSISTENT;
          push(recs, cap, nrec, &r);
        }
        if (!dirty) break;
        if (attempt == 0) {
          stats->rollbacks++;                        /* rollback to t - delta */
          if (p->recovery == 1) {
            /* stencil locality, reading Q28: an error
               injected in this window of L sweeps has spread at most L - 1
               layers from its origin, and every layer it made flag lies
               within that reach, so everything it touched is within
               2 (L - 1) layers of a flagged one: the layers to re-execute
               are the union of those neighbourhoods over the flagged layers */
            const int64_t r = 2 * (wend - s - 1);
            int wraps = 0;
            memset(redo, 0, (size_t)nz);
            for (int64_t f = 0; f < nz; f++) {
              if (!flagged[f]) continue;
              if (f - r < 0 || f + r > nz - 1) wraps = 1;
              for (int64_t z = f - r; z <= f + r; z++)
                if (z >= 0 && z < nz) redo[z] = 1;
            }
            /* periodic z: a reach past a face wraps to the far layers -- take
               every layer then */
            if (p->bc == OR_BC_PERIODIC && wraps) memset(redo, 1, (size_t)nz);
            memcpy(first, cur, fb);
          }
          if (cur != ckpt) memcpy(cur, ckpt, fb);
        } else {
          stats->persistent++;
          worst = 3;
        }
      }
      double* t;
      t = Ap; Ap = An; An = t;                       /* verified state's checksums */
      t = Bp; Bp = Bn; Bn = t;
      s = wend;
    }
    free(ckpt);
    free(first);
    free(redo);
    free(flagged);
  }
  if (cur != u) memcpy(u, cur, fb);
  free(tmp);
  memcpy(Aout, Ap, sizeof(double) * nz * nx);
  memcpy(Bout, Bp, sizeof(double) * nz * ny);
  free(Ap); free(Bp); free(An); free(Bn); free(PA); free(PB); free(QA); free(QB);
  free(cA); free(cB);
  return worst;
}
