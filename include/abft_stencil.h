/*
 * abft_stencil.h -- C-ABI of the B200-native ABFT-protected stencil library
 * (libabft_stencil.so, built from paper_1909_00709_b200/csrc/).
 *
 * The method is Cavelan & Ciorba, "Algorithm-Based Fault Tolerance for
 * Parallel Stencil Computations" (arXiv 1909.00709); passages are cited as
 * PAPER.md line numbers (P:<line>) with their section / equation / listing.
 *
 * One protected sweep s (s = 1, 2, ...) is, in the paper's order (fig.abft
 * caption):
 *   (1) u^s = C + sum_S w u^{s-1}                       Eq. 1
 *       and the actual checksums a^s_x = sum_y u^s,     Eqs. 2-3
 *       b^s_y = sum_x u^s of every z-layer, in the same pass (fig.sweep)
 *   (2) the predicted checksums a', b' from a^{s-1}, b^{s-1} and the
 *       boundary terms alpha, beta                      Theorem 1
 *   (3) compare |a'/a - 1| > epsilon                    fig.detect
 *   (4) locate the corrupted cell as the intersection of the flagged
 *       row and column
 *   (5) online: correct it and repair the checksums     Eq. 8, fig.correction
 *       offline: compare once per window of `delta` sweeps and roll back to
 *       the window's checkpoint on mismatch             Section IV
 *
 * Layout.  A field is u[z][y][x], x contiguous, dtype float (ABFT_F32) or
 * double (ABFT_F64).  The domain is nx * ny * nz_global; this process owns
 * the z-slab [z_begin, z_begin + z_count).  Checksums are fp64 per z-layer:
 * A[z][x] = sum_y u (the paper's a, length nx) and B[z][y] = sum_x u (b,
 * length ny).  Coordinates in faults and records are GLOBAL.
 *
 * Ownership.  The caller owns every device buffer (field buffers, aux
 * workspace, source fields) and the CUDA stream, and keeps them alive until
 * abft_stencil_destroy.  The library owns only the opaque handle and, when
 * nranks > 1, its NCCL communicator.  It never allocates device memory.
 * One handle per rank and stream; handles are not thread-safe.
 *
 * Errors.  Every function returns an int status: 0 = ABFT_OK, negative =
 * hard error (nothing was launched or the handle is unusable for ECUDA),
 * positive = resilience outcome.  abft_strerror() names a status.
 */
#ifndef ABFT_STENCIL_H
#define ABFT_STENCIL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------------- */
#define ABFT_OK 0
#define ABFT_DETECTED_UNCORRECTABLE 1 /* a flag that was not corrected (unlocated or >1 per vector) */
#define ABFT_PERSISTENT_ERROR 3       /* offline: window still dirty after its rollback */
#define ABFT_EINVAL (-1)              /* invalid configuration or argument */
#define ABFT_ENOSPACE (-2)            /* a buffer is smaller than abft_stencil_workspace_size says */
#define ABFT_ECUDA (-3)               /* CUDA runtime / driver error */
#define ABFT_ENCCL (-4)               /* NCCL error (nranks > 1) */
#define ABFT_EUNSUPPORTED (-5)        /* valid per the paper but not implemented on this path */
#define ABFT_ETIMEOUT (-6)            /* IPC job: a neighbour rank made no progress (ABFT_IPC_TIMEOUT_S) */

/* ---- enums ---------------------------------------------------------------- */
typedef enum { ABFT_F32 = 0, ABFT_F64 = 1 } abft_dtype;
/* Boundary condition of Eq. 1 at the domain edge ("bounce-back" =
 * clamp/replicate; P:407-415 periodic, zero and constant ghosts). */
typedef enum {
  ABFT_BC_CLAMP = 0,
  ABFT_BC_PERIODIC = 1,
  ABFT_BC_ZERO = 2,
  ABFT_BC_CONSTANT = 3
} abft_bc;
/* NONE = unprotected sweep (the paper's No-ABFT baseline), ONLINE =
 * detect + correct every sweep (Section III), OFFLINE = detect every `delta`
 * sweeps + checkpoint rollback (Section IV). */
typedef enum { ABFT_MODE_NONE = 0, ABFT_MODE_ONLINE = 1, ABFT_MODE_OFFLINE = 2 } abft_mode;
/* Which actual checksum vectors an online step() computes.  BOTH: a and b of
 * every layer every sweep, both compared.  LAZY: the paper's recommendation
 * ("only one checksum vector is computed during the stencil sweep";
 * P:496-497 "only necessary to perform the detection on one of the two
 * checksums.  If one or more errors are detected, only then ... interpolate
 * the other checksum"): b every sweep; for a layer whose b flags, a^{s-1} and
 * a^s are computed from the fields and a' compared, to locate and correct.
 * OFFLINE windows under LAZY predict, sum and compare b alone: a window is
 * rolled back, never corrected, so a is never needed (Q29; dirty
 * records carry nflag_a = 0, x = -1).  The explicit sweep()/check()/correct()
 * API always uses BOTH. */
typedef enum { ABFT_CK_BOTH = 0, ABFT_CK_LAZY = 1 } abft_checksum_policy;
/* What a dirty OFFLINE window re-executes.  ROLLBACK: the whole window from
 * its checkpoint.  PARTIAL: stencil locality (P:107-108,
 * P:743-745 "exploit stencil locality to reduce the re-execution cost"): an
 * error injected in a window of L sweeps spreads at most L - 1 layers, so
 * only the layers within 2 (L - 1) of a flagged layer (the union of those
 * neighbourhoods over the flagged layers of all ranks: several disjoint
 * ranges when the flags are clustered) are re-executed from the checkpoint
 * -- the light cones of those ranges, sweep by sweep -- and re-checked;
 * every other layer keeps its first execution (Q28).  Equal to
 * ROLLBACK whenever every error of the window is detected; an undetected
 * one outside those layers is not erased. */
typedef enum { ABFT_RECOVER_ROLLBACK = 0, ABFT_RECOVER_PARTIAL = 1 } abft_recovery;
/* Schedule of an ONLINE step() on a single slab (nranks == 1).  AUTO: when
 * init is given a third field buffer, the checks of sweep s (steps (2)-(5))
 * run on a side stream beside the stencil update of sweep s + 1, which reads
 * u^s while it is being checked; a cell the checks rewrite is then recomputed
 * in u^{s+1} (with its checksums) before anything reads u^{s+1}, so every
 * result is bitwise that of the SERIAL order -- the paper's (fig.abft caption
 * detect and correct after each sweep) -- and an error-free sweep
 * never waits for its check.  SERIAL (or two buffers, or nranks > 1): each
 * sweep's checks finish before the next sweep starts. */
typedef enum { ABFT_SCHED_AUTO = 0, ABFT_SCHED_SERIAL = 1 } abft_schedule;
/* abft_record.status */
typedef enum {
  ABFT_REC_CORRECTED = 1,     /* located by intersection, corrected (Eq. 8)      */
  ABFT_REC_UNLOCATED = 2,     /* only one checksum vector flagged        */
  ABFT_REC_UNCORRECTABLE = 3, /* >= 2 flagged entries in a vector of one layer    */
  ABFT_REC_WINDOW_DIRTY = 4,  /* offline: layer flagged at a window end   */
  ABFT_REC_PERSISTENT = 5,    /* offline: layer still flagged after the rollback  */
  ABFT_REC_RECOMPUTED = 6,    /* correction_form 2, flags not intersecting in one
                                 cell: the layer was recomputed from u^{s-1} and
                                 this cell differed (rewritten)                  */
  ABFT_REC_VERIFIED = 7       /* correction_form 2, flags not intersecting in one
                                 cell: the layer was recomputed, no cell differed */
} abft_record_status;

/* ---- problem statement ---------------------------------------------------- */
/* One stencil point {i, j, w} of S plus the vertical offset dk of
 * the 3D extension.  |di|, |dj|, |dk| <= 1.  The sweep evaluates
 * the points in array order: acc = w0*v0, then acc = fma(w_p, v_p, acc). */
typedef struct {
  int32_t di, dj, dk, pad;
  double w; /* rounded to the field dtype before use */
} abft_point;

/* One term of the constant C_{x,y} of Eq. 1: coef * field[z][y][x]
 * if field != NULL, else coef * scalar.  Terms are added after the points,
 * in array order, as acc = fma(coef, src, acc).  `field` is a DEVICE pointer
 * to this rank's slab, dense [z_count][ny][nx] of the field dtype, read-only.
 * At most one term may have a field. */
typedef struct {
  double coef;
  const void* field;
  double scalar;
} abft_source;

typedef struct {
  int64_t nx, ny;       /* layer extent, >= 1 each */
  int64_t nz_global;    /* number of z-layers of the whole domain, >= 1 */
  int64_t z_begin;      /* first global layer of this rank's slab */
  int64_t z_count;      /* layers owned by this rank, >= 1 */
  int32_t dtype;        /* abft_dtype */
  int32_t bc;           /* abft_bc: all four; PERIODIC over several ranks closes
                           the z ring (rank 0 and the last rank are neighbours) */
  double bc_value;      /* ghost value for ABFT_BC_CONSTANT */
  int32_t npoints;      /* 1 .. 27 */
  int32_t nsources;     /* 0 .. 4 */
  const abft_point* points;   /* host array, copied at init */
  const abft_source* sources; /* host array, copied at init */
  double epsilon;       /* detection threshold of fig.detect, > 0 */
  int32_t mode;         /* abft_mode */
  int32_t delta;        /* offline detection period, >= 1 */
  int32_t correction_form; /* 0: Eq. 8 with (a - u) re-summed over the other cells
                              (default); 1: literal fig.correction listing; 2: the
                              located cell recomputed from u^{s-1} with Eq. 1
                              (stencil locality: exact
                              repair); when the flags do not intersect in one
                              cell, the whole layer is recomputed, the differing
                              cells rewritten and a, b of the layer re-summed
                              (Q27) */
  int32_t rank, nranks; /* z-slab decomposition; nranks == 1: single process */
  int32_t checksum_policy; /* abft_checksum_policy (ONLINE and OFFLINE step()) */
  const void* nccl_unique_id; /* host pointer to a 128-byte ncclUniqueId shared by
                                 all ranks (one process per GPU, nranks > 1); NULL
                                 for nranks == 1 or for a local group member (see
                                 abft_stencil_group) */
  int32_t recovery;     /* abft_recovery: what an OFFLINE dirty window re-executes */
  int32_t schedule;     /* abft_schedule: how an ONLINE step() of a single slab
                           orders the checks against the sweeps */
} abft_config;

/* A scheduled single bit-flip (fault model P:783-785): at sweep `sweep`
 * (1-based) the value of cell (z, y, x) gets bit `bit` flipped after its
 * update and before it is stored, so the checksums see the corrupted value.
 * Each fault fires once; a rollback re-executes without it (transient). */
typedef struct {
  int64_t sweep, z, y, x;
  int32_t bit, pad;
} abft_fault;

/* One detection event of one z-layer. */
typedef struct {
  int64_t sweep, z, y, x; /* y / x: located (or first flagged) row / column, -1 if none */
  double observed;        /* value before correction */
  double corrected;       /* value written back (Eq. 8) */
  double vx, vy;          /* the two Eq. 8 estimates from a and from b */
  int32_t status;         /* abft_record_status */
  int32_t nflag_a, nflag_b; /* flagged entries of a (over x) and of b (over y) */
  int32_t pad;
} abft_record;

/* Counters since init.  sweeps: sweeps executed, including the re-executed
 * ones after offline rollbacks; detections: (sweep, layer) events with a
 * flag; located / corrected / unlocated / uncorrectable: online outcomes;
 * rollbacks, windows, persistent: offline windows checked, rolled back, and
 * still dirty after their rollback. */
typedef struct {
  int64_t sweeps, detections, located, corrected, unlocated, uncorrectable,
      rollbacks, windows, persistent;
} abft_stats;

typedef struct abft_stencil abft_stencil;

/* ---- API ------------------------------------------------------------------ */

/* Bytes of each of the (up to three) field buffers and of the aux workspace
 * for `cfg`.  A field buffer holds the slab plus two halo layers with a
 * padded row pitch; aux holds three generations of A/B (with halo entries),
 * the offline prediction vectors, the constant sums c_x/c_y (Theorem 1,
 * P:321), the device record ring and counters.  Returns ABFT_EINVAL for an
 * invalid cfg, ABFT_EUNSUPPORTED for a valid one this build does not run. */
int abft_stencil_workspace_size(const abft_config* cfg, size_t* field_bytes, size_t* aux_bytes);

/* Number of field buffers init uses for `cfg` on the current device: 3 for
 * OFFLINE (checkpoint rotation) and for an ONLINE single slab that runs the
 * pipelined schedule (schedule AUTO and K1 z-chunks of at most two layers, or
 * ABFT_PIPELINE=1), else 2.  Errors as abft_stencil_workspace_size, plus
 * ABFT_ECUDA without a device. */
int abft_stencil_field_buffers(const abft_config* cfg, int32_t* n);

/* Create a handle.  field_bufs: 2 device buffers (NONE / ONLINE) or 3
 * (OFFLINE: the third holds the checkpoint, rotated without copies; ONLINE
 * single slab with the pipelined schedule, see abft_stencil_field_buffers: the
 * third keeps u^{s-1} for the checks of sweep s while sweep s + 1 runs -- NULL
 * selects the serial schedule), each of field_bytes; aux: device buffer of aux_bytes.  u0: this rank's initial
 * slab, dense [z_count][ny][nx] of dtype, HOST or DEVICE pointer (copied).
 * stream: cudaStream_t to run on (NULL = default stream).  Computes the
 * trusted initial checksums a^0, b^0 and c_x, c_y, and (nranks > 1) creates
 * the NCCL communicator and exchanges the initial halo.  Asynchronous on
 * `stream` except for NCCL initialisation.  Ordering is the caller's: u0,
 * the source fields and the buffers must be ready for work on `stream` (a
 * producer on another stream is waited for first), and stay allocated until
 * destroy() (which synchronises `stream`). */
int abft_stencil_init(const abft_config* cfg, void* const field_bufs[3], void* aux,
                      const void* u0, void* stream, abft_stencil** out);

/* Run n protected sweeps in the configured mode (steps (1)-(5) above).
 * NONE / ONLINE: fully asynchronous, no host synchronisation; online
 * detection outcomes are reported by abft_stencil_stats / _records /
 * _status.  OFFLINE: windows of `delta` sweeps (the last one may be shorter:
 * the call's final sweep is always checked); one host synchronisation per
 * window to read the verdict; returns ABFT_PERSISTENT_ERROR if a window
 * stayed dirty after its rollback. */
int abft_stencil_step(abft_stencil* h, int32_t nsweeps);

/* Prepare step(nsweeps) from the current state without running it.  A
 * single-slab ONLINE (either schedule) or NONE step with no
 * bit-flip scheduled in its range, runs as one CUDA graph: the launch
 * sequence depends only on the rotation phase (field buffer, checksum
 * generation, sweep parity), so step() captures it on first use and replays
 * it whenever the phase and length recur (up to 8 cached per handle).  plan()
 * does that capture ahead of time, so the first step() of that phase does not
 * pay it.  A no-op (ABFT_OK) for any other step.  ABFT_GRAPHS=0 in the
 * environment disables the graphs (every call enqueued directly). */
int abft_stencil_plan(abft_stencil* h, int32_t nsweeps);

/* Local group: n handles created by THIS process for the n slabs of one
 * domain (cfg.nranks = n, cfg.rank = i, cfg.nccl_unique_id = NULL, slabs
 * contiguous in rank order), on one GPU or on several peer GPUs.  group()
 * links them and exchanges the initial halo.  Halos then move inside the
 * kernels (fused halo): K1 stores each slab's boundary layers
 * also into the neighbours' halo layers, K2/K3 store the boundary layers'
 * checksum (or offline prediction) rows and any correction there too --
 * straight to the neighbour's memory (same device, or a peer GPU over NVLink
 * with peer access enabled by group()); events order each slab's next sweep
 * after its neighbours' sweep.  ABFT_GROUP_COPY=1 or GPUs without peer access
 * fall back to device copies after each sweep.  step_group() runs n
 * protected sweeps of every slab in lockstep (offline: windows, verdicts and
 * rollbacks are collective).  abft_stencil_step / _sweep / _check / _correct
 * reject grouped handles (ABFT_EINVAL).  Destroying a member dissolves the
 * group. */
int abft_stencil_group(abft_stencil* const* hs, int32_t n);

/* The z-slab halo plan of cfg (one process per GPU, NCCL): for the lower
 * (plan[0..2]) and upper (plan[3..5]) face, the peer rank, the buffer layer
 * sent (1 or z_count) and the halo layer received (0 or z_count + 1); -1
 * where there is no neighbour (a periodic ring has none).  No device needed. */
int abft_stencil_halo_plan(const abft_config* cfg, int32_t plan[6]);
int abft_stencil_step_group(abft_stencil* const* hs, int32_t n, int32_t nsweeps);

/* Multi-process job over CUDA IPC (one process per slab and GPU, or several
 * processes sharing a GPU): the fused halo of local groups across processes
 * (the paper's distributed-memory claim).  Each rank
 * creates its handle with cfg.nranks = n, cfg.rank = its rank and
 * cfg.nccl_unique_id = NULL, then
 *   1. abft_stencil_ipc_export(h, blob): writes ABFT_IPC_BLOB_BYTES describing
 *      its buffers (cudaIpcMemHandle + offset of each field buffer and of aux,
 *      the aux layout) and two interprocess events; synchronises the handle's
 *      stream (its initial state is ready for the neighbours to read);
 *   2. the blobs travel to the neighbours by any host channel (bench.py and the
 *      tests use torch.distributed all_gather_object);
 *   3. abft_stencil_ipc_link(h, lo_blob, hi_blob, shm): maps the neighbours'
 *      buffers (peer access over NVLink, or the same GPU), opens their events,
 *      pulls the initial halo and zeroes this rank's progress slot.  lo_blob /
 *      hi_blob: the blob of rank - 1 / rank + 1 (modulo nranks for a periodic
 *      ring), NULL at a global face.  shm:
 *      an array of nranks abft_ipc_slot in host memory mapped by every
 *      process of the job (e.g. a /dev/shm segment), zero-initialised; the
 *      caller keeps it mapped until destroy.  Every rank must have linked (a
 *      barrier) before any rank steps.
 * Then step() stores each sweep's boundary layers, their checksum (or
 * prediction) rows and any correction of a boundary cell straight into the
 * neighbours' halo slots from K1 / K2 / K3, and orders the next sweep after
 * the neighbours' through the events (a rank publishes its sweep count in
 * its slot; a neighbour enqueues the wait once the count is there).  Offline
 * window verdicts and the flagged layers (partial re-execution) are reduced
 * over all ranks through the slots.  Every rank
 * calls step() with the same counts (lockstep).  Errors: ABFT_EINVAL for a
 * handle that is grouped, has a communicator, has stepped, or a blob that
 * does not describe the expected neighbour; ABFT_EUNSUPPORTED for recovery
 * PARTIAL with a slab of more than 32 * ABFT_IPC_ZWORDS layers (its flagged
 * layers travel as bits in the slot); ABFT_ECUDA if a handle or event cannot
 * be opened. */
#define ABFT_IPC_BLOB_BYTES 1024
#define ABFT_IPC_ZWORDS 256   /* recovery PARTIAL over IPC: z_count <= 32 * ABFT_IPC_ZWORDS per rank */
typedef struct {
  int64_t seq;        /* halo exchanges this rank has published */
  int64_t wseq;       /* offline windows whose verdict this rank has published */
  int64_t wdone;      /* offline windows this rank has reduced */
  int32_t val[2][3];  /* verdict per window parity: flagged layers, extent words */
  int32_t z_begin;    /* this rank's slab (set by ipc_link) */
  int32_t z_count;
  uint32_t zbits[2][ABFT_IPC_ZWORDS];  /* per window parity: flagged layers of the slab, bit z - z_begin */
} abft_ipc_slot;
int abft_stencil_ipc_export(abft_stencil* h, void* blob);
int abft_stencil_ipc_link(abft_stencil* h, const void* lo_blob, const void* hi_blob, void* shm);

/* Explicit-control API (ONLINE / NONE handles), the paper's listings one by
 * one.  sweep(): one sweep with the actual checksums of the result (fig.sweep).
 * check(): predicted checksums of the last sweep (Theorem 1, fig.interpolation)
 * compared with the actual ones (fig.detect); returns the number of flagged
 * entries of a and b over the slab (synchronises).  correct(): locate and
 * correct the flags of the last check (fig.correction); *ncorrected = cells
 * written back.  step(n) is n x (sweep, check, correct) without host syncs. */
int abft_stencil_sweep(abft_stencil* h);
int abft_stencil_check(abft_stencil* h, int64_t* nflag_a, int64_t* nflag_b);
int abft_stencil_correct(abft_stencil* h, int64_t* ncorrected);

/* Schedule bit-flips (test / measurement hook).  Replaces the pending list;
 * faults outside this rank's slab are ignored by this rank.  A cell listed k
 * times for one sweep is flipped in k executions of that sweep (the first and
 * k - 1 offline re-executions: a fault that strikes again, i.e. a persistent
 * error).  ABFT_EINVAL (and an empty list) if a fault is out of range or more
 * than 64 entries fall in this slab in one sweep. */
int abft_stencil_set_faults(abft_stencil* h, const abft_fault* faults, int32_t n);

/* Read-back.  All synchronise the handle's stream. */
/* device pointer to u[z_begin][0][0] of the current field and its row pitch
   in elements (layer pitch = pitch * ny) */
int abft_stencil_field(abft_stencil* h, void** dev_ptr, int64_t* pitch);
/* copy the current slab, dense [z_count][ny][nx], to dst (HOST or DEVICE) */
int abft_stencil_read_field(abft_stencil* h, void* dst);
/* copy the current actual checksums A [z_count][nx], B [z_count][ny] (HOST or DEVICE);
   under LAZY (a not carried) A is summed from the current field first */
int abft_stencil_checksums(abft_stencil* h, double* A, double* B);
int abft_stencil_stats(abft_stencil* h, abft_stats* out);
/* copy up to cap records (in device append order) to the host array out;
   *n = total recorded (may exceed cap; the ring keeps the first entries) */
int abft_stencil_records(abft_stencil* h, abft_record* out, int32_t cap, int64_t* n);
/* worst resilience status so far: ABFT_OK, _DETECTED_UNCORRECTABLE or _PERSISTENT_ERROR */
int abft_stencil_status(abft_stencil* h);
/* logical sweep index of the current state (rollbacks do not count twice) */
int64_t abft_stencil_sweep_count(const abft_stencil* h);

/* Kernel launches issued by this handle so far (for launch accounting). */
int64_t abft_stencil_launch_count(const abft_stencil* h);

/* Measurement hook.  enable != 0: every K1 (fused sweep + checksums) launch
 * and every check launch -- K2 (predict / compare / locate / correct) and,
 * under the LAZY policy, K3 (second checksum of flagged layers) -- is
 * bracketed by CUDA events on the handle's stream (the events also disable
 * the programmatic-dependent-launch overlap between them).  profile_read
 * synchronises, returns the summed device time (ms) and launch counts of K1
 * and of the checks (k2_*) since the last read, and resets them.  Also
 * reports the K1 launch geometry (grid x, y, z, threads per CTA, dynamic
 * shared memory bytes, layers per CTA) when geo != NULL. */
int abft_stencil_profile(abft_stencil* h, int32_t enable);
int abft_stencil_profile_read(abft_stencil* h, double* k1_ms, int64_t* k1_launches,
                              double* k2_ms, int64_t* k2_launches, int32_t geo[6]);

/* Free the handle and its NCCL communicator; never the caller's buffers. */
int abft_stencil_destroy(abft_stencil* h);

const char* abft_strerror(int status);

#ifdef __cplusplus
}
#endif
#endif /* ABFT_STENCIL_H */
