// abft_stencil.cu -- host side of libabft_stencil.so: the C-ABI of
// include/abft_stencil.h, workspace carving, the online / offline sweep loop,
// the fault schedule, and the z-slab halo exchange over NCCL (NVLink).
//
// Everything numeric runs in the sm_100a kernels of sweep.cuh / check.cuh;
// this file only validates, lays out memory, encodes TMA descriptors and
// sequences launches on the caller's stream.  There is no CPU fallback: a
// missing device or driver entry point is a hard ABFT_ECUDA.
#include <dlfcn.h>
#include <sched.h>
#include <time.h>
#include <map>
#include <array>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <tuple>
#include <cstdlib>
#include <vector>

#include "check.cuh"
#include "common.cuh"
#include "launch.h"
#include "nccl.h"

using namespace abft;

namespace {

// ------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.ok ? &api : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
#define NSYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
  NSYM(commInitRank, "ncclCommInitRank");
  NSYM(commDestroy, "ncclCommDestroy");
  NSYM(groupStart, "ncclGroupStart");
  NSYM(groupEnd, "ncclGroupEnd");
  NSYM(send, "ncclSend");
  NSYM(recv, "ncclRecv");
  NSYM(allReduce, "ncclAllReduce");
#undef NSYM
  api.ok = api.commInitRank && api.commDestroy && api.groupStart && api.groupEnd && api.send &&
           api.recv && api.allReduce;
  return api.ok ? &api : nullptr;
}

// One communicator per (job, rank): handles created with the same unique id
// share it (reference counted), so a process that runs several handles of one
// job in turn -- bench.py's runs -- pays one ncclCommInitRank.  Handles that
// share a communicator must not run concurrently.
struct CommCache {
  std::map<std::array<char, sizeof(ncclUniqueId)>, std::pair<ncclComm_t, int>> m;
};
CommCache& comm_cache() {
  static CommCache c;
  return c;
}
int comm_acquire(const void* id_bytes, int nranks, int rank, ncclComm_t* out) {
  NcclApi* n = nccl_api();
  if (!n) return ABFT_ENCCL;
  std::array<char, sizeof(ncclUniqueId)> key;
  memcpy(key.data(), id_bytes, key.size());
  auto it = comm_cache().m.find(key);
  if (it != comm_cache().m.end()) {
    it->second.second++;
    *out = it->second.first;
    return ABFT_OK;
  }
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof(id));
  if (n->commInitRank(out, nranks, id, rank) != ncclSuccess) return ABFT_ENCCL;
  comm_cache().m[key] = {*out, 1};
  return ABFT_OK;
}
void comm_release(ncclComm_t c) {
  for (auto it = comm_cache().m.begin(); it != comm_cache().m.end(); ++it)
    if (it->second.first == c) {
      if (--it->second.second == 0) {
        if (NcclApi* n = nccl_api()) n->commDestroy(c);
        comm_cache().m.erase(it);
      }
      return;
    }
}

// ------------------------------------------------------- TMA descriptor encode
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool encode3d(CUtensorMap* m, int dtype, void* base, uint64_t d0, uint64_t d1, uint64_t d2,
              uint64_t pitch_bytes, uint64_t layer_bytes, uint32_t b0, uint32_t b1, uint32_t b2 = 1,
              CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {pitch_bytes, layer_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, dtype == ABFT_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                  3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
  int esz;
  int64_t px, plane;
  size_t field_bytes;
  // aux offsets
  size_t off_gA[kGens], off_gB[kGens], off_PA[2], off_PB[2], off_cA, off_cB, off_summ, off_lazy, off_st, off_src, off_zflag;
  size_t off_EX[3];  // x-edge ledger of each field buffer, [2][zc+2][ny] of dtype
  size_t aux_bytes;
  size_t hot_bytes;  // prefix of aux touched every sweep
  bool pad_src;
};

// K1 launch geometry of a config on a device, and whether an online step()
// runs the pipelined schedule
struct K1Plan {
  int zchunk;
  dim3 grid;
  bool pipe;
};
K1Plan k1_plan(const abft_config* cfg, int dev) {
  const K1Geometry geo = k1_geometry(cfg->dtype);
  const int64_t nx = cfg->nx, ny = cfg->ny, zc = cfg->z_count;
  int nsm = 148;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm < 1) nsm = 148;
  const int tiles_x = (int)((nx + geo.tile_x - 1) / geo.tile_x);
  const int tiles_y = (int)((ny + geo.tile_y - 1) / geo.tile_y);
  const int64_t tiles = (int64_t)tiles_x * tiles_y;
  // z-chunks: ~32 waves of resident CTAs (the last, partial wave then costs
  // little; measured on cfg4: 8 waves / 103 layers per CTA -> 32 waves / 28
  // layers: protected K1 -3%), but >= 16 layers per CTA (each chunk re-stages
  // its two z-halo layers)
  const int per_sm = std::max(1, (228 * 1024) / (geo.smem + 1024));
  const int64_t target = (int64_t)32 * nsm * per_sm;
  int64_t nch = std::max<int64_t>(1, std::min<int64_t>(zc, (target + tiles - 1) / tiles));
  int64_t zch = std::max<int64_t>((zc + nch - 1) / nch, std::min<int64_t>(zc, 16));
  // ... unless that leaves SMs idle (few tiles and layers: cfg2, cfg3), then
  // about four waves of short chunks (cfg3: 13 -> 4 layers per CTA measured
  // 42.2 -> 37.2 us per unprotected sweep; cfg2 stays at 1)
  const int64_t slots = (int64_t)nsm * per_sm;
  if (tiles * ((zc + zch - 1) / zch) < slots)
    zch = std::max<int64_t>(1, (tiles * zc + 4 * slots - 1) / (4 * slots));
  K1Plan k;
  k.zchunk = (int)zch;
  if (const char* e = getenv("ABFT_ZCHUNK")) k.zchunk = std::max(1, std::min((int)zc, atoi(e)));
  k.grid = dim3(tiles_x, tiles_y, (unsigned)((zc + k.zchunk - 1) / k.zchunk));
  // The pipelined schedule pays where K1's CTAs are short-lived (one or two
  // layers each: cfg1, cfg2): the checks' CTAs get SM slots as K1's retire.
  // With long z-chunks K1 holds every slot (two CTAs use the whole register
  // file) until its last wave, so the checks cannot run beside it and the
  // serial order is as fast or faster (measured).
  // ABFT_PIPELINE=0/1 overrides the choice where the schedule is allowed.
  k.pipe = cfg->mode == ABFT_MODE_ONLINE && cfg->nranks == 1 && cfg->schedule == ABFT_SCHED_AUTO;
  if (k.pipe) {
    const char* e = getenv("ABFT_PIPELINE");
    k.pipe = e ? atoi(e) != 0 : k.zchunk <= 2;
  }
  return k;
}

int field_source(const abft_config* c) {
  int fs = -1;
  for (int q = 0; q < c->nsources; ++q)
    if (c->sources[q].field) fs = q;
  return fs;
}

int validate(const abft_config* c) {
  if (!c) return ABFT_EINVAL;
  if (c->nx < 1 || c->ny < 1 || c->nz_global < 1 || c->z_count < 1 || c->z_begin < 0 ||
      c->z_begin + c->z_count > c->nz_global)
    return ABFT_EINVAL;
  if (c->nx > (1LL << 30) || c->ny > (1LL << 30) || c->z_count > (1LL << 30)) return ABFT_EINVAL;
  if (c->dtype != ABFT_F32 && c->dtype != ABFT_F64) return ABFT_EINVAL;
  if (c->bc < 0 || c->bc > 3) return ABFT_EINVAL;
  if (c->npoints < 1 || c->npoints > kMaxPoints || !c->points) return ABFT_EINVAL;
  for (int q = 0; q < c->npoints; ++q) {
    const abft_point& p = c->points[q];
    if (p.di < -1 || p.di > 1 || p.dj < -1 || p.dj > 1 || p.dk < -1 || p.dk > 1) return ABFT_EUNSUPPORTED;
    if (!isfinite(p.w)) return ABFT_EINVAL;
    for (int r = 0; r < q; ++r)
      if (c->points[r].di == p.di && c->points[r].dj == p.dj && c->points[r].dk == p.dk) return ABFT_EINVAL;
  }
  if (c->nsources < 0 || c->nsources > kMaxSources || (c->nsources > 0 && !c->sources)) return ABFT_EINVAL;
  int nf = 0;
  for (int q = 0; q < c->nsources; ++q) {
    if (!isfinite(c->sources[q].coef) || !isfinite(c->sources[q].scalar)) return ABFT_EINVAL;
    if (c->sources[q].field) nf++;
  }
  if (nf > 1) return ABFT_EUNSUPPORTED;
  if (!(c->epsilon > 0.0) || !isfinite(c->epsilon)) return ABFT_EINVAL;
  if (c->mode < 0 || c->mode > 2) return ABFT_EINVAL;
  if (c->mode == ABFT_MODE_OFFLINE && c->delta < 1) return ABFT_EINVAL;
  if (c->correction_form < 0 || c->correction_form > 2) return ABFT_EINVAL;
  if (c->checksum_policy != ABFT_CK_BOTH && c->checksum_policy != ABFT_CK_LAZY) return ABFT_EINVAL;
  if (c->recovery != ABFT_RECOVER_ROLLBACK && c->recovery != ABFT_RECOVER_PARTIAL) return ABFT_EINVAL;
  if (c->schedule != ABFT_SCHED_AUTO && c->schedule != ABFT_SCHED_SERIAL) return ABFT_EINVAL;
  if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) return ABFT_EINVAL;
  if (c->nranks > 1) {
    if ((c->rank == 0) != (c->z_begin == 0)) return ABFT_EINVAL;
    if ((c->rank == c->nranks - 1) != (c->z_begin + c->z_count == c->nz_global)) return ABFT_EINVAL;
  } else if (c->z_begin != 0 || c->z_count != c->nz_global) {
    return ABFT_EINVAL;
  }
  if (c->bc == ABFT_BC_CONSTANT && !isfinite(c->bc_value)) return ABFT_EINVAL;
  return ABFT_OK;
}

Layout layout(const abft_config* c) {
  Layout L;
  L.esz = c->dtype == ABFT_F32 ? 4 : 8;
  const int64_t align_elems = 128 / L.esz;  // 128-byte rows: TMA strides + coalescing
  L.px = (c->nx + align_elems - 1) / align_elems * align_elems;
  L.plane = L.px * c->ny;
  L.field_bytes = align_up((size_t)L.plane * (c->z_count + 2) * L.esz, 256);
  const size_t zc2 = (size_t)c->z_count + 2;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  // per-sweep vectors first (checksum generations, c_x / c_y, edge ledgers).
  // A persisting-L2 window over them was measured: K2 unchanged, K1 2x slower
  // (the carve-out starves the streaming sweep), so none is set.
  for (int g = 0; g < kGens; ++g) { L.off_gA[g] = take(zc2 * c->nx * 8); L.off_gB[g] = take(zc2 * c->ny * 8); }
  L.off_cA = take((size_t)c->z_count * c->nx * 8);
  L.off_cB = take((size_t)c->z_count * c->ny * 8);
  for (int b = 0; b < 3; ++b) L.off_EX[b] = take((size_t)2 * zc2 * c->ny * L.esz);
  L.off_summ = take((size_t)c->z_count * sizeof(LayerSummary));
  L.off_lazy = take((size_t)c->z_count * sizeof(int) + (size_t)4 * zc2 * sizeof(int));
  L.off_st = take(sizeof(DevState));
  L.hot_bytes = o;
  for (int g = 0; g < 2; ++g) { L.off_PA[g] = take(zc2 * c->nx * 8); L.off_PB[g] = take(zc2 * c->ny * 8); }
  const int fs = field_source(c);
  L.pad_src = fs >= 0 && ((c->nx * L.esz) % 16 != 0 ||
                          (reinterpret_cast<uintptr_t>(c->sources[fs].field) % 16) != 0);
  L.off_src = L.pad_src ? take((size_t)L.plane * c->z_count * L.esz) : 0;
  // offline: one word per global layer, set by a window check that flags it
  L.off_zflag = take((size_t)c->nz_global * sizeof(int));
  L.aux_bytes = o;
  return L;
}

struct PendingFault {
  abft_fault f;
  bool fired;
};

}  // namespace

struct abft_stencil;
using Group = std::vector<abft_stencil*>;

namespace {
// A whole step(n) of a single slab captured as one CUDA graph.  What a step
// enqueues depends only on the rotation phase (field buffer, checksum
// generation, sweep parity, generations known zero) and n, so a later call in
// the same phase replays the instantiated graph; the sweep numbers the checks
// record are offset on the device (DevState::sweep_off, set by the graph's
// first node).
struct StepGraph {
  int n, cur, gen, par;
  unsigned zmask;
  int64_t sweeps0;                 // sweep count at capture
  cudaGraph_t graph = nullptr;     // kept: its node handles address the exec's nodes
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t off = nullptr;   // memset node: sweep_off = sweeps - sweeps0
  int cur2, prev2, gen2, gen_prev2;
  unsigned zmask2;
  int64_t launches;
  uint64_t used;
};
constexpr size_t kMaxGraphs = 8;
}  // namespace

struct abft_stencil {
  abft_config cfg;
  std::vector<abft_point> points;
  std::vector<abft_source> sources;
  Layout L;
  int nbuf = 2;
  char* fb[3] = {nullptr, nullptr, nullptr};
  char* aux = nullptr;
  char* EX[3] = {nullptr, nullptr, nullptr};
  double* gA[kGens];
  double* gB[kGens];
  double* PA[2];
  double* PB[2];
  double *cA, *cB;
  LayerSummary* summ;
  int* lazy_list;
  int* lazy_rowlist;
  int* lazy_mark;
  DevState* st;
  const void* src_field = nullptr;
  int64_t src_px = 0;
  int field_src = -1;
  cudaStream_t stream = nullptr;
  CUtensorMap tm_u[3];
  int shape = SHAPE_GENERIC;
  K1Geometry geo;
  dim3 grid1;
  int zchunk = 1;
  SweepParams sp;
  CheckParams cp;
  int cur = 0;       // buffer holding the current field
  int prev = 1;      // buffer holding the previous field (explicit API)
  int gen = 0;       // checksum generation of the current state
  int gen_prev = 0;
  bool pending_check = false;
  unsigned zmask = 0;      // bit g: checksum generation g is known to be zero
  bool summ_dirty = false; // check() left layer summaries that correct() did not consume
  int64_t sweeps = 0;      // logical sweep index of the current state
  int64_t executed = 0;    // sweeps executed, incl. re-executions after rollbacks
  int64_t launches = 0;
  int64_t rollbacks = 0, windows = 0, persistent = 0;
  int host_worst = 0;
  int* zflag = nullptr;    // [nz_global] offline: layers the last window check flagged (Q28)
  // offline, single slab: while the host waits for window w's verdict the GPU
  // already runs sweep 1 of window w + 1 (into the buffer that is neither
  // w's checkpoint nor its result); kept if w is clean, dropped otherwise
  bool spec_on = true;              // ABFT_OFFLINE_SPEC=0: wait idle instead
  bool spec_done = false;           // sweep 1 of the next window has run
  int* pin_dirty = nullptr;         // pinned host copy of the window verdict
  cudaEvent_t ev_verdict = nullptr;
  std::vector<PendingFault> faults;
  ncclComm_t comm = nullptr;
  // multi-process job over CUDA IPC (abft_stencil_ipc_link): neighbour proxies
  // (mapped buffers + IPC events), the host-shared progress slots, counters
  bool ipc = false;
  abft_ipc_slot* shm = nullptr;
  int64_t xseq = 0, wseq = 0;
  cudaEvent_t ev_ipc[2] = {nullptr, nullptr};
  std::vector<void*> ipc_opened;   // bases from cudaIpcOpenMemHandle (closed at destroy)
  abft_stencil* proxy[2] = {nullptr, nullptr};
  bool is_proxy = false;
  int has_lo = 0, has_hi = 0;
  // local group (several slabs in one process): neighbours and sync events
  abft_stencil* lo_peer = nullptr;
  abft_stencil* hi_peer = nullptr;
  bool grouped = false;
  std::vector<abft_stencil*> members;
  // fused halo (local group): the sweep's kernels store the boundary layers,
  // their checksum / prediction rows and corrections straight into the
  // neighbours' halo slots; fwd_* name what crosses a face this sweep
  bool fused = false;
  int fwd_buf = -1, fwd_kind = 0, fwd_idx = 0;
  int dev = 0;
  cudaEvent_t ev_ready = nullptr, ev_pulled = nullptr;
  // pipelined online schedule (single slab, three field buffers): the checks
  // of sweep s on the side stream s2, beside K1 of sweep s + 1 (online_pipelined)
  bool pipe = false;
  cudaStream_t s2 = nullptr;
  cudaStream_t cs = nullptr;        // capture stream of the step graphs
  bool graphs_on = true;            // ABFT_GRAPHS=0: enqueue every call directly
  bool pipe_pdl = false;            // pipelined K1 with programmatic serialization (experiment)
  std::vector<StepGraph> graphs;
  uint64_t graph_tick = 0;
  cudaEvent_t ev_k1 = nullptr, ev_chk[2] = {nullptr, nullptr};
  // measurement hook: event pairs around K1 / K2 launches
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_kind;  // 1 = K1, 2 = K2, per pair
  size_t ev_used = 0;        // pairs in use
};

namespace {

// Every per-handle CUDA call runs on the handle's device (a local group may
// span peer GPUs); the C-ABI entry points restore the caller's device.
inline void on_dev(const abft_stencil* h) {
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess || d != h->dev) cudaSetDevice(h->dev);
}
struct DevScope {
  int old = -1;
  explicit DevScope(const abft_stencil* h) {
    if (cudaGetDevice(&old) != cudaSuccess) old = -1;
    if (h && old != h->dev) cudaSetDevice(h->dev);
    else old = -1;
  }
  ~DevScope() { if (old >= 0) cudaSetDevice(old); }
};

cudaEvent_t* prof_begin(abft_stencil* h, int kind, cudaStream_t s) {
  if (!h->prof) return nullptr;
  if (h->ev_used * 2 + 2 > h->ev.size()) {
    for (int i = 0; i < 2; ++i) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      h->ev.push_back(e);
    }
    h->ev_kind.push_back(0);
  }
  cudaEvent_t* pair = &h->ev[h->ev_used * 2];
  h->ev_kind[h->ev_used] = kind;
  h->ev_used++;
  cudaEventRecord(pair[0], s);
  return pair;
}
void prof_end(cudaEvent_t* pair, cudaStream_t s) {
  if (pair) cudaEventRecord(pair[1], s);
}

#define CK(x)                                              \
  do {                                                     \
    cudaError_t e_ = (x);                                  \
    if (e_ != cudaSuccess) {                               \
      fprintf(stderr, "abft_stencil: %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return ABFT_ECUDA;                                   \
    }                                                      \
  } while (0)

int match_shape(const abft_config* c) {
  auto same = [&](auto shape_tag) {
    using S = decltype(shape_tag);
    if (c->npoints != S::NP) return false;
    for (int q = 0; q < S::NP; ++q)
      if (c->points[q].di != S::off(q, 0) || c->points[q].dj != S::off(q, 1) ||
          c->points[q].dk != S::off(q, 2))
        return false;
    return true;
  };
  if (same(Shape<SHAPE_HOTSPOT7>{})) {
    const bool fs = c->nsources == 2 && c->sources[0].field && !c->sources[1].field;
    return fs ? SHAPE_HOTSPOT7_FS : SHAPE_HOTSPOT7;
  }
  if (same(Shape<SHAPE_FIG2_5PT>{})) return SHAPE_FIG2_5PT;
  if (same(Shape<SHAPE_BOX27>{})) return SHAPE_BOX27;
  return SHAPE_GENERIC;
}

double rnd(int dtype, double v) { return dtype == ABFT_F32 ? (double)(float)v : v; }

// steps (2)-(5) parameters for one sweep (see CheckParams)
constexpr int XV_GEN_ID = 1, XV_P_ID = 2;   // = XV_GEN, XV_P below

CheckParams make_check(abft_stencil* h, int uprev, int ucur, const double* Ap, const double* Bp,
                       double* Ac, double* Bc, double* PAo, double* PBo, double* zA, double* zB,
                       int flags, int64_t sweep) {
  CheckParams p = h->cp;
  p.uprev = h->fb[uprev];
  p.ucur = h->fb[ucur];
  p.Ap = Ap; p.Bp = Bp; p.Ac = Ac; p.Bc = Bc; p.PAo = PAo; p.PBo = PBo; p.zA = zA; p.zB = zB;
  p.EXp = h->EX[uprev];
  p.EXc = h->EX[ucur];
  p.flags = flags;
  p.sweep = sweep;
  for (int f = 0; f < 2; ++f) { p.peerU[f] = nullptr; p.fwdA[f] = p.fwdB[f] = nullptr; }
  if (h->fused && h->fwd_buf == ucur) {
    abft_stencil* nb[2] = {h->lo_peer, h->hi_peer};
    const size_t lb = (size_t)h->L.plane * h->L.esz;
    for (int f = 0; f < 2; ++f) {
      abft_stencil* q = nb[f];
      if (!q) continue;
      const int64_t row = f == 0 ? q->cfg.z_count + 1 : 0;   // the neighbour's halo slot
      p.peerU[f] = q->fb[ucur] + (size_t)row * lb;
      double *qa = nullptr, *qb = nullptr;
      if (h->fwd_kind == XV_GEN_ID) { qa = q->gA[h->fwd_idx]; qb = q->gB[h->fwd_idx]; }
      if (h->fwd_kind == XV_P_ID) { qa = q->PA[h->fwd_idx]; qb = q->PB[h->fwd_idx]; }
      // lazy policy: a rows are K3 scratch, recomputed from the field by the neighbour
      if (qa && !(flags & CK_LAZY)) p.fwdA[f] = qa + (size_t)row * q->cfg.nx;
      if (qb) p.fwdB[f] = qb + (size_t)row * q->cfg.ny;
    }
  }
  return p;
}

// this slab's armed flips of `sweep` (at most one per cell per execution);
// `mark`: they fire now
int sweep_faults(abft_stencil* h, int64_t sweep, LocalFault* out, bool mark) {
  int n = 0;
  for (auto& pf : h->faults) {
    if (pf.fired || pf.f.sweep != sweep) continue;
    const int64_t zl = pf.f.z - h->cfg.z_begin;
    if (zl < 0 || zl >= h->cfg.z_count) continue;
    bool dup = false;
    for (int k = 0; k < n; ++k)
      if (out[k].z == zl && out[k].y == pf.f.y && out[k].x == pf.f.x) dup = true;
    if (dup || n == kMaxFaultsPerLaunch) continue;
    out[n++] = LocalFault{(int)zl, (int)pf.f.y, (int)pf.f.x, pf.f.bit};
    if (mark) pf.fired = true;
  }
  return n;
}

// CTAs of a whole-slab K1 launch
unsigned long long k1_grid_ctas(const abft_stencil* h) {
  const unsigned long long gz = (h->cfg.z_count + h->zchunk - 1) / h->zchunk;
  return (unsigned long long)h->grid1.x * h->grid1.y * gz;
}

// K1: step (1)
// za / zb: the slab-local layers [za, zb) to compute (partial re-execution;
// zb < 0: the whole slab); count: add its CTAs to DevState::k1_cnt[sweep & 1] as they
// finish (pipelined schedule)
int launch_k1(abft_stencil* h, int src, int dst, double* A, double* B, int chk, int64_t sweep,
              int za = 0, int zb = -1, bool count = false) {
  SweepParams p = h->sp;
  if (zb < 0) zb = (int)h->cfg.z_count;
  p.zr0 = za;
  p.zr1 = zb;
  dim3 grid = h->grid1;
  grid.z = (unsigned)((zb - za + h->zchunk - 1) / h->zchunk);
  p.out = h->fb[dst];
  p.uin = h->fb[src];
  p.peerU[0] = p.peerU[1] = nullptr;
  if (h->fused && h->fwd_buf == dst) {
    const size_t lb = (size_t)h->L.plane * h->L.esz;
    if (h->lo_peer) p.peerU[0] = h->lo_peer->fb[dst] + (size_t)(h->lo_peer->cfg.z_count + 1) * lb;
    if (h->hi_peer) p.peerU[1] = h->hi_peer->fb[dst];
  }
  p.EX = h->cfg.mode != ABFT_MODE_NONE ? h->EX[dst] : nullptr;
  p.A = A;
  p.B = B;
  p.done = count ? &h->st->k1_cnt[sweep & 1] : nullptr;
  p.nfaults = sweep_faults(h, sweep, p.faults, true);
  // K1 variant: constant / periodic ghosts need the general one; scheduled
  // flips the injecting one; everything else runs the hot path
  const bool inj = p.nfaults > 0;
  on_dev(h);
  const int var = ((h->cfg.bc == ABFT_BC_CONSTANT || h->cfg.bc == ABFT_BC_PERIODIC) ? K1_GEN
                   : (inj ? K1_INJ : K1_HOT)) | (count && !h->pipe_pdl ? K1_NO_PDL : 0);
  h->executed++;
  cudaEvent_t* pe = prof_begin(h, 1, h->stream);
  const cudaError_t e = h->cfg.dtype == ABFT_F32
            ? launch_k1_f32(h->shape, chk, var, grid, h->stream, h->tm_u[src], p)
            : launch_k1_f64(h->shape, chk, var, grid, h->stream, h->tm_u[src], p);
  prof_end(pe, h->stream);
  h->launches++;
  CK(e);
  return ABFT_OK;
}

// K2: steps (2)-(5) as their own launch (on the handle's stream, or the
// side stream of the pipelined schedule)
int launch_check(abft_stencil* h, const CheckParams& p, cudaStream_t s = nullptr) {
  on_dev(h);
  if (!s) s = h->stream;
  cudaEvent_t* pe = prof_begin(h, 2, s);
  cudaError_t e = launch_k2(h->cfg.dtype, h->shape, s, p);
  prof_end(pe, s);
  h->launches++;
  CK(e);
  return ABFT_OK;
}

// K3 (lazy policy): a vectors + locate / correct of the layers K2 handed over
int launch_lazy(abft_stencil* h, const CheckParams& p, cudaStream_t s = nullptr) {
  on_dev(h);
  if (!s) s = h->stream;
  cudaEvent_t* pe = prof_begin(h, 2, s);
  cudaError_t e = launch_k3(h->cfg.dtype, h->shape, s, p);
  prof_end(pe, s);
  h->launches++;
  CK(e);
  return ABFT_OK;
}

int launch_check(abft_stencil* h, int uprev, int ucur, const double* Ap, const double* Bp,
                 double* Ac, double* Bc, double* PAo, double* PBo, double* zA, double* zB,
                 int flags, int64_t sweep) {
  return launch_check(h, make_check(h, uprev, ucur, Ap, Bp, Ac, Bc, PAo, PBo, zA, zB, flags, sweep));
}

// a checked sweep: K1 (step (1)) then K2 (steps (2)-(5))
int sweep_checked(abft_stencil* h, int src, int dst, double* A, double* B, const CheckParams& ck,
                  int64_t sweep) {
  int r = launch_k1(h, src, dst, A, B, K1_CK_AB, sweep);
  if (r) return r;
#ifdef ABFT_EXP_NO_K2  // experiment builds only (tools/exp_build.py): K1 cost in isolation
  return ABFT_OK;
#endif
  return launch_check(h, ck);
}

// ------------------------------------------------------------------ halos
// What crosses a slab face after a sweep: the boundary layer of field buffer
// `buf` plus the matching entries of one pair of per-layer vectors (a
// checksum generation or an offline prediction slot), SURVEY §8(e).
enum { XV_NONE = 0, XV_GEN = 1, XV_P = 2 };
struct XSpec {
  int buf, kind, idx;
};

void xvecs(abft_stencil* h, const XSpec& x, double** a, double** b) {
  *a = *b = nullptr;
  if (x.kind == XV_GEN) { *a = h->gA[x.idx]; *b = h->gB[x.idx]; }
  if (x.kind == XV_P) { *a = h->PA[x.idx]; *b = h->PB[x.idx]; }
}

// NCCL transport (one process per GPU): send / recv to rank -+ 1 in one group
// the z-slab halo plan of (rank, nranks, z_count): per face (0 = lower,
// 1 = upper) the peer rank, the buffer layer sent and the halo layer received
// (-1 when there is no neighbour) -- the plan paper_1909_00709_b200/dist.py
// states and tests with gloo
// Periodic z over several ranks closes the ring: rank 0's lower neighbour is
// the last rank and vice versa.
bool z_ring(const abft_config& c) { return c.bc == ABFT_BC_PERIODIC && c.nranks > 1; }
void halo_plan(const abft_config& c, int32_t plan[6]) {
  for (int side = 0; side < 2; ++side) {
    const bool has = z_ring(c) || (side == 0 ? c.rank > 0 : c.rank < c.nranks - 1);
    plan[3 * side + 0] = has ? (c.rank + (side == 0 ? -1 : 1) + c.nranks) % c.nranks : -1;
    plan[3 * side + 1] = has ? (side == 0 ? 1 : (int32_t)c.z_count) : -1;
    plan[3 * side + 2] = has ? (side == 0 ? 0 : (int32_t)c.z_count + 1) : -1;
  }
}

int exchange_nccl(abft_stencil* h, const XSpec& x) {
  NcclApi* n = nccl_api();
  if (!n) return ABFT_ENCCL;
  const ncclDataType_t dt = h->cfg.dtype == ABFT_F32 ? ncclFloat32 : ncclFloat64;
  const size_t lb = (size_t)h->L.plane, esz = h->L.esz;
  char* buf = h->fb[x.buf];
  double *va, *vb;
  xvecs(h, x, &va, &vb);
  const std::pair<double*, int64_t> vecs[2] = {{va, h->cfg.nx}, {vb, h->cfg.ny}};
  int32_t plan[6];
  halo_plan(h->cfg, plan);
  if (n->groupStart() != ncclSuccess) return ABFT_ENCCL;
  // sends / receives to one peer are matched in posting order: with a ring of
  // two ranks both faces face the same peer, so rank 1 posts its upper face
  // first (rank 0's lower-face send lands in rank 1's upper halo)
  const bool swap = z_ring(h->cfg) && h->cfg.nranks == 2 && h->cfg.rank == 1;
  for (int k = 0; k < 2; ++k) {
    const int side = swap ? 1 - k : k;
    const int peer = plan[3 * side];
    if (peer < 0) continue;
    const int64_t send_l = plan[3 * side + 1], recv_l = plan[3 * side + 2];
    n->send(buf + send_l * lb * esz, lb, dt, peer, h->comm, h->stream);
    n->recv(buf + recv_l * lb * esz, lb, dt, peer, h->comm, h->stream);
    for (const auto& v : vecs) {
      if (!v.first) continue;
      n->send(v.first + send_l * v.second, v.second, ncclFloat64, peer, h->comm, h->stream);
      n->recv(v.first + recv_l * v.second, v.second, ncclFloat64, peer, h->comm, h->stream);
    }
  }
  if (n->groupEnd() != ncclSuccess) return ABFT_ENCCL;
  return ABFT_OK;
}

// local transport (several slabs driven by one process, same or peer GPUs):
// every handle pulls its two halo layers from its neighbours with device
// copies, ordered by events across the handles' streams.
int exchange_local(Group& G, const XSpec& x) {
  for (abft_stencil* h : G) { on_dev(h); CK(cudaEventRecord(h->ev_ready, h->stream)); }
  for (abft_stencil* h : G) {
    on_dev(h);
    const size_t lb = (size_t)h->L.plane * h->L.esz;
    for (int side = 0; side < 2; ++side) {
      abft_stencil* q = side == 0 ? h->lo_peer : h->hi_peer;
      if (!q) continue;
      CK(cudaStreamWaitEvent(h->stream, q->ev_ready, 0));
      const int64_t src_l = side == 0 ? q->cfg.z_count : 1;
      const int64_t dst_l = side == 0 ? 0 : h->cfg.z_count + 1;
      CK(cudaMemcpyAsync(h->fb[x.buf] + dst_l * lb, q->fb[x.buf] + src_l * lb, lb, cudaMemcpyDefault,
                         h->stream));
      double *ha, *hb, *qa, *qb;
      xvecs(h, x, &ha, &hb);
      xvecs(q, x, &qa, &qb);
      if (ha) {
        const int64_t nx = h->cfg.nx, ny = h->cfg.ny;
        CK(cudaMemcpyAsync(ha + dst_l * nx, qa + src_l * nx, nx * 8, cudaMemcpyDefault, h->stream));
        CK(cudaMemcpyAsync(hb + dst_l * ny, qb + src_l * ny, ny * 8, cudaMemcpyDefault, h->stream));
      }
    }
    CK(cudaEventRecord(h->ev_pulled, h->stream));
  }
  // a neighbour may overwrite the layers we pulled only after our copies ran
  for (abft_stencil* h : G) {
    on_dev(h);
    for (abft_stencil* q : {h->lo_peer, h->hi_peer})
      if (q) CK(cudaStreamWaitEvent(h->stream, q->ev_pulled, 0));
  }
  return ABFT_OK;
}

// fused halo: the kernels already wrote every neighbour's halo; order the next
// sweep of each slab after this sweep of its neighbours
int sync_local(Group& G) {
  for (abft_stencil* h : G) { on_dev(h); CK(cudaEventRecord(h->ev_ready, h->stream)); }
  for (abft_stencil* h : G) {
    on_dev(h);
    for (abft_stencil* q : {h->lo_peer, h->hi_peer})
      if (q) CK(cudaStreamWaitEvent(h->stream, q->ev_ready, 0));
  }
  return ABFT_OK;
}

// what crosses the faces of this sweep, for the fused halo (set before launching)
void set_fwd(Group& G, const XSpec& x) {
  for (abft_stencil* h : G) {
    h->fwd_buf = h->fused ? x.buf : -1;
    h->fwd_kind = x.kind;
    h->fwd_idx = x.idx;
  }
}

// IPC transport (one process per slab): the kernels stored the halos into
// the neighbours' mapped buffers; order the next sweep of each slab after its
// neighbours' sweep.  Exchange #s records this rank's event of parity s,
// publishes s in its host-shared slot, waits until each neighbour published
// s and enqueues a wait on the neighbour's event of parity s.  A neighbour
// re-records that event only at exchange s + 2, which it reaches after this
// rank published s + 1 -- i.e. after the wait below was enqueued.
#define TRY(...)            \
  do {                      \
    int r_ = (__VA_ARGS__); \
    if (r_) return r_;      \
  } while (0)

// Wait until a neighbour's progress word reaches `want`.  A rank that died or
// never linked would leave the others spinning: give up after
// ABFT_IPC_TIMEOUT_S seconds (default 120) with ABFT_ETIMEOUT.
int ipc_wait(const volatile int64_t* word, int64_t want) {
  static const double limit = [] {
    const char* e = getenv("ABFT_IPC_TIMEOUT_S");
    return e ? atof(e) : 120.0;
  }();
  if (__atomic_load_n(word, __ATOMIC_ACQUIRE) >= want) return ABFT_OK;
  timespec t0, t;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (unsigned k = 0;; ++k) {
    if (__atomic_load_n(word, __ATOMIC_ACQUIRE) >= want) return ABFT_OK;
    if ((k & 1023) == 1023) {
      clock_gettime(CLOCK_MONOTONIC, &t);
      if ((t.tv_sec - t0.tv_sec) + 1e-9 * (t.tv_nsec - t0.tv_nsec) > limit) return ABFT_ETIMEOUT;
    }
    sched_yield();
  }
}

int sync_ipc(abft_stencil* h) {
  on_dev(h);
  const int64_t s = ++h->xseq;
  CK(cudaEventRecord(h->ev_ipc[s & 1], h->stream));
  __atomic_store_n(&h->shm[h->cfg.rank].seq, s, __ATOMIC_RELEASE);
  for (abft_stencil* q : {h->lo_peer, h->hi_peer}) {
    if (!q) continue;
    TRY(ipc_wait(&h->shm[q->cfg.rank].seq, s));
    CK(cudaStreamWaitEvent(h->stream, q->ev_ipc[s & 1], 0));
  }
  return ABFT_OK;
}

int halo_exchange(Group& G, const XSpec& x) {
  if (G.size() == 1 && G[0]->ipc) {
    G[0]->fwd_buf = -1;
    return sync_ipc(G[0]);
  }
  if (G.size() > 1 && G[0]->fused) {
    for (abft_stencil* h : G) h->fwd_buf = -1;
    return sync_local(G);
  }
  if (G.size() > 1) return exchange_local(G, x);
  abft_stencil* h = G[0];
  if (h->cfg.nranks == 1) return ABFT_OK;
  return exchange_nccl(h, x);
}

int zero_gen(abft_stencil* h, int g, int za = 0, int zb = -1);
// the buffer an online / unprotected sweep writes (three rotate on a
// pipelined handle, so u^{s-1} survives the next sweep)
int next_buf(const abft_stencil* h) { return h->nbuf == 3 ? (h->cur + 1) % 3 : 1 - h->cur; }
// K1 accumulates into generation g: clear it first unless it is known zero
int take_gen(abft_stencil* h, int g) {
  if (!((h->zmask >> g) & 1u)) {
    int r = zero_gen(h, g);
    if (r) return r;
  }
  h->zmask &= ~(1u << g);
  return ABFT_OK;
}

// the interior rows of a checksum generation, which K1 accumulates into; the
// halo rows belong to the neighbours' exchange (a fused neighbour may already
// have written them on its own stream)
int zero_gen(abft_stencil* h, int g, int za, int zb) {
  on_dev(h);
  const int64_t nx = h->cfg.nx, ny = h->cfg.ny;
  if (zb < 0) zb = (int)h->cfg.z_count;
  if (zb <= za) return ABFT_OK;
  CK(cudaMemsetAsync(h->gA[g] + (za + 1) * nx, 0, sizeof(double) * (zb - za) * nx, h->stream));
  CK(cudaMemsetAsync(h->gB[g] + (za + 1) * ny, 0, sizeof(double) * (zb - za) * ny, h->stream));
  return ABFT_OK;
}


// one online sweep s = sweeps + 1 of every slab of the group: K1 (sweep +
// actual checksums) then K2 (predict, compare, locate, correct, clear the
// generation of sweep s + 1), then the halo of the corrected layers
int online_sweep(Group& G) {
  abft_stencil* h0 = G[0];
  const int64_t s = h0->sweeps + 1;
  const int src = h0->cur, dst = next_buf(h0);
  const int gp = h0->gen, gn = (h0->gen + 1) % kGens, gz = (h0->gen + 2) % kGens;
  set_fwd(G, XSpec{dst, XV_GEN, gn});
  for (abft_stencil* h : G) {
    TRY(take_gen(h, gn));
    if (h->cfg.checksum_policy == ABFT_CK_LAZY) {
      // b in the pass; a (generations used as scratch) by K3 only
      // for layers whose b flagged
      TRY(launch_k1(h, src, dst, nullptr, h->gB[gn], K1_CK_B, s));
      CheckParams ck = make_check(h, src, dst, h->gA[gp], h->gB[gp], h->gA[gn], h->gB[gn], nullptr,
                                  nullptr, nullptr, h->gB[gz], CK_COMPARE | CK_CORRECT | CK_LAZY, s);
      ck.Aw = h->gA[gp];
      TRY(launch_check(h, ck));
      TRY(launch_lazy(h, ck));
      continue;
    }
    TRY(sweep_checked(h, src, dst, h->gA[gn], h->gB[gn],
                      make_check(h, src, dst, h->gA[gp], h->gB[gp], h->gA[gn], h->gB[gn], nullptr,
                                 nullptr, h->gA[gz], h->gB[gz], CK_COMPARE | CK_CORRECT, s),
                      s));
  }
  TRY(halo_exchange(G, XSpec{dst, XV_GEN, gn}));
  for (abft_stencil* h : G) {
    h->prev = src;
    h->cur = dst;
    h->gen_prev = gp;
    h->gen = gn;
    h->sweeps = s;
    h->zmask |= 1u << gz;  // K2 cleared the generation of sweep s + 1
  }
  return ABFT_OK;
}

// Pipelined online schedule (single slab, three field buffers):
// K1 of sweep s + 1 is launched right behind K1 of sweep s, and the checks of
// sweep s (K2, and K3 under LAZY) run beside it on the side stream.  They
// read u^{s-1} (the third buffer, which K1 of s + 1 does not write) and u^s,
// and K1 of s + 2 waits for them (it overwrites u^{s-1} and accumulates into
// the generation they cleared).  A cell of u^s the checks rewrite may already
// have been read by K1 of s + 1: the kernel that finishes the checks then
// recomputes the cells of u^{s+1} that read it (fix_next), so the result is
// bitwise the serial schedule's -- the paper's order -- while error-free
// sweeps never wait for a check.
int online_pipelined(abft_stencil* h, int32_t n) {
  on_dev(h);
  const bool lazy = h->cfg.checksum_policy == ABFT_CK_LAZY;
  for (int i = 0; i < n; ++i) {
    const int64_t s = h->sweeps + 1;
    const int src = h->cur, dst = (h->cur + 1) % 3;
    const int gp = h->gen, gn = (gp + 1) % kGens, g1 = (gp + 2) % kGens, g2 = (gp + 3) % kGens;
    TRY(take_gen(h, gn));
    // after the checks of sweep s - 2 (the previous call's are complete)
    if (i >= 2) CK(cudaStreamWaitEvent(h->stream, h->ev_chk[s & 1], 0));
    TRY(launch_k1(h, src, dst, lazy ? nullptr : h->gA[gn], h->gB[gn], lazy ? K1_CK_B : K1_CK_AB, s, 0, -1,
                  true));
    CK(cudaEventRecord(h->ev_k1, h->stream));
    CK(cudaStreamWaitEvent(h->s2, h->ev_k1, 0));
    // the checks of s clear the generation of sweep s + 2
    CheckParams ck = make_check(h, src, dst, h->gA[gp], h->gB[gp], h->gA[gn], h->gB[gn], nullptr, nullptr,
                                lazy ? nullptr : h->gA[g2], h->gB[g2],
                                CK_COMPARE | CK_CORRECT | (lazy ? CK_LAZY : 0), s);
    if (lazy) ck.Aw = h->gA[gp];
    ck.k1_reset = 1;
    if (i + 1 < n) {   // K1 of s + 1 will be in flight beside these checks
      const int nb = (dst + 1) % 3;
      ck.fix = 1;
      ck.k1_target = (unsigned)k1_grid_ctas(h);
      ck.unext = h->fb[nb];
      ck.Anext = lazy ? nullptr : h->gA[g1];
      ck.Bnext = h->gB[g1];
      ck.EXnext = h->EX[nb];
      ck.nfn = sweep_faults(h, s + 1, ck.fn, false);
    }
    TRY(launch_check(h, ck, h->s2));
    if (lazy) TRY(launch_lazy(h, ck, h->s2));
    CK(cudaEventRecord(h->ev_chk[s & 1], h->s2));
    h->zmask |= 1u << g2;
    h->prev = src;
    h->cur = dst;
    h->gen_prev = gp;
    h->gen = gn;
    h->sweeps = s;
  }
  // the caller's stream orders everything after the last check
  if (n > 0) CK(cudaStreamWaitEvent(h->stream, h->ev_chk[h->sweeps & 1], 0));
  return ABFT_OK;
}

int none_sweep(Group& G) {
  abft_stencil* h0 = G[0];
  const int64_t s = h0->sweeps + 1;
  const int src = h0->cur, dst = 1 - h0->cur;
  set_fwd(G, XSpec{dst, XV_NONE, 0});
  for (abft_stencil* h : G) TRY(launch_k1(h, src, dst, nullptr, nullptr, K1_CK_NONE, s));
  TRY(halo_exchange(G, XSpec{dst, XV_NONE, 0}));
  for (abft_stencil* h : G) {
    h->prev = src;
    h->cur = dst;
    h->sweeps = s;
  }
  return ABFT_OK;
}

// IPC transport: the window verdict (dirty, extent) is max-reduced over every
// rank through the host-shared slots.  Window w's values go to parity w & 1
// once every rank has reduced window w - 2 (nobody still reads that parity).
int read_dirty_ipc(abft_stencil* h, int* dirty, int64_t* zmin, int64_t* zmax, std::vector<uint8_t>* F) {
  on_dev(h);
  int d[3] = {0, 0, 0};
  CK(cudaMemcpyAsync(d, &h->st->dirty, sizeof(d), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const int64_t w = ++h->wseq;
  const int n = h->cfg.nranks, me = h->cfg.rank, par = (int)(w & 1);
  for (int r = 0; r < n; ++r)
    TRY(ipc_wait(&h->shm[r].wdone, w - 2));
  if (F) {
    // this slab's flagged layers as bits (bit z - z_begin), beside the verdict
    const int64_t zc = h->cfg.z_count, zb = h->cfg.z_begin;
    uint32_t* bits = h->shm[me].zbits[par];
    for (int64_t i = 0; i < (zc + 31) / 32; ++i) bits[i] = 0;
    if (d[0] > 0) {
      std::vector<int> own((size_t)zc);
      CK(cudaMemcpyAsync(own.data(), h->zflag + zb, sizeof(int) * (size_t)zc, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      for (int64_t i = 0; i < zc; ++i)
        if (own[(size_t)i]) bits[i >> 5] |= 1u << (i & 31);
    }
    F->assign((size_t)h->cfg.nz_global, 0);
  }
  for (int k = 0; k < 3; ++k) h->shm[me].val[par][k] = d[k];
  __atomic_store_n(&h->shm[me].wseq, w, __ATOMIC_RELEASE);
  int m[3] = {0, 0, 0};
  for (int r = 0; r < n; ++r) {
    TRY(ipc_wait(&h->shm[r].wseq, w));
    for (int k = 0; k < 3; ++k) m[k] = std::max(m[k], h->shm[r].val[par][k]);
    if (F && h->shm[r].val[par][0] > 0) {
      const int64_t zb = h->shm[r].z_begin, zc = h->shm[r].z_count;
      for (int64_t i = 0; i < zc; ++i)
        if (h->shm[r].zbits[par][i >> 5] >> (i & 31) & 1u) (*F)[(size_t)(zb + i)] = 1;
    }
  }
  __atomic_store_n(&h->shm[me].wdone, w, __ATOMIC_RELEASE);
  *dirty = m[0];
  *zmin = 0x7fffffffLL - m[1];
  *zmax = (int64_t)m[2] - 1;
  return ABFT_OK;
}

// the last window check over every slab of the job: flagged layers (> 0:
// dirty) and the global extent [zmin, zmax] of the flagged layers
int read_dirty(Group& G, int* dirty, int64_t* zmin, int64_t* zmax, std::vector<uint8_t>* F) {
  *dirty = 0;
  int ext[2] = {0, 0};
  if (G.size() == 1 && G[0]->ipc) return read_dirty_ipc(G[0], dirty, zmin, zmax, F);
  for (abft_stencil* h : G) {
    on_dev(h);
    if (G.size() == 1 && h->cfg.nranks > 1) {
      // dirty, zext[0], zext[1] are adjacent ints: one max-reduction (a
      // count's maximum is nonzero iff any rank's is)
      NcclApi* n = nccl_api();
      if (!n) return ABFT_ENCCL;
      if (n->allReduce(&h->st->dirty, &h->st->dirty, 3, ncclInt32, ncclMax, h->comm, h->stream) !=
          ncclSuccess)
        return ABFT_ENCCL;
    }
    int d[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(d, &h->st->dirty, sizeof(d), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    *dirty += d[0];
    ext[0] = std::max(ext[0], d[1]);
    ext[1] = std::max(ext[1], d[2]);
  }
  *zmin = 0x7fffffffLL - ext[0];
  *zmax = (int64_t)ext[1] - 1;
  return ABFT_OK;
}

// the global layers the last window check flagged, over every slab of the
// job (partial re-execution, Q28): each slab's check marked its own layers in
// its zflag array (indexed by global layer).  NCCL ranks max-reduce the array
// in place; the IPC transport carries the marks with the verdict instead
// (read_dirty_ipc).  Called by every rank once the verdict is dirty.
int read_flagged(Group& G, std::vector<uint8_t>* F) {
  const int64_t nzg = G[0]->cfg.nz_global;
  F->assign((size_t)nzg, 0);
  std::vector<int> w((size_t)nzg);
  for (abft_stencil* h : G) {
    on_dev(h);
    int64_t z0 = h->cfg.z_begin, n = h->cfg.z_count;
    if (G.size() == 1 && h->cfg.nranks > 1) {
      NcclApi* a = nccl_api();
      if (!a) return ABFT_ENCCL;
      if (a->allReduce(h->zflag, h->zflag, (size_t)nzg, ncclInt32, ncclMax, h->comm, h->stream) != ncclSuccess)
        return ABFT_ENCCL;
      z0 = 0;
      n = nzg;
    }
    CK(cudaMemcpyAsync(w.data() + z0, h->zflag + z0, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (int64_t z = z0; z < z0 + n; ++z)
      if (w[(size_t)z]) (*F)[(size_t)z] = 1;
  }
  return ABFT_OK;
}

using ZRanges = std::vector<std::pair<int64_t, int64_t>>;
// the ranges, each widened by m layers, clipped to the domain and merged
// where they touch (ascending, disjoint)
ZRanges widen(const ZRanges& R, int64_t m, int64_t nzg) {
  ZRanges out;
  for (const auto& r : R) {
    const int64_t lo = std::max<int64_t>(0, r.first - m), hi = std::min<int64_t>(nzg - 1, r.second + m);
    if (!out.empty() && lo <= out.back().second + 1) out.back().second = std::max(out.back().second, hi);
    else out.push_back({lo, hi});
  }
  return out;
}

// Partial re-execution of a dirty window of L sweeps (recovery PARTIAL,
// P:107-108, Q28): only the global layers of R (ascending
// disjoint ranges: the layers within 2 (L - 1) of a flagged one) are
// recomputed from the checkpoint.  Sweep k re-executes the light cones of
// those ranges -- each widened by L - k layers, merged where they meet --
// reading sweep k - 1's cones; the cones of sweep k < L go to the two
// buffers other than `last` (the first execution's result), ping-pong -- the
// checkpoint is read by sweep 1 only -- and sweep L writes the ranges into
// `last`, whose other layers keep the first execution.  The predictions P
// are re-advanced over the same cones, the actual checksums of the ranges
// recomputed and compared.
int partial_window(Group& G, int L, const ZRanges& R, int ck, int last, int ckgen, int gend, int64_t s0) {
  int other = 0;
  while (other == ck || other == last) ++other;
  int src = ck;
  for (int k = 1; k <= L; ++k) {
    const int64_t s = s0 + k;
    const bool end = k == L;
    const int dst = end ? last : (src == ck ? other : ck);
    const ZRanges cones = widen(R, L - k, G[0]->cfg.nz_global);
    set_fwd(G, end ? XSpec{dst, XV_GEN, gend} : XSpec{dst, XV_P, k & 1});
    for (abft_stencil* h : G) {
      const int64_t zb0 = h->cfg.z_begin;
      const double* pA = k == 1 ? h->gA[ckgen] : h->PA[(k - 1) & 1];
      const double* pB = k == 1 ? h->gB[ckgen] : h->PB[(k - 1) & 1];
      const bool bonly = h->cfg.checksum_policy == ABFT_CK_LAZY;   // Q29
      const int64_t executed0 = h->executed;
      for (const auto& cone : cones) {
        const int za = (int)std::max<int64_t>(0, cone.first - zb0);
        const int zb = (int)std::min<int64_t>(h->cfg.z_count, cone.second - zb0 + 1);
        if (za >= zb) continue;   // the cone misses this slab
        CheckParams c;
        if (!end) {
          TRY(launch_k1(h, src, dst, nullptr, nullptr, K1_CK_NONE, s, za, zb));
          c = make_check(h, src, dst, pA, pB, nullptr, nullptr, h->PA[k & 1], h->PB[k & 1], nullptr,
                         nullptr, CK_STORE_PRED | (bonly ? CK_BONLY : 0), s);
        } else {
          TRY(zero_gen(h, gend, za, zb));
          TRY(launch_k1(h, src, dst, bonly ? nullptr : h->gA[gend], h->gB[gend], bonly ? K1_CK_B : K1_CK_AB, s,
                        za, zb));
          c = make_check(h, src, dst, pA, pB, h->gA[gend], h->gB[gend], nullptr, nullptr, nullptr,
                         nullptr, CK_COMPARE | CK_OFFLINE_END | CK_PERSIST | (bonly ? CK_BONLY : 0), s);
        }
        c.zr0 = za;
        c.zr1 = zb;
        TRY(launch_check(h, c));
      }
      h->executed = executed0 + 1;   // one sweep, whatever the number of cones
    }
    TRY(halo_exchange(G, end ? XSpec{dst, XV_GEN, gend} : XSpec{dst, XV_P, k & 1}));
    for (abft_stencil* h : G) h->sweeps = s;
    src = dst;
  }
  return ABFT_OK;
}

// Offline ABFT (Section IV): one window of L sweeps starting from
// the checkpoint (current buffer + its actual checksums), the prediction
// vectors advanced once per sweep (Q17), compared at the window end; on
// mismatch -- anywhere in the job -- every slab recomputes the window from
// its checkpoint (rotation of three field buffers: no copy), or only the
// light cone of the flagged layers (recovery PARTIAL); a second mismatch is a
// persistent error.
// sweep 1 of the window after this one, run while the host waits for this
// window's verdict (single slab): from this window's result `last` into the
// buffer that is neither `last` nor this window's checkpoint `ck`, predicting
// from this window's actual checksums into slot 1 -- exactly what the next
// window's first sweep does, so the next window adopts it (the buffer order
// below makes that sweep write the same buffer).  No flip may be scheduled in
// it (a dropped speculation would have consumed it).
bool spec_allowed(const abft_stencil* h, int64_t s) {
  if (!h->spec_on || h->cfg.nranks != 1 || h->grouped || h->ipc || h->prof) return false;
  for (const PendingFault& pf : h->faults)
    if (!pf.fired && pf.f.sweep == s) return false;
  return true;
}
int spec_sweep(abft_stencil* h, int ck, int last, int gend, int64_t s) {
  const int x = 3 - ck - last;
  const int bf = h->cfg.checksum_policy == ABFT_CK_LAZY ? CK_BONLY : 0;
  TRY(launch_k1(h, last, x, nullptr, nullptr, K1_CK_NONE, s));
  TRY(launch_check(h, last, x, h->gA[gend], h->gB[gend], nullptr, nullptr, h->PA[1], h->PB[1], nullptr,
                   nullptr, CK_STORE_PRED | bf, s));
  return ABFT_OK;
}
// the window verdict of a single slab: copied to pinned memory behind the
// window's check, then (after the caller enqueued more work) waited for
int verdict_post(abft_stencil* h) {
  on_dev(h);
  if (!h->pin_dirty) CK(cudaHostAlloc(reinterpret_cast<void**>(&h->pin_dirty), 4 * sizeof(int), cudaHostAllocDefault));
  if (!h->ev_verdict) CK(cudaEventCreateWithFlags(&h->ev_verdict, cudaEventDisableTiming));
  CK(cudaMemcpyAsync(h->pin_dirty, &h->st->dirty, 3 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaEventRecord(h->ev_verdict, h->stream));
  return ABFT_OK;
}
int verdict_wait(abft_stencil* h, int* dirty, int64_t* zmin, int64_t* zmax) {
  CK(cudaEventSynchronize(h->ev_verdict));
  *dirty = h->pin_dirty[0];
  *zmin = 0x7fffffffLL - h->pin_dirty[1];
  *zmax = (int64_t)h->pin_dirty[2] - 1;
  return ABFT_OK;
}

int offline_window(Group& G, int L, bool spec_next) {
  abft_stencil* h0 = G[0];
  const int ck = h0->cur, ckgen = h0->gen, gend = (h0->gen + 1) % kGens;
  const int64_t s0 = h0->sweeps;
  const bool partial = h0->cfg.recovery == ABFT_RECOVER_PARTIAL;
  // the two buffers besides the checkpoint, the one that is not the previous
  // window's checkpoint first (a speculative first sweep wrote it, see above)
  int others[2], k = 0;
  for (int b = 0; b < 3; ++b)
    if (b != ck && b != h0->prev) others[k++] = b;
  for (int b = 0; b < 3; ++b)
    if (b != ck && b == h0->prev) others[k++] = b;
  if (k != 2) {   // prev == ck (first window after init): plain order
    k = 0;
    for (int b = 0; b < 3; ++b)
      if (b != ck) others[k++] = b;
  }
  const bool adopt = h0->spec_done;   // sweep 1 already ran (previous window's speculation)
  h0->spec_done = false;
  const bool single = G.size() == 1 && h0->cfg.nranks == 1;
  int last = ck;
  int worst = ABFT_OK;
  ZRanges redo;
  std::vector<uint8_t> flagged;
  for (int attempt = 0; attempt < 2; ++attempt) {
    for (abft_stencil* h : G) {
      on_dev(h);
      CK(cudaMemsetAsync(&h->st->dirty, 0, 3 * sizeof(int), h->stream));
      if (partial && attempt == 0) CK(cudaMemsetAsync(h->zflag, 0, sizeof(int) * (size_t)h->cfg.nz_global, h->stream));
    }
    if (attempt == 1 && partial) {
      TRY(partial_window(G, L, redo, ck, last, ckgen, gend, s0));
    } else {
      int src = ck;
      for (int t = 1; t <= L; ++t) {
        const int64_t s = s0 + t;
        const int dst = (src == others[0]) ? others[1] : others[0];
        const bool end = (t == L);
        set_fwd(G, end ? XSpec{dst, XV_GEN, gend} : XSpec{dst, XV_P, t & 1});
        // P^{t-1}: the checkpoint's actual checksums for t = 1, else slot (t-1)&1
        for (abft_stencil* h : G) {
          const double* pA = t == 1 ? h->gA[ckgen] : h->PA[(t - 1) & 1];
          const double* pB = t == 1 ? h->gB[ckgen] : h->PB[(t - 1) & 1];
          // policy LAZY offline (Q29): b predicted, summed and compared alone
          const bool bonly = h->cfg.checksum_policy == ABFT_CK_LAZY;
          const int bf = bonly ? CK_BONLY : 0;
          if (!end) {
            if (!(adopt && attempt == 0 && t == 1)) {
              TRY(launch_k1(h, src, dst, nullptr, nullptr, K1_CK_NONE, s));
              TRY(launch_check(h, src, dst, pA, pB, nullptr, nullptr, h->PA[t & 1], h->PB[t & 1],
                               nullptr, nullptr, CK_STORE_PRED | bf, s));
            }
          } else {
            TRY(zero_gen(h, gend));
            TRY(launch_k1(h, src, dst, bonly ? nullptr : h->gA[gend], h->gB[gend], bonly ? K1_CK_B : K1_CK_AB,
                          s));
            TRY(launch_check(h, make_check(h, src, dst, pA, pB, h->gA[gend], h->gB[gend], nullptr, nullptr,
                                           nullptr, nullptr,
                                           CK_COMPARE | CK_OFFLINE_END | (attempt ? CK_PERSIST : 0) | bf, s)));
          }
        }
        TRY(halo_exchange(G, end ? XSpec{dst, XV_GEN, gend} : XSpec{dst, XV_P, t & 1}));
        for (abft_stencil* h : G) h->sweeps = s;
        src = dst;
      }
      last = src;
    }
    int dirty = 0;
    int64_t zmin = 0, zmax = 0;
    const bool spec = single && spec_next && attempt == 0 && spec_allowed(h0, s0 + L + 1);
    if (single) {
      TRY(verdict_post(h0));
      if (spec) TRY(spec_sweep(h0, ck, last, gend, s0 + L + 1));
      TRY(verdict_wait(h0, &dirty, &zmin, &zmax));
    } else {
      TRY(read_dirty(G, &dirty, &zmin, &zmax, partial && attempt == 0 ? &flagged : nullptr));
    }
    for (abft_stencil* h : G) h->windows++;
    if (!dirty) {
      h0->spec_done = spec;
      break;
    }
    if (spec) h0->executed--;   // the speculative sweep is dropped (it ran on a dirty result)
    if (attempt == 0 && partial) {
      // layers a partial recovery re-executes: every layer an error of this
      // window that was flagged can have reached -- within 2 (L - 1) layers
      // of a flagged one (Q28)
      if (!(G.size() == 1 && h0->ipc)) TRY(read_flagged(G, &flagged));
      const int64_t nzg = h0->cfg.nz_global, r = 2 * (L - 1);
      ZRanges fl;
      for (int64_t z = 0; z < nzg; ++z)
        if (flagged[(size_t)z]) fl.push_back({z, z});
      redo = widen(fl, r, nzg);
      // periodic z: a reach past a face wraps to the far layers -- take them all
      if (h0->cfg.bc == ABFT_BC_PERIODIC && (zmin - r < 0 || zmax + r > nzg - 1)) redo = {{0, nzg - 1}};
    }
    for (abft_stencil* h : G) {
      if (attempt == 0) {
        h->rollbacks++;  // rollback to the checkpoint, recompute
        h->sweeps = s0;
      } else {
        h->persistent++;
        h->host_worst = 3;
        worst = ABFT_PERSISTENT_ERROR;
      }
    }
  }
  for (abft_stencil* h : G) {
    h->prev = ck;
    h->cur = last;
    h->gen_prev = ckgen;
    h->gen = gend;
    h->zmask &= ~(1u << gend);
  }
  return worst;
}

int clear_summaries(abft_stencil* h) {
  if (h->summ_dirty) {
    on_dev(h);
    CK(cudaMemsetAsync(h->summ, 0, sizeof(LayerSummary) * h->cfg.z_count, h->stream));
    h->summ_dirty = false;
  }
  return ABFT_OK;
}

// ---------------------------------------------------------- step graphs
// a step of this handle that may run as a captured graph: one slab, the
// pipelined online schedule or unprotected sweeps, no flip scheduled in the
// range (flips change the launch parameters; those calls enqueue directly)
bool graph_eligible(const abft_stencil* h, int32_t n) {
  if (!h->graphs_on || h->prof || n < 1 || h->grouped || h->ipc || h->cfg.nranks != 1) return false;
  if (h->cfg.mode == ABFT_MODE_OFFLINE) return false;   // one host verdict per window
  for (const PendingFault& pf : h->faults)
    if (!pf.fired && pf.f.sweep > h->sweeps && pf.f.sweep <= h->sweeps + n + 1) return false;
  return true;
}

StepGraph* graph_find(abft_stencil* h, int32_t n) {
  for (StepGraph& g : h->graphs)
    if (g.n == n && g.cur == h->cur && g.gen == h->gen && g.par == (int)(h->sweeps & 1) && g.zmask == h->zmask)
      return &g;
  return nullptr;
}

int run_direct(abft_stencil* h, int32_t n);

// the sweep-offset memset node on stream st (inside a capture)
int offset_node(abft_stencil* h, cudaStream_t st, cudaGraphNode_t* out) {
  cudaStreamCaptureStatus cst;
  cudaGraph_t cg;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(st, &cst, nullptr, &cg, &deps, &nd));
  cudaMemsetParams mp = {};
  mp.dst = &h->st->sweep_off;
  mp.value = 0;
  mp.elementSize = 4;
  mp.width = 1;
  mp.height = 1;
  mp.pitch = 4;
  CK(cudaGraphAddMemsetNode(out, cg, deps, nd, &mp));
  CK(cudaStreamUpdateCaptureDependencies(st, out, 1, cudaStreamSetCaptureDependencies));
  return ABFT_OK;
}

// capture step(n) from the current state (which is left unchanged)
int graph_capture(abft_stencil* h, int32_t n, StepGraph** out) {
  on_dev(h);
  if (!h->cs && cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking) != cudaSuccess) return ABFT_ECUDA;
  StepGraph g;
  g.n = n; g.cur = h->cur; g.gen = h->gen; g.par = (int)(h->sweeps & 1); g.zmask = h->zmask;
  g.sweeps0 = h->sweeps;
  const int prev0 = h->prev, gen_prev0 = h->gen_prev;
  const int64_t sweeps0 = h->sweeps, executed0 = h->executed, launches0 = h->launches;
  cudaStream_t user = h->stream;
  h->stream = h->cs;
  cudaGraph_t graph = nullptr;
  int r = ABFT_OK;
  if (cudaStreamBeginCapture(h->cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) r = ABFT_ECUDA;
  if (r == ABFT_OK && h->pipe) {   // records of this graph's checks: sweep numbers offset per replay
    if (cudaEventRecord(h->ev_k1, h->cs) != cudaSuccess || cudaStreamWaitEvent(h->s2, h->ev_k1, 0) != cudaSuccess)
      r = ABFT_ECUDA;
    if (r == ABFT_OK) r = offset_node(h, h->s2, &g.off);
  } else if (r == ABFT_OK && h->cfg.mode == ABFT_MODE_ONLINE) {
    r = offset_node(h, h->cs, &g.off);
  }
  if (r == ABFT_OK) r = run_direct(h, n);
  if (r == ABFT_OK && h->pipe) {   // back to 0 for calls enqueued directly
    cudaGraphNode_t z;
    if (cudaStreamWaitEvent(h->s2, h->ev_chk[h->sweeps & 1], 0) != cudaSuccess) r = ABFT_ECUDA;
    if (r == ABFT_OK) r = offset_node(h, h->s2, &z);
    if (r == ABFT_OK && (cudaEventRecord(h->ev_k1, h->s2) != cudaSuccess ||
                         cudaStreamWaitEvent(h->cs, h->ev_k1, 0) != cudaSuccess))
      r = ABFT_ECUDA;
  } else if (r == ABFT_OK && h->cfg.mode == ABFT_MODE_ONLINE) {
    cudaGraphNode_t z;
    r = offset_node(h, h->cs, &z);
  }
  const cudaError_t ee = cudaStreamEndCapture(h->cs, &graph);
  if (r == ABFT_OK && ee != cudaSuccess) r = ABFT_ECUDA;
  if (r == ABFT_OK) {
    cudaGraphExec_t ex = nullptr;
    if (cudaGraphInstantiate(&ex, graph, 0) != cudaSuccess) r = ABFT_ECUDA;
    g.exec = ex;
    // the device-side copy of the graph now, not at its first launch
    if (r == ABFT_OK && cudaGraphUpload(ex, user) != cudaSuccess) r = ABFT_ECUDA;
  }
  g.graph = graph;
  g.cur2 = h->cur; g.prev2 = h->prev; g.gen2 = h->gen; g.gen_prev2 = h->gen_prev; g.zmask2 = h->zmask;
  g.launches = h->launches - launches0;
  // the state as before: the graph runs when launched
  h->stream = user;
  h->cur = g.cur; h->prev = prev0; h->gen = g.gen; h->gen_prev = gen_prev0; h->zmask = g.zmask;
  h->sweeps = sweeps0; h->executed = executed0; h->launches = launches0;
  if (r != ABFT_OK) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    cudaGetLastError();
    return r;
  }
  if (h->graphs.size() >= kMaxGraphs) {   // evict the least recently used
    size_t v = 0;
    for (size_t i = 1; i < h->graphs.size(); ++i)
      if (h->graphs[i].used < h->graphs[v].used) v = i;
    cudaGraphExecDestroy(h->graphs[v].exec);
    cudaGraphDestroy(h->graphs[v].graph);
    h->graphs.erase(h->graphs.begin() + v);
  }
  g.used = ++h->graph_tick;
  h->graphs.push_back(g);
  *out = &h->graphs.back();
  return ABFT_OK;
}

int graph_launch(abft_stencil* h, StepGraph* g) {
  on_dev(h);
  if (g->off) {
    cudaMemsetParams mp = {};
    mp.dst = &h->st->sweep_off;
    mp.value = (unsigned)(h->sweeps - g->sweeps0);
    mp.elementSize = 4;
    mp.width = 1;
    mp.height = 1;
    mp.pitch = 4;
    CK(cudaGraphExecMemsetNodeSetParams(g->exec, g->off, &mp));
  }
  CK(cudaGraphLaunch(g->exec, h->stream));
  g->used = ++h->graph_tick;
  h->cur = g->cur2; h->prev = g->prev2; h->gen = g->gen2; h->gen_prev = g->gen_prev2; h->zmask = g->zmask2;
  h->sweeps += g->n;
  h->executed += g->n;
  h->launches += g->launches;
  return ABFT_OK;
}

// online (pipelined or serial) or unprotected sweeps of one slab, enqueued directly
int run_direct(abft_stencil* h, int32_t n) {
  if (h->cfg.mode == ABFT_MODE_ONLINE && h->pipe) return online_pipelined(h, n);
  Group G{h};
  for (int i = 0; i < n; ++i) TRY(h->cfg.mode == ABFT_MODE_ONLINE ? online_sweep(G) : none_sweep(G));
  return ABFT_OK;
}

int step_group(Group& G, int32_t n) {
  for (abft_stencil* h : G) {
    h->pending_check = false;
    TRY(clear_summaries(h));
  }
  const int mode = G[0]->cfg.mode;
  if (mode == ABFT_MODE_OFFLINE) {
    int worst = ABFT_OK;
    while (n > 0) {
      const int L = std::min<int>(n, G[0]->cfg.delta);
      // the next window's first sweep may run while this window's verdict
      // is read back when that window has an in-window sweep (length >= 2)
      int r = offline_window(G, L, n - L >= 2 && G[0]->cfg.delta >= 2);
      if (r < 0) return r;
      worst = std::max(worst, r);
      n -= L;
    }
    return worst;
  }
  if (G.size() == 1 && graph_eligible(G[0], n)) {
    abft_stencil* h = G[0];
    StepGraph* g = graph_find(h, n);
    if (!g) TRY(graph_capture(h, n, &g));
    return graph_launch(h, g);
  }
  if (mode == ABFT_MODE_ONLINE && G.size() == 1 && G[0]->pipe) return online_pipelined(G[0], n);
  for (int i = 0; i < n; ++i) TRY(mode == ABFT_MODE_ONLINE ? online_sweep(G) : none_sweep(G));
  return ABFT_OK;
}

// ---------------------------------------------------------------- IPC
// What a rank shares with its neighbours (abft_stencil_ipc_export): IPC
// handles of its field buffers and aux workspace (each with the offset of the
// handle's buffer in its allocation), the aux layout, and its two IPC events.
struct IpcBlob {
  uint32_t magic, version;
  int32_t rank, nranks, nbuf, pad;
  int64_t nx, ny, z_count, z_begin, plane, esz;
  cudaIpcMemHandle_t mem[4];   // field buffers 0..2, aux
  uint64_t off[4];
  uint64_t off_gA[kGens], off_gB[kGens], off_PA[2], off_PB[2];
  cudaIpcEventHandle_t ev[2];
};
static_assert(sizeof(IpcBlob) <= ABFT_IPC_BLOB_BYTES, "blob size");
constexpr uint32_t kIpcMagic = 0xAB5F1C01u;

typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<AddrRangeFn>(p);
  }
  return fn;
}

// the allocation containing ptr: IPC handle + offset of ptr in it
int ipc_handle(const void* ptr, cudaIpcMemHandle_t* hd, uint64_t* off) {
  AddrRangeFn fn = addr_range_fn();
  if (!fn) return ABFT_ECUDA;
  CUdeviceptr base = 0;
  size_t sz = 0;
  if (fn(&base, &sz, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return ABFT_ECUDA;
  CK(cudaIpcGetMemHandle(hd, reinterpret_cast<void*>(base)));
  *off = reinterpret_cast<uintptr_t>(ptr) - base;
  return ABFT_OK;
}

// map a neighbour's allocation once per process (an allocation may hold
// several of its buffers)
int ipc_open(abft_stencil* h, std::vector<std::pair<cudaIpcMemHandle_t, char*>>& seen,
             const cudaIpcMemHandle_t& hd, char** base) {
  for (auto& e : seen)
    if (!memcmp(&e.first, &hd, sizeof(hd))) { *base = e.second; return ABFT_OK; }
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
  h->ipc_opened.push_back(p);
  seen.push_back({hd, static_cast<char*>(p)});
  *base = static_cast<char*>(p);
  return ABFT_OK;
}

void ipc_unlink(abft_stencil* h) {
  if (h->proxy[1] == h->proxy[0]) h->proxy[1] = nullptr;
  for (int f = 0; f < 2; ++f) {
    abft_stencil* q = h->proxy[f];
    if (!q) continue;
    for (auto e : q->ev_ipc)
      if (e) cudaEventDestroy(e);
    delete q;
    h->proxy[f] = nullptr;
  }
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  h->ipc_opened.clear();
  for (auto e : h->ev_ipc)
    if (e) cudaEventDestroy(e);
  h->ev_ipc[0] = h->ev_ipc[1] = nullptr;
  if (h->ipc) { h->lo_peer = h->hi_peer = nullptr; h->ipc = false; h->fused = false; }
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int abft_stencil_halo_plan(const abft_config* cfg, int32_t plan[6]) {
  if (!plan) return ABFT_EINVAL;
  const int v = validate(cfg);
  if (v) return v;
  halo_plan(*cfg, plan);
  return ABFT_OK;
}

const char* abft_strerror(int s) {
  switch (s) {
    case ABFT_OK: return "ok";
    case ABFT_DETECTED_UNCORRECTABLE: return "detected, not corrected";
    case ABFT_PERSISTENT_ERROR: return "persistent error after rollback";
    case ABFT_EINVAL: return "invalid argument";
    case ABFT_ENOSPACE: return "workspace too small";
    case ABFT_ECUDA: return "CUDA error";
    case ABFT_ENCCL: return "NCCL error";
    case ABFT_EUNSUPPORTED: return "unsupported by this build";
    case ABFT_ETIMEOUT: return "timed out waiting for a neighbour rank (IPC)";
    default: return "unknown status";
  }
}

int abft_stencil_field_buffers(const abft_config* cfg, int32_t* n) {
  if (!n) return ABFT_EINVAL;
  const int v = validate(cfg);
  if (v) return v;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return ABFT_ECUDA;
  *n = (cfg->mode == ABFT_MODE_OFFLINE || k1_plan(cfg, dev).pipe) ? 3 : 2;
  return ABFT_OK;
}

int abft_stencil_workspace_size(const abft_config* cfg, size_t* field_bytes, size_t* aux_bytes) {
  int v = validate(cfg);
  if (v) return v;
  Layout L = layout(cfg);
  if (field_bytes) *field_bytes = L.field_bytes;
  if (aux_bytes) *aux_bytes = L.aux_bytes;
  return ABFT_OK;
}

int abft_stencil_init(const abft_config* cfg, void* const field_bufs[3], void* aux, const void* u0,
                      void* stream, abft_stencil** out) {
  if (!out || !field_bufs || !aux || !u0) return ABFT_EINVAL;
  *out = nullptr;
  int v = validate(cfg);
  if (v) return v;
  abft_stencil* h = new abft_stencil();
  h->cfg = *cfg;
  h->points.assign(cfg->points, cfg->points + cfg->npoints);
  h->sources.assign(cfg->sources, cfg->sources + cfg->nsources);
  h->cfg.points = h->points.data();
  h->cfg.sources = h->sources.data();
  h->L = layout(cfg);
  {
    int dev0 = 0;
    if (cudaGetDevice(&dev0) != cudaSuccess) { delete h; return ABFT_ECUDA; }
    h->pipe = field_bufs[2] && k1_plan(cfg, dev0).pipe;
  }
  h->nbuf = (cfg->mode == ABFT_MODE_OFFLINE || h->pipe) ? 3 : 2;
  for (int b = 0; b < h->nbuf; ++b) {
    if (!field_bufs[b]) { delete h; return ABFT_EINVAL; }
    h->fb[b] = static_cast<char*>(field_bufs[b]);
  }
  h->aux = static_cast<char*>(aux);
  h->stream = static_cast<cudaStream_t>(stream);
  const Layout& L = h->L;
  for (int g = 0; g < kGens; ++g) {
    h->gA[g] = reinterpret_cast<double*>(h->aux + L.off_gA[g]);
    h->gB[g] = reinterpret_cast<double*>(h->aux + L.off_gB[g]);
  }
  for (int g = 0; g < 2; ++g) {
    h->PA[g] = reinterpret_cast<double*>(h->aux + L.off_PA[g]);
    h->PB[g] = reinterpret_cast<double*>(h->aux + L.off_PB[g]);
  }
  h->cA = reinterpret_cast<double*>(h->aux + L.off_cA);
  h->cB = reinterpret_cast<double*>(h->aux + L.off_cB);
  h->summ = reinterpret_cast<LayerSummary*>(h->aux + L.off_summ);
  h->lazy_list = reinterpret_cast<int*>(h->aux + L.off_lazy);
  h->lazy_rowlist = h->lazy_list + cfg->z_count;
  h->lazy_mark = h->lazy_rowlist + 2 * (cfg->z_count + 2);
  for (int b = 0; b < 3; ++b) h->EX[b] = h->aux + L.off_EX[b];
  h->st = reinterpret_cast<DevState*>(h->aux + L.off_st);
  h->zflag = reinterpret_cast<int*>(h->aux + L.off_zflag);
  h->has_lo = z_ring(*cfg) || cfg->rank > 0;
  h->has_hi = z_ring(*cfg) || cfg->rank < cfg->nranks - 1;
  const int64_t nx = cfg->nx, ny = cfg->ny, zc = cfg->z_count;
  const int esz = L.esz;
  auto fail = [&](int code) { delete h; return code; };
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(ABFT_ECUDA);
  h->dev = dev;
  if (!encode_fn()) return fail(ABFT_ECUDA);

  // field: u0 (host or device, dense) -> buffer 0 layers 1..zc (padded pitch)
  if (cudaMemsetAsync(h->fb[0], 0, L.field_bytes, h->stream) != cudaSuccess) return fail(ABFT_ECUDA);
  if (cudaMemcpy2DAsync(h->fb[0] + (size_t)L.plane * esz, L.px * esz, u0, nx * esz, nx * esz, ny * zc,
                        cudaMemcpyDefault, h->stream) != cudaSuccess)
    return fail(ABFT_ECUDA);
  for (int b = 1; b < h->nbuf; ++b)
    if (cudaMemsetAsync(h->fb[b], 0, L.field_bytes, h->stream) != cudaSuccess) return fail(ABFT_ECUDA);
  if (cudaMemsetAsync(h->aux, 0, L.aux_bytes, h->stream) != cudaSuccess) return fail(ABFT_ECUDA);

  // source field (HotSpot power): used in place when TMA-legal, else a padded copy
  h->field_src = field_source(cfg);
  if (h->field_src >= 0) {
    const void* f = cfg->sources[h->field_src].field;
    if (L.pad_src) {
      char* dstp = h->aux + L.off_src;
      if (cudaMemcpy2DAsync(dstp, L.px * esz, f, nx * esz, nx * esz, ny * zc, cudaMemcpyDefault,
                            h->stream) != cudaSuccess)
        return fail(ABFT_ECUDA);
      h->src_field = dstp;
      h->src_px = L.px;
    } else {
      h->src_field = f;
      h->src_px = nx;
    }
  }

  // x-edge ledger of u0 (columns 0 and nx-1 of layers 1..zc), read by the first check
  for (int side = 0; side < 2; ++side) {
    char* dst = h->EX[0] + ((size_t)side * (zc + 2) * ny + ny) * esz;
    const char* src = h->fb[0] + ((size_t)L.plane + (side ? nx - 1 : 0)) * esz;
    if (cudaMemcpy2DAsync(dst, esz, src, L.px * esz, esz, ny * zc, cudaMemcpyDeviceToDevice,
                          h->stream) != cudaSuccess)
      return fail(ABFT_ECUDA);
  }

  // TMA descriptors
  h->geo = k1_geometry(cfg->dtype);
  const int HV = 16 / esz;
  for (int b = 0; b < h->nbuf; ++b)
    if (!encode3d(&h->tm_u[b], cfg->dtype, h->fb[b], nx, ny, zc + 2, L.px * esz, L.plane * esz,
                  h->geo.tile_x + 2 * HV, h->geo.tile_y + 2))
      return fail(ABFT_ECUDA);

  // launch geometry and schedule (k1_plan)
  h->shape = match_shape(cfg);
  {
    const K1Plan kp = k1_plan(cfg, dev);
    h->zchunk = kp.zchunk;
    h->grid1 = kp.grid;
  }

  // parameter blocks (weights and coefficients rounded to the dtype)
  SweepParams& sp = h->sp;
  memset(&sp, 0, sizeof(sp));
  sp.nx = (int)nx; sp.ny = (int)ny; sp.zc = (int)zc; sp.zchunk = h->zchunk;
  sp.zr0 = 0; sp.zr1 = (int)zc;
  sp.bc = cfg->bc;
  sp.g = cfg->bc == ABFT_BC_CONSTANT ? rnd(cfg->dtype, cfg->bc_value) : 0.0;
  sp.src = h->src_field;
  sp.spx = h->src_px;
  sp.splane = h->src_px * ny;
  sp.px = L.px; sp.plane = L.plane; sp.has_lo = h->has_lo; sp.has_hi = h->has_hi;
  sp.npoints = cfg->npoints; sp.nsources = cfg->nsources; sp.field_src = h->field_src;
  for (int q = 0; q < cfg->npoints; ++q) {
    sp.di[q] = cfg->points[q].di; sp.dj[q] = cfg->points[q].dj; sp.dk[q] = cfg->points[q].dk;
    sp.w[q] = rnd(cfg->dtype, cfg->points[q].w);
    sp.wf[q] = (float)sp.w[q];
  }
  for (int q = 0; q < cfg->nsources; ++q) {
    sp.coef[q] = rnd(cfg->dtype, cfg->sources[q].coef);
    sp.scalar[q] = rnd(cfg->dtype, cfg->sources[q].scalar);
    sp.coeff[q] = (float)sp.coef[q];
    sp.scalarf[q] = (float)sp.scalar[q];
  }
  CheckParams& cp = h->cp;
  memset(&cp, 0, sizeof(cp));
  cp.nx = (int)nx; cp.ny = (int)ny; cp.zc = (int)zc; cp.px = L.px; cp.plane = L.plane;
  cp.has_lo = h->has_lo; cp.has_hi = h->has_hi;
  cp.bc = cfg->bc;
  cp.g = sp.g;
  cp.cA = h->cA; cp.cB = h->cB; cp.summ = h->summ; cp.st = h->st; cp.zflag = h->zflag; cp.lazy_list = h->lazy_list;
  cp.lazy_rowlist = h->lazy_rowlist; cp.lazy_mark = h->lazy_mark;
  cp.npoints = cfg->npoints;
  for (int q = 0; q < cfg->npoints; ++q) {
    cp.di[q] = sp.di[q]; cp.dj[q] = sp.dj[q]; cp.dk[q] = sp.dk[q]; cp.w[q] = sp.w[q];
  }
  cp.nsources = cfg->nsources;
  cp.field_src = h->field_src;
  for (int q = 0; q < cfg->nsources; ++q) { cp.coef[q] = sp.coef[q]; cp.scalar[q] = sp.scalar[q]; }
  cp.src = h->src_field;
  cp.spx = h->src_px;
  cp.splane = h->src_px * ny;
  cp.eps = cfg->epsilon;
  cp.form = cfg->correction_form;
  cp.z_begin = cfg->z_begin;
  cp.zr0 = 0; cp.zr1 = (int)zc;

  // constant ghosts: the halo layers no neighbour owns are the
  // ghost layers of z (zmap); zero ghosts are the init memset
  if (cfg->bc == ABFT_BC_CONSTANT) {
    for (int b = 0; b < h->nbuf; ++b) {
      if (!h->has_lo && launch_fill(cfg->dtype, h->fb[b], L.plane, sp.g, h->stream) != cudaSuccess)
        return fail(ABFT_ECUDA);
      if (!h->has_hi && launch_fill(cfg->dtype, h->fb[b] + (size_t)(zc + 1) * L.plane * esz, L.plane, sp.g,
                                    h->stream) != cudaSuccess)
        return fail(ABFT_ECUDA);
    }
  }

  // load every kernel variant this handle may launch (hot / flip / general K1
  // for each checksum mode, K2, K3) now: with CUDA's lazy module loading the
  // first sweep carrying a flip would otherwise pay the load inside the run
  {
    const int vars[3] = {K1_HOT, K1_INJ, K1_GEN};
    const int chks[3] = {K1_CK_NONE, K1_CK_AB, K1_CK_B};
    for (int ci = 0; ci < 3; ++ci)
      for (int vi = 0; vi < 3; ++vi) {
        const cudaError_t e = cfg->dtype == ABFT_F32
                                  ? launch_k1_f32(h->shape, chks[ci], vars[vi], dim3(0), h->stream, h->tm_u[0], sp)
                                  : launch_k1_f64(h->shape, chks[ci], vars[vi], dim3(0), h->stream, h->tm_u[0], sp);
        if (e != cudaSuccess) return fail(ABFT_ECUDA);
      }
  }
  if (prime_checks(cfg->dtype, h->shape, cfg->bc) != cudaSuccess) return fail(ABFT_ECUDA);

  // K0: trusted a^0, b^0 of u0 and the pre-computed c_x, c_y
  if (launch_k0_field(cfg->dtype, h->fb[0], L.px, L.plane, (int)nx, (int)ny, (int)zc, h->gA[0], h->gB[0],
                      1, h->stream) != cudaSuccess)
    return fail(ABFT_ECUDA);
  if (launch_k0_const(cfg->dtype, h->src_field, h->src_px, (int)nx, (int)ny, (int)zc, cfg->nsources,
                      h->field_src, sp.coef, sp.scalar, h->cA, h->cB, h->stream) != cudaSuccess)
    return fail(ABFT_ECUDA);
  h->launches += 4;
  h->zmask = ((1u << kGens) - 1) & ~1u;   // aux cleared, K0 wrote generation 0
  if (const char* e = getenv("ABFT_GRAPHS")) h->graphs_on = atoi(e) != 0;
  if (const char* e = getenv("ABFT_OFFLINE_SPEC")) h->spec_on = atoi(e) != 0;
  if (const char* e = getenv("ABFT_PIPE_PDL")) h->pipe_pdl = atoi(e) != 0;
  if (h->pipe) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const char* pe = getenv("ABFT_S2_PRIO");   // experiment: 1 high, -1 low, 0 default
    const int pv = pe ? atoi(pe) : 0;
    const int prio = pv > 0 ? hi : (pv < 0 ? lo : 0);
    if (cudaStreamCreateWithPriority(&h->s2, cudaStreamNonBlocking, prio) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_k1, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_chk[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_chk[1], cudaEventDisableTiming) != cudaSuccess)
      return fail(ABFT_ECUDA);
  }

  // multi-GPU: NCCL communicator over NVLink, initial halo.  Without an id the
  // handle is a member of a local group (abft_stencil_group links them).
  if (cfg->nranks > 1 && cfg->nccl_unique_id) {
    int r = comm_acquire(cfg->nccl_unique_id, cfg->nranks, cfg->rank, &h->comm);
    if (r) return fail(r);
    r = exchange_nccl(h, XSpec{0, XV_GEN, 0});
    if (r) { comm_release(h->comm); return fail(r); }
  }
  *out = h;
  return ABFT_OK;
}

}  // extern "C"

namespace {
// the members of a group (or the ranks of a job) state the same problem: grid,
// dtype, stencil S and C (Eq. 1), boundary, threshold, mode, period, policy
bool same_problem(const abft_config& a, const abft_config& b) {
  if (a.nx != b.nx || a.ny != b.ny || a.nz_global != b.nz_global || a.dtype != b.dtype ||
      a.mode != b.mode || a.delta != b.delta || a.npoints != b.npoints || a.nsources != b.nsources ||
      a.bc != b.bc || a.epsilon != b.epsilon || a.correction_form != b.correction_form ||
      a.checksum_policy != b.checksum_policy || a.recovery != b.recovery)
    return false;
  if (a.bc == ABFT_BC_CONSTANT && a.bc_value != b.bc_value) return false;
  for (int q = 0; q < a.npoints; ++q) {
    const abft_point &p = a.points[q], &r = b.points[q];
    if (p.di != r.di || p.dj != r.dj || p.dk != r.dk || p.w != r.w) return false;
  }
  for (int q = 0; q < a.nsources; ++q) {
    const abft_source &s = a.sources[q], &r = b.sources[q];
    if (s.coef != r.coef || s.scalar != r.scalar || (s.field == nullptr) != (r.field == nullptr)) return false;
  }
  return true;
}
}  // namespace

extern "C" {

int abft_stencil_group(abft_stencil* const* hs, int32_t n) {
  if (!hs || n < 2) return ABFT_EINVAL;
  for (int i = 0; i < n; ++i) {
    abft_stencil* h = hs[i];
    if (!h || h->grouped || h->comm || h->ipc || h->cfg.nranks != n || h->cfg.rank != i) return ABFT_EINVAL;
    const abft_config &a = h->cfg, &b = hs[0]->cfg;
    if (!same_problem(a, b)) return ABFT_EINVAL;
    if (i + 1 < n && a.z_begin + a.z_count != hs[i + 1]->cfg.z_begin) return ABFT_EINVAL;
    if (h->sweeps != 0) return ABFT_EINVAL;
  }
  Group G(hs, hs + n);
  DevScope ds(hs[0]);
  // fused halo when every neighbour's memory is directly addressable: same
  // device, or a peer GPU with peer access (NVLink); ABFT_GROUP_COPY=1 keeps
  // the device-copy exchange
  bool fused = !(getenv("ABFT_GROUP_COPY") && getenv("ABFT_GROUP_COPY")[0] == '1');
  int cur_dev = 0;
  CK(cudaGetDevice(&cur_dev));
  for (int i = 0; i + 1 < n && fused; ++i) {
    const int a = hs[i]->dev, b = hs[i + 1]->dev;
    if (a == b) continue;
    int ab = 0, ba = 0;
    cudaDeviceCanAccessPeer(&ab, a, b);
    cudaDeviceCanAccessPeer(&ba, b, a);
    if (!ab || !ba) { fused = false; break; }
    for (int pr = 0; pr < 2; ++pr) {
      CK(cudaSetDevice(pr ? b : a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(pr ? a : b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) fused = false;
      cudaGetLastError();
    }
  }
  CK(cudaSetDevice(cur_dev));
  for (int i = 0; i < n; ++i) {
    abft_stencil* h = hs[i];
    const bool ring = z_ring(h->cfg);
    h->lo_peer = i > 0 ? hs[i - 1] : (ring ? hs[n - 1] : nullptr);
    h->hi_peer = i + 1 < n ? hs[i + 1] : (ring ? hs[0] : nullptr);
    h->grouped = true;
    h->fused = fused;
    h->members = G;
    on_dev(h);   // events belong to the member's device (recorded on its stream)
    CK(cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_pulled, cudaEventDisableTiming));
  }
  return exchange_local(G, XSpec{0, XV_GEN, 0});  // initial halo of u^0 and a^0, b^0
}

int abft_stencil_ipc_export(abft_stencil* h, void* blob) {
  if (!h || !blob || h->is_proxy || h->grouped || h->comm || h->cfg.nranks < 2) return ABFT_EINVAL;
  DevScope ds(h);
  IpcBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kIpcMagic;
  b.version = 2;
  b.rank = h->cfg.rank; b.nranks = h->cfg.nranks; b.nbuf = h->nbuf;
  b.nx = h->cfg.nx; b.ny = h->cfg.ny; b.z_count = h->cfg.z_count; b.z_begin = h->cfg.z_begin;
  b.plane = h->L.plane; b.esz = h->L.esz;
  for (int k = 0; k < h->nbuf; ++k) TRY(ipc_handle(h->fb[k], &b.mem[k], &b.off[k]));
  TRY(ipc_handle(h->aux, &b.mem[3], &b.off[3]));
  for (int g = 0; g < kGens; ++g) { b.off_gA[g] = h->L.off_gA[g]; b.off_gB[g] = h->L.off_gB[g]; }
  for (int g = 0; g < 2; ++g) { b.off_PA[g] = h->L.off_PA[g]; b.off_PB[g] = h->L.off_PB[g]; }
  for (int k = 0; k < 2; ++k) {
    if (!h->ev_ipc[k]) CK(cudaEventCreateWithFlags(&h->ev_ipc[k], cudaEventDisableTiming | cudaEventInterprocess));
    CK(cudaIpcGetEventHandle(&b.ev[k], h->ev_ipc[k]));
  }
  // a neighbour reads this slab's initial state as soon as it has the blob
  CK(cudaStreamSynchronize(h->stream));
  memset(blob, 0, ABFT_IPC_BLOB_BYTES);
  memcpy(blob, &b, sizeof(b));
  return ABFT_OK;
}

int abft_stencil_ipc_link(abft_stencil* h, const void* lo_blob, const void* hi_blob, void* shm) {
  if (!h || !shm || h->is_proxy || h->grouped || h->comm || h->ipc || h->cfg.nranks < 2 || h->sweeps != 0)
    return ABFT_EINVAL;
  if ((h->has_lo != 0) != (lo_blob != nullptr) || (h->has_hi != 0) != (hi_blob != nullptr)) return ABFT_EINVAL;
  if (!h->ev_ipc[0]) return ABFT_EINVAL;   // export first (it creates the events the neighbours open)
  // the slots carry a slab's flagged layers (partial re-execution) as bits
  if (h->cfg.recovery == ABFT_RECOVER_PARTIAL && h->cfg.z_count > 32 * (int64_t)ABFT_IPC_ZWORDS)
    return ABFT_EUNSUPPORTED;
  DevScope ds(h);
  const void* blobs[2] = {lo_blob, hi_blob};
  std::vector<std::pair<cudaIpcMemHandle_t, char*>> seen;
  int r = ABFT_OK;
  for (int f = 0; f < 2 && r == ABFT_OK; ++f) {
    if (!blobs[f]) continue;
    IpcBlob b;
    memcpy(&b, blobs[f], sizeof(b));
    const int64_t nzg = h->cfg.nz_global;
    const int want = (h->cfg.rank + (f == 0 ? -1 : 1) + h->cfg.nranks) % h->cfg.nranks;
    const int64_t want_z = ((f == 0 ? h->cfg.z_begin - b.z_count : h->cfg.z_begin + h->cfg.z_count) + nzg) % nzg;
    if (f == 1 && h->proxy[0] && lo_blob && !memcmp(lo_blob, hi_blob, sizeof(IpcBlob))) {
      h->proxy[1] = h->proxy[0];   // a ring of two ranks: one neighbour on both faces
      continue;
    }
    if (b.magic != kIpcMagic || b.version != 2 || b.rank != want || b.nranks != h->cfg.nranks ||
        b.nx != h->cfg.nx || b.ny != h->cfg.ny || b.plane != h->L.plane || b.esz != h->L.esz ||
        b.nbuf != h->nbuf || b.z_begin != want_z) {
      r = ABFT_EINVAL;
      break;
    }
    abft_stencil* q = new abft_stencil();
    q->is_proxy = true;
    q->cfg = h->cfg;
    q->cfg.rank = b.rank;
    q->cfg.z_begin = b.z_begin;
    q->cfg.z_count = b.z_count;
    q->L = h->L;
    q->dev = h->dev;
    h->proxy[f] = q;
    for (int k = 0; k < b.nbuf && r == ABFT_OK; ++k) {
      char* base = nullptr;
      r = ipc_open(h, seen, b.mem[k], &base);
      if (r == ABFT_OK) q->fb[k] = base + b.off[k];
    }
    char* base = nullptr;
    if (r == ABFT_OK) r = ipc_open(h, seen, b.mem[3], &base);
    if (r != ABFT_OK) break;
    char* aux = base + b.off[3];
    for (int g = 0; g < kGens; ++g) {
      q->gA[g] = reinterpret_cast<double*>(aux + b.off_gA[g]);
      q->gB[g] = reinterpret_cast<double*>(aux + b.off_gB[g]);
    }
    for (int g = 0; g < 2; ++g) {
      q->PA[g] = reinterpret_cast<double*>(aux + b.off_PA[g]);
      q->PB[g] = reinterpret_cast<double*>(aux + b.off_PB[g]);
    }
    for (int k = 0; k < 2 && r == ABFT_OK; ++k)
      if (cudaIpcOpenEventHandle(&q->ev_ipc[k], b.ev[k]) != cudaSuccess) r = ABFT_ECUDA;
  }
  if (r != ABFT_OK) {
    ipc_unlink(h);
    return r;
  }
  h->lo_peer = h->proxy[0];
  h->hi_peer = h->proxy[1];
  h->ipc = true;
  h->fused = true;
  h->shm = static_cast<abft_ipc_slot*>(shm);
  h->xseq = h->wseq = 0;
  memset(&h->shm[h->cfg.rank], 0, sizeof(abft_ipc_slot));
  h->shm[h->cfg.rank].z_begin = (int32_t)h->cfg.z_begin;
  h->shm[h->cfg.rank].z_count = (int32_t)h->cfg.z_count;
  // initial halo of u^0 and a^0, b^0: pull the neighbours' boundary layers
  // (their exports synchronised their init); their first writes into these
  // buffers come after their first sweep, which waits for this rank's
  const size_t lb = (size_t)h->L.plane * h->L.esz;
  const int64_t nx = h->cfg.nx, ny = h->cfg.ny, zc = h->cfg.z_count;
  for (int f = 0; f < 2; ++f) {
    abft_stencil* q = h->proxy[f];
    if (!q) continue;
    const int64_t src_l = f == 0 ? q->cfg.z_count : 1, dst_l = f == 0 ? 0 : zc + 1;
    CK(cudaMemcpyAsync(h->fb[0] + dst_l * lb, q->fb[0] + src_l * lb, lb, cudaMemcpyDefault, h->stream));
    CK(cudaMemcpyAsync(h->gA[0] + dst_l * nx, q->gA[0] + src_l * nx, nx * 8, cudaMemcpyDefault, h->stream));
    CK(cudaMemcpyAsync(h->gB[0] + dst_l * ny, q->gB[0] + src_l * ny, ny * 8, cudaMemcpyDefault, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  return ABFT_OK;
}

int abft_stencil_step_group(abft_stencil* const* hs, int32_t n, int32_t nsweeps) {
  if (!hs || n < 1 || nsweeps < 0) return ABFT_EINVAL;
  if (n == 1) return abft_stencil_step(hs[0], nsweeps);
  for (int i = 0; i < n; ++i)
    if (!hs[i] || !hs[i]->grouped || hs[i]->members.size() != (size_t)n || hs[i]->members[i] != hs[i])
      return ABFT_EINVAL;
  Group G(hs, hs + n);
  DevScope ds(hs[0]);
  return step_group(G, nsweeps);
}

int abft_stencil_step(abft_stencil* h, int32_t n) {
  if (!h || n < 0 || h->grouped) return ABFT_EINVAL;
  DevScope ds(h);
  Group G{h};
  return step_group(G, n);
}

int abft_stencil_plan(abft_stencil* h, int32_t n) {
  if (!h || n < 0 || h->grouped) return ABFT_EINVAL;
  DevScope ds(h);
  if (!graph_eligible(h, n) || graph_find(h, n)) return ABFT_OK;
  StepGraph* g = nullptr;
  return graph_capture(h, n, &g);
}

int abft_stencil_sweep(abft_stencil* h) {
  if (!h || h->grouped) return ABFT_EINVAL;
  DevScope ds(h);
  if (h->cfg.mode == ABFT_MODE_OFFLINE) return ABFT_EINVAL;
  Group G{h};
  if (h->cfg.mode == ABFT_MODE_NONE) return none_sweep(G);
  const int64_t s = h->sweeps + 1;
  const int src = h->cur, dst = next_buf(h);
  const int gn = (h->gen + 1) % kGens;
  TRY(clear_summaries(h));
  TRY(zero_gen(h, gn));
  h->zmask &= ~(1u << gn);
  TRY(launch_k1(h, src, dst, h->gA[gn], h->gB[gn], K1_CK_AB, s));
  TRY(halo_exchange(G, XSpec{dst, XV_GEN, gn}));
  h->prev = src;
  h->cur = dst;
  h->gen_prev = h->gen;
  h->gen = gn;
  h->sweeps = s;
  h->pending_check = true;
  return ABFT_OK;
}

int abft_stencil_check(abft_stencil* h, int64_t* nflag_a, int64_t* nflag_b) {
  if (!h || h->grouped || h->cfg.mode != ABFT_MODE_ONLINE || !h->pending_check) return ABFT_EINVAL;
  DevScope ds(h);
  TRY(clear_summaries(h));
  CK(cudaMemsetAsync(&h->st->flag_a, 0, 2 * sizeof(long long), h->stream));
  int r = launch_check(h, h->prev, h->cur, h->gA[h->gen_prev], h->gB[h->gen_prev], h->gA[h->gen],
                       h->gB[h->gen], nullptr, nullptr, nullptr, nullptr, CK_COMPARE | CK_SUMMARY,
                       h->sweeps);
  if (r) return r;
  h->summ_dirty = true;
  long long f[2];
  CK(cudaMemcpyAsync(f, &h->st->flag_a, sizeof(f), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (nflag_a) *nflag_a = f[0];
  if (nflag_b) *nflag_b = f[1];
  return ABFT_OK;
}

int abft_stencil_correct(abft_stencil* h, int64_t* ncorrected) {
  if (!h || h->grouped || h->cfg.mode != ABFT_MODE_ONLINE || !h->pending_check) return ABFT_EINVAL;
  DevScope ds(h);
  CK(cudaMemsetAsync(&h->st->ncorr, 0, sizeof(long long), h->stream));
  int r = launch_check(h, h->prev, h->cur, h->gA[h->gen_prev], h->gB[h->gen_prev], h->gA[h->gen],
                       h->gB[h->gen], nullptr, nullptr, nullptr, nullptr, CK_FROM_SUMMARY | CK_CORRECT,
                       h->sweeps);
  if (r) return r;
  h->summ_dirty = false;
  Group G{h};
  TRY(halo_exchange(G, XSpec{h->cur, XV_GEN, h->gen}));
  long long c = 0;
  CK(cudaMemcpyAsync(&c, &h->st->ncorr, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (ncorrected) *ncorrected = c;
  h->pending_check = false;
  return ABFT_OK;
}

int abft_stencil_set_faults(abft_stencil* h, const abft_fault* f, int32_t n) {
  if (!h || n < 0 || (n > 0 && !f)) return ABFT_EINVAL;
  h->faults.clear();
  for (int i = 0; i < n; ++i) {
    const abft_fault& a = f[i];
    if (a.z < 0 || a.z >= h->cfg.nz_global || a.y < 0 || a.y >= h->cfg.ny || a.x < 0 || a.x >= h->cfg.nx ||
        a.bit < 0 || a.bit >= 8 * h->L.esz || a.sweep < 1)
      return ABFT_EINVAL;
    h->faults.push_back(PendingFault{a, false});
  }
  // one K1 launch carries a sweep's flips in its parameter block: at most
  // kMaxFaultsPerLaunch per sweep in this slab (a cell listed k times for one
  // sweep strikes k executions of it: the first and k - 1 re-executions)
  std::vector<const abft_fault*> mine;
  for (const PendingFault& pf : h->faults) {
    const int64_t zl = pf.f.z - h->cfg.z_begin;
    if (zl >= 0 && zl < h->cfg.z_count) mine.push_back(&pf.f);
  }
  std::sort(mine.begin(), mine.end(), [](const abft_fault* a, const abft_fault* b) {
    return std::tie(a->sweep, a->z, a->y, a->x) < std::tie(b->sweep, b->z, b->y, b->x);
  });
  for (size_t i = 0, run = 1; i < mine.size(); ++i, ++run) {
    if (i > 0 && mine[i]->sweep != mine[i - 1]->sweep) run = 1;
    if (run > (size_t)kMaxFaultsPerLaunch) {
      h->faults.clear();
      return ABFT_EINVAL;
    }
  }
  return ABFT_OK;
}

int abft_stencil_field(abft_stencil* h, void** dev_ptr, int64_t* pitch) {
  if (!h || !dev_ptr) return ABFT_EINVAL;
  DevScope ds(h);
  CK(cudaStreamSynchronize(h->stream));
  *dev_ptr = h->fb[h->cur] + (size_t)h->L.plane * h->L.esz;
  if (pitch) *pitch = h->L.px;
  return ABFT_OK;
}

int abft_stencil_read_field(abft_stencil* h, void* dst) {
  if (!h || !dst) return ABFT_EINVAL;
  DevScope ds(h);
  const size_t esz = h->L.esz;
  CK(cudaMemcpy2DAsync(dst, h->cfg.nx * esz, h->fb[h->cur] + (size_t)h->L.plane * esz, h->L.px * esz,
                       h->cfg.nx * esz, h->cfg.ny * h->cfg.z_count, cudaMemcpyDefault, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return ABFT_OK;
}

int abft_stencil_checksums(abft_stencil* h, double* A, double* B) {
  if (!h || !A || !B) return ABFT_EINVAL;
  DevScope ds(h);
  const int64_t nx = h->cfg.nx, ny = h->cfg.ny, zc = h->cfg.z_count;
  int g = h->gen, ga = h->gen;
  if (h->cfg.mode == ABFT_MODE_NONE) {  // no running checksums: compute them now (Eqs. 2-3)
    g = ga = (h->gen + 1) % kGens;
    h->zmask &= ~(1u << g);
    if (launch_k0_field(h->cfg.dtype, h->fb[h->cur], h->L.px, h->L.plane, (int)nx, (int)ny, (int)zc,
                        h->gA[g], h->gB[g], 1, h->stream) != cudaSuccess)
      return ABFT_ECUDA;
    h->launches += 2;
  } else if (h->cfg.checksum_policy == ABFT_CK_LAZY &&
             ((h->cfg.mode == ABFT_MODE_ONLINE && !h->pending_check) || h->cfg.mode == ABFT_MODE_OFFLINE)) {
    // lazy policy: a is not carried (online: K3 computes it for flagged
    // layers only; offline: never, Q29); compute it now into generation
    // gen + 2 (cleared again before it is accumulated into)
    ga = (h->gen + 2) % kGens;
    h->zmask &= ~(1u << ga);
    if (launch_k0_field(h->cfg.dtype, h->fb[h->cur], h->L.px, h->L.plane, (int)nx, (int)ny, (int)zc,
                        h->gA[ga], h->gB[ga], 1, h->stream) != cudaSuccess)
      return ABFT_ECUDA;
    h->launches += 2;
  }
  CK(cudaMemcpyAsync(A, h->gA[ga] + nx, sizeof(double) * nx * zc, cudaMemcpyDefault, h->stream));
  CK(cudaMemcpyAsync(B, h->gB[g] + ny, sizeof(double) * ny * zc, cudaMemcpyDefault, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return ABFT_OK;
}

int abft_stencil_stats(abft_stencil* h, abft_stats* o) {
  if (!h || !o) return ABFT_EINVAL;
  DevScope ds(h);
  long long c[9];
  CK(cudaMemcpyAsync(c, h->st->cnt, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  o->sweeps = h->executed;
  o->detections = c[ST_DETECT];
  o->located = c[ST_LOCATED];
  o->corrected = c[ST_CORRECTED];
  o->unlocated = c[ST_UNLOCATED];
  o->uncorrectable = c[ST_UNCORR];
  o->rollbacks = h->rollbacks;
  o->windows = h->windows;
  o->persistent = h->persistent;
  return ABFT_OK;
}

int abft_stencil_records(abft_stencil* h, abft_record* out, int32_t cap, int64_t* n) {
  if (!h || cap < 0 || (cap > 0 && !out)) return ABFT_EINVAL;
  DevScope ds(h);
  unsigned long long nrec = 0;
  CK(cudaMemcpyAsync(&nrec, &h->st->nrec, sizeof(nrec), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const int64_t m = std::min<int64_t>({(int64_t)nrec, (int64_t)cap, (int64_t)kRecordCap});
  if (m > 0) {
    CK(cudaMemcpyAsync(out, h->st->rec, sizeof(abft_record) * m, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  if (n) *n = (int64_t)nrec;
  return ABFT_OK;
}

int abft_stencil_status(abft_stencil* h) {
  if (!h) return ABFT_EINVAL;
  DevScope ds(h);
  int w = 0;
  CK(cudaMemcpyAsync(&w, &h->st->worst, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return std::max(w, h->host_worst);
}

int64_t abft_stencil_sweep_count(const abft_stencil* h) { return h ? h->sweeps : -1; }
int64_t abft_stencil_launch_count(const abft_stencil* h) { return h ? h->launches : -1; }

int abft_stencil_profile(abft_stencil* h, int32_t enable) {
  if (!h) return ABFT_EINVAL;
  h->prof = enable != 0;
  return ABFT_OK;
}

int abft_stencil_profile_read(abft_stencil* h, double* k1_ms, int64_t* k1_n, double* k2_ms,
                              int64_t* k2_n, int32_t geo[6]) {
  if (!h) return ABFT_EINVAL;
  DevScope ds(h);
  CK(cudaStreamSynchronize(h->stream));
  double t[3] = {0, 0, 0};
  int64_t n[3] = {0, 0, 0};
  for (size_t i = 0; i < h->ev_used; ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev[2 * i], h->ev[2 * i + 1]));
    t[h->ev_kind[i]] += ms;
    n[h->ev_kind[i]]++;
  }
  h->ev_used = 0;
  if (k1_ms) *k1_ms = t[1];
  if (k1_n) *k1_n = n[1];
  if (k2_ms) *k2_ms = t[2];
  if (k2_n) *k2_n = n[2];
  if (geo) {
    geo[0] = h->grid1.x; geo[1] = h->grid1.y; geo[2] = h->grid1.z;
    geo[3] = h->geo.threads; geo[4] = h->geo.smem; geo[5] = h->zchunk;
  }
  return ABFT_OK;
}

int abft_stencil_destroy(abft_stencil* h) {
  if (!h) return ABFT_EINVAL;
  DevScope ds(h);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (auto e : h->ev) cudaEventDestroy(e);
  if (h->s2) { cudaStreamSynchronize(h->s2); cudaStreamDestroy(h->s2); }
  for (StepGraph& g : h->graphs) { cudaGraphExecDestroy(g.exec); cudaGraphDestroy(g.graph); }
  if (h->cs) cudaStreamDestroy(h->cs);
  if (h->ev_verdict) cudaEventDestroy(h->ev_verdict);
  if (h->pin_dirty) cudaFreeHost(h->pin_dirty);
  for (cudaEvent_t e : {h->ev_k1, h->ev_chk[0], h->ev_chk[1]})
    if (e) cudaEventDestroy(e);
  if (h->ev_ready) cudaEventDestroy(h->ev_ready);
  if (h->ev_pulled) cudaEventDestroy(h->ev_pulled);
  for (abft_stencil* q : h->members)   // unlink: the group is unusable once a member is gone
    if (q != h) { q->lo_peer = q->lo_peer == h ? nullptr : q->lo_peer;
                  q->hi_peer = q->hi_peer == h ? nullptr : q->hi_peer; q->members.clear(); }
  if (h->comm) comm_release(h->comm);
  ipc_unlink(h);
  delete h;
  return ABFT_OK;
}

}  // extern "C"
