// abi.cu — the C ABI of include/gscl.h: validation, grid storage and layout,
// z-slab decomposition, NCCL halo exchange and cross-rank combine, and the
// device-resident Jacobi driver.  No exception or abort crosses the ABI.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gscl.h"
#include "internal.h"
#include "ops.cuh"

using namespace gscl;

struct gscl_grid_s {
  int64_t nx = 0, ny = 0, nz = 0;  // global interior extents
  int h = 0;
  int dtype = 0;
  size_t es = 8;
  int64_t z_begin = 0, z_end = 0, nzl = 0;  // this rank's slab
  int64_t pitch = 0, plane = 0, ox = 0;     // elements
  // storage (swapped as a unit by gscl_swap)
  void* base = nullptr;
  size_t bytes = 0;
  bool owned = false;
  cudaEvent_t ready = nullptr;  // completion of an asynchronous upload into this storage
  bool pending = false;         // the library stream must wait on `ready` before use
};

namespace {

// NVTX ranges on the host timeline (Nsight Systems): one per ABI call and per
// enqueued sweep / pass / exchange / combine (SURVEY §5 tracing).
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

thread_local std::string t_err;

gscl_status fail(gscl_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return s;
}

struct TimedPair {
  cudaEvent_t a, b;
  int kind;
};

struct GraphEntry {
  std::vector<int64_t> key;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
  bool final_in_v = false;
};

// Peer-memory transport of the multi-rank two-sweep schedule (option
// "transport" = 1): IPC mappings of the neighbours' u / v storage and of every
// rank's "arena" = [ghost planes for input storage 0 | ... 1 | counters |
// reduction slots].  Storage index 0 / 1 = the u / v storage at export time.
constexpr int kRedSlots = 64;
constexpr int kFlagsBytes = 256;  // counters: [0] from below, [1] from above, [2] barrier from below,
                                  // [3] barrier from above, [4] reduction arrivals
struct PeerBlob {
  int32_t magic, rank, world, dtype;
  int64_t nx, ny, nzl, h, pitch, plane, z_begin;
  cudaIpcMemHandle_t handle[3];  // u storage, v storage, arena
  int64_t offset[3];             // of the storage / arena inside its allocation
};
struct PeerSet {
  bool ready = false;
  void* store_base[2] = {nullptr, nullptr};  // my u / v storage at export
  void* arena = nullptr;                     // mine (cudaMalloc, exported)
  size_t plane_bytes = 0;
  int64_t nzl_nb[2] = {0, 0};                // planes of the lower / upper neighbour
  void* nb_store[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [lower/upper][storage] (base of grid data)
  char* arena_of[8] = {};                    // every rank's arena (mine included)
  std::vector<void*> opened;                 // IPC mappings to close
  unsigned tgt[5] = {0, 0, 0, 0, 0};         // host mirrors of what my counters will reach
  unsigned red_next = 0;                     // reduction slot ring position
  int64_t units = 0;                         // boundary units per side per step
  // arena layout: ghost planes for input storage 0 (2 planes: below, above),
  // for input storage 1, then the counters, then the reduction slots
  static size_t arena_bytes(size_t pb, int world) {
    return 4 * pb + kFlagsBytes + (size_t)kRedSlots * world * sizeof(double);
  }
  static unsigned* flags_of(char* ar, size_t pb) { return reinterpret_cast<unsigned*>(ar + 4 * pb); }
  static double* red_of(char* ar, size_t pb) { return reinterpret_cast<double*>(ar + 4 * pb + kFlagsBytes); }
  static char* ghost_of(char* ar, size_t pb, int storage) { return ar + (size_t)storage * 2 * pb; }
};

struct State {
  bool inited = false;
  int rank = 0, world = 1, device = 0, num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  double* d_partials = nullptr;
  int max_partials = 1 << 22;
  unsigned* d_counter = nullptr;
  double* d_scratch = nullptr;  // [0] result, [1..world] gathered partials
  double* d_hist = nullptr;     // [0, hist_cap): global check values
  double* d_lochist = nullptr;  // [0, hist_cap): this rank's partials (d_hist + hist_cap)
  size_t hist_cap = 0;
  void* d_ghost = nullptr;      // two planes below / above the halo (multi-rank passes)
  size_t ghost_cap = 0;
  void* d_rb = nullptr;         // red-black GS: the second buffer of the out-of-place passes
  size_t rb_cap = 0;
  unsigned long long* d_digest = nullptr;
  int* d_conv = nullptr;  // [0] converged, [1] iterations, [2] halt, [3] skip redo, [4] final half
  unsigned* d_bflag = nullptr;  // boundary-plane counter of the overlapped schedule
  cudaStream_t copy_stream = nullptr;  // asynchronous uploads (gscl_grid_copy_from_host_async)
  cudaEvent_t ev_to_copy = nullptr;
  void* up_stage[2] = {nullptr, nullptr};
  size_t up_cap[2] = {0, 0};
  unsigned up_next = 0;
  unsigned bflag_target = 0;    // host mirror of what the counter will reach
  double* h_pinned = nullptr;  // 64 doubles
  void* d_stage = nullptr;     // host-copy staging buffer (dense planes)
  size_t stage_cap = 0;
  cudaStream_t comm_stream = nullptr;  // halo exchange / cross-rank combine in jacobi_run
  cudaEvent_t ev_to_comm = nullptr, ev_to_main = nullptr, ev_halo = nullptr;
  int split = 0;  // force the overlapped (boundary-first) jacobi schedule at world 1
  int tblock = 0;  // jacobi_run sweeps per HBM pass: 0 = auto (2 for JACOBI7 on one rank), 1, 2
  int graph = 0;   // jacobi_run as a CUDA graph: 0 = auto (small grids), 1 = always, 2 = never
  int zalt = 0;    // 1: jacobi_run alternates the z-chunk walk of consecutive sweeps
                   // (ablation: 2.4 % slower at 512^3, profiles/r01_ablations.md)
  std::vector<GraphEntry> graphs;
  int variant = 0;
  int transport = 0;  // multi-rank jacobi_run halo transport: 0 = NCCL, 1 = peer memory (IPC / NVLink)
  PeerSet peer;
  int impl = 0;
  int zchunks = 0;
  int sched = 0;
  int l2promo = 0;
  int stages = 0;  // 0 = per-op default (8 for 7-point fp64, else 4)
  bool timing = false;
  std::vector<TimedPair> pool, pending;
  double kind_ms[4] = {0, 0, 0, 0};
  int64_t kind_n[4] = {0, 0, 0, 0};
  int64_t launches = 0;
  std::set<gscl_grid_s*> live;
};
State S;

#define GSCL_TRY try {
#define GSCL_CATCH                                                   \
  }                                                                  \
  catch (...) {                                                      \
    return fail(GSCL_E_INVALID_ARG, "internal exception caught at ABI"); \
  }

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) return fail(GSCL_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)
#define NK(x)                                                                            \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess) return fail(GSCL_E_NCCL, "%s: %s", #x, ncclGetErrorString(r_)); \
  } while (0)
#define NEED_INIT() \
  if (!S.inited) return fail(GSCL_E_STATE, "gscl_init has not been called (or gscl_finalize was)")

int64_t ox_of(int dtype) { return dtype == 0 ? 16 : 32; }
int max_halo(int dtype) { return (int)ox_of(dtype); }

void slab(int64_t nz, int rank, int world, int64_t* z0, int64_t* z1) {
  int64_t base = nz / world, rem = nz % world;
  int64_t r = rank;
  *z0 = r * base + std::min<int64_t>(r, rem);
  *z1 = *z0 + base + (r < rem ? 1 : 0);
}

gscl_status layout(gscl_grid_s* g, int64_t nx, int64_t ny, int64_t nz, int halo, int dtype,
                   int rank, int world) {
  if (nx <= 0 || ny <= 0 || nz <= 0)
    return fail(GSCL_E_INVALID_DOMAIN, "extents must be positive (got %lld x %lld x %lld)",
                (long long)nx, (long long)ny, (long long)nz);
  if (dtype != GSCL_F64 && dtype != GSCL_F32) return fail(GSCL_E_INVALID_ARG, "bad dtype %d", dtype);
  if (halo < 0 || halo > max_halo(dtype))
    return fail(GSCL_E_INVALID_DOMAIN, "halo %d outside 0..%d", halo, max_halo(dtype));
  if (nx > (1ll << 30) || ny > (1ll << 30) || nz > (1ll << 30))
    return fail(GSCL_E_INVALID_DOMAIN, "extent too large");
  g->nx = nx; g->ny = ny; g->nz = nz; g->h = halo; g->dtype = dtype;
  g->es = dtype == 0 ? 8 : 4;
  slab(nz, rank, world, &g->z_begin, &g->z_end);
  g->nzl = g->z_end - g->z_begin;
  if (g->nzl <= 0 || (world > 1 && g->nzl < halo))
    return fail(GSCL_E_INVALID_DOMAIN, "slab of rank %d has %lld planes (nz=%lld, world=%d, halo=%d)",
                rank, (long long)g->nzl, (long long)nz, world, halo);
  g->ox = ox_of(dtype);
  g->pitch = (g->ox + nx + halo + g->ox - 1) / g->ox * g->ox;
  g->plane = g->pitch * (ny + 2 * halo);
  g->bytes = (size_t)(g->plane * (g->nzl + 2 * halo)) * g->es;
  return GSCL_OK;
}

View view_of(const gscl_grid_s* g) {
  View v;
  v.base = g->base;
  v.origin = static_cast<char*>(g->base) + (size_t)(g->h * g->plane + g->h * g->pitch + g->ox) * g->es;
  v.nx = g->nx; v.ny = g->ny; v.nzl = g->nzl; v.h = g->h;
  v.pitch = g->pitch; v.plane = g->plane; v.ox = g->ox; v.dtype = g->dtype;
  return v;
}

bool live(gscl_grid_t g) { return g && S.live.count(g); }

gscl_status check_grid(gscl_grid_t g, const char* what) {
  if (!g) return fail(GSCL_E_INVALID_ARG, "%s is NULL", what);
  if (!live(g)) return fail(GSCL_E_INVALID_ARG, "%s is not a live grid handle", what);
  if (g->pending) {  // an asynchronous upload into it: order it before any use
    CK(cudaStreamWaitEvent(S.stream, g->ready, 0));
    g->pending = false;
  }
  return GSCL_OK;
}

gscl_status same_shape(gscl_grid_t a, gscl_grid_t b) {
  if (a->nx != b->nx || a->ny != b->ny || a->nz != b->nz)
    return fail(GSCL_E_SHAPE_MISMATCH, "grid extents differ (%lldx%lldx%lld vs %lldx%lldx%lld)",
                (long long)a->nx, (long long)a->ny, (long long)a->nz, (long long)b->nx,
                (long long)b->ny, (long long)b->nz);
  if (a->dtype != b->dtype) return fail(GSCL_E_DTYPE, "grid element types differ");
  return GSCL_OK;
}

// Global range -> local box (clipped to this rank's slab).
gscl_status local_box(const gscl_grid_s* g, const gscl_range* r, Box* b) {
  gscl_range R = r ? *r : gscl_range{0, g->nx, 0, g->ny, 0, g->nz};
  if (R.x0 < 0 || R.x1 > g->nx || R.y0 < 0 || R.y1 > g->ny || R.z0 < 0 || R.z1 > g->nz ||
      R.x0 > R.x1 || R.y0 > R.y1 || R.z0 > R.z1)
    return fail(GSCL_E_RANGE, "range [%lld,%lld)x[%lld,%lld)x[%lld,%lld) not inside the interior",
                (long long)R.x0, (long long)R.x1, (long long)R.y0, (long long)R.y1, (long long)R.z0,
                (long long)R.z1);
  b->x0 = R.x0; b->x1 = R.x1; b->y0 = R.y0; b->y1 = R.y1;
  b->z0 = std::max(R.z0, g->z_begin) - g->z_begin;
  b->z1 = std::min(R.z1, g->z_end) - g->z_begin;
  if (b->z1 < b->z0) b->z1 = b->z0;
  return GSCL_OK;
}

int op_arity(int op) { return op == GSCL_OP_VARCOEF8 ? 8 : 1; }

gscl_status record_start(TimedPair* tp) {
  if (!S.timing) return GSCL_OK;
  if (S.pool.empty()) {
    TimedPair p;
    CK(cudaEventCreate(&p.a));
    CK(cudaEventCreate(&p.b));
    S.pool.push_back(p);
  }
  *tp = S.pool.back();
  S.pool.pop_back();
  CK(cudaEventRecord(tp->a, S.stream));
  return GSCL_OK;
}
gscl_status record_end(TimedPair tp, int kind) {
  if (!S.timing) return GSCL_OK;
  CK(cudaEventRecord(tp.b, S.stream));
  tp.kind = kind;
  S.pending.push_back(tp);
  return GSCL_OK;
}

RedTarget red_target(double* result, int comb) {
  RedTarget t;
  t.partials = S.d_partials;
  t.counter = S.d_counter;
  t.result = result;
  t.comb = comb;
  t.max_partials = S.max_partials;
  return t;
}

// Launch one sweep (timed when instrumentation is on).
gscl_status run_sweep(SweepPlan& p) {
  Nvtx nv(p.tsteps == 2 ? "gscl.pass" : p.write ? "gscl.sweep" : "gscl.reduce_sweep");
  p.stream = S.stream;
  p.impl = S.impl;
  p.zchunks = S.zchunks;
  p.sched = S.sched;
  p.l2promo = S.l2promo;
  p.stages = S.stages;
  p.variant = S.variant;
  p.num_sms = S.num_sms;
  if (p.rv != RV_NONE && p.box.empty()) {
    CK(launch_fold(nullptr, 0, p.red.comb, p.red.result, S.stream, &S.launches));
    return GSCL_OK;
  }
  TimedPair tp{};
  gscl_status st = record_start(&tp);
  if (st != GSCL_OK) return st;
  cudaError_t e = p.tsteps == 2 ? launch_sweep2(p, &S.launches) : launch_sweep(p, &S.launches);
  if (e != cudaSuccess) return fail(GSCL_E_CUDA, "sweep launch failed: %s", cudaGetErrorString(e));
  const int kind = p.tsteps == 2 ? 3 : p.rv == RV_NONE ? 0 : (p.write ? 1 : 2);
  return record_end(tp, kind);
}

// Combine this rank's device scalar d_loc across ranks into d_out (same bits
// on every rank): all-gather, then fold in rank order (R14).
gscl_status cross_rank(double* d_loc, int comb, double* d_out, cudaStream_t st) {
  Nvtx nv("gscl.combine");
  if (S.world == 1) {
    if (d_loc != d_out) CK(cudaMemcpyAsync(d_out, d_loc, 8, cudaMemcpyDeviceToDevice, st));
    return GSCL_OK;
  }
  if (!S.comm) return fail(GSCL_E_STATE, "no NCCL communicator (gscl_init had no nccl_id)");
  NK(ncclAllGather(d_loc, S.d_scratch + 1, 1, ncclDouble, S.comm, st));
  CK(launch_fold(S.d_scratch + 1, S.world, comb, d_out, st, &S.launches));
  return GSCL_OK;
}

// Make stream `to` wait for everything issued so far on stream `from`.
gscl_status hand_off(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
  CK(cudaEventRecord(ev, from));
  CK(cudaStreamWaitEvent(to, ev, 0));
  return GSCL_OK;
}

// The halo-exchange plan of one rank (byte offsets into its slab allocation).
// Local plane k (k = -h .. nzl+h-1) starts at byte (k + h) * plane * es.
int halo_plan(const gscl_grid_s* g, int rank, int world, gscl_halo_op* ops) {
  if (world == 1 || g->h == 0) return 0;
  const int64_t pb = g->plane * (int64_t)g->es;
  const int64_t n = g->h * pb;  // h contiguous planes
  int k = 0;
  if (rank > 0) {
    ops[k++] = gscl_halo_op{rank - 1, 1, g->h * pb, n};        // planes 0..h-1 -> below
    ops[k++] = gscl_halo_op{rank - 1, 0, 0, n};                // ghost planes -h..-1
  }
  if (rank < world - 1) {
    ops[k++] = gscl_halo_op{rank + 1, 1, g->nzl * pb, n};      // planes nzl-h..nzl-1 -> above
    ops[k++] = gscl_halo_op{rank + 1, 0, (g->nzl + g->h) * pb, n};  // ghost planes nzl..
  }
  return k;
}

gscl_status exchange(gscl_grid_s* g, cudaStream_t st) {
  Nvtx nv("gscl.halo");
  gscl_halo_op ops[4];
  const int n = halo_plan(g, S.rank, S.world, ops);
  if (n == 0) return GSCL_OK;
  if (!S.comm) return fail(GSCL_E_STATE, "no NCCL communicator (gscl_init had no nccl_id)");
  char* base = static_cast<char*>(g->base);
  NK(ncclGroupStart());
  for (int i = 0; i < n; ++i) {
    if (ops[i].is_send)
      NK(ncclSend(base + ops[i].offset, (size_t)ops[i].bytes, ncclUint8, ops[i].peer, S.comm, st));
    else
      NK(ncclRecv(base + ops[i].offset, (size_t)ops[i].bytes, ncclUint8, ops[i].peer, S.comm, st));
  }
  NK(ncclGroupEnd());
  return GSCL_OK;
}
gscl_status exchange(gscl_grid_s* g) { return exchange(g, S.stream); }

gscl_status ensure_hist(size_t n) {
  if (n <= S.hist_cap) return GSCL_OK;
  if (S.d_hist) {
    CK(cudaStreamSynchronize(S.stream));
    CK(cudaFree(S.d_hist));
  }
  S.d_hist = nullptr;
  CK(cudaMalloc(&S.d_hist, 2 * n * sizeof(double)));
  S.d_lochist = S.d_hist + n;
  S.hist_cap = n;
  return GSCL_OK;
}

gscl_status ensure_ghost(size_t bytes) {
  if (bytes <= S.ghost_cap) return GSCL_OK;
  if (S.d_ghost) {
    CK(cudaStreamSynchronize(S.stream));
    CK(cudaFree(S.d_ghost));
  }
  S.d_ghost = nullptr;
  CK(cudaMalloc(&S.d_ghost, bytes));
  S.ghost_cap = bytes;
  return GSCL_OK;
}

// The depth-2 halo exchange of a two-sweep pass: each side sends its first /
// last two interior planes, one plane per transfer, and receives the
// neighbour's into local planes -1, -2 (below) and nzl, nzl+1 (above).  A
// received plane inside the grid's halo (|offset| <= h) lands in the grid;
// one beyond it (h = 1) lands in the ghost buffer (plane 0 below, 1 above).
// Per neighbour the transfers are listed nearest plane first on both sides,
// so NCCL matches them in order.
int pass_plan(const gscl_grid_s* g, int rank, int world, gscl_pass_xfer* ops) {
  if (world == 1) return 0;
  int k = 0;
  const int64_t n = g->nzl, h = g->h;
  auto recv_at = [&](int peer, int64_t z) {
    gscl_pass_xfer o{peer, 0, z, 0};
    if (z < -h) o.ghost_plane = 1;       // ghost plane 0 (1-based flag + index)
    else if (z >= n + h) o.ghost_plane = 2;  // ghost plane 1
    ops[k++] = o;
  };
  if (rank > 0) {
    ops[k++] = gscl_pass_xfer{rank - 1, 1, 0, 0};
    ops[k++] = gscl_pass_xfer{rank - 1, 1, 1, 0};
    recv_at(rank - 1, -1);
    recv_at(rank - 1, -2);
  }
  if (rank < world - 1) {
    ops[k++] = gscl_pass_xfer{rank + 1, 1, n - 1, 0};
    ops[k++] = gscl_pass_xfer{rank + 1, 1, n - 2, 0};
    recv_at(rank + 1, n);
    recv_at(rank + 1, n + 1);
  }
  return k;
}

gscl_status exchange_pass(gscl_grid_s* g, cudaStream_t st) {
  Nvtx nv("gscl.halo2");
  gscl_pass_xfer ops[8];
  const int n = pass_plan(g, S.rank, S.world, ops);
  if (n == 0) return GSCL_OK;
  if (!S.comm) return fail(GSCL_E_STATE, "no NCCL communicator (gscl_init had no nccl_id)");
  const int64_t pb = g->plane * (int64_t)g->es;
  if (g->h < 2)
    if (gscl_status s = ensure_ghost(2 * (size_t)pb); s != GSCL_OK) return s;
  char* base = static_cast<char*>(g->base);
  char* ghost = static_cast<char*>(S.d_ghost);
  NK(ncclGroupStart());
  for (int i = 0; i < n; ++i) {
    char* ptr = ops[i].ghost_plane ? ghost + (ops[i].ghost_plane - 1) * pb : base + (ops[i].z + g->h) * pb;
    if (ops[i].is_send)
      NK(ncclSend(ptr, (size_t)pb, ncclUint8, ops[i].peer, S.comm, st));
    else
      NK(ncclRecv(ptr, (size_t)pb, ncclUint8, ops[i].peer, S.comm, st));
  }
  NK(ncclGroupEnd());
  return GSCL_OK;
}

void swap_storage(gscl_grid_s* a, gscl_grid_s* b) {
  std::swap(a->base, b->base);
  std::swap(a->bytes, b->bytes);
  std::swap(a->owned, b->owned);
  std::swap(a->ready, b->ready);
  std::swap(a->pending, b->pending);
}

// Release every IPC mapping and the arena of the peer transport.
void peer_reset() {
  PeerSet& P = S.peer;
  if (P.arena || !P.opened.empty()) cudaStreamSynchronize(S.stream);
  for (void* q : P.opened) cudaIpcCloseMemHandle(q);
  if (P.arena) cudaFree(P.arena);
  P = PeerSet();
}

// Open (once per process) the allocation behind an IPC handle.
struct OpenedHandle {
  cudaIpcMemHandle_t h;
  void* ptr;
};
std::vector<OpenedHandle> g_opened;
gscl_status open_handle(const cudaIpcMemHandle_t& h, void** ptr) {
  for (auto& o : g_opened)
    if (std::memcmp(&o.h, &h, sizeof h) == 0) {
      *ptr = o.ptr;
      return GSCL_OK;
    }
  void* q = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(GSCL_E_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  g_opened.push_back({h, q});
  S.peer.opened.push_back(q);
  *ptr = q;
  return GSCL_OK;
}

}  // namespace

extern "C" {

const char* gscl_last_error(void) { return t_err.c_str(); }

const char* gscl_version(void) {
  return "gscl-b200 0.1 (sm_100a; TMA 2.5-D sweep; NCCL z-slab halo exchange)";
}

gscl_status gscl_slab_range(int64_t nz, int rank, int world, int64_t* z_begin, int64_t* z_end) {
  if (nz <= 0 || world <= 0 || rank < 0 || rank >= world || !z_begin || !z_end)
    return fail(GSCL_E_INVALID_ARG, "bad slab arguments");
  slab(nz, rank, world, z_begin, z_end);
  return GSCL_OK;
}

gscl_status gscl_grid_bytes(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype, int rank,
                            int world, size_t* bytes) {
  GSCL_TRY
  if (!bytes || world <= 0 || rank < 0 || rank >= world) return fail(GSCL_E_INVALID_ARG, "bad arguments");
  gscl_grid_s g;
  gscl_status s = layout(&g, nx, ny, nz, halo, dtype, rank, world);
  if (s != GSCL_OK) return s;
  *bytes = g.bytes;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_halo_plan(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype, int rank,
                           int world, gscl_halo_op* ops, int* n_ops) {
  GSCL_TRY
  if (!ops || !n_ops || world <= 0 || rank < 0 || rank >= world)
    return fail(GSCL_E_INVALID_ARG, "bad arguments");
  gscl_grid_s g;
  gscl_status s = layout(&g, nx, ny, nz, halo, dtype, rank, world);
  if (s != GSCL_OK) return s;
  *n_ops = halo_plan(&g, rank, world, ops);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_pass_plan(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype, int rank,
                           int world, gscl_pass_xfer* ops, int* n_ops) {
  GSCL_TRY
  if (!ops || !n_ops || world <= 0 || rank < 0 || rank >= world)
    return fail(GSCL_E_INVALID_ARG, "bad arguments");
  gscl_grid_s g;
  gscl_status s = layout(&g, nx, ny, nz, halo, dtype, rank, world);
  if (s != GSCL_OK) return s;
  if (world > 1 && g.nzl < 2)
    return fail(GSCL_E_INVALID_DOMAIN, "a two-sweep pass needs >= 2 planes per rank (rank %d has %lld)",
                rank, (long long)g.nzl);
  *n_ops = pass_plan(&g, rank, world, ops);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_get_nccl_unique_id(void* out128) {
  GSCL_TRY
  if (!out128) return fail(GSCL_E_INVALID_ARG, "out128 is NULL");
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, 128);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_init(int rank, int world, const void* nccl_id, int device, void* cuda_stream) {
  GSCL_TRY
  if (S.inited) return fail(GSCL_E_STATE, "gscl_init called twice");
  if (world < 1 || rank < 0 || rank >= world) return fail(GSCL_E_INVALID_ARG, "bad rank/world");
  // world > 1 without an NCCL id: no communicator — only the peer-memory
  // transport of gscl_jacobi_run works across ranks (gscl_peer_export/import)
  CK(cudaSetDevice(device));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major < 10) return fail(GSCL_E_UNSUPPORTED, "device %d has compute capability %d.x; sm_100a required", device, major);
  CK(cudaDeviceGetAttribute(&S.num_sms, cudaDevAttrMultiProcessorCount, device));
  S.rank = rank;
  S.world = world;
  S.device = device;
  // NULL is the legacy default stream (CUDA's convention, and the handle torch
  // reports for its default stream): library work must be ordered with the
  // caller's allocations and fills on that same stream.
  S.stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : cudaStreamLegacy;
  S.own_stream = false;
  CK(cudaMalloc(&S.d_partials, (size_t)S.max_partials * sizeof(double)));
  CK(cudaMalloc(&S.d_counter, 64 * sizeof(unsigned)));
  CK(cudaMemset(S.d_counter, 0, 64 * sizeof(unsigned)));
  CK(cudaMalloc(&S.d_scratch, (size_t)(world + 8) * sizeof(double)));
  CK(cudaMalloc(&S.d_digest, sizeof(unsigned long long)));
  CK(cudaMalloc(&S.d_conv, 8 * sizeof(int)));
  CK(cudaMalloc(&S.d_bflag, sizeof(unsigned)));
  CK(cudaMemset(S.d_bflag, 0, sizeof(unsigned)));
  S.bflag_target = 0;
  CK(cudaMallocHost(&S.h_pinned, 64 * sizeof(double)));
  CK(cudaStreamCreateWithFlags(&S.comm_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&S.ev_to_comm, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&S.ev_to_main, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&S.ev_halo, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&S.copy_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&S.ev_to_copy, cudaEventDisableTiming));
  if (world > 1 && nccl_id) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, 128);
    NK(ncclCommInitRank(&S.comm, world, id, rank));
  }
  S.inited = true;
  S.launches = 0;
  t_err.clear();
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_finalize(void) {
  GSCL_TRY
  NEED_INIT();
  cudaStreamSynchronize(S.stream);
  peer_reset();
  g_opened.clear();
  if (S.copy_stream) cudaStreamSynchronize(S.copy_stream);
  for (gscl_grid_s* g : S.live) {
    if (g->owned && g->base) cudaFree(g->base);
    if (g->ready) cudaEventDestroy(g->ready);
    delete g;
  }
  S.live.clear();
  if (S.comm) ncclCommDestroy(S.comm);
  S.comm = nullptr;
  for (auto& p : S.pool) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  for (auto& p : S.pending) { cudaEventDestroy(p.a); cudaEventDestroy(p.b); }
  S.pool.clear();
  S.pending.clear();
  cudaFree(S.d_partials);
  cudaFree(S.d_counter);
  cudaFree(S.d_scratch);
  cudaFree(S.d_digest);
  cudaFree(S.d_conv);
  cudaFree(S.d_bflag);
  if (S.d_hist) cudaFree(S.d_hist);
  if (S.d_ghost) cudaFree(S.d_ghost);
  if (S.d_rb) cudaFree(S.d_rb);
  if (S.d_stage) cudaFree(S.d_stage);
  cudaFreeHost(S.h_pinned);
  for (auto& e : S.graphs) cudaGraphExecDestroy(e.exec);
  S.graphs.clear();
  if (S.comm_stream) {
    cudaStreamSynchronize(S.comm_stream);
    cudaStreamDestroy(S.comm_stream);
  }
  for (cudaEvent_t e : {S.ev_to_comm, S.ev_to_main, S.ev_halo, S.ev_to_copy})
    if (e) cudaEventDestroy(e);
  if (S.copy_stream) cudaStreamDestroy(S.copy_stream);
  for (void* p : S.up_stage)
    if (p) cudaFree(p);
  if (S.own_stream) cudaStreamDestroy(S.stream);
  S = State();
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_sync(void) {
  GSCL_TRY
  NEED_INIT();
  CK(cudaStreamSynchronize(S.stream));
  if (S.comm) {
    ncclResult_t async_err;
    NK(ncclCommGetAsyncError(S.comm, &async_err));
    if (async_err != ncclSuccess) return fail(GSCL_E_NCCL, "NCCL async error: %s", ncclGetErrorString(async_err));
  }
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_create(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype,
                             gscl_grid_t* out) {
  GSCL_TRY
  NEED_INIT();
  if (!out) return fail(GSCL_E_INVALID_ARG, "out is NULL");
  auto* g = new gscl_grid_s();
  gscl_status s = layout(g, nx, ny, nz, halo, dtype, S.rank, S.world);
  if (s != GSCL_OK) { delete g; return s; }
  cudaError_t e = cudaMalloc(&g->base, g->bytes);
  if (e != cudaSuccess) {
    delete g;
    cudaGetLastError();
    return fail(GSCL_E_OOM, "cudaMalloc(%zu) failed: %s", g->bytes, cudaGetErrorString(e));
  }
  g->owned = true;
  e = cudaMemsetAsync(g->base, 0, g->bytes, S.stream);
  if (e != cudaSuccess) { cudaFree(g->base); delete g; return fail(GSCL_E_CUDA, "memset failed"); }
  S.live.insert(g);
  *out = g;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_wrap(void* dev_ptr, size_t bytes, int64_t nx, int64_t ny, int64_t nz, int halo,
                           gscl_dtype dtype, gscl_grid_t* out) {
  GSCL_TRY
  NEED_INIT();
  if (!out || !dev_ptr) return fail(GSCL_E_INVALID_ARG, "NULL pointer");
  if (reinterpret_cast<uintptr_t>(dev_ptr) % 256 != 0)
    return fail(GSCL_E_INVALID_ARG, "dev_ptr must be 256-byte aligned");
  auto* g = new gscl_grid_s();
  gscl_status s = layout(g, nx, ny, nz, halo, dtype, S.rank, S.world);
  if (s != GSCL_OK) { delete g; return s; }
  if (bytes < g->bytes) {
    size_t need = g->bytes;
    delete g;
    return fail(GSCL_E_INVALID_ARG, "wrapped buffer has %zu bytes, layout needs %zu", bytes, need);
  }
  g->base = dev_ptr;
  g->owned = false;
  S.live.insert(g);
  *out = g;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_destroy(gscl_grid_t g) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  CK(cudaStreamSynchronize(S.stream));
  if (g->owned) CK(cudaFree(g->base));
  if (g->ready) CK(cudaEventDestroy(g->ready));
  S.live.erase(g);
  delete g;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_layout(gscl_grid_t g, int64_t* pitch, int64_t* z_begin, int64_t* z_end,
                             int64_t* origin_offset_elems) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  if (pitch) *pitch = g->pitch;
  if (z_begin) *z_begin = g->z_begin;
  if (z_end) *z_end = g->z_end;
  if (origin_offset_elems) *origin_offset_elems = g->h * g->plane + g->h * g->pitch + g->ox;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_device_ptr(gscl_grid_t g, void** dev_ptr) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  if (!dev_ptr) return fail(GSCL_E_INVALID_ARG, "dev_ptr is NULL");
  *dev_ptr = g->base;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_fill_random(gscl_grid_t g, uint64_t seed, uint32_t grid_id, double scale) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  CK(launch_fill_random(view_of(g), g->z_begin, seed, grid_id, scale, S.stream, &S.launches));
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_fill_const(gscl_grid_t g, double value) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  CK(launch_fill_const(view_of(g), value, S.stream, &S.launches));
  return GSCL_OK;
  GSCL_CATCH
}

// Host <-> device copy of the dense slab.  Large copies go through a device
// staging buffer in chunks of whole planes: one contiguous (full PCIe rate)
// cudaMemcpyAsync per chunk plus an on-device repack into / out of the padded
// layout; small ones use a strided 2-D copy.
static gscl_status host_copy(gscl_grid_t g, void* host, size_t bytes, bool to_host) {
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  if (!host) return fail(GSCL_E_INVALID_ARG, "host pointer is NULL");
  const size_t w = (size_t)(g->nx + 2 * g->h) * g->es;
  const size_t rows_per_plane = (size_t)(g->ny + 2 * g->h);
  const size_t planes = (size_t)(g->nzl + 2 * g->h);
  const size_t rows = rows_per_plane * planes;
  if (bytes != w * rows) return fail(GSCL_E_INVALID_ARG, "host buffer has %zu bytes, dense slab needs %zu", bytes, w * rows);
  const size_t plane_bytes = w * rows_per_plane;
  const size_t kChunk = (size_t)256 << 20;
  if (bytes < ((size_t)8 << 20) || plane_bytes > kChunk) {
    char* dev = static_cast<char*>(g->base) + (size_t)(g->ox - g->h) * g->es;
    const size_t dp = (size_t)g->pitch * g->es;
    if (to_host)
      CK(cudaMemcpy2DAsync(host, w, dev, dp, w, rows, cudaMemcpyDeviceToHost, S.stream));
    else
      CK(cudaMemcpy2DAsync(dev, dp, host, w, w, rows, cudaMemcpyHostToDevice, S.stream));
    CK(cudaStreamSynchronize(S.stream));
    return GSCL_OK;
  }
  const size_t per = std::max<size_t>(1, kChunk / plane_bytes);  // planes per chunk
  const size_t need = per * plane_bytes;
  if (S.stage_cap < need) {
    if (S.d_stage) CK(cudaFree(S.d_stage));
    S.d_stage = nullptr;
    S.stage_cap = 0;
    CK(cudaMalloc(&S.d_stage, need));
    S.stage_cap = need;
  }
  const View v = view_of(g);
  char* hp = static_cast<char*>(host);
  for (size_t p0 = 0; p0 < planes; p0 += per) {
    const size_t np = std::min(per, planes - p0);
    if (to_host) {
      CK(launch_repack(v, S.d_stage, (int64_t)p0, (int64_t)np, false, S.stream, &S.launches));
      CK(cudaMemcpyAsync(hp + p0 * plane_bytes, S.d_stage, np * plane_bytes, cudaMemcpyDeviceToHost, S.stream));
    } else {
      CK(cudaMemcpyAsync(S.d_stage, hp + p0 * plane_bytes, np * plane_bytes, cudaMemcpyHostToDevice, S.stream));
      CK(launch_repack(v, S.d_stage, (int64_t)p0, (int64_t)np, true, S.stream, &S.launches));
    }
  }
  CK(cudaStreamSynchronize(S.stream));
  return GSCL_OK;
}

gscl_status gscl_grid_copy_to_host(gscl_grid_t g, void* host, size_t bytes) {
  GSCL_TRY
  return host_copy(g, host, bytes, true);
  GSCL_CATCH
}

gscl_status gscl_grid_copy_from_host(gscl_grid_t g, const void* host, size_t bytes) {
  GSCL_TRY
  return host_copy(g, const_cast<void*>(host), bytes, false);
  GSCL_CATCH
}

gscl_status gscl_grid_copy_from_host_async(gscl_grid_t g, const void* host, size_t bytes) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  if (!host) return fail(GSCL_E_INVALID_ARG, "host pointer is NULL");
  const size_t w = (size_t)(g->nx + 2 * g->h) * g->es;
  const size_t planes = (size_t)(g->nzl + 2 * g->h);
  const size_t need = w * (size_t)(g->ny + 2 * g->h) * planes;
  if (bytes != need) return fail(GSCL_E_INVALID_ARG, "host buffer has %zu bytes, dense slab needs %zu", bytes, need);
  // the upload must not overwrite storage the library stream still uses
  CK(cudaEventRecord(S.ev_to_copy, S.stream));
  CK(cudaStreamWaitEvent(S.copy_stream, S.ev_to_copy, 0));
  const unsigned slot = S.up_next++ & 1u;  // two staging slots: consecutive uploads overlap
  if (S.up_cap[slot] < bytes) {
    CK(cudaStreamSynchronize(S.copy_stream));
    if (S.up_stage[slot]) CK(cudaFree(S.up_stage[slot]));
    S.up_stage[slot] = nullptr;
    S.up_cap[slot] = 0;
    CK(cudaMalloc(&S.up_stage[slot], bytes));
    S.up_cap[slot] = bytes;
  }
  CK(cudaMemcpyAsync(S.up_stage[slot], host, bytes, cudaMemcpyHostToDevice, S.copy_stream));
  CK(launch_repack(view_of(g), S.up_stage[slot], 0, (int64_t)planes, true, S.copy_stream, &S.launches));
  if (!g->ready) CK(cudaEventCreateWithFlags(&g->ready, cudaEventDisableTiming));
  CK(cudaEventRecord(g->ready, S.copy_stream));
  g->pending = true;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_grid_digest(gscl_grid_t g, uint64_t* out) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  if (!out) return fail(GSCL_E_INVALID_ARG, "out is NULL");
  CK(cudaMemsetAsync(S.d_digest, 0, 8, S.stream));
  CK(launch_digest(view_of(g), g->z_begin, reinterpret_cast<uint64_t*>(S.d_digest), S.stream, &S.launches));
  if (S.world > 1) NK(ncclAllReduce(S.d_digest, S.d_digest, 1, ncclUint64, ncclSum, S.comm, S.stream));
  CK(cudaMemcpyAsync(S.h_pinned, S.d_digest, 8, cudaMemcpyDeviceToHost, S.stream));
  CK(cudaStreamSynchronize(S.stream));
  std::memcpy(out, S.h_pinned, 8);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_swap(gscl_grid_t a, gscl_grid_t b) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(a, "a"); s != GSCL_OK) return s;
  if (gscl_status s = check_grid(b, "b"); s != GSCL_OK) return s;
  if (gscl_status s = same_shape(a, b); s != GSCL_OK) return s;
  if (a->h != b->h) return fail(GSCL_E_SHAPE_MISMATCH, "halo widths differ");
  swap_storage(a, b);
  return GSCL_OK;
  GSCL_CATCH
}

static gscl_status validate_inputs(const gscl_grid_t* in, int n, gscl_grid_t out) {
  for (int i = 0; i < n; ++i) {
    if (gscl_status s = check_grid(in[i], "input grid"); s != GSCL_OK) return s;
    if (gscl_status s = same_shape(in[0], in[i]); s != GSCL_OK) return s;
  }
  if (out) {
    if (gscl_status s = check_grid(out, "out"); s != GSCL_OK) return s;
    if (gscl_status s = same_shape(in[0], out); s != GSCL_OK) return s;
    for (int i = 0; i < n; ++i)
      if (in[i] == out || in[i]->base == out->base)
        return fail(GSCL_E_INVALID_ARG, "out aliases input %d (write-only output, PAPER.md:63)", i);
  }
  return GSCL_OK;
}

gscl_status gscl_do_all(gscl_op op, const gscl_grid_t* in, int n_in, gscl_grid_t out,
                        const gscl_range* range, const double* params, int n_params) {
  GSCL_TRY
  Nvtx nv_call("gscl.do_all");
  (void)params; (void)n_params;
  NEED_INIT();
  if (op < GSCL_OP_FIG1B || op > GSCL_OP_VARCOEF8) return fail(GSCL_E_INVALID_ARG, "unknown op %d", (int)op);
  if (!in) return fail(GSCL_E_INVALID_ARG, "in is NULL");
  if (n_in != op_arity(op)) return fail(GSCL_E_ARITY, "op %d takes %d input grids, got %d", (int)op, op_arity(op), n_in);
  if (!out) return fail(GSCL_E_INVALID_ARG, "out is NULL");
  if (gscl_status s = validate_inputs(in, n_in, out); s != GSCL_OK) return s;
  if (in[0]->h < 1) return fail(GSCL_E_HALO_VIOLATION, "input 0 has halo %d, the op reads offset 1", in[0]->h);
  Box b;
  if (gscl_status s = local_box(out, range, &b); s != GSCL_OK) return s;
  SweepPlan p;
  p.op = op;
  p.rv = RV_NONE;
  p.write = true;
  p.n_in = n_in;
  for (int i = 0; i < n_in; ++i) p.in[i] = view_of(in[i]);
  p.out = view_of(out);
  p.box = b;
  return run_sweep(p);
  GSCL_CATCH
}

gscl_status gscl_do_reduce(gscl_rop rop, const gscl_grid_t* grids, int n, gscl_grid_t out,
                           gscl_combine combine, const gscl_range* range, const double* params,
                           int n_params, double* result) {
  GSCL_TRY
  Nvtx nv_call("gscl.do_reduce");
  NEED_INIT();
  if (rop < GSCL_R_VALUE || rop > GSCL_R_FIG1B_CONV) return fail(GSCL_E_INVALID_ARG, "unknown rop %d", (int)rop);
  if (combine < GSCL_SUM || combine > GSCL_AND) return fail(GSCL_E_INVALID_ARG, "unknown combine %d", (int)combine);
  if (!grids || !result) return fail(GSCL_E_INVALID_ARG, "NULL pointer");
  const int need = (rop == GSCL_R_ABSDIFF || rop == GSCL_R_CONV) ? 2 : 1;
  if (n != need) return fail(GSCL_E_ARITY, "rop %d takes %d grids, got %d", (int)rop, need, n);
  const bool fused = rop >= GSCL_R_JACOBI7_RESID7_SQ;
  if (fused && !out) return fail(GSCL_E_INVALID_ARG, "fused rop %d writes `out`, which is NULL", (int)rop);
  if (!fused && out) return fail(GSCL_E_INVALID_ARG, "rop %d does not write; pass out = NULL", (int)rop);
  if (gscl_status s = validate_inputs(grids, n, out); s != GSCL_OK) return s;
  const bool needs_eps = rop == GSCL_R_CONV || rop == GSCL_R_FIG1B_CONV;
  if (needs_eps && (!params || n_params < 1)) return fail(GSCL_E_INVALID_ARG, "eps (params[0]) required");
  const bool stencil = rop == GSCL_R_RESID7_SQ || rop == GSCL_R_RESID27_SQ || fused;
  if (stencil && grids[0]->h < 1) return fail(GSCL_E_HALO_VIOLATION, "stencil rop needs halo >= 1");
  Box b;
  if (gscl_status s = local_box(grids[0], range, &b); s != GSCL_OK) return s;
  double* d_loc = S.d_scratch;
  RedTarget red = red_target(d_loc, combine);
  if (!stencil) {
    View v[2];
    for (int i = 0; i < n; ++i) v[i] = view_of(grids[i]);
    if (b.empty()) {
      CK(launch_fold(nullptr, 0, combine, d_loc, S.stream, &S.launches));
    } else {
      CK(launch_reduce_points((int)rop, v, n, b, needs_eps ? params[0] : 0.0, red, S.num_sms,
                              S.stream, &S.launches));
    }
  } else {
    SweepPlan p;
    p.n_in = 1;
    p.in[0] = view_of(grids[0]);
    p.box = b;
    p.red = red;
    p.eps = needs_eps ? params[0] : 0.0;
    switch (rop) {
      case GSCL_R_RESID7_SQ: p.op = OP_JACOBI7; p.rv = RV_RESID; p.write = false; break;
      case GSCL_R_RESID27_SQ: p.op = OP_JACOBI27; p.rv = RV_RESID; p.write = false; break;
      case GSCL_R_JACOBI7_RESID7_SQ: p.op = OP_JACOBI7; p.rv = RV_RESID; p.write = true; break;
      case GSCL_R_JACOBI27_RESID27_SQ: p.op = OP_JACOBI27; p.rv = RV_RESID; p.write = true; break;
      default: p.op = OP_FIG1B; p.rv = RV_CONV; p.write = true; break;
    }
    if (p.write) p.out = view_of(out);
    if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
  }
  if (gscl_status s = cross_rank(d_loc, combine, d_loc, S.stream); s != GSCL_OK) return s;
  CK(cudaMemcpyAsync(S.h_pinned, d_loc, 8, cudaMemcpyDeviceToHost, S.stream));
  CK(cudaStreamSynchronize(S.stream));
  *result = S.h_pinned[0];
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_halo_exchange(const gscl_grid_t* grids, int n) {
  GSCL_TRY
  Nvtx nv_call("gscl.halo_exchange");
  NEED_INIT();
  if (n < 0 || (n > 0 && !grids)) return fail(GSCL_E_INVALID_ARG, "bad grid list");
  for (int i = 0; i < n; ++i)
    if (gscl_status s = check_grid(grids[i], "grid"); s != GSCL_OK) return s;
  for (int i = 0; i < n; ++i)
    if (gscl_status s = exchange(grids[i]); s != GSCL_OK) return s;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_pass_units(int64_t nx, int64_t ny, gscl_dtype dtype, int64_t* units) {
  GSCL_TRY
  if (!units || nx <= 0 || ny <= 0 || (dtype != GSCL_F64 && dtype != GSCL_F32))
    return fail(GSCL_E_INVALID_ARG, "bad arguments");
  *units = pass_tiles(nx, ny, dtype == GSCL_F64 ? 0 : 1, S.variant);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_do_all_pass2(gscl_op op, gscl_grid_t in, gscl_grid_t out, const void* ghost, int phys_lo,
                              int phys_hi, const gscl_pass_peer* peer) {
  GSCL_TRY
  Nvtx nv_call("gscl.do_all_pass2");
  NEED_INIT();
  if (op != GSCL_OP_JACOBI7) return fail(GSCL_E_UNSUPPORTED, "two-sweep passes support JACOBI7 (got %d)", (int)op);
  if (gscl_status s = check_grid(in, "in"); s != GSCL_OK) return s;
  if (gscl_status s = check_grid(out, "out"); s != GSCL_OK) return s;
  if (gscl_status s = same_shape(in, out); s != GSCL_OK) return s;
  if (in == out || in->base == out->base) return fail(GSCL_E_INVALID_ARG, "in and out alias");
  if (in->h < 1) return fail(GSCL_E_HALO_VIOLATION, "in needs halo >= 1");
  if (!ghost && in->h < 2 && (!phys_lo || !phys_hi))
    return fail(GSCL_E_INVALID_ARG, "ghost planes are needed for a non-physical z side when halo < 2");
  Box full;
  if (gscl_status s = local_box(in, nullptr, &full); s != GSCL_OK) return s;
  if (full.empty()) return GSCL_OK;
  SweepPlan p;
  p.op = OP_JACOBI7;
  p.n_in = 1;
  p.in[0] = view_of(in);
  p.out = view_of(out);
  p.box = full;
  p.write = true;
  p.tsteps = 2;
  p.phys_lo = phys_lo != 0;
  p.phys_hi = phys_hi != 0;
  p.ghost = ghost;
  if (peer) {
    if (in->nzl < 6) return fail(GSCL_E_INVALID_DOMAIN, "the peer transport needs >= 6 planes per slab");
    p.bnd_h = 1;  // boundary-first units carry the remote stores
    for (int i = 0; i < 2; ++i) {
      p.peer_lo[i] = peer->lo[i];
      p.peer_hi[i] = peer->hi[i];
    }
    p.peer_flag_lo = peer->lo_flag;
    p.peer_flag_hi = peer->hi_flag;
  }
  return run_sweep(p);
  GSCL_CATCH
}

// The device work of one gscl_jacobi_run (everything but the history copy and
// the host sync), issued on the library streams; *final_in_v reports whether
// the final iterate ends in v's storage.
// Whether jacobi_run takes the multi-rank two-sweep schedule: JACOBI7 on the
// TMA path, tblock auto or 2, several ranks (or "split" on one), and at least 6
// planes on every rank (2 boundary planes per end + the interior; the same
// decision on every rank, so the NCCL call sequences match).
static bool pairs_multirank(gscl_op op, const gscl_grid_s* u) {
  return op == GSCL_OP_JACOBI7 && S.impl == 0 && (S.tblock == 0 || S.tblock == 2) &&
         (S.world > 1 || S.split) && u->nz / S.world >= 6 && u->nx > 0 && u->ny > 0;
}

// The multi-rank two-sweep schedule over the peer-memory transport (option
// transport = 1, after gscl_peer_export / gscl_peer_import): no NCCL and no
// comm-stream exchange.  Each pass's boundary units store their planes
// straight into the neighbours' next-input halo / ghost planes (IPC / NVLink
// mappings) and bump the neighbours' arrival counters; before its next pass a
// rank's stream waits (cuStreamWaitValue32) until both neighbours' counters
// say their previous pass's boundary planes have landed — which also means
// they have finished reading the planes this pass overwrites.  Two ghost
// buffers (one per input storage) keep a neighbour's early writes for pass
// k+1 away from the planes this rank still reads in pass k.  Unpaired single
// sweeps copy their boundary planes with cudaMemcpyAsync and signal the same
// counters.  Residual checks: each rank publishes its partial into every
// rank's slot array (peer stores + a counter), and the comm stream folds the
// slots in rank order once all have arrived (R14).  A start barrier
// (two counter rounds) orders this call's setup copies after the neighbours'
// previous calls.
static gscl_status enqueue_jacobi_p2p(gscl_op op, gscl_grid_s* u, gscl_grid_s* v, const gscl_grid_t* coeffs,
                                      int nc, int iters, int check_every, int nh, bool* final_in_v) {
  PeerSet& P = S.peer;
  // JACOBI7 pairs sweeps into two-sweep passes (a slab needs >= 6 planes);
  // JACOBI27 / VARCOEF8 run single sweeps whose boundary planes are copied
  const bool can_pair = op == GSCL_OP_JACOBI7 && S.impl == 0 && (S.tblock == 0 || S.tblock == 2) &&
                        u->nz / S.world >= 6;
  const int check_rv = op == GSCL_OP_VARCOEF8 ? RV_SQ : RV_RESID;
  // operators that never pair (JACOBI27, VARCOEF8): their sweeps store the
  // boundary planes into the neighbours from the kernel (the h planes each
  // next sweep needs); JACOBI7's unpaired steps copy 2 planes (a pass follows)
  const bool fuse_single = op != GSCL_OP_JACOBI7 && S.impl == 0 && u->nz / S.world > 2 * u->h;
  int cur;  // storage index of the current input
  if (u->base == P.store_base[0] && v->base == P.store_base[1]) cur = 0;
  else if (u->base == P.store_base[1] && v->base == P.store_base[0]) cur = 1;
  else return fail(GSCL_E_INVALID_ARG, "u / v are not the grids of gscl_peer_export");
  const View vu = view_of(u), vv = view_of(v);
  CK(launch_copy_halo(vu, vv, S.stream, &S.launches));  // Dirichlet shell travels (R11)
  Box full;
  if (gscl_status s = local_box(u, nullptr, &full); s != GSCL_OK) return s;
  struct Step { bool pair, check; int slot; };
  std::vector<Step> steps;
  for (int it = 1; it <= iters; ++it) {
    const bool check = check_every > 0 && it % check_every == 0;
    if (can_pair && !check && it + 1 <= iters) {
      const bool c2 = check_every > 0 && (it + 1) % check_every == 0;
      steps.push_back({true, c2, c2 ? (it + 1) / check_every - 1 : -1});
      ++it;
    } else {
      steps.push_back({false, check, check ? it / check_every - 1 : -1});
    }
  }
  const size_t pb = P.plane_bytes;
  const int64_t h = u->h, n = u->nzl;
  const bool lo = S.rank > 0, hi = S.rank < S.world - 1;
  char* my_ar = P.arena_of[S.rank];
  unsigned* my_flags = PeerSet::flags_of(my_ar, pb);
  unsigned* lo_flags = lo ? PeerSet::flags_of(P.arena_of[S.rank - 1], pb) : nullptr;
  unsigned* hi_flags = hi ? PeerSet::flags_of(P.arena_of[S.rank + 1], pb) : nullptr;
  const int64_t es = u->es;
  auto plane_ptr = [&](void* base, int64_t z) {  // start of local plane z of a storage
    return static_cast<char*>(base) + (z + h) * pb;
  };
  auto origin = [&](char* plane_start) {  // interior (0,0) of a plane
    return static_cast<void*>(plane_start + (h * u->pitch + u->ox) * es);
  };
  // receiving plane k (0 nearest) on a neighbour for an output in storage st
  auto recv_plane = [&](int side, int st, int k) -> char* {
    if (side == 0) {  // lower: its planes nzl, nzl+1
      const int64_t z = P.nzl_nb[0] + k;
      if (z < P.nzl_nb[0] + h) return plane_ptr(P.nb_store[0][st], z);
      return PeerSet::ghost_of(P.arena_of[S.rank - 1], pb, st) + pb;  // its ghost plane "above"
    }
    const int64_t z = -1 - k;  // upper: its planes -1, -2
    if (z >= -h) return plane_ptr(P.nb_store[1][st], z);
    return PeerSet::ghost_of(P.arena_of[S.rank + 1], pb, st);  // its ghost plane "below"
  };
  auto signal = [&](unsigned* lof, unsigned* hif, unsigned add) -> gscl_status {
    PeerPtrs8 f{};
    if (lof) f.p[f.n++] = lof;
    if (hif) f.p[f.n++] = hif;
    if (f.n) CK(launch_signal(f, add, S.stream, &S.launches));
    return GSCL_OK;
  };
  auto wait_nb = [&](int idx_lo, int idx_hi) -> gscl_status {
    if (lo) CK(stream_wait_geq(S.stream, my_flags + idx_lo, P.tgt[idx_lo]));
    if (hi) CK(stream_wait_geq(S.stream, my_flags + idx_hi, P.tgt[idx_hi]));
    return GSCL_OK;
  };
  // copy whole boundary planes of storage st (both depths) into the neighbours
  auto copy_planes = [&](int st) -> gscl_status {
    for (int k = 0; k < 2; ++k) {
      if (lo) CK(cudaMemcpyAsync(recv_plane(0, st, k), plane_ptr(P.store_base[st], k), pb,
                                 cudaMemcpyDeviceToDevice, S.stream));
      if (hi) CK(cudaMemcpyAsync(recv_plane(1, st, k), plane_ptr(P.store_base[st], n - 1 - k), pb,
                                 cudaMemcpyDeviceToDevice, S.stream));
    }
    return GSCL_OK;
  };
  // ---- start barrier: neighbours are done with the previous call; setup copies
  // of both storages (the x/y boundary ring of every receiving plane, and the
  // first input's planes); second barrier round: their copies into us landed
  for (int round = 0; round < 2; ++round) {
    if (round == 1) {
      if (gscl_status s = copy_planes(cur); s != GSCL_OK) return s;
      if (gscl_status s = copy_planes(1 - cur); s != GSCL_OK) return s;
    }
    if (gscl_status s = signal(lo ? lo_flags + 3 : nullptr, hi ? hi_flags + 2 : nullptr, 1); s != GSCL_OK)
      return s;
    if (lo) ++P.tgt[2];
    if (hi) ++P.tgt[3];
    if (gscl_status s = wait_nb(2, 3); s != GSCL_OK) return s;
  }
  cudaStream_t CS = S.comm_stream;
  // residual partial -> every rank's slot q; the comm stream folds slot q
  auto check_combine = [&](double* loc, double* glob) -> gscl_status {
    const unsigned q = P.red_next++ % kRedSlots;
    PeerPtrs8 dst{}, cnt{};
    for (int r = 0; r < S.world; ++r) {
      dst.p[dst.n++] = PeerSet::red_of(P.arena_of[r], pb) + (size_t)q * S.world + S.rank;
      cnt.p[cnt.n++] = PeerSet::flags_of(P.arena_of[r], pb) + 4;
    }
    CK(launch_publish(loc, dst, cnt, S.stream, &S.launches));
    P.tgt[4] += (unsigned)S.world;
    if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
    CK(stream_wait_geq(CS, my_flags + 4, P.tgt[4]));
    CK(launch_fold(PeerSet::red_of(my_ar, pb) + (size_t)q * S.world, S.world, GSCL_SUM, glob, CS,
                   &S.launches));
    return GSCL_OK;
  };
  View a = vu, b = vv;
  gscl_grid_s* ga = u;
  gscl_grid_s* gb = v;
  for (size_t k = 0; k < steps.size(); ++k) {
    const Step& st = steps[k];
    if (k > 0)
      if (gscl_status s = wait_nb(0, 1); s != GSCL_OK) return s;
    double* glob = st.check ? S.d_hist + st.slot : nullptr;
    double* loc = st.check ? S.d_lochist + st.slot : nullptr;
    SweepPlan p;
    p.op = op;
    p.n_in = 1 + nc;
    p.in[0] = a;
    for (int i = 0; i < nc; ++i) p.in[1 + i] = view_of(coeffs[i]);
    p.out = b;
    p.box = full;
    p.write = true;
    p.rv = st.check ? (st.pair ? RV_RESID : check_rv) : RV_NONE;
    if (st.check) p.red = red_target(loc, GSCL_SUM);
    const int out_st = 1 - cur;
    unsigned inc = (unsigned)P.units;  // what each neighbour's counter grows by this step
    if (st.pair) {
      p.tsteps = 2;
      p.phys_lo = !lo;
      p.phys_hi = !hi;
      p.ghost = PeerSet::ghost_of(my_ar, pb, cur);
      p.bnd_h = 1;
      for (int i = 0; i < 2; ++i) {
        p.peer_lo[i] = lo ? origin(recv_plane(0, out_st, i)) : nullptr;
        p.peer_hi[i] = hi ? origin(recv_plane(1, out_st, i)) : nullptr;
      }
      p.peer_flag_lo = lo ? lo_flags + 1 : nullptr;  // the lower neighbour hears from above
      p.peer_flag_hi = hi ? hi_flags + 0 : nullptr;
      int64_t units = 0;
      p.bnd_units = &units;
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      if (units != 2 * P.units)  // (tiles at each end)
        return fail(GSCL_E_STATE, "pass boundary units %lld != 2 x %lld", (long long)units, (long long)P.units);
    } else if (fuse_single) {
      // one sweep whose boundary units (the h planes at each end, first) also
      // store those planes into the neighbours' halo planes and bump their
      // counters: the transfer overlaps the interior units of the same launch
      p.bnd_h = (int)h;
      for (int i = 0; i < 2 && i < h; ++i) {
        p.peer_lo[i] = lo ? origin(recv_plane(0, out_st, i)) : nullptr;
        p.peer_hi[i] = hi ? origin(recv_plane(1, out_st, i)) : nullptr;
      }
      p.peer_flag_lo = lo ? lo_flags + 1 : nullptr;
      p.peer_flag_hi = hi ? hi_flags + 0 : nullptr;
      int64_t units = 0;
      p.bnd_units = &units;
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      inc = (unsigned)(units / 2);
    } else {
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      if (gscl_status s = copy_planes(out_st); s != GSCL_OK) return s;
      if (gscl_status s = signal(lo ? lo_flags + 1 : nullptr, hi ? hi_flags + 0 : nullptr, (unsigned)P.units);
          s != GSCL_OK)
        return s;
    }
    if (lo) P.tgt[0] += inc;
    if (hi) P.tgt[1] += inc;
    if (st.check)
      if (gscl_status s = check_combine(loc, glob); s != GSCL_OK) return s;
    std::swap(a, b);
    std::swap(ga, gb);
    cur = out_st;
  }
  if (check_every > 0) {  // the final iterate's neighbour planes: the last step's signal
    if (!steps.empty())
      if (gscl_status s = wait_nb(0, 1); s != GSCL_OK) return s;
    double* glob = S.d_hist + (nh - 1);
    double* loc = S.d_lochist + (nh - 1);
    if (op == GSCL_OP_VARCOEF8) {
      CK(launch_reduce_points(1 /*SQ*/, &a, 1, full, 0.0, red_target(loc, GSCL_SUM), S.num_sms, S.stream,
                              &S.launches));
    } else {
      SweepPlan p;
      p.op = op;
      p.rv = RV_RESID;
      p.write = false;
      p.n_in = 1;
      p.in[0] = a;
      p.box = full;
      p.red = red_target(loc, GSCL_SUM);
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
    }
    if (gscl_status s = check_combine(loc, glob); s != GSCL_OK) return s;
  }
  if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
  *final_in_v = (ga != u);
  return GSCL_OK;
}

// JACOBI7 as two-sweep passes on a z-slab of several ranks (or one rank with
// the "split" option): temporal blocking with a depth-2 halo.  Every pass is
// ONE launch whose first units compute the 2 output planes at each end of the
// slab and bump d_bflag; the comm stream waits for the counter
// (cuStreamWaitValue32) and runs the depth-2 NCCL exchange of those planes
// (into the next input's halo plane and the ghost buffer) while the interior
// units of the same launch still run; the next pass waits for the exchange.
// A check pass reduces the residual of its intermediate iterate into a
// per-check slot, combined across ranks on the comm stream after the pass.
// Check sweeps that cannot be paired (odd check_every) run as single fused
// sweeps with a depth-1 exchange.  Same results, bit for bit, as single sweeps.
static gscl_status enqueue_jacobi_pairs(gscl_grid_s* u, gscl_grid_s* v, int iters, int check_every, int nh,
                                        bool* final_in_v) {
  const View vu = view_of(u), vv = view_of(v);
  CK(launch_copy_halo(vu, vv, S.stream, &S.launches));  // Dirichlet shell travels (R11)
  Box full;
  if (gscl_status s = local_box(u, nullptr, &full); s != GSCL_OK) return s;
  struct Step { bool pair, check; int slot; };
  std::vector<Step> steps;
  for (int it = 1; it <= iters; ++it) {
    const bool check = check_every > 0 && it % check_every == 0;
    if (!check && it + 1 <= iters) {
      const bool c2 = check_every > 0 && (it + 1) % check_every == 0;
      steps.push_back({true, c2, c2 ? (it + 1) / check_every - 1 : -1});
      ++it;
    } else {
      steps.push_back({false, check, check ? it / check_every - 1 : -1});
    }
  }
  const bool multi = S.world > 1;
  cudaStream_t CS = S.comm_stream;
  if (multi && u->h < 2)
    if (gscl_status s = ensure_ghost(2 * (size_t)(u->plane * (int64_t)u->es)); s != GSCL_OK) return s;
  auto xchg = [&](gscl_grid_s* g, int depth) { return depth == 2 ? exchange_pass(g, CS) : exchange(g, CS); };
  auto depth_of = [&](size_t k) { return k < steps.size() && steps[k].pair ? 2 : 1; };
  View a = vu, b = vv;
  gscl_grid_s* ga = u;
  gscl_grid_s* gb = v;
  if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
  if (gscl_status s = xchg(ga, depth_of(0)); s != GSCL_OK) return s;
  if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
  for (size_t k = 0; k < steps.size(); ++k) {
    const Step& st = steps[k];
    double* glob = st.check ? S.d_hist + st.slot : nullptr;
    double* res = st.check ? (multi ? S.d_lochist + st.slot : glob) : nullptr;
    const int next = depth_of(k + 1);
    SweepPlan p;
    p.op = OP_JACOBI7;
    p.n_in = 1;
    p.in[0] = a;
    p.out = b;
    p.box = full;
    p.write = true;
    p.rv = st.check ? RV_RESID : RV_NONE;
    if (st.check) p.red = red_target(res, GSCL_SUM);
    if (st.pair) {
      p.tsteps = 2;
      p.phys_lo = S.rank == 0;
      p.phys_hi = S.rank == S.world - 1;
      p.ghost = S.d_ghost;
      p.bnd_h = 1;
      p.bflag = S.d_bflag;
      int64_t units = 0;
      p.bnd_units = &units;
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      if (st.check && multi) CK(cudaEventRecord(S.ev_to_comm, S.stream));  // the pass's end
      if (units > 0) {
        S.bflag_target += (unsigned)units;
        CK(stream_wait_geq(CS, S.d_bflag, S.bflag_target));
      } else {
        CK(cudaEventRecord(S.ev_to_main, S.stream));
        CK(cudaStreamWaitEvent(CS, S.ev_to_main, 0));
      }
      if (gscl_status s = xchg(gb, next); s != GSCL_OK) return s;
      CK(cudaEventRecord(S.ev_halo, CS));
      if (st.check && multi) {
        CK(cudaStreamWaitEvent(CS, S.ev_to_comm, 0));
        if (gscl_status s = cross_rank(res, GSCL_SUM, glob, CS); s != GSCL_OK) return s;
      }
      CK(cudaStreamWaitEvent(S.stream, S.ev_halo, 0));
    } else {
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
      if (st.check && multi)
        if (gscl_status s = cross_rank(res, GSCL_SUM, glob, CS); s != GSCL_OK) return s;
      if (gscl_status s = xchg(gb, next); s != GSCL_OK) return s;
      if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
    }
    std::swap(a, b);
    std::swap(ga, gb);
  }
  if (check_every > 0) {  // the final iterate's halo arrived with the last exchange
    double* glob = S.d_hist + (nh - 1);
    double* res = multi ? S.d_lochist + (nh - 1) : glob;
    SweepPlan p;
    p.op = OP_JACOBI7;
    p.rv = RV_RESID;
    p.write = false;
    p.n_in = 1;
    p.in[0] = a;
    p.box = full;
    p.red = red_target(res, GSCL_SUM);
    if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
    if (multi) {
      if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
      if (gscl_status s = cross_rank(res, GSCL_SUM, glob, CS); s != GSCL_OK) return s;
    }
  }
  // the library stream ends after all comm-stream work of the run
  if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
  *final_in_v = (ga != u);
  return GSCL_OK;
}

static gscl_status enqueue_jacobi(gscl_op op, gscl_grid_s* u, gscl_grid_s* v, const gscl_grid_t* coeffs,
                                  int nc, int iters, int check_every, int nh, bool* final_in_v) {
  if (S.transport == 1 && S.world > 1) {
    if (!S.peer.ready) return fail(GSCL_E_STATE, "transport = 1 needs gscl_peer_export / gscl_peer_import");
    if (u->nz / S.world < 2) return fail(GSCL_E_INVALID_DOMAIN, "the peer transport needs >= 2 planes per rank");
    return enqueue_jacobi_p2p(op, u, v, coeffs, nc, iters, check_every, nh, final_in_v);
  }
  if (pairs_multirank(op, u)) return enqueue_jacobi_pairs(u, v, iters, check_every, nh, final_in_v);
  View vu = view_of(u), vv = view_of(v);
  CK(launch_copy_halo(vu, vv, S.stream, &S.launches));  // Dirichlet shell travels (R11)
  Box full;
  if (gscl_status s = local_box(u, nullptr, &full); s != GSCL_OK) return s;
  View a = vu, bview = vv;
  gscl_grid_s* ga = u;
  gscl_grid_s* gb = v;
  const int check_rv = op == GSCL_OP_VARCOEF8 ? RV_SQ : RV_RESID;
  double* d_loc = S.d_scratch;
  const int64_t h = u->h;
  cudaStream_t CS = S.comm_stream;
  // Overlapped schedule (multi-rank, or forced with the "split" option): the
  // h boundary planes at each end of the slab are swept first, their halo
  // exchange runs on the comm stream while the interior sweeps, and the next
  // sweep waits for the exchange.  All NCCL work of the loop is on CS.
  const bool split = (S.world > 1 || S.split) && S.impl == 0 && full.z1 - full.z0 > 2 * h;
  int nsweep = 0;  // alternate the chunk walk so each sweep starts in L2-resident planes
  auto sweep = [&](const View& in, const View& out, const Box& box, int rv, double* res) {
    SweepPlan p;
    p.reverse = S.zalt && (nsweep++ & 1);
    p.op = op;
    p.n_in = 1 + nc;
    p.in[0] = in;
    for (int i = 0; i < nc; ++i) p.in[1 + i] = view_of(coeffs[i]);
    p.out = out;
    p.box = box;
    p.write = true;
    p.rv = rv;
    if (rv != RV_NONE) p.red = red_target(res, GSCL_SUM);
    return run_sweep(p);
  };
  if (split) {  // ghost planes of the first input
    if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
    if (gscl_status s = exchange(ga, CS); s != GSCL_OK) return s;
    if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
  }
  // Temporal blocking (NEXT-2): on a single rank, JACOBI7 sweeps it and it+1
  // run as one two-sweep pass unless sweep it itself carries a check (the
  // pass can reduce the residual of its intermediate = the input of it+1).
  // (auto: every single-rank JACOBI7 run of the default TMA path; the split
  // schedule and the plain-kernel ablation keep single sweeps unless forced)
  const bool pairs = (S.tblock == 2 || (S.tblock == 0 && !S.split && S.impl == 0)) && S.world == 1 &&
                     op == GSCL_OP_JACOBI7 && !full.empty();
  for (int it = 1; it <= iters; ++it) {
    const bool check = check_every > 0 && it % check_every == 0;
    double* slot = S.d_hist + (it / std::max(check_every, 1) - 1);
    double* res = S.world == 1 ? slot : d_loc;
    if (pairs && !check && it + 1 <= iters) {
      const bool check2 = check_every > 0 && (it + 1) % check_every == 0;
      SweepPlan p;
      p.op = op;
      p.n_in = 1;
      p.in[0] = a;
      p.out = bview;
      p.box = full;
      p.write = true;
      p.tsteps = 2;
      p.rv = check2 ? RV_RESID : RV_NONE;
      if (check2) p.red = red_target(S.d_hist + ((it + 1) / check_every - 1), GSCL_SUM);
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      std::swap(a, bview);
      std::swap(ga, gb);
      ++it;  // two sweeps done
      continue;
    }
    if (!split) {
      if (gscl_status s = exchange(ga); s != GSCL_OK) return s;
      if (gscl_status s = sweep(a, bview, full, check ? check_rv : RV_NONE, res); s != GSCL_OK) return s;
      if (check && S.world > 1)
        if (gscl_status s = cross_rank(d_loc, GSCL_SUM, slot, S.stream); s != GSCL_OK) return s;
    } else if (check) {
      // check sweeps are not split: one fused pass, then combine + exchange on CS
      if (gscl_status s = sweep(a, bview, full, check_rv, res); s != GSCL_OK) return s;
      if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
      if (S.world > 1)
        if (gscl_status s = cross_rank(d_loc, GSCL_SUM, slot, CS); s != GSCL_OK) return s;
      if (gscl_status s = exchange(gb, CS); s != GSCL_OK) return s;
      if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
    } else {
      // one launch whose first units sweep the h planes at each end of the
      // slab; each bumps d_bflag after its stores, and the comm stream waits
      // for the counter (cuStreamWaitValue32) before the NCCL exchange of those
      // planes, which thus overlaps the interior units of the same launch
      SweepPlan p;
      p.op = op;
      p.n_in = 1 + nc;
      p.in[0] = a;
      for (int i = 0; i < nc; ++i) p.in[1 + i] = view_of(coeffs[i]);
      p.out = bview;
      p.box = full;
      p.write = true;
      p.rv = RV_NONE;
      p.bnd_h = (int)h;
      p.bflag = S.d_bflag;
      int64_t units = 0;
      p.bnd_units = &units;
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      S.bflag_target += (unsigned)units;
      CK(stream_wait_geq(CS, S.d_bflag, S.bflag_target));
      if (gscl_status s = exchange(gb, CS); s != GSCL_OK) return s;
      CK(cudaEventRecord(S.ev_halo, CS));
      CK(cudaStreamWaitEvent(S.stream, S.ev_halo, 0));
    }
    std::swap(a, bview);
    std::swap(ga, gb);
  }
  if (check_every > 0) {
    double* slot = S.d_hist + (nh - 1);
    double* res = S.world == 1 ? slot : d_loc;
    if (!split)
      if (gscl_status s = exchange(ga); s != GSCL_OK) return s;  // (split: already received)
    if (op == GSCL_OP_VARCOEF8) {
      RedTarget red = red_target(res, GSCL_SUM);
      if (full.empty()) CK(launch_fold(nullptr, 0, GSCL_SUM, red.result, S.stream, &S.launches));
      else CK(launch_reduce_points(1 /*SQ*/, &a, 1, full, 0.0, red, S.num_sms, S.stream, &S.launches));
    } else {
      SweepPlan p;
      p.op = op;
      p.rv = RV_RESID;
      p.write = false;
      p.n_in = 1;
      p.in[0] = a;
      p.box = full;
      p.red = red_target(res, GSCL_SUM);
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
    }
    if (S.world > 1) {
      if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
      if (gscl_status s = cross_rank(d_loc, GSCL_SUM, slot, CS); s != GSCL_OK) return s;
      if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
    }
  }
  *final_in_v = (ga != u);
  return GSCL_OK;
}

gscl_status gscl_jacobi_run(gscl_op op, gscl_grid_t u, gscl_grid_t v, const gscl_grid_t* coeffs,
                            int n_coeffs, int iters, int check_every, double* history) {
  GSCL_TRY
  Nvtx nv_call("gscl.jacobi_run");
  NEED_INIT();
  if (op != GSCL_OP_JACOBI7 && op != GSCL_OP_JACOBI27 && op != GSCL_OP_VARCOEF8)
    return fail(GSCL_E_UNSUPPORTED, "jacobi_run supports JACOBI7, JACOBI27, VARCOEF8 (got %d)", (int)op);
  if (iters < 0 || check_every < 0) return fail(GSCL_E_INVALID_ARG, "negative iters/check_every");
  if (check_every > 0 && !history) return fail(GSCL_E_INVALID_ARG, "history is NULL but check_every > 0");
  if (gscl_status s = check_grid(u, "u"); s != GSCL_OK) return s;
  if (gscl_status s = check_grid(v, "v"); s != GSCL_OK) return s;
  if (gscl_status s = same_shape(u, v); s != GSCL_OK) return s;
  if (u == v || u->base == v->base) return fail(GSCL_E_INVALID_ARG, "u and v alias");
  if (u->h != v->h) return fail(GSCL_E_SHAPE_MISMATCH, "u and v halo widths differ");
  if (u->h < 1) return fail(GSCL_E_HALO_VIOLATION, "u needs halo >= 1");
  const int nc = op == GSCL_OP_VARCOEF8 ? 7 : 0;
  if (n_coeffs != nc) return fail(GSCL_E_ARITY, "op %d takes %d coefficient grids, got %d", (int)op, nc, n_coeffs);
  if (nc) {
    if (!coeffs) return fail(GSCL_E_INVALID_ARG, "coeffs is NULL");
    for (int i = 0; i < nc; ++i) {
      if (gscl_status s = check_grid(coeffs[i], "coefficient grid"); s != GSCL_OK) return s;
      if (gscl_status s = same_shape(u, coeffs[i]); s != GSCL_OK) return s;
      if (coeffs[i]->base == u->base || coeffs[i]->base == v->base)
        return fail(GSCL_E_INVALID_ARG, "coefficient grid aliases u or v");
    }
  }
  const int nh = check_every > 0 ? iters / check_every + 1 : 0;
  if (gscl_status s = ensure_hist((size_t)std::max(nh, 1)); s != GSCL_OK) return s;

  bool final_in_v = false;
  const int64_t local_pts = u->nx * u->ny * u->nzl;
  // (not with the overlapped schedule: its stream-wait targets change per call)
  const bool overlapped = ((S.world > 1 || S.split) && S.impl == 0 && u->nzl > 2 * u->h) ||
                          pairs_multirank(op, u) || (S.transport == 1 && S.world > 1);
  const bool use_graph = !overlapped && (S.graph == 1 || (S.graph == 0 && !S.timing &&
                                                          local_pts <= (int64_t(1) << 24)));
  if (use_graph) {
    // small grids are launch-bound: the whole launch sequence is captured once
    // per (storage, shape, schedule, options) and replayed as one CUDA graph
    std::vector<int64_t> key = {(int64_t)op, (int64_t)(uintptr_t)u->base, (int64_t)(uintptr_t)v->base,
                                u->nx, u->ny, u->nz, u->h, u->dtype, iters, check_every,
                                (int64_t)(uintptr_t)S.d_hist, S.impl, S.zchunks, S.sched, S.stages,
                                S.l2promo, S.split, S.tblock, S.variant, S.zalt};
    for (int i = 0; i < nc; ++i) key.push_back((int64_t)(uintptr_t)coeffs[i]->base);
    GraphEntry* hit = nullptr;
    for (auto& e : S.graphs)
      if (e.key == key) hit = &e;
    if (hit) {
      CK(cudaGraphLaunch(hit->exec, S.stream));
      S.launches += hit->kernels;
      final_in_v = hit->final_in_v;
    } else {
      CK(cudaStreamBeginCapture(S.stream, cudaStreamCaptureModeRelaxed));
      const int64_t l0 = S.launches;
      gscl_status st = enqueue_jacobi(op, u, v, coeffs, nc, iters, check_every, nh, &final_in_v);
      cudaGraph_t g = nullptr;
      cudaError_t ec = cudaStreamEndCapture(S.stream, &g);
      if (st != GSCL_OK) {
        if (g) cudaGraphDestroy(g);
        return st;
      }
      if (ec != cudaSuccess) return fail(GSCL_E_CUDA, "graph capture failed: %s", cudaGetErrorString(ec));
      GraphEntry e;
      e.key = key;
      e.kernels = S.launches - l0;
      e.final_in_v = final_in_v;
      cudaError_t ei = cudaGraphInstantiate(&e.exec, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) return fail(GSCL_E_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ei));
      if (S.graphs.size() >= 16) {
        cudaGraphExecDestroy(S.graphs.front().exec);
        S.graphs.erase(S.graphs.begin());
      }
      S.graphs.push_back(e);
      CK(cudaGraphLaunch(e.exec, S.stream));
    }
  } else {
    if (gscl_status st = enqueue_jacobi(op, u, v, coeffs, nc, iters, check_every, nh, &final_in_v);
        st != GSCL_OK)
      return st;
  }
  if (check_every > 0)
    CK(cudaMemcpyAsync(history, S.d_hist, (size_t)nh * sizeof(double), cudaMemcpyDeviceToHost, S.stream));
  CK(cudaStreamSynchronize(S.stream));
  for (int i = 0; i < nh; ++i) history[i] = std::sqrt(history[i]);
  if (final_in_v) swap_storage(u, v);  // u holds the final iterate on return
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_converge_run(gscl_op op, gscl_grid_t u, gscl_grid_t v, double eps, int max_iters,
                              int batch, int* iters_done, int* converged) {
  GSCL_TRY
  Nvtx nv_call("gscl.converge_run");
  NEED_INIT();
  if (op != GSCL_OP_FIG1B && op != GSCL_OP_JACOBI7)
    return fail(GSCL_E_UNSUPPORTED, "converge_run supports FIG1B and JACOBI7 (got %d)", (int)op);
  if (max_iters < 0 || batch < 0) return fail(GSCL_E_INVALID_ARG, "negative max_iters/batch");
  if (!iters_done || !converged) return fail(GSCL_E_INVALID_ARG, "NULL output pointer");
  if (gscl_status s = check_grid(u, "u"); s != GSCL_OK) return s;
  if (gscl_status s = check_grid(v, "v"); s != GSCL_OK) return s;
  if (gscl_status s = same_shape(u, v); s != GSCL_OK) return s;
  if (u == v || u->base == v->base) return fail(GSCL_E_INVALID_ARG, "u and v alias");
  if (u->h != v->h) return fail(GSCL_E_SHAPE_MISMATCH, "u and v halo widths differ");
  if (u->h < 1) return fail(GSCL_E_HALO_VIOLATION, "u needs halo >= 1");
  if (batch == 0) batch = 16;
  View a = view_of(u), b = view_of(v);
  CK(launch_copy_halo(a, b, S.stream, &S.launches));  // Dirichlet shell travels (R11)
  CK(cudaMemsetAsync(S.d_conv, 0, 8 * sizeof(int), S.stream));
  Box full;
  if (gscl_status s = local_box(u, nullptr, &full); s != GSCL_OK) return s;
  gscl_grid_s* ga = u;
  gscl_grid_s* gb = v;
  double* d_loc = S.d_scratch;       // this rank's AND of the iteration
  double* d_res = S.d_scratch + 2 + S.world;  // the global AND
  int* h_flags = reinterpret_cast<int*>(S.h_pinned);
  int done = 0, conv = 0;
  // One rank: the whole loop is ONE graph launch — a conditional WHILE node
  // whose body runs two iterations (a -> b, b -> a: fixed buffer roles) and
  // whose condition the last bookkeeping kernel sets from the device halt
  // flag, so the host synchronises once, at the end.
  if (S.world == 1 && S.graph != 2 && !S.timing && max_iters > 0) {
    // two iterations per HBM pass (the two-sweep kernel) unless tblock = 1
    const bool pairs = S.tblock != 1 && S.impl == 0;
    std::vector<int64_t> key = {-1, (int64_t)op, (int64_t)(uintptr_t)u->base, (int64_t)(uintptr_t)v->base,
                                u->nx, u->ny, u->nz, u->h, u->dtype, max_iters, S.impl, S.variant,
                                S.zchunks, S.sched, S.stages, S.l2promo, pairs ? 1 : 0};
    int64_t eb;
    std::memcpy(&eb, &eps, sizeof eb);
    key.push_back(eb);
    GraphEntry* hit = nullptr;
    for (auto& e : S.graphs)
      if (e.key == key) hit = &e;
    if (!hit) {
      cudaGraph_t g = nullptr;
      CK(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle cond;
      cudaGraphNodeParams cp = {};
      cudaGraphNode_t node;
      cudaError_t e = cudaGraphConditionalHandleCreate(&cond, g, 1u, cudaGraphCondAssignDefault);
      if (e == cudaSuccess) {
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = cond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
      }
      if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(S.stream, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed);
      if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        return fail(GSCL_E_CUDA, "conditional graph setup failed: %s", cudaGetErrorString(e));
      }
      const int64_t l0 = S.launches;
      gscl_status st = GSCL_OK;
      View x = a, y = b;
      for (int half = 0; half < 2 && st == GSCL_OK; ++half) {
        SweepPlan p;
        p.op = op;
        p.n_in = 1;
        p.in[0] = x;
        p.out = y;
        p.box = full;
        p.write = true;
        p.eps = eps;
        p.stop = S.d_conv + 2;
        p.red = red_target(d_loc, GSCL_AND);
        if (pairs) {
          // iterations k+1, k+2 in one two-sweep pass, both tests reduced; if
          // k+1 is the last (converged, or the budget), a single sweep redoes it
          p.tsteps = 2;
          p.rv = RV_CONV2;
          p.red2 = red_target(d_loc + 1, GSCL_AND);
          p.red2.partials = S.d_partials + S.max_partials / 2;
          p.red2.counter = S.d_counter + 1;
          st = run_sweep(p);
          if (st == GSCL_OK) {
            cudaError_t el = launch_conv_pair(d_loc, d_loc + 1, S.d_conv, max_iters, half,
                                              (unsigned long long)cond, half, S.stream, &S.launches);
            if (el != cudaSuccess) st = fail(GSCL_E_CUDA, "conv pair: %s", cudaGetErrorString(el));
          }
          if (st == GSCL_OK) {
            SweepPlan q;
            q.op = op;
            q.n_in = 1;
            q.in[0] = x;
            q.out = y;
            q.box = full;
            q.write = true;
            q.rv = RV_NONE;
            q.stop = S.d_conv + 3;  // runs only when flagged
            st = run_sweep(q);
          }
        } else {
          p.rv = RV_CONV;
          st = run_sweep(p);
          if (st == GSCL_OK) {
            cudaError_t el = launch_conv_step(d_loc, S.d_conv, max_iters, (unsigned long long)cond, half,
                                              S.stream, &S.launches);
            if (el != cudaSuccess) st = fail(GSCL_E_CUDA, "conv step: %s", cudaGetErrorString(el));
          }
        }
        std::swap(x, y);
      }
      cudaGraph_t body = nullptr;
      cudaError_t ec = cudaStreamEndCapture(S.stream, &body);
      if (st != GSCL_OK || ec != cudaSuccess) {
        cudaGraphDestroy(g);
        return st != GSCL_OK ? st : fail(GSCL_E_CUDA, "capture failed: %s", cudaGetErrorString(ec));
      }
      GraphEntry ge;
      ge.key = key;
      ge.kernels = S.launches - l0;
      ge.final_in_v = false;
      cudaError_t ei = cudaGraphInstantiate(&ge.exec, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) return fail(GSCL_E_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ei));
      if (S.graphs.size() >= 16) {
        cudaGraphExecDestroy(S.graphs.front().exec);
        S.graphs.erase(S.graphs.begin());
      }
      S.graphs.push_back(ge);
      hit = &S.graphs.back();
    }
    CK(cudaGraphLaunch(hit->exec, S.stream));
    CK(cudaMemcpyAsync(h_flags, S.d_conv, 5 * sizeof(int), cudaMemcpyDeviceToHost, S.stream));
    CK(cudaStreamSynchronize(S.stream));
    conv = h_flags[0];
    done = h_flags[1];
    // single iterations: iteration k wrote v when k is odd; pairs: the half of
    // the body that halted (half 0 writes v, half 1 writes u)
    const bool in_v = pairs ? (h_flags[4] == 0) : (done % 2 == 1);
    if (in_v) swap_storage(u, v);
    *iters_done = done;
    *converged = conv;
    return GSCL_OK;
  }
  for (int it = 1; it <= max_iters; ++it) {
    // one iteration of the paper's loop: b = OP(a) fused with the AND-reduced
    // convergence test |b - a| <= eps; skipped on device once converged
    if (gscl_status s = exchange(ga); s != GSCL_OK) return s;
    SweepPlan p;
    p.op = op;
    p.n_in = 1;
    p.in[0] = a;
    p.out = b;
    p.box = full;
    p.write = true;
    p.rv = RV_CONV;
    p.eps = eps;
    p.stop = S.d_conv;  // (the converged flag: this loop halts on the host)
    p.red = red_target(d_loc, GSCL_AND);
    if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
    if (gscl_status s = cross_rank(d_loc, GSCL_AND, d_res, S.stream); s != GSCL_OK) return s;
    CK(launch_conv_update(d_res, S.d_conv, S.d_conv + 1, it, S.stream, &S.launches));
    std::swap(a, b);
    std::swap(ga, gb);
    if (it % batch == 0 || it == max_iters) {
      CK(cudaMemcpyAsync(h_flags, S.d_conv, 2 * sizeof(int), cudaMemcpyDeviceToHost, S.stream));
      CK(cudaStreamSynchronize(S.stream));
      conv = h_flags[0];
      done = h_flags[1];
      if (conv) break;
    }
  }
  // iteration k wrote v when k is odd, u when k is even
  if (done % 2 == 1) swap_storage(u, v);
  *iters_done = done;
  *converged = conv;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_rbgs_run(gscl_grid_t u, int iters, int check_every, double* history) {
  GSCL_TRY
  Nvtx nv_call("gscl.rbgs_run");
  NEED_INIT();
  if (gscl_status s = check_grid(u, "u"); s != GSCL_OK) return s;
  if (iters < 0 || check_every < 0) return fail(GSCL_E_INVALID_ARG, "negative iters/check_every");
  if (check_every > 0 && !history) return fail(GSCL_E_INVALID_ARG, "history is NULL but check_every > 0");
  if (u->h < 1) return fail(GSCL_E_HALO_VIOLATION, "u needs halo >= 1");
  const int nh = check_every > 0 ? iters / check_every + 1 : 0;
  if (gscl_status s = ensure_hist((size_t)std::max(nh, 1)); s != GSCL_OK) return s;
  Box full;
  if (gscl_status s = local_box(u, nullptr, &full); s != GSCL_OK) return s;
  const View a = view_of(u);
  double* d_loc = S.d_scratch;
  auto resid = [&](double* slot) -> gscl_status {
    if (gscl_status s = exchange(u); s != GSCL_OK) return s;
    SweepPlan p;
    p.op = OP_JACOBI7;
    p.rv = RV_RESID;
    p.write = false;
    p.n_in = 1;
    p.in[0] = a;
    p.box = full;
    p.red = red_target(S.world == 1 ? slot : d_loc, GSCL_SUM);
    if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
    if (S.world > 1) return cross_rank(d_loc, GSCL_SUM, slot, S.stream);
    return GSCL_OK;
  };
  // One rank: an iteration is ONE two-sweep pass (red then black as
  // colour-masked Jacobi sweeps, sweep2r.cu), out of place between u and a
  // library buffer; a check fuses RESID7^2 of the pass's input.  An odd
  // iteration count leaves the result in the buffer: copied back to u.
  if (S.world == 1 && S.tblock != 1 && S.impl == 0 && !full.empty() && iters > 0) {
    if (S.rb_cap < u->bytes) {
      if (S.d_rb) {
        CK(cudaStreamSynchronize(S.stream));
        CK(cudaFree(S.d_rb));
      }
      S.d_rb = nullptr;
      CK(cudaMalloc(&S.d_rb, u->bytes));
      S.rb_cap = u->bytes;
    }
    View b = a;
    b.base = S.d_rb;
    b.origin = static_cast<char*>(S.d_rb) + (static_cast<char*>(a.origin) - static_cast<char*>(a.base));
    CK(launch_copy_halo(a, b, S.stream, &S.launches));  // the Dirichlet shell of both buffers
    View x = a, y = b;
    for (int it = 1; it <= iters; ++it) {
      const bool check = check_every > 0 && it % check_every == 0;
      SweepPlan p;
      p.op = OP_JACOBI7;
      p.n_in = 1;
      p.in[0] = x;
      p.out = y;
      p.box = full;
      p.write = true;
      p.tsteps = 2;
      p.rbgs = true;
      p.zoff = u->z_begin;
      p.rv = check ? RV_RESID_IN : RV_NONE;
      if (check) p.red = red_target(S.d_hist + (it / check_every - 1), GSCL_SUM);
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      std::swap(x, y);
    }
    if (x.base != a.base) CK(cudaMemcpyAsync(a.base, x.base, u->bytes, cudaMemcpyDeviceToDevice, S.stream));
  } else {
  for (int it = 1; it <= iters; ++it) {
    if (check_every > 0 && it % check_every == 0)
      if (gscl_status s = resid(S.d_hist + (it / check_every - 1)); s != GSCL_OK) return s;
    for (int color = 0; color < 2; ++color) {
      // in place: a half-sweep writes only its colour, whose points read only
      // points of the other colour (unchanged during the half-sweep)
      if (gscl_status s = exchange(u); s != GSCL_OK) return s;
      SweepPlan p;
      p.op = OP_JACOBI7;
      p.rv = RV_NONE;
      p.write = true;
      p.n_in = 1;
      p.in[0] = a;
      p.out = a;
      p.box = full;
      p.color = color;
      p.zoff = u->z_begin;
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
    }
  }
  }
  if (check_every > 0) {
    if (gscl_status s = resid(S.d_hist + (nh - 1)); s != GSCL_OK) return s;
    CK(cudaMemcpyAsync(history, S.d_hist, (size_t)nh * sizeof(double), cudaMemcpyDeviceToHost, S.stream));
  }
  CK(cudaStreamSynchronize(S.stream));
  for (int i = 0; i < nh; ++i) history[i] = std::sqrt(history[i]);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_do_ordered(gscl_space space, gscl_oop op, gscl_grid_t in, gscl_grid_t out) {
  GSCL_TRY
  Nvtx nv_call("gscl.do_ordered");
  NEED_INIT();
  if (space < GSCL_DO_I_INC || space > GSCL_DO_DIAMOND) return fail(GSCL_E_INVALID_ARG, "unknown space %d", (int)space);
  if (op < GSCL_O_PREFIX || op > GSCL_O_PASCAL) return fail(GSCL_E_INVALID_ARG, "unknown op %d", (int)op);
  if ((op == GSCL_O_PASCAL) != (space == GSCL_DO_DIAMOND))
    return fail(GSCL_E_UNSUPPORTED, "PASCAL goes with DIAMOND, PREFIX with the axis spaces");
  if (gscl_status s = check_grid(out, "out"); s != GSCL_OK) return s;
  if (out->h < 1) return fail(GSCL_E_HALO_VIOLATION, "out needs halo >= 1 (it holds the values before the first cell)");
  if (op == GSCL_O_PREFIX) {
    if (gscl_status s = check_grid(in, "in"); s != GSCL_OK) return s;
    if (gscl_status s = same_shape(in, out); s != GSCL_OK) return s;
    if (in == out || in->base == out->base) return fail(GSCL_E_INVALID_ARG, "out aliases in");
  } else if (in) {
    return fail(GSCL_E_ARITY, "PASCAL reads no input grid (pass NULL)");
  }
  View vo = view_of(out), vi;
  if (in) vi = view_of(in);
  // the k spaces cross ranks: ranks run in order, each receiving the plane
  // before its first one from the previous rank (sequential by definition)
  const bool kspace = space == GSCL_DO_K_INC || space == GSCL_DO_K_DEC;
  const bool inc = space == GSCL_DO_K_INC;
  const int prev = inc ? S.rank - 1 : S.rank + 1;
  const int next = inc ? S.rank + 1 : S.rank - 1;
  const int64_t pb = out->plane * (int64_t)out->es;
  char* base = static_cast<char*>(out->base);
  if (kspace && S.world > 1 && prev >= 0 && prev < S.world) {
    // ghost plane before my first: plane -1 (inc) or plane nzl (dec)
    char* ghost = base + (inc ? (out->h - 1) : (out->nzl + out->h)) * pb;
    NK(ncclRecv(ghost, (size_t)pb, ncclUint8, prev, S.comm, S.stream));
  }
  CK(launch_ordered((int)space, (int)op, in ? &vi : nullptr, vo, S.stream, &S.launches));
  if (kspace && S.world > 1 && next >= 0 && next < S.world) {
    char* last = base + (inc ? (out->nzl - 1 + out->h) : out->h) * pb;
    NK(ncclSend(last, (size_t)pb, ncclUint8, next, S.comm, S.stream));
  }
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_timing_enable(int on) {
  GSCL_TRY
  NEED_INIT();
  S.timing = on != 0;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_timing_read(double* ms, int64_t* n, int64_t* launches) {
  GSCL_TRY
  NEED_INIT();
  CK(cudaStreamSynchronize(S.stream));
  for (auto& tp : S.pending) {
    float t = 0;
    CK(cudaEventElapsedTime(&t, tp.a, tp.b));
    S.kind_ms[tp.kind] += t;
    S.kind_n[tp.kind] += 1;
    S.pool.push_back(tp);
  }
  S.pending.clear();
  for (int k = 0; k < 4; ++k) {
    if (ms) ms[k] = S.kind_ms[k];
    if (n) n[k] = S.kind_n[k];
    S.kind_ms[k] = 0;
    S.kind_n[k] = 0;
  }
  if (launches) *launches = S.launches;
  S.launches = 0;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_peer_export(gscl_grid_t u, gscl_grid_t v, void* blob, size_t cap, size_t* bytes) {
  GSCL_TRY
  NEED_INIT();
  if (!bytes) return fail(GSCL_E_INVALID_ARG, "bytes is NULL");
  *bytes = sizeof(PeerBlob);
  if (!blob) return GSCL_OK;  // size query
  if (cap < sizeof(PeerBlob)) return fail(GSCL_E_INVALID_ARG, "blob buffer too small (%zu < %zu)", cap, sizeof(PeerBlob));
  if (S.world > 8) return fail(GSCL_E_UNSUPPORTED, "the peer transport supports up to 8 ranks");
  if (gscl_status s = check_grid(u, "u"); s != GSCL_OK) return s;
  if (gscl_status s = check_grid(v, "v"); s != GSCL_OK) return s;
  if (gscl_status s = same_shape(u, v); s != GSCL_OK) return s;
  if (u->base == v->base) return fail(GSCL_E_INVALID_ARG, "u and v alias");
  peer_reset();
  g_opened.clear();
  PeerSet& P = S.peer;
  P.plane_bytes = (size_t)(u->plane * (int64_t)u->es);
  const size_t ab = PeerSet::arena_bytes(P.plane_bytes, S.world);
  CK(cudaMalloc(&P.arena, ab));
  CK(cudaMemset(P.arena, 0, ab));
  P.store_base[0] = u->base;
  P.store_base[1] = v->base;
  PeerBlob b{};
  b.magic = 0x4c435347;  // "GSCL"
  b.rank = S.rank;
  b.world = S.world;
  b.dtype = u->dtype;
  b.nx = u->nx; b.ny = u->ny; b.nzl = u->nzl; b.h = u->h;
  b.pitch = u->pitch; b.plane = u->plane; b.z_begin = u->z_begin;
  void* ptrs[3] = {u->base, v->base, P.arena};
  for (int k = 0; k < 3; ++k) {
    void* base = nullptr;
    CK(alloc_base(ptrs[k], &base, nullptr));
    CK(cudaIpcGetMemHandle(&b.handle[k], base));
    b.offset[k] = static_cast<char*>(ptrs[k]) - static_cast<char*>(base);
  }
  std::memcpy(blob, &b, sizeof b);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_peer_import(gscl_grid_t u, gscl_grid_t v, const void* blobs, size_t bytes_each) {
  GSCL_TRY
  NEED_INIT();
  PeerSet& P = S.peer;
  if (!P.arena) return fail(GSCL_E_STATE, "gscl_peer_export must precede gscl_peer_import");
  if (!blobs || bytes_each != sizeof(PeerBlob)) return fail(GSCL_E_INVALID_ARG, "bad blob array");
  if (gscl_status s = check_grid(u, "u"); s != GSCL_OK) return s;
  if (gscl_status s = check_grid(v, "v"); s != GSCL_OK) return s;
  if (!((u->base == P.store_base[0] && v->base == P.store_base[1]) ||
        (u->base == P.store_base[1] && v->base == P.store_base[0])))
    return fail(GSCL_E_INVALID_ARG, "u / v are not the grids passed to gscl_peer_export");
  for (int r = 0; r < S.world; ++r) {
    PeerBlob b;
    std::memcpy(&b, static_cast<const char*>(blobs) + (size_t)r * bytes_each, sizeof b);
    if (b.magic != 0x4c435347 || b.rank != r || b.world != S.world)
      return fail(GSCL_E_INVALID_ARG, "blob %d is not rank %d's export of this job", r, r);
    if (b.nx != u->nx || b.ny != u->ny || b.h != u->h || b.pitch != u->pitch || b.plane != u->plane ||
        b.dtype != u->dtype)
      return fail(GSCL_E_SHAPE_MISMATCH, "rank %d exported a different grid layout", r);
    if (r == S.rank) {
      P.arena_of[r] = static_cast<char*>(P.arena);
      continue;
    }
    void* q = nullptr;
    if (gscl_status s = open_handle(b.handle[2], &q); s != GSCL_OK) return s;
    P.arena_of[r] = static_cast<char*>(q) + b.offset[2];
    const int side = r == S.rank - 1 ? 0 : r == S.rank + 1 ? 1 : -1;
    if (side >= 0) {
      for (int k = 0; k < 2; ++k) {
        if (gscl_status s = open_handle(b.handle[k], &q); s != GSCL_OK) return s;
        P.nb_store[side][k] = static_cast<char*>(q) + b.offset[k];
      }
      P.nzl_nb[side] = b.nzl;
    }
  }
  P.units = pass_tiles(u->nx, u->ny, u->dtype, S.variant);
  P.ready = true;
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_set_option(const char* name, int64_t value) {
  GSCL_TRY
  NEED_INIT();
  if (!name) return fail(GSCL_E_INVALID_ARG, "name is NULL");
  std::string n(name);
  if (n == "sweep_impl") {
    if (value < 0 || value > 2) return fail(GSCL_E_INVALID_ARG, "sweep_impl must be 0, 1 or 2");
    S.impl = (int)value;
  } else if (n == "zchunks") {
    if (value < 0) return fail(GSCL_E_INVALID_ARG, "zchunks must be >= 0");
    S.zchunks = (int)value;
  } else if (n == "zalt") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "zalt must be 0 or 1");
    S.zalt = (int)value;
  } else if (n == "graph") {
    if (value < 0 || value > 2) return fail(GSCL_E_INVALID_ARG, "graph must be 0, 1 or 2");
    S.graph = (int)value;
  } else if (n == "variant") {
    // 1, 2: sweep_tma ablations; 1..4: sweep2.cu geometries; 11, 12, 14: sweep2r.cu
    if (value < 0 || (value > 4 && value != 11 && value != 12 && value != 14))
      return fail(GSCL_E_INVALID_ARG, "variant must be 0..4, 11, 12 or 14");
    S.variant = (int)value;
  } else if (n == "transport") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "transport must be 0 (NCCL) or 1 (peer memory)");
    S.transport = (int)value;
  } else if (n == "tblock") {
    if (value != 0 && value != 1 && value != 2) return fail(GSCL_E_INVALID_ARG, "tblock must be 0, 1 or 2");
    S.tblock = (int)value;
  } else if (n == "split") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "split must be 0 or 1");
    S.split = (int)value;
  } else if (n == "sched") {
    if (value < 0 || value > 2) return fail(GSCL_E_INVALID_ARG, "sched must be 0, 1 or 2");
    S.sched = (int)value;
  } else if (n == "stages") {
    if (value != 0 && value != 4 && value != 8) return fail(GSCL_E_INVALID_ARG, "stages must be 0, 4 or 8");
    S.stages = (int)value;
  } else if (n == "l2promo") {
    if (value < 0 || value > 3) return fail(GSCL_E_INVALID_ARG, "l2promo must be 0..3");
    S.l2promo = (int)value;
  } else {
    return fail(GSCL_E_UNSUPPORTED, "unknown option '%s'", name);
  }
  return GSCL_OK;
  GSCL_CATCH
}

}  // extern "C"
