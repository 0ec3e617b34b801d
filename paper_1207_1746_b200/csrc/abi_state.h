// abi_state.h — the library's process-wide state and the host-side helpers
// shared by the ABI translation units (abi.cu: context, grids, do_all /
// do_reduce / halo exchange; jacobi.cu: the Jacobi, convergence and red-black
// drivers; peer.cu: the peer-memory transport).  Internal: not part of the C
// ABI (include/gscl.h).  C++17 inline variables / functions, so every unit
// shares one definition.
#pragma once
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <thread>
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
  cudaEvent_t read_done = nullptr;  // an asynchronous download has finished reading this storage
  bool dl_pending = false;          // the library stream must wait on `read_done` before use
};


namespace gscl_abi {


// NVTX ranges on the host timeline (Nsight Systems): one per ABI call and per
// enqueued sweep / pass / exchange / combine (SURVEY §5 tracing).
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

inline thread_local std::string t_err;

inline gscl_status fail(gscl_status s, const char* fmt, ...) {
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
  int count = 1;  // launches the pair brackets (a run of consecutive passes: several)
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
constexpr int kSlotFlag0 = 64;    // counter index of reduction slot 0
constexpr int kFlagsBytes = 4 * (kSlotFlag0 + kRedSlots);
// counters: [0] from below, [1] from above, [2] barrier from below, [3] barrier
// from above, [kSlotFlag0 + q] arrivals into reduction slot q (one counter per
// slot: a rank's wait for check m is satisfied only by check m's publishes,
// never by a later check of a rank that ran ahead)
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
  unsigned tgt[4] = {0, 0, 0, 0};            // host mirrors of what my counters will reach
  unsigned tgt_slot[kRedSlots] = {};         // ... and the reduction slots' counters
  unsigned red_next = 0;                     // reduction slot ring position
  int64_t units = 0;                         // boundary units per side per step
  size_t cplane_bytes = 0;                   // a plane of a halo-0 grid of u's extents (coefficients)
  // arena layout: ghost planes for input storage 0 (2 planes: below, above),
  // for input storage 1, then the counters, then the reduction slots (room
  // for 8 ranks), then 14 coefficient planes (VARCOEF8 passes: plane 2c =
  // coefficient grid c's plane below the slab, 2c + 1 = above)
  static size_t cghost_offset(size_t pb) {
    return (4 * pb + kFlagsBytes + (size_t)kRedSlots * 8 * sizeof(double) + 255) / 256 * 256;
  }
  static size_t arena_bytes(size_t pb, size_t cpb) { return cghost_offset(pb) + 14 * cpb; }
  static unsigned* flags_of(char* ar, size_t pb) { return reinterpret_cast<unsigned*>(ar + 4 * pb); }
  static double* red_of(char* ar, size_t pb) { return reinterpret_cast<double*>(ar + 4 * pb + kFlagsBytes); }
  static char* ghost_of(char* ar, size_t pb, int storage) { return ar + (size_t)storage * 2 * pb; }
  static char* cghost_of(char* ar, size_t pb) { return ar + cghost_offset(pb); }
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
  void* d_cghost = nullptr;     // VARCOEF8 passes on slabs: 7 x 2 coefficient planes outside the slab
  size_t cghost_cap = 0;
  void* d_rb = nullptr;         // red-black GS: the second buffer of the out-of-place passes
  size_t rb_cap = 0;
  unsigned long long* d_digest = nullptr;
  int* d_conv = nullptr;  // [0] converged, [1] iterations, [2] halt, [3] skip redo, [4] final half
  unsigned* d_bflag = nullptr;  // boundary-plane counter of the overlapped schedule
  cudaStream_t copy_stream = nullptr;  // asynchronous uploads (gscl_grid_copy_from_host_async)
  cudaStream_t down_stream = nullptr;  // asynchronous downloads (gscl_grid_copy_to_host_async)
  cudaEvent_t ev_to_down = nullptr;
  void* down_stage[2] = {nullptr, nullptr};
  size_t down_cap[2] = {0, 0};
  unsigned down_next = 0;
  cudaEvent_t ev_to_copy = nullptr;
  void* up_stage[2] = {nullptr, nullptr};
  size_t up_cap[2] = {0, 0};
  unsigned up_next = 0;
  unsigned bflag_target = 0;    // host mirror of what the counter will reach
  double* h_pinned = nullptr;  // 64 doubles
  double* h_hist = nullptr;    // [0, hist_cap): pinned landing zone of the history (a D2H copy
                               // into pageable memory would block the host before the watchdog)
  void* d_stage = nullptr;     // host-copy staging buffer (dense planes)
  size_t stage_cap = 0;
  cudaStream_t comm_stream = nullptr;  // halo exchange / cross-rank combine in jacobi_run
  cudaStream_t cap_stream = nullptr;   // graph captures when S.stream is the legacy default stream
  cudaEvent_t ev_to_comm = nullptr, ev_to_main = nullptr, ev_halo = nullptr;
  cudaEvent_t ev_bnd = nullptr;  // jacobi_run pairs: the boundary-chunk launch of the last pass ended
  int split = 0;  // force the overlapped (boundary-first) jacobi schedule at world 1
  int split_one = 0;  // ablation: the boundary-first JACOBI7 pass as ONE multi-rank launch
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
  int halo_off = 0;              // timing only: skip the halo exchanges (option "halo_off")
  int64_t timeout_ms = 120000;  // multi-rank watchdog (option "timeout_ms")
  bool poisoned = false;        // a multi-rank wait timed out: only gscl_finalize is accepted
  std::vector<TimedPair> pool, pending;
  double kind_ms[4] = {0, 0, 0, 0};
  int64_t kind_n[4] = {0, 0, 0, 0};
  int64_t launches = 0;
  std::set<gscl_grid_s*> live;
};
inline State S;

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
#define NEED_INIT()                                                                              \
  if (!S.inited) return fail(GSCL_E_STATE, "gscl_init has not been called (or gscl_finalize was)"); \
  if (S.poisoned)                                                                                  \
  return fail(GSCL_E_STATE, "a multi-rank call timed out waiting for its peers; call gscl_finalize")

// ---- the multi-rank watchdog.  On one rank a stream synchronisation cannot
// wait on anything but this GPU, so it is a plain cudaStreamSynchronize.  On
// several ranks the library stream may be parked on a peer: a
// cuStreamWaitValue32 on a counter a neighbour bumps (peer transport), or an
// NCCL kernel waiting for its partner.  A rank that died or never calls would
// hang the job, so the wait polls with a deadline (option "timeout_ms"); on
// expiry it (1) releases every pending counter wait of this rank by raising
// its counters past their targets (the waits compare cyclically, (int)(*addr -
// value) >= 0), written from the host on a stream the parked one does not
// block, (2) aborts the NCCL communicator, which ends its kernels, (3) lets
// the stream drain for a bounded time and (4) poisons the context: the
// results are garbage, so every later call but gscl_finalize is refused.
inline void release_peer_waits() {
  PeerSet& P = S.peer;
  if (!P.ready || !P.arena) return;
  unsigned v[kSlotFlag0 + kRedSlots] = {};
  for (int i = 0; i < 4; ++i) v[i] = P.tgt[i] + (1u << 30);
  for (int q = 0; q < kRedSlots; ++q) v[kSlotFlag0 + q] = P.tgt_slot[q] + (1u << 30);
  unsigned* flags = PeerSet::flags_of(static_cast<char*>(P.arena), P.plane_bytes);
  cudaMemcpyAsync(flags, v, sizeof v, cudaMemcpyHostToDevice, S.cap_stream);
  cudaStreamSynchronize(S.cap_stream);
}

inline gscl_status sync_stream(cudaStream_t st) {
  if (S.world == 1) {
    CK(cudaStreamSynchronize(st));
    return GSCL_OK;
  }
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  auto ms_since = [](clk::time_point t) {
    return (int64_t)std::chrono::duration_cast<std::chrono::milliseconds>(clk::now() - t).count();
  };
  for (int spin = 0;; ++spin) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return GSCL_OK;
    if (e != cudaErrorNotReady) return fail(GSCL_E_CUDA, "stream: %s", cudaGetErrorString(e));
    if (S.comm && (spin & 63) == 0) {
      ncclResult_t ar = ncclSuccess;
      if (ncclCommGetAsyncError(S.comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
        S.poisoned = true;
        ncclCommAbort(S.comm);
        S.comm = nullptr;
        return fail(GSCL_E_NCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ar));
      }
    }
    if (ms_since(t0) > S.timeout_ms) break;
    if (spin < 2000) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  S.poisoned = true;
  release_peer_waits();
  if (S.comm) {
    ncclCommAbort(S.comm);
    S.comm = nullptr;
  }
  const auto t1 = clk::now();
  while (cudaStreamQuery(st) == cudaErrorNotReady && ms_since(t1) < 10000)
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  return fail(GSCL_E_TIMEOUT, "rank %d: no progress from the peer ranks within %lld ms (peer waits released, "
              "NCCL aborted; the context is poisoned - call gscl_finalize)", S.rank, (long long)S.timeout_ms);
}
inline gscl_status sync_main() { return sync_stream(S.stream); }

inline int64_t ox_of(int dtype) { return dtype == 0 ? 16 : 32; }
inline int max_halo(int dtype) { return (int)ox_of(dtype); }

inline void slab(int64_t nz, int rank, int world, int64_t* z0, int64_t* z1) {
  int64_t base = nz / world, rem = nz % world;
  int64_t r = rank;
  *z0 = r * base + std::min<int64_t>(r, rem);
  *z1 = *z0 + base + (r < rem ? 1 : 0);
}

inline gscl_status layout(gscl_grid_s* g, int64_t nx, int64_t ny, int64_t nz, int halo, int dtype,
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

inline View view_of(const gscl_grid_s* g) {
  View v;
  v.base = g->base;
  v.origin = static_cast<char*>(g->base) + (size_t)(g->h * g->plane + g->h * g->pitch + g->ox) * g->es;
  v.nx = g->nx; v.ny = g->ny; v.nzl = g->nzl; v.h = g->h;
  v.pitch = g->pitch; v.plane = g->plane; v.ox = g->ox; v.dtype = g->dtype;
  return v;
}

inline bool live(gscl_grid_t g) { return g && S.live.count(g); }

inline gscl_status check_grid(gscl_grid_t g, const char* what) {
  if (!g) return fail(GSCL_E_INVALID_ARG, "%s is NULL", what);
  if (!live(g)) return fail(GSCL_E_INVALID_ARG, "%s is not a live grid handle", what);
  if (g->pending) {  // an asynchronous upload into it: order it before any use
    CK(cudaStreamWaitEvent(S.stream, g->ready, 0));
    g->pending = false;
  }
  if (g->dl_pending) {  // an asynchronous download still reads it: no overwrite before
    CK(cudaStreamWaitEvent(S.stream, g->read_done, 0));
    g->dl_pending = false;
  }
  return GSCL_OK;
}

inline gscl_status same_shape(gscl_grid_t a, gscl_grid_t b) {
  if (a->nx != b->nx || a->ny != b->ny || a->nz != b->nz)
    return fail(GSCL_E_SHAPE_MISMATCH, "grid extents differ (%lldx%lldx%lld vs %lldx%lldx%lld)",
                (long long)a->nx, (long long)a->ny, (long long)a->nz, (long long)b->nx,
                (long long)b->ny, (long long)b->nz);
  if (a->dtype != b->dtype) return fail(GSCL_E_DTYPE, "grid element types differ");
  return GSCL_OK;
}

// Global range -> local box (clipped to this rank's slab).
inline gscl_status local_box(const gscl_grid_s* g, const gscl_range* r, Box* b) {
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

inline int op_arity(int op) { return op == GSCL_OP_VARCOEF8 ? 8 : 1; }

inline gscl_status record_start(TimedPair* tp) {
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
inline gscl_status record_end(TimedPair tp, int kind, int count = 1) {
  if (!S.timing) return GSCL_OK;
  CK(cudaEventRecord(tp.b, S.stream));
  tp.kind = kind;
  tp.count = count;
  S.pending.push_back(tp);
  return GSCL_OK;
}

inline RedTarget red_target(double* result, int comb) {
  RedTarget t;
  t.partials = S.d_partials;
  t.counter = S.d_counter;
  t.result = result;
  t.comb = comb;
  t.max_partials = S.max_partials;
  return t;
}

// Launch one sweep (timed when instrumentation is on).
inline gscl_status run_sweep(SweepPlan& p) {
  Nvtx nv(p.tsteps == 2 ? "gscl.pass" : p.write ? "gscl.sweep" : "gscl.reduce_sweep");
  p.stream = S.stream;
  p.impl = S.impl;
  p.zchunks = S.zchunks;
  p.sched = S.sched;
  p.l2promo = S.l2promo;
  p.stages = S.stages;
  p.variant = S.variant;
  p.num_sms = S.num_sms;
  p.ticket = S.d_counter + 8;
  if (p.rv != RV_NONE && p.box.empty()) {
    CK(launch_fold(nullptr, 0, p.red.comb, p.red.result, S.stream, &S.launches));
    return GSCL_OK;
  }
  TimedPair tp{};
  if (!p.untimed)
    if (gscl_status st = record_start(&tp); st != GSCL_OK) return st;
  cudaError_t e = p.tsteps == 2 ? launch_sweep2(p, &S.launches) : launch_sweep(p, &S.launches);
  if (e != cudaSuccess) return fail(GSCL_E_CUDA, "sweep launch failed: %s", cudaGetErrorString(e));
  const int kind = p.tsteps == 2 ? 3 : p.rv == RV_NONE ? 0 : (p.write ? 1 : 2);
  return p.untimed ? GSCL_OK : record_end(tp, kind);
}

// Peer-memory combine: this rank's value goes into slot q of every rank's
// arena (peer stores on stream `pub`, then each rank's slot-q counter is
// bumped); stream `fold` waits until slot q's counter has grown by `world`
// (all ranks' values of THIS use of slot q have landed) and folds the slot in
// rank order (R14).  The slot ring has kRedSlots entries and ranks drift apart
// by at most world - 1 passes (each pass waits on its neighbours), so a slot is
// never republished before every rank has folded it.
inline gscl_status peer_combine(double* d_loc, int comb, double* d_out, cudaStream_t pub, cudaStream_t fold,
                                cudaEvent_t ev) {
  PeerSet& P = S.peer;
  const size_t pb = P.plane_bytes;
  const unsigned q = P.red_next++ % kRedSlots;
  PeerPtrs8 dst{}, cnt{};
  for (int r = 0; r < S.world; ++r) {
    dst.p[dst.n++] = PeerSet::red_of(P.arena_of[r], pb) + (size_t)q * S.world + S.rank;
    cnt.p[cnt.n++] = PeerSet::flags_of(P.arena_of[r], pb) + kSlotFlag0 + q;
  }
  CK(launch_publish(d_loc, dst, cnt, pub, &S.launches));
  P.tgt_slot[q] += (unsigned)S.world;
  if (fold != pub) {
    CK(cudaEventRecord(ev, pub));
    CK(cudaStreamWaitEvent(fold, ev, 0));
  }
  CK(stream_wait_geq(fold, PeerSet::flags_of(P.arena_of[S.rank], pb) + kSlotFlag0 + q, P.tgt_slot[q]));
  CK(launch_fold(PeerSet::red_of(P.arena_of[S.rank], pb) + (size_t)q * S.world, S.world, comb, d_out, fold,
                 &S.launches));
  return GSCL_OK;
}

// Combine this rank's device scalar d_loc across ranks into d_out (same bits
// on every rank): all-gather, then fold in rank order (R14).
inline gscl_status cross_rank(double* d_loc, int comb, double* d_out, cudaStream_t st) {
  Nvtx nv("gscl.combine");
  if (S.world == 1) {
    if (d_loc != d_out) CK(cudaMemcpyAsync(d_out, d_loc, 8, cudaMemcpyDeviceToDevice, st));
    return GSCL_OK;
  }
  if (!S.comm) {
    // no communicator: the peer-memory arena (after gscl_peer_export/import)
    if (!S.peer.ready) return fail(GSCL_E_STATE, "no NCCL communicator and no peer set (gscl_peer_export/import)");
    return peer_combine(d_loc, comb, d_out, st, st, nullptr);
  }
  NK(ncclAllGather(d_loc, S.d_scratch + 1, 1, ncclDouble, S.comm, st));
  CK(launch_fold(S.d_scratch + 1, S.world, comb, d_out, st, &S.launches));
  return GSCL_OK;
}

// A CUDA graph cannot be captured on the legacy default stream (what a NULL
// cuda_stream at gscl_init selects), so while a capture is open the library
// enqueues on a private stream instead; the graph it yields is launched on
// S.stream after the scope closes, in order with the caller's work.
struct CaptureScope {
  cudaStream_t saved;
  CaptureScope() : saved(S.stream) {
    if (S.stream == cudaStreamLegacy) S.stream = S.cap_stream;
  }
  ~CaptureScope() { S.stream = saved; }
  CaptureScope(const CaptureScope&) = delete;
  CaptureScope& operator=(const CaptureScope&) = delete;
};

// Make stream `to` wait for everything issued so far on stream `from`.
inline gscl_status hand_off(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
  CK(cudaEventRecord(ev, from));
  CK(cudaStreamWaitEvent(to, ev, 0));
  return GSCL_OK;
}

// The halo-exchange plan of one rank (byte offsets into its slab allocation).
// Local plane k (k = -h .. nzl+h-1) starts at byte (k + h) * plane * es.
inline int halo_plan(const gscl_grid_s* g, int rank, int world, gscl_halo_op* ops) {
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

inline gscl_status exchange(gscl_grid_s* g, cudaStream_t st) {
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
inline gscl_status exchange(gscl_grid_s* g) { return exchange(g, S.stream); }

inline gscl_status ensure_hist(size_t n) {
  if (n <= S.hist_cap) return GSCL_OK;
  if (S.d_hist) {
    if (gscl_status ss = sync_main(); ss != GSCL_OK) return ss;
    CK(cudaFree(S.d_hist));
  }
  S.d_hist = nullptr;
  CK(cudaMalloc(&S.d_hist, 2 * n * sizeof(double)));
  if (S.h_hist) cudaFreeHost(S.h_hist);
  S.h_hist = nullptr;
  CK(cudaMallocHost(&S.h_hist, n * sizeof(double)));
  S.d_lochist = S.d_hist + n;
  S.hist_cap = n;
  return GSCL_OK;
}

inline gscl_status ensure_ghost(size_t bytes) {
  if (bytes <= S.ghost_cap) return GSCL_OK;
  if (S.d_ghost) {
    if (gscl_status ss = sync_main(); ss != GSCL_OK) return ss;
    CK(cudaFree(S.d_ghost));
  }
  S.d_ghost = nullptr;
  CK(cudaMalloc(&S.d_ghost, bytes));
  S.ghost_cap = bytes;
  return GSCL_OK;
}

// The coefficient planes a VARCOEF8 two-sweep pass reads just outside the
// slab (u1 is computed on a rank boundary's halo plane, and it needs the
// coefficients there; the coefficient grids have no halo): grid c's plane 0
// goes to the lower neighbour's d_cghost plane 2c + 1 (its plane "above"),
// its plane nzl - 1 to the upper neighbour's plane 2c (its plane "below").
// Sends and receives per peer are issued in c order on both sides.
inline gscl_status exchange_coeff_ghosts(const gscl_grid_t* coeffs, int nc, cudaStream_t st) {
  Nvtx nv("gscl.coeff_ghosts");
  if (S.world == 1 || nc == 0) return GSCL_OK;
  if (!S.comm) return fail(GSCL_E_STATE, "no NCCL communicator (gscl_init had no nccl_id)");
  const gscl_grid_s* c0 = coeffs[0];
  const size_t pb = (size_t)(c0->plane * (int64_t)c0->es);
  const size_t need = (size_t)2 * nc * pb;
  if (need > S.cghost_cap) {
    if (S.d_cghost) {
      if (gscl_status ss = sync_main(); ss != GSCL_OK) return ss;
      CK(cudaFree(S.d_cghost));
    }
    S.d_cghost = nullptr;
    CK(cudaMalloc(&S.d_cghost, need));
    S.cghost_cap = need;
  }
  char* g = static_cast<char*>(S.d_cghost);
  NK(ncclGroupStart());
  for (int c = 0; c < nc; ++c) {
    const gscl_grid_s* cg = coeffs[c];
    char* base = static_cast<char*>(cg->base) + (size_t)cg->h * pb;  // plane 0
    if (S.rank > 0) {
      NK(ncclSend(base, pb, ncclUint8, S.rank - 1, S.comm, st));
      NK(ncclRecv(g + (size_t)(2 * c) * pb, pb, ncclUint8, S.rank - 1, S.comm, st));
    }
    if (S.rank < S.world - 1) {
      NK(ncclSend(base + (size_t)(cg->nzl - 1) * pb, pb, ncclUint8, S.rank + 1, S.comm, st));
      NK(ncclRecv(g + (size_t)(2 * c + 1) * pb, pb, ncclUint8, S.rank + 1, S.comm, st));
    }
  }
  NK(ncclGroupEnd());
  return GSCL_OK;
}

// The depth-2 halo exchange of a two-sweep pass: each side sends its first /
// last two interior planes, one plane per transfer, and receives the
// neighbour's into local planes -1, -2 (below) and nzl, nzl+1 (above).  A
// received plane inside the grid's halo (|offset| <= h) lands in the grid;
// one beyond it (h = 1) lands in the ghost buffer (plane 0 below, 1 above).
// Per neighbour the transfers are listed nearest plane first on both sides,
// so NCCL matches them in order.
inline int pass_plan(const gscl_grid_s* g, int rank, int world, gscl_pass_xfer* ops) {
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

inline gscl_status exchange_pass(gscl_grid_s* g, cudaStream_t st) {
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


inline void swap_storage(gscl_grid_s* a, gscl_grid_s* b) {
  std::swap(a->base, b->base);
  std::swap(a->bytes, b->bytes);
  std::swap(a->owned, b->owned);
  std::swap(a->ready, b->ready);
  std::swap(a->pending, b->pending);
  std::swap(a->read_done, b->read_done);
  std::swap(a->dl_pending, b->dl_pending);
}

// Release every IPC mapping and the arena of the peer transport.
inline void peer_reset() {
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
inline std::vector<OpenedHandle> g_opened;
inline gscl_status open_handle(const cudaIpcMemHandle_t& h, void** ptr) {
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


}  // namespace gscl_abi
