// abi.cu — the C ABI of include/gscl.h: context, grid storage and layout,
// z-slab decomposition, do_all / do_reduce, NCCL halo exchange and
// cross-rank combine, timing and options.  The Jacobi / convergence /
// red-black drivers are in jacobi.cu, the peer-memory transport in peer.cu;
// the shared state in abi_state.h.  No exception or abort crosses the ABI.
#include <cstdlib>

#include "abi_state.h"

using namespace gscl;
using namespace gscl_abi;


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
  {
    // the halo exchange / combine stream runs at the highest priority: its
    // NCCL kernels then take the first SM a pass CTA frees instead of queueing
    // behind the rest of the pass's grid, so the exchange overlaps the
    // interior units
    int lo_prio = 0, hi_prio = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    CK(cudaStreamCreateWithPriority(&S.comm_stream, cudaStreamNonBlocking, hi_prio));
  }
  CK(cudaStreamCreateWithFlags(&S.cap_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&S.ev_to_comm, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&S.ev_to_main, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&S.ev_halo, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&S.ev_bnd, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&S.copy_stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&S.down_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&S.ev_to_down, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&S.ev_to_copy, cudaEventDisableTiming));
  if (world > 1) {
    // every kernel loaded now: a lazy load later, behind a parked peer wait,
    // would block the host before the watchdog (internal.h, GSCL_MODULE_ANCHOR)
    int nfun = 0;
    CK(preload_modules(&nfun));
    if (std::getenv("GSCL_TRACE")) std::fprintf(stderr, "gscl[%d]: preloaded %d kernels\n", rank, nfun);
  }
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
  if (!S.inited) return fail(GSCL_E_STATE, "gscl_init has not been called (or gscl_finalize was)");
  if (S.poisoned) {
    // after a watchdog timeout the streams were released and drained (bounded);
    // if one is still parked, freeing memory under it would block: give up
    // the resources instead of hanging the caller's exit
    for (cudaStream_t st : {S.stream, S.comm_stream, S.copy_stream, S.down_stream})
      if (st && cudaStreamQuery(st) == cudaErrorNotReady) {
        S = State();
        return fail(GSCL_E_TIMEOUT, "finalize after a timeout: a stream is still blocked; resources leaked");
      }
  }
  cudaStreamSynchronize(S.stream);
  peer_reset();
  g_opened.clear();
  if (S.copy_stream) cudaStreamSynchronize(S.copy_stream);
  if (S.down_stream) cudaStreamSynchronize(S.down_stream);
  for (gscl_grid_s* g : S.live) {
    if (g->owned && g->base) cudaFree(g->base);
    if (g->ready) cudaEventDestroy(g->ready);
    if (g->read_done) cudaEventDestroy(g->read_done);
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
  if (S.h_hist) cudaFreeHost(S.h_hist);
  for (auto& e : S.graphs) cudaGraphExecDestroy(e.exec);
  S.graphs.clear();
  if (S.comm_stream) {
    cudaStreamSynchronize(S.comm_stream);
    cudaStreamDestroy(S.comm_stream);
  }
  for (cudaEvent_t e : {S.ev_to_comm, S.ev_to_main, S.ev_halo, S.ev_to_copy, S.ev_bnd})
    if (e) cudaEventDestroy(e);
  if (S.copy_stream) cudaStreamDestroy(S.copy_stream);
  if (S.down_stream) cudaStreamDestroy(S.down_stream);
  if (S.ev_to_down) cudaEventDestroy(S.ev_to_down);
  for (void* p : S.down_stage)
    if (p) cudaFree(p);
  for (void* p : S.up_stage)
    if (p) cudaFree(p);
  if (S.cap_stream) cudaStreamDestroy(S.cap_stream);
  if (S.d_cghost) cudaFree(S.d_cghost);
  if (S.own_stream) cudaStreamDestroy(S.stream);
  S = State();
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_sync(void) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
  CK(cudaStreamSynchronize(S.down_stream));  // asynchronous downloads have landed in host memory
  CK(cudaStreamSynchronize(S.copy_stream));
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
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
  if (g->owned) CK(cudaFree(g->base));
  if (g->ready) CK(cudaEventDestroy(g->ready));
  if (g->read_done) CK(cudaEventDestroy(g->read_done));
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
  // (a copy to or from pageable memory blocks the host until the stream
  // reaches it: drain the stream first, under the multi-rank watchdog)
  if (gscl_status ss = sync_main(); ss != GSCL_OK) return ss;
  const size_t plane_bytes = w * rows_per_plane;
  const size_t kChunk = (size_t)256 << 20;
  if (bytes < ((size_t)8 << 20) || plane_bytes > kChunk) {
    char* dev = static_cast<char*>(g->base) + (size_t)(g->ox - g->h) * g->es;
    const size_t dp = (size_t)g->pitch * g->es;
    if (to_host)
      CK(cudaMemcpy2DAsync(host, w, dev, dp, w, rows, cudaMemcpyDeviceToHost, S.stream));
    else
      CK(cudaMemcpy2DAsync(dev, dp, host, w, w, rows, cudaMemcpyHostToDevice, S.stream));
    if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
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
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
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

gscl_status gscl_grid_copy_to_host_async(gscl_grid_t g, void* host, size_t bytes) {
  GSCL_TRY
  NEED_INIT();
  if (gscl_status s = check_grid(g, "grid"); s != GSCL_OK) return s;
  if (!host) return fail(GSCL_E_INVALID_ARG, "host pointer is NULL");
  const size_t w = (size_t)(g->nx + 2 * g->h) * g->es;
  const size_t planes = (size_t)(g->nzl + 2 * g->h);
  const size_t need = w * (size_t)(g->ny + 2 * g->h) * planes;
  if (bytes != need) return fail(GSCL_E_INVALID_ARG, "host buffer has %zu bytes, dense slab needs %zu", bytes, need);
  // the download reads what the library stream has written so far
  CK(cudaEventRecord(S.ev_to_down, S.stream));
  CK(cudaStreamWaitEvent(S.down_stream, S.ev_to_down, 0));
  const unsigned slot = S.down_next++ & 1u;  // two staging slots (in order on the download stream)
  if (S.down_cap[slot] < bytes) {
    CK(cudaStreamSynchronize(S.down_stream));
    if (S.down_stage[slot]) CK(cudaFree(S.down_stage[slot]));
    S.down_stage[slot] = nullptr;
    S.down_cap[slot] = 0;
    CK(cudaMalloc(&S.down_stage[slot], bytes));
    S.down_cap[slot] = bytes;
  }
  CK(launch_repack(view_of(g), S.down_stage[slot], 0, (int64_t)planes, false, S.down_stream, &S.launches));
  if (!g->read_done) CK(cudaEventCreateWithFlags(&g->read_done, cudaEventDisableTiming));
  CK(cudaEventRecord(g->read_done, S.down_stream));  // the grid may be overwritten after this
  g->dl_pending = true;
  CK(cudaMemcpyAsync(host, S.down_stage[slot], bytes, cudaMemcpyDeviceToHost, S.down_stream));
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
  if (S.world > 1) {
    if (S.comm) {
      NK(ncclAllReduce(S.d_digest, S.d_digest, 1, ncclUint64, ncclSum, S.comm, S.stream));
    } else if (S.peer.ready) {  // no communicator: the peer arena's slots, an integer fold
      double* d = reinterpret_cast<double*>(S.d_digest);
      if (gscl_status s = peer_combine(d, kFoldU64Sum, d, S.stream, S.stream, nullptr); s != GSCL_OK) return s;
    } else {
      return fail(GSCL_E_STATE, "no NCCL communicator and no peer set (gscl_peer_export/import)");
    }
  }
  CK(cudaMemcpyAsync(S.h_pinned, S.d_digest, 8, cudaMemcpyDeviceToHost, S.stream));
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
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
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
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

gscl_status gscl_pass_units_op(gscl_op op, int64_t nx, int64_t ny, gscl_dtype dtype, int64_t* units) {
  GSCL_TRY
  if (!units || nx <= 0 || ny <= 0 || (dtype != GSCL_F64 && dtype != GSCL_F32))
    return fail(GSCL_E_INVALID_ARG, "bad arguments");
  if (op == GSCL_OP_JACOBI7) *units = pass_tiles(nx, ny, dtype == GSCL_F64 ? 0 : 1, S.variant);
  else if (op == GSCL_OP_VARCOEF8) *units = pass_tiles_v(nx, ny, dtype == GSCL_F64 ? 0 : 1);
  else return fail(GSCL_E_UNSUPPORTED, "two-sweep passes support JACOBI7 and VARCOEF8 (got %d)", (int)op);
  return GSCL_OK;
  GSCL_CATCH
}

gscl_status gscl_do_all_pass2_coeffs(gscl_op op, gscl_grid_t in, const gscl_grid_t* coeffs, int n_coeffs,
                                     gscl_grid_t out, const void* ghost, const void* cghost, int phys_lo,
                                     int phys_hi, const gscl_pass_peer* peer) {
  GSCL_TRY
  Nvtx nv_call("gscl.do_all_pass2");
  NEED_INIT();
  if (op != GSCL_OP_JACOBI7 && op != GSCL_OP_VARCOEF8)
    return fail(GSCL_E_UNSUPPORTED, "two-sweep passes support JACOBI7 and VARCOEF8 (got %d)", (int)op);
  const int nc = op == GSCL_OP_VARCOEF8 ? 7 : 0;
  if (n_coeffs != nc) return fail(GSCL_E_ARITY, "op %d takes %d coefficient grids, got %d", (int)op, nc, n_coeffs);
  if (gscl_status s = check_grid(in, "in"); s != GSCL_OK) return s;
  if (gscl_status s = check_grid(out, "out"); s != GSCL_OK) return s;
  if (gscl_status s = same_shape(in, out); s != GSCL_OK) return s;
  if (nc && !coeffs) return fail(GSCL_E_INVALID_ARG, "coeffs is NULL");
  for (int i = 0; i < nc; ++i) {
    if (gscl_status s = check_grid(coeffs[i], "coefficient grid"); s != GSCL_OK) return s;
    if (gscl_status s = same_shape(in, coeffs[i]); s != GSCL_OK) return s;
    if (coeffs[i]->h != 0) return fail(GSCL_E_INVALID_ARG, "coefficient grids of a pass have halo 0");
    if (coeffs[i]->base == out->base) return fail(GSCL_E_INVALID_ARG, "out aliases a coefficient grid");
  }
  if (in == out || in->base == out->base) return fail(GSCL_E_INVALID_ARG, "in and out alias");
  if (in->h < 1) return fail(GSCL_E_HALO_VIOLATION, "in needs halo >= 1");
  if (!ghost && in->h < 2 && (!phys_lo || !phys_hi))
    return fail(GSCL_E_INVALID_ARG, "ghost planes are needed for a non-physical z side when halo < 2");
  if (nc && !cghost && (!phys_lo || !phys_hi))
    return fail(GSCL_E_INVALID_ARG, "coefficient ghost planes are needed for a non-physical z side");
  Box full;
  if (gscl_status s = local_box(in, nullptr, &full); s != GSCL_OK) return s;
  if (full.empty()) return GSCL_OK;
  SweepPlan p;
  p.op = op == GSCL_OP_VARCOEF8 ? OP_VARCOEF8 : OP_JACOBI7;
  p.n_in = 1 + nc;
  p.in[0] = view_of(in);
  for (int i = 0; i < nc; ++i) p.in[1 + i] = view_of(coeffs[i]);
  p.out = view_of(out);
  p.box = full;
  p.write = true;
  p.tsteps = 2;
  p.phys_lo = phys_lo != 0;
  p.phys_hi = phys_hi != 0;
  p.ghost = ghost;
  p.cghost = nc ? cghost : nullptr;
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

gscl_status gscl_do_all_pass2(gscl_op op, gscl_grid_t in, gscl_grid_t out, const void* ghost, int phys_lo,
                              int phys_hi, const gscl_pass_peer* peer) {
  if (op != GSCL_OP_JACOBI7) return fail(GSCL_E_UNSUPPORTED, "gscl_do_all_pass2 is JACOBI7 (got %d)", (int)op);
  return gscl_do_all_pass2_coeffs(op, in, nullptr, 0, out, ghost, nullptr, phys_lo, phys_hi, peer);
}

// Ordered iteration spaces (NEXT-4): do_{i,j,k}_{inc,dec}
// with PREFIX and do_diamond with PASCAL; the kernels are in ordered.cu.
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
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
  for (auto& tp : S.pending) {
    float t = 0;
    CK(cudaEventElapsedTime(&t, tp.a, tp.b));
    S.kind_ms[tp.kind] += t;
    S.kind_n[tp.kind] += tp.count;
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

gscl_status gscl_set_option(const char* name, int64_t value) {
  GSCL_TRY
  NEED_INIT();
  if (!name) return fail(GSCL_E_INVALID_ARG, "name is NULL");
  std::string n(name);
  if (n == "graph") {
    if (value < 0 || value > 2) return fail(GSCL_E_INVALID_ARG, "graph must be 0, 1 or 2");
    S.graph = (int)value;
  } else if (n == "transport") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "transport must be 0 (NCCL) or 1 (peer memory)");
    S.transport = (int)value;
  } else if (n == "tblock") {
    if (value != 0 && value != 1 && value != 2) return fail(GSCL_E_INVALID_ARG, "tblock must be 0, 1 or 2");
    S.tblock = (int)value;
  } else if (n == "halo_off") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "halo_off must be 0 or 1");
    S.halo_off = (int)value;
  } else if (n == "timeout_ms") {
    if (value < 0) return fail(GSCL_E_INVALID_ARG, "timeout_ms must be >= 0");
    S.timeout_ms = value == 0 ? 120000 : value;
  } else if (n == "split") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "split must be 0 or 1");
    S.split = (int)value;
#ifdef GSCL_ABLATIONS
  // ablation knobs (GSCL_ABLATIONS builds only; results in profiles/)
  } else if (n == "split_one") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "split_one must be 0 or 1");
    S.split_one = (int)value;
  } else if (n == "sweep_impl") {
    if (value < 0 || value > 2) return fail(GSCL_E_INVALID_ARG, "sweep_impl must be 0, 1 or 2");
    S.impl = (int)value;
  } else if (n == "zchunks") {
    if (value < 0) return fail(GSCL_E_INVALID_ARG, "zchunks must be >= 0");
    S.zchunks = (int)value;
  } else if (n == "zalt") {
    if (value != 0 && value != 1) return fail(GSCL_E_INVALID_ARG, "zalt must be 0 or 1");
    S.zalt = (int)value;
  } else if (n == "variant") {
    // 1..5: sweep_tma geometries; 1..4: sweep2.cu; 11..16, 40..59, 91..97: sweep2r.cu (sweep2v/k: 11..16)
    if (value < 0 || (value > 5 && !(value >= 11 && value <= 16) && !(value >= 40 && value <= 60) &&
                      !(value >= 90 && value <= 99)))
      return fail(GSCL_E_INVALID_ARG, "variant must be 0..5, 11..16, 40..59 or 91..99");
    S.variant = (int)value;
  } else if (n == "sched") {
    if (value < 0 || value > 2) return fail(GSCL_E_INVALID_ARG, "sched must be 0, 1 or 2");
    S.sched = (int)value;
  } else if (n == "stages") {
    if (value != 0 && value != 4 && value != 8) return fail(GSCL_E_INVALID_ARG, "stages must be 0, 4 or 8");
    S.stages = (int)value;
  } else if (n == "l2promo") {
    if (value < 0 || value > 3) return fail(GSCL_E_INVALID_ARG, "l2promo must be 0..3");
    S.l2promo = (int)value;
#else
  } else if (n == "sweep_impl" || n == "zchunks" || n == "zalt" || n == "variant" || n == "sched" ||
             n == "stages" || n == "l2promo") {
    if (value != 0)
      return fail(GSCL_E_UNSUPPORTED, "'%s' is an ablation knob: build with GSCL_ABLATIONS=1", name);
#endif
  } else {
    return fail(GSCL_E_UNSUPPORTED, "unknown option '%s'", name);
  }
  return GSCL_OK;
  GSCL_CATCH
}

}  // extern "C"

