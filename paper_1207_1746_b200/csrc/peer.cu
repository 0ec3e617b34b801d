// peer.cu — the collective setup of the peer-memory halo transport
// (gscl_peer_export / gscl_peer_import: CUDA IPC mappings of the neighbours'
// grid storage and of every rank's arena); the schedule that uses it is
// enqueue_jacobi_p2p in jacobi.cu.
#include "abi_state.h"

using namespace gscl;
using namespace gscl_abi;

extern "C" {

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
  {
    gscl_grid_s c;  // the layout of a halo-0 grid of u's extents (VARCOEF8's coefficients)
    if (gscl_status s = layout(&c, u->nx, u->ny, u->nz, 0, u->dtype, S.rank, S.world); s != GSCL_OK) return s;
    P.cplane_bytes = (size_t)(c.plane * (int64_t)c.es);
  }
  const size_t ab = PeerSet::arena_bytes(P.plane_bytes, P.cplane_bytes);
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


}  // extern "C"
