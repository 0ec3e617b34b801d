// jacobi.cu — the device-resident drivers of include/gscl.h: gscl_jacobi_run
// (single sweeps, two-sweep passes, the overlapped multi-rank schedules over
// NCCL or peer memory), gscl_converge_run (the paper's convergence loop as a
// conditional-WHILE CUDA graph) and gscl_rbgs_run (red-black Gauss-Seidel).
#include "abi_state.h"

using namespace gscl;
using namespace gscl_abi;

extern "C" {

// Whether jacobi_run takes the multi-rank two-sweep schedule: JACOBI7 on the
// TMA path, tblock auto or 2, several ranks (or "split" on one), and at least 6
// planes on every rank (2 boundary planes per end + the interior; the same
// decision on every rank, so the NCCL call sequences match).
static bool pairs_multirank(gscl_op op, const gscl_grid_s* u) {
  // (h <= 2: after a pass only the 2 boundary planes at each end are final when
  // the comm stream starts the exchange; a deeper halo would send planes the
  // pass's interior units may still be writing)
  return (op == GSCL_OP_JACOBI7 || op == GSCL_OP_VARCOEF8) && S.impl == 0 && (S.tblock == 0 || S.tblock == 2) &&
         (S.world > 1 || S.split) && u->nz / S.world >= 6 && u->nx > 0 && u->ny > 0 && u->h <= 2;
}

// VARCOEF8 passes on slabs read the coefficient planes next to the slab from a
// ghost buffer in the layout of a halo-0 coefficient grid; coefficient grids
// with a halo keep the single-sweep schedule on several ranks.
static bool coeffs_pass_ok(const gscl_grid_t* coeffs, int nc) {
  for (int i = 0; i < nc; ++i)
    if (coeffs[i]->h != 0) return false;
  return true;
}

// The per-call plumbing of the peer-memory transport: a rank's view of its
// neighbours' storage / arena, the counters, and the start barrier.
struct P2PLink {
  PeerSet& P;
  const gscl_grid_s* g;
  size_t pb;
  int64_t h, n;
  bool lo, hi;
  char* my_ar;
  unsigned *my_flags, *lo_flags, *hi_flags;
  explicit P2PLink(const gscl_grid_s* grid) : P(S.peer), g(grid) {
    pb = P.plane_bytes;
    h = g->h;
    n = g->nzl;
    lo = S.rank > 0;
    hi = S.rank < S.world - 1;
    my_ar = P.arena_of[S.rank];
    my_flags = PeerSet::flags_of(my_ar, pb);
    lo_flags = lo ? PeerSet::flags_of(P.arena_of[S.rank - 1], pb) : nullptr;
    hi_flags = hi ? PeerSet::flags_of(P.arena_of[S.rank + 1], pb) : nullptr;
  }
  // storage index (0 / 1 = u / v at export) of u's current storage
  gscl_status input_storage(const gscl_grid_s* u, const gscl_grid_s* v, int* cur) const {
    if (u->base == P.store_base[0] && v->base == P.store_base[1]) *cur = 0;
    else if (u->base == P.store_base[1] && v->base == P.store_base[0]) *cur = 1;
    else return fail(GSCL_E_INVALID_ARG, "u / v are not the grids of gscl_peer_export");
    return GSCL_OK;
  }
  char* plane_ptr(void* base, int64_t z) const { return static_cast<char*>(base) + (z + h) * pb; }
  void* origin(char* plane_start) const {
    return static_cast<void*>(plane_start + (h * g->pitch + g->ox) * (int64_t)g->es);
  }
  // receiving plane k (0 nearest) on a neighbour for an output in storage st
  char* recv_plane(int side, int st, int k) const {
    if (side == 0) {  // lower: its planes nzl, nzl+1
      const int64_t z = P.nzl_nb[0] + k;
      if (z < P.nzl_nb[0] + h) return plane_ptr(P.nb_store[0][st], z);
      return PeerSet::ghost_of(P.arena_of[S.rank - 1], pb, st) + pb;  // its ghost plane "above"
    }
    const int64_t z = -1 - k;  // upper: its planes -1, -2
    if (z >= -h) return plane_ptr(P.nb_store[1][st], z);
    return PeerSet::ghost_of(P.arena_of[S.rank + 1], pb, st);  // its ghost plane "below"
  }
  gscl_status signal(unsigned* lof, unsigned* hif, unsigned add) const {
    PeerPtrs8 f{};
    if (lof) f.p[f.n++] = lof;
    if (hif) f.p[f.n++] = hif;
    if (f.n) CK(launch_signal(f, add, S.stream, &S.launches));
    return GSCL_OK;
  }
  gscl_status wait_nb(int idx_lo, int idx_hi, cudaStream_t st = nullptr) const {
    if (!st) st = S.stream;
    if (lo) CK(stream_wait_geq(st, my_flags + idx_lo, P.tgt[idx_lo]));
    if (hi) CK(stream_wait_geq(st, my_flags + idx_hi, P.tgt[idx_hi]));
    return GSCL_OK;
  }
  // copy whole boundary planes of storage st (both depths) into the neighbours
  gscl_status copy_planes(int st) const {
    for (int k = 0; k < 2; ++k) {
      if (lo) CK(cudaMemcpyAsync(recv_plane(0, st, k), plane_ptr(P.store_base[st], k), pb,
                                 cudaMemcpyDeviceToDevice, S.stream));
      if (hi) CK(cudaMemcpyAsync(recv_plane(1, st, k), plane_ptr(P.store_base[st], n - 1 - k), pb,
                                 cudaMemcpyDeviceToDevice, S.stream));
    }
    return GSCL_OK;
  }
  // one step's boundary planes (depth 2) copied, then the neighbours signalled
  gscl_status copy_and_signal(int st) {
    if (gscl_status s = copy_planes(st); s != GSCL_OK) return s;
    if (gscl_status s = signal(lo ? lo_flags + 1 : nullptr, hi ? hi_flags + 0 : nullptr, (unsigned)P.units);
        s != GSCL_OK)
      return s;
    if (lo) P.tgt[0] += (unsigned)P.units;
    if (hi) P.tgt[1] += (unsigned)P.units;
    return GSCL_OK;
  }
  // ---- start barrier: neighbours are done with their previous call; setup
  // copies of both storages (the x/y boundary ring of every receiving plane,
  // and the first input's planes); second round: their copies into us landed
  // the coefficient planes next to the slab into the neighbours' arenas
  // (VARCOEF8 passes; the coefficient grids have no halo): grid c's plane 0
  // -> the lower neighbour's coefficient ghost plane 2c + 1, plane nzl - 1 ->
  // the upper neighbour's plane 2c
  gscl_status copy_coeff_planes(const gscl_grid_t* coeffs, int nc) const {
    const size_t cpb = P.cplane_bytes;
    for (int c = 0; c < nc; ++c) {
      const char* base = static_cast<const char*>(coeffs[c]->base);
      if (lo)
        CK(cudaMemcpyAsync(PeerSet::cghost_of(P.arena_of[S.rank - 1], pb) + (size_t)(2 * c + 1) * cpb, base, cpb,
                           cudaMemcpyDeviceToDevice, S.stream));
      if (hi)
        CK(cudaMemcpyAsync(PeerSet::cghost_of(P.arena_of[S.rank + 1], pb) + (size_t)(2 * c) * cpb,
                           base + (size_t)(n - 1) * cpb, cpb, cudaMemcpyDeviceToDevice, S.stream));
    }
    return GSCL_OK;
  }
  gscl_status begin(int cur, const gscl_grid_t* coeffs = nullptr, int nc = 0) {
    for (int round = 0; round < 2; ++round) {
      if (round == 1) {
        if (gscl_status s = copy_planes(cur); s != GSCL_OK) return s;
        if (gscl_status s = copy_planes(1 - cur); s != GSCL_OK) return s;
        if (gscl_status s = copy_coeff_planes(coeffs, nc); s != GSCL_OK) return s;
      }
      if (gscl_status s = signal(lo ? lo_flags + 3 : nullptr, hi ? hi_flags + 2 : nullptr, 1); s != GSCL_OK)
        return s;
      if (lo) ++P.tgt[2];
      if (hi) ++P.tgt[3];
      if (gscl_status s = wait_nb(2, 3); s != GSCL_OK) return s;
    }
    return GSCL_OK;
  }
};

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
  // JACOBI7 and VARCOEF8 pair sweeps into two-sweep passes (a slab needs >= 6
  // planes); JACOBI27 runs single sweeps
  const bool can_pair = (op == GSCL_OP_JACOBI7 || op == GSCL_OP_VARCOEF8) && S.impl == 0 &&
                        (S.tblock == 0 || S.tblock == 2) && u->nz / S.world >= 6 && u->h <= 2 &&
                        coeffs_pass_ok(coeffs, nc);
  const int check_rv = op == GSCL_OP_VARCOEF8 ? RV_SQ : RV_RESID;
  // single sweeps of a schedule without passes store the boundary planes into
  // the neighbours from the kernel (the h planes each next sweep needs); the
  // unpaired steps of a pass schedule copy 2 planes (a pass follows)
  const bool fuse_single = !can_pair && S.impl == 0 && u->nz / S.world > 2 * u->h;
  // what each neighbour's counter grows by per pass: the pass kernel's
  // boundary units per side (its x-y tiles)
  const int64_t pu = op == GSCL_OP_VARCOEF8 ? pass_tiles_v(u->nx, u->ny, u->dtype) : P.units;
  P2PLink L(u);
  int cur;  // storage index of the current input
  if (gscl_status s = L.input_storage(u, v, &cur); s != GSCL_OK) return s;
  // the boundary units a pass signals per side follow the pass geometry in
  // effect now: check them against the peer set's count before anything is
  // launched or signalled (a mismatch found after a launch would leave the
  // neighbours waiting on counters that never reach their targets)
  if (can_pair && op == GSCL_OP_JACOBI7 && pass_tiles(u->nx, u->ny, u->dtype, S.variant) != P.units)
    return fail(GSCL_E_STATE, "pass geometry changed since gscl_peer_import (re-run the peer setup)");
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
  const int64_t h = u->h;
  const bool lo = L.lo, hi = L.hi;
  const size_t pb = L.pb;
  char* my_ar = L.my_ar;
  unsigned* my_flags = L.my_flags;
  unsigned* lo_flags = L.lo_flags;
  unsigned* hi_flags = L.hi_flags;
  auto origin = [&](char* plane_start) { return L.origin(plane_start); };
  auto recv_plane = [&](int side, int st, int k) { return L.recv_plane(side, st, k); };
  auto signal = [&](unsigned* lof, unsigned* hif, unsigned add) { return L.signal(lof, hif, add); };
  auto wait_nb = [&](int idx_lo, int idx_hi) { return L.wait_nb(idx_lo, idx_hi); };
  auto copy_planes = [&](int st) { return L.copy_planes(st); };
  if (gscl_status s = L.begin(cur, can_pair ? coeffs : nullptr, can_pair ? nc : 0); s != GSCL_OK) return s;
  cudaStream_t CS = S.comm_stream;
  // residual partial -> every rank's slot q; the comm stream folds slot q
  auto check_combine = [&](double* loc, double* glob) -> gscl_status {
    return peer_combine(loc, GSCL_SUM, glob, S.stream, CS, S.ev_to_comm);
  };
  View a = vu, b = vv;
  gscl_grid_s* ga = u;
  gscl_grid_s* gb = v;
  // JACOBI7 passes as two launches, as in enqueue_jacobi_pairs: the boundary
  // chunks B(k) on the comm stream after the neighbour wait (only they read
  // the received planes and store into the neighbours), the middle chunks
  // M(k) on the library stream, waiting only for B(k-1) — never for a
  // neighbour.  `joined` = the library stream has waited for the comm stream.
  // (default geometry only: the launcher splits exactly those passes, so a
  // pass issued as `two` always runs as two launches)
  const bool split2 = op == GSCL_OP_JACOBI7 && !S.split_one && S.variant == 0;
  bool joined = true;
  auto join = [&]() -> gscl_status {
    if (joined) return GSCL_OK;
    joined = true;
    return hand_off(CS, S.stream, S.ev_to_main);
  };
  for (size_t k = 0; k < steps.size(); ++k) {
    const Step& st = steps[k];
    const bool two = split2 && st.pair;
    if (!two)
      if (gscl_status s = join(); s != GSCL_OK) return s;
    if (k > 0 && !two)
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
      inc = (unsigned)pu;
      p.tsteps = 2;
      p.phys_lo = !lo;
      p.phys_hi = !hi;
      p.ghost = PeerSet::ghost_of(my_ar, pb, cur);
      if (nc) p.cghost = PeerSet::cghost_of(my_ar, pb);
      p.bnd_h = 1;
      for (int i = 0; i < 2; ++i) {
        p.peer_lo[i] = lo ? origin(recv_plane(0, out_st, i)) : nullptr;
        p.peer_hi[i] = hi ? origin(recv_plane(1, out_st, i)) : nullptr;
      }
      p.peer_flag_lo = lo ? lo_flags + 1 : nullptr;  // the lower neighbour hears from above
      p.peer_flag_hi = hi ? hi_flags + 0 : nullptr;
      int64_t units = 0;
      p.bnd_units = &units;
      bool did2 = false;
      if (two) {
        // B(k): after everything on the library stream (M(k-1)) and the
        // neighbours' B(k-1) signals; M(k): after B(k-1)
        if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
        if (k > 0)
          if (gscl_status s = L.wait_nb(0, 1, CS); s != GSCL_OK) return s;
        if (!joined) CK(cudaStreamWaitEvent(S.stream, S.ev_bnd, 0));
        p.bnd_stream = CS;
        p.bnd_split = &did2;
      }
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      if (units != 2 * pu)  // (tiles at each end)
        return fail(GSCL_E_STATE, "pass boundary units %lld != 2 x %lld", (long long)units, (long long)pu);
      if (two && !did2) return fail(GSCL_E_STATE, "the two-launch pass was not split");
      if (two) {
        CK(cudaEventRecord(S.ev_bnd, CS));
        joined = false;
        // (the residual of a check pass is final once both launches ended)
        if (st.check) CK(cudaStreamWaitEvent(S.stream, S.ev_bnd, 0));
      }
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
  if (gscl_status s = join(); s != GSCL_OK) return s;
  // The neighbours' last stores into this rank's halo / ghost planes (their
  // last step's signal) must land before the call returns, checks or not: a
  // later call that reads or overwrites those planes would race the remote
  // stores otherwise.
  if (!steps.empty())
    if (gscl_status s = wait_nb(0, 1); s != GSCL_OK) return s;
  if (check_every > 0) {
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
static gscl_status enqueue_jacobi_pairs(gscl_op op, gscl_grid_s* u, gscl_grid_s* v, const gscl_grid_t* coeffs,
                                        int nc, int iters, int check_every, int nh, bool* final_in_v) {
  const View vu = view_of(u), vv = view_of(v);
  const int check_rv = op == GSCL_OP_VARCOEF8 ? RV_SQ : RV_RESID;
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
  auto xchg = [&](gscl_grid_s* g, int depth) -> gscl_status {
    if (S.halo_off) return GSCL_OK;  // (timing only: the compute-only step)
    return depth == 2 ? exchange_pass(g, CS) : exchange(g, CS);
  };
  auto depth_of = [&](size_t k) { return k < steps.size() && steps[k].pair ? 2 : 1; };
  View a = vu, b = vv;
  gscl_grid_s* ga = u;
  gscl_grid_s* gb = v;
  if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
  // VARCOEF8: the coefficient planes just outside the slab (the coefficient
  // grids have no halo), exchanged once per call — they never change
  if (multi && nc > 0)
    if (gscl_status s = exchange_coeff_ghosts(coeffs, nc, CS); s != GSCL_OK) return s;
  if (gscl_status s = xchg(ga, depth_of(0)); s != GSCL_OK) return s;
  if (gscl_status s = hand_off(CS, S.stream, S.ev_to_main); s != GSCL_OK) return s;
  // JACOBI7 passes run as two launches (SweepPlan::bnd_stream): the boundary
  // chunks B(k) on the comm stream, then the exchange of their planes there;
  // the middle chunks M(k) on the library stream.  B(k) reads planes M(k-1)
  // wrote (and the exchanged halo: comm-stream order); M(k) reads planes
  // B(k-1) wrote but never the halo — so M(k) waits only for B(k-1) (ev_bnd),
  // not for the exchange, which overlaps M(k) whole.  `joined` = the library
  // stream has waited for everything on the comm stream.
  // (JACOBI7 only: for VARCOEF8 the multi-rank kernel costs nothing and its
  // 2-plane boundary units as a launch of their own made the pass 2 % slower,
  // profiles/r02_sweep2r.md)
  // (default geometry only: the launcher splits exactly those passes)
  const bool split2 = op == GSCL_OP_JACOBI7 && !S.split_one && S.variant == 0;
  bool joined = true;
  auto join = [&]() -> gscl_status {
    if (joined) return GSCL_OK;
    joined = true;
    return hand_off(CS, S.stream, S.ev_to_main);
  };
  for (size_t k = 0; k < steps.size(); ++k) {
    const Step& st = steps[k];
    double* glob = st.check ? S.d_hist + st.slot : nullptr;
    double* res = st.check ? (multi ? S.d_lochist + st.slot : glob) : nullptr;
    const int next = depth_of(k + 1);
    SweepPlan p;
    p.op = op;
    p.n_in = 1 + nc;
    p.in[0] = a;
    for (int i = 0; i < nc; ++i) p.in[1 + i] = view_of(coeffs[i]);
    p.out = b;
    p.box = full;
    p.write = true;
    p.rv = st.check ? check_rv : RV_NONE;
    if (st.check) p.red = red_target(res, GSCL_SUM);
    if (st.pair) {
      p.tsteps = 2;
      p.phys_lo = S.rank == 0;
      p.phys_hi = S.rank == S.world - 1;
      p.ghost = S.d_ghost;
      if (nc > 0 && multi) p.cghost = S.d_cghost;
      p.bnd_h = 1;
      p.bflag = S.d_bflag;
      int64_t units = 0;
      p.bnd_units = &units;
      bool did2 = false;
      if (split2) {
        // B(k) after everything issued on the library stream (M(k-1)); M(k)
        // after B(k-1) (recorded on the comm stream before its exchange)
        if (gscl_status s = hand_off(S.stream, CS, S.ev_to_comm); s != GSCL_OK) return s;
        if (!joined) CK(cudaStreamWaitEvent(S.stream, S.ev_bnd, 0));
        p.bnd_stream = CS;
        p.bnd_split = &did2;
      } else {
        if (gscl_status s = join(); s != GSCL_OK) return s;
      }
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      if (split2 && !did2) return fail(GSCL_E_STATE, "the two-launch pass was not split");
      if (did2) CK(cudaEventRecord(S.ev_bnd, CS));
      if (st.check && multi) CK(cudaEventRecord(S.ev_to_comm, S.stream));  // the pass's end
      if (did2) {
        S.bflag_target += (unsigned)units;  // (the boundary units still bump the counter)
      } else if (units > 0) {
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
      if (did2 && next == 2) {
        joined = false;  // the next pass's M waits for this B only
      } else {
        CK(cudaStreamWaitEvent(S.stream, S.ev_halo, 0));
        joined = true;  // (a pending cross_rank only writes the history: joined at the end)
      }
    } else {
      if (gscl_status s = join(); s != GSCL_OK) return s;
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
  if (gscl_status s = join(); s != GSCL_OK) return s;
  if (check_every > 0) {  // the final iterate's halo arrived with the last exchange
    double* glob = S.d_hist + (nh - 1);
    double* res = multi ? S.d_lochist + (nh - 1) : glob;
    if (op == GSCL_OP_VARCOEF8) {
      CK(launch_reduce_points(1 /*SQ*/, &a, 1, full, 0.0, red_target(res, GSCL_SUM), S.num_sms, S.stream,
                              &S.launches));
    } else {
      SweepPlan p;
      p.op = OP_JACOBI7;
      p.rv = RV_RESID;
      p.write = false;
      p.n_in = 1;
      p.in[0] = a;
      p.box = full;
      p.red = red_target(res, GSCL_SUM);
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
    }
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

// The device work of one gscl_jacobi_run (everything but the history copy and
// the host sync), issued on the library streams; *final_in_v reports whether
// the final iterate ends in v's storage.
static gscl_status enqueue_jacobi(gscl_op op, gscl_grid_s* u, gscl_grid_s* v, const gscl_grid_t* coeffs,
                                  int nc, int iters, int check_every, int nh, bool* final_in_v) {
  if (S.transport == 1 && S.world > 1 && !(S.halo_off && pairs_multirank(op, u) && coeffs_pass_ok(coeffs, nc))) {
    if (!S.peer.ready) return fail(GSCL_E_STATE, "transport = 1 needs gscl_peer_export / gscl_peer_import");
    if (u->nz / S.world < 2) return fail(GSCL_E_INVALID_DOMAIN, "the peer transport needs >= 2 planes per rank");
    return enqueue_jacobi_p2p(op, u, v, coeffs, nc, iters, check_every, nh, final_in_v);
  }
  if (pairs_multirank(op, u) && coeffs_pass_ok(coeffs, nc))
    return enqueue_jacobi_pairs(op, u, v, coeffs, nc, iters, check_every, nh, final_in_v);
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
  // (VARCOEF8: sweep2v.cu reads the 7 coefficient grids once per pass;
  // JACOBI27: sweep2k.cu, opt-in with tblock = 2 in ablation builds only —
  // measured slower than single sweeps, profiles/r01_sweep2k.md)
#ifdef GSCL_ABLATIONS
  constexpr bool kJ27Pairs = true;
#else
  constexpr bool kJ27Pairs = false;
#endif
  const bool pairs = S.world == 1 && !full.empty() &&
                     ((op == GSCL_OP_JACOBI7 && (S.tblock == 2 || (S.tblock == 0 && !S.split && S.impl == 0))) ||
                      (op == GSCL_OP_VARCOEF8 && (S.tblock == 2 || (S.tblock == 0 && !S.split)) && S.impl == 0) ||
                      (kJ27Pairs && op == GSCL_OP_JACOBI27 && S.tblock == 2 && S.impl == 0));
  // Instrumentation (gscl_timing_enable): one event pair around each run of
  // consecutive passes, booked as that many pass launches — events between
  // the launches of a run would add their own gaps to the step (1.4-2 % of a
  // config-2 step when every launch was bracketed).
  TimedPair run_tp{};
  int run_n = 0;
  auto run_close = [&]() -> gscl_status {
    if (run_n == 0) return GSCL_OK;
    const int n = run_n;
    run_n = 0;
    return record_end(run_tp, 3, n);
  };
  for (int it = 1; it <= iters; ++it) {
    const bool check = check_every > 0 && it % check_every == 0;
    double* slot = S.d_hist + (it / std::max(check_every, 1) - 1);
    double* res = S.world == 1 ? slot : d_loc;
    if (pairs && !check && it + 1 <= iters) {
      const bool check2 = check_every > 0 && (it + 1) % check_every == 0;
      SweepPlan p;
      p.op = op;
      p.n_in = 1 + nc;
      p.in[0] = a;
      for (int i = 0; i < nc; ++i) p.in[1 + i] = view_of(coeffs[i]);
      p.out = bview;
      p.box = full;
      p.write = true;
      p.tsteps = 2;
      p.rv = check2 ? check_rv : RV_NONE;
      if (check2) p.red = red_target(S.d_hist + ((it + 1) / check_every - 1), GSCL_SUM);
      if (run_n == 0)
        if (gscl_status s = record_start(&run_tp); s != GSCL_OK) return s;
      p.untimed = true;
      if (gscl_status s = run_sweep(p); s != GSCL_OK) return s;
      ++run_n;
      std::swap(a, bview);
      std::swap(ga, gb);
      ++it;  // two sweeps done
      continue;
    }
    if (gscl_status s = run_close(); s != GSCL_OK) return s;
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
  if (gscl_status s = run_close(); s != GSCL_OK) return s;
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

gscl_status gscl_halo_exchange_depth(const gscl_grid_t* grids, int n, int depth) {
  GSCL_TRY
  Nvtx nv_call("gscl.halo_exchange_depth");
  NEED_INIT();
  if (n < 0 || (n > 0 && !grids)) return fail(GSCL_E_INVALID_ARG, "bad grid list");
  if (depth != 1 && depth != 2) return fail(GSCL_E_INVALID_ARG, "depth must be 1 or 2 (got %d)", depth);
  for (int i = 0; i < n; ++i)
    if (gscl_status s = check_grid(grids[i], "grid"); s != GSCL_OK) return s;
  if (S.world == 1) return GSCL_OK;
  if (S.transport == 1) {
    if (n != 1) return fail(GSCL_E_INVALID_ARG, "the peer transport exchanges one grid per call");
    PeerSet& P = S.peer;
    if (!P.ready) return fail(GSCL_E_STATE, "transport = 1 needs gscl_peer_export / gscl_peer_import");
    gscl_grid_s* g = grids[0];
    int st = -1;
    for (int k = 0; k < 2; ++k)
      if (g->base == P.store_base[k]) st = k;
    if (st < 0) return fail(GSCL_E_INVALID_ARG, "grid is not one of the gscl_peer_export pair");
    if (g->nzl < 2) return fail(GSCL_E_INVALID_DOMAIN, "the peer transport needs >= 2 planes per rank");
    P2PLink L(g);
    // ready round: a neighbour's earlier stream work on its grid (a fill, a
    // sweep writing its halo shell) must be done before this rank's copies
    // land in its halo planes — NCCL gets that from the matched receive
    if (gscl_status s = L.signal(L.lo ? L.lo_flags + 3 : nullptr, L.hi ? L.hi_flags + 2 : nullptr, 1);
        s != GSCL_OK)
      return s;
    if (L.lo) ++P.tgt[2];
    if (L.hi) ++P.tgt[3];
    if (gscl_status s = L.wait_nb(2, 3); s != GSCL_OK) return s;
    // (always both planes: the receiving side's layout is the pass's)
    if (gscl_status s = L.copy_and_signal(st); s != GSCL_OK) return s;
    return L.wait_nb(0, 1);
  }
  for (int i = 0; i < n; ++i) {
    gscl_status s = depth == 2 ? exchange_pass(grids[i], S.stream) : exchange(grids[i], S.stream);
    if (s != GSCL_OK) return s;
  }
  return GSCL_OK;
  GSCL_CATCH
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
      const int64_t l0 = S.launches;
      gscl_status st;
      cudaGraph_t g = nullptr;
      cudaError_t ec;
      {
        CaptureScope cs;
        CK(cudaStreamBeginCapture(S.stream, cudaStreamCaptureModeRelaxed));
        st = enqueue_jacobi(op, u, v, coeffs, nc, iters, check_every, nh, &final_in_v);
        ec = cudaStreamEndCapture(S.stream, &g);
      }
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
    CK(cudaMemcpyAsync(S.h_hist, S.d_hist, (size_t)nh * sizeof(double), cudaMemcpyDeviceToHost, S.stream));
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
  for (int i = 0; i < nh; ++i) history[i] = std::sqrt(S.h_hist[i]);
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
      CaptureScope capture_scope;  // (the body is captured on a capturable stream)
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
    if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
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
  // several ranks over the peer-memory transport: the halo planes of each
  // iteration's output are copied into the neighbours (IPC / NVLink) and
  // signalled; the next iteration waits for the neighbours' signals
  const bool p2p = S.world > 1 && S.transport == 1;
  if (p2p && !S.peer.ready) return fail(GSCL_E_STATE, "transport = 1 needs gscl_peer_export / gscl_peer_import");
  P2PLink L(u);
  int cur = 0;
  if (p2p) {
    if (u->nz / S.world < 2) return fail(GSCL_E_INVALID_DOMAIN, "the peer transport needs >= 2 planes per rank");
    if (gscl_status s = L.input_storage(u, v, &cur); s != GSCL_OK) return s;
    if (gscl_status s = L.begin(cur); s != GSCL_OK) return s;
  }
  for (int it = 1; it <= max_iters; ++it) {
    // one iteration of the paper's loop: b = OP(a) fused with the AND-reduced
    // convergence test |b - a| <= eps; skipped on device once converged
    if (p2p) {
      if (it > 1)
        if (gscl_status s = L.wait_nb(0, 1); s != GSCL_OK) return s;
    } else if (gscl_status s = exchange(ga); s != GSCL_OK) {
      return s;
    }
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
    if (p2p) {
      if (gscl_status s = L.copy_and_signal(1 - cur); s != GSCL_OK) return s;
      cur = 1 - cur;
    }
    if (gscl_status s = cross_rank(d_loc, GSCL_AND, d_res, S.stream); s != GSCL_OK) return s;
    CK(launch_conv_update(d_res, S.d_conv, S.d_conv + 1, it, S.stream, &S.launches));
    std::swap(a, b);
    std::swap(ga, gb);
    if (it % batch == 0 || it == max_iters) {
      CK(cudaMemcpyAsync(h_flags, S.d_conv, 2 * sizeof(int), cudaMemcpyDeviceToHost, S.stream));
      if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
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
        if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
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
    CK(cudaMemcpyAsync(S.h_hist, S.d_hist, (size_t)nh * sizeof(double), cudaMemcpyDeviceToHost, S.stream));
  }
  if (gscl_status ss_ = sync_main(); ss_ != GSCL_OK) return ss_;
  for (int i = 0; i < nh; ++i) history[i] = std::sqrt(S.h_hist[i]);
  return GSCL_OK;
  GSCL_CATCH
}


}  // extern "C"
