// internal.h — host-side declarations shared by the ABI layer and the kernel
// translation units (not part of the public C ABI; see include/gscl.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gscl {

// Local box in LOCAL interior coordinates (z relative to the slab), half open.
struct Box {
  int64_t x0, x1, y0, y1, z0, z1;
  bool empty() const { return x0 >= x1 || y0 >= y1 || z0 >= z1; }
  int64_t points() const { return empty() ? 0 : (x1 - x0) * (y1 - y0) * (z1 - z0); }
};

// A device view of one local slab: the allocation, its geometry, and the
// interior origin.  dtype 0 = f64, 1 = f32.
struct View {
  void* base = nullptr;     // start of the allocation (TMA global address)
  void* origin = nullptr;   // element (0,0,0) of the local interior
  int64_t nx = 0, ny = 0, nzl = 0;
  int h = 0;
  int64_t pitch = 0, plane = 0, ox = 0;  // elements
  int dtype = 0;
};

// Reduction destination of one kernel launch: the last CTA folds the
// per-CTA partials in index order into *result (deterministic).
struct RedTarget {
  double* partials = nullptr;
  unsigned* counter = nullptr;
  double* result = nullptr;
  int comb = 0;
  int max_partials = 0;
};

// One sweep launch: op over `box`, reading in[0..n_in) and writing out
// (when write), reducing the rv value into red (when rv != RV_NONE).
struct SweepPlan {
  int op = 0;
  int rv = 0;       // RedVal
  bool write = true;
  int n_in = 1;
  View in[8];
  View out;
  Box box;
  double eps = 0;
  RedTarget red;
  RedTarget red2;   // RV_CONV2 (two-sweep pass): the second iteration's AND
  int impl = 0;     // 0 = TMA ring, 1 = plain per-point kernel
  int zchunks = 0;  // 0 = auto
  int sched = 0;    // 0 = auto, 1 = multi-wave (all chunks stream up), 2 = single wave, alternating
  int l2promo = 0;  // TMA L2 promotion: 0 none, 1 64B, 2 128B, 3 256B
  int stages = 0;   // TMA ring depth: 0 = default, 4, 8 (8 only for 7-point fp64)
  int tsteps = 1;   // sweeps per pass: 1, or 2 (temporal blocking, sweep2.cu)
  int variant = 0;  // kernel variant for ablations (sweep2: x-neighbour source, occupancy)
  const int* stop = nullptr;  // device flag: skip the sweep when set (converge loop)
  int color = -1;             // >= 0: red-black half-sweep, store only this colour (in place)
  bool rbgs = false;          // two-sweep pass = one red-black GS iteration (out of place)
  // boundary-first (multi-rank overlap): the h planes at each end of the box are
  // the first two chunks; each of their units bumps *bflag when its stores are
  // done; *bnd_units (out) receives how many such units the launch has
  int bnd_h = 0;
  unsigned* bflag = nullptr;
  int64_t* bnd_units = nullptr;
  // two-sweep JACOBI7 pass with boundary-first chunks: when set, the boundary
  // chunks run as their own launch of the multi-rank kernel on this stream
  // (the comm stream: the exchange then simply follows in stream order, no
  // counter wait) and the middle chunks as a launch of the single-rank kernel
  // on `stream` — they never touch the slab ends, so they run the leaner code
  // (the multi-rank kernel needs 255 registers with spills, the plain one 245)
  cudaStream_t bnd_stream = nullptr;
  bool* bnd_split = nullptr;  // (out) set when the pass was split that way
  // instrumentation: the caller times this launch together with its
  // neighbours (one event pair around a run of consecutive passes)
  bool untimed = false;
  // walk the z chunks top-down: a sweep that starts where the previous one
  // ended finds those planes still in L2 (jacobi_run alternates it)
  bool reverse = false;
  int64_t zoff = 0;           // global z of local plane 0 (colour parity)
  // two-sweep passes on a multi-rank slab: z ends that are physical
  // boundaries (Dirichlet rule for the intermediate iterate), and a buffer of
  // two planes (the grid's plane layout) holding the input planes below / above
  // the grid's halo (z = -2 / nzl + 1 when h = 1)
  bool phys_lo = true, phys_hi = true;
  const void* ghost = nullptr;
  // VARCOEF8 pass on a multi-rank slab: the coefficient planes just outside
  // the slab (the coefficient grids have no halo): 14 planes of the
  // coefficient grids' plane layout, plane 2c = grid c's plane below the slab,
  // 2c + 1 = above
  const void* cghost = nullptr;
  // peer-memory transport of a boundary-first two-sweep pass: receiving planes
  // on the lower / upper neighbour (interior origins; [0] nearest) and their
  // arrival counters, bumped by each boundary unit after its stores
  void* peer_lo[2] = {nullptr, nullptr};
  void* peer_hi[2] = {nullptr, nullptr};
  unsigned* peer_flag_lo = nullptr;
  unsigned* peer_flag_hi = nullptr;
  // two unsigneds of device memory, zero between launches: the unit ticket
  // and exit count of the persistent (dynamically scheduled) pass kernel
  unsigned* ticket = nullptr;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
};

// Kernel launchers (return cudaError_t of the launch).  *launches is
// incremented by the number of kernels issued.
cudaError_t launch_sweep(const SweepPlan& p, int64_t* launches);
// Two sweeps in one pass (JACOBI7, whole single-rank interior; rv RV_NONE or
// RV_RESID of the intermediate iterate).
cudaError_t launch_sweep2(const SweepPlan& p, int64_t* launches);
// Register-resident two-sweep kernel (sweep2r.cu); launch_sweep2 dispatches to it.
cudaError_t launch_sweep2r(const SweepPlan& p, int64_t* launches);
// VARCOEF8 two-sweep pass (sweep2v.cu; in = u + 7 coefficient grids).
cudaError_t launch_sweep2v(const SweepPlan& p, int64_t* launches);
#ifdef GSCL_ABLATIONS
// Ablation builds only: the JACOBI27 two-sweep pass (sweep2k.cu; rv RV_NONE or
// RV_RESID of the intermediate iterate) and the first JACOBI7 two-sweep design
// with u1 in shared memory (sweep2.cu, variants 1..4).
cudaError_t launch_sweep2k(const SweepPlan& p, int64_t* launches);
cudaError_t launch_sweep2_smem(const SweepPlan& p, int64_t* launches);
#endif
// x-y tiles of the two-sweep pass kernel of `variant` (= boundary units per
// side of a boundary-first pass).  dtype 0 = f64, 1 = f32.
int64_t pass_tiles(int64_t nx, int64_t ny, int dtype, int variant);
// x-y tiles of the VARCOEF8 two-sweep pass (sweep2v.cu).
int64_t pass_tiles_v(int64_t nx, int64_t ny, int dtype);
#ifdef GSCL_ABLATIONS
// JACOBI7 two-sweep pass with u1 rows handed between warps (sweep2x.cu; ablation).
cudaError_t launch_sweep2x(const SweepPlan& p, int64_t* launches);
int64_t pass_tiles_x(int64_t nx, int64_t ny, int dtype);
#endif
cudaError_t launch_reduce_points(int rop, const View* g, int n, const Box& box, double eps,
                                 const RedTarget& red, int num_sms, cudaStream_t s, int64_t* launches);
cudaError_t launch_fill_random(const View& v, int64_t z_begin, uint64_t seed, uint32_t grid_id,
                               double scale, cudaStream_t s, int64_t* launches);
cudaError_t launch_fill_const(const View& v, double value, cudaStream_t s, int64_t* launches);
cudaError_t launch_copy_halo(const View& src, const View& dst, cudaStream_t s, int64_t* launches);
cudaError_t launch_digest(const View& v, int64_t z_begin, uint64_t* d_out, cudaStream_t s,
                          int64_t* launches);
// Repack array planes [p0, p0+np) between a dense staging buffer
// ([np][ny+2h][nx+2h]) and the padded grid layout.
cudaError_t launch_repack(const View& v, void* dense, int64_t p0, int64_t np, bool to_padded,
                          cudaStream_t s, int64_t* launches);
cudaError_t launch_fold(const double* d_vals, int n, int comb, double* d_out, cudaStream_t s,
                        int64_t* launches);
// launch_fold's comb for 64-bit integer words summed mod 2^64 (the digest)
constexpr int kFoldU64Sum = 100;

// Ordered iteration spaces (ordered.cu): space 0..5 = I_INC, I_DEC, J_INC,
// J_DEC, K_INC, K_DEC with op 0 (PREFIX); space 6 = DIAMOND with op 1 (PASCAL).
cudaError_t launch_ordered(int space, int op, const View* in, const View& out, cudaStream_t s,
                           int64_t* launches);

// Up to 8 device pointers passed by value (peer-memory signalling).
struct PeerPtrs8 {
  void* p[8];
  int n;
};
// atomicAdd_system(flags.p[i], add) for every non-null pointer, after a
// system-scope fence (orders the stream's earlier peer stores / copies).
cudaError_t launch_signal(const PeerPtrs8& flags, unsigned add, cudaStream_t s, int64_t* launches);
// *dst.p[i] = *val for every i, a system fence, then atomicAdd_system(cnt.p[i], 1).
cudaError_t launch_publish(const double* val, const PeerPtrs8& dst, const PeerPtrs8& cnt, cudaStream_t s,
                           int64_t* launches);
// Base and size of the device allocation that contains ptr (cuMemGetAddressRange).
cudaError_t alloc_base(const void* ptr, void** base, size_t* size);

// Make stream s wait until (int32)(*flag - value) >= 0 (cuStreamWaitValue32).
cudaError_t stream_wait_geq(cudaStream_t s, unsigned* flag, unsigned value);

// Convergence bookkeeping of gscl_converge_run: if *conv is clear, record
// iteration `it` in *iters and set *conv when the AND-reduced result is 1.
cudaError_t launch_conv_update(const double* res, int* conv, int* iters, int it, cudaStream_t s,
                               int64_t* launches);

// One iteration's bookkeeping of the device-terminated convergence loop
// (flags: converged, iterations, halt); set_cond: also set the WHILE
// condition `cond` of the enclosing graph to !halt.
cudaError_t launch_conv_step(const double* res, int* flags, int max_iters, unsigned long long cond,
                             int set_cond, cudaStream_t s, int64_t* launches);

// Bookkeeping of one two-sweep pass of the convergence loop (util.cu k_conv_pair).
cudaError_t launch_conv_pair(const double* res1, const double* res2, int* flags, int max_iters, int half,
                             unsigned long long cond, int set_cond, cudaStream_t s, int64_t* launches);

// TMA descriptor encoding (driver entry point resolved at runtime).
bool encode_tma_3d(CUtensorMap* map, const View& v, uint32_t box_x, uint32_t box_y, int l2promo);

// Every translation unit with kernels is its own CUDA module.  Under lazy
// module loading (CUDA_MODULE_LOADING=LAZY, the default) a kernel's first
// launch loads it, and a load may synchronise the context: with the library
// stream parked on a peer's counter (cuStreamWaitValue32) that launch would
// block the host forever, before the multi-rank watchdog could run.  Each
// unit therefore exports an anchor kernel, and preload_modules() loads every
// function of every unit's module up front (gscl_init with world > 1).
#define GSCL_MODULE_ANCHOR(name)                                    \
  namespace {                                                       \
  __global__ void k_module_anchor() {}                              \
  }                                                                 \
  const void* name() { return reinterpret_cast<const void*>(&k_module_anchor); }
const void* anchor_util();
const void* anchor_sweep();
const void* anchor_sweep2r();
const void* anchor_sweep2v();
const void* anchor_ordered();
const void* anchor_sweep2x();
// Load every function of the library's modules; *n = functions loaded.
cudaError_t preload_modules(int* n);

}  // namespace gscl
