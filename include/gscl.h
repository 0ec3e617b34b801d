/*
 * gscl.h — C ABI of the B200-native GSCL hot path (arXiv 1207.1746).
 *
 * The library implements the data-parallel iteration spaces of GSCL
 * (§3): do_all ("does not guarantee any order of application
 * of the stencil operator") and do_reduce (return values
 * "(commutatively) reduced to a single value"), the fused
 * operator of the §5.2 Jacobi loop, the halo exchange that
 * joins z-slab subdomains (the MPI level of PAPER.md:113,180, here NCCL over
 * NVLink), and a device-resident Jacobi driver.
 * Operators are a compiled-in catalogue; grids live in HBM
 * between calls ("keep data on the GPU's memory between invocations",
 * PAPER.md:133).
 *
 * Conventions
 *  - Every entry point returns gscl_status; nothing aborts and no C++
 *    exception crosses this boundary.  gscl_last_error() returns a
 *    thread-local, human-readable message for the most recent failure.
 *  - Extents are GLOBAL.  On a world of P ranks each rank owns a z-slab:
 *    the first (nz mod P) ranks get ceil(nz/P) planes, the rest floor(nz/P)
 *    (SPEC.md:539).  Ranges are half-open boxes in GLOBAL interior
 *    coordinates and are clipped to the caller's slab.
 *  - Layout in HBM (see gscl_grid_layout): element type T (binary64 or
 *    binary32), x fastest, z slowest.  Interior x = 0 sits at element offset
 *    OX = 128 / sizeof(T) inside each row, so every interior row starts on a
 *    128-byte boundary; pitch = round_up(OX + nx + halo, OX) elements; a
 *    plane is pitch * (ny + 2*halo) elements; the local array holds
 *    nz_local + 2*halo planes.  Halo cells hold boundary values (Dirichlet)
 *    and are never written by do_all / do_reduce.
 *  - Asynchrony: gscl_do_all, gscl_halo_exchange, gscl_swap and the fills
 *    are stream-ordered on the library stream and return immediately.
 *    gscl_do_reduce, gscl_jacobi_run, gscl_sync and the host copies block
 *    until their host outputs are valid; asynchronous CUDA errors surface at
 *    those calls as GSCL_E_CUDA.
 *  - One controlling host thread per process.
 */
#ifndef GSCL_H
#define GSCL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gscl_grid_s* gscl_grid_t; /* opaque, library-owned handle */

typedef enum { GSCL_F64 = 0, GSCL_F32 = 1 } gscl_dtype;

typedef enum {
  GSCL_OK = 0,
  GSCL_E_INVALID_ARG = 1,    /* NULL pointer, bad enum, out grid aliases an input */
  GSCL_E_INVALID_DOMAIN = 2, /* extent <= 0, halo < 0 or too wide */
  GSCL_E_SHAPE_MISMATCH = 3, /* grids of one call differ in extents */
  GSCL_E_HALO_VIOLATION = 4, /* a grid's halo is below the op's footprint */
  GSCL_E_ARITY = 5,          /* wrong number of grids for the op */
  GSCL_E_RANGE = 6,          /* range not inside the global interior */
  GSCL_E_DTYPE = 7,          /* grids of one call differ in element type */
  GSCL_E_STATE = 8,          /* call before gscl_init / after gscl_finalize */
  GSCL_E_OOM = 9,
  GSCL_E_CUDA = 10,
  GSCL_E_NCCL = 11,
  GSCL_E_UNSUPPORTED = 12,
  GSCL_E_TIMEOUT = 13        /* multi-rank: a synchronising call waited longer than option
                                "timeout_ms" for its peers (a missing or failed rank); the
                                pending peer waits are released, the NCCL communicator is
                                aborted, and every later call except gscl_finalize returns
                                GSCL_E_STATE */
} gscl_status;

/* do_all catalogue (readings R1-R7).  u(dx,dy,dz) is the
 * neighbour at that offset; every + - * / is one IEEE-754 operation, round to
 * nearest, no contraction.
 *  FIG1B    v = fl(1/36) * ((((((6u - u(+x)) - u(-x)) - u(+y)) - u(-y)) - u(+z)) - u(-z))
 *           PAPER.md:68-71 (Fig 1.b), left to right as printed.  1 input, halo >= 1.
 *  LAP7     L = ((sx + sy) + sz) - 6u,  sx = u(-x)+u(+x), sy, sz likewise.
 *  JACOBI7  v = ((sx + sy) + sz) * fl(1/6).   (PAPER.md:157 Jacobi iteration)
 *  LAP27    L = (B - 128u) / 30 with the z-plane grouped bracket B of R5
 *           (weights (1/30)[-128 centre, 14 face, 3 edge, 1 corner]).
 *  JACOBI27 v = B * 2^-7.
 *  VARCOEF8 v = c0 u + cxm u(-x) + cxp u(+x) + cym u(-y) + cyp u(+y)
 *               + czm u(-z) + czp u(+z), accumulated left to right.
 *           8 inputs: in[0] = u (halo >= 1), in[1..7] = c0,cxm,cxp,cym,cyp,czm,czp
 *           (any halo >= 0).  "real applications ... take 5 to 15 grids at
 *           once". */
typedef enum {
  GSCL_OP_FIG1B = 0,
  GSCL_OP_LAP7 = 1,
  GSCL_OP_JACOBI7 = 2,
  GSCL_OP_LAP27 = 3,
  GSCL_OP_JACOBI27 = 4,
  GSCL_OP_VARCOEF8 = 5
} gscl_op;

/* do_reduce value operators (R8).  grids[0] = a, grids[1] = b.
 *  VALUE a; SQ a*a; ABSDIFF |a-b|; CONV (|a-b| <= eps) ? 1 : 0 (PAPER.md:157,
 *  the infinite-norm test of sten_op_convergence); RESID7_SQ L*L with L = LAP7(a);
 *  RESID27_SQ L*L with L = LAP27(a).
 * Fused operators (PAPER.md:166 fuse(...)) also WRITE out = op(a) in the same
 * scan ("only one scan of the grids is needed"):
 *  JACOBI7_RESID7_SQ   out = JACOBI7(a),  value = RESID7_SQ(a)
 *  JACOBI27_RESID27_SQ out = JACOBI27(a), value = RESID27_SQ(a)
 *  FIG1B_CONV          out = FIG1B(a),    value = CONV(eps)(out, a)
 * eps = params[0] for CONV and FIG1B_CONV (fp32 grids compare in binary32). */
typedef enum {
  GSCL_R_VALUE = 0,
  GSCL_R_SQ = 1,
  GSCL_R_ABSDIFF = 2,
  GSCL_R_CONV = 3,
  GSCL_R_RESID7_SQ = 4,
  GSCL_R_RESID27_SQ = 5,
  GSCL_R_JACOBI7_RESID7_SQ = 6,
  GSCL_R_JACOBI27_RESID27_SQ = 7,
  GSCL_R_FIG1B_CONV = 8
} gscl_rop;

/* Combines: SUM (identity +0), MAX (-inf), MIN (+inf), AND (1; values are
 * 0/1).  Values are widened to binary64 before combining. */
typedef enum { GSCL_SUM = 0, GSCL_MAX = 1, GSCL_MIN = 2, GSCL_AND = 3 } gscl_combine;

/* Half-open box [x0,x1) x [y0,y1) x [z0,z1) in GLOBAL interior coordinates. */
typedef struct {
  int64_t x0, x1, y0, y1, z0, z1;
} gscl_range;

/* ---------------------------------------------------------------- context */

/* Writes a fresh 128-byte NCCL unique id into out128 (rank 0 calls this and
 * broadcasts the bytes, e.g. with torch.distributed).  Does not need a GPU
 * context; returns GSCL_E_NCCL on failure. */
gscl_status gscl_get_nccl_unique_id(void* out128);

/* Initialise the library for this process: rank in [0, world), the CUDA
 * device ordinal, and the CUDA stream all work is issued on (a cudaStream_t,
 * e.g. torch.cuda.current_stream().cuda_stream; NULL = the legacy default
 * stream, which is what torch reports for its default stream).  Memory the
 * caller fills or frees for wrapped grids must be ordered on this stream.
 * nccl_id: the 128 bytes from gscl_get_nccl_unique_id (ignored when world ==
 * 1); NULL with world > 1 creates no communicator — after gscl_peer_export /
 * import, gscl_jacobi_run and the cross-rank combine of gscl_do_reduce then
 * run over peer memory; gscl_halo_exchange returns GSCL_E_STATE.  Calling init twice without finalize
 * returns GSCL_E_STATE. */
gscl_status gscl_init(int rank, int world, const void* nccl_id, int device, void* cuda_stream);

/* Release NCCL/CUDA resources owned by the library (grids still alive are
 * destroyed).  Afterwards every call except gscl_init returns GSCL_E_STATE. */
gscl_status gscl_finalize(void);

/* Wait for all library work on this rank; reports asynchronous errors. */
gscl_status gscl_sync(void);

/* Thread-local message for the last non-OK status ("" if none). */
const char* gscl_last_error(void);

/* The library's version string and build flags. */
const char* gscl_version(void);

/* ---------------------------------------------------------------- grids */

/* Allocate a grid of GLOBAL interior extents nx, ny, nz with halo width
 * `halo` (0..16 for f64, 0..32 for f32) on every side.  This rank allocates
 * its z-slab (plus halo planes).  Memory is zero-filled.  *out receives the
 * handle (library-owned; release with gscl_grid_destroy). */
gscl_status gscl_grid_create(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype,
                             gscl_grid_t* out);

/* Wrap caller-owned device memory (e.g. a torch tensor) laid out exactly as
 * gscl_grid_layout describes; `bytes` must be at least the slab size and
 * dev_ptr 256-byte aligned.  The library never frees it. */
gscl_status gscl_grid_wrap(void* dev_ptr, size_t bytes, int64_t nx, int64_t ny, int64_t nz,
                           int halo, gscl_dtype dtype, gscl_grid_t* out);

gscl_status gscl_grid_destroy(gscl_grid_t g);

/* Bytes a grid of these extents needs on `rank` of `world` (no GPU needed). */
gscl_status gscl_grid_bytes(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype,
                            int rank, int world, size_t* bytes);

/* Layout of the local slab: pitch (elements per row), this rank's global
 * z range [z_begin, z_end), and the element offset of interior (0,0,z_begin)
 * from the start of the allocation.  Any output pointer may be NULL. */
gscl_status gscl_grid_layout(gscl_grid_t g, int64_t* pitch, int64_t* z_begin, int64_t* z_end,
                             int64_t* origin_offset_elems);

/* Device pointer of the allocation (for wrapping as a tensor in tests). */
gscl_status gscl_grid_device_ptr(gscl_grid_t g, void** dev_ptr);

/* Balanced z-slab of `rank` among `world` ranks; no GPU needed. */
gscl_status gscl_slab_range(int64_t nz, int rank, int world, int64_t* z_begin, int64_t* z_end);

/* Fill the interior with the counter-based generator of DESIGN.md R9:
 * value = U[0,1)(splitmix64(seed ^ (grid_id << 48) ^ gidx)) * scale with
 * gidx = (z*ny + y)*nx + x over GLOBAL coordinates; halo cells are zeroed. */
gscl_status gscl_grid_fill_random(gscl_grid_t g, uint64_t seed, uint32_t grid_id, double scale);

/* Fill every cell (interior and halo) with one value. */
gscl_status gscl_grid_fill_const(gscl_grid_t g, double value);

/* Copy the local slab to / from host memory in the DENSE layout
 * [(nz_local+2h)][(ny+2h)][(nx+2h)] (x fastest), halo included.
 * `bytes` must equal that size.  Host memory may be pageable or pinned;
 * both calls are synchronous. */
gscl_status gscl_grid_copy_to_host(gscl_grid_t g, void* host, size_t bytes);
gscl_status gscl_grid_copy_from_host(gscl_grid_t g, const void* host, size_t bytes);

/* Asynchronous upload of the dense slab (same layout and size rule as
 * gscl_grid_copy_from_host): a contiguous host->device copy into one of two
 * device staging slots and an on-device repack, both on the library's copy
 * stream, so consecutive uploads and library work on OTHER grids overlap.
 * Returns at once; the next library call that uses `g` (any entry point taking
 * it) orders itself after the upload.  `host` must stay valid and unmodified
 * until then; pinned memory makes the copy truly asynchronous. */
gscl_status gscl_grid_copy_from_host_async(gscl_grid_t g, const void* host, size_t bytes);

/* Asynchronous download of the dense slab (same layout and size rule as
 * gscl_grid_copy_to_host): an on-device repack of the grid's current contents
 * (everything the library stream has written before the call) into one of
 * two device staging slots and a contiguous device->host copy, both on the
 * library's download stream, so the download of one result overlaps library
 * work on other grids and uploads on the copy stream (PCIe is full duplex).
 * Returns at once; later library calls that use `g` order themselves after
 * the repack has read it; the host buffer holds the data after the next
 * gscl_sync.  `host` must be pinned for the copy to be asynchronous. */
gscl_status gscl_grid_copy_to_host_async(gscl_grid_t g, void* host, size_t bytes);

/* Order-independent 64-bit digest of the GLOBAL interior (R10),
 * identical on every rank: sum over cells of
 * splitmix64(bits(value) ^ splitmix64(gidx)) mod 2^64.  Synchronous. */
gscl_status gscl_grid_digest(gscl_grid_t g, uint64_t* out);

/* Exchange the storage of two grids of identical shape in O(1)
 * (swap_grids(); halos travel with the storage). */
gscl_status gscl_swap(gscl_grid_t a, gscl_grid_t b);

/* ---------------------------------------------------------------- iteration spaces */

/* do_all: out(p) = op(in[0..n_in-1])(p) for every interior p in `range`
 * (NULL = the whole interior).  in[] grids are read-only, out is write-only
 * (the access list of PAPER.md:63); out must not alias any input.  Reads at
 * z-offsets use the halo planes as they are: call gscl_halo_exchange first
 * on a multi-rank run.  params unused (may be NULL). */
gscl_status gscl_do_all(gscl_op op, const gscl_grid_t* in, int n_in, gscl_grid_t out,
                        const gscl_range* range, const double* params, int n_params);

/* do_reduce: *result = combine over p in range of rop(grids)(p), the global
 * result on every rank.  Fused rops also write `out` (must be non-NULL for
 * them and NULL otherwise).  SUM order is fixed for a given launch
 * configuration (deterministic), not the oracle's order. */
gscl_status gscl_do_reduce(gscl_rop rop, const gscl_grid_t* grids, int n, gscl_grid_t out,
                           gscl_combine combine, const gscl_range* range, const double* params,
                           int n_params, double* result);

/* Exchange z-halo planes of each grid with the neighbouring ranks (whole
 * padded planes; physical-boundary halos are untouched).  No-op on world 1.
 * Issued as one NCCL group per grid on the library stream; the transfers are
 * exactly the ops gscl_halo_plan lists. */
gscl_status gscl_halo_exchange(const gscl_grid_t* grids, int n);

/* The halo exchange at a given depth ("wide ghost areas"; the
 * exchange step of gscl_jacobi_run's multi-rank schedules, callable alone so
 * its cost can be timed apart from the sweeps — SURVEY §8(d).1).
 * depth 1: the planes gscl_halo_exchange moves (h per side).  depth 2: the
 * exchange that precedes a two-sweep pass (gscl_pass_plan: the first / last
 * two interior planes per side; with halo 1 the second received plane lands
 * in the library's ghost buffer).  Transport: option "transport" 0 = NCCL
 * grouped send/recv on the library stream; 1 = peer memory (n must be 1 and
 * the grid one of the pair given to gscl_peer_export): a ready handshake with
 * the neighbours (their earlier work on the grid is done), then both boundary
 * planes are copied into the neighbours' receiving planes over the IPC
 * mappings, the neighbours are signalled, and the stream waits for their
 * signals (stream-ordered).  Asynchronous; no-op on world 1. */
gscl_status gscl_halo_exchange_depth(const gscl_grid_t* grids, int n, int depth);

/* One two-sweep pass (temporal blocking) of JACOBI7 over the
 * local interior of `in` into `out`: out = OP(OP(in)) with the intermediate
 * iterate u1 = OP(in) on interior points and u1 = in on halo points (the
 * Dirichlet rule of gscl_jacobi_run) — except that on a z side with
 * phys_lo / phys_hi = 0 (a neighbour's slab, not the domain boundary) u1 IS
 * computed on the halo plane -1 / nzl, from the neighbour's planes the caller
 * has placed in in's halo plane and, when in's halo is 1, in `ghost`: a
 * device buffer of 2 planes in in's plane layout (pitch x (ny + 2h) elements
 * each) holding plane -2 (first) and nzl + 1 (second); NULL when both sides
 * are physical or halo >= 2.  This is the kernel gscl_jacobi_run uses on
 * several ranks, exposed so a caller can drive its own transport.  Stream-
 * ordered; `out`'s halo is not written.  UNSUPPORTED for ops other than
 * JACOBI7; SHAPE_MISMATCH / DTYPE / INVALID_ARG (aliasing, missing ghost).
 *
 * peer (may be NULL): the peer-memory halo transport — the pass ALSO stores
 * its output planes 0 and 1 into lo[0] / lo[1] (the lower neighbour's planes
 * nzl, nzl+1 of ITS output grid: the halo plane and, for halo 1, its ghost
 * plane) and planes nzl-1, nzl-2 into hi[0] / hi[1] (the upper neighbour's
 * planes -1, -2), from the same registers as the local stores, tile by tile;
 * each pointer is the interior origin (x = 0, y = 0) of such a plane in the
 * same plane layout (device memory of this GPU, a peer GPU over NVLink, or an
 * IPC mapping); NULL skips it.  The launch's boundary units (2-plane z-chunks
 * at each end, scheduled first) bump *lo_flag / *hi_flag (system-scope
 * atomics, after a system fence) once their planes are stored: gscl_pass_units
 * of them per side per pass.  The x/y halo ring of a receiving plane is not
 * written (it holds boundary values that never change). */
typedef struct {
  void* lo[2];
  void* hi[2];
  unsigned* lo_flag;
  unsigned* hi_flag;
} gscl_pass_peer;
gscl_status gscl_do_all_pass2(gscl_op op, gscl_grid_t in, gscl_grid_t out, const void* ghost, int phys_lo,
                              int phys_hi, const gscl_pass_peer* peer);

/* The same pass for JACOBI7 (n_coeffs 0) or VARCOEF8 (coeffs = the 7
 * coefficient grids, halo 0, same extents; "5 to 15 grids at
 * once").  For VARCOEF8 on a non-physical z side u1 on the halo plane also
 * needs the coefficients of planes -1 / nzl, which the coefficient grids do
 * not hold: cghost is a device buffer of 14 planes in the coefficient grids'
 * plane layout, plane 2c = grid c's plane -1 and 2c + 1 = its plane nzl (the
 * neighbours' boundary planes); NULL when both z sides are physical.  Errors
 * as gscl_do_all_pass2, plus ARITY for a wrong n_coeffs. */
gscl_status gscl_do_all_pass2_coeffs(gscl_op op, gscl_grid_t in, const gscl_grid_t* coeffs, int n_coeffs,
                                     gscl_grid_t out, const void* ghost, const void* cghost, int phys_lo,
                                     int phys_hi, const gscl_pass_peer* peer);

/* Boundary units per side of a boundary-first two-sweep pass over a slab of
 * these extents (what a neighbour's arrival counter grows by per pass):
 * gscl_pass_units for JACOBI7, gscl_pass_units_op for JACOBI7 or VARCOEF8. */
gscl_status gscl_pass_units(int64_t nx, int64_t ny, gscl_dtype dtype, int64_t* units);
gscl_status gscl_pass_units_op(gscl_op op, int64_t nx, int64_t ny, gscl_dtype dtype, int64_t* units);

/* One transfer of the halo exchange: send (is_send = 1) or receive `bytes`
 * contiguous bytes at byte `offset` of this rank's slab allocation to / from
 * rank `peer`. */
typedef struct {
  int peer;
  int is_send;
  int64_t offset;
  int64_t bytes;
} gscl_halo_op;

/* The exchange plan of `rank` for a grid of these GLOBAL extents (no GPU
 * needed): at most 4 ops, written to ops[0..*n_ops).  Interior ranks send
 * their first/last h interior planes and receive into their h ghost planes
 * on each side; ranks 0 and world-1 skip their physical boundary. */
gscl_status gscl_halo_plan(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype,
                           int rank, int world, gscl_halo_op* ops, int* n_ops);

/* One plane of the depth-2 exchange that precedes a two-sweep pass of
 * gscl_jacobi_run on several ranks (temporal blocking; "wide
 * ghost areas"): send (is_send = 1) or receive local plane z
 * (local interior coordinates, -2 <= z <= nzl + 1) to / from rank `peer`.
 * ghost_plane = 0: the plane is in the grid (interior or halo); 1 / 2: it is
 * beyond the grid's halo (h = 1) and lives in the library's ghost buffer,
 * plane 0 (below) / 1 (above). */
typedef struct {
  int peer;
  int is_send;
  int64_t z;
  int ghost_plane;
} gscl_pass_xfer;

/* The depth-2 exchange plan of `rank` (no GPU needed): at most 8 transfers,
 * one plane each, written to ops[0..*n_ops).  Per neighbour the sends are the
 * two boundary planes nearest-first and the receives fill planes -1, -2
 * (below) / nzl, nzl+1 (above) nearest-first, so NCCL matches them in order.
 * Physical boundaries (rank 0 below, world-1 above) exchange nothing. */
gscl_status gscl_pass_plan(int64_t nx, int64_t ny, int64_t nz, int halo, gscl_dtype dtype,
                           int rank, int world, gscl_pass_xfer* ops, int* n_ops);

/* Jacobi driver (PAPER.md:157-170 with a fixed iteration count, DESIGN.md
 * R11): op in {JACOBI7, JACOBI27, VARCOEF8}; coeffs = the 7 coefficient grids
 * for VARCOEF8 (else NULL / 0).  Copies u's halo shell into v, then for
 * it = 1..iters: [halo exchange of the input]; sweep (fused with the check
 * value of its INPUT when check_every > 0 and it % check_every == 0; the
 * check is RESID7_SQ / RESID27_SQ / SQ for JACOBI7 / JACOBI27 / VARCOEF8);
 * swap.  history (iters/check_every + 1 doubles, or NULL; needed when
 * check_every > 0) receives sqrt(global sum) of each check and, last, of a
 * standalone pass over the final iterate.  On return u holds the final
 * iterate (handles are swapped as needed); v holds an earlier iterate (the
 * one before, or two before when sweeps were fused in pairs). */
gscl_status gscl_jacobi_run(gscl_op op, gscl_grid_t u, gscl_grid_t v, const gscl_grid_t* coeffs,
                            int n_coeffs, int iters, int check_every, double* history);

/* The paper's convergence-terminated fused loop (§5.2):
 *   do { swap_grids(); res = do_reduce(ctx, now, before,
 *          fuse(sten_op_diffusion(), sten_op_convergence(EPSI)), logical_and) }
 *   while (!res);
 * op in {FIG1B (the paper's operator), JACOBI7}.  Copies u's halo shell into v,
 * then iteration it = 1, 2, ... computes out = op(in) in one pass fused with
 * res = AND over the interior of (|out - in| <= eps), the global AND on every
 * rank, and stops after the first iteration with res = 1 or after max_iters.
 * Device-resident.  One rank: the loop is ONE launch of a CUDA graph with a
 * conditional WHILE node (two iterations per body; a device flag sets the
 * condition), so the host synchronises once; `batch` is unused.  Several
 * ranks (or option graph = 2): once converged, the remaining kernels of a
 * batch return immediately and the host reads the flag every `batch`
 * iterations (0 = 16).
 * On return u holds the final iterate, *iters_done the iterations executed
 * (including the converging one) and *converged whether res became 1. */
gscl_status gscl_converge_run(gscl_op op, gscl_grid_t u, gscl_grid_t v, double eps, int max_iters,
                              int batch, int* iters_done, int* converged);

/* Red-black Gauss-Seidel for the 7-point Laplace equation (NEXT-3; the paper's
 * "stateful" stencil shapes are "useful ... for implementing red-black
 * Gauss-Siedel").  In place on u (halo >= 1, Dirichlet halo
 * values): iteration = red half-sweep then black, a half-sweep setting
 * u(p) = JACOBI7(u)(p) at the interior points with (x + y + z) mod 2 = colour
 * (global coordinates; red = 0).  history as gscl_jacobi_run (RESID7 of the
 * iterate before iteration it when it % check_every == 0, then of the final
 * iterate).  One rank (default): each iteration is ONE two-sweep pass (red,
 * then black from the red-updated field), out of place between u and a
 * library buffer, the result copied back into u after an odd count; option
 * tblock = 1 or several ranks: two in-place half-sweeps, the z ghost planes
 * exchanged before every half-sweep.  Same results either way. */
gscl_status gscl_rbgs_run(gscl_grid_t u, int iters, int check_every, double* history);

/* Ordered iteration spaces (NEXT-4; §3): do_i_inc, do_j_inc,
 * do_k_inc process cell (i-1,j,k), (i,j-1,k), (i,j,k-1) before (i,j,k) (the
 * paper's "(i,j-1,j)" read as (i,j-1,k)); the _dec spaces the +1 cells;
 * do_diamond processes (i-1,j) and (i,j-1) before (i,j) ("available only for
 * 2D": applied to every z plane). */
typedef enum {
  GSCL_DO_I_INC = 0,
  GSCL_DO_I_DEC = 1,
  GSCL_DO_J_INC = 2,
  GSCL_DO_J_DEC = 3,
  GSCL_DO_K_INC = 4,
  GSCL_DO_K_DEC = 5,
  GSCL_DO_DIAMOND = 6
} gscl_space;

/* Ordered operators: PREFIX out(p) = out(p - d) + in(p) along the space's axis
 * (d = the predecessor offset; a running sum / suffix sum); PASCAL (diamond
 * only) out(i,j) = out(i-1,j) + out(i,j-1).  The halo of `out` supplies the
 * values before the first cell (boundary values). */
typedef enum { GSCL_O_PREFIX = 0, GSCL_O_PASCAL = 1 } gscl_oop;

/* Apply `op` over the interior of `out` in the order of `space`.  in: same
 * extents as out (PREFIX) or NULL (PASCAL); out: halo >= 1, must not alias in.
 * Results equal the sequential recurrence bit for bit.  The k spaces cross
 * ranks in order (rank r receives the plane before its first from its
 * predecessor); the others stay inside each slab.  Stream-ordered. */
gscl_status gscl_do_ordered(gscl_space space, gscl_oop op, gscl_grid_t in, gscl_grid_t out);

/* ---------------------------------------------------------------- measurement */

/* Kernel-level instrumentation: when on, the library brackets every sweep
 * kernel it launches with CUDA events on its stream — except that a run of
 * consecutive two-sweep passes inside one single-rank gscl_jacobi_run gets
 * ONE pair of events around the whole run, booked as that many launches of
 * kind 3 (events between the passes would add their own gaps to the step;
 * the run's time includes the few-microsecond launch gaps between its
 * passes, so the per-pass average is conservative).  gscl_timing_read
 * returns (and clears) per sweep kind k the summed device milliseconds ms[k]
 * and launch count n[k] — k = 0: do_all sweep (write only), 1: fused sweep
 * (write + reduce), 2: stencil reduce-only pass, 3: two-sweep pass — and
 * *launches, the number of kernels the library launched since the last read
 * (sweeps, reductions, copies, fills, folds).  ms and n point to 4 elements
 * each (may be NULL). */
gscl_status gscl_timing_enable(int on);
gscl_status gscl_timing_read(double* ms, int64_t* n, int64_t* launches);

/* Peer-memory halo transport for gscl_jacobi_run on several ranks (option
 * "transport" = 1): the sweep kernels (the two-sweep pass for
 * JACOBI7, the single sweep for JACOBI27 / VARCOEF8) store their
 * boundary planes directly into the neighbours' halo / ghost planes through
 * CUDA IPC mappings (NVLink peer memory on a multi-GPU node) and signals
 * arrival counters; no NCCL call on the halo path.  Collective setup, once per
 * (u, v) pair: every rank calls gscl_peer_export (blob == NULL: *bytes = the
 * blob size), the caller all-gathers the blobs in rank order (any channel —
 * torch.distributed, MPI, NCCL), then every rank calls gscl_peer_import with
 * the world * bytes array.  u / v may later be swapped by jacobi_run (the
 * storages are tracked).  Grids must live in cudaMalloc'd memory (the torch
 * caching allocator's default); up to 8 ranks.  gscl_init may be given a NULL
 * nccl_id when world > 1: then only this transport works across ranks
 * (NCCL-based calls return GSCL_E_STATE). */
gscl_status gscl_peer_export(gscl_grid_t u, gscl_grid_t v, void* blob, size_t cap, size_t* bytes);
gscl_status gscl_peer_import(gscl_grid_t u, gscl_grid_t v, const void* blobs, size_t bytes_each);

/* Tuning / ablation knobs, process-wide:
 *  "sweep_impl" 0 = TMA ring (default), 1 = plain per-point kernel, 2 = 3-D
 *               blocked kernel without z streaming (7-point do_all; ablations);
 *  "zchunks"    z chunks per tile column, 0 = auto;
 *  "sched"      0 = auto, 1 = multi-wave (chunks all stream up),
 *               2 = single wave with alternating chunk direction;
 *  "l2promo"    TMA L2 promotion 0 = none (default), 1 = 64B, 2 = 128B, 3 = 256B;
 *  "stages"     TMA ring depth of the 7-point fp64 sweeps: 0 = default (8
 *               for reduction sweeps, else 4), 4, 8 (fp64 27-point sweeps
 *               always use 8);
 *  "tblock"     sweeps per HBM pass in jacobi_run: 0 = auto (default: pairs of
 *               JACOBI7 or VARCOEF8 sweeps fused into one two-sweep pass on a
 *               single rank — temporal blocking, results unchanged), 1 = one
 *               sweep per pass, 2 = pairs (JACOBI7, VARCOEF8, and JACOBI27 —
 *               measured slower, profiles/r01_sweep2k.md; single rank);
 *  "zalt"       1 = jacobi_run walks the z chunks of consecutive sweeps in
 *               alternating order (meant for L2 reuse; measured slower), 0 = off;
 *  "graph"      jacobi_run as one CUDA graph per (grids, shape, schedule,
 *               options): 0 = auto (grids of <= 2^24 local points, timing
 *               off), 1 = always, 2 = never;
 *  "variant"    kernel geometry (ablation): two-sweep pass 0 = register-
 *               resident u1 (sweep2r.cu, 7 warps x 4 rows), 11 / 12 / 14 / 15
 *               = its other geometries (8 x 2 rows; 2 CTAs of 3 x 4; 8-stage
 *               ring; 8 x 4 rows + a setmaxnreg producer warpgroup),
 *               1..4 = the shared-memory-u1 kernel (sweep2.cu); VARCOEF8
 *               pass (sweep2v.cu): 11 = 4-stage ring, 12 = 12 warps,
 *               14 = 2 CTAs of 4 warps; JACOBI27 pass (sweep2k.cu): 11 / 12 =
 *               1 / 3 rows per lane, 14 = 2 CTAs of 4 warps, 15 = 4-stage
 *               ring, 16 = 2 points per lane;
 *               single sweeps: 1 = shuffled x neighbours, 2 = 27-point R = 2,
 *               3 = fp64 27-point at 3 CTAs/SM, 4 = fp64 7-point at 2
 *               CTAs/SM, 5 = fp64 27-point with a 4-stage ring;
 *  "transport"  multi-rank jacobi_run halo transport: 0 = NCCL (default),
 *               1 = peer memory (after gscl_peer_export / gscl_peer_import);
 *  "timeout_ms" multi-rank watchdog (world > 1): the longest a synchronising
 *               call (jacobi_run, converge_run, rbgs_run, do_reduce, sync, the
 *               host copies, digest) waits for the library stream before it
 *               gives up with GSCL_E_TIMEOUT; 0 = the default, 120000;
 *  "halo_off"   TIMING ONLY (results are wrong on several ranks): jacobi_run's
 *               multi-rank schedule runs with every halo exchange skipped —
 *               the compute-only step that the exposed halo time (overlapped
 *               step minus compute-only step) is measured
 *               against; 0 = off (default);
 *  "split"      1 = run jacobi_run's overlapped multi-rank schedule (boundary
 *               planes first, exchange on a comm stream, interior overlapped)
 *               also on a single rank (testing); multi-rank always uses it.
 * Unknown names return GSCL_E_UNSUPPORTED; no option changes results. */
gscl_status gscl_set_option(const char* name, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* GSCL_H */
