// sweep2.cu — two Jacobi sweeps per HBM pass (temporal blocking, SURVEY §8(f)
// NEXT-2; "wide ghost areas").
//
// out = OP(OP(u)) for JACOBI7 / JACOBI27 with the Dirichlet halo of
// gscl_jacobi_run (halo cells are boundary values and are never updated, so
// the intermediate iterate u1 equals u on the halo).  Both sweeps evaluate the
// per-point trees of ops.cuh, so the result is bitwise the result of two
// single sweeps.
//
// Tile geometry (fp64, V = 2): a CTA outputs a 60 x 14 tile (lanes 1..30 x
// rows 1..14 of the warps' bands); the intermediate u1 is computed on the
// 62 x 16 ring around it (lanes 0..31 x 2 rows per warp, 8 warps), and the
// input u is staged by TMA as a 64 x 18 box per plane (2 extra on each side).
// Per input plane:
//   1. wait for the TMA stage, build sweep-1 tuples of u at my 2 x 2 points,
//      release the stage (fence.proxy.async + mbarrier arrive);
//   2. when three tuples are available, u1(z-1) = OP(...) (or the halo value
//      u(z-1) outside the interior) is written to a 3-plane u1 ring in shared
//      memory; a named barrier makes the plane visible to all warps;
//   3. build sweep-2 tuples of u1(z-1) from the ring and, when three are
//      available, out(z-2) = OP(...) is stored (16-byte st.global).
// A chunk of output planes [zs, ze) needs u1 on [zs-1, ze] and u on
// [zs-2, ze+1]: np = (ze - zs) + 4 input planes.
#include <algorithm>
#include <type_traits>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

#ifdef GSCL_ABLATIONS  // the first two-sweep design: an ablation, not in the product library
namespace {

constexpr int kR = 2;          // u1 rows per lane
constexpr int kS = 6;          // input ring stages
constexpr int kHeader = 1024;  // barriers + reduction scratch

template <typename T, int kNW> struct Geo2 {
  static constexpr int V = Vec<T>::N;
  static constexpr int W = 32 * V;              // u1 strip width = input box width
  static constexpr int TXO = W - 2 * V;         // output tile width (lanes 1..30)
  static constexpr int U1ROWS = kNW * kR;       // 16
  static constexpr int TYO = U1ROWS - 2;        // 14 output rows
  static constexpr int INROWS = U1ROWS + 2;     // 18 input rows
  static constexpr int INBYTES = INROWS * W * (int)sizeof(T);
  static constexpr int INBYTES_AL = (INBYTES + 127) / 128 * 128;
  static constexpr int U1BYTES = U1ROWS * W * (int)sizeof(T);
  static constexpr int U1BYTES_AL = (U1BYTES + 127) / 128 * 128;
  // + 128: with smem x neighbours lane 31 reads one element past the last u1 row
  static constexpr int SMEM = kHeader + kS * INBYTES_AL + 3 * U1BYTES_AL + 128;
};

template <typename T> struct Sweep2Args {
  T* out;
  int64_t osy, osz;
  int nx, ny, nz;          // local interior extents (u1 halo rule)
  int tiles_x, tiles_y, chunk, nzr;
  int col0, row0, pln0;    // array coords of interior (0,0,0) of u
  double* partials;
  unsigned* counter;
  double* result;
};

// In-plane neighbourhood of point (j, k) of a lane from rows cv[0..kR+1] and
// x neighbours xl/xr (kR+2 rows) — the same construction as sweep_tma.
template <typename T, int OP>
__device__ __forceinline__ typename OpT<OP, T>::Tup tuple_at(const T (&cv)[kR + 2][Vec<T>::N],
                                                             const T (&h)[kR + 2][Vec<T>::N],
                                                             const T (&xl)[kR + 2], const T (&xr)[kR + 2],
                                                             int j, int k) {
  constexpr int V = Vec<T>::N;
  Nbr<T> n;
  n.c = cv[j + 1][k];
  n.xm = k > 0 ? cv[j + 1][k - 1] : xl[j + 1];
  n.xp = k < V - 1 ? cv[j + 1][k + 1] : xr[j + 1];
  n.ym = cv[j][k];
  n.yp = cv[j + 2][k];
  n.h0 = h[j + 1][k];
  if constexpr (OpT<OP, T>::DIAG) {
    n.hm = h[j][k];
    n.hp = h[j + 2][k];
  }
  T cf[1] = {T(0)};
  return OpT<OP, T>::plane(n, cf);
}

// Build the tuples of my kR x V points from a W-wide smem plane whose row 0 is
// the row above my first point (rows rbase .. rbase+kR+1).
template <typename T, int OP, int XS>
__device__ __forceinline__ void plane_tuples(const T* P, int rbase, int lane,
                                             typename OpT<OP, T>::Tup (&t)[kR][Vec<T>::N]) {
  constexpr int V = Vec<T>::N;
  constexpr int W = 32 * V;
  using O = OpT<OP, T>;
  T cv[kR + 2][V];
#pragma unroll
  for (int r = 0; r < kR + 2; ++r) vload<T>(P + (rbase + r) * W + V * lane, cv[r]);
  // x neighbours from the adjacent lanes (warp shuffles, no shared-memory
  // traffic); lanes 0 / 31 get their own values, and the points that would need
  // the true neighbour (x = xt0 - V, x = xt0 + 31V - 1) are never used
  T xl[kR + 2], xr[kR + 2];
#pragma unroll
  for (int r = 0; r < kR + 2; ++r) {
    if (O::DIAG || (r >= 1 && r <= kR)) {
      if constexpr (XS == 1) {
        xl[r] = __shfl_up_sync(0xffffffffu, cv[r][V - 1], 1);
        xr[r] = __shfl_down_sync(0xffffffffu, cv[r][0], 1);
      } else {  // lanes 0 / 31 read one element outside the strip (inside shared memory)
        xl[r] = P[(rbase + r) * W + V * lane - 1];
        xr[r] = P[(rbase + r) * W + V * lane + V];
      }
    } else {
      xl[r] = T(0);
      xr[r] = T(0);
    }
  }
  T h[kR + 2][V];
#pragma unroll
  for (int r = 0; r < kR + 2; ++r)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (O::DIAG || (r >= 1 && r <= kR))
        h[r][k] = add(k > 0 ? cv[r][k - 1] : xl[r], k < V - 1 ? cv[r][k + 1] : xr[r]);
#pragma unroll
  for (int j = 0; j < kR; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) t[j][k] = tuple_at<T, OP>(cv, h, xl, xr, j, k);
}

template <int OP, int RV, typename T, int XS, int MINB, int kNW>
__global__ void __launch_bounds__(32 * (kNW + 1), MINB)
    sweep2_tma(const __grid_constant__ Sweep2Args<T> a, const __grid_constant__ CUtensorMap map) {
  using G = Geo2<T, kNW>;
  using O = OpT<OP, T>;
  using Tup = typename O::Tup;
  constexpr int V = G::V;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kS;
  double* red = reinterpret_cast<double*>(empty + kS);
  int* flag = reinterpret_cast<int*>(red + kNW);
  unsigned char* in_stages = smem + kHeader;
  T* u1ring = reinterpret_cast<T*>(smem + kHeader + kS * G::INBYTES_AL);
  constexpr int U1P = G::U1BYTES_AL / (int)sizeof(T);  // elements per u1 plane slot

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int unit = blockIdx.x;
  const int tx = unit % a.tiles_x;
  unit /= a.tiles_x;
  const int ty = unit % a.tiles_y;
  const int zc = unit / a.tiles_y;
  const int xt0 = tx * G::TXO;           // first output x of the tile
  const int yt0 = ty * G::TYO;           // first output y of the tile
  const int zs = zc * a.chunk;
  const int ze = min(zs + a.chunk, a.nzr);
  const int np = ze - zs + 4;            // input planes zs-2 .. ze+1

  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kNW) {  // ---------------- producer
    if (lane == 0) {
      tma_prefetch_desc(&map);
      int s = 0;
      uint32_t ph = 0;
      for (int p = 0; p < np; ++p) {
        if (p >= kS) mbar_wait(&empty[s], ph ^ 1);
        const int z = zs - 2 + p;
        mbar_arrive_expect_tx(&full[s], G::INBYTES);
        tma_load_3d(in_stages + s * G::INBYTES_AL, &map, a.col0 + xt0 - V, a.row0 + yt0 - 2,
                    a.pln0 + z, &full[s]);
        if (++s == kS) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumers: lane l owns strip columns V*l .. V*l+V-1
  // (x = xt0 - V + V*l + k), warp w owns u1 rows 2w, 2w+1 (y = yt0 - 1 + 2w + j).
  const int rbase = warp * kR;
  const int xs = xt0 - V + V * lane;  // x of my first point
  const int ys = yt0 - 1 + rbase;     // y of my first u1 row
  // u1 rule: interior points get OP, halo points keep u (never updated)
  bool interior_xy[kR][V];
#pragma unroll
  for (int j = 0; j < kR; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k)
      interior_xy[j][k] = xs + k >= 0 && xs + k < a.nx && ys + j >= 0 && ys + j < a.ny;
  // output: lanes 1..30, u1 rows 1..14 of the 16, inside the grid
  bool ok[kR][V];
#pragma unroll
  for (int j = 0; j < kR; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k)
      ok[j][k] = lane >= 1 && lane <= 30 && rbase + j >= 1 && rbase + j <= G::TYO &&
                 xs + k < a.nx && ys + j < a.ny;
  const bool fast = lane >= 1 && lane <= 30 && rbase >= 1 && rbase + kR - 1 <= G::TYO &&
                    xs + V <= a.nx && ys + kR <= a.ny;
  T* optr = a.out + (int64_t)ys * a.osy + xs + (int64_t)zs * a.osz;
  int64_t roff[kR];
#pragma unroll
  for (int j = 0; j < kR; ++j) roff[j] = (int64_t)j * a.osy;
  double acc[kR][V];
#pragma unroll
  for (int j = 0; j < kR; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) acc[j][k] = 0.0;

  int s = 0;
  uint32_t ph = 0;
  // sweep-1 tuples of input planes (3-set rotation), sweep-2 tuples of u1 planes
  auto load_in = [&](Tup (&t)[kR][V]) {
    mbar_wait(&full[s], ph);
    // input box row 0 is y = yt0 - 2: my u1 rows need input rows rbase .. rbase+3
    plane_tuples<T, OP, XS>(reinterpret_cast<const T*>(in_stages + s * G::INBYTES_AL), rbase, lane, t);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == kS) {
      s = 0;
      ph ^= 1;
    }
  };
  // u1 at plane z (from input tuples of z-1, z, z+1) -> ring slot z % 3
  T own[kR][V];  // my u1 rows of the plane just made (kept for its sweep-2 tuples)
  auto make_u1 = [&](const Tup (&lo)[kR][V], const Tup (&mid)[kR][V], const Tup (&hi)[kR][V], int z) {
    T* P = u1ring + ((z + 3) % 3) * U1P;
    const bool zin = z >= 0 && z < a.nz;
#pragma unroll
    for (int j = 0; j < kR; ++j) {
#pragma unroll
      for (int k = 0; k < V; ++k)
        own[j][k] = (zin && interior_xy[j][k]) ? O::out(lo[j][k], mid[j][k], hi[j][k]) : mid[j][k].c;
      vstore<T>(P + (rbase + j) * G::W + V * lane, own[j]);
    }
  };
  // sweep-2 tuples of u1 plane z; needs all warps' rows of that plane
  auto load_u1 = [&](Tup (&t)[kR][V], int z) {
    named_bar_sync(1, kNW * 32);
    const T* P = u1ring + ((z + 3) % 3) * U1P;
    // rows rbase-1 .. rbase+kR of u1: shift so row index r maps to u1 row rbase-1+r
    T cv[kR + 2][V];
    T xl[kR + 2], xr[kR + 2];
#pragma unroll
    for (int r = 0; r < kR + 2; ++r) {
      if (r >= 1 && r <= kR) {  // my own rows: still in registers
#pragma unroll
        for (int k = 0; k < V; ++k) cv[r][k] = own[r - 1][k];
        continue;
      }
      int row = rbase - 1 + r;
      row = row < 0 ? 0 : (row >= G::U1ROWS ? G::U1ROWS - 1 : row);  // edge rows: unused values
      vload<T>(P + row * G::W + V * lane, cv[r]);
    }
#pragma unroll
    for (int r = 0; r < kR + 2; ++r) {
      int row = rbase - 1 + r;
      row = row < 0 ? 0 : (row >= G::U1ROWS ? G::U1ROWS - 1 : row);
      if (O::DIAG || (r >= 1 && r <= kR)) {
        if constexpr (XS == 1) {
          xl[r] = __shfl_up_sync(0xffffffffu, cv[r][V - 1], 1);
          xr[r] = __shfl_down_sync(0xffffffffu, cv[r][0], 1);
        } else {
          xl[r] = P[row * G::W + V * lane - 1];
          xr[r] = P[row * G::W + V * lane + V];
        }
      } else {
        xl[r] = T(0);
        xr[r] = T(0);
      }
    }
    T h[kR + 2][V];
#pragma unroll
    for (int r = 0; r < kR + 2; ++r)
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (O::DIAG || (r >= 1 && r <= kR))
          h[r][k] = add(k > 0 ? cv[r][k - 1] : xl[r], k < V - 1 ? cv[r][k + 1] : xr[r]);
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) t[j][k] = tuple_at<T, OP>(cv, h, xl, xr, j, k);
  };
  auto emit = [&](const Tup (&lo)[kR][V], const Tup (&mid)[kR][V], const Tup (&hi)[kR][V]) {
    T v[kR][V];
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) v[j][k] = O::out(lo[j][k], mid[j][k], hi[j][k]);
    if constexpr (RV == RV_RESID) {
#pragma unroll
      for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const double rv = (double)O::resid(lo[j][k], mid[j][k], hi[j][k]);
          acc[j][k] = __dadd_rn(acc[j][k], ok[j][k] ? rv : 0.0);
        }
    }
    if (fast) {
#pragma unroll
      for (int j = 0; j < kR; ++j) vstore<T>(optr + roff[j], v[j]);
    } else {
#pragma unroll
      for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k)
          if (ok[j][k]) optr[roff[j] + k] = v[j][k];
    }
    optr += a.osz;
  };

  // Input plane p is z = zs - 2 + p.  After input p (p >= 2): u1(z-1) =
  // u1(zs - 3 + p) and its sweep-2 tuple; with three of those (p >= 4):
  // out(zs + p - 4).
  Tup A[kR][V], B[kR][V], C[kR][V];   // sweep-1 tuples (input planes)
  Tup X[kR][V], Y[kR][V], Z[kR][V];   // sweep-2 tuples (u1 planes)
  // prologue: input planes 0, 1
  load_in(A);
  load_in(B);
  // p = 2, 3, 4 handled in the steady loop with guards on the u1 pipeline
  int p = 2;
  auto step = [&](Tup (&lo)[kR][V], Tup (&mid)[kR][V], Tup (&hi)[kR][V],
                  Tup (&ulo)[kR][V], Tup (&umid)[kR][V], Tup (&uhi)[kR][V]) {
    load_in(hi);
    const int zu = zs - 3 + p;  // u1 plane completed by this step
    make_u1(lo, mid, hi, zu);
    load_u1(uhi, zu);
    if (p >= 4) emit(ulo, umid, uhi);
    ++p;
  };
  for (; p + 3 <= np; ) {
    step(A, B, C, X, Y, Z);
    step(B, C, A, Y, Z, X);
    step(C, A, B, Z, X, Y);
  }
  if (p < np) {
    step(A, B, C, X, Y, Z);
    if (p < np) step(B, C, A, Y, Z, X);
  }

  if constexpr (RV != RV_NONE) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) t = __dadd_rn(t, acc[j][k]);
    cta_reduce_finish(t, CB_SUM, red, flag, kNW * 32, a.partials, a.counter, a.result, gridDim.x,
                      blockIdx.x);
  }
}

}  // namespace

// Two sweeps (out = OP(OP(in))) over the whole local interior of a single-rank
// grid (z-halo = physical boundary).  With rv == RV_RESID the residual of the
// INTERMEDIATE iterate (the input of the second sweep) is reduced into red.
template <int OP, int RV, typename T, int XS, int MINB, int kNW>
static cudaError_t launch2(const SweepPlan& p, int64_t* launches) {
  using G = Geo2<T, kNW>;
  auto kern = sweep2_tma<OP, RV, T, XS, MINB, kNW>;
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * (kNW + 1), G::SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  const View& in = p.in[0];
  Sweep2Args<T> a{};
  a.out = static_cast<T*>(p.out.origin);
  a.osy = p.out.pitch;
  a.osz = p.out.plane;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  a.nz = (int)in.nzl;
  a.nzr = (int)in.nzl;
  a.tiles_x = (int)((in.nx + G::TXO - 1) / G::TXO);
  a.tiles_y = (int)((in.ny + G::TYO - 1) / G::TYO);
  const int64_t tiles = (int64_t)a.tiles_x * a.tiles_y;
  const int64_t slots = (int64_t)occ * p.num_sms;
  int chunks = tiles * 2 <= slots ? (int)std::max<int64_t>(1, std::min<int64_t>(slots / tiles, a.nzr))
                                  : (int)std::max<int64_t>(1, (a.nzr + 31) / 32);
  if (p.zchunks > 0) chunks = (int)std::min<int64_t>(p.zchunks, a.nzr);
  a.chunk = (a.nzr + chunks - 1) / chunks;
  chunks = (a.nzr + a.chunk - 1) / a.chunk;
  a.col0 = (int)in.ox;
  a.row0 = in.h;
  a.pln0 = in.h;
  a.partials = p.red.partials;
  a.counter = p.red.counter;
  a.result = p.red.result;
  CUtensorMap map;
  if (!encode_tma_3d(&map, in, G::W, G::INROWS, p.l2promo)) return cudaErrorInvalidValue;
  const int64_t units = tiles * chunks;
  if (RV != RV_NONE && units > p.red.max_partials) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)units, 32 * (kNW + 1), G::SMEM, p.stream>>>(a, map);
  ++*launches;
  return cudaGetLastError();
}

template <int XS, int MINB, int NW>
static cudaError_t launch2v(const SweepPlan& p, int64_t* launches) {
  const bool f64 = p.in[0].dtype == 0;
  const bool resid = p.rv == RV_RESID;
  if (f64) return resid ? launch2<OP_JACOBI7, RV_RESID, double, XS, MINB, NW>(p, launches)
                        : launch2<OP_JACOBI7, RV_NONE, double, XS, MINB, NW>(p, launches);
  return resid ? launch2<OP_JACOBI7, RV_RESID, float, XS, MINB, NW>(p, launches)
               : launch2<OP_JACOBI7, RV_NONE, float, XS, MINB, NW>(p, launches);
}

// The first design's geometries (gscl_set_option "variant" 1..4; measured at
// 512^3 fp64, ms per 100-sweep step: smem/2 CTAs/8 warps 30.2, shfl/1/8 34.3,
// smem/1/8 33.5; 4 = its former default).
cudaError_t launch_sweep2_smem(const SweepPlan& p, int64_t* launches) {
  switch (p.variant) {
    case 1: return launch2v<1, 1, 8>(p, launches);
    case 2: return launch2v<0, 1, 8>(p, launches);
    case 3: return launch2v<0, 1, 16>(p, launches);
    case 4: return launch2v<0, 2, 8>(p, launches);
    default: return cudaErrorInvalidValue;
  }
}

#endif  // GSCL_ABLATIONS

}  // namespace gscl
