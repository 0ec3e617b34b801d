// sweep2k.cu — two JACOBI27 sweeps per HBM pass (temporal blocking for the
// 27-point operator).
//
// out = OP(OP(u)) with OP = JACOBI27 (B(u)/128 over the 3x3x3 neighbourhood,
// DESIGN.md R6) and the Dirichlet rule of gscl_jacobi_run for the
// intermediate u1 (a point outside the interior keeps its halo value).  Same
// per-plane tuples (c, X = edge pairs, D = corner pairs; ops.cuh Sum27) as the
// single sweep, so the result is bitwise that of two single sweeps; the
// residual check of the pass is RESID27² of u1 (= the input of the second
// sweep), formed from the very tuples the second sweep uses.
//
// Layout: like sweep2v.cu — a lane owns V consecutive x points of R output
// rows, warps stack in y, one producer warp streams one TMA box per input
// plane (u rows y0-2 .. y0+TYO+1) into an S-stage ring; a lane computes u1 on
// its R + 2 rows itself (x neighbours, including the corner pairs, by warp
// shuffle) and keeps the z pipelines of both sweeps in registers.
#include <algorithm>

#include "internal.h"
#include "reduce_common.cuh"

#ifdef GSCL_ABLATIONS  // opt-in JACOBI27 two-sweep pass: measured slower, ablation build only
namespace gscl {

namespace {

template <typename T, int NW, int R, int V, int S> struct GeoK {
  static constexpr int W = 32 * V;          // x points the lanes own
  // two sweeps need two halo columns per side: HL halo lanes per side
  static constexpr int HL = V >= 2 ? 1 : 2;
  static constexpr int TXO = W - 2 * HL * V;
  static constexpr int TYO = NW * R;
  static constexpr int UROWS = TYO + 4;
  // the TMA box must start 16-byte aligned: it starts LEFT >= V columns left
  // of the tile, lane 0's first point is column OFF of the box row, BW wide
  static constexpr int AL = 16 / (int)sizeof(T);
  static constexpr int LEFT = HL * V > AL ? HL * V : AL;
  static constexpr int OFF = LEFT - HL * V;
  static constexpr int BW = (OFF + W + AL - 1) / AL * AL;
  static constexpr int STAGE = UROWS * BW * (int)sizeof(T);
  static constexpr int STAGE_AL = (STAGE + 127) / 128 * 128;
  static constexpr int HEADER = 1024;
  static constexpr int SMEM = HEADER + S * STAGE_AL;
  static_assert((TXO * (int)sizeof(T)) % 16 == 0, "tile starts stay 16-byte aligned");
  static_assert((R + 2) * V <= 32 && R * V <= 32, "point masks");
};

template <typename T> struct Sweep2KArgs {
  T* out;
  int64_t osy, osz;
  int nx, ny, nz;
  int tiles_x, tiles_y, chunk, nzr;
  int col0, row0, pln0;
  double* partials;
  unsigned* counter;
  double* result;
};

struct Map1 {
  CUtensorMap m;
};

template <typename T> __device__ __forceinline__ T kshfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T> __device__ __forceinline__ T kshfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// Sum27 tuples of rows 1..NR-2 of `rows` (NR rows of V values per lane): the
// tuple of row j + 1 goes to t[j].
template <typename T, int NR, int V, typename Tup>
__device__ __forceinline__ void tuples27(const T (&rows)[NR][V], Tup (&t)[NR - 2][V]) {
  using O = OpT<OP_JACOBI27, T>;
  T h[NR][V];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const T xl = kshfl_up1(rows[r][V - 1]);
    const T xr = kshfl_dn1(rows[r][0]);
#pragma unroll
    for (int k = 0; k < V; ++k) h[r][k] = add(k > 0 ? rows[r][k - 1] : xl, k < V - 1 ? rows[r][k + 1] : xr);
  }
#pragma unroll
  for (int j = 0; j < NR - 2; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) {
      Nbr<T> n;
      n.c = rows[j + 1][k];
      n.xm = n.xp = T(0);  // Sum27 reads only the pair sums
      n.ym = rows[j][k];
      n.yp = rows[j + 2][k];
      n.h0 = h[j + 1][k];
      n.hm = h[j][k];
      n.hp = h[j + 2][k];
      t[j][k] = O::plane(n, nullptr);
    }
}

template <int RV, typename T, int NW, int R, int V, int S, int MINB>
__global__ void __launch_bounds__(32 * (NW + 1), MINB)
    sweep2k_tma(const __grid_constant__ Sweep2KArgs<T> a, const __grid_constant__ Map1 map) {
  using G = GeoK<T, NW, R, V, S>;
  using O = OpT<OP_JACOBI27, T>;
  using Tup = typename O::Tup;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  double* red = reinterpret_cast<double*>(empty + S);
  int* flag = reinterpret_cast<int*>(red + NW);
  unsigned char* stages = smem + G::HEADER;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int unit = blockIdx.x;
  const int tx = unit % a.tiles_x;
  unit /= a.tiles_x;
  const int ty = unit % a.tiles_y;
  const int zc = unit / a.tiles_y;
  const int xt0 = tx * G::TXO, yt0 = ty * G::TYO;
  const int zs = zc * a.chunk;
  const int ze = min(zs + a.chunk, a.nzr);
  const int np = ze - zs + 4;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // ---------------- producer: one u box per input plane
    if (lane == 0) {
      tma_prefetch_desc(&map.m);
      int s = 0;
      uint32_t ph = 0;
      for (int p = 0; p < np; ++p) {
        if (p >= S) mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], G::STAGE);
        tma_load_3d(stages + s * G::STAGE_AL, &map.m, a.col0 + xt0 - G::LEFT, a.row0 + yt0 - 2, a.pln0 + zs - 2 + p,
                    &full[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumers: warp w's output rows y = yt0 + w*R + r; its u1
  // rows j = 0..R+1 are y = yt0 + w*R - 1 + j; its u rows are box rows w*R .. w*R + R + 3.
  const int xs = xt0 - G::HL * V + V * lane;
  const int yb = yt0 + warp * R;
  uint32_t in1 = 0;
#pragma unroll
  for (int j = 0; j < R + 2; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (xs + k >= 0 && xs + k < a.nx && yb - 1 + j >= 0 && yb - 1 + j < a.ny) in1 |= 1u << (j * V + k);
  uint32_t okm = 0;
  const bool lane_out = lane >= G::HL && lane < 32 - G::HL;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (lane_out && xs + k < a.nx && yb + r < a.ny) okm |= 1u << (r * V + k);
  constexpr uint32_t kAll1 = ((R + 2) * V == 32) ? 0xffffffffu : ((1u << ((R + 2) * V)) - 1u);
  constexpr uint32_t kAllO = (R * V == 32) ? 0xffffffffu : ((1u << (R * V)) - 1u);
  const bool fast = okm == kAllO;
  const bool warp_int = __all_sync(0xffffffffu, in1 == kAll1);
  T* optr = a.out + (int64_t)yb * a.osy + xs + (int64_t)zs * a.osz;
  double acc = 0.0;

  int s = 0;
  uint32_t ph = 0;
  // sweep-1 tuples of the next input plane (R + 2 u1 rows)
  auto load_in = [&](Tup (&t)[R + 2][V]) {
    mbar_wait(&full[s], ph);
    const T* U = reinterpret_cast<const T*>(stages + s * G::STAGE_AL) + warp * R * G::BW + G::OFF + V * lane;
    T rows[R + 4][V];
#pragma unroll
    for (int r = 0; r < R + 4; ++r) vload<T>(U + r * G::BW, rows[r]);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
    tuples27<T, R + 4, V>(rows, t);
  };
  // u1 plane z (R + 2 rows) from the tuples of z-1, z, z+1, then its
  // second-sweep tuples at my R output rows
  auto make_u1 = [&](const Tup (&lo)[R + 2][V], const Tup (&mid)[R + 2][V], const Tup (&hi)[R + 2][V], int z,
                     Tup (&t2)[R][V]) {
    const bool zin = z >= 0 && z < a.nz;
    T u1[R + 2][V];
#pragma unroll
    for (int j = 0; j < R + 2; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k)
        u1[j][k] = (zin && (warp_int || ((in1 >> (j * V + k)) & 1u))) ? O::out(lo[j][k], mid[j][k], hi[j][k])
                                                                      : mid[j][k].c;
    tuples27<T, R + 2, V>(u1, t2);
  };
  auto emit = [&](const Tup (&lo)[R][V], const Tup (&mid)[R][V], const Tup (&hi)[R][V]) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      T v[V];
#pragma unroll
      for (int k = 0; k < V; ++k) v[k] = O::out(lo[r][k], mid[r][k], hi[r][k]);
      if constexpr (RV == RV_RESID) {  // RESID27² of the intermediate iterate at my output points
#pragma unroll
        for (int k = 0; k < V; ++k)
          acc = __dadd_rn(acc, ((okm >> (r * V + k)) & 1u) ? (double)O::resid_sum(lo[r][k], mid[r][k], hi[r][k])
                                                           : 0.0);
      }
      T* o = optr + (int64_t)r * a.osy;
      if (fast) {
        vstore<T>(o, v);
      } else {
#pragma unroll
        for (int k = 0; k < V; ++k)
          if ((okm >> (r * V + k)) & 1u) o[k] = v[k];
      }
    }
    optr += a.osz;
  };

  // input plane p is z = zs-2+p; after p >= 2: u1(zs-3+p) and its second-sweep
  // tuples; p >= 4: out(zs+p-4)
  Tup A[R + 2][V], B[R + 2][V], C[R + 2][V];
  Tup X[R][V], Y[R][V], Z[R][V];
  load_in(A);
  load_in(B);
  int p = 2;
  auto step = [&](Tup (&lo)[R + 2][V], Tup (&mid)[R + 2][V], Tup (&hi)[R + 2][V], Tup (&ulo)[R][V],
                  Tup (&umid)[R][V], Tup (&uhi)[R][V]) {
    load_in(hi);
    make_u1(lo, mid, hi, zs - 3 + p, uhi);
    if (p >= 4) emit(ulo, umid, uhi);
    ++p;
  };
  for (; p + 3 <= np;) {
    step(A, B, C, X, Y, Z);
    step(B, C, A, Y, Z, X);
    step(C, A, B, Z, X, Y);
  }
  if (p < np) {
    step(A, B, C, X, Y, Z);
    if (p < np) step(B, C, A, Y, Z, X);
  }

  if constexpr (RV != RV_NONE)
    cta_reduce_finish(acc, CB_SUM, red, flag, NW * 32, a.partials, a.counter, a.result, gridDim.x, blockIdx.x);
}

template <int RV, typename T, int NW, int R, int V, int S, int MINB>
cudaError_t launch2k(const SweepPlan& p, int64_t* launches) {
  using G = GeoK<T, NW, R, V, S>;
  auto kern = sweep2k_tma<RV, T, NW, R, V, S, MINB>;
  constexpr int NT = 32 * (NW + 1);
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, G::SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  const View& in = p.in[0];
  Sweep2KArgs<T> a{};
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
  int best = 1;
  double best_cost = 1e300;
  for (int c = 1; c <= a.nzr; ++c) {
    const int64_t chunk = (a.nzr + c - 1) / c;
    const int64_t cc = (a.nzr + chunk - 1) / chunk;
    const int64_t waves = (tiles * cc + slots - 1) / slots;
    const double cost = (double)waves * (double)(chunk + 4);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = (int)cc;
    }
  }
  int chunks = p.zchunks > 0 ? (int)std::min<int64_t>(p.zchunks, a.nzr) : best;
  a.chunk = (a.nzr + chunks - 1) / chunks;
  chunks = (a.nzr + a.chunk - 1) / a.chunk;
  Map1 map;
  if (!encode_tma_3d(&map.m, in, G::BW, G::UROWS, p.l2promo)) return cudaErrorInvalidValue;
  a.col0 = (int)in.ox;
  a.row0 = in.h;
  a.pln0 = in.h;
  a.partials = p.red.partials;
  a.counter = p.red.counter;
  a.result = p.red.result;
  const int64_t units = tiles * chunks;
  if (RV != RV_NONE && units > p.red.max_partials) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)units, NT, G::SMEM, p.stream>>>(a, map);
  ++*launches;
  return cudaGetLastError();
}

template <typename T, int NW, int R, int V, int S, int MINB>
cudaError_t launch2k_rv(const SweepPlan& p, int64_t* launches) {
  return p.rv == RV_RESID ? launch2k<RV_RESID, T, NW, R, V, S, MINB>(p, launches)
                          : launch2k<RV_NONE, T, NW, R, V, S, MINB>(p, launches);
}

}  // namespace

// JACOBI27 two-sweep pass (single rank).  fp64: 8 consumer warps x R = 2
// output rows of one point per lane (28 x 16 tile), 6-stage ring of u boxes;
// fp32: 4 points per lane, one row (120 x 8 tile).
cudaError_t launch_sweep2k(const SweepPlan& p, int64_t* launches) {
  if (p.op != OP_JACOBI27 || p.n_in != 1) return cudaErrorInvalidValue;
  if (p.rv != RV_NONE && p.rv != RV_RESID) return cudaErrorInvalidValue;
  if (p.in[0].dtype == 0) {
    switch (p.variant) {  // geometry ablations (gscl_set_option "variant")
      case 11: return launch2k_rv<double, 8, 1, 1, 6, 1>(p, launches);
      case 12: return launch2k_rv<double, 8, 3, 1, 6, 1>(p, launches);
      case 14: return launch2k_rv<double, 4, 2, 1, 6, 2>(p, launches);
      case 15: return launch2k_rv<double, 8, 2, 1, 4, 1>(p, launches);
      case 16: return launch2k_rv<double, 8, 1, 2, 4, 1>(p, launches);
      default: return launch2k_rv<double, 8, 2, 1, 6, 1>(p, launches);
    }
  }
  return launch2k_rv<float, 8, 1, 4, 6, 1>(p, launches);
}

}  // namespace gscl
#endif  // GSCL_ABLATIONS
