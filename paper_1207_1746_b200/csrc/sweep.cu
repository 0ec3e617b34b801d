// sweep.cu — the do_all / fused do_reduce sweep kernels for sm_100a.
//
// sweep_tma: TMA-staged 2.5-D z-streaming.
//   * One CTA owns an xy tile of TX x TY points (TX = 32 lanes x 16 bytes) and a
//     chunk of z planes.  Warp NW is the producer: one elected lane issues, per
//     input plane, a 3-D cp.async.bulk.tensor of the (TY+2) x (TX+2V) halo tile
//     (plus the 7 coefficient tiles for VARCOEF8) into an S-stage shared-memory
//     ring, completing on that stage's mbarrier (expect_tx).
//   * Warps 0..NW-1 consume: each lane reads its R rows x V points (16-byte
//     ld.shared.v2.f64 / v4.f32) and x/y neighbours from the landed plane,
//     computes the operator's per-plane tuple (ops.cuh), releases the stage,
//     and combines the tuples of planes z-1, z, z+1 held in registers (the z
//     register queue) into out(z), stored with 16-byte st.global.
//   * Fused reductions fold per point in registers and finish with the
//     deterministic CTA/grid epilogue (reduce_common.cuh).
// sweep_plain: one thread per point, every neighbour loaded from global
//   memory; the same ops.cuh trees.  Used as an ablation baseline and as a
//   second GPU implementation in the tests.
#include <algorithm>
#include <cstdio>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

template <typename T, int NW, int R> struct Geo {
  static constexpr int VEC = Vec<T>::N;
  static constexpr int TX = 32 * VEC;
  static constexpr int TY = NW * R;
  static constexpr int ROWW = TX + 2 * VEC;  // smem row: [V pad | TX interior | V pad]
  static constexpr int UROWS = TY + 2;
  static constexpr int UBYTES = UROWS * ROWW * (int)sizeof(T);
  static constexpr int UBYTES_AL = (UBYTES + 127) / 128 * 128;
  static constexpr int CBYTES = TY * TX * (int)sizeof(T);
};

// Geometry per operator: rows per lane R, consumer warps NW, ring stages S.
template <int OP> struct Cfg {
  static constexpr int NW = 8;
  static constexpr int R = (OP == OP_VARCOEF8) ? 1 : 2;
  static constexpr int S = (OP == OP_VARCOEF8) ? 4 : 6;
};

constexpr int kHeaderBytes = 1024;  // mbarriers + reduction scratch

template <typename T> struct SweepArgs {
  T* out;
  int64_t osy, osz;
  int x0, x1, y0, y1, z0, z1;  // local interior box (outputs)
  int tx_first, tiles_x, tiles_y, chunk;
  int col0[8], row0[8], pln0[8];  // array coords of interior (0,0,0) per input
  T eps;
  double* partials;
  unsigned* counter;
  double* result;
  int comb;
};
struct Maps {
  CUtensorMap m[8];
};

template <int OP, int RV, bool WRITE, typename T>
__global__ void __launch_bounds__(32 * (Cfg<OP>::NW + 1))
    sweep_tma(const __grid_constant__ SweepArgs<T> a, const __grid_constant__ Maps maps) {
  constexpr int NW = Cfg<OP>::NW, R = Cfg<OP>::R, S = Cfg<OP>::S;
  using G = Geo<T, NW, R>;
  using O = OpT<OP, T>;
  using Tup = typename O::Tup;
  constexpr int V = G::VEC;
  constexpr int NC = O::NCOEF;
  constexpr int STAGE = G::UBYTES_AL + NC * G::CBYTES;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  double* red = reinterpret_cast<double*>(empty + S);
  int* flag = reinterpret_cast<int*>(red + NW);
  unsigned char* stages = smem + kHeaderBytes;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int unit = blockIdx.x;
  const int tx = unit % a.tiles_x;
  unit /= a.tiles_x;
  const int ty = unit % a.tiles_y;
  const int zc = unit / a.tiles_y;
  const int xt0 = (a.tx_first + tx) * G::TX;
  const int yt0 = a.y0 + ty * G::TY;
  const int zs = a.z0 + zc * a.chunk;
  const int ze = min(zs + a.chunk, a.z1);
  const int np = ze - zs + 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // ---------------- producer warp
    if (lane == 0) {
      for (int c = 0; c <= NC; ++c) tma_prefetch_desc(&maps.m[c]);
      for (int p = 0; p < np; ++p) {
        const int s = p % S;
        if (p >= S) mbar_wait(&empty[s], ((p / S) - 1) & 1);
        const int z = zs - 1 + p;
        const bool coef = NC > 0 && p >= 1 && p <= np - 2;
        mbar_arrive_expect_tx(&full[s], G::UBYTES + (coef ? NC * G::CBYTES : 0));
        unsigned char* st = stages + s * STAGE;
        tma_load_3d(st, &maps.m[0], a.col0[0] + xt0 - V, a.row0[0] + yt0 - 1, a.pln0[0] + z, &full[s]);
        if (coef) {
#pragma unroll
          for (int c = 1; c <= NC; ++c)
            tma_load_3d(st + G::UBYTES_AL + (c - 1) * G::CBYTES, &maps.m[c], a.col0[c] + xt0,
                        a.row0[c] + yt0, a.pln0[c] + z, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  double acc = 0.0;
  if constexpr (RV != RV_NONE) acc = comb_identity(a.comb);
  Tup lo[R][V], mid[R][V], hi[R][V];
  const int xb = xt0 + V * lane;
  const int rbase = warp * R;  // smem row of tile row (rbase - 1)

  for (int p = 0; p < np; ++p) {
    const int s = p % S;
    mbar_wait(&full[s], (p / S) & 1);
    const T* U = reinterpret_cast<const T*>(stages + s * STAGE);
    T cv[R + 2][V];
#pragma unroll
    for (int r = 0; r < R + 2; ++r) vload<T>(U + (rbase + r) * G::ROWW + V + V * lane, cv[r]);
    T xl[R + 2], xr[R + 2];
#pragma unroll
    for (int r = 0; r < R + 2; ++r) {
      if (O::DIAG || (r >= 1 && r <= R)) {
        xl[r] = U[(rbase + r) * G::ROWW + V + V * lane - 1];
        xr[r] = U[(rbase + r) * G::ROWW + V + V * lane + V];
      } else {
        xl[r] = T(0);
        xr[r] = T(0);
      }
    }
    T cf[NC > 0 ? NC : 1][R][V];
    if constexpr (NC > 0) {
      if (p >= 1 && p <= np - 2) {
        const T* C = reinterpret_cast<const T*>(stages + s * STAGE + G::UBYTES_AL);
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < R; ++j) vload<T>(C + c * (G::TY * G::TX) + (rbase + j) * G::TX + V * lane, cf[c][j]);
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int j = 0; j < R; ++j)
#pragma unroll
            for (int k = 0; k < V; ++k) cf[c][j][k] = T(0);
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
#pragma unroll
      for (int k = 0; k < V; ++k) {
        Nbr<T> n;
        n.c = cv[j + 1][k];
        n.xm = k > 0 ? cv[j + 1][k - 1] : xl[j + 1];
        n.xp = k < V - 1 ? cv[j + 1][k + 1] : xr[j + 1];
        n.ym = cv[j][k];
        n.yp = cv[j + 2][k];
        if constexpr (O::DIAG) {
          n.mm = k > 0 ? cv[j][k - 1] : xl[j];
          n.pm = k < V - 1 ? cv[j][k + 1] : xr[j];
          n.mp = k > 0 ? cv[j + 2][k - 1] : xl[j + 2];
          n.pp = k < V - 1 ? cv[j + 2][k + 1] : xr[j + 2];
        }
        T cfk[NC > 0 ? NC : 1];
#pragma unroll
        for (int c = 0; c < (NC > 0 ? NC : 1); ++c) cfk[c] = NC > 0 ? cf[c][j][k] : T(0);
        hi[j][k] = O::plane(n, cfk);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    if (p >= 2) {
      const int z = zs + p - 2;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int y = yt0 + rbase + j;
        if (y < a.y1) {
          T v[V];
#pragma unroll
          for (int k = 0; k < V; ++k) v[k] = O::out(lo[j][k], mid[j][k], hi[j][k]);
          if constexpr (RV != RV_NONE) {
#pragma unroll
            for (int k = 0; k < V; ++k)
              if (xb + k >= a.x0 && xb + k < a.x1)
                acc = comb_apply(a.comb, acc, red_value<OP, RV, T>(lo[j][k], mid[j][k], hi[j][k], v[k], a.eps));
          }
          if constexpr (WRITE) {
            T* o = a.out + (int64_t)z * a.osz + (int64_t)y * a.osy + xb;
            if (xb >= a.x0 && xb + V <= a.x1) {
              vstore<T>(o, v);
            } else {
#pragma unroll
              for (int k = 0; k < V; ++k)
                if (xb + k >= a.x0 && xb + k < a.x1) o[k] = v[k];
            }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) {
        lo[j][k] = mid[j][k];
        mid[j][k] = hi[j][k];
      }
  }

  if constexpr (RV != RV_NONE)
    cta_reduce_finish(acc, a.comb, red, flag, NW * 32, a.partials, a.counter, a.result, gridDim.x,
                      blockIdx.x);
}

// ------------------------------------------------------------------ plain
template <typename T> struct PlainArgs {
  const T* in[8];
  int64_t sy[8], sz[8];
  T* out;
  int64_t osy, osz;
  int x0, x1, y0, y1, z0, z1;
  int bx, by;  // blocks along x, y
  T eps;
  double* partials;
  unsigned* counter;
  double* result;
  int comb;
};

template <int OP, typename T>
__device__ __forceinline__ typename OpT<OP, T>::Tup plain_plane(const PlainArgs<T>& a, int x, int y, int z) {
  using O = OpT<OP, T>;
  const T* u = a.in[0] + (int64_t)z * a.sz[0] + (int64_t)y * a.sy[0] + x;
  const int64_t sy = a.sy[0];
  Nbr<T> n;
  n.c = __ldg(u);
  n.xm = __ldg(u - 1);
  n.xp = __ldg(u + 1);
  n.ym = __ldg(u - sy);
  n.yp = __ldg(u + sy);
  if constexpr (O::DIAG) {
    n.mm = __ldg(u - sy - 1);
    n.pm = __ldg(u - sy + 1);
    n.mp = __ldg(u + sy - 1);
    n.pp = __ldg(u + sy + 1);
  }
  T cf[O::NCOEF > 0 ? O::NCOEF : 1];
  if constexpr (O::NCOEF > 0) {
#pragma unroll
    for (int c = 0; c < O::NCOEF; ++c)
      cf[c] = __ldg(a.in[c + 1] + (int64_t)z * a.sz[c + 1] + (int64_t)y * a.sy[c + 1] + x);
  } else {
    cf[0] = T(0);
  }
  return O::plane(n, cf);
}

template <int OP, int RV, bool WRITE, typename T>
__global__ void __launch_bounds__(256) sweep_plain(const __grid_constant__ PlainArgs<T> a) {
  __shared__ double red[8];
  __shared__ int flag;
  using O = OpT<OP, T>;
  int b = blockIdx.x;
  const int bxi = b % a.bx;
  b /= a.bx;
  const int byi = b % a.by;
  const int z = a.z0 + b / a.by;
  const int x = a.x0 + bxi * 32 + (threadIdx.x & 31);
  const int y = a.y0 + byi * 8 + (threadIdx.x >> 5);
  double acc = 0.0;
  if constexpr (RV != RV_NONE) acc = comb_identity(a.comb);
  if (x < a.x1 && y < a.y1) {
    auto lo = plain_plane<OP, T>(a, x, y, z - 1);
    auto mid = plain_plane<OP, T>(a, x, y, z);
    auto hi = plain_plane<OP, T>(a, x, y, z + 1);
    T v = O::out(lo, mid, hi);
    if constexpr (WRITE) a.out[(int64_t)z * a.osz + (int64_t)y * a.osy + x] = v;
    if constexpr (RV != RV_NONE) acc = comb_apply(a.comb, acc, red_value<OP, RV, T>(lo, mid, hi, v, a.eps));
  }
  if constexpr (RV != RV_NONE)
    cta_reduce_finish(acc, a.comb, red, &flag, 256, a.partials, a.counter, a.result, gridDim.x, blockIdx.x);
}

// ------------------------------------------------------------------ host side
namespace {

template <typename T> T* origin_of(const View& v) { return static_cast<T*>(v.origin); }

int auto_chunks(int64_t tiles, int64_t nzr, int resident) {
  int best = 1;
  double best_cost = 1e30;
  int cmax = (int)std::min<int64_t>(nzr, 128);
  for (int c = 1; c <= cmax; ++c) {
    int64_t L = (nzr + c - 1) / c;
    int64_t ceff = (nzr + L - 1) / L;
    int64_t units = tiles * ceff;
    int64_t waves = (units + resident - 1) / resident;
    double eff = (double)units / (double)(waves * resident);
    double over = (double)(L + 2) / (double)L;
    double cost = over / eff;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = (int)ceff;
    }
  }
  return best;
}

template <int OP, int RV, bool WRITE, typename T>
cudaError_t launch_tma(const SweepPlan& p, int64_t* launches) {
  constexpr int NW = Cfg<OP>::NW, R = Cfg<OP>::R, S = Cfg<OP>::S;
  using G = Geo<T, NW, R>;
  constexpr int NC = OpT<OP, T>::NCOEF;
  constexpr int STAGE = G::UBYTES_AL + NC * G::CBYTES;
  constexpr int SMEM = kHeaderBytes + S * STAGE;
  constexpr int THREADS = 32 * (NW + 1);
  auto kern = sweep_tma<OP, RV, WRITE, T>;
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  const Box& b = p.box;
  SweepArgs<T> a{};
  a.out = WRITE ? origin_of<T>(p.out) : nullptr;
  a.osy = p.out.pitch;
  a.osz = p.out.plane;
  a.x0 = (int)b.x0; a.x1 = (int)b.x1; a.y0 = (int)b.y0; a.y1 = (int)b.y1;
  a.z0 = (int)b.z0; a.z1 = (int)b.z1;
  a.tx_first = (int)(b.x0 / G::TX);
  a.tiles_x = (int)((b.x1 - 1) / G::TX) - a.tx_first + 1;
  a.tiles_y = (int)((b.y1 - b.y0 + G::TY - 1) / G::TY);
  int64_t tiles = (int64_t)a.tiles_x * a.tiles_y;
  int64_t nzr = b.z1 - b.z0;
  int chunks = p.zchunks > 0 ? (int)std::min<int64_t>(p.zchunks, nzr)
                             : auto_chunks(tiles, nzr, occ * p.num_sms);
  a.chunk = (int)((nzr + chunks - 1) / chunks);
  chunks = (int)((nzr + a.chunk - 1) / a.chunk);
  Maps maps;
  for (int i = 0; i < p.n_in; ++i) {
    const View& v = p.in[i];
    bool ok = (i == 0) ? encode_tma_3d(&maps.m[i], v, G::ROWW, G::UROWS)
                       : encode_tma_3d(&maps.m[i], v, G::TX, G::TY);
    if (!ok) return cudaErrorInvalidValue;
    a.col0[i] = (int)v.ox;
    a.row0[i] = v.h;
    a.pln0[i] = v.h;
  }
  a.eps = (T)p.eps;
  a.partials = p.red.partials;
  a.counter = p.red.counter;
  a.result = p.red.result;
  a.comb = p.red.comb;
  int64_t units = tiles * chunks;
  if (RV != RV_NONE && units > p.red.max_partials) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)units, THREADS, SMEM, p.stream>>>(a, maps);
  ++*launches;
  return cudaGetLastError();
}

template <int OP, int RV, bool WRITE, typename T>
cudaError_t launch_plain(const SweepPlan& p, int64_t* launches) {
  const Box& b = p.box;
  PlainArgs<T> a{};
  for (int i = 0; i < p.n_in; ++i) {
    a.in[i] = origin_of<T>(p.in[i]);
    a.sy[i] = p.in[i].pitch;
    a.sz[i] = p.in[i].plane;
  }
  a.out = WRITE ? origin_of<T>(p.out) : nullptr;
  a.osy = p.out.pitch;
  a.osz = p.out.plane;
  a.x0 = (int)b.x0; a.x1 = (int)b.x1; a.y0 = (int)b.y0; a.y1 = (int)b.y1;
  a.z0 = (int)b.z0; a.z1 = (int)b.z1;
  a.bx = (int)((b.x1 - b.x0 + 31) / 32);
  a.by = (int)((b.y1 - b.y0 + 7) / 8);
  a.eps = (T)p.eps;
  a.partials = p.red.partials;
  a.counter = p.red.counter;
  a.result = p.red.result;
  a.comb = p.red.comb;
  int64_t blocks = (int64_t)a.bx * a.by * (b.z1 - b.z0);
  if (RV != RV_NONE && blocks > p.red.max_partials) return cudaErrorInvalidConfiguration;
  sweep_plain<OP, RV, WRITE, T><<<(unsigned)blocks, 256, 0, p.stream>>>(a);
  ++*launches;
  return cudaGetLastError();
}

template <int OP, int RV, bool WRITE, typename T>
cudaError_t launch_impl(const SweepPlan& p, int64_t* launches) {
  return p.impl == 1 ? launch_plain<OP, RV, WRITE, T>(p, launches)
                     : launch_tma<OP, RV, WRITE, T>(p, launches);
}

template <typename T> cudaError_t dispatch(const SweepPlan& p, int64_t* launches) {
  if (p.rv == RV_NONE) {
    switch (p.op) {
      case OP_FIG1B: return launch_impl<OP_FIG1B, RV_NONE, true, T>(p, launches);
      case OP_LAP7: return launch_impl<OP_LAP7, RV_NONE, true, T>(p, launches);
      case OP_JACOBI7: return launch_impl<OP_JACOBI7, RV_NONE, true, T>(p, launches);
      case OP_LAP27: return launch_impl<OP_LAP27, RV_NONE, true, T>(p, launches);
      case OP_JACOBI27: return launch_impl<OP_JACOBI27, RV_NONE, true, T>(p, launches);
      case OP_VARCOEF8: return launch_impl<OP_VARCOEF8, RV_NONE, true, T>(p, launches);
    }
  } else if (p.rv == RV_RESID) {
    if (p.op == OP_JACOBI7 || p.op == OP_LAP7)
      return p.write ? launch_impl<OP_JACOBI7, RV_RESID, true, T>(p, launches)
                     : launch_impl<OP_JACOBI7, RV_RESID, false, T>(p, launches);
    if (p.op == OP_JACOBI27 || p.op == OP_LAP27)
      return p.write ? launch_impl<OP_JACOBI27, RV_RESID, true, T>(p, launches)
                     : launch_impl<OP_JACOBI27, RV_RESID, false, T>(p, launches);
  } else if (p.rv == RV_CONV && p.op == OP_FIG1B && p.write) {
    return launch_impl<OP_FIG1B, RV_CONV, true, T>(p, launches);
  } else if (p.rv == RV_SQ && p.op == OP_VARCOEF8 && p.write) {
    return launch_impl<OP_VARCOEF8, RV_SQ, true, T>(p, launches);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_sweep(const SweepPlan& p, int64_t* launches) {
  if (p.box.empty()) return cudaSuccess;
  return p.out.dtype == 0 && p.in[0].dtype == 0 ? dispatch<double>(p, launches)
                                                 : dispatch<float>(p, launches);
}

}  // namespace gscl
