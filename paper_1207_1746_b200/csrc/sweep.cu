// sweep.cu — the do_all / fused do_reduce sweep kernels for sm_100a.
//
// sweep_tma: TMA-staged 2.5-D z-streaming.
//   * One CTA owns an xy tile of TX x TY points (TX = 32 lanes x 16 bytes) and a
//     chunk of z planes.  Warp NW is the producer: one lane issues, per input
//     plane, a 3-D cp.async.bulk.tensor of the (TY+2) x (TX+2V) halo tile (plus
//     the 7 coefficient tiles for VARCOEF8) into an S-stage shared-memory ring,
//     completing on that stage's mbarrier (expect_tx).
//   * Warps 0..NW-1 consume: each lane reads its R rows x V points (16-byte
//     ld.shared.v2.f64 / v4.f32) and x/y neighbours from the landed plane,
//     computes the operator's per-plane tuple (ops.cuh) and releases the stage.
//     The tuples of planes z-1, z, z+1 live in three register sets that rotate
//     roles (the z loop is unrolled by 3, so no register moves), and
//     out(z) = combine(z-1, z, z+1) is stored with 16-byte st.global.
//   * Scheduling: when every (tile, chunk) unit fits on the GPU at once, the
//     grid is ONE wave and odd chunks stream downward, so both chunks that
//     share a boundary read it at the same moment (L2 hit, not a second DRAM
//     read); otherwise tiles run in waves with all chunks streaming upward.
//   * Fused reductions fold per point in registers and finish with the
//     deterministic CTA/grid epilogue (reduce_common.cuh).
// sweep_plain: one thread per point, every neighbour loaded from global
//   memory; the same ops.cuh trees.  An ablation baseline and a second GPU
//   implementation for the tests.
#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

GSCL_MODULE_ANCHOR(anchor_sweep)


template <typename T, int NW, int R, int VV = 0> struct Geo {
  static constexpr int VEC = VV > 0 ? VV : Vec<T>::N;  // points per lane along x
  // left/right pad of a smem row = one 16-byte vector, so the TMA box (which
  // starts PAD elements left of the tile) begins 16-byte aligned in global memory
  static constexpr int PAD = Vec<T>::N;
  static constexpr int TX = 32 * VEC;
  static constexpr int TY = NW * R;
  static constexpr int ROWW = TX + 2 * PAD;  // smem row: [pad | TX interior | pad]
  static constexpr int UROWS = TY + 2;
  static constexpr int UBYTES = UROWS * ROWW * (int)sizeof(T);
  static constexpr int UBYTES_AL = (UBYTES + 127) / 128 * 128;
  static constexpr int CBYTES = TY * TX * (int)sizeof(T);
};

// Geometry per operator and type: consumer warps NW, rows per lane R, ring stages S.
template <int OP, typename T, int RW = 0> struct Cfg {
  static constexpr bool K27 = (OP == OP_LAP27 || OP == OP_JACOBI27);
  // 27-point fp64: one point per lane (V = 1) so the x neighbours are
  // consecutive 8-byte words (conflict-free) and 3 rows per lane fit the
  // register budget: 5/3 rows read per output row instead of 3
  static constexpr bool K27V1 = K27 && sizeof(T) == 8 && RW <= 0;
  // consumer warps.  A CTA is NW + 1 warps, and the register file is split
  // per scheduler (4 x 16K registers): 2 CTAs of 9 warps put 5 warps on two
  // schedulers, capping a thread at 96 registers (the 27-point sweeps spilled
  // 12-100 B there); 2 CTAs of 8 warps put 4 on each, 128 registers.
  // fp64 7-point sweeps: 7 consumer warps too (14-row tiles): 3 CTAs of 8
  // warps per SM fit 80 registers (4 / 20 B spills) where 9-warp CTAs were
  // capped at 72 (112 / 224 B spills) — the do_all sweep 0.360 -> 0.348 ms
  // (RW = -6: the read-only 7-point reductions keep 8 warps — 7 measured 6 %
  // slower there: 0.236-0.249 -> 0.250-0.267 ms)
  static constexpr bool K7D = (OP == OP_FIG1B || OP == OP_LAP7 || OP == OP_JACOBI7) && sizeof(T) == 8;
  static constexpr int NW = ((K27V1 || K7D) && RW == 0) ? 7 : 8;
  static constexpr int VV = K27V1 ? 1 : 0;
  static constexpr int R = RW > 0 ? RW : K27V1 ? 3 : (OP == OP_VARCOEF8 || K27) ? 1 : 2;
  // register cap: 3 CTAs of 288 threads per SM (<= 72 registers) for the fp64
  // 7-point sweeps with a 4-stage ring; 2 CTAs for the 8-stage ring (shared
  // memory allows no more), 27-point and fp32 (more live values per lane: at
  // 3 CTAs the fp64 27-point sweeps spilled 224-1096 B and ran 2-6 % slower —
  // kept as variant 3, RW = -1); none for the shared-memory-bound VARCOEF8
  // (one CTA per SM).
  static constexpr int minb(int S) {
    return (OP == OP_VARCOEF8 || RW > 0) ? 1 : RW == -1 ? 3 : RW == -2 ? 2 : K27V1 ? 2
           : (sizeof(T) == 8 && S == 4) ? 3 : 2;
  }
};

constexpr int kHeaderBytes = 1024;  // mbarriers + reduction scratch
// z planes per (tile, chunk) unit in multi-wave mode.  Short units keep the
// tiles that share halo rows/planes resident together, so the shared data comes
// from L2: 8-plane units cut the 7-point do_all's DRAM reads from 1.17 to
// 1.15 GB per 512^3 sweep (profiles/r01_chunking.md).  Reduction sweeps keep
// 32-plane units (fewer CTA partials to fold), as do the 27-point sweeps.
// The 27-point reduction sweeps use 64-plane units: their CTA epilogue (the
// warps of a CTA meet at the reduction barrier, the slowest sets the pace)
// and ring start-up recur per unit — ncu of the fused JACOBI27 + RESID27^2
// sweep put 12 % of its stall samples at that barrier with 32-plane units;
// 64 planes: 0.442 -> 0.403 ms per 512^3 sweep, the RESID27-only pass 0.322 ->
// 0.296 ms (profiles/r02_sweep2r.md).  The plain 27-point sweep keeps 32.
template <int OP, int RV> constexpr int chunk_planes() {
  return ((OP == OP_JACOBI7 || OP == OP_LAP7 || OP == OP_FIG1B) && RV == RV_NONE) ? 8
         : ((OP == OP_JACOBI27 || OP == OP_LAP27) && RV != RV_NONE)               ? 64
                                                                                  : 32;
}

template <typename T> struct SweepArgs {
  T* out;
  int64_t osy, osz;
  int x0, x1, y0, y1, z0, z1;  // local interior box (outputs)
  int tx_first, tiles_x, tiles_y, chunk;
  int dir_alt;                    // odd chunks stream downward
  const int* stop;                // if non-null and set: the iteration is skipped (converged)
  int color;                      // >= 0: store only points with (x+y+z+zoff) % 2 == color
  int zoff;                       // global z of local plane 0 (colour parity)
  int bnd_h;                      // > 0: chunks 0 / 1 are the bnd_h planes at each end
  unsigned* bflag;                // bumped by every boundary unit after its stores
  // peer-memory transport: boundary units also store output planes z0 + i into
  // rlo[i] (the lower neighbour's planes nzl + i) and z1 - 1 - i into rhi[i]
  // (the upper neighbour's planes -1 - i) — interior origins, same pitch — and
  // bump the neighbour's arrival counter (system scope) after their stores
  T* rlo[2];
  T* rhi[2];
  unsigned* rflag_lo;
  unsigned* rflag_hi;
  int nchunks;                    // chunks per tile column
  int rev;                        // walk the chunks top-down (units in reverse z order)
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

// Combine with a compile-time combine when CB >= 0, else the runtime one.
template <int CB> __device__ __forceinline__ double comb_t(int rt, double a, double b) {
  if constexpr (CB == CB_SUM) return __dadd_rn(a, b);
  else return comb_apply(rt, a, b);
}

template <int OP, int RV, bool WRITE, typename T, int CB, int S, bool XSHFL, int RW>
__global__ void __launch_bounds__(32 * (Cfg<OP, T, RW>::NW + 1), Cfg<OP, T, RW>::minb(S))
    sweep_tma(const __grid_constant__ SweepArgs<T> a, const __grid_constant__ Maps maps) {
  constexpr int NW = Cfg<OP, T, RW>::NW, R = Cfg<OP, T, RW>::R;
  using G = Geo<T, NW, R, Cfg<OP, T, RW>::VV>;
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
  const int zc = a.rev ? a.nchunks - 1 - unit / a.tiles_y : unit / a.tiles_y;
  const int xt0 = (a.tx_first + tx) * G::TX;
  const int yt0 = a.y0 + ty * G::TY;
  int zs, ze;
  if (a.bnd_h > 0) {  // boundary-first: [z0, z0+h), [z1-h, z1), then the interior
    if (zc < 2) {
      zs = zc == 0 ? a.z0 : a.z1 - a.bnd_h;
      ze = zs + a.bnd_h;
    } else {
      zs = a.z0 + a.bnd_h + (zc - 2) * a.chunk;
      ze = min(zs + a.chunk, a.z1 - a.bnd_h);
    }
  } else {
    zs = a.z0 + zc * a.chunk;
    ze = min(zs + a.chunk, a.z1);
  }
  const int np = ze - zs + 2;
  const bool down = a.dir_alt && (zc & 1);
  // converged earlier (gscl_converge_run): one thread reads the flag and the
  // CTA leaves together (a uniform decision, never a divergent barrier)
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    s_stop = a.stop ? *(volatile const int*)a.stop : 0;
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (s_stop) return;

  if (warp == NW) {  // ---------------- producer warp
    if (lane == 0) {
      for (int c = 0; c <= NC; ++c) tma_prefetch_desc(&maps.m[c]);
      int s = 0;
      uint32_t ph = 0;
      for (int p = 0; p < np; ++p) {
        if (p >= S) mbar_wait(&empty[s], ph ^ 1);
        const int z = down ? ze - p : zs - 1 + p;
        const bool coef = NC > 0 && p >= 1 && p <= np - 2;
        mbar_arrive_expect_tx(&full[s], G::UBYTES + (coef ? NC * G::CBYTES : 0));
        unsigned char* st = stages + s * STAGE;
        tma_load_3d(st, &maps.m[0], a.col0[0] + xt0 - G::PAD, a.row0[0] + yt0 - 1, a.pln0[0] + z, &full[s]);
        if (coef) {
#pragma unroll
          for (int c = 1; c <= NC; ++c)
            tma_load_3d(st + G::UBYTES_AL + (c - 1) * G::CBYTES, &maps.m[c], a.col0[c] + xt0,
                        a.row0[c] + yt0, a.pln0[c] + z, &full[s]);
        }
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  const int xb = xt0 + V * lane;
  const int rbase = warp * R;  // smem row of tile row (rbase - 1)
  const int y0t = yt0 + rbase;
  bool ok[R][V];  // point inside the box (loop invariant)
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) ok[j][k] = y0t + j < a.y1 && xb + k >= a.x0 && xb + k < a.x1;
  const bool fast = xb >= a.x0 && xb + V <= a.x1 && y0t + R <= a.y1;  // all my points inside
  // Output pointer of row 0 at the first output plane; it moves one plane per step.
  T* optr = nullptr;
  int64_t ostep = 0, roff[R];
  int zo = down ? ze - 1 : zs;  // the plane the next emit stores
  // colour-masked (red-black) sweeps: parity of my point (j, k) at the first
  // output plane; it flips with every plane
  int cpar = (xb + y0t + (down ? ze - 1 : zs) + a.zoff) & 1;
  if constexpr (WRITE) {
    optr = a.out + (int64_t)y0t * a.osy + xb + (int64_t)(down ? ze - 1 : zs) * a.osz;
    ostep = down ? -a.osz : a.osz;
#pragma unroll
    for (int j = 0; j < R; ++j) roff[j] = (int64_t)j * a.osy;
  }
  // one accumulator per point of the lane: no serial dependency between the
  // points of a step; folded in (j,k) order at the end (deterministic).
  double acc[R][V];
  const double ident = RV != RV_NONE ? comb_identity(a.comb) : 0.0;
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) acc[j][k] = ident;
  int s = 0;
  uint32_t ph = 0;

  // Wait for input step p's plane, build its tuples into t, release the stage.
  auto load = [&](Tup (&t)[R][V], int p) {
    mbar_wait(&full[s], ph);
    const T* U = reinterpret_cast<const T*>(stages + s * STAGE);
    T cv[R + 2][V];
#pragma unroll
    for (int r = 0; r < R + 2; ++r) vload<T>(U + (rbase + r) * G::ROWW + G::PAD + V * lane, cv[r]);
    T xl[R + 2], xr[R + 2];
#pragma unroll
    for (int r = 0; r < R + 2; ++r) {
      if (O::DIAG || (r >= 1 && r <= R)) {
        if constexpr (XSHFL) {
          // x neighbours from the adjacent lanes; the edge lanes read the tile's
          // pad column (a one-lane shared load instead of a 4-way-conflicted one)
          const T l = __shfl_up_sync(0xffffffffu, cv[r][V - 1], 1);
          const T rr = __shfl_down_sync(0xffffffffu, cv[r][0], 1);
          xl[r] = lane == 0 ? U[(rbase + r) * G::ROWW + G::PAD - 1] : l;
          xr[r] = lane == 31 ? U[(rbase + r) * G::ROWW + G::PAD + G::TX] : rr;
        } else {
          xl[r] = U[(rbase + r) * G::ROWW + G::PAD + V * lane - 1];
          xr[r] = U[(rbase + r) * G::ROWW + G::PAD + V * lane + V];
        }
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
    // x pair sums h[r][k] = u(x-1) + u(x+1) of every row this lane needs
    T h[R + 2][V];
#pragma unroll
    for (int r = 0; r < R + 2; ++r)
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (O::DIAG || (r >= 1 && r <= R))
          h[r][k] = add(k > 0 ? cv[r][k - 1] : xl[r], k < V - 1 ? cv[r][k + 1] : xr[r]);
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
        n.h0 = h[j + 1][k];
        if constexpr (O::DIAG) {
          n.hm = h[j][k];
          n.hp = h[j + 2][k];
        }
        T cfk[NC > 0 ? NC : 1];
#pragma unroll
        for (int c = 0; c < (NC > 0 ? NC : 1); ++c) cfk[c] = NC > 0 ? cf[c][j][k] : T(0);
        t[j][k] = O::plane(n, cfk);
      }
    }
    fence_proxy_async_smem();  // generic reads of the stage before its TMA refill
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  };

  // out(z) from the tuples of planes z-1 (lo), z (mid), z+1 (hi); z = the plane
  // optr points at (it advances by one plane per call).
  auto emit = [&](const Tup (&lo)[R][V], const Tup (&mid)[R][V], const Tup (&hi)[R][V]) {
    T v[R][V];
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) v[j][k] = O::out(lo[j][k], mid[j][k], hi[j][k]);
    if constexpr (RV != RV_NONE) {
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const double rv = red_value<OP, RV, T, CB>(lo[j][k], mid[j][k], hi[j][k], v[j][k], a.eps);
          acc[j][k] = comb_t<CB>(a.comb, acc[j][k], ok[j][k] ? rv : ident);
        }
    }
    if constexpr (WRITE) {
      if (a.color >= 0) {  // red-black half-sweep (in place): my colour only
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (ok[j][k] && ((cpar + j + k) & 1) == a.color) optr[roff[j] + k] = v[j][k];
        cpar ^= 1;
      } else if (fast) {
#pragma unroll
        for (int j = 0; j < R; ++j) vstore<T>(optr + roff[j], v[j]);
      } else {
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (ok[j][k]) optr[roff[j] + k] = v[j][k];
      }
      if (a.bnd_h > 0 && zc < 2) {  // boundary plane: also into the neighbour's receiving plane
        T* rp = nullptr;
        if (zc == 0) {
          const int i = zo - a.z0;
          if (i >= 0 && i < 2) rp = a.rlo[i];
        } else {
          const int i = a.z1 - 1 - zo;
          if (i >= 0 && i < 2) rp = a.rhi[i];
        }
        if (rp && a.color < 0) {
          rp += (int64_t)y0t * a.osy + xb;
          if (fast) {
#pragma unroll
            for (int j = 0; j < R; ++j) vstore<T>(rp + roff[j], v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < R; ++j)
#pragma unroll
              for (int k = 0; k < V; ++k)
                if (ok[j][k]) rp[roff[j] + k] = v[j][k];
          }
        }
      }
      optr += ostep;
      zo += down ? -1 : 1;
    }
  };

  // The z loop, unrolled by 3 so the three tuple sets rotate roles in place.
  auto run = [&](auto dtag) {
    constexpr bool D = decltype(dtag)::value;
    Tup A[R][V], B[R][V], C[R][V];
    // step p (>= 2) completes output plane: up zs + p - 2, down ze - p + 1
    auto E = [&](const Tup (&o)[R][V], const Tup (&m)[R][V], const Tup (&n)[R][V], int) {
      if constexpr (D) emit(n, m, o);
      else emit(o, m, n);
    };
    load(A, 0);
    load(B, 1);
    int p = 2;
    for (; p + 3 <= np; p += 3) {
      load(C, p);
      E(A, B, C, p);
      load(A, p + 1);
      E(B, C, A, p + 1);
      load(B, p + 2);
      E(C, A, B, p + 2);
    }
    if (p < np) {
      load(C, p);
      E(A, B, C, p);
      ++p;
      if (p < np) {
        load(A, p);
        E(B, C, A, p);
      }
    }
  };
  if (down) run(std::true_type{});
  else run(std::false_type{});

  if constexpr (RV != RV_NONE) {
    double t = ident;
#pragma unroll
    for (int j = 0; j < R; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) t = comb_t<CB>(a.comb, t, acc[j][k]);
    cta_reduce_finish(t, a.comb, red, flag, NW * 32, a.partials, a.counter, a.result, gridDim.x,
                      blockIdx.x);
  }
  if (a.bnd_h > 0 && zc < 2) {
    // boundary planes stored: publish them to the comm stream, which waits on
    // the counter (cuStreamWaitValue32) before the NCCL halo exchange
    named_bar_sync(2, NW * 32);
    if (threadIdx.x == 0) {
      __threadfence();
      if (a.bflag) atomicAdd(a.bflag, 1u);
      unsigned* rf = zc == 0 ? a.rflag_lo : a.rflag_hi;
      if (rf) {  // the neighbour's planes are written (NVLink / IPC memory)
        __threadfence_system();
        atomicAdd_system(rf, 1u);
      }
    }
  }
}

// ------------------------------------------------------------------ plain
#ifdef GSCL_ABLATIONS  // sweep_plain / sweep_block3d: ablation baselines
template <typename T> struct PlainArgs {
  const T* in[8];
  int64_t sy[8], sz[8];
  T* out;
  int64_t osy, osz;
  int x0, x1, y0, y1, z0, z1;
  int bx, by;  // blocks along x, y
  const int* stop;
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
  n.h0 = add(n.xm, n.xp);
  if constexpr (O::DIAG) {
    n.hm = add(__ldg(u - sy - 1), __ldg(u - sy + 1));
    n.hp = add(__ldg(u + sy - 1), __ldg(u + sy + 1));
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

template <int OP, int RV, bool WRITE, typename T, int CB>
__global__ void __launch_bounds__(256) sweep_plain(const __grid_constant__ PlainArgs<T> a) {
  __shared__ double red[8];
  __shared__ int flag;
  __shared__ int s_stop;
  using O = OpT<OP, T>;
  if (threadIdx.x == 0) s_stop = a.stop ? *(volatile const int*)a.stop : 0;
  __syncthreads();
  if (s_stop) return;
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
    if constexpr (RV != RV_NONE) acc = comb_t<CB>(a.comb, acc, red_value<OP, RV, T, CB>(lo, mid, hi, v, a.eps));
  }
  if constexpr (RV != RV_NONE)
    cta_reduce_finish(acc, a.comb, red, &flag, 256, a.partials, a.counter, a.result, gridDim.x, blockIdx.x);
}

// ------------------------------------------------------------------ host side
#endif  // GSCL_ABLATIONS

namespace {

template <typename T> T* origin_of(const View& v) { return static_cast<T*>(v.origin); }

// Multi-wave chunking: balance wave quantisation against boundary re-reads.
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

template <int OP, int RV, bool WRITE, typename T, int CB, int S, bool XSHFL, int RW = 0>
cudaError_t launch_tma(const SweepPlan& p, int64_t* launches) {
  constexpr int NW = Cfg<OP, T, RW>::NW, R = Cfg<OP, T, RW>::R;
  using G = Geo<T, NW, R, Cfg<OP, T, RW>::VV>;
  constexpr int NC = OpT<OP, T>::NCOEF;
  constexpr int STAGE = G::UBYTES_AL + NC * G::CBYTES;
  constexpr int SMEM = kHeaderBytes + S * STAGE;
  constexpr int THREADS = 32 * (NW + 1);
  auto kern = sweep_tma<OP, RV, WRITE, T, CB, S, XSHFL, RW>;
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
  const int64_t tiles = (int64_t)a.tiles_x * a.tiles_y;
  const int64_t nzr = b.z1 - b.z0 - (p.bnd_h > 0 ? 2 * p.bnd_h : 0);  // planes chunked normally
  const int64_t slots = (int64_t)occ * p.num_sms;
  int chunks;
  bool single = false;
  if (p.zchunks > 0) {
    chunks = (int)std::min<int64_t>(p.zchunks, nzr);
    single = p.sched == 2 || (p.sched == 0 && tiles * chunks <= slots);
  } else if (p.sched == 2 || (p.sched == 0 && 2 * tiles <= slots)) {
    // few tiles (small grids): one wave, fill the GPU with z chunks
    chunks = (int)std::max<int64_t>(1, std::min<int64_t>(slots / tiles, nzr));
    single = true;
  } else if (p.sched == 0) {
    // many tiles: waves of ~32-plane chunks.  Short units balance the waves and
    // keep z-neighbouring chunks of a tile resident together, so their shared
    // boundary planes come from L2 (measured best at 512^3, profiles/).
    constexpr int L = chunk_planes<OP, RV>();
    chunks = (int)std::max<int64_t>(1, (nzr + L - 1) / L);
  } else {
    chunks = auto_chunks(tiles, nzr, (int)slots);
  }
  a.chunk = (int)((nzr + chunks - 1) / chunks);
  chunks = (int)((nzr + a.chunk - 1) / a.chunk);
  a.dir_alt = single && p.sched != 1 ? 1 : 0;
  if (p.bnd_h > 0) {  // two boundary chunks first, all streaming up
    chunks += 2;
    a.dir_alt = 0;
    a.bnd_h = p.bnd_h;
    a.bflag = p.bflag;
    for (int i = 0; i < 2; ++i) {
      a.rlo[i] = static_cast<T*>(p.peer_lo[i]);
      a.rhi[i] = static_cast<T*>(p.peer_hi[i]);
    }
    a.rflag_lo = p.peer_flag_lo;
    a.rflag_hi = p.peer_flag_hi;
    if (p.bnd_units) *p.bnd_units = 2 * tiles;
  }
  a.nchunks = chunks;
  a.rev = (p.reverse && p.bnd_h == 0) ? 1 : 0;
  a.stop = p.stop;
  a.color = p.color;
  a.zoff = (int)(p.zoff & 1);
  Maps maps;
  for (int i = 0; i < p.n_in; ++i) {
    const View& v = p.in[i];
    bool ok = (i == 0) ? encode_tma_3d(&maps.m[i], v, G::ROWW, G::UROWS, p.l2promo)
                       : encode_tma_3d(&maps.m[i], v, G::TX, G::TY, p.l2promo);
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
  const int64_t units = tiles * chunks;
  if (RV != RV_NONE && units > p.red.max_partials) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)units, THREADS, SMEM, p.stream>>>(a, maps);
  ++*launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ 3-D blocked
// Ablation ("register-queue z-streaming vs a 3-D-blocked
// kernel without streaming"): a CTA loads a (32+2) x (8+2) x (8+2) block of u
// (halo included) into shared memory with plain coalesced loads, then each
// thread computes its (x, y) column for 8 planes from shared memory.  No TMA,
// no ring, no z streaming: every block re-reads its halo planes and rows.
#ifdef GSCL_ABLATIONS
template <int OP, typename T>
__global__ void __launch_bounds__(256) sweep_block3d(const __grid_constant__ PlainArgs<T> a) {
  using O = OpT<OP, T>;
  constexpr int BX = 32, BY = 8, BZ = 8;
  __shared__ T sm[BZ + 2][BY + 2][BX + 2];
  int b = blockIdx.x;
  const int bxi = b % a.bx;
  b /= a.bx;
  const int byi = b % a.by;
  const int bzi = b / a.by;
  const int x0 = a.x0 + bxi * BX, y0 = a.y0 + byi * BY, z0 = a.z0 + bzi * BZ;
  const T* in = a.in[0];
  for (int i = threadIdx.x; i < (BZ + 2) * (BY + 2) * (BX + 2); i += blockDim.x) {
    const int lx = i % (BX + 2), ly = (i / (BX + 2)) % (BY + 2), lz = i / ((BX + 2) * (BY + 2));
    const int x = x0 - 1 + lx, y = y0 - 1 + ly, z = z0 - 1 + lz;
    // cells beyond the box's outer halo are never used by a stored point
    const bool ok = x <= a.x1 && y <= a.y1 && z <= a.z1;
    sm[lz][ly][lx] = ok ? __ldg(in + (int64_t)z * a.sz[0] + (int64_t)y * a.sy[0] + x) : T(0);
  }
  __syncthreads();
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x = x0 + tx, y = y0 + ty;
  if (x >= a.x1 || y >= a.y1) return;
  auto tup = [&](int lz) {
    Nbr<T> n;
    n.c = sm[lz][ty + 1][tx + 1];
    n.xm = sm[lz][ty + 1][tx];
    n.xp = sm[lz][ty + 1][tx + 2];
    n.ym = sm[lz][ty][tx + 1];
    n.yp = sm[lz][ty + 2][tx + 1];
    n.h0 = add(n.xm, n.xp);
    T cf[1] = {T(0)};
    return O::plane(n, cf);
  };
  for (int k = 0; k < BZ && z0 + k < a.z1; ++k) {
    const T v = O::out(tup(k), tup(k + 1), tup(k + 2));
    a.out[(int64_t)(z0 + k) * a.osz + (int64_t)y * a.osy + x] = v;
  }
}

template <int OP, typename T>
cudaError_t launch_block3d(const SweepPlan& p, int64_t* launches) {
  const Box& b = p.box;
  PlainArgs<T> a{};
  a.in[0] = origin_of<T>(p.in[0]);
  a.sy[0] = p.in[0].pitch;
  a.sz[0] = p.in[0].plane;
  a.out = origin_of<T>(p.out);
  a.osy = p.out.pitch;
  a.osz = p.out.plane;
  a.x0 = (int)b.x0; a.x1 = (int)b.x1; a.y0 = (int)b.y0; a.y1 = (int)b.y1;
  a.z0 = (int)b.z0; a.z1 = (int)b.z1;
  a.bx = (int)((b.x1 - b.x0 + 31) / 32);
  a.by = (int)((b.y1 - b.y0 + 7) / 8);
  const int64_t bz = (b.z1 - b.z0 + 7) / 8;
  sweep_block3d<OP, T><<<(unsigned)(a.bx * a.by * bz), 256, 0, p.stream>>>(a);
  ++*launches;
  return cudaGetLastError();
}

template <int OP, int RV, bool WRITE, typename T, int CB>
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
  a.stop = p.stop;
  a.eps = (T)p.eps;
  a.partials = p.red.partials;
  a.counter = p.red.counter;
  a.result = p.red.result;
  a.comb = p.red.comb;
  int64_t blocks = (int64_t)a.bx * a.by * (b.z1 - b.z0);
  if (RV != RV_NONE && blocks > p.red.max_partials) return cudaErrorInvalidConfiguration;
  sweep_plain<OP, RV, WRITE, T, CB><<<(unsigned)blocks, 256, 0, p.stream>>>(a);
  ++*launches;
  return cudaGetLastError();
}

// Ring depth: the 7-point fp64 reduction sweeps run 32-plane units with an
// 8-stage ring (fewer, longer-lived CTAs need more bytes in flight each); the
// do_all sweeps run 8-plane units with 4 stages (3 CTAs per SM).
#endif  // GSCL_ABLATIONS

template <int OP, int RV, bool WRITE, typename T, int CB>
cudaError_t launch_impl(const SweepPlan& p, int64_t* launches) {
  constexpr bool k7 = (OP == OP_JACOBI7 || OP == OP_LAP7 || OP == OP_FIG1B) && sizeof(T) == 8;
  constexpr bool k27r = (OP == OP_JACOBI27 || OP == OP_LAP27) && sizeof(T) == 8;
#ifdef GSCL_ABLATIONS
  // sweep_impl 1 (one thread per point) / 2 (3-D blocked), and the geometry
  // variants of the TMA kernel (measured: profiles/r01_ablations.md)
  if (p.impl == 1) return launch_plain<OP, RV, WRITE, T, CB>(p, launches);
  if constexpr ((OP == OP_JACOBI7 || OP == OP_LAP7 || OP == OP_FIG1B) && RV == RV_NONE && WRITE)
    if (p.impl == 2 && p.color < 0 && p.bnd_h == 0) return launch_block3d<OP, T>(p, launches);
  if constexpr (k7) {
    if (p.stages == 8 && RV == RV_NONE) return launch_tma<OP, RV, WRITE, T, CB, 8, false>(p, launches);
    if (p.stages == 4 && RV != RV_NONE) return launch_tma<OP, RV, WRITE, T, CB, 4, false>(p, launches);
  }
  if (p.variant == 1) return launch_tma<OP, RV, WRITE, T, CB, 4, true>(p, launches);
  if constexpr (k7)
    if (p.variant == 4) return launch_tma<OP, RV, WRITE, T, CB, 4, false, -2>(p, launches);  // 2 CTAs/SM
  constexpr bool k27 = (OP == OP_JACOBI27 || OP == OP_LAP27) && sizeof(T) == 8 && RV == RV_NONE;
  if constexpr (k27) {
    if (p.variant == 2) return launch_tma<OP, RV, WRITE, T, CB, 4, false, 2>(p, launches);
    if (p.variant == 3) return launch_tma<OP, RV, WRITE, T, CB, 4, false, -1>(p, launches);  // 3 CTAs/SM (spills)
  }
  if constexpr (k27r)
    if (p.variant == 5) return launch_tma<OP, RV, WRITE, T, CB, 4, false>(p, launches);
#endif
  // Ring depth: the 7-point fp64 reduction sweeps run 32-plane units with an
  // 8-stage ring (fewer, longer-lived CTAs need more bytes in flight each); the
  // do_all sweeps run 8-plane units with 4 stages (3 CTAs per SM).
  if constexpr (k7 && RV != RV_NONE) {
    if constexpr (!WRITE) return launch_tma<OP, RV, WRITE, T, CB, 8, false, -6>(p, launches);
    return launch_tma<OP, RV, WRITE, T, CB, 8, false>(p, launches);
  }
  // fp64 27-point: 2 CTAs/SM with an 8-stage ring (more bytes in flight per
  // CTA; 4 stages = variant 5, 5-6 % slower on config 3)
  if constexpr (k27r) return launch_tma<OP, RV, WRITE, T, CB, 8, false>(p, launches);
  return launch_tma<OP, RV, WRITE, T, CB, 4, false>(p, launches);
}

template <int OP, int RV, bool WRITE, typename T>
cudaError_t launch_cb(const SweepPlan& p, int64_t* launches) {
  return p.red.comb == CB_SUM ? launch_impl<OP, RV, WRITE, T, CB_SUM>(p, launches)
                              : launch_impl<OP, RV, WRITE, T, -1>(p, launches);
}

template <typename T> cudaError_t dispatch(const SweepPlan& p, int64_t* launches) {
  if (p.rv == RV_NONE) {
    switch (p.op) {
      case OP_FIG1B: return launch_impl<OP_FIG1B, RV_NONE, true, T, -1>(p, launches);
      case OP_LAP7: return launch_impl<OP_LAP7, RV_NONE, true, T, -1>(p, launches);
      case OP_JACOBI7: return launch_impl<OP_JACOBI7, RV_NONE, true, T, -1>(p, launches);
      case OP_LAP27: return launch_impl<OP_LAP27, RV_NONE, true, T, -1>(p, launches);
      case OP_JACOBI27: return launch_impl<OP_JACOBI27, RV_NONE, true, T, -1>(p, launches);
      case OP_VARCOEF8: return launch_impl<OP_VARCOEF8, RV_NONE, true, T, -1>(p, launches);
    }
  } else if (p.rv == RV_RESID) {
    if (p.op == OP_JACOBI7 || p.op == OP_LAP7)
      return p.write ? launch_cb<OP_JACOBI7, RV_RESID, true, T>(p, launches)
                     : launch_cb<OP_JACOBI7, RV_RESID, false, T>(p, launches);
    if (p.op == OP_JACOBI27 || p.op == OP_LAP27)
      return p.write ? launch_cb<OP_JACOBI27, RV_RESID, true, T>(p, launches)
                     : launch_cb<OP_JACOBI27, RV_RESID, false, T>(p, launches);
  } else if (p.rv == RV_CONV && p.op == OP_FIG1B && p.write) {
    return launch_impl<OP_FIG1B, RV_CONV, true, T, -1>(p, launches);
  } else if (p.rv == RV_CONV && p.op == OP_JACOBI7 && p.write) {
    return launch_impl<OP_JACOBI7, RV_CONV, true, T, -1>(p, launches);
  } else if (p.rv == RV_SQ && p.op == OP_VARCOEF8 && p.write) {
    return launch_cb<OP_VARCOEF8, RV_SQ, true, T>(p, launches);
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
