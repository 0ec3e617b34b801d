// sweep2x.cu — two JACOBI7 sweeps per HBM pass with the intermediate iterate
// u1 computed ONCE per CTA row: each warp computes u1 on its own rows only
// and hands its first and last u1 row of every plane to the neighbouring
// warps through a shared-memory ring (temporal blocking, SURVEY §8(f) NEXT-2;
// "wide ghost areas").
//
// ABLATION (measured 15 % slower than sweep2r.cu, profiles/r02_sweep2r.md;
// compiled into GSCL_ABLATIONS builds only, variant 60).
// Why it was tried (sweep2r.cu is the register-resident default): there, every warp computes u1 on R + 2 rows for
// its R output rows, so 2 of every 6 u1 rows are recomputed by the
// neighbouring warp — a third of the first sweep's FP64 work, shuffles and
// shared loads.  The pass is bound by that instruction stream at one CTA per
// SM (registers), not by HBM.  Here a warp computes u1 on 4 rows; the u1 band
// of the CTA (NW x 4 rows) is one row wider than the output tile on each side,
// so the outputs are the band minus its first and last row.  Round 1's
// attempt at sharing u1 rows used named barriers between warp pairs every
// plane (no drift allowed between warps) and ran 35 % slower; here the hand-
// over is a ring of D plane slots with one mbarrier per slot, and a warp forms
// the second-sweep tuples of u1 plane q only one plane step after it computed
// u1(q) itself — by then its neighbours, which progress within the same TMA
// ring, have normally published u1(q) too.
//
// Per input plane z (one step):
//   sweep-1 tuples of z  ->  u1(z-1) on my 4 rows (Dirichlet rule)
//   -> publish my rows 0 / 3 of u1(z-1)
//   -> second-sweep tuples of u1(z-2) (my 4 rows; the rows above / below
//      them from the neighbours' published rows)
//   -> out(z-3) from the tuples of u1(z-4), u1(z-3), u1(z-2)
// Both sweeps evaluate the per-plane tuples of ops.cuh: results are bitwise
// those of two single sweeps.
#include <algorithm>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

GSCL_MODULE_ANCHOR(anchor_sweep2x)

#ifdef GSCL_ABLATIONS  // measured slower than sweep2r.cu (profiles/r02_sweep2r.md): ablation builds only

namespace {

constexpr int kHeaderX = 1024;

template <typename T, int NW, int S, int D> struct GeoX {
  static constexpr int V = Vec<T>::N;              // points per lane (one 16-byte vector)
  static constexpr int W = 32 * V;                 // warp strip / box width
  static constexpr int XB = V;                     // box columns left of the tile
  static constexpr int TXO = W - 2 * V;            // output tile width (lanes 1..30)
  static constexpr int RU = 4;                     // u1 rows per warp
  static constexpr int NB = NW * RU;               // u1 band rows (y = yt0 - 1 .. yt0 + NB - 2)
  static constexpr int TYO = NB - 2;               // output rows (the band minus its first / last row)
  static constexpr int INROWS = NB + 2;            // box rows: y = yt0 - 2 .. yt0 + NB - 1
  static constexpr int INBYTES = INROWS * W * (int)sizeof(T);
  static constexpr int INBYTES_AL = (INBYTES + 127) / 128 * 128;
  static constexpr int EROW = W * (int)sizeof(T);  // one published u1 row
  static constexpr int EBYTES = D * NW * 2 * EROW; // edge ring: [slot][warp][first/last][W]
  static constexpr int SMEM = kHeaderX + S * INBYTES_AL + EBYTES;
  static_assert(S * 16 + D * 8 + NW * 8 + 16 <= kHeaderX, "header");
  static_assert(INROWS <= 256, "TMA box height");
};

template <typename T> struct Sweep2XArgs {
  T* out;
  int64_t osy, osz;
  int nx, ny, nz;
  int tiles_x, tiles_y, chunk, nzr, nchunks;
  int col0, row0, pln0;
  int zlo, zhi;      // u1 = OP(u) on planes zlo <= z < zhi (multi-rank: halo planes of rank boundaries)
  int h, glo, ghi;   // ghost planes beyond the halo (plane 0 below, 1 above) when glo / ghi
  int bnd;           // boundary-first chunks (multi-rank)
  unsigned* bflag;
  T* rlo[2];
  T* rhi[2];
  unsigned* rflag_lo;
  unsigned* rflag_hi;
  double* partials;
  unsigned* counter;
  double* result;
};

template <typename T> __device__ __forceinline__ T xshfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T> __device__ __forceinline__ T xshfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <int OP, int RV, typename T, int NW, int S, int D, bool MR>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    sweep2x_tma(const __grid_constant__ Sweep2XArgs<T> a, const __grid_constant__ CUtensorMap map,
                const __grid_constant__ CUtensorMap gmap) {
  using G = GeoX<T, NW, S, D>;
  using O = OpT<OP, T>;
  using Tup = typename O::Tup;
  static_assert(!O::DIAG && O::NCOEF == 0, "7-point single-grid operators only");
  static_assert(RV == RV_NONE || RV == RV_RESID, "plain or residual passes");
  constexpr int V = G::V;
  constexpr int RU = G::RU;

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  uint64_t* ebar = empty + S;                          // edge slot q: every warp published plane q
  double* red = reinterpret_cast<double*>(ebar + D);
  int* flag = reinterpret_cast<int*>(red + NW);
  unsigned char* stages = smem + kHeaderX;
  T* edges = reinterpret_cast<T*>(stages + S * G::INBYTES_AL);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // one unit per CTA: (x tile, y tile, z chunk), x fastest
  int unit = blockIdx.x;
  const int tx = unit % a.tiles_x;
  unit /= a.tiles_x;
  const int ty = unit % a.tiles_y;
  const int zc = unit / a.tiles_y;
  const int xt0 = tx * G::TXO, yt0 = ty * G::TYO;
  int zs, ze;
  if (MR && a.bnd > 0) {
    if (zc < 2) {
      zs = zc == 0 ? 0 : a.nz - a.bnd;
      ze = zs + a.bnd;
    } else {
      zs = a.bnd + (zc - 2) * a.chunk;
      ze = min(zs + a.chunk, a.nz - a.bnd);
    }
  } else {
    zs = zc * a.chunk;
    ze = min(zs + a.chunk, a.nzr);
  }
  const int np = ze - zs + 4;  // input planes zs-2 .. ze+1

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    for (int q = 0; q < D; ++q) mbar_init(&ebar[q], NW);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // ---------------- producer: one TMA box per input plane
    if (lane == 0) {
      tma_prefetch_desc(&map);
      if (MR && (a.glo | a.ghi)) tma_prefetch_desc(&gmap);
      const int xb = a.col0 + xt0 - G::XB, yb = a.row0 + yt0 - 2;
      int s = 0;
      uint32_t ph = 0;
      for (int p = 0; p < np; ++p) {
        if (p >= S) mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], G::INBYTES);
        const int z = zs - 2 + p;
        if (MR && a.glo && z < -a.h)
          tma_load_3d(stages + s * G::INBYTES_AL, &gmap, xb, yb, 0, &full[s]);
        else if (MR && a.ghi && z >= a.nz + a.h)
          tma_load_3d(stages + s * G::INBYTES_AL, &gmap, xb, yb, 1, &full[s]);
        else
          tma_load_3d(stages + s * G::INBYTES_AL, &map, xb, yb, a.pln0 + z, &full[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumers.  Warp w: u1 band rows 4w .. 4w+3 (y = yt0-1+4w+j),
  // input box rows 4w .. 4w+5 (y = yt0-2+4w+r); lane l: x = xs .. xs+V-1.
  const int rb = warp * RU;
  const int xs = xt0 - G::XB + V * lane;
  const int yb1 = yt0 - 1 + rb;  // y of my u1 row 0
  uint32_t in1 = 0;  // bit j*V+k: u1 point (j,k) is an interior (x,y) point
#pragma unroll
  for (int j = 0; j < RU; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (xs + k >= 0 && xs + k < a.nx && yb1 + j >= 0 && yb1 + j < a.ny) in1 |= 1u << (j * V + k);
  constexpr uint32_t kAll1 = (RU * V == 32) ? 0xffffffffu : ((1u << (RU * V)) - 1u);
  const bool warp_int = __all_sync(0xffffffffu, in1 == kAll1);
  uint32_t okm = 0;  // bit j*V+k: output point (j,k) is stored (band rows 1 .. NB-2 only)
  const bool lane_out = lane >= 1 && lane <= 30;
#pragma unroll
  for (int j = 0; j < RU; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int bj = rb + j;
      if (lane_out && bj >= 1 && bj <= G::NB - 2 && xs + k < a.nx && yb1 + j < a.ny) okm |= 1u << (j * V + k);
    }
  const int osy = (int)a.osy;  // (a row pitch fits 32 bits)
  T* optr = a.out + (int64_t)yb1 * a.osy + xs + (int64_t)zs * a.osz;  // (row j: + j * osy)

  double acc[RU];
#pragma unroll
  for (int j = 0; j < RU; ++j) acc[j] = 0.0;

  int s = 0;
  uint32_t ph = 0;
  T nrows[RU + 2][V];
  auto fetch = [&]() {
    mbar_wait(&full[s], ph);
    const T* P = reinterpret_cast<const T*>(stages + s * G::INBYTES_AL) + rb * G::W + V * lane;
#pragma unroll
    for (int r = 0; r < RU + 2; ++r) vload<T>(P + r * G::W, nrows[r]);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  };
  // tuples of rows 1..NR of rows[0..NR+1]; x neighbours by shuffle
  auto tuples = [&](auto& rows, auto& t) {
    constexpr int NR = sizeof(t) / sizeof(t[0]);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const T xl = xshfl_up1(rows[j + 1][V - 1]);
      const T xr = xshfl_dn1(rows[j + 1][0]);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        Nbr<T> n;
        n.c = rows[j + 1][k];
        n.xm = k > 0 ? rows[j + 1][k - 1] : xl;
        n.xp = k < V - 1 ? rows[j + 1][k + 1] : xr;
        n.ym = rows[j][k];
        n.yp = rows[j + 2][k];
        n.h0 = add(n.xm, n.xp);
        t[j][k] = O::plane(n, nullptr);
      }
    }
  };

  // edge ring: the e-th published u1 plane (e = 0: plane zs-1) goes to slot
  // e % D with barrier parity (e / D) & 1 — kept as running slot / parity
  // counters.  Row layout: [slot][warp][first / last][W], lane l at V*l.
  int wr_slot = 0, rd_slot = 0;
  uint32_t wr_par = 0, rd_par = 0;
  constexpr int kSlotElems = NW * 2 * G::W;
  T* const my_first = edges + (warp * 2) * G::W + V * lane;
  const T* const up_last = edges + ((warp - 1) * 2 + 1) * G::W + V * lane;   // warp w-1's last row
  const T* const dn_first = edges + ((warp + 1) * 2) * G::W + V * lane;      // warp w+1's first row
  auto publish = [&](const T (&u1)[RU][V]) {
    vstore<T>(my_first + wr_slot * kSlotElems, u1[0]);
    vstore<T>(my_first + wr_slot * kSlotElems + G::W, u1[RU - 1]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&ebar[wr_slot]);
    if (++wr_slot == D) {
      wr_slot = 0;
      wr_par ^= 1;
    }
  };

  Tup A[RU][V], B[RU][V], C[RU][V];  // sweep-1 tuples of input planes (rotating)
  Tup X[RU][V], Y[RU][V], Z[RU][V];  // sweep-2 tuples of u1 planes (rotating)
  T u1p[RU][V];                      // u1 of the previous step (its tuples are formed one step later)

  // u1(z) on my rows from the sweep-1 tuples of z-1, z, z+1 (Dirichlet rule)
  auto make_u1 = [&](const Tup (&lo)[RU][V], const Tup (&mid)[RU][V], const Tup (&hi)[RU][V], int z,
                     T (&u1)[RU][V]) {
    const bool zin = z >= a.zlo && z < a.zhi;
    if (warp_int && zin) {
#pragma unroll
      for (int j = 0; j < RU; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) u1[j][k] = O::out(lo[j][k], mid[j][k], hi[j][k]);
    } else {
#pragma unroll
      for (int j = 0; j < RU; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k)
          u1[j][k] = (zin && ((in1 >> (j * V + k)) & 1u)) ? O::out(lo[j][k], mid[j][k], hi[j][k]) : mid[j][k].c;
    }
  };
  // second-sweep tuples of the u1 plane published e_rd (my rows u1p; the rows
  // above / below from the neighbouring warps' published rows)
  auto tuples2 = [&](Tup (&t2)[RU][V]) {
    mbar_wait(&ebar[rd_slot], rd_par);
    T rows[RU + 2][V];
    if (warp > 0) vload<T>(up_last + rd_slot * kSlotElems, rows[0]);
    else {
#pragma unroll
      for (int k = 0; k < V; ++k) rows[0][k] = u1p[0][k];  // (row 0 of warp 0 is not an output)
    }
    if (warp < NW - 1) vload<T>(dn_first + rd_slot * kSlotElems, rows[RU + 1]);
    else {
#pragma unroll
      for (int k = 0; k < V; ++k) rows[RU + 1][k] = u1p[RU - 1][k];  // (row 3 of the last warp is not an output)
    }
#pragma unroll
    for (int j = 0; j < RU; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) rows[j + 1][k] = u1p[j][k];
    if (++rd_slot == D) {
      rd_slot = 0;
      rd_par ^= 1;
    }
    tuples(rows, t2);
  };
  auto emit = [&](const Tup (&lo)[RU][V], const Tup (&mid)[RU][V], const Tup (&hi)[RU][V], int zo) {
    T v[RU][V];
#pragma unroll
    for (int j = 0; j < RU; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) v[j][k] = O::out(lo[j][k], mid[j][k], hi[j][k]);
    if constexpr (RV == RV_RESID) {  // the residual of u1 (the second sweep's input) at my stored points
#pragma unroll
      for (int j = 0; j < RU; ++j)
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const double rv = (double)O::resid(lo[j][k], mid[j][k], hi[j][k]);
          acc[j] = __dadd_rn(acc[j], ((okm >> (j * V + k)) & 1u) ? rv : 0.0);
        }
    }
    auto store_rows = [&](T* base) {
#pragma unroll
      for (int j = 0; j < RU; ++j) {
        const uint32_t m = (okm >> (j * V)) & ((1u << V) - 1u);
        if (m == (1u << V) - 1u) {
          vstore<T>(base + j * osy, v[j]);
        } else if (m) {  // (ragged edge tiles only)
#pragma unroll
          for (int k = 0; k < V; ++k)
            if ((m >> k) & 1u) base[j * osy + k] = v[j][k];
        }
      }
    };
    store_rows(optr);
    optr += a.osz;
    if (MR && a.bnd > 0 && zc < 2) {  // boundary plane: also into the neighbour's receiving plane
      T* rp = nullptr;
      if (zc == 0) {
        if (zo < 2) rp = a.rlo[zo];
      } else {
        const int q = a.nz - 1 - zo;
        if (q >= 0 && q < 2) rp = a.rhi[q];
      }
      if (rp) store_rows(rp + (int64_t)yb1 * a.osy + xs);
    }
  };

  // Input plane p is z = zs-2+p.  Step p >= 2: u1(z-1); p >= 3: tuples of
  // u1(z-2); p >= 5: out(z-3).  One drain step after the last input plane.
  fetch();
  tuples(nrows, A);
  fetch();
  tuples(nrows, B);
  fetch();
  int p = 2;
  auto step = [&](Tup (&lo)[RU][V], Tup (&mid)[RU][V], Tup (&hi)[RU][V], Tup (&ulo)[RU][V], Tup (&umid)[RU][V],
                  Tup (&uhi)[RU][V]) {
    // p < np: a new input plane (its rows are in nrows)
    T u1n[RU][V];
    tuples(nrows, hi);
    make_u1(lo, mid, hi, zs - 3 + p, u1n);
    publish(u1n);
    if (p + 1 < np) fetch();
    if (p >= 3) {
      tuples2(uhi);  // of u1(zs-4+p), computed last step
      if (p >= 5) emit(ulo, umid, uhi, zs + p - 5);
    }
#pragma unroll
    for (int j = 0; j < RU; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) u1p[j][k] = u1n[j][k];
    ++p;
  };
  // sweep-1 sets rotate with period 3 (A, B, C); sweep-2 sets with period 3,
  // offset so that uhi of step p is the set of u1(zs-4+p)
  for (; p + 3 <= np;) {
    step(A, B, C, Y, Z, X);
    step(B, C, A, Z, X, Y);
    step(C, A, B, X, Y, Z);
  }
  // tail: at most 2 more input steps, then the drain step (p == np)
  auto drain = [&](Tup (&ulo)[RU][V], Tup (&umid)[RU][V], Tup (&uhi)[RU][V]) {
    tuples2(uhi);
    emit(ulo, umid, uhi, zs + p - 5);
  };
  if (p < np) {
    step(A, B, C, Y, Z, X);
    if (p < np) {
      step(B, C, A, Z, X, Y);
      drain(X, Y, Z);
    } else {
      drain(Z, X, Y);
    }
  } else {
    drain(Y, Z, X);
  }

  if (MR && a.bnd > 0 && zc < 2) {
    named_bar_sync(2, NW * 32);
    if (threadIdx.x == 0) {
      __threadfence();
      if (a.bflag) atomicAdd(a.bflag, 1u);
      unsigned* rf = zc == 0 ? a.rflag_lo : a.rflag_hi;
      if (rf) {
        __threadfence_system();
        atomicAdd_system(rf, 1u);
      }
    }
  }
  if constexpr (RV == RV_RESID) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < RU; ++j) t = __dadd_rn(t, acc[j]);
    cta_reduce_finish(t, CB_SUM, red, flag, NW * 32, a.partials, a.counter, a.result, gridDim.x, blockIdx.x);
  }
}

template <int OP, int RV, typename T, int NW, int S, int D, bool MR>
cudaError_t launch2x_k(const SweepPlan& p, int64_t* launches) {
  using G = GeoX<T, NW, S, D>;
  auto kern = sweep2x_tma<OP, RV, T, NW, S, D, MR>;
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
  Sweep2XArgs<T> a{};
  a.out = static_cast<T*>(p.out.origin);
  a.osy = p.out.pitch;
  a.osz = p.out.plane;
  a.nx = (int)in.nx;
  a.ny = (int)in.ny;
  a.nz = (int)in.nzl;
  a.nzr = (int)in.nzl;
  a.tiles_x = (int)((in.nx + G::TXO - 1) / G::TXO);
  a.tiles_y = (int)((in.ny + G::TYO - 1) / G::TYO);
  a.h = in.h;
  a.zlo = p.phys_lo ? 0 : -1;
  a.zhi = p.phys_hi ? a.nz : a.nz + 1;
  a.glo = (p.ghost && !p.phys_lo && in.h < 2) ? 1 : 0;
  a.ghi = (p.ghost && !p.phys_hi && in.h < 2) ? 1 : 0;
  a.bnd = (p.bnd_h > 0 && a.nz >= 6) ? 2 : 0;
  if (a.bnd) a.nzr = a.nz - 2 * a.bnd;
  const int64_t tiles = (int64_t)a.tiles_x * a.tiles_y;
  const int64_t slots = (int64_t)occ * p.num_sms;
  int best = 1;
  double best_cost = 1e300;
  for (int c = 1; c <= a.nzr; ++c) {
    const int64_t chunk = (a.nzr + c - 1) / c;
    const int64_t cc = (a.nzr + chunk - 1) / chunk;
    const int64_t waves = (tiles * cc + slots - 1) / slots;
    const double cost = (double)waves * (double)(chunk + 5);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = (int)cc;
    }
  }
  int chunks = best;
  if (p.zchunks > 0) chunks = (int)std::min<int64_t>(p.zchunks, a.nzr);
  a.chunk = (a.nzr + chunks - 1) / chunks;
  chunks = (a.nzr + a.chunk - 1) / a.chunk;
  if (a.bnd) {
    chunks += 2;
    a.bflag = p.bflag;
    for (int i = 0; i < 2; ++i) {
      a.rlo[i] = static_cast<T*>(p.peer_lo[i]);
      a.rhi[i] = static_cast<T*>(p.peer_hi[i]);
    }
    a.rflag_lo = p.peer_flag_lo;
    a.rflag_hi = p.peer_flag_hi;
    if (p.bnd_units) *p.bnd_units = 2 * tiles;
  } else if (p.bnd_units) {
    *p.bnd_units = 0;
  }
  a.col0 = (int)in.ox;
  a.row0 = in.h;
  a.pln0 = in.h;
  a.partials = p.red.partials;
  a.counter = p.red.counter;
  a.result = p.red.result;
  CUtensorMap map, gmap;
  if (!encode_tma_3d(&map, in, G::W, G::INROWS, p.l2promo)) return cudaErrorInvalidValue;
  gmap = map;
  if (a.glo | a.ghi) {
    View gv = in;
    gv.base = const_cast<void*>(p.ghost);
    gv.h = 1;
    gv.nzl = 0;
    gv.ny = in.ny + 2 * in.h - 2;
    if (!encode_tma_3d(&gmap, gv, G::W, G::INROWS, p.l2promo)) return cudaErrorInvalidValue;
  }
  a.nchunks = chunks;
  const int64_t units = tiles * chunks;
  if (RV != RV_NONE && units > p.red.max_partials) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)units, NT, G::SMEM, p.stream>>>(a, map, gmap);
  ++*launches;
  return cudaGetLastError();
}

template <int RV, typename T, int NW, int S, int D>
cudaError_t launch2x_mr(const SweepPlan& p, int64_t* launches) {
  const bool mr = p.bnd_h > 0 || !p.phys_lo || !p.phys_hi || p.ghost || p.peer_lo[0] || p.peer_lo[1] ||
                  p.peer_hi[0] || p.peer_hi[1];
  return mr ? launch2x_k<OP_JACOBI7, RV, T, NW, S, D, true>(p, launches)
            : launch2x_k<OP_JACOBI7, RV, T, NW, S, D, false>(p, launches);
}

}  // namespace

// Geometry: 7 consumer warps x 4 u1 rows (26 output rows), a producer warp,
// an 8-stage TMA ring and a 12-slot edge ring (fp64: 60 x 26 output tile).
#define GSCL_PASSX_DEFAULT 7, 8, 12

int64_t pass_tiles_x(int64_t nx, int64_t ny, int dtype) {
  if (dtype == 0) {
    using G = GeoX<double, 7, 8, 12>;
    return ((nx + G::TXO - 1) / G::TXO) * ((ny + G::TYO - 1) / G::TYO);
  }
  using G = GeoX<float, 7, 8, 12>;
  return ((nx + G::TXO - 1) / G::TXO) * ((ny + G::TYO - 1) / G::TYO);
}

cudaError_t launch_sweep2x(const SweepPlan& p, int64_t* launches) {
  if (p.op != OP_JACOBI7 || p.rbgs || (p.rv != RV_NONE && p.rv != RV_RESID)) return cudaErrorInvalidValue;
  const bool f64 = p.in[0].dtype == 0;
  if (p.rv == RV_RESID)
    return f64 ? launch2x_mr<RV_RESID, double, GSCL_PASSX_DEFAULT>(p, launches)
               : launch2x_mr<RV_RESID, float, GSCL_PASSX_DEFAULT>(p, launches);
  return f64 ? launch2x_mr<RV_NONE, double, GSCL_PASSX_DEFAULT>(p, launches)
             : launch2x_mr<RV_NONE, float, GSCL_PASSX_DEFAULT>(p, launches);
}

#endif  // GSCL_ABLATIONS

}  // namespace gscl
