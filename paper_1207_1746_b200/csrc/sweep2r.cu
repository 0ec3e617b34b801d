// sweep2r.cu — two Jacobi sweeps per HBM pass with the intermediate iterate
// kept in registers (temporal blocking; "wide ghost
// areas").
//
// out = OP(OP(u)) for the 7-point operators with the Dirichlet rule of
// gscl_jacobi_run: halo cells are boundary values and are never updated, so the
// intermediate iterate u1 equals u outside the interior.  Both sweeps evaluate
// the per-plane tuples of ops.cuh, so the result is bitwise the result of two
// single sweeps.
//
// Why a second design (sweep2.cu is the first): there, u1 went through a
// shared-memory ring so that every warp could read its y neighbours, which cost
// a CTA-wide named barrier per plane, 4-way bank-conflicted x-neighbour loads
// and, at 96 registers, local-memory spills (ncu: L1/TEX 85 %, 0.59 ms per
// 512^3 pass).  Here each warp is independent: a lane owns V consecutive x
// points (one 16-byte vector) of R output rows, computes u1 on the R + 2 rows
// around them itself (the y neighbours of u1 are then its own registers), and
// takes every x neighbour — of u and of u1 — from the adjacent lane by warp
// shuffle.  Shared memory holds only the TMA-staged input planes, read once per
// lane row with conflict-free 16-byte loads; the only CTA-level coupling is the
// stage ring (mbarriers), which lets warps drift apart by up to S planes.
//
// Tile (fp64, V = 2): a warp spans 32V = 64 x-columns (2 halo columns each
// side: output lanes 1..30 = 60 points), R output rows, R + 2 u1 rows, R + 4
// input rows; NW warps stack in y, so a CTA outputs 60 x NW*R from a
// 64 x (NW*R + 4) TMA box per plane.  A unit = (tile, z-chunk); the chunk
// [zs, ze) reads input planes zs-2 .. ze+1.
#include <algorithm>
#include <type_traits>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

GSCL_MODULE_ANCHOR(anchor_sweep2r)


namespace {

constexpr int kHeaderR = 1024;  // barriers + reduction scratch

// V = points per lane: one 16-byte vector (Vec<T>::N) or, for fp64, one
// point (V = 1: half the per-lane tuple state, so two CTAs fit per SM).
// WP: warp-private rings — each consumer warp streams its own (R + 4)-row box
// per plane into S stages of its own and refills a stage itself as soon as it
// has read it (no producer warp, no cross-warp release barrier).
template <typename T, int V_, int NW, int R, int S, bool WP = false> struct GeoR {
  static constexpr int V = V_;
  static constexpr int W = 32 * V;                 // box width = warp strip width
  static constexpr int XB = V == 1 ? 2 : V;        // box columns left of the tile (>= 2)
  static constexpr int TXO = W - 2 * XB;           // output tile width (V = 2: lanes 1..30, V = 1: 2..29)
  static constexpr int LO0 = XB / V, LO1 = (W - XB) / V;  // output lanes [LO0, LO1)
  static constexpr int TYO = NW * R;               // output tile height
  static constexpr int INROWS = WP ? R + 4 : TYO + 4;  // rows of one TMA box
  static constexpr int INBYTES = INROWS * W * (int)sizeof(T);
  static constexpr int INBYTES_AL = (INBYTES + 127) / 128 * 128;
  static constexpr int NSTAGE = WP ? NW * S : S;
  static constexpr int SMEM = kHeaderR + NSTAGE * INBYTES_AL;
  static_assert(NSTAGE * 8 + NW * 8 + 8 + S * 4 <= kHeaderR, "header");
  static_assert(INROWS <= 256, "TMA box height");
  static_assert((R + 2) * V <= 32 && R * V <= 32, "row masks are 32-bit");
};

template <typename T> struct Sweep2RArgs {
  T* out;
  int64_t osy, osz;
  int nx, ny, nz;          // local interior extents (u1 halo rule)
  int tiles_x, tiles_y, chunk, nzr, nchunks;
  int col0, row0, pln0;    // array coords of interior (0,0,0) of u
  // z-slab of several ranks: the u1 Dirichlet rule applies only at physical
  // z boundaries (u1 IS computed on the halo planes -1 / nz of a rank boundary)
  int zlo, zhi;            // u1 = OP(u) on planes zlo <= z < zhi (0, nz on one rank)
  // planes beyond the grid's halo (z < -h or z >= nz + h) come from the ghost
  // buffer's map (plane 0 below, plane 1 above) when glo / ghi are set
  int h, glo, ghi;
  // boundary-first (multi-rank overlap): units of z-chunk 0 / 1 are the bnd
  // output planes at each end; each bumps *bflag after its stores
  int bnd;
  unsigned* bflag;
  // peer-memory halo transport (multi-rank, NVLink P2P): the boundary units
  // also store output planes 0, 1 into the lower neighbour's receiving planes
  // rlo[0], rlo[1] (its planes nzl, nzl+1) and planes nzl-1, nzl-2 into the
  // upper neighbour's rhi[0], rhi[1] (its planes -1, -2); each pointer is the
  // interior origin (x = 0, y = 0) of that plane, same pitch as `out`.  After
  // its stores a unit bumps the neighbour's arrival counter (system scope).
  T* rlo[2];
  T* rhi[2];
  unsigned* rflag_lo;
  unsigned* rflag_hi;
  double* partials;
  unsigned* counter;
  double* result;
  // RV_CONV2: the second iteration's AND goes to partials2 / counter2 / result2
  double* partials2;
  unsigned* counter2;
  double* result2;
  double eps;
  const int* stop;  // if non-null and set: the pass is skipped (converged loop)
  int zpar;         // RB: parity of the global z of local plane 0
  // DYN: units claimed in increasing order from *ticket; the last CTA's
  // producer resets ticket[0] and ticket[1] (the exit count) to 0
  unsigned* ticket;
  int slots;  // resident CTAs (occupancy x SMs): the unit a CTA's SM runs next is ~ blockIdx.x + slots
  // reductions of a pass split into two launches (boundary chunks, middle
  // chunks): this launch's CTAs write partials[unit0 + blockIdx.x] and the
  // last of all nparts CTAs (both launches share the counter) folds them all
  int unit0, nparts;
};

template <typename T> __device__ __forceinline__ T shfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T> __device__ __forceinline__ T shfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// Tuples of `NR` consecutive rows (rows 1..NR of rows[0..NR+1]) of a lane's V
// points, x neighbours from the adjacent lanes.  Lanes 0 / 31 receive their
// own edge value, which only feeds points whose results are never used.
template <int OP, typename T, int NR, int V>
__device__ __forceinline__ void row_tuples(const T (&rows)[NR + 2][V], typename OpT<OP, T>::Tup (&t)[NR][V]) {
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const T xl = shfl_up1(rows[j + 1][V - 1]);
    const T xr = shfl_dn1(rows[j + 1][0]);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      Nbr<T> n;
      n.c = rows[j + 1][k];
      n.xm = k > 0 ? rows[j + 1][k - 1] : xl;
      n.xp = k < V - 1 ? rows[j + 1][k + 1] : xr;
      n.ym = rows[j][k];
      n.yp = rows[j + 2][k];
      n.h0 = add(n.xm, n.xp);
      t[j][k] = OpT<OP, T>::plane(n, nullptr);
    }
  }
}

// The same tuples computed in place: t[j][k].c already holds row j + 1 of the
// staged rows (the fetch loaded it there), e[0] / e[1] rows 0 / NR + 1.
// plane() keeps c, so the y neighbours read from t are still the loaded rows.
template <int OP, typename T, int NR, int V>
__device__ __forceinline__ void row_tuples_inplace(typename OpT<OP, T>::Tup (&t)[NR][V], const T (&e)[2][V]) {
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    const T xl = shfl_up1(t[j][V - 1].c);
    const T xr = shfl_dn1(t[j][0].c);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      Nbr<T> n;
      n.c = t[j][k].c;
      n.xm = k > 0 ? t[j][k - 1].c : xl;
      n.xp = k < V - 1 ? t[j][k + 1].c : xr;
      n.ym = j > 0 ? t[j - 1][k].c : e[0][k];
      n.yp = j < NR - 1 ? t[j + 1][k].c : e[1][k];
      n.h0 = add(n.xm, n.xp);
      t[j][k] = OpT<OP, T>::plane(n, nullptr);
    }
  }
}

// One CTA = NW consumer warps + one producer warp (lane 0 issues one TMA box
// per input plane into an S-stage ring; consumers release a stage through its
// "empty" mbarrier); one unit (x tile, y tile, z chunk) per CTA.  The units in
// flight at any time are consecutive in (x tile, y tile, z chunk) order, so
// x/y-neighbour tiles that share halo rows are read together and their shared
// bytes come from L2.  (Ablations — persistent CTAs, a producer-less ring,
// centre values re-read from the ring, suspend-hinted waits, shared-memory x
// neighbours — were all slower or no better: profiles/r01_sweep2r.md.)
// RB: red-black Gauss-Seidel iteration as one pass (NEXT-3): the first sweep
// updates only the red points ((x + y + z) even, global coordinates), the
// second only the black ones from the updated field — each a colour-masked
// Jacobi step, which is exactly the in-place half-sweep order.
// MR: the multi-rank features (boundary-first chunks + arrival counter, ghost
// map, peer stores); a single-rank launch compiles them out.
// MINB == 0 (ablation): a warpgroup of 4 producer warps (one issues the TMA
// boxes) hands its registers to the NW consumer warps with setmaxnreg.
// MINB == -1: no producer warp — lane 0 of consumer warp 0 issues the TMA
// boxes itself (the "inline producer": 8 consumer warps = 2 per scheduler,
// where 7 consumers + a producer warp leave one scheduler with 1 consumer).
template <int NW, int MINB, bool WP = false> struct ThreadsR {
  static constexpr int PW = (WP || MINB == -1) ? 0 : MINB == 0 ? 4 : 1;
  static constexpr int NT = 32 * (NW + PW);
  static constexpr int MB = MINB <= 0 ? 1 : MINB;
};

// DBG (ablation probes only, 0 in every product instantiation; 1-4 use the round-1 step order): 1 = memory only
// (the ring and the stores, no arithmetic), 2 = compute only (no TMA, no ring
// waits), 3 = stage release without the proxy fence, 4 = Dirichlet select
// skipped.
// DYN: persistent CTAs (one per SM slot) with dynamic unit claiming — the
// producer claims units in increasing order from a global ticket and streams
// their planes through ONE continuous ring, writing each unit's id into the
// header slot of the unit's first stage; consumers read it there.  The ring
// never drains between units (the startup of a non-persistent CTA — an empty
// ring, ~2 us before its first plane lands — recurs ~7 times per SM per pass),
// and the claim order keeps the units in flight a contiguous window as the
// hardware's wave order does.  Residual partials are per UNIT, folded in unit
// order: the result does not depend on which CTA ran which unit.
template <int OP, int RV, typename T, int V_, int NW, int R, int S, int MINB, bool WP, bool RB = false,
          bool MR = false, int DBG = 0, bool DYN = false>
__global__ void __launch_bounds__(ThreadsR<NW, MINB, WP>::NT, ThreadsR<NW, MINB, WP>::MB)
    sweep2r_tma(const __grid_constant__ Sweep2RArgs<T> a, const __grid_constant__ CUtensorMap map,
                const __grid_constant__ CUtensorMap gmap) {
  static_assert(!DYN || (!WP && !RB && (RV == RV_NONE || RV == RV_RESID)), "DYN: plain / residual passes");
  constexpr bool IP = MINB == -1;  // inline producer (see ThreadsR)
  static_assert(!IP || (!WP && !DYN), "inline producer: plain ring");
  using G = GeoR<T, V_, NW, R, S, WP>;
  using O = OpT<OP, T>;
  using Tup = typename O::Tup;
  static_assert(!O::DIAG && O::NCOEF == 0, "7-point single-grid operators only");
  constexpr int V = G::V;
  constexpr int R1 = R + 2;  // u1 rows per lane

  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + G::NSTAGE;
  double* red = reinterpret_cast<double*>(empty + (WP ? 0 : S));
  int* flag = reinterpret_cast<int*>(red + NW);
  int* unit_of = flag + 2;  // DYN: unit id of the unit whose first plane is in stage s (-1: no more)
  unsigned char* stages = smem + kHeaderR;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int units = a.tiles_x * a.tiles_y * a.nchunks;
  const int ustep = units;  // one unit per CTA
  struct Unit { int xt0, yt0, zs, np, zc; };
  auto decode = [&](int u) {
    Unit d;
    const int tx = u % a.tiles_x;
    u /= a.tiles_x;
    const int ty = u % a.tiles_y;
    const int zc = u / a.tiles_y;
    d.xt0 = tx * G::TXO;
    d.yt0 = ty * G::TYO;
    d.zc = zc;
    int ze;
    if (MR && a.bnd > 0) {  // boundary-first: [0, chunk), [nz - chunk, nz), then [chunk, nz - chunk)
      if (zc == 0) {
        d.zs = 0;
        ze = a.chunk;
      } else if (zc == 1) {
        d.zs = a.nz - a.chunk;
        ze = a.nz;
      } else {
        d.zs = a.chunk + (zc - 2) * a.chunk;
        ze = min(d.zs + a.chunk, a.nz - a.chunk);
      }
    } else {
      d.zs = zc * a.chunk;
      ze = min(d.zs + a.chunk, a.nzr);
    }
    d.np = ze - d.zs + 4;  // input planes zs-2 .. ze+1
    return d;
  };

  // Consumer warps whose output rows all lie below the grid (the last tile
  // row: 512 rows in 28-row tiles leave 5 of its 7 warps outside) take no part
  // in the ring — the stages' release count is the number of warps that do —
  // and go straight to the epilogue, leaving the SM's issue slots to the
  // others.  (Single-rank, one unit per CTA, shared ring only: the multi-rank
  // boundary publishing needs every warp at its barrier.)
  constexpr bool kIdleOut = !MR && !DYN && !WP && !IP;
  int nact = NW;
  if constexpr (kIdleOut) {
    const int yt0 = ((int)blockIdx.x / a.tiles_x % a.tiles_y) * G::TYO;
    nact = min(NW, max(1, (a.ny - yt0 + R - 1) / R));
  }
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    s_stop = a.stop ? *(volatile const int*)a.stop : 0;
    for (int s = 0; s < G::NSTAGE; ++s) mbar_init(&full[s], 1);
    if constexpr (!WP)
      for (int s = 0; s < S; ++s) mbar_init(&empty[s], nact);
    fence_mbar_init();
  }
  __syncthreads();
  if (s_stop) return;  // (uniform: the whole CTA leaves)

  if (!WP && warp >= NW) {  // ---------------- producer: one TMA box per input plane
    if constexpr (MINB == 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
    if (warp == NW && lane == 0 && DBG != 2) {
      tma_prefetch_desc(&map);
      if (a.glo | a.ghi) tma_prefetch_desc(&gmap);
      int s = 0, issued = 0;
      uint32_t ph = 0;
      for (int u = DYN ? (int)atomicAdd(a.ticket, 1u) : (int)blockIdx.x; u < units;
           u = DYN ? (int)atomicAdd(a.ticket, 1u) : u + ustep) {
        const Unit d = decode(u);
        const int xb = a.col0 + d.xt0 - G::XB, yb = a.row0 + d.yt0 - 2, zb = a.pln0 + d.zs - 2;
        for (int p = 0; p < d.np; ++p, ++issued) {
          if (issued >= S) mbar_wait(&empty[s], ph ^ 1);
          if (DYN && p == 0) unit_of[s] = u;  // (visible to the consumers through the stage's barrier)
          mbar_arrive_expect_tx(&full[s], G::INBYTES);
          const int z = d.zs - 2 + p;  // local interior z of the plane
          if (MR && a.glo && z < -a.h)
            tma_load_3d(stages + s * G::INBYTES_AL, &gmap, xb, yb, 0, &full[s]);
          else if (MR && a.ghi && z >= a.nz + a.h)
            tma_load_3d(stages + s * G::INBYTES_AL, &gmap, xb, yb, 1, &full[s]);
          else
            tma_load_3d(stages + s * G::INBYTES_AL, &map, xb, yb, zb + p, &full[s]);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      if constexpr (DBG == 8 && !DYN && !WP) {
        // all planes of this unit issued (~S planes before the CTA ends): warm
        // L2 with the first planes of the unit the next wave starts about now
        // on some SM (one unit per CTA, launched in index order), so that
        // CTA's ring does not start on a cold HBM latency
        const int un = (int)blockIdx.x + a.slots;
        if (un < units) {
          const Unit dn = decode(un);
          const int xbn = a.col0 + dn.xt0 - G::XB, ybn = a.row0 + dn.yt0 - 2, zbn = a.pln0 + dn.zs - 2;
          for (int q = 0; q < 4 && q < dn.np; ++q)
            if (!(MR && ((a.glo && dn.zs - 2 + q < -a.h) || (a.ghi && dn.zs - 2 + q >= a.nz + a.h))))
              tma_prefetch_l2_3d(&map, xbn, ybn, zbn + q);
        }
      }
      if constexpr (DYN) {
        // no more units: a sentinel stage (no data) tells the consumers to stop
        if (issued >= S) mbar_wait(&empty[s], ph ^ 1);
        unit_of[s] = -1;
        mbar_arrive(&full[s]);
        // the last producer to finish claiming resets the ticket for the next launch
        if (atomicAdd(a.ticket + 1, 1u) == gridDim.x - 1) {
          atomicExch(a.ticket, 0u);
          atomicExch(a.ticket + 1, 0u);
        }
      }
    }
    return;
  }

  if constexpr (MINB == 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 240;" ::: "memory");
  // ---------------- consumers.  Lane l owns x = xs .. xs+V-1; warp w's input
  // rows are box rows rb .. rb+R+3 (y = yt0-2+rb+r), its u1 rows j = 0..R+1
  // are y = yt0-1+rb+j, its output rows i = 0..R-1 are y = yt0+rb+i.
  const int rb = warp * R;
  constexpr uint32_t kAll1 = (R1 * V == 32) ? 0xffffffffu : ((1u << (R1 * V)) - 1u);
  constexpr uint32_t kAllO = (R * V == 32) ? 0xffffffffu : ((1u << (R * V)) - 1u);
  double acc[R];            // RESID: one running sum per output row (no long serial chain)
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = 0.0;
  unsigned ok1 = 1u, ok2 = 1u;  // CONV2: ANDs of iterations 1 and 2 (integer: no FP dependency chain)
  const T eps = (T)a.eps;
  int s = 0;
  uint32_t ph = 0;

  auto next_unit = [&](int u) -> int {  // DYN: the id in the header of the next stage
    if constexpr (DYN) {
      mbar_wait(&full[s], ph);
      // (broadcast from lane 0: lets the compiler treat the unit — and its
      // loop bounds — as warp-uniform, as it does for blockIdx.x)
      return __shfl_sync(0xffffffffu, unit_of[s], 0);
    } else {
      return u;
    }
  };
  for (int u = next_unit(blockIdx.x); (DYN ? u >= 0 : u < units) && warp < nact; u = next_unit(u + ustep)) {
    const Unit d = decode(u);
    const int zs = d.zs, np = d.np;
    const int xs = d.xt0 - G::XB + V * lane;
    const int yo = d.yt0 + rb;
    uint32_t in1 = 0;  // bit j*V+k: u1 point (j,k) is an interior (x,y) point
#pragma unroll
    for (int j = 0; j < R1; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (xs + k >= 0 && xs + k < a.nx && yo - 1 + j >= 0 && yo - 1 + j < a.ny) in1 |= 1u << (j * V + k);
    uint32_t okm = 0;  // bit i*V+k: output point (i,k) is stored
    const bool lane_out = lane >= G::LO0 && lane < G::LO1;
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (lane_out && xs + k < a.nx && yo + i < a.ny) okm |= 1u << (i * V + k);
    // all stored (lanes 1..30 of interior tiles) -> 16-byte stores; lanes 0 / 31
    // store nothing, so the per-element path runs only on ragged edge tiles
    const bool fast = okm == kAllO;
    // every u1 point of the warp is an interior (x, y) point: the Dirichlet
    // select is skipped (warp-uniform branch) on planes inside the slab
    const bool warp_int = DBG == 4 || __all_sync(0xffffffffu, in1 == kAll1);
    T* optr = a.out + (int64_t)yo * a.osy + xs + (int64_t)zs * a.osz;

    // WP: lane 0 streams the warp's own box (input rows yo-2 .. yo+R+1) of
    // plane p of the unit into ring slot `st` of the warp
    int ld = 0;  // planes of this unit read so far
    auto issue_wp = [&](int p, int st) {
      const int xb = a.col0 + d.xt0 - G::XB, yb = a.row0 + yo - 2;
      uint64_t* bar = &full[warp * S + st];
      unsigned char* dst = stages + (warp * S + st) * G::INBYTES_AL;
      mbar_arrive_expect_tx(bar, G::INBYTES);
      const int z = zs - 2 + p;  // local interior z of the plane
      if (MR && a.glo && z < -a.h)
        tma_load_3d(dst, &gmap, xb, yb, 0, bar);
      else if (MR && a.ghi && z >= a.nz + a.h)
        tma_load_3d(dst, &gmap, xb, yb, 1, bar);
      else
        tma_load_3d(dst, &map, xb, yb, a.pln0 + z, bar);
    };
    if constexpr (WP) {
      if (lane == 0) {
        int st = s;
        for (int p = 0; p < S && p < np; ++p) {
          issue_wp(p, st);
          if (++st == S) st = 0;
        }
      }
    }

    // sweep-1 tuples of the next input plane (u1 rows), from the staged box
    auto load_in = [&](Tup (&t)[R1][V]) {
      T rows[R + 4][V];
      if constexpr (WP) {
        mbar_wait(&full[warp * S + s], ph);
        const T* P = reinterpret_cast<const T*>(stages + (warp * S + s) * G::INBYTES_AL) + V * lane;
#pragma unroll
        for (int r = 0; r < R + 4; ++r) vload<T>(P + r * G::W, rows[r]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && ld + S < np) issue_wp(ld + S, s);
        ++ld;
      } else {
        if (DBG != 2) mbar_wait(&full[s], ph);
        const T* P = reinterpret_cast<const T*>(stages + s * G::INBYTES_AL) + rb * G::W + V * lane;
#pragma unroll
        for (int r = 0; r < R + 4; ++r) vload<T>(P + r * G::W, rows[r]);
        if (DBG != 3) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && DBG != 2) mbar_arrive(&empty[s]);
      }
      if (DBG == 1) {
        if (ld >= 4) {
#pragma unroll
          for (int i = 0; i < R; ++i) vstore<T>(optr + (int64_t)i * a.osy, rows[i + 2]);
          optr += a.osz;
        }
        ++ld;
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
        return;
      }
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
      row_tuples<OP, T, R1, V>(rows, t);
    };
    // u1 plane z from the tuples of z-1, z, z+1; then its sweep-2 tuples
    auto make_u1 = [&](const Tup (&lo)[R1][V], const Tup (&mid)[R1][V], const Tup (&hi)[R1][V], int z,
                       Tup (&t2)[R][V]) {
      const bool zin = z >= a.zlo && z < a.zhi;
      T u1[R1][V];
      if constexpr (RB) {  // red points only: parity of (x + y + z) even
        const int b0 = (xs + (yo - 1) + z + a.zpar) & 1;
#pragma unroll
        for (int j = 0; j < R1; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const bool red = ((b0 + j + k) & 1) == 0;
            u1[j][k] = (red && zin && ((in1 >> (j * V + k)) & 1u)) ? O::out(lo[j][k], mid[j][k], hi[j][k])
                                                                   : mid[j][k].c;
          }
      } else if (warp_int && zin) {
#pragma unroll
        for (int j = 0; j < R1; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k) u1[j][k] = O::out(lo[j][k], mid[j][k], hi[j][k]);
      } else {
#pragma unroll
        for (int j = 0; j < R1; ++j)
#pragma unroll
          for (int k = 0; k < V; ++k)
            u1[j][k] = (zin && ((in1 >> (j * V + k)) & 1u)) ? O::out(lo[j][k], mid[j][k], hi[j][k])
                                                            : mid[j][k].c;
      }
      if constexpr (RV == RV_RESID_IN) {  // RESID7^2 of the input at my output points
        if (z >= zs && z < zs + np - 4) {
#pragma unroll
          for (int i = 0; i < R; ++i)
#pragma unroll
            for (int k = 0; k < V; ++k) {
              const double rv = (double)O::resid(lo[i + 1][k], mid[i + 1][k], hi[i + 1][k]);
              acc[i] = __dadd_rn(acc[i], ((okm >> (i * V + k)) & 1u) ? rv : 0.0);
            }
        }
      }
      if constexpr (RV == RV_CONV2) {
        // iteration 1 of the pass converged at my output points of this plane?
        if (z >= zs && z < zs + np - 4) {
#pragma unroll
          for (int i = 0; i < R; ++i)
#pragma unroll
            for (int k = 0; k < V; ++k)
              ok1 &= (((okm >> (i * V + k)) & 1u) == 0u) |
                     (unsigned)(fabs(sub(u1[i + 1][k], mid[i + 1][k].c)) <= eps);
        }
      }
      row_tuples<OP, T, R, V>(u1, t2);
    };
    auto emit = [&](const Tup (&lo)[R][V], const Tup (&mid)[R][V], const Tup (&hi)[R][V], int zo) {
      T v[R][V];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int k = 0; k < V; ++k) v[i][k] = O::out(lo[i][k], mid[i][k], hi[i][k]);
      if constexpr (RB) {  // black points only; red ones keep the first sweep's value
        const int b0 = (xs + yo + zo + a.zpar) & 1;
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
          for (int k = 0; k < V; ++k)
            if (((b0 + i + k) & 1) == 0) v[i][k] = mid[i][k].c;
      }
      if constexpr (RV == RV_CONV2) {  // iteration 2: |u2 - u1| <= eps
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
          for (int k = 0; k < V; ++k)
            ok2 &= (((okm >> (i * V + k)) & 1u) == 0u) | (unsigned)(fabs(sub(v[i][k], mid[i][k].c)) <= eps);
      }
      if constexpr (RV == RV_RESID) {
        // residual of u1 (the input of the second sweep) at the stored points,
        // one fixed fold order per lane
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const double rv = (double)O::resid(lo[i][k], mid[i][k], hi[i][k]);
            acc[i] = __dadd_rn(acc[i], ((okm >> (i * V + k)) & 1u) ? rv : 0.0);
          }
      }
      if (fast) {
#pragma unroll
        for (int i = 0; i < R; ++i) vstore<T>(optr + (int64_t)i * a.osy, v[i]);
      } else if (okm) {
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
          for (int k = 0; k < V; ++k)
            if ((okm >> (i * V + k)) & 1u) optr[(int64_t)i * a.osy + k] = v[i][k];
      }
      optr += a.osz;
      if (MR && a.bnd > 0 && d.zc < 2) {  // boundary plane: also into the neighbour's receiving plane
        T* rp = nullptr;
        if (d.zc == 0) {
          if (zo < 2) rp = a.rlo[zo];
        } else {
          const int q = a.nz - 1 - zo;
          if (q >= 0 && q < 2) rp = a.rhi[q];
        }
        if (rp) {
          rp += (int64_t)yo * a.osy + xs;
          if (fast) {
#pragma unroll
            for (int i = 0; i < R; ++i) vstore<T>(rp + (int64_t)i * a.osy, v[i]);
          } else if (okm) {
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
              for (int k = 0; k < V; ++k)
                if ((okm >> (i * V + k)) & 1u) rp[(int64_t)i * a.osy + k] = v[i][k];
          }
        }
      }
    };

    // Input plane p is z = zs-2+p.  After input p (p >= 2): u1(zs-3+p) and its
    // sweep-2 tuples; with three of those (p >= 4): out(zs+p-4).
    Tup A[R1][V], B[R1][V], C[R1][V];  // sweep-1 tuples (input planes)
    Tup X[R][V], Y[R][V], Z[R][V];     // sweep-2 tuples (u1 planes)
    // Software-pipelined steps (the default; DBG 7 = the round-1 order): the
    // next plane's rows are fetched (ring wait + shared loads + stage release)
    // before this plane's second-sweep output is formed, so the loads overlap
    // the output's arithmetic instead of queueing behind the ring-wait loop (a
    // basic-block boundary the scheduler does not cross).  0.3868 -> 0.3836 ms
    // per 512^3 pass (r02).  DBG 6 = the same without the proxy fence (probe).
    // (fp64 only, not the two-test convergence pass: with the prefetched rows
    // live across the output those instantiations spill at 255 registers)
    constexpr bool kPF = !WP && sizeof(T) == 8 && RV != RV_CONV2 && (DBG == 0 || DBG == 5 || DBG == 6 || DBG == 8);
    static_assert(!IP || kPF, "inline producer: software-pipelined steps");
    // (software-pipelined steps: the next plane's rows 1 .. R + 2 are loaded
    // straight into the c fields of the tuple set that becomes `hi` — the
    // current `lo`, dead once u1 is formed — and rows 0 / R + 3 into nedge, so
    // no row is copied between registers afterwards)
    T nedge[2][V];
    // IP: lane 0 of warp 0 issues plane q into stage q % S (one unit per CTA,
    // the ring starts at stage 0); plane q >= S needs use q/S - 1 of the stage
    // released by every warp.  Before warp 0 waits for a plane it has not
    // issued it blocks on that release (the other warps only need planes
    // already issued, so they get there); after each of its own releases it
    // issues every further plane whose stage is free, without blocking.
    int nq = 0;  // IP: planes issued
    const int xb_ip = a.col0 + d.xt0 - G::XB, yb_ip = a.row0 + d.yt0 - 2;
    auto issue_ip = [&](int q) {
      const int st = q % S;
      mbar_arrive_expect_tx(&full[st], G::INBYTES);
      const int z = zs - 2 + q;
      if (MR && a.glo && z < -a.h)
        tma_load_3d(stages + st * G::INBYTES_AL, &gmap, xb_ip, yb_ip, 0, &full[st]);
      else if (MR && a.ghi && z >= a.nz + a.h)
        tma_load_3d(stages + st * G::INBYTES_AL, &gmap, xb_ip, yb_ip, 1, &full[st]);
      else
        tma_load_3d(stages + st * G::INBYTES_AL, &map, xb_ip, yb_ip, a.pln0 + z, &full[st]);
    };
    int q_next = 0;  // IP: the plane this warp fetches next
    if constexpr (IP) {
      if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&map);
        if (MR && (a.glo | a.ghi)) tma_prefetch_desc(&gmap);
        for (; nq < S && nq < np; ++nq) issue_ip(nq);
      }
    }
    auto fetch = [&](Tup (&t)[R1][V]) {
      if constexpr (IP) {
        if (warp == 0 && lane == 0) {
          for (; nq <= q_next && nq < np; ++nq) {  // must not wait for a plane nobody issued
            mbar_wait(&empty[nq % S], ((nq / S) - 1) & 1);
            issue_ip(nq);
          }
        }
        ++q_next;
      }
      mbar_wait(&full[s], ph);
      const T* P = reinterpret_cast<const T*>(stages + s * G::INBYTES_AL) + rb * G::W + V * lane;
      vload<T>(P, nedge[0]);
#pragma unroll
      for (int j = 0; j < R1; ++j) {
        T w[V];
        vload<T>(P + (j + 1) * G::W, w);
#pragma unroll
        for (int k = 0; k < V; ++k) t[j][k].c = w[k];
      }
      vload<T>(P + (R + 3) * G::W, nedge[1]);
      if (DBG != 6) fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == S) {
        s = 0;
        ph ^= 1;
      }
      if constexpr (IP) {
        if (warp == 0 && lane == 0)
          while (nq < np && mbar_test(&empty[nq % S], ((nq / S) - 1) & 1)) issue_ip(nq++);
      }
    };
    if constexpr (kPF) {
      fetch(A);
      row_tuples_inplace<OP, T, R1, V>(A, nedge);
      fetch(B);
      row_tuples_inplace<OP, T, R1, V>(B, nedge);
      fetch(C);
    } else {
      load_in(A);
      load_in(B);
    }
    int p = 2;
    // boundary-first units publish the slab's boundary planes (the comm
    // stream waits on bflag before the NCCL exchange; the peer transport's
    // neighbour waits on its counter): the first chunk after its second
    // output (planes 0, 1 — mid-unit), the last chunk at its end
    auto publish = [&]() {
      named_bar_sync(2, NW * 32);
      if (threadIdx.x == 0) {
        __threadfence();
        if (a.bflag) atomicAdd(a.bflag, 1u);
        unsigned* rf = d.zc == 0 ? a.rflag_lo : a.rflag_hi;
        if (rf) {  // the neighbour's planes are written (NVLink / IPC memory)
          __threadfence_system();
          atomicAdd_system(rf, 1u);
        }
      }
    };
    auto step = [&](Tup (&lo)[R1][V], Tup (&mid)[R1][V], Tup (&hi)[R1][V], Tup (&ulo)[R][V],
                    Tup (&umid)[R][V], Tup (&uhi)[R][V]) {
      if constexpr (kPF) {
        row_tuples_inplace<OP, T, R1, V>(hi, nedge);
        make_u1(lo, mid, hi, zs - 3 + p, uhi);
        if (p + 1 < np) fetch(lo);  // (lo is dead now; it is the next step's hi)
        if (p >= 4) emit(ulo, umid, uhi, zs + p - 4);
      } else {
        load_in(hi);
        if (DBG == 1) { ++p; return; }
        make_u1(lo, mid, hi, zs - 3 + p, uhi);
        if (p >= 4) emit(ulo, umid, uhi, zs + p - 4);
      }
      if (MR && a.bnd > 0 && d.zc == 0 && p == 5) publish();
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
    if (MR && a.bnd > 0 && d.zc == 1) publish();
    if constexpr (DYN && RV == RV_RESID) {  // the unit's partial, in unit order
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        t = __dadd_rn(t, acc[i]);
        acc[i] = 0.0;
      }
      cta_partial(t, CB_SUM, red, NW * 32, &a.partials[u]);
    }
  }

  if constexpr (DYN) {
    if constexpr (RV == RV_RESID)
      grid_fold_last(CB_SUM, red, flag, NW * 32, a.partials, a.counter, a.result, gridDim.x, (unsigned)units);
  } else if constexpr (RV == RV_CONV2) {
    cta_reduce_finish(ok1 ? 1.0 : 0.0, CB_AND, red, flag, NW * 32, a.partials, a.counter, a.result, gridDim.x,
                      blockIdx.x);
    cta_reduce_finish(ok2 ? 1.0 : 0.0, CB_AND, red, flag, NW * 32, a.partials2, a.counter2, a.result2,
                      gridDim.x, blockIdx.x);
  } else if constexpr (RV == RV_RESID || RV == RV_RESID_IN) {
    double t = 0.0;  // rows folded in a fixed order (deterministic for the launch)
#pragma unroll
    for (int i = 0; i < R; ++i) t = __dadd_rn(t, acc[i]);
    cta_reduce_finish(t, CB_SUM, red, flag, NW * 32, a.partials, a.counter, a.result, (unsigned)a.nparts,
                      (unsigned)(a.unit0 + blockIdx.x));
  }
}

}  // namespace

// Two sweeps (out = OP(OP(in))) over the whole local interior of a single-rank
// grid.  With rv == RV_RESID the residual of the intermediate iterate (the
// input of the second sweep) is reduced into p.red.
template <int OP, int RV, typename T, int V, int NW, int R, int S, int MINB, bool WP, bool RB = false,
          bool MR = false, int DBG = 0, bool DYN = false>
static cudaError_t launch2r_k(const SweepPlan& p, int64_t* launches) {
  using G = GeoR<T, V, NW, R, S, WP>;
  auto kern = sweep2r_tma<OP, RV, T, V, NW, R, S, MINB, WP, RB, MR, DBG, DYN>;
  constexpr int NT = ThreadsR<NW, MINB, WP>::NT;
  static int occ = -1;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, G::SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  const View& in = p.in[0];
  Sweep2RArgs<T> a{};
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
  // boundary-first: the first and the last z-chunk (what holds the 2 output
  // planes at each end the neighbours' next pass needs) are scheduled first;
  // the first chunk publishes its boundary planes as soon as they are stored,
  // the last one when it ends — about a wave into a ~7-wave pass, so the
  // exchange still overlaps the rest of the pass.  (Round 1 gave the boundary
  // planes 2-plane chunks of their own: 3 input planes per output and a ring
  // start-up per tiny unit, 5-10 % per pass — tools/mr_probe.py.)
  a.bnd = (p.bnd_h > 0 && a.nz >= 6) ? 2 : 0;
  const int64_t tiles = (int64_t)a.tiles_x * a.tiles_y;
  const int64_t slots = (int64_t)occ * p.num_sms;
  // z-chunks: minimise (waves) x (planes streamed per unit, incl. the 4 extra)
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
  int chunks = best;
  if (p.zchunks > 0) chunks = (int)std::min<int64_t>(p.zchunks, a.nzr);
  a.chunk = (a.nzr + chunks - 1) / chunks;
  chunks = (a.nzr + a.chunk - 1) / a.chunk;
  if (a.bnd) {  // the two boundary chunks have `chunk` (>= 2) planes each, the middle ones at most that
    a.chunk = std::max(2, std::min(a.chunk, a.nz / 2));
    chunks = 2 + (a.nz - 2 * a.chunk + a.chunk - 1) / a.chunk;
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
  a.partials2 = p.red2.partials;
  a.counter2 = p.red2.counter;
  a.result2 = p.red2.result;
  a.eps = p.eps;
  a.stop = p.stop;
  a.zpar = (int)(p.zoff & 1);
  CUtensorMap map, gmap;
  if (!encode_tma_3d(&map, in, G::W, G::INROWS, p.l2promo)) return cudaErrorInvalidValue;
  gmap = map;
  if (a.glo | a.ghi) {  // two planes of the grid's plane layout (below, above)
    View gv = in;
    gv.base = const_cast<void*>(p.ghost);
    gv.h = 1;
    gv.nzl = 0;
    gv.ny = in.ny + 2 * in.h - 2;  // rows per plane unchanged
    if (!encode_tma_3d(&gmap, gv, G::W, G::INROWS, p.l2promo)) return cudaErrorInvalidValue;
  }
  a.nchunks = chunks;
  const int64_t units = tiles * chunks;
  const int64_t grid = DYN ? std::min<int64_t>(units, slots) : units;
  a.ticket = p.ticket;
  a.slots = (int)slots;
  a.unit0 = 0;
  a.nparts = (int)grid;
  if (DYN && !p.ticket) return cudaErrorInvalidValue;
  if (RV != RV_NONE && units > p.red.max_partials) return cudaErrorInvalidConfiguration;
  if constexpr (MR && !DYN && !WP && !RB && MINB == 1 && (RV == RV_NONE || RV == RV_RESID)) {
    if (a.bnd && p.bnd_stream) {
      // boundary chunks (z-chunks 0 and 1 of the multi-rank decode) on the
      // boundary stream, issued first; the middle chunks [chunk, nz - chunk)
      // as the single-rank kernel on a view shifted by `chunk` planes, where
      // every u1 plane it computes (local -1 .. nzr) is interior
      kern<<<(unsigned)(2 * tiles), NT, G::SMEM, p.bnd_stream>>>(a, map, gmap);
      ++*launches;
      if (p.bnd_split) *p.bnd_split = true;
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess || chunks == 2) return e;
      auto kmid = sweep2r_tma<OP, RV, T, V, NW, R, S, MINB, WP, RB, false, DBG, false>;
      static bool attr = false;
      if (!attr) {
        e = cudaFuncSetAttribute(kmid, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
      }
      Sweep2RArgs<T> m = a;
      m.out = a.out + (int64_t)a.chunk * a.osz;
      m.pln0 = a.pln0 + a.chunk;
      m.nz = m.nzr = a.nz - 2 * a.chunk;
      m.nchunks = chunks - 2;
      m.zlo = -1;
      m.zhi = m.nz + 1;
      m.glo = m.ghi = 0;
      m.bnd = 0;
      m.bflag = nullptr;
      m.unit0 = (int)(2 * tiles);
      kmid<<<(unsigned)(tiles * (chunks - 2)), NT, G::SMEM, p.stream>>>(m, map, map);
      ++*launches;
      return cudaGetLastError();
    }
  }
  kern<<<(unsigned)grid, NT, G::SMEM, p.stream>>>(a, map, gmap);
  ++*launches;
  return cudaGetLastError();
}

// A launch needs the multi-rank features when it has boundary-first chunks,
// a non-physical z side, or peer stores.
template <int OP, int RV, typename T, int V, int NW, int R, int S, int MINB, bool WP = false, bool RB = false,
          bool DYN = false>
static cudaError_t launch2r(const SweepPlan& p, int64_t* launches) {
  const bool mr = p.bnd_h > 0 || !p.phys_lo || !p.phys_hi || p.ghost || p.peer_lo[0] || p.peer_lo[1] ||
                  p.peer_hi[0] || p.peer_hi[1];
  return mr ? launch2r_k<OP, RV, T, V, NW, R, S, MINB, WP, RB, true, 0, DYN>(p, launches)
            : launch2r_k<OP, RV, T, V, NW, R, S, MINB, WP, RB, false, 0, DYN>(p, launches);
}

template <typename T, int V, int NW, int R, int S, int MINB, bool WP = false, bool DYN = false>
static cudaError_t launch2r_rv(const SweepPlan& p, int64_t* launches) {
  return p.rv == RV_RESID ? launch2r<OP_JACOBI7, RV_RESID, T, V, NW, R, S, MINB, WP, false, DYN>(p, launches)
                          : launch2r<OP_JACOBI7, RV_NONE, T, V, NW, R, S, MINB, WP, false, DYN>(p, launches);
}

template <typename T, int V, int NW, int R>
static int64_t tiles_of(int64_t nx, int64_t ny) {
  using G = GeoR<T, V, NW, R, 4>;
  return ((nx + G::TXO - 1) / G::TXO) * ((ny + G::TYO - 1) / G::TYO);
}

// Ablation geometries (GSCL_ABLATIONS builds only): V (points per lane), NW
// (consumer warps), R (rows per lane), S (ring stages), MINB (CTAs per SM; 0 =
// producer warpgroup with setmaxnreg), WP (warp-private rings).  fp32 always
// runs the default geometry with V = 4.  Results: profiles/r01_sweep2r.md,
// profiles/r02_sweep2r.md.
#ifdef GSCL_ABLATIONS
#define GSCL_PASS_VARIANTS(X)                                                                  \
  X(11, 2, 8, 2, 6, 1, false) /* 8 warps x 2 rows (60 x 16 tile), 6 stages */                  \
  X(12, 2, 3, 4, 4, 2, false) /* 2 CTAs/SM of 3 warps x 4 rows */                              \
  X(14, 2, 7, 4, 8, 1, false) /* default geometry, 8-stage ring */                             \
  X(15, 2, 8, 4, 4, 0, false) /* 8 consumer warps x 4 rows + producer warpgroup, setmaxnreg */ \
  X(40, 1, 7, 4, 4, 2, false) /* one point per lane: 28 x 28 tile, 2 CTAs/SM (128 registers) */ \
  X(41, 1, 7, 4, 8, 2, false) /* the same with an 8-stage ring */                                  \
  X(44, 2, 7, 4, 10, 1, false) /* default geometry, 10-stage ring */                                 \
  X(45, 2, 7, 4, 12, 1, false) /* default geometry, 12-stage ring */                                 \
  X(42, 1, 7, 3, 8, 2, false) /* one point per lane, 3 rows: 28 x 21 tile, 2 CTAs/SM */             \
  X(46, 1, 3, 4, 6, 4, false) /* 28 x 12, 4 CTAs/SM */                                         \
  X(50, 2, 8, 4, 4, 1, true)  /* warp-private rings: 60 x 32 tile, 4 stages per warp */        \
  X(51, 2, 8, 4, 6, 1, true)  /* warp-private rings, 6 stages per warp */                      \
  X(52, 2, 7, 4, 5, 1, true)  /* warp-private rings, 60 x 28, 5 stages */                      \
  X(53, 1, 8, 4, 6, 2, true)  /* warp-private rings, one point per lane, 2 CTAs/SM */          \
  X(54, 1, 4, 4, 6, 4, true)  /* warp-private rings, one point per lane, 4 CTAs/SM */ \
  X(55, 2, 7, 4, 4, 1, false) /* the round-1 default: 4-stage ring */                          \
  X(56, 2, 7, 4, 6, 1, false) /* 6-stage ring */
#endif

// Default geometry: 7 consumer warps x 4 rows (60 x 28 tile for fp64, 120 x 28
// for fp32) + a producer warp, one CTA per SM (up to 255 registers), an
// 8-stage ring (128 KB): the deeper ring keeps ~100 KB of loads in flight per
// SM — 4 stages left the consumers waiting on the TMA (ncu long-scoreboard
// stalls on the ring barrier; 0.406 -> 0.380 ms per 512^3 pass, r02).
#define GSCL_PASS_DEFAULT_F64 2, 7, 4, 8, 1
#define GSCL_PASS_DEFAULT_F32 4, 7, 4, 8, 1

int64_t pass_tiles(int64_t nx, int64_t ny, int dtype, int variant) {
#ifdef GSCL_ABLATIONS
  if (variant == 60) return pass_tiles_x(nx, ny, dtype);
#endif
  if (dtype != 0) return tiles_of<float, 4, 7, 4>(nx, ny);
  switch (variant) {
#ifdef GSCL_ABLATIONS
#define X(id, V, NW, R, S, MINB, WP) \
  case id: return tiles_of<double, V, NW, R>(nx, ny);
    GSCL_PASS_VARIANTS(X)
#undef X
#endif
    default: return tiles_of<double, 2, 7, 4>(nx, ny);
  }
}

// variant: 0 = default geometry; the others (ablation build only) are the
// geometries of GSCL_PASS_VARIANTS and the memory-only / compute-only probes.
cudaError_t launch_sweep2r(const SweepPlan& p, int64_t* launches) {
  const bool f64 = p.in[0].dtype == 0;
  if (p.rbgs) {  // red-black GS iteration (JACOBI7 colour-masked sweeps), default geometry
    if (p.op != OP_JACOBI7) return cudaErrorInvalidValue;
    if (p.rv == RV_RESID_IN)
      return f64 ? launch2r<OP_JACOBI7, RV_RESID_IN, double, GSCL_PASS_DEFAULT_F64, false, true>(p, launches)
                 : launch2r<OP_JACOBI7, RV_RESID_IN, float, GSCL_PASS_DEFAULT_F32, false, true>(p, launches);
    return f64 ? launch2r<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, true>(p, launches)
               : launch2r<OP_JACOBI7, RV_NONE, float, GSCL_PASS_DEFAULT_F32, false, true>(p, launches);
  }
  if (p.rv == RV_CONV2) {  // the convergence loop's pass (FIG1B, JACOBI7), default geometry
    if (p.op == OP_FIG1B)
      return f64 ? launch2r<OP_FIG1B, RV_CONV2, double, GSCL_PASS_DEFAULT_F64>(p, launches)
                 : launch2r<OP_FIG1B, RV_CONV2, float, GSCL_PASS_DEFAULT_F32>(p, launches);
    if (p.op == OP_JACOBI7)
      return f64 ? launch2r<OP_JACOBI7, RV_CONV2, double, GSCL_PASS_DEFAULT_F64>(p, launches)
                 : launch2r<OP_JACOBI7, RV_CONV2, float, GSCL_PASS_DEFAULT_F32>(p, launches);
    return cudaErrorInvalidValue;
  }
  if (p.op != OP_JACOBI7) return cudaErrorInvalidValue;
  if (!f64) return launch2r_rv<float, GSCL_PASS_DEFAULT_F32>(p, launches);
  switch (p.variant) {
#ifdef GSCL_ABLATIONS
#define X(id, V, NW, R, S, MINB, WP) \
  case id: return launch2r_rv<double, V, NW, R, S, MINB, WP>(p, launches);
    GSCL_PASS_VARIANTS(X)
#undef X
    // probes of the default geometry: 91 memory only (loads + stores, no
    // arithmetic), 92 compute only (no ring waits, no TMA), 93 = 91 with the
    // round-1 4-stage ring, 96 without the proxy fence (unsafe), 97 with the
    // Dirichlet select skipped (wrong at the tile edges): timings only
    case 91: return launch2r_k<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, false, false, 1>(p, launches);
    case 92: return launch2r_k<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, false, false, 2>(p, launches);
    case 93: return launch2r_k<OP_JACOBI7, RV_NONE, double, 2, 7, 4, 4, 1, false, false, false, 1>(p, launches);
    case 96: return launch2r_k<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, false, false, 3>(p, launches);
    case 97: return launch2r_k<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, false, false, 4>(p, launches);
    // 94: the round-1 step order (no software pipelining); 95: the default
    // without the proxy fence (unsafe, timing only)
    case 94:
      return p.rv == RV_RESID
                 ? launch2r_k<OP_JACOBI7, RV_RESID, double, GSCL_PASS_DEFAULT_F64, false, false, false, 7>(p, launches)
                 : launch2r_k<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, false, false, 7>(p, launches);
    // 90: L2 prefetch of the next wave's first planes
    case 90: return launch2r_k<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, false, false, 8>(p, launches);
    // 98: persistent CTAs claiming units dynamically (one continuous ring)
    case 98: return launch2r_rv<double, GSCL_PASS_DEFAULT_F64, false, true>(p, launches);
    // 60: u1 rows handed between warps (sweep2x.cu)
    case 60: return launch_sweep2x(p, launches);
    // 99: 8 consumer warps x 4 rows (60 x 32 tile), no producer warp (inline producer)
    case 99: return launch2r_rv<double, 2, 8, 4, 8, -1>(p, launches);
    case 95: return launch2r_k<OP_JACOBI7, RV_NONE, double, GSCL_PASS_DEFAULT_F64, false, false, false, 6>(p, launches);
#endif
    default:
      return launch2r_rv<double, GSCL_PASS_DEFAULT_F64>(p, launches);
  }
}

// Two sweeps per pass: dispatch by operator.  JACOBI7 (and the red-black and
// convergence passes) -> sweep2r_tma; VARCOEF8 -> sweep2v_tma (sweep2v.cu).
// Ablation builds also reach the first design (sweep2.cu, variants 1..4) and
// the JACOBI27 pass (sweep2k.cu).
cudaError_t launch_sweep2(const SweepPlan& p, int64_t* launches) {
  if (p.rv == RV_CONV2 || p.rbgs) return launch_sweep2r(p, launches);
  if (p.op == OP_VARCOEF8) return launch_sweep2v(p, launches);
#ifdef GSCL_ABLATIONS
  if (p.op == OP_JACOBI27) return launch_sweep2k(p, launches);
  if (p.op == OP_JACOBI7 && p.variant >= 1 && p.variant <= 4) return launch_sweep2_smem(p, launches);
#endif
  if (p.op != OP_JACOBI7) return cudaErrorInvalidValue;
  return launch_sweep2r(p, launches);
}

}  // namespace gscl
