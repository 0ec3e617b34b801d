// sweep2v.cu — two VARCOEF8 sweeps per HBM pass (temporal blocking for the
// 8-grid operator).
//
// out = OP(OP(u)) with OP = VARCOEF8 (u plus 7 centre-only coefficient grids,
// DESIGN.md R7) and the Dirichlet rule of gscl_jacobi_run for the
// intermediate u1.  The coefficient grids are constant, so one pass reads u
// and the 7 coefficients ONCE for two sweeps: 72 B per point per pass instead
// of 144 B for two single sweeps.  Same per-plane tuples as ops.cuh, so the
// result is bitwise that of two single sweeps.
//
// Layout: like sweep2r.cu (a lane owns V consecutive x points, warps stack in
// y, the z pipelines of both sweeps in registers, x neighbours by shuffle),
// with R = 1 output row per lane — each stage carries u (TYO + 4 rows) and the
// 7 coefficient tiles of the u1 band (TYO + 2 rows) — and the coefficients a
// lane needs for its second-sweep tuple of plane z kept in registers from the
// plane's load until that tuple is formed one plane later.
#include <algorithm>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

GSCL_MODULE_ANCHOR(anchor_sweep2v)


namespace {

template <typename T, int NW, int S> struct GeoV {
  static constexpr int V = Vec<T>::N;
  static constexpr int W = 32 * V;
  static constexpr int TXO = W - 2 * V;
  static constexpr int TYO = NW;            // R = 1 output row per warp
  static constexpr int UROWS = TYO + 4;     // u rows: y0-2 .. y0+TYO+1
  static constexpr int CROWS = TYO + 2;     // coefficient rows: the u1 band y0-1 .. y0+TYO
  static constexpr int UBYTES = UROWS * W * (int)sizeof(T);
  static constexpr int CBYTES = CROWS * W * (int)sizeof(T);
  static constexpr int STAGE = UBYTES + 7 * CBYTES;
  static constexpr int STAGE_AL = (STAGE + 127) / 128 * 128;
  static constexpr int HEADER = 1024;
  static constexpr int SMEM = HEADER + S * STAGE_AL;
  static_assert(UBYTES % 128 == 0 && CBYTES % 128 == 0, "tile alignment");
};

template <typename T> struct Sweep2VArgs {
  T* out;
  int64_t osy, osz;
  int nx, ny, nz;
  int tiles_x, tiles_y, chunk, nzr;
  int col0[8], row0[8], pln0[8];
  double* partials;
  unsigned* counter;
  double* result;
  // z-slab of several ranks (MR), as in sweep2r.cu: u1 = OP(u) on planes
  // zlo <= z < zhi (the Dirichlet rule only at physical z ends); u planes
  // beyond the grid's halo come from the u ghost map (plane 0 below, 1 above)
  // when glo / ghi; the coefficient planes -1 / nz of a rank boundary (the
  // coefficient grids have no halo) come from the coefficient ghost map
  // (plane 2c below, 2c + 1 above) when cglo / cghi
  int zlo, zhi, h, glo, ghi, cglo, cghi;
  // boundary-first: units of z-chunk 0 / 1 are the bnd output planes at each
  // end; each bumps *bflag (and, peer transport, the neighbour's counter)
  // after its stores, which also go into the neighbours' receiving planes
  int bnd;
  unsigned* bflag;
  T* rlo[2];
  T* rhi[2];
  unsigned* rflag_lo;
  unsigned* rflag_hi;
};
// maps: [0] u, [1..7] coefficients, [8] u ghost planes, [9] coefficient ghost planes
struct Maps10 {
  CUtensorMap m[10];
};

template <typename T> __device__ __forceinline__ T vshfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T> __device__ __forceinline__ T vshfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <int RV, typename T, int NW, int S, int MINB, bool MR = false>
__global__ void __launch_bounds__(32 * (NW + 1), MINB)
    sweep2v_tma(const __grid_constant__ Sweep2VArgs<T> a, const __grid_constant__ Maps10 maps) {
  using G = GeoV<T, NW, S>;
  using O = OpT<OP_VARCOEF8, T>;
  using Tup = typename O::Tup;
  constexpr int V = G::V;

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
  int zs, ze;
  if (MR && a.bnd > 0) {  // [0, bnd), [nz-bnd, nz), then the interior chunks
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
  const int np = ze - zs + 4;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // ---------------- producer: u box + 7 coefficient boxes per plane
    if (lane == 0) {
      for (int c = 0; c < (MR ? 10 : 8); ++c) tma_prefetch_desc(&maps.m[c]);
      int s = 0;
      uint32_t ph = 0;
      for (int p = 0; p < np; ++p) {
        if (p >= S) mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], G::STAGE);
        unsigned char* st = stages + s * G::STAGE_AL;
        const int z = zs - 2 + p;
        const int xb = a.col0[0] + xt0 - V;
        if (MR && a.glo && z < -a.h)
          tma_load_3d(st, &maps.m[8], xb, a.row0[0] + yt0 - 2, 0, &full[s]);
        else if (MR && a.ghi && z >= a.nz + a.h)
          tma_load_3d(st, &maps.m[8], xb, a.row0[0] + yt0 - 2, 1, &full[s]);
        else
          tma_load_3d(st, &maps.m[0], xb, a.row0[0] + yt0 - 2, a.pln0[0] + z, &full[s]);
        // (coefficient planes outside the grid and outside a rank boundary's
        // ghost planes are zero-filled by the TMA; they only meet u1 points
        // the Dirichlet rule keeps at their halo value)
        const bool cg = MR && ((a.cglo && z == -1) || (a.cghi && z == a.nz));
#pragma unroll
        for (int c = 1; c < 8; ++c) {
          if (cg)
            tma_load_3d(st + G::UBYTES + (c - 1) * G::CBYTES, &maps.m[9], a.col0[c] + xt0 - V,
                        yt0 - 1, 2 * (c - 1) + (z < 0 ? 0 : 1), &full[s]);
          else
            tma_load_3d(st + G::UBYTES + (c - 1) * G::CBYTES, &maps.m[c], a.col0[c] + xt0 - V,
                        a.row0[c] + yt0 - 1, a.pln0[c] + z, &full[s]);
        }
        if (++s == S) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumers: warp w's output row y = yt0 + w; its u1 rows
  // j = 0..2 are y = yt0 - 1 + w + j (coefficient rows w + j of the band);
  // its u rows are box rows w .. w + 4.
  const int xs = xt0 - V + V * lane;
  const int yo = yt0 + warp;
  uint32_t in1 = 0;
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int k = 0; k < V; ++k)
      if (xs + k >= 0 && xs + k < a.nx && yo - 1 + j >= 0 && yo - 1 + j < a.ny) in1 |= 1u << (j * V + k);
  uint32_t okm = 0;
  const bool lane_out = lane >= 1 && lane <= 30;
#pragma unroll
  for (int k = 0; k < V; ++k)
    if (lane_out && xs + k < a.nx && yo < a.ny) okm |= 1u << k;
  constexpr uint32_t kAll1 = (3 * V == 32) ? 0xffffffffu : ((1u << (3 * V)) - 1u);
  constexpr uint32_t kAllO = (1u << V) - 1u;
  const bool fast = okm == kAllO;
  const bool warp_int = __all_sync(0xffffffffu, in1 == kAll1);
  T* optr = a.out + (int64_t)yo * a.osy + xs + (int64_t)zs * a.osz;
  double acc = 0.0;

  int s = 0;
  uint32_t ph = 0;
  // the coefficients of my output points for the second sweep, per plane
  struct Cf {
    T c[7][V];
  };
  // sweep-1 tuples of the next input plane (3 u1 rows) + my output row's
  // coefficients (u1 row 1) for that plane's second-sweep tuple
  auto load_in = [&](Tup (&t)[3][V], Cf& cf2) {
    mbar_wait(&full[s], ph);
    const unsigned char* st = stages + s * G::STAGE_AL;
    const T* U = reinterpret_cast<const T*>(st) + warp * G::W + V * lane;
    T rows[5][V];
#pragma unroll
    for (int r = 0; r < 5; ++r) vload<T>(U + r * G::W, rows[r]);
    T cf[3][7][V];
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const T* C = reinterpret_cast<const T*>(st + G::UBYTES + c * G::CBYTES) + warp * G::W + V * lane;
#pragma unroll
      for (int j = 0; j < 3; ++j) vload<T>(C + j * G::W, cf[j][c]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
#pragma unroll
    for (int c = 0; c < 7; ++c)
#pragma unroll
      for (int k = 0; k < V; ++k) cf2.c[c][k] = cf[1][c][k];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const T xl = vshfl_up1(rows[j + 1][V - 1]);
      const T xr = vshfl_dn1(rows[j + 1][0]);
#pragma unroll
      for (int k = 0; k < V; ++k) {
        Nbr<T> n;
        n.c = rows[j + 1][k];
        n.xm = k > 0 ? rows[j + 1][k - 1] : xl;
        n.xp = k < V - 1 ? rows[j + 1][k + 1] : xr;
        n.ym = rows[j][k];
        n.yp = rows[j + 2][k];
        n.h0 = add(n.xm, n.xp);
        T c7[7];
#pragma unroll
        for (int c = 0; c < 7; ++c) c7[c] = cf[j][c][k];
        t[j][k] = O::plane(n, c7);
      }
    }
  };
  // u1 plane z (3 rows) from the tuples of z-1, z, z+1, then its second-sweep
  // tuple at my output row with the coefficients of plane z
  auto make_u1 = [&](const Tup (&lo)[3][V], const Tup (&mid)[3][V], const Tup (&hi)[3][V], int z, const Cf& cfz,
                     Tup (&t2)[V]) {
    const bool zin = MR ? (z >= a.zlo && z < a.zhi) : (z >= 0 && z < a.nz);
    T u1[3][V];
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k)
        u1[j][k] = (zin && (warp_int || ((in1 >> (j * V + k)) & 1u))) ? O::out(lo[j][k], mid[j][k], hi[j][k])
                                                                      : mid[j][k].c;
    const T xl = vshfl_up1(u1[1][V - 1]);
    const T xr = vshfl_dn1(u1[1][0]);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      Nbr<T> n;
      n.c = u1[1][k];
      n.xm = k > 0 ? u1[1][k - 1] : xl;
      n.xp = k < V - 1 ? u1[1][k + 1] : xr;
      n.ym = u1[0][k];
      n.yp = u1[2][k];
      n.h0 = add(n.xm, n.xp);
      T c7[7];
#pragma unroll
      for (int c = 0; c < 7; ++c) c7[c] = cfz.c[c][k];
      t2[k] = O::plane(n, c7);
    }
  };
  auto emit = [&](const Tup (&lo)[V], const Tup (&mid)[V], const Tup (&hi)[V], int zo) {
    T v[V];
#pragma unroll
    for (int k = 0; k < V; ++k) v[k] = O::out(lo[k], mid[k], hi[k]);
    if constexpr (RV == RV_SQ) {  // the intermediate iterate's SQ at my output points
#pragma unroll
      for (int k = 0; k < V; ++k)
        acc = __dadd_rn(acc, ((okm >> k) & 1u) ? (double)mul(mid[k].c, mid[k].c) : 0.0);
    }
    if (fast) {
      vstore<T>(optr, v);
    } else if (okm) {
#pragma unroll
      for (int k = 0; k < V; ++k)
        if ((okm >> k) & 1u) optr[k] = v[k];
    }
    optr += a.osz;
    if (MR && a.bnd > 0 && zc < 2) {  // boundary plane: also into the neighbour's receiving plane
      T* rp = nullptr;
      if (zc == 0) {
        if (zo < 2) rp = a.rlo[zo];
      } else {
        const int q = a.nz - 1 - zo;
        if (q >= 0 && q < 2) rp = a.rhi[q];
      }
      if (rp) {
        rp += (int64_t)yo * a.osy + xs;
        if (fast) {
          vstore<T>(rp, v);
        } else if (okm) {
#pragma unroll
          for (int k = 0; k < V; ++k)
            if ((okm >> k) & 1u) rp[k] = v[k];
        }
      }
    }
  };

  // input plane p is z = zs-2+p; after p >= 2: u1(zs-3+p) and its second-sweep
  // tuple (with the coefficients loaded with plane zs-3+p); p >= 4: out(zs+p-4)
  Tup A[3][V], B[3][V], C[3][V];
  Tup X[V], Y[V], Z[V];
  Cf F0, F1, F2;  // coefficients of the planes held in A, B, C
  load_in(A, F0);
  load_in(B, F1);
  int p = 2;
  auto step = [&](Tup (&lo)[3][V], Tup (&mid)[3][V], Tup (&hi)[3][V], const Cf& fmid, Cf& fhi,
                  Tup (&ulo)[V], Tup (&umid)[V], Tup (&uhi)[V]) {
    load_in(hi, fhi);
    make_u1(lo, mid, hi, zs - 3 + p, fmid, uhi);
    if (p >= 4) emit(ulo, umid, uhi, zs + p - 4);
    ++p;
  };
  for (; p + 3 <= np;) {
    step(A, B, C, F1, F2, X, Y, Z);
    step(B, C, A, F2, F0, Y, Z, X);
    step(C, A, B, F0, F1, Z, X, Y);
  }
  if (p < np) {
    step(A, B, C, F1, F2, X, Y, Z);
    if (p < np) step(B, C, A, F2, F0, Y, Z, X);
  }
  if (MR && a.bnd > 0 && zc < 2) {
    // boundary planes stored: publish them (the comm stream waits on bflag
    // before the NCCL exchange; the peer transport's neighbour waits on its
    // counter)
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

  if constexpr (RV != RV_NONE)
    cta_reduce_finish(acc, CB_SUM, red, flag, NW * 32, a.partials, a.counter, a.result, gridDim.x, blockIdx.x);
}

template <int RV, typename T, int NW, int S, int MINB, bool MR>
cudaError_t launch2v_k(const SweepPlan& p, int64_t* launches) {
  using G = GeoV<T, NW, S>;
  auto kern = sweep2v_tma<RV, T, NW, S, MINB, MR>;
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
  Sweep2VArgs<T> a{};
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
  a.cglo = (p.cghost && !p.phys_lo) ? 1 : 0;
  a.cghi = (p.cghost && !p.phys_hi) ? 1 : 0;
  if ((!p.phys_lo || !p.phys_hi) && !p.cghost) return cudaErrorInvalidValue;  // coefficient planes needed
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
    const double cost = (double)waves * (double)(chunk + 4);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = (int)cc;
    }
  }
  int chunks = p.zchunks > 0 ? (int)std::min<int64_t>(p.zchunks, a.nzr) : best;
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
  Maps10 maps;
  for (int i = 0; i < 8; ++i) {
    const View& v = p.in[i];
    if (!encode_tma_3d(&maps.m[i], v, G::W, i == 0 ? G::UROWS : G::CROWS, p.l2promo)) return cudaErrorInvalidValue;
    a.col0[i] = (int)v.ox;
    a.row0[i] = v.h;
    a.pln0[i] = v.h;
  }
  maps.m[8] = maps.m[0];
  maps.m[9] = maps.m[1];
  if (a.glo | a.ghi) {  // two u planes of the grid's plane layout (below, above)
    View gv = in;
    gv.base = const_cast<void*>(p.ghost);
    gv.h = 1;
    gv.nzl = 0;
    gv.ny = in.ny + 2 * in.h - 2;
    if (!encode_tma_3d(&maps.m[8], gv, G::W, G::UROWS, p.l2promo)) return cudaErrorInvalidValue;
  }
  if (a.cglo | a.cghi) {  // 14 coefficient planes (plane 2c below, 2c + 1 above), coefficient layout
    View cv = p.in[1];
    cv.base = const_cast<void*>(p.cghost);
    cv.nzl = 14 + 2 * cv.h;  // (h = 0 for the coefficient grids)
    cv.nzl = 14;
    if (cv.h != 0) return cudaErrorInvalidValue;
    if (!encode_tma_3d(&maps.m[9], cv, G::W, G::CROWS, p.l2promo)) return cudaErrorInvalidValue;
  }
  a.partials = p.red.partials;
  a.counter = p.red.counter;
  a.result = p.red.result;
  const int64_t units = tiles * chunks;
  if (RV != RV_NONE && units > p.red.max_partials) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)units, NT, G::SMEM, p.stream>>>(a, maps);
  ++*launches;
  return cudaGetLastError();
}

// the multi-rank features (boundary chunks, ghost maps, peer stores) are
// compiled only into the launches that need them
template <int RV, typename T, int NW, int S, int MINB>
cudaError_t launch2v(const SweepPlan& p, int64_t* launches) {
  const bool mr = p.bnd_h > 0 || !p.phys_lo || !p.phys_hi || p.ghost || p.cghost || p.peer_lo[0] ||
                  p.peer_lo[1] || p.peer_hi[0] || p.peer_hi[1];
  return mr ? launch2v_k<RV, T, NW, S, MINB, true>(p, launches) : launch2v_k<RV, T, NW, S, MINB, false>(p, launches);
}

}  // namespace

int64_t pass_tiles_v(int64_t nx, int64_t ny, int dtype) {
  if (dtype == 0) {
    using G = GeoV<double, 8, 3>;
    return ((nx + G::TXO - 1) / G::TXO) * ((ny + G::TYO - 1) / G::TYO);
  }
  using G = GeoV<float, 8, 3>;
  return ((nx + G::TXO - 1) / G::TXO) * ((ny + G::TYO - 1) / G::TYO);
}

// VARCOEF8 two-sweep pass: 8 warps x 1 output row (60 x 8 tile for fp64),
// 3-stage ring of u + 7 coefficient tiles; on a multi-rank slab with the
// boundary-first chunks, ghost maps and peer stores of sweep2r.cu.
cudaError_t launch_sweep2v(const SweepPlan& p, int64_t* launches) {
  if (p.op != OP_VARCOEF8 || p.n_in != 8) return cudaErrorInvalidValue;
  const bool f64 = p.in[0].dtype == 0;
  const bool sq = p.rv == RV_SQ;
  if (f64) {
#ifdef GSCL_ABLATIONS
    // geometry ablations (gscl_set_option "variant"): 11 = 4-stage ring,
    // 12 = 12 warps (less y-halo re-read), 14 = 4 warps x 2 CTAs per SM
    if (p.variant == 11)
      return sq ? launch2v<RV_SQ, double, 8, 4, 1>(p, launches) : launch2v<RV_NONE, double, 8, 4, 1>(p, launches);
    if (p.variant == 12)
      return sq ? launch2v<RV_SQ, double, 12, 3, 1>(p, launches) : launch2v<RV_NONE, double, 12, 3, 1>(p, launches);
    if (p.variant == 14)
      return sq ? launch2v<RV_SQ, double, 4, 4, 2>(p, launches) : launch2v<RV_NONE, double, 4, 4, 2>(p, launches);
#endif
    return sq ? launch2v<RV_SQ, double, 8, 3, 1>(p, launches) : launch2v<RV_NONE, double, 8, 3, 1>(p, launches);
  }
  return sq ? launch2v<RV_SQ, float, 8, 3, 1>(p, launches) : launch2v<RV_NONE, float, 8, 3, 1>(p, launches);
}

}  // namespace gscl
