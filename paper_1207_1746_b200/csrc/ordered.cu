// ordered.cu — GSCL's ordered iteration spaces (
// PAPER.md:54-56): do_{i,j,k}_{inc,dec} process (i-1,j,k) / (i,j-1,k) /
// (i,j,k-1) (resp. +1) before (i,j,k); do_diamond processes (i-1,j) and
// (i,j-1) before (i,j) in every z plane.  Catalogue: PREFIX
// out(p) = out(p - d) + in(p) and (diamond) PASCAL out = out(i-1,j) + out(i,j-1);
// out's halo supplies the values before the first cell.  Each recurrence runs
// in its defined order, so results are bitwise those of the sequential loops.
//
//  * k / j spaces: one thread per (x, y) / (x, z) line marching the ordered
//    axis — lanes are consecutive x, so every step is a coalesced row access;
//    the loads of the next 8 cells are issued before the dependent adds.
//  * i spaces: a warp per 32 rows, 32 x 32 tiles transposed through shared
//    memory so loads and stores stay coalesced while each lane scans its row.
//  * diamond: one warp per z plane, a skewed wavefront in registers (lane l
//    computes row y at step y + l; left neighbours by shuffle) — see
//    k_pascal_lanes.
#include <algorithm>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

GSCL_MODULE_ANCHOR(anchor_ordered)


namespace {

struct OrdArgs {
  const void* in;
  void* out;
  int64_t isy, isz, osy, osz;  // element strides of in / out (origin-relative)
  int nx, ny, nz;
};

constexpr int kUnroll = 8;

// PREFIX along an axis with `stride` (elements) between consecutive cells;
// `n` cells starting at `first` (origin-relative offsets), stepping +/-.
template <typename T, bool INC>
__device__ __forceinline__ void prefix_line(const T* in, T* out, int64_t in_first, int64_t out_first,
                                            int64_t istride, int64_t ostride, int n) {
  const int64_t dir = INC ? 1 : -1;
  T run = out[out_first - dir * ostride];  // the halo cell before the first one
  int s = 0;
  for (; s + kUnroll <= n; s += kUnroll) {
    T v[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) v[q] = __ldg(in + in_first + dir * (s + q) * istride);
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) {
      run = add(run, v[q]);
      out[out_first + dir * (s + q) * ostride] = run;
    }
  }
  for (; s < n; ++s) {
    run = add(run, __ldg(in + in_first + dir * s * istride));
    out[out_first + dir * s * ostride] = run;
  }
}

template <typename T, int AXIS, bool INC> __global__ void k_prefix(const OrdArgs a) {
  const T* in = static_cast<const T*>(a.in);
  T* out = static_cast<T*>(a.out);
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if constexpr (AXIS == 2) {  // k: thread per (x, y)
    if (t >= (int64_t)a.nx * a.ny) return;
    const int x = (int)(t % a.nx), y = (int)(t / a.nx);
    const int z0 = INC ? 0 : a.nz - 1;
    prefix_line<T, INC>(in, out, (int64_t)z0 * a.isz + (int64_t)y * a.isy + x,
                        (int64_t)z0 * a.osz + (int64_t)y * a.osy + x, a.isz, a.osz, a.nz);
  } else if constexpr (AXIS == 1) {  // j: thread per (x, z)
    if (t >= (int64_t)a.nx * a.nz) return;
    const int x = (int)(t % a.nx), z = (int)(t / a.nx);
    const int y0 = INC ? 0 : a.ny - 1;
    prefix_line<T, INC>(in, out, (int64_t)z * a.isz + (int64_t)y0 * a.isy + x,
                        (int64_t)z * a.osz + (int64_t)y0 * a.osy + x, a.isy, a.osy, a.ny);
  } else {  // i: thread per (y, z) row
    if (t >= (int64_t)a.ny * a.nz) return;
    const int y = (int)(t % a.ny), z = (int)(t / a.ny);
    const int x0 = INC ? 0 : a.nx - 1;
    prefix_line<T, INC>(in, out, (int64_t)z * a.isz + (int64_t)y * a.isy + x0,
                        (int64_t)z * a.osz + (int64_t)y * a.osy + x0, 1, 1, a.nx);
  }
}

// k / j spaces, fp64 with even nx: a thread marches TWO adjacent x lines
// (one 16-byte vector per cell pair: 512-byte warp accesses instead of 256,
// and two independent dependency chains per thread).  Each line's sum is
// still formed in its own order, so results are bitwise those of k_prefix.
template <bool INC>
__device__ __forceinline__ void prefix_line2(const double* in, double* out, int64_t in_first, int64_t out_first,
                                             int64_t istride, int64_t ostride, int n) {
  const int64_t dir = INC ? 1 : -1;
  double2 run = *reinterpret_cast<const double2*>(out + out_first - dir * ostride);
  int s = 0;
  for (; s + kUnroll <= n; s += kUnroll) {
    double2 v[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) v[q] = __ldg(reinterpret_cast<const double2*>(in + in_first + dir * (s + q) * istride));
#pragma unroll
    for (int q = 0; q < kUnroll; ++q) {
      run.x = add(run.x, v[q].x);
      run.y = add(run.y, v[q].y);
      *reinterpret_cast<double2*>(out + out_first + dir * (s + q) * ostride) = run;
    }
  }
  for (; s < n; ++s) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(in + in_first + dir * s * istride));
    run.x = add(run.x, v.x);
    run.y = add(run.y, v.y);
    *reinterpret_cast<double2*>(out + out_first + dir * s * ostride) = run;
  }
}

template <int AXIS, bool INC> __global__ void k_prefix2(const OrdArgs a) {
  const double* in = static_cast<const double*>(a.in);
  double* out = static_cast<double*>(a.out);
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int hx = a.nx / 2;
  if constexpr (AXIS == 2) {  // k: thread per (x pair, y)
    if (t >= (int64_t)hx * a.ny) return;
    const int x = 2 * (int)(t % hx), y = (int)(t / hx);
    const int z0 = INC ? 0 : a.nz - 1;
    prefix_line2<INC>(in, out, (int64_t)z0 * a.isz + (int64_t)y * a.isy + x,
                      (int64_t)z0 * a.osz + (int64_t)y * a.osy + x, a.isz, a.osz, a.nz);
  } else {  // j: thread per (x pair, z)
    if (t >= (int64_t)hx * a.nz) return;
    const int x = 2 * (int)(t % hx), z = (int)(t / hx);
    const int y0 = INC ? 0 : a.ny - 1;
    prefix_line2<INC>(in, out, (int64_t)z * a.isz + (int64_t)y0 * a.isy + x,
                      (int64_t)z * a.osz + (int64_t)y0 * a.osy + x, a.isy, a.osy, a.ny);
  }
}

// i spaces: a warp owns 32 consecutive rows; per 32-column tile it loads the
// 32 x 32 block with coalesced row reads (all 32 issued before any is used:
// 8 KB in flight per warp), stages it in shared memory, each lane scans its
// own row across the tile in order (carrying the running sum), and the block is
// written back with coalesced row stores.  Row offsets are computed once per
// lane (one division) and broadcast with shuffles.
template <typename T, bool INC> __global__ void __launch_bounds__(128) k_prefix_rows(const OrdArgs a) {
  __shared__ T tile[4][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)a.ny * a.nz;
  const int64_t r0 = ((int64_t)blockIdx.x * 4 + warp) * 32;  // first row of my warp
  if (r0 >= rows) return;
  const T* in = static_cast<const T*>(a.in);
  T* out = static_cast<T*>(a.out);
  const int64_t my_row = r0 + lane;
  const bool my_ok = my_row < rows;
  const int64_t zr = my_ok ? my_row / a.ny : 0, yr = my_ok ? my_row % a.ny : 0;
  const int64_t my_in = zr * a.isz + yr * a.isy, my_out = zr * a.osz + yr * a.osy;
  const int nvalid = rows - r0 < 32 ? (int)(rows - r0) : 32;  // rows of this warp that exist
  T run = T(0);
  if (my_ok) run = out[my_out + (INC ? -1 : a.nx)];  // halo before the first cell
  T(&t)[32][33] = tile[warp];
  const int ntiles = (a.nx + 31) / 32;
  // Row r of the warp's group: with ny >= 32 the group spans at most two
  // planes, so its offsets follow from the (warp-uniform) first row with
  // integer arithmetic instead of a shuffle per row per tile (the shuffles
  // and the shared-memory transposes were the kernel's MIO bottleneck).
  const bool arith = a.ny >= 32;
  const int64_t zg = r0 / a.ny, yg = r0 % a.ny;
  const int split = (int)(a.ny - yg < 32 ? a.ny - yg : 32);  // rows r < split lie in plane zg
  const int64_t ib0c = zg * a.isz + yg * a.isy, ib1c = (zg + 1) * a.isz - split * a.isy;
  const int64_t ob0c = zg * a.osz + yg * a.osy, ob1c = (zg + 1) * a.osz - split * a.osy;
  for (int ti = 0; ti < ntiles; ++ti) {
    // (re-read each tile through an opaque move, so the compiler does not
    // hoist 2 x 32 row offsets out of the tile loop into registers)
    int64_t ib0, ib1, ob0, ob1;
    asm volatile("mov.b64 %0, %1;" : "=l"(ib0) : "l"(ib0c));
    asm volatile("mov.b64 %0, %1;" : "=l"(ib1) : "l"(ib1c));
    asm volatile("mov.b64 %0, %1;" : "=l"(ob0) : "l"(ob0c));
    asm volatile("mov.b64 %0, %1;" : "=l"(ob1) : "l"(ob1c));
    auto row_off = [&](int r, int64_t sy, int64_t b0, int64_t b1, int64_t mine) -> int64_t {
      if (!arith) return __shfl_sync(0xffffffffu, mine, r);
      return (r < split ? b0 : b1) + r * sy;
    };
    const int tt = INC ? ti : ntiles - 1 - ti;
    const int x = tt * 32 + lane;
    const bool xok = x < a.nx;
    T v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int64_t off = row_off(r, a.isy, ib0, ib1, my_in);
      v[r] = (r < nvalid && xok) ? __ldg(in + off + x) : T(0);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) t[r][lane] = v[r];
    __syncwarp();
    // lane scans its row in the space's order
    const int x0 = tt * 32;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      const int cc = INC ? c : 31 - c;
      if (x0 + cc < a.nx) {
        run = add(run, t[lane][cc]);
        t[lane][cc] = run;
      }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int64_t off = row_off(r, a.osy, ob0, ob1, my_out);
      if (r < nvalid && xok) out[off + x] = t[r][lane];
    }
    __syncwarp();
  }
}

// diamond as a skewed wavefront (default): ONE WARP per z plane.  Lane l owns
// C consecutive columns x = 32 C b + C l .. + C - 1 of column block b and
// computes row y of them at step t = y + l: the left neighbour of its first
// column, (x - 1, y), is lane l - 1's last column at the previous step (a warp
// shuffle), every other left neighbour its own previous column, and every
// upper neighbour its own value of row y - 1 (registers).  Lane 0 of a block
// takes column x - 1 from the halo / the previous block (read 32 rows at a
// time, one window ahead).  No barrier at all on the dependency chain; a plane
// costs ny + 31 steps of C dependent additions per column block.  Each cell is
// out(x, y) = add(out(x - 1, y), out(x, y - 1)) after both predecessors, so
// the table is bitwise the sequential one.
template <typename T, int C> __global__ void __launch_bounds__(128) k_pascal_lanes(const OrdArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int plane = blockIdx.x * 4 + warp;
  if (plane >= a.nz) return;
  T* out = static_cast<T*>(a.out) + (int64_t)plane * a.osz;
  const int nblk = (a.nx + 32 * C - 1) / (32 * C);
  for (int b = 0; b < nblk; ++b) {
    const int xb = b * 32 * C;       // first column of the block
    const int x0 = xb + C * lane;    // my first column
    T up[C];
#pragma unroll
    for (int c = 0; c < C; ++c) up[c] = (x0 + c < a.nx) ? out[-a.osy + x0 + c] : T(0);  // halo row
    T last = up[C - 1];
    auto col_load = [&](int t0) {
      return (t0 + lane < a.ny) ? out[(int64_t)(t0 + lane) * a.osy + xb - 1] : T(0);
    };
    T col_cur = col_load(0), col_nxt = col_load(32);
    const bool full = x0 + C <= a.nx;
    for (int t = 0; t < a.ny + 31; ++t) {
      const int y = t - lane;
      if ((t & 31) == 0 && t > 0) {
        col_cur = col_nxt;
        col_nxt = col_load(t + 32);
      }
      const T c0 = __shfl_sync(0xffffffffu, col_cur, t & 31);
      T left = __shfl_up_sync(0xffffffffu, last, 1);
      if (lane == 0) left = c0;
      if (y >= 0 && y < a.ny && x0 < a.nx) {
        T v = left;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          v = add(v, up[c]);
          up[c] = v;
        }
        last = v;
        T* row = out + (int64_t)y * a.osy + x0;
        if (full && (sizeof(T) * C) % 16 == 0) {
          constexpr int VN = Vec<T>::N;
#pragma unroll
          for (int c = 0; c < C; c += VN) {
            T w[VN];
#pragma unroll
            for (int q = 0; q < VN; ++q) w[q] = up[c + q];
            vstore<T>(row + c, w);
          }
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (x0 + c < a.nx) row[c] = up[c];
        }
      }
    }
    __syncwarp();
  }
}


}  // namespace

cudaError_t launch_ordered(int space, int op, const View* in, const View& out, cudaStream_t s,
                           int64_t* launches) {
  OrdArgs a{};
  a.in = in ? in->origin : nullptr;
  a.out = out.origin;
  if (in) {
    a.isy = in->pitch;
    a.isz = in->plane;
  }
  a.osy = out.pitch;
  a.osz = out.plane;
  a.nx = (int)out.nx;
  a.ny = (int)out.ny;
  a.nz = (int)out.nzl;
  const bool f64 = out.dtype == 0;
  if (space == 6) {
    if (op != 1) return cudaErrorInvalidValue;
    const unsigned blocks = (unsigned)((a.nz + 3) / 4);
    if (f64) k_pascal_lanes<double, 16><<<blocks, 128, 0, s>>>(a);
    else k_pascal_lanes<float, 16><<<blocks, 128, 0, s>>>(a);
    ++*launches;
    return cudaGetLastError();
  }
  if (op != 0 || !in) return cudaErrorInvalidValue;
  const int axis = space / 2;
  const bool inc = (space % 2) == 0;
  if (axis == 0) {  // rows: coalesced through a shared-memory transpose
    const int64_t rows = (int64_t)a.ny * a.nz;
    const unsigned blocks = (unsigned)((rows + 127) / 128);
    if (f64) {
      if (inc) k_prefix_rows<double, true><<<blocks, 128, 0, s>>>(a);
      else k_prefix_rows<double, false><<<blocks, 128, 0, s>>>(a);
    } else {
      if (inc) k_prefix_rows<float, true><<<blocks, 128, 0, s>>>(a);
      else k_prefix_rows<float, false><<<blocks, 128, 0, s>>>(a);
    }
    ++*launches;
    return cudaGetLastError();
  }
  if (f64 && a.nx % 2 == 0 && axis >= 1) {  // two x lines per thread (16-byte cells)
    const int64_t pairs = (int64_t)(a.nx / 2) * (axis == 2 ? a.ny : a.nz);
    const unsigned blocks = (unsigned)((pairs + 255) / 256);
    if (axis == 2) {
      if (inc) k_prefix2<2, true><<<blocks, 256, 0, s>>>(a);
      else k_prefix2<2, false><<<blocks, 256, 0, s>>>(a);
    } else {
      if (inc) k_prefix2<1, true><<<blocks, 256, 0, s>>>(a);
      else k_prefix2<1, false><<<blocks, 256, 0, s>>>(a);
    }
    ++*launches;
    return cudaGetLastError();
  }
  const int64_t lines = axis == 2 ? (int64_t)a.nx * a.ny : axis == 1 ? (int64_t)a.nx * a.nz
                                                                     : (int64_t)a.ny * a.nz;
  const unsigned blocks = (unsigned)((lines + 255) / 256);
#define GSCL_ORD(T, AX, INC) k_prefix<T, AX, INC><<<blocks, 256, 0, s>>>(a)
#define GSCL_ORD_T(T)                                              \
  switch (axis * 2 + (inc ? 0 : 1)) {                              \
    case 0: GSCL_ORD(T, 0, true); break;                           \
    case 1: GSCL_ORD(T, 0, false); break;                          \
    case 2: GSCL_ORD(T, 1, true); break;                           \
    case 3: GSCL_ORD(T, 1, false); break;                          \
    case 4: GSCL_ORD(T, 2, true); break;                           \
    default: GSCL_ORD(T, 2, false); break;                         \
  }
  if (f64) {
    GSCL_ORD_T(double)
  } else {
    GSCL_ORD_T(float)
  }
#undef GSCL_ORD_T
#undef GSCL_ORD
  ++*launches;
  return cudaGetLastError();
}

}  // namespace gscl
