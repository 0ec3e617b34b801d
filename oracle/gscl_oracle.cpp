/*
 * gscl_oracle.cpp — the plain, slow CPU oracle for the GSCL hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1207_1746_b200/) never links, imports or calls it,
 * and this file includes nothing from the product tree: it has its own dense
 * layout, its own copy of the counter-based input generator, its own digest.
 *
 * What it computes (paper = /root/reference/PAPER.md):
 *   do_all     PAPER.md:47,51 (§3: "reads elements of the grids at fixed
 *              offsets ... can write elements corresponding to the core
 *              elements"; do_all "does not guarantee any order") and
 *              PAPER.md:60-73 (Fig 1.b, the operator this build calls FIG1B).
 *   do_reduce  PAPER.md:53 (§3: return values "(commutatively) reduced to a
 *              single value"), PAPER.md:192 (§5.3: "the sum of all elements").
 *   fused      PAPER.md:159-172 (§5.2: fuse(sten_op_diffusion(),
 *              sten_op_convergence(EPSI)), "only one scan of the grids").
 *   jacobi     PAPER.md:157,161-170 (§5.2 Jacobi iteration with swap_grids()).
 * Every per-point expression tree is the one fixed in DESIGN.md §3 (readings
 * R1-R11); each + - * / is a single IEEE-754 operation, round-to-nearest, with
 * no contraction (compiled -ffp-contract=off).  Sums accumulate in long double
 * per z-plane and the plane partials are folded in plane order, so the result
 * does not depend on the OpenMP thread count.
 *
 * Layout (oracle-private, deliberately different from the GPU's padded one):
 *   dense [(nz+2h)][(ny+2h)][(nx+2h)], x fastest; interior (x,y,z) sits at
 *   ((z+h)*(ny+2h) + (y+h))*(nx+2h) + (x+h).
 */
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

/* ---- catalogue numbering (kept equal to the ABI's by convention only; the
 *      tests map both sides by name) ---- */
enum Op { FIG1B = 0, LAP7 = 1, JACOBI7 = 2, LAP27 = 3, JACOBI27 = 4, VARCOEF8 = 5 };
enum Rop {
  R_VALUE = 0, R_SQ = 1, R_ABSDIFF = 2, R_CONV = 3, R_RESID7_SQ = 4, R_RESID27_SQ = 5,
  R_JACOBI7_RESID7_SQ = 6, R_JACOBI27_RESID27_SQ = 7, R_FIG1B_CONV = 8
};
enum Comb { SUM = 0, MAX = 1, MIN = 2, AND = 3 };

/* A borrowed dense grid with its own halo width. */
template <typename T> struct G {
  T* p; int64_t nx, ny, nz; int h;
  T& at(int64_t x, int64_t y, int64_t z) const {
    return p[((z + h) * (ny + 2 * h) + (y + h)) * (nx + 2 * h) + (x + h)];
  }
};

/* Constants: the correctly rounded literals (R3). 1.0/36.0 and
 * 1.0/6.0 are folded by the compiler exactly as C++ folds Fig 1.b's
 * "1.0/36.0". */
template <typename T> struct K;
template <> struct K<double> {
  static constexpr double c36 = 1.0 / 36.0, c6 = 1.0 / 6.0, inv128 = 0.0078125;
};
template <> struct K<float> {
  static constexpr float c36 = 1.0f / 36.0f, c6 = 1.0f / 6.0f, inv128 = 0.0078125f;
};

/* ---------------- per-point expression trees -------------- */

/* FIG1B, left to right as printed:
 *   v() = 1.0/36.0 *(6*u() - u(1,0,0) - u(-1,0,0) - u(0,1,0) - u(0,-1,0)
 *                          - u(0,0,1) - u(0,0,-1));
 * with the paper's u(a,b,c) read as u(dx,dy,dz) (reading R2). */
template <typename T> T fig1b(const G<T>& u, int64_t x, int64_t y, int64_t z) {
  T s = T(6) * u.at(x, y, z);
  s = s - u.at(x + 1, y, z);
  s = s - u.at(x - 1, y, z);
  s = s - u.at(x, y + 1, z);
  s = s - u.at(x, y - 1, z);
  s = s - u.at(x, y, z + 1);
  s = s - u.at(x, y, z - 1);
  return K<T>::c36 * s;
}

/* The 7-point neighbour sum S = (sx + sy) + sz (reading R4). */
template <typename T> T sum6(const G<T>& u, int64_t x, int64_t y, int64_t z) {
  T sx = u.at(x - 1, y, z) + u.at(x + 1, y, z);
  T sy = u.at(x, y - 1, z) + u.at(x, y + 1, z);
  T sz = u.at(x, y, z - 1) + u.at(x, y, z + 1);
  return (sx + sy) + sz;
}
/* LAP7: L = S - 6*u (unit spacing). */
template <typename T> T lap7(const G<T>& u, int64_t x, int64_t y, int64_t z) {
  T S = sum6(u, x, y, z);
  T c = T(6) * u.at(x, y, z);
  return S - c;
}
/* JACOBI7 (Laplace, f = 0): v = S * fl(1/6). */
template <typename T> T jacobi7(const G<T>& u, int64_t x, int64_t y, int64_t z) {
  return sum6(u, x, y, z) * K<T>::c6;
}

/* 27-point bracket B = (14*Sf + 3*Se) + Sc, grouped by z-plane (reading R5):
 *   C_q = u(0,0,q)
 *   X_q = (u(-1,0,q) + u(+1,0,q)) + (u(0,-1,q) + u(0,+1,q))
 *   D_q = (u(-1,-1,q) + u(+1,-1,q)) + (u(-1,+1,q) + u(+1,+1,q))
 *   Sf = X_0 + (C_-1 + C_+1);  Se = D_0 + (X_-1 + X_+1);  Sc = D_-1 + D_+1 */
template <typename T> T bracket27(const G<T>& u, int64_t x, int64_t y, int64_t z) {
  T C[3], X[3], D[3];
  for (int q = -1; q <= 1; ++q) {
    C[q + 1] = u.at(x, y, z + q);
    X[q + 1] = (u.at(x - 1, y, z + q) + u.at(x + 1, y, z + q)) +
               (u.at(x, y - 1, z + q) + u.at(x, y + 1, z + q));
    D[q + 1] = (u.at(x - 1, y - 1, z + q) + u.at(x + 1, y - 1, z + q)) +
               (u.at(x - 1, y + 1, z + q) + u.at(x + 1, y + 1, z + q));
  }
  T Sf = X[1] + (C[0] + C[2]);
  T Se = D[1] + (X[0] + X[2]);
  T Sc = D[0] + D[2];
  T a = T(14) * Sf;
  T b = T(3) * Se;
  return (a + b) + Sc;
}
/* LAP27: L = (B - 128*u0) / 30, weights (1/30)[-128, 14, 3, 1] (reading R6). */
template <typename T> T lap27(const G<T>& u, int64_t x, int64_t y, int64_t z) {
  T B = bracket27(u, x, y, z);
  T c = T(128) * u.at(x, y, z);
  return (B - c) / T(30);
}
/* JACOBI27: v = B * 2^-7, the point where LAP27 vanishes. */
template <typename T> T jacobi27(const G<T>& u, int64_t x, int64_t y, int64_t z) {
  return bracket27(u, x, y, z) * K<T>::inv128;
}

/* VARCOEF8: u plus seven centre-only coefficient grids (reading R7). */
template <typename T>
T varcoef8(const G<T>* g, int64_t x, int64_t y, int64_t z) {
  const G<T>& u = g[0];
  T a = g[1].at(x, y, z) * u.at(x, y, z);
  a = a + g[2].at(x, y, z) * u.at(x - 1, y, z);
  a = a + g[3].at(x, y, z) * u.at(x + 1, y, z);
  a = a + g[4].at(x, y, z) * u.at(x, y - 1, z);
  a = a + g[5].at(x, y, z) * u.at(x, y + 1, z);
  a = a + g[6].at(x, y, z) * u.at(x, y, z - 1);
  a = a + g[7].at(x, y, z) * u.at(x, y, z + 1);
  return a;
}

template <typename T> T apply_op(int op, const G<T>* in, int64_t x, int64_t y, int64_t z) {
  switch (op) {
    case FIG1B: return fig1b(in[0], x, y, z);
    case LAP7: return lap7(in[0], x, y, z);
    case JACOBI7: return jacobi7(in[0], x, y, z);
    case LAP27: return lap27(in[0], x, y, z);
    case JACOBI27: return jacobi27(in[0], x, y, z);
    default: return varcoef8(in, x, y, z);
  }
}

int op_arity(int op) { return op == VARCOEF8 ? 8 : 1; }
int op_footprint(int op, int grid) { return (op == VARCOEF8 && grid > 0) ? 0 : 1; }

/* The value a reduce op contributes at one point, computed in T and then
 * widened (R8).  For the fused ops *w receives the written value. */
template <typename T>
T reduce_val(int rop, const G<T>* g, int64_t x, int64_t y, int64_t z, double eps, T* w) {
  switch (rop) {
    case R_VALUE: return g[0].at(x, y, z);
    case R_SQ: { T a = g[0].at(x, y, z); return a * a; }
    case R_ABSDIFF: { T d = g[0].at(x, y, z) - g[1].at(x, y, z); return std::fabs(d); }
    case R_CONV: { T d = g[0].at(x, y, z) - g[1].at(x, y, z); return std::fabs(d) <= T(eps) ? T(1) : T(0); }
    case R_RESID7_SQ: { T L = lap7(g[0], x, y, z); return L * L; }
    case R_RESID27_SQ: { T L = lap27(g[0], x, y, z); return L * L; }
    case R_JACOBI7_RESID7_SQ: { *w = jacobi7(g[0], x, y, z); T L = lap7(g[0], x, y, z); return L * L; }
    case R_JACOBI27_RESID27_SQ: { *w = jacobi27(g[0], x, y, z); T L = lap27(g[0], x, y, z); return L * L; }
    default: { /* R_FIG1B_CONV: v = FIG1B(u); ok = |v - u| <= eps */
      T v = fig1b(g[0], x, y, z); *w = v; T d = v - g[0].at(x, y, z);
      return std::fabs(d) <= T(eps) ? T(1) : T(0);
    }
  }
}
bool rop_writes(int rop) { return rop >= R_JACOBI7_RESID7_SQ; }

long double comb_identity(int c) {
  switch (c) {
    case SUM: return 0.0L;
    case MAX: return -INFINITY;
    case MIN: return INFINITY;
    default: return 1.0L;
  }
}
long double comb(int c, long double a, long double b) {
  switch (c) {
    case SUM: return a + b;
    case MAX: return b > a ? b : a;
    case MIN: return b < a ? b : a;
    default: return (a != 0.0L && b != 0.0L) ? 1.0L : 0.0L;
  }
}

struct Range { int64_t x0, x1, y0, y1, z0, z1; };

template <typename T>
void do_all(int op, const G<T>* in, const G<T>& out, const Range& r) {
#pragma omp parallel for schedule(static)
  for (int64_t z = r.z0; z < r.z1; ++z)
    for (int64_t y = r.y0; y < r.y1; ++y)
      for (int64_t x = r.x0; x < r.x1; ++x) out.at(x, y, z) = apply_op(op, in, x, y, z);
}

template <typename T>
void do_reduce(int rop, const G<T>* g, const G<T>* out, int c, const Range& r, double eps,
               double* result, double* abs_sum) {
  int64_t nzr = r.z1 > r.z0 ? r.z1 - r.z0 : 0;
  std::vector<long double> part(nzr), apart(nzr);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nzr; ++k) {
    int64_t z = r.z0 + k;
    long double acc = comb_identity(c), aacc = 0.0L;
    for (int64_t y = r.y0; y < r.y1; ++y)
      for (int64_t x = r.x0; x < r.x1; ++x) {
        T w = T(0);
        T v = reduce_val(rop, g, x, y, z, eps, &w);
        if (out) out->at(x, y, z) = w;
        acc = comb(c, acc, (long double)v);
        aacc += std::fabs((long double)v);
      }
    part[k] = acc; apart[k] = aacc;
  }
  long double acc = comb_identity(c), aacc = 0.0L;
  for (int64_t k = 0; k < nzr; ++k) { acc = comb(c, acc, part[k]); aacc += apart[k]; }
  *result = (double)acc;
  if (abs_sum) *abs_sum = (double)aacc;
}

/* splitmix64 (Steele, Lea, Flood 2014): the counter hash of reading R9. */
uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T> T u01(uint64_t h);
template <> double u01<double>(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
template <> float u01<float>(uint64_t h) { return (float)(h >> 40) * 0x1.0p-24f; }

template <typename T> G<T> mk(void* p, int64_t nx, int64_t ny, int64_t nz, int h) {
  return G<T>{static_cast<T*>(p), nx, ny, nz, h};
}

}  // namespace

/* ============================== C interface ============================== */
/* dtype: 0 = binary64, 1 = binary32.  All extents are LOCAL (the array's own
 * nz); z_off is the global z of local plane 0 and NX, NY, NZ the global
 * interior extents, used only by the generator and the digest. */
extern "C" {

uint64_t og_splitmix64(uint64_t x) { return splitmix64(x); }

int og_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void og_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* Reading R9: interior value = U[0,1)(splitmix64(seed ^ grid_id<<48 ^ gidx))
 * * scale, gidx = (z*NY + y)*NX + x over GLOBAL interior coordinates; halo
 * cells are set to 0 (zero Dirichlet boundary). */
void og_fill_random(int dtype, void* p, int64_t nx, int64_t ny, int64_t nz, int h, int64_t z_off,
                    uint64_t seed, uint32_t grid_id, double scale) {
  int64_t n = (nx + 2 * h) * (ny + 2 * h) * (nz + 2 * h);
  uint64_t base = seed ^ ((uint64_t)grid_id << 48);
  if (dtype == 0) {
    G<double> g = mk<double>(p, nx, ny, nz, h);
    std::memset(p, 0, (size_t)n * sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < nz; ++z)
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) {
          uint64_t gidx = (uint64_t)(((z + z_off) * ny + y) * nx + x);
          g.at(x, y, z) = u01<double>(splitmix64(base ^ gidx)) * scale;
        }
  } else {
    G<float> g = mk<float>(p, nx, ny, nz, h);
    std::memset(p, 0, (size_t)n * sizeof(float));
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < nz; ++z)
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) {
          uint64_t gidx = (uint64_t)(((z + z_off) * ny + y) * nx + x);
          g.at(x, y, z) = u01<float>(splitmix64(base ^ gidx)) * (float)scale;
        }
  }
}

/* A window of the global generated field (reading R9): a dense array of
 * interior size bx*by*bz plus halo h whose interior cell (i,j,k) is the global
 * point (x_off+i, y_off+j, z_off+k) of an NX*NY*NZ grid; cells outside the
 * global interior (its halo) are 0.  Used for sampled parity at full size. */
void og_fill_random_window(int dtype, void* p, int64_t bx, int64_t by, int64_t bz, int h,
                           int64_t x_off, int64_t y_off, int64_t z_off, int64_t NX, int64_t NY,
                           int64_t NZ, uint64_t seed, uint32_t grid_id, double scale) {
  uint64_t base = seed ^ ((uint64_t)grid_id << 48);
  for (int64_t k = -h; k < bz + h; ++k)
    for (int64_t j = -h; j < by + h; ++j)
      for (int64_t i = -h; i < bx + h; ++i) {
        int64_t x = x_off + i, y = y_off + j, z = z_off + k;
        bool in = x >= 0 && x < NX && y >= 0 && y < NY && z >= 0 && z < NZ;
        uint64_t gidx = in ? (uint64_t)((z * NY + y) * NX + x) : 0;
        if (dtype == 0) {
          G<double> g = mk<double>(p, bx, by, bz, h);
          g.at(i, j, k) = in ? u01<double>(splitmix64(base ^ gidx)) * scale : 0.0;
        } else {
          G<float> g = mk<float>(p, bx, by, bz, h);
          g.at(i, j, k) = in ? u01<float>(splitmix64(base ^ gidx)) * (float)scale : 0.0f;
        }
      }
}

/* Order-independent digest of the interior (reading R10):
 *   sum over interior cells of splitmix64(bits(value) ^ splitmix64(gidx)) mod 2^64. */
uint64_t og_digest(int dtype, const void* p, int64_t nx, int64_t ny, int64_t nz, int h,
                   int64_t z_off) {
  std::vector<uint64_t> part(nz > 0 ? nz : 0);
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < nz; ++z) {
    uint64_t acc = 0;
    for (int64_t y = 0; y < ny; ++y)
      for (int64_t x = 0; x < nx; ++x) {
        uint64_t gidx = (uint64_t)(((z + z_off) * ny + y) * nx + x);
        uint64_t bits;
        if (dtype == 0) {
          double v = mk<double>(const_cast<void*>(p), nx, ny, nz, h).at(x, y, z);
          std::memcpy(&bits, &v, 8);
        } else {
          float v = mk<float>(const_cast<void*>(p), nx, ny, nz, h).at(x, y, z);
          uint32_t b32; std::memcpy(&b32, &v, 4); bits = b32;
        }
        acc += splitmix64(bits ^ splitmix64(gidx));
      }
    part[z] = acc;
  }
  uint64_t acc = 0;
  for (int64_t z = 0; z < nz; ++z) acc += part[z];
  return acc;
}

/* do_all: out(p) = OP(in...) for every p in the LOCAL half-open range r
 * (x0,x1,y0,y1,z0,z1).  halos[i] is the halo of in[i]; out_h that of out.
 * Returns 0, or -1 on a bad argument (arity, halo below the footprint). */
int og_do_all(int op, int dtype, void* const* in, const int* halos, int n_in, void* out,
              int out_h, int64_t nx, int64_t ny, int64_t nz, const int64_t* r6) {
  if (op < FIG1B || op > VARCOEF8 || n_in != op_arity(op)) return -1;
  for (int i = 0; i < n_in; ++i)
    if (halos[i] < op_footprint(op, i)) return -1;
  Range r{r6[0], r6[1], r6[2], r6[3], r6[4], r6[5]};
  if (dtype == 0) {
    G<double> g[8];
    for (int i = 0; i < n_in; ++i) g[i] = mk<double>(in[i], nx, ny, nz, halos[i]);
    do_all(op, g, mk<double>(out, nx, ny, nz, out_h), r);
  } else {
    G<float> g[8];
    for (int i = 0; i < n_in; ++i) g[i] = mk<float>(in[i], nx, ny, nz, halos[i]);
    do_all(op, g, mk<float>(out, nx, ny, nz, out_h), r);
  }
  return 0;
}

/* do_reduce (fused ops also write `out`, which may be NULL otherwise).
 * result = the combine over r; abs_sum = sum |val| (the tolerance scale). */
int og_do_reduce(int rop, int dtype, void* const* g_in, const int* halos, int n, void* out,
                 int out_h, int64_t nx, int64_t ny, int64_t nz, const int64_t* r6, int combine,
                 double eps, double* result, double* abs_sum) {
  int need = (rop == R_ABSDIFF || rop == R_CONV) ? 2 : 1;
  if (rop < R_VALUE || rop > R_FIG1B_CONV || n != need) return -1;
  if (combine < SUM || combine > AND) return -1;
  if (rop_writes(rop) && !out) return -1;
  bool stencil = rop == R_RESID7_SQ || rop == R_RESID27_SQ || rop_writes(rop);
  if (stencil && halos[0] < 1) return -1;
  Range r{r6[0], r6[1], r6[2], r6[3], r6[4], r6[5]};
  if (dtype == 0) {
    G<double> g[2];
    for (int i = 0; i < n; ++i) g[i] = mk<double>(g_in[i], nx, ny, nz, halos[i]);
    G<double> o = mk<double>(out, nx, ny, nz, out_h);
    do_reduce(rop, g, rop_writes(rop) ? &o : nullptr, combine, r, eps, result, abs_sum);
  } else {
    G<float> g[2];
    for (int i = 0; i < n; ++i) g[i] = mk<float>(g_in[i], nx, ny, nz, halos[i]);
    G<float> o = mk<float>(out, nx, ny, nz, out_h);
    do_reduce(rop, g, rop_writes(rop) ? &o : nullptr, combine, r, eps, result, abs_sum);
  }
  return 0;
}

/* Single-domain jacobi_run (PAPER.md:161-170 with a fixed iteration count,
 * reading R11).  u, v: state buffers with halo h >= 1; coeffs: 7 grids with
 * halo ch (VARCOEF8 only).  Before the first sweep u's halo shell is copied
 * into v (Dirichlet boundary travels with both buffers).  Sweep it = 1..iters:
 *   if check_every > 0 and it % check_every == 0, the sweep is fused with the
 *   check value of its INPUT iterate and hist[it/check_every - 1] = sqrt(sum);
 *   then swap.  If check_every > 0, hist[iters/check_every] = the check value
 *   of the final iterate (a standalone pass).  The check value is RESID7_SQ
 *   for JACOBI7, RESID27_SQ for JACOBI27 and SQ (of u) for VARCOEF8.
 * On return the final iterate is in *u_final (0 = u, 1 = v). */
int og_jacobi_run(int op, int dtype, void* u, void* v, int h, void* const* coeffs, int ch,
                  int64_t nx, int64_t ny, int64_t nz, int iters, int check_every, double* hist,
                  int* u_final) {
  if (op != JACOBI7 && op != JACOBI27 && op != VARCOEF8) return -1;
  if (h < 1 || iters < 0 || check_every < 0) return -1;
  size_t es = dtype == 0 ? 8 : 4;
  int64_t px = nx + 2 * h, py = ny + 2 * h, pz = nz + 2 * h;
  /* copy the halo shell of u into v */
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < pz; ++z)
    for (int64_t y = 0; y < py; ++y)
      for (int64_t x = 0; x < px; ++x) {
        bool halo = z < h || z >= nz + h || y < h || y >= ny + h || x < h || x >= nx + h;
        if (halo) {
          size_t o = (size_t)(((z * py) + y) * px + x) * es;
          std::memcpy((char*)v + o, (char*)u + o, es);
        }
      }
  int64_t r6[6] = {0, nx, 0, ny, 0, nz};
  void* a = u;
  void* b = v;
  int check_rop = op == JACOBI7 ? R_RESID7_SQ : op == JACOBI27 ? R_RESID27_SQ : R_SQ;
  for (int it = 1; it <= iters; ++it) {
    void* in[8] = {a};
    int hal[8] = {h};
    for (int i = 0; i < 7 && op == VARCOEF8; ++i) { in[i + 1] = coeffs[i]; hal[i + 1] = ch; }
    bool check = check_every > 0 && it % check_every == 0;
    if (check) {
      double s = 0, as = 0;
      if (op == VARCOEF8) {
        og_do_reduce(R_SQ, dtype, in, hal, 1, nullptr, 0, nx, ny, nz, r6, SUM, 0, &s, &as);
        og_do_all(op, dtype, in, hal, 8, b, h, nx, ny, nz, r6);
      } else {
        int frop = op == JACOBI7 ? R_JACOBI7_RESID7_SQ : R_JACOBI27_RESID27_SQ;
        og_do_reduce(frop, dtype, in, hal, 1, b, h, nx, ny, nz, r6, SUM, 0, &s, &as);
      }
      hist[it / check_every - 1] = std::sqrt(s);
    } else {
      og_do_all(op, dtype, in, hal, op == VARCOEF8 ? 8 : 1, b, h, nx, ny, nz, r6);
    }
    void* t = a; a = b; b = t;
  }
  if (check_every > 0) {
    void* in[1] = {a};
    int hal[1] = {h};
    double s = 0, as = 0;
    og_do_reduce(check_rop, dtype, in, hal, 1, nullptr, 0, nx, ny, nz, r6, SUM, 0, &s, &as);
    hist[iters / check_every] = std::sqrt(s);
  }
  *u_final = (a == u) ? 0 : 1;
  return 0;
}

/* The paper's convergence-terminated fused loop (§5.2):
 *   do { swap_grids(); res = do_reduce(now, before, fuse(OP, convergence(EPSI)), and) }
 *   while (!res);
 * Iteration it (1-based) computes b = OP(a) and res = AND_p (|b(p) - a(p)| <= eps)
 * (FIG1B_CONV for FIG1B, the same test after JACOBI7 for JACOBI7), then the
 * roles swap.  Stops at the first iteration with res = 1, or after max_iters.
 * Before the first sweep u's halo shell is copied into v (reading R11).
 * *iters_done = iterations executed, *converged = res of the last one; the
 * final iterate is in u (*u_final = 0) or v (1). */
int og_converge_run(int op, int dtype, void* u, void* v, int h, int64_t nx, int64_t ny, int64_t nz,
                    double eps, int max_iters, int* iters_done, int* converged, int* u_final) {
  if (op != FIG1B && op != JACOBI7) return -1;
  if (h < 1 || max_iters < 0) return -1;
  size_t es = dtype == 0 ? 8 : 4;
  int64_t px = nx + 2 * h, py = ny + 2 * h, pz = nz + 2 * h;
#pragma omp parallel for schedule(static)
  for (int64_t z = 0; z < pz; ++z)
    for (int64_t y = 0; y < py; ++y)
      for (int64_t x = 0; x < px; ++x) {
        bool halo = z < h || z >= nz + h || y < h || y >= ny + h || x < h || x >= nx + h;
        if (halo) {
          size_t o = (size_t)(((z * py) + y) * px + x) * es;
          std::memcpy((char*)v + o, (char*)u + o, es);
        }
      }
  int64_t r6[6] = {0, nx, 0, ny, 0, nz};
  void* a = u;
  void* b = v;
  int it = 0;
  double res = 0.0;
  while (it < max_iters) {
    ++it;
    void* in[1] = {a};
    int hal[1] = {h};
    double as = 0;
    if (op == FIG1B) {
      og_do_reduce(R_FIG1B_CONV, dtype, in, hal, 1, b, h, nx, ny, nz, r6, AND, eps, &res, &as);
    } else {
      og_do_all(JACOBI7, dtype, in, hal, 1, b, h, nx, ny, nz, r6);
      void* pair[2] = {b, a};
      int hh[2] = {h, h};
      og_do_reduce(R_CONV, dtype, pair, hh, 2, nullptr, 0, nx, ny, nz, r6, AND, eps, &res, &as);
    }
    void* t = a; a = b; b = t;
    if (res != 0.0) break;
  }
  *iters_done = it;
  *converged = res != 0.0 ? 1 : 0;
  *u_final = (a == u) ? 0 : 1;
  return 0;
}

/* Red-black Gauss-Seidel for the 7-point Laplace equation (NEXT-3; PAPER.md:
 * 107-109: "stateful" stencil shapes expose the indices of the accessed
 * elements, "useful ... for implementing red-black Gauss-Siedel").  Colour of a
 * point = (x + y + z_global) mod 2 (global coordinates; z_global = z + z_off).
 * One iteration = the red half-sweep (colour 0) then the black one (colour 1);
 * a half-sweep sets u(p) = JACOBI7(u)(p) in place at every interior point of
 * its colour (those points read only points of the other colour).  History as
 * jacobi_run: when it % check_every == 0, hist[it/k - 1] = sqrt(sum RESID7^2)
 * of the iterate before iteration it; hist[iters/k] of the final iterate. */
int og_rbgs_run(int dtype, void* u, int h, int64_t nx, int64_t ny, int64_t nz, int64_t z_off,
                int iters, int check_every, double* hist) {
  if (h < 1 || iters < 0 || check_every < 0) return -1;
  int64_t r6[6] = {0, nx, 0, ny, 0, nz};
  auto resid = [&](double* out) {
    void* in[1] = {u};
    int hal[1] = {h};
    double s = 0, as = 0;
    og_do_reduce(R_RESID7_SQ, dtype, in, hal, 1, nullptr, 0, nx, ny, nz, r6, SUM, 0, &s, &as);
    *out = std::sqrt(s);
  };
  for (int it = 1; it <= iters; ++it) {
    if (check_every > 0 && it % check_every == 0) resid(&hist[it / check_every - 1]);
    for (int color = 0; color < 2; ++color) {
      if (dtype == 0) {
        G<double> g = mk<double>(u, nx, ny, nz, h);
#pragma omp parallel for schedule(static)
        for (int64_t z = 0; z < nz; ++z)
          for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x)
              if (((x + y + z + z_off) & 1) == color) g.at(x, y, z) = jacobi7(g, x, y, z);
      } else {
        G<float> g = mk<float>(u, nx, ny, nz, h);
#pragma omp parallel for schedule(static)
        for (int64_t z = 0; z < nz; ++z)
          for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x)
              if (((x + y + z + z_off) & 1) == color) g.at(x, y, z) = jacobi7(g, x, y, z);
      }
    }
  }
  if (check_every > 0) resid(&hist[iters / check_every]);
  return 0;
}

/* Ordered iteration spaces (NEXT-4; §3):
 *   do_i_inc / do_j_inc / do_k_inc: cell (i-1,j,k) / (i,j-1,k) / (i,j,k-1) is
 *   processed before (i,j,k) (the paper's "(i,j-1,j)" read as (i,j-1,k));
 *   *_dec: (i+1,..) etc. before (i,j,k); do_diamond: (i-1,j) and (i,j-1) before
 *   (i,j) (2-D: applied to every z plane).
 * space: 0 I_INC, 1 I_DEC, 2 J_INC, 3 J_DEC, 4 K_INC, 5 K_DEC, 6 DIAMOND.
 * op: 0 PREFIX  out(p) = out(p - d) + in(p), d the space's predecessor offset
 *               (out's halo supplies out before the first cell);
 *     1 PASCAL  (DIAMOND only) out(i,j) = out(i-1,j) + out(i,j-1).
 * Evaluated literally in the space's order. */
int og_do_ordered(int space, int op, int dtype, const void* in, int in_h, void* out, int out_h,
                  int64_t nx, int64_t ny, int64_t nz) {
  if (space < 0 || space > 6 || op < 0 || op > 1) return -1;
  if ((op == 1) != (space == 6)) return -1;
  if (out_h < 1 || (op == 0 && !in)) return -1;
  auto run = [&](auto tag) {
    using T = decltype(tag);
    G<T> o = mk<T>(out, nx, ny, nz, out_h);
    G<T> u = mk<T>(const_cast<void*>(in), nx, ny, nz, in_h);
    if (space == 6) {
      for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
          for (int64_t x = 0; x < nx; ++x) o.at(x, y, z) = o.at(x - 1, y, z) + o.at(x, y - 1, z);
      return;
    }
    const int axis = space / 2;
    const bool inc = (space % 2) == 0;
    const int64_t n[3] = {nx, ny, nz};
    for (int64_t a = 0; a < n[(axis + 1) % 3]; ++a)
      for (int64_t b = 0; b < n[(axis + 2) % 3]; ++b)
        for (int64_t s = 0; s < n[axis]; ++s) {
          const int64_t t = inc ? s : n[axis] - 1 - s;
          int64_t c[3];
          c[axis] = t;
          c[(axis + 1) % 3] = a;
          c[(axis + 2) % 3] = b;
          int64_t p[3] = {c[0], c[1], c[2]};
          p[axis] += inc ? -1 : 1;
          o.at(c[0], c[1], c[2]) = o.at(p[0], p[1], p[2]) + u.at(c[0], c[1], c[2]);
        }
  };
  if (dtype == 0) run(double{});
  else run(float{});
  return 0;
}

}  /* extern "C" */
