// ops.cuh — the compiled-in operator catalogue as plane-pipelined functors.
//
// Every operator is written as   out(z) = combine(tuple(z-1), tuple(z), tuple(z+1))
// where tuple(q) is computed once per point from plane q alone.  The 2.5-D
// streaming kernel computes each plane's tuple when the plane lands in shared
// memory and keeps the last three in registers (the z register queue).  The
// grouping below IS the expression tree of DESIGN.md §3 (readings R1-R8), so
// the result equals the oracle's per-point evaluation bit for bit:
//  FIG1B    PAPER.md:68-71 (Fig 1.b), left to right:
//           q = ((((6c - xp) - xm) - yp) - ym);  v = fl(1/36) * ((q - c(z+1)) - c(z-1))
//  LAP7 / JACOBI7   p = (xm + xp) + (ym + yp);  S = p + (c(z-1) + c(z+1))
//           LAP7: S - 6c   JACOBI7: S * fl(1/6)
//  LAP27 / JACOBI27 per plane C = c, X = (xm+xp)+(ym+yp), D = (mm+pm)+(mp+pp);
//           Sf = X0 + (C-1 + C+1); Se = D0 + (X-1 + X+1); Sc = D-1 + D+1;
//           B = (14 Sf + 3 Se) + Sc;  LAP27: (B - 128c)/30   JACOBI27: B * 2^-7
//  VARCOEF8 a = c0 c; a += cxm xm; a += cxp xp; a += cym ym; a += cyp yp  (plane z)
//           v = (a + czm c(z-1)) + czp c(z+1)
// All arithmetic goes through gscl::add/sub/mul/dvd (IEEE RN, never fused).
#pragma once
#include "device.cuh"

namespace gscl {

enum OpCode { OP_FIG1B = 0, OP_LAP7 = 1, OP_JACOBI7 = 2, OP_LAP27 = 3, OP_JACOBI27 = 4, OP_VARCOEF8 = 5 };

// What the sweep kernel reduces besides (or instead of) writing.
enum RedVal {
  RV_NONE = 0,   // do_all
  RV_RESID = 1,  // RESID7_SQ for 7-point ops, RESID27_SQ for 27-point ops (of the input)
  RV_CONV = 2,   // (|out - u| <= eps) ? 1 : 0   (FIG1B_CONV; also JACOBI7)
  RV_SQ = 3,     // u * u of the input centre (the VARCOEF8 jacobi check)
  RV_CONV2 = 4,  // two-sweep pass: AND of |u1 - u| <= eps and AND of |u2 - u1| <= eps
                 // (the convergence tests of both iterations of the pass)
  RV_RESID_IN = 5  // two-sweep pass: RESID7_SQ of the pass's INPUT (red-black GS check)
};

enum Comb { CB_SUM = 0, CB_MAX = 1, CB_MIN = 2, CB_AND = 3 };

__device__ __forceinline__ double comb_identity(int c) {
  return c == CB_SUM ? 0.0 : c == CB_MAX ? -__longlong_as_double(0x7ff0000000000000ll)
                         : c == CB_MIN ? __longlong_as_double(0x7ff0000000000000ll) : 1.0;
}
__device__ __forceinline__ double comb_apply(int c, double a, double b) {
  switch (c) {
    case CB_SUM: return __dadd_rn(a, b);
    case CB_MAX: return b > a ? b : a;
    case CB_MIN: return b < a ? b : a;
    default: return (a != 0.0 && b != 0.0) ? 1.0 : 0.0;
  }
}

// In-plane neighbourhood of one point: centre c, x faces xm/xp, y faces ym/yp,
// and the x pair sums of the point's row and the rows below / above:
//   h0 = xm + xp,  hm = u(-1,-1) + u(+1,-1),  hp = u(-1,+1) + u(+1,+1)
// (hm/hp only for the 27-point ops).  A pair sum is one IEEE addition, so a
// row's h is computed once and shared by the rows above and below it without
// changing any tree: X = h0 + (ym + yp), D = hm + hp.
template <typename T> struct Nbr { T c, xm, xp, ym, yp, h0, hm, hp; };

template <typename T> struct Cst;
template <> struct Cst<double> {
  static __device__ __forceinline__ double c36() { return 1.0 / 36.0; }
  static __device__ __forceinline__ double c6() { return 1.0 / 6.0; }
  static __device__ __forceinline__ double inv128() { return 0.0078125; }
  static __device__ __forceinline__ double c30inv() { return 1.0 / 30.0; }
};
template <> struct Cst<float> {
  static __device__ __forceinline__ float c36() { return 1.0f / 36.0f; }
  static __device__ __forceinline__ float c6() { return 1.0f / 6.0f; }
  static __device__ __forceinline__ float inv128() { return 0.0078125f; }
  static __device__ __forceinline__ float c30inv() { return 1.0f / 30.0f; }
};

template <int OP, typename T> struct OpT;

// ---- FIG1B -----------------------------------------------------------------
template <typename T> struct OpT<OP_FIG1B, T> {
  static constexpr bool DIAG = false;
  static constexpr int NCOEF = 0;
  struct Tup { T c, q; };
  __device__ __forceinline__ static Tup plane(const Nbr<T>& n, const T*) {
    T q = mul(T(6), n.c);
    q = sub(q, n.xp);
    q = sub(q, n.xm);
    q = sub(q, n.yp);
    q = sub(q, n.ym);
    return {n.c, q};
  }
  __device__ __forceinline__ static T out(const Tup& lo, const Tup& mid, const Tup& hi) {
    T s = sub(sub(mid.q, hi.c), lo.c);
    return mul(Cst<T>::c36(), s);
  }
  __device__ __forceinline__ static T resid(const Tup&, const Tup&, const Tup&) { return T(0); }
  __device__ __forceinline__ static T resid_sum(const Tup&, const Tup&, const Tup&) { return T(0); }
};

// ---- LAP7 / JACOBI7 ----------------------------------------------------------
template <typename T> struct Sum7 {
  static constexpr bool DIAG = false;
  static constexpr int NCOEF = 0;
  struct Tup { T c, p; };
  __device__ __forceinline__ static Tup plane(const Nbr<T>& n, const T*) {
    T sy = add(n.ym, n.yp);
    return {n.c, add(n.h0, sy)};  // (sx + sy), sx = h0
  }
  __device__ __forceinline__ static T S(const Tup& lo, const Tup& mid, const Tup& hi) {
    return add(mid.p, add(lo.c, hi.c));
  }
  __device__ __forceinline__ static T lap(const Tup& lo, const Tup& mid, const Tup& hi) {
    return sub(S(lo, mid, hi), mul(T(6), mid.c));
  }
  __device__ __forceinline__ static T resid(const Tup& lo, const Tup& mid, const Tup& hi) {
    T L = lap(lo, mid, hi);
    return mul(L, L);
  }
  __device__ __forceinline__ static T resid_sum(const Tup& lo, const Tup& mid, const Tup& hi) {
    return resid(lo, mid, hi);
  }
};
template <typename T> struct OpT<OP_LAP7, T> : Sum7<T> {
  using Tup = typename Sum7<T>::Tup;
  __device__ __forceinline__ static T out(const Tup& lo, const Tup& mid, const Tup& hi) { return Sum7<T>::lap(lo, mid, hi); }
};
template <typename T> struct OpT<OP_JACOBI7, T> : Sum7<T> {
  using Tup = typename Sum7<T>::Tup;
  __device__ __forceinline__ static T out(const Tup& lo, const Tup& mid, const Tup& hi) {
    return mul(Sum7<T>::S(lo, mid, hi), Cst<T>::c6());
  }
};

// ---- LAP27 / JACOBI27 --------------------------------------------------------
template <typename T> struct Sum27 {
  static constexpr bool DIAG = true;
  static constexpr int NCOEF = 0;
  struct Tup { T c, x, d; };
  __device__ __forceinline__ static Tup plane(const Nbr<T>& n, const T*) {
    T X = add(n.h0, add(n.ym, n.yp));  // (xm + xp) + (ym + yp)
    T D = add(n.hm, n.hp);             // (mm + pm) + (mp + pp)
    return {n.c, X, D};
  }
  __device__ __forceinline__ static T B(const Tup& lo, const Tup& mid, const Tup& hi) {
    T Sf = add(mid.x, add(lo.c, hi.c));
    T Se = add(mid.d, add(lo.x, hi.x));
    T Sc = add(lo.d, hi.d);
    return add(add(mul(T(14), Sf), mul(T(3), Se)), Sc);
  }
  __device__ __forceinline__ static T lap(const Tup& lo, const Tup& mid, const Tup& hi) {
    return dvd(sub(B(lo, mid, hi), mul(T(128), mid.c)), T(30));
  }
  __device__ __forceinline__ static T resid(const Tup& lo, const Tup& mid, const Tup& hi) {
    T L = lap(lo, mid, hi);
    return mul(L, L);
  }
  // fp64 SUM reductions use L = (B - 128c) * fl(1/30) instead of the division
  // of LAP27's tree: within 2 ulp of it, so each L^2 term is within ~1e-15
  // relative (SUMs are compared within 1e-10, R15), without the
  // multi-instruction IEEE division in the fused sweep.  MAX / MIN (exact
  // combines) and fp32 (whose ulp exceeds the 1e-10 bar) keep the division.
  __device__ __forceinline__ static T resid_sum(const Tup& lo, const Tup& mid, const Tup& hi) {
    if constexpr (sizeof(T) == 8) {
      T L = mul(sub(B(lo, mid, hi), mul(T(128), mid.c)), Cst<T>::c30inv());
      return mul(L, L);
    } else {
      return resid(lo, mid, hi);
    }
  }
};
template <typename T> struct OpT<OP_LAP27, T> : Sum27<T> {
  using Tup = typename Sum27<T>::Tup;
  __device__ __forceinline__ static T out(const Tup& lo, const Tup& mid, const Tup& hi) { return Sum27<T>::lap(lo, mid, hi); }
};
template <typename T> struct OpT<OP_JACOBI27, T> : Sum27<T> {
  using Tup = typename Sum27<T>::Tup;
  __device__ __forceinline__ static T out(const Tup& lo, const Tup& mid, const Tup& hi) {
    return mul(Sum27<T>::B(lo, mid, hi), Cst<T>::inv128());
  }
};

// ---- VARCOEF8 ---------------------------------------------------------------
// cf[] = c0, cxm, cxp, cym, cyp, czm, czp at this point (centre-only reads).
template <typename T> struct OpT<OP_VARCOEF8, T> {
  static constexpr bool DIAG = false;
  static constexpr int NCOEF = 7;
  struct Tup { T c, a, czm, czp; };
  __device__ __forceinline__ static Tup plane(const Nbr<T>& n, const T* cf) {
    T a = mul(cf[0], n.c);
    a = add(a, mul(cf[1], n.xm));
    a = add(a, mul(cf[2], n.xp));
    a = add(a, mul(cf[3], n.ym));
    a = add(a, mul(cf[4], n.yp));
    return {n.c, a, cf[5], cf[6]};
  }
  __device__ __forceinline__ static T out(const Tup& lo, const Tup& mid, const Tup& hi) {
    T a = add(mid.a, mul(mid.czm, lo.c));
    return add(a, mul(mid.czp, hi.c));
  }
  __device__ __forceinline__ static T resid(const Tup&, const Tup&, const Tup&) { return T(0); }
  __device__ __forceinline__ static T resid_sum(const Tup&, const Tup&, const Tup&) { return T(0); }
};

// The value the sweep epilogue reduces at one point (widened to double).
template <int OP, int RV, typename T, int CB = -1>
__device__ __forceinline__ double red_value(const typename OpT<OP, T>::Tup& lo,
                                            const typename OpT<OP, T>::Tup& mid,
                                            const typename OpT<OP, T>::Tup& hi, T v, T eps) {
  if constexpr (RV == RV_RESID) {
    if constexpr (CB == CB_SUM) return (double)OpT<OP, T>::resid_sum(lo, mid, hi);
    return (double)OpT<OP, T>::resid(lo, mid, hi);
  } else if constexpr (RV == RV_CONV) {
    T d = sub(v, mid.c);
    return fabs(d) <= eps ? 1.0 : 0.0;
  } else if constexpr (RV == RV_SQ) {
    return (double)mul(mid.c, mid.c);
  } else {
    return 0.0;
  }
}

}  // namespace gscl
