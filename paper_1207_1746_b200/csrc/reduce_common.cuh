// reduce_common.cuh — deterministic CTA -> grid reduction epilogue.
//
// Each thread folds its own points in a fixed order; a warp butterfly
// (commutative IEEE ops, so every lane ends with the same bits) and an
// in-order fold over warps give the CTA partial; the last CTA to finish (atomic
// ticket) folds the per-CTA partials with all its threads in a fixed order.  The result depends only
// on the launch configuration, never on scheduling (PAPER.md:53 allows any
// order for a commutative reduction; R8).
#pragma once
#include "ops.cuh"

namespace gscl {

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double warp_fold(int comb, double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = comb_apply(comb, v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One partial of the first `nthreads` threads of the CTA (a multiple of 32):
// warp butterfly, in-order fold over the warps, written to *out by thread 0.
// red_smem: >= nthreads/32 doubles (free again on return).
__device__ __forceinline__ void cta_partial(double acc, int comb, double* red_smem, int nthreads, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = nthreads >> 5;
  acc = warp_fold(comb, acc);
  if (lane == 0) red_smem[warp] = acc;
  named_bar_sync(1, nthreads);
  if (threadIdx.x == 0) {
    double t = comb_identity(comb);
    for (int w = 0; w < nw; ++w) t = comb_apply(comb, t, red_smem[w]);
    *out = t;
  }
  named_bar_sync(1, nthreads);
}

__device__ __forceinline__ void grid_fold_last(int comb, double* red_smem, int* flag_smem, int nthreads,
                                               double* partials, unsigned* counter, double* result,
                                               unsigned nblocks, unsigned nparts);

// Called by the first `nthreads` threads of the CTA (a multiple of 32).
// red_smem: >= nthreads/32 doubles; flag_smem: one int.
__device__ __forceinline__ void cta_reduce_finish(double acc, int comb, double* red_smem,
                                                  int* flag_smem, int nthreads, double* partials,
                                                  unsigned* counter, double* result,
                                                  unsigned nblocks, unsigned block_id) {
  cta_partial(acc, comb, red_smem, nthreads, &partials[block_id]);
  grid_fold_last(comb, red_smem, flag_smem, nthreads, partials, counter, result, nblocks, nblocks);
}

// After every CTA has written its partials: the last CTA to arrive (atomic
// ticket over nblocks CTAs) folds partials[0 .. nparts) in index order.
__device__ __forceinline__ void grid_fold_last(int comb, double* red_smem, int* flag_smem, int nthreads,
                                               double* partials, unsigned* counter, double* result,
                                               unsigned nblocks, unsigned nparts) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = nthreads >> 5;
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned ticket = atomicAdd(counter, 1u);
    *flag_smem = (ticket == nblocks - 1) ? 1 : 0;
  }
  named_bar_sync(1, nthreads);
  const unsigned nblk = nparts;
  if (*flag_smem) {  // uniform across the CTA
    __threadfence();
    // all threads of the last CTA fold the partials: thread t takes t, t+n,
    // t+2n, ... in index order (loads issued 8 at a time), then the warp
    // butterfly and the in-order fold over warps — a fixed order per launch
    // configuration, so the result is deterministic.
    double t = comb_identity(comb);
    unsigned i = threadIdx.x;
    const unsigned step = (unsigned)nthreads;
    for (; i + 7 * step < nblk; i += 8 * step) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcg(&partials[i + q * step]);
#pragma unroll
      for (int q = 0; q < 8; ++q) t = comb_apply(comb, t, v[q]);
    }
    for (; i < nblk; i += step) t = comb_apply(comb, t, __ldcg(&partials[i]));
    t = warp_fold(comb, t);
    named_bar_sync(1, nthreads);  // red_smem reuse
    if (lane == 0) red_smem[warp] = t;
    named_bar_sync(1, nthreads);
    if (threadIdx.x == 0) {
      double r = comb_identity(comb);
      for (int w = 0; w < nw; ++w) r = comb_apply(comb, r, red_smem[w]);
      *result = r;
      atomicExch(counter, 0u);
    }
  }
}

}  // namespace gscl
