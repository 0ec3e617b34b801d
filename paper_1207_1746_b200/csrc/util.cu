// util.cu — the non-stencil kernels of the hot path: the counter-based input
// generator (R9), constant fill, halo-shell copy (R11), the
// order-independent digest (R10), point-wise do_reduce (R8) and the
// rank-order fold used after the cross-GPU all-gather (R14); plus the TMA
// descriptor encoder.
#include <algorithm>
#include <mutex>

#include <cudaTypedefs.h>

#include <vector>

#include "internal.h"
#include "reduce_common.cuh"

namespace gscl {

GSCL_MODULE_ANCHOR(anchor_util)


namespace {

template <typename T> __device__ __forceinline__ T u01(uint64_t h);
template <> __device__ __forceinline__ double u01<double>(uint64_t h) {
  return (double)(h >> 11) * 0x1.0p-53;
}
template <> __device__ __forceinline__ float u01<float>(uint64_t h) {
  return (float)(h >> 40) * 0x1.0p-24f;
}

// Cell linear index over the whole allocation -> (col,row,plane) array coords.
struct Geom {
  int64_t pitch, rows, planes;  // rows = ny+2h, planes = nzl+2h
  int64_t ox;                   // column of interior x = 0
  int64_t nx, ny, nzl;
  int h;
};

__host__ Geom geom_of(const View& v) {
  return Geom{v.pitch, v.ny + 2 * v.h, v.nzl + 2 * v.h, v.ox, v.nx, v.ny, v.nzl, v.h};
}

template <typename T>
__global__ void k_fill_random(T* base, Geom g, int64_t z_begin, uint64_t key, T scale) {
  const int64_t n = g.pitch * g.rows * g.planes;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i % g.pitch;
    const int64_t rp = i / g.pitch;
    const int64_t row = rp % g.rows;
    const int64_t pl = rp / g.rows;
    const int64_t x = col - g.ox, y = row - g.h, z = pl - g.h;
    T v = T(0);
    if (x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < g.nzl) {
      const uint64_t gidx = (uint64_t)(((z + z_begin) * g.ny + y) * g.nx + x);
      v = mul(u01<T>(splitmix64(key ^ gidx)), scale);
    }
    base[i] = v;
  }
}

template <typename T> __global__ void k_fill_const(T* base, int64_t n, T value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    base[i] = value;
}

// Copy every cell of the logical halo shell (not the row padding) src -> dst.
// One block row per array plane (blockIdx.y): halo planes are copied whole;
// interior planes copy their h first / last rows and the 2h edge cells of each
// interior row — only halo cells are touched.
template <typename T> __global__ void k_copy_halo(const T* src, T* dst, Geom g) {
  const int64_t w = g.nx + 2 * g.h;
  const int64_t pl = blockIdx.y;
  const int64_t base = pl * g.rows * g.pitch + (g.ox - g.h);
  const bool halo_plane = pl < g.h || pl >= g.nzl + g.h;
  const int64_t n = halo_plane ? g.rows * w : 2 * g.h * w + g.ny * 2 * g.h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row, xx;
    if (halo_plane) {
      row = i / w;
      xx = i % w;
    } else if (i < 2 * g.h * w) {  // the h rows below and above the interior
      const int64_t r = i / w;
      row = r < g.h ? r : g.ny + r;
      xx = i % w;
    } else {  // left / right edge cells of the interior rows
      const int64_t j = i - 2 * g.h * w;
      row = g.h + j / (2 * g.h);
      const int64_t e = j % (2 * g.h);
      xx = e < g.h ? e : g.nx + e;
    }
    const int64_t o = base + row * g.pitch + xx;
    dst[o] = src[o];
  }
}

// Dense <-> padded repack of whole planes [p0, p0+np) (array plane indices):
// dense rows hold nx+2h elements, padded rows start at column ox-h.
template <typename T>
__global__ void k_repack(T* padded, T* dense, Geom g, int64_t p0, int64_t np, int to_padded) {
  const int64_t w = g.nx + 2 * g.h;
  const int64_t n = w * g.rows * np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t xx = i % w;
    const int64_t rp = i / w;  // row within the chunk, plane-major
    const int64_t o = (p0 * g.rows + rp) * g.pitch + (g.ox - g.h + xx);
    if (to_padded) padded[o] = dense[i];
    else dense[i] = padded[o];
  }
}

template <typename T> __device__ __forceinline__ uint64_t bits_of(T v);
template <> __device__ __forceinline__ uint64_t bits_of<double>(double v) {
  return (uint64_t)__double_as_longlong(v);
}
template <> __device__ __forceinline__ uint64_t bits_of<float>(float v) {
  return (uint64_t)(uint32_t)__float_as_uint(v);
}

template <typename T>
__global__ void k_digest(const T* base, Geom g, int64_t z_begin, unsigned long long* out) {
  const int64_t n = g.nx * g.ny * g.nzl;
  uint64_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % g.nx;
    const int64_t yz = i / g.nx;
    const int64_t y = yz % g.ny;
    const int64_t z = yz / g.ny;
    const T v = base[((z + g.h) * g.rows + (y + g.h)) * g.pitch + g.ox + x];
    const uint64_t gidx = (uint64_t)(((z + z_begin) * g.ny + y) * g.nx + x);
    acc += splitmix64(bits_of<T>(v) ^ splitmix64(gidx));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);  // mod 2^64: order-free
}

// Point-wise reduce: VALUE(0) SQ(1) ABSDIFF(2) CONV(3).  Rows (y,z) of the box
// are dealt to warps in a fixed pattern; lanes stride x.
struct PointArgs {
  const void* a;
  const void* b;
  int64_t asy, asz, bsy, bsz;
  int x0, x1, y0, y1, z0, z1;
  double eps;
  double* partials;
  unsigned* counter;
  double* result;
  int comb;
};

template <int ROP, typename T> __global__ void __launch_bounds__(256) k_reduce_points(const __grid_constant__ PointArgs p) {
  __shared__ double red[8];
  __shared__ int flag;
  const T* A = static_cast<const T*>(p.a);
  const T* B = static_cast<const T*>(p.b);
  const T eps = (T)p.eps;
  double acc = comb_identity(p.comb);
  const int lane = threadIdx.x & 31;
  const int64_t ny = p.y1 - p.y0;
  const int64_t rows = ny * (p.z1 - p.z0);
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t r = gw; r < rows; r += nwarps) {
    const int64_t y = p.y0 + r % ny, z = p.z0 + r / ny;
    const T* ar = A + z * p.asz + y * p.asy;
    const T* br = (ROP >= 2) ? B + z * p.bsz + y * p.bsy : nullptr;
    for (int x = p.x0 + lane; x < p.x1; x += 32) {
      T v;
      if constexpr (ROP == 0) {
        v = __ldg(ar + x);
      } else if constexpr (ROP == 1) {
        T t = __ldg(ar + x);
        v = mul(t, t);
      } else if constexpr (ROP == 2) {
        v = fabs(sub(__ldg(ar + x), __ldg(br + x)));
      } else {
        v = fabs(sub(__ldg(ar + x), __ldg(br + x))) <= eps ? T(1) : T(0);
      }
      acc = comb_apply(p.comb, acc, (double)v);
    }
  }
  cta_reduce_finish(acc, p.comb, red, &flag, 256, p.partials, p.counter, p.result, gridDim.x, blockIdx.x);
}

__global__ void k_conv_update(const double* res, int* conv, int* iters, int it) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && *conv == 0) {
    *iters = it;
    if (*res != 0.0) *conv = 1;
  }
}

// One iteration's bookkeeping inside the conditional-WHILE graph of
// gscl_converge_run: flags[0] converged, [1] iterations executed, [2] halt
// (converged or max_iters reached: later sweeps return at once).  The last
// update of the loop body sets the WHILE condition from the halt flag.
__global__ void k_conv_step(const double* res, int* flags, int max_iters, cudaGraphConditionalHandle cond,
                            int set_cond) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (flags[2] == 0) {
      flags[1] += 1;
      if (*res != 0.0) flags[0] = 1;
      flags[2] = (flags[0] != 0 || flags[1] >= max_iters) ? 1 : 0;
    }
    if (set_cond) cudaGraphSetConditional(cond, flags[2] ? 0u : 1u);
  }
}

// Bookkeeping of a two-sweep pass of the convergence loop (iterations k+1,
// k+2 computed by one pass; res1 / res2 their AND-reduced tests): flags[0]
// converged, [1] iterations, [2] halt, [3] skip the redo sweep (0: the pass's
// output must be replaced by iteration k+1 alone — it converged, or only one
// iteration of the budget was left), [4] the half of the graph body whose
// output buffer holds the final iterate.
__global__ void k_conv_pair(const double* res1, const double* res2, int* flags, int max_iters, int half,
                            cudaGraphConditionalHandle cond, int set_cond) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (flags[2] == 0) {
      if (*res1 != 0.0 || max_iters - flags[1] == 1) {
        flags[1] += 1;
        flags[0] = *res1 != 0.0 ? 1 : 0;
        flags[3] = 0;
      } else {
        flags[1] += 2;
        flags[0] = *res2 != 0.0 ? 1 : 0;
        flags[3] = 1;
      }
      flags[2] = (flags[0] != 0 || flags[1] >= max_iters) ? 1 : 0;
      if (flags[2]) flags[4] = half;
    } else {
      flags[3] = 1;
    }
    if (set_cond) cudaGraphSetConditional(cond, flags[2] ? 0u : 1u);
  }
}

__global__ void k_fold(const double* vals, int n, int comb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (comb == kFoldU64Sum) {  // the digest across ranks: 64-bit words summed mod 2^64
      unsigned long long t = 0;
      for (int i = 0; i < n; ++i) t += reinterpret_cast<const unsigned long long*>(vals)[i];
      *reinterpret_cast<unsigned long long*>(out) = t;
      return;
    }
    double t = comb_identity(comb);
    for (int i = 0; i < n; ++i) t = comb_apply(comb, t, vals[i]);
    *out = t;
  }
}

int grid_for(int64_t n, int threads, int num_sms = 148) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms * 16));
}

}  // namespace

cudaError_t launch_fill_random(const View& v, int64_t z_begin, uint64_t seed, uint32_t grid_id,
                               double scale, cudaStream_t s, int64_t* launches) {
  Geom g = geom_of(v);
  const int64_t n = g.pitch * g.rows * g.planes;
  const uint64_t key = seed ^ ((uint64_t)grid_id << 48);
  if (v.dtype == 0)
    k_fill_random<double><<<grid_for(n, 256), 256, 0, s>>>((double*)v.base, g, z_begin, key, scale);
  else
    k_fill_random<float><<<grid_for(n, 256), 256, 0, s>>>((float*)v.base, g, z_begin, key, (float)scale);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_const(const View& v, double value, cudaStream_t s, int64_t* launches) {
  const int64_t n = v.pitch * (v.ny + 2 * v.h) * (v.nzl + 2 * v.h);
  if (v.dtype == 0)
    k_fill_const<double><<<grid_for(n, 256), 256, 0, s>>>((double*)v.base, n, value);
  else
    k_fill_const<float><<<grid_for(n, 256), 256, 0, s>>>((float*)v.base, n, (float)value);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_copy_halo(const View& src, const View& dst, cudaStream_t s, int64_t* launches) {
  Geom g = geom_of(src);
  if (g.h == 0) return cudaSuccess;
  const int64_t per_plane = g.rows * (g.nx + 2 * g.h);  // upper bound of a plane's halo cells
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((per_plane + 255) / 256, 8)),
            (unsigned)g.planes);
  if (src.dtype == 0)
    k_copy_halo<double><<<grid, 256, 0, s>>>((const double*)src.base, (double*)dst.base, g);
  else
    k_copy_halo<float><<<grid, 256, 0, s>>>((const float*)src.base, (float*)dst.base, g);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_repack(const View& v, void* dense, int64_t p0, int64_t np, bool to_padded,
                          cudaStream_t s, int64_t* launches) {
  Geom g = geom_of(v);
  const int64_t n = (g.nx + 2 * g.h) * g.rows * np;
  if (n == 0) return cudaSuccess;
  if (v.dtype == 0)
    k_repack<double><<<grid_for(n, 256), 256, 0, s>>>((double*)v.base, (double*)dense, g, p0, np, to_padded);
  else
    k_repack<float><<<grid_for(n, 256), 256, 0, s>>>((float*)v.base, (float*)dense, g, p0, np, to_padded);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_digest(const View& v, int64_t z_begin, uint64_t* d_out, cudaStream_t s,
                          int64_t* launches) {
  Geom g = geom_of(v);
  const int64_t n = g.nx * g.ny * g.nzl;
  if (n == 0) return cudaSuccess;
  auto* o = reinterpret_cast<unsigned long long*>(d_out);
  if (v.dtype == 0)
    k_digest<double><<<grid_for(n, 256), 256, 0, s>>>((const double*)v.base, g, z_begin, o);
  else
    k_digest<float><<<grid_for(n, 256), 256, 0, s>>>((const float*)v.base, g, z_begin, o);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_reduce_points(int rop, const View* gv, int n, const Box& box, double eps,
                                 const RedTarget& red, int num_sms, cudaStream_t s,
                                 int64_t* launches) {
  PointArgs p{};
  p.a = gv[0].origin;
  p.asy = gv[0].pitch;
  p.asz = gv[0].plane;
  if (n > 1) {
    p.b = gv[1].origin;
    p.bsy = gv[1].pitch;
    p.bsz = gv[1].plane;
  }
  p.x0 = (int)box.x0; p.x1 = (int)box.x1; p.y0 = (int)box.y0; p.y1 = (int)box.y1;
  p.z0 = (int)box.z0; p.z1 = (int)box.z1;
  p.eps = eps;
  p.partials = red.partials;
  p.counter = red.counter;
  p.result = red.result;
  p.comb = red.comb;
  const int64_t rows = (box.y1 - box.y0) * (box.z1 - box.z0);
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, (int64_t)num_sms * 8));
  blocks = std::min(blocks, red.max_partials);
  const bool f64 = gv[0].dtype == 0;
#define GSCL_RP(R)                                                                       \
  if (f64) k_reduce_points<R, double><<<blocks, 256, 0, s>>>(p);                         \
  else k_reduce_points<R, float><<<blocks, 256, 0, s>>>(p);
  switch (rop) {
    case 0: GSCL_RP(0); break;
    case 1: GSCL_RP(1); break;
    case 2: GSCL_RP(2); break;
    case 3: GSCL_RP(3); break;
    default: return cudaErrorInvalidValue;
  }
#undef GSCL_RP
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_conv_update(const double* res, int* conv, int* iters, int it, cudaStream_t s,
                               int64_t* launches) {
  k_conv_update<<<1, 32, 0, s>>>(res, conv, iters, it);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_conv_step(const double* res, int* flags, int max_iters, unsigned long long cond,
                             int set_cond, cudaStream_t s, int64_t* launches) {
  k_conv_step<<<1, 32, 0, s>>>(res, flags, max_iters, (cudaGraphConditionalHandle)cond, set_cond);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_conv_pair(const double* res1, const double* res2, int* flags, int max_iters, int half,
                             unsigned long long cond, int set_cond, cudaStream_t s, int64_t* launches) {
  k_conv_pair<<<1, 32, 0, s>>>(res1, res2, flags, max_iters, half, (cudaGraphConditionalHandle)cond, set_cond);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fold(const double* d_vals, int n, int comb, double* d_out, cudaStream_t s,
                        int64_t* launches) {
  k_fold<<<1, 32, 0, s>>>(d_vals, n, comb, d_out);
  ++*launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ peer-memory signalling
namespace {
__global__ void k_signal(PeerPtrs8 f, unsigned add) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    __threadfence_system();  // the caller's preceding copies / stores into the peers' memory
    for (int i = 0; i < f.n; ++i)
      if (f.p[i]) atomicAdd_system(static_cast<unsigned*>(f.p[i]), add);
  }
}
__global__ void k_publish(const double* val, PeerPtrs8 dst, PeerPtrs8 cnt) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double v = *val;
    for (int i = 0; i < dst.n; ++i) static_cast<double*>(dst.p[i])[0] = v;
    __threadfence_system();
    for (int i = 0; i < cnt.n; ++i) atomicAdd_system(static_cast<unsigned*>(cnt.p[i]), 1u);
  }
}
}  // namespace

cudaError_t launch_signal(const PeerPtrs8& flags, unsigned add, cudaStream_t s, int64_t* launches) {
  k_signal<<<1, 32, 0, s>>>(flags, add);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_publish(const double* val, const PeerPtrs8& dst, const PeerPtrs8& cnt, cudaStream_t s,
                           int64_t* launches) {
  k_publish<<<1, 32, 0, s>>>(val, dst, cnt);
  ++*launches;
  return cudaGetLastError();
}

namespace {
PFN_cuMemGetAddressRange_v3020 g_range = nullptr;
std::once_flag g_range_once;
}  // namespace

cudaError_t alloc_base(const void* ptr, void** base, size_t* size) {
  std::call_once(g_range_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  });
  if (!g_range) return cudaErrorNotSupported;
  CUdeviceptr b = 0;
  size_t n = 0;
  CUresult r = g_range(&b, &n, reinterpret_cast<CUdeviceptr>(ptr));
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  *base = reinterpret_cast<void*>(b);
  if (size) *size = n;
  return cudaSuccess;
}

// ------------------------------------------------------------------ stream memory ops
namespace {
PFN_cuStreamWaitValue32_v11070 g_wait32 = nullptr;
std::once_flag g_wait32_once;
}  // namespace

cudaError_t preload_modules(int* n) {
  using PGetModule = CUresult (*)(CUmodule*, CUfunction);
  using PCount = CUresult (*)(unsigned*, CUmodule);
  using PEnum = CUresult (*)(CUfunction*, unsigned, CUmodule);
  using PLoad = CUresult (*)(CUfunction);
  auto entry = [](const char* sym) -> void* {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(sym, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      return nullptr;
    return fn;
  };
  auto get_module = reinterpret_cast<PGetModule>(entry("cuFuncGetModule"));
  auto count = reinterpret_cast<PCount>(entry("cuModuleGetFunctionCount"));
  auto enumerate = reinterpret_cast<PEnum>(entry("cuModuleEnumerateFunctions"));
  auto load = reinterpret_cast<PLoad>(entry("cuFuncLoad"));
  if (!get_module || !count || !enumerate || !load) return cudaErrorNotSupported;
  const void* (*anchors[])() = {anchor_util, anchor_sweep, anchor_sweep2r, anchor_sweep2v, anchor_ordered,
                                anchor_sweep2x};
  int total = 0;
  for (auto a : anchors) {
    cudaFunction_t f = nullptr;
    cudaError_t e = cudaGetFuncBySymbol(&f, a());
    if (e != cudaSuccess) return e;
    CUmodule m = nullptr;
    if (get_module(&m, reinterpret_cast<CUfunction>(f)) != CUDA_SUCCESS) return cudaErrorUnknown;
    unsigned c = 0;
    if (count(&c, m) != CUDA_SUCCESS) return cudaErrorUnknown;
    std::vector<CUfunction> fs(c);
    if (c && enumerate(fs.data(), c, m) != CUDA_SUCCESS) return cudaErrorUnknown;
    for (CUfunction g : fs)
      if (load(g) != CUDA_SUCCESS) return cudaErrorUnknown;
    total += (int)c;
  }
  if (n) *n = total;
  return cudaSuccess;
}

cudaError_t stream_wait_geq(cudaStream_t s, unsigned* flag, unsigned value) {
  std::call_once(g_wait32_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fn);
  });
  if (!g_wait32) return cudaErrorNotSupported;
  CUresult r = g_wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

// ------------------------------------------------------------------ TMA maps
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
}  // namespace

bool encode_tma_3d(CUtensorMap* map, const View& v, uint32_t box_x, uint32_t box_y, int l2promo) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return false;
  const size_t es = v.dtype == 0 ? 8 : 4;
  cuuint64_t dims[3] = {(cuuint64_t)v.pitch, (cuuint64_t)(v.ny + 2 * v.h), (cuuint64_t)(v.nzl + 2 * v.h)};
  cuuint64_t strides[2] = {(cuuint64_t)(v.pitch * es), (cuuint64_t)(v.plane * es)};
  cuuint32_t box[3] = {box_x, box_y, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, v.dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, v.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE,
                        l2promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                        : l2promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                        : l2promo == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                       : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace gscl
