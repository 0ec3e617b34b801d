// Does programmatic dependent launch overlap consecutive grids on this box?
// A chain of K grids of 1026 one-CTA-per-SM blocks (big dynamic smem), each
// CTA busy-waits a pseudo-random 40-70 us; with PDL each CTA executes
// griddepcontrol.launch_dependents first.  Prints the chain time with and
// without the launch attribute, and the overlap seen by %globaltimer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void work(int k, uint64_t* first_start, uint64_t* last_end, int pdl) {
  extern __shared__ char sm[];
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t t0 = gtime();
  if (threadIdx.x == 0) atomicMin((unsigned long long*)&first_start[k], (unsigned long long)t0);
  uint32_t h = blockIdx.x * 2654435761u + k * 40503u;
  h ^= h >> 13;
  const uint64_t dur = 40000 + (h % 30000);  // ns
  while (gtime() - t0 < dur) {
  }
  sm[threadIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax((unsigned long long*)&last_end[k], (unsigned long long)gtime());
}

int main() {
  const int K = 20, G = 1026, T = 256;
  const size_t smem = 150 * 1024;
  cudaFuncSetAttribute(work, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  uint64_t *fs, *le;
  cudaMalloc(&fs, K * 8);
  cudaMalloc(&le, K * 8);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep)
    for (int pdl = 0; pdl <= 1; ++pdl) {
      cudaMemset(fs, 0xff, K * 8);
      cudaMemset(le, 0, K * 8);
      cudaDeviceSynchronize();
      cudaEventRecord(e0, st);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(T);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = (pdl && k > 0) ? 1 : 0;
        cudaLaunchKernelEx(&cfg, work, k, fs, le, pdl);
      }
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      uint64_t hfs[K], hle[K];
      cudaMemcpy(hfs, fs, sizeof hfs, cudaMemcpyDeviceToHost);
      cudaMemcpy(hle, le, sizeof hle, cudaMemcpyDeviceToHost);
      double ov = 0;
      for (int k = 1; k < K; ++k) ov += (double)((int64_t)hle[k - 1] - (int64_t)hfs[k]) / 1e3;
      printf("{\"pdl\": %d, \"chain_ms\": %.3f, \"per_grid_ms\": %.4f, \"mean_overlap_us\": %.2f, \"err\": \"%s\"}\n", pdl,
             ms, ms / K, ov / (K - 1), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
