// Does a cluster-launched, ~224 KB-smem kernel (the FFN1 GEMM's footprint) start while a
// small PDL primary kernel (the ordered push's footprint) is still resident?  Prints when the
// secondary's CTAs start relative to the primary's start / end (diagnostics).
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_t[4096][2];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256, 4) primary(int us, int trigger) {
  if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) g_t[blockIdx.x][0] = t0;
  while (gt() - t0 < (unsigned long long)us * 1000ull) {
  }
  if (threadIdx.x == 0) g_t[blockIdx.x][1] = gt();
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1) secondary() {
  extern __shared__ char smem[];
  if (threadIdx.x == 0) {
    smem[0] = 1;
    g_t[2048 + blockIdx.x][0] = gt();
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

int main() {
  const int smem = 228624;
  cudaFuncSetAttribute(secondary, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int carve : {-1, 100}) {
    for (int pdl : {0, 1}) {
      if (carve >= 0) cudaFuncSetAttribute(primary, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
      primary<<<nsm, 256>>>(50, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nsm & ~1);
      cfg.blockDim = dim3(320);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl;
      cudaError_t e = cudaLaunchKernelEx(&cfg, secondary);
      cudaError_t e2 = cudaDeviceSynchronize();
      static unsigned long long h[4096][2];
      cudaMemcpyFromSymbol(h, g_t, sizeof(h));
      unsigned long long p0 = ~0ull, p1 = 0, s0 = ~0ull, s1 = 0;
      for (int i = 0; i < nsm; ++i) {
        p0 = h[i][0] < p0 ? h[i][0] : p0;
        p1 = h[i][1] > p1 ? h[i][1] : p1;
      }
      for (int i = 0; i < (nsm & ~1); ++i) {
        s0 = h[2048 + i][0] < s0 ? h[2048 + i][0] : s0;
        s1 = h[2048 + i][0] > s1 ? h[2048 + i][0] : s1;
      }
      printf("carveout %d pdl %d (%s/%s): primary %.1f us; secondary CTAs start %.1f .. %.1f us after primary start\n",
             carve, pdl, cudaGetErrorString(e), cudaGetErrorString(e2), (p1 - p0) / 1e3, ((long long)(s0 - p0)) / 1e3,
             ((long long)(s1 - p0)) / 1e3);
    }
  }
  return 0;
}
