// Microbenchmark: cost of a block barrier vs a 2-CTA cluster barrier (16 warps/CTA).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(512, 1) k_block(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k_cluster(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) k_cluster_relaxed(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 1024 * sizeof(long long));
  long long h[1024];
  const int iters = 10000;
  auto rep = [&](const char* name, void (*k)(int, long long*)) {
    k<<<148, 512, 180 * 1024>>>(iters, d);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
    k<<<148, 512, 180 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    printf("%s: %s %.1f cycles/barrier\n", name, cudaGetErrorString(e), (double)h[0] / iters);
  };
  rep("block", k_block);
  rep("cluster2 acq/rel", k_cluster);
  rep("cluster2 relaxed", k_cluster_relaxed);
  return 0;
}
