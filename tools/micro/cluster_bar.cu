// Microbenchmark: cost of barrier.cluster (16-CTA and 8-CTA clusters, 512
// threads) and of __syncthreads, per barrier.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_cbar(int iters, double* sink) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (acc == -1.0) sink[0] = acc;
}
__global__ void k_cbar_relaxed(int iters, double* sink) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  }
  if (acc == -1.0) sink[0] = acc;
}
__global__ void k_sync(int iters, double* sink) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    __syncthreads();
  }
  if (acc == -1.0) sink[0] = acc;
}

template <typename K>
float run(K kern, int csize, int iters, double* sink) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, kern, iters, sink);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kern, iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("  err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return ms * 1e3f / iters;
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  for (int cs : {16, 8, 4, 2, 1}) {
    printf("cluster %2d: barrier.cluster release/acquire %.3f us, relaxed %.3f us\n", cs,
           run(k_cbar, cs, 20000, sink), run(k_cbar_relaxed, cs, 20000, sink));
  }
  printf("__syncthreads (1 CTA, 512 thr): %.3f us\n", run(k_sync, 1, 20000, sink));
  return 0;
}
