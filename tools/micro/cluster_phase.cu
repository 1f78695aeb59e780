// Microbenchmark: cost of one "phase" of a persistent multigrid tail.
// Every row sums K products a_m * x[c_m] with the row's columns/values in
// shared memory (SELL-like column-major layout: conflict-free) and x in
// shared memory (random gathers); the new value is stored to x in EVERY CTA
// of the cluster (replicated vector, DSMEM remote stores) or locally
// (CS = 1), then a cluster barrier / __syncthreads.  rows = 0 measures the
// bare barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cphase tools/micro/cluster_phase.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr int NX = 2048;   // x entries (replicated)
constexpr int K = 14;      // entries per row (coarse AMG levels: 12-18)
constexpr int RMAX = 128;  // distinct row records in smem (rows wrap)

template <int CS, int NT>
__global__ void __launch_bounds__(NT, 1) k_phase(int phases, int rows, double* sink) {
  __shared__ double x[NX];
  __shared__ int cols[K * RMAX];
  __shared__ double vals[K * RMAX];
  const int tid = threadIdx.x;
  for (int i = tid; i < NX; i += NT) x[i] = 1.0 + 1e-3 * i;
  for (int i = tid; i < K * RMAX; i += NT) {
    cols[i] = (int)((i * 2654435761u) % NX);
    vals[i] = 1e-3 * (i % 7);
  }
  unsigned rank = 0;
  if constexpr (CS > 1) {
    cg::cluster_group cl = cg::this_cluster();
    rank = cl.block_rank();
    cl.sync();
  } else {
    __syncthreads();
  }
  const int per = (rows + CS - 1) / CS;
  double acc = 0.0;
  for (int p = 0; p < phases; ++p) {
    for (int t = tid; t < per; t += NT) {
      const int row = (rank * per + t + p * 37) % NX;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) s = s + vals[k * RMAX + (t & (RMAX - 1))] * x[cols[k * RMAX + (t & (RMAX - 1))]];
      s = 1.0 + 1e-3 * s;
      if constexpr (CS > 1) {
        cg::cluster_group cl = cg::this_cluster();
#pragma unroll
        for (int r = 0; r < CS; ++r) cl.map_shared_rank(x, r)[row] = s;
      } else {
        x[row] = s;
      }
      acc += s;
    }
    if constexpr (CS > 1) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      __syncthreads();
    }
  }
  if (acc == -1.0) sink[0] = acc;
}

template <int CS, int NT>
void run(int rows, double* sink) {
  auto kern = k_phase<CS, NT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(NT);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ph = 4000;
  cudaLaunchKernelEx(&cfg, kern, ph, rows, sink);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kern, ph, rows, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  printf("cluster %2d threads %4d rows %5d : %.3f us/phase %s\n", CS, NT, rows, ms * 1e3 / ph,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  double* sink;
  cudaMalloc(&sink, 8);
  for (int rows : {0, 32, 128, 512, 2048}) {
    if (rows <= 512) {
      run<1, 128>(rows, sink);
      run<1, 512>(rows, sink);
    }
    if (rows <= 1024) run<2, 512>(rows, sink);
    run<4, 512>(rows, sink);
    run<8, 256>(rows, sink);
    run<16, 128>(rows, sink);
  }
  return 0;
}
