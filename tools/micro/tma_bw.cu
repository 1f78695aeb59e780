// Microbenchmark: per-SM streaming rate of cp.async.bulk (global -> shared)
// with a DEPTH-slot ring, vs. plain coalesced LDG.  Used to size the BILU
// wave pipeline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int DEPTH>
__global__ void k_tma(const uint8_t* src, size_t per_cta, int piece, int npieces_per_slot, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[DEPTH];
  const int slot_bytes = piece * npieces_per_slot;
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const int nsteps = (int)(per_cta / slot_bytes);
  if (threadIdx.x == 0) {
    for (int d = 0; d < DEPTH; ++d) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[d])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long acc = 0;
  if (threadIdx.x == 0) {
    auto issue = [&](int k) {
      const int st = k % DEPTH;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(slot_bytes) : "memory");
      for (int p = 0; p < npieces_per_slot; ++p)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(sm + (size_t)st * slot_bytes + p * piece)), "l"(base + (size_t)k * slot_bytes + p * piece),
                     "r"(piece), "r"(su32(&full[st])) : "memory");
    };
    for (int k = 0; k < DEPTH && k < nsteps; ++k) issue(k);
    for (int k = 0; k < nsteps; ++k) {
      const int st = k % DEPTH;
      const uint32_t par = (k / DEPTH) & 1;
      asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(su32(&full[st])), "r"(par) : "memory");
      acc += sm[(size_t)st * slot_bytes + 64];
      if (k + DEPTH < nsteps) issue(k + DEPTH);
    }
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

__global__ void k_ldg(const double* src, size_t per_cta_d, unsigned long long* sink) {
  const double* base = src + (size_t)blockIdx.x * per_cta_d;
  double acc = 0;
  for (size_t i = threadIdx.x; i < per_cta_d; i += blockDim.x) acc += __ldg(base + i);
  if (acc == 1.2345) sink[0] = 1;
}

int main() {
  const size_t per_cta = 8u << 20;  // 8 MB per CTA (~ one BILU chunk)
  const int nctas[] = {1, 43, 85, 148};
  uint8_t* src;
  unsigned long long* sink;
  cudaMalloc(&src, per_cta * 148);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 1, per_cta * 148);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int piece, npieces; };
  Cfg cfgs[] = {{30720, 1}, {4096, 8}, {2048, 15}, {16384, 1}, {1024, 30}};
  for (int nc : nctas) {
    for (auto c : cfgs) {
      const int slot = c.piece * c.npieces;
      const size_t smem = 4 * (size_t)slot;
      cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_tma<4><<<nc, 32, smem>>>(src, per_cta, c.piece, c.npieces, sink);
      cudaEventRecord(e0);
      k_tma<4><<<nc, 32, smem>>>(src, per_cta, c.piece, c.npieces, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("TMA depth4 ctas=%3d slot=%6d (%d x %5d): %7.1f GB/s per SM, %8.1f GB/s total  err=%s\n", nc, slot, c.npieces,
             c.piece, per_cta / (ms * 1e-3) / 1e9, nc * per_cta / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    {
      const int slot = 15360;
      cudaFuncSetAttribute(k_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * slot);
      k_tma<8><<<nc, 32, 8 * slot>>>(src, per_cta, slot, 1, sink);
      cudaEventRecord(e0);
      k_tma<8><<<nc, 32, 8 * slot>>>(src, per_cta, slot, 1, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("TMA depth8 ctas=%3d slot=%6d: %7.1f GB/s per SM\n", nc, slot, per_cta / (ms * 1e-3) / 1e9);
    }
    for (int thr : {64, 128, 256, 1024}) {
      k_ldg<<<nc, thr>>>((const double*)src, per_cta / 8, sink);
      cudaEventRecord(e0);
      k_ldg<<<nc, thr>>>((const double*)src, per_cta / 8, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("LDG ctas=%3d threads=%4d: %7.1f GB/s per SM\n", nc, thr, per_cta / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
