// Device steps of the slab-partitioned solve: each
// rank owns a contiguous range of block rows (whole z-slabs of the grid for
// the generated problems) and its vectors hold only those rows; the
// operators read a contiguous column window [w0, w1) whose halo parts are
// exchanged between ranks by the host layer (partition.py).
//
// Reductions are GPU-count invariant: a dot product is the fixed-order sum
// of per-SEGMENT partials, a segment being a fixed global range of rows
// (rank boundaries are segment boundaries), each partial reduced by one CTA
// in a fixed thread/shuffle order.  The same partials in the same order are
// summed on every rank, so H, norms and every host decision are bitwise
// identical for 1, 2, 4 or 8 ranks.
#include <cmath>

#include "device.cuh"
#include "engine.h"

namespace cprb {

constexpr int SEG_THREADS = 256;

__device__ __forceinline__ double seg_block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(CPRB_FULL, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s = s + sh[k];
  return s;  // valid in thread 0
}

// one CTA per segment: optionally w -= (*hprev) * vprev (MGS), then the
// segment's partial of (w, vdot) ((w, w) when vdot == nullptr)
__global__ void __launch_bounds__(SEG_THREADS)
    k_seg_partials(int64_t n, int64_t seg_len, double* w, const double* __restrict__ vprev,
                   const double* __restrict__ hprev, const double* __restrict__ vdot,
                   double* __restrict__ partials) {
  __shared__ double sh[SEG_THREADS / 32];
  const int64_t lo = (int64_t)blockIdx.x * seg_len;
  const int64_t hi = lo + seg_len < n ? lo + seg_len : n;
  const double h = vprev ? *hprev : 0.0;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += SEG_THREADS) {
    double wi = w[i];
    if (vprev) {
      wi = wi - h * vprev[i];
      w[i] = wi;
    }
    const double d = vdot ? vdot[i] : wi;
    acc = acc + wi * d;
  }
  const double s = seg_block_sum(acc, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// fixed-order sum of all segment partials (global segment order via map)
__global__ void __launch_bounds__(SEG_THREADS)
    k_seg_finish(int nseg, const double* __restrict__ partials, const int32_t* __restrict__ map,
                 double* out, int sq) {
  __shared__ double sh[SEG_THREADS / 32];
  double acc = 0.0;
  for (int s = threadIdx.x; s < nseg; s += SEG_THREADS) acc = acc + partials[map ? map[s] : s];
  const double t = seg_block_sum(acc, sh);
  if (threadIdx.x == 0) *out = sq ? sqrt(t) : t;
}

__global__ void k_div_nz(int64_t n, double* w, const double* __restrict__ h) {
  const double hv = *h;
  if (hv == 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = w[i] / hv;
}

__global__ void k_scatter_add(int64_t n, const int32_t* __restrict__ idx,
                              const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = dst[idx[i]] + src[i];
}

__global__ void k_gather_s(int64_t n, const int32_t* __restrict__ idx,
                           const double* __restrict__ src, int stride,
                           double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[(int64_t)stride * (idx ? idx[i] : i)];
}

// padded all-gather layout [rank][cap] -> packed rank-ordered vector
__global__ void k_unpad(int nranks, int64_t cap, const int64_t* __restrict__ offs,
                        const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nranks * cap) return;
  const int q = (int)(i / cap);
  const int64_t e = i - (int64_t)q * cap;
  const int64_t o = offs[q];
  if (e < offs[q + 1] - o) dst[o + e] = src[i];
}

// z = Pi zp + y  (src/cpr.py:184-186: z1 = zeros + scatter(zp); z1 + y)
__global__ void k_cpr_combine(int64_t ncells, int b, const double* __restrict__ zp,
                              const double* __restrict__ y, double* __restrict__ z) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ncells * b) return;
  const int64_t c = e / b;
  const double z1 = (e - c * b) == 0 ? zp[c] : 0.0;
  z[e] = z1 + y[e];
}

static inline int eblk(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : g);
}

static inline int eblk_cap(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace cprb

using namespace cprb;

extern "C" {

int cprb_seg_partials(int64_t n, int64_t seg_len, double* w, const double* vprev,
                      const double* hprev, const double* vdot, double* partials, void* stream) {
  if (n <= 0) return CPRB_OK;
  if (seg_len <= 0) return set_error(CPRB_EINVAL, "segment length must be positive");
  const int64_t nseg = (n + seg_len - 1) / seg_len;
  k_seg_partials<<<(unsigned)nseg, SEG_THREADS, 0, (cudaStream_t)stream>>>(n, seg_len, w, vprev,
                                                                          hprev, vdot, partials);
  return check_launch("segment partials");
}

int cprb_seg_finish(int32_t nseg, const double* partials, const int32_t* map, double* out,
                    int32_t sqrt_, void* stream) {
  k_seg_finish<<<1, SEG_THREADS, 0, (cudaStream_t)stream>>>(nseg, partials, map, out, sqrt_);
  return check_launch("segment finish");
}

int cprb_div_if_nonzero(int64_t n, double* w, const double* h, void* stream) {
  if (n <= 0) return CPRB_OK;
  k_div_nz<<<eblk_cap(n), 256, 0, (cudaStream_t)stream>>>(n, w, h);
  return check_launch("div if nonzero");
}

int cprb_scatter_add(int64_t n, const int32_t* idx, const double* src, double* dst,
                     void* stream) {
  if (n <= 0) return CPRB_OK;
  k_scatter_add<<<eblk(n), 256, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  return check_launch("scatter add");
}

int cprb_gather(int64_t n, const int32_t* idx, const double* src, int32_t stride, double* dst,
                void* stream) {
  if (n <= 0) return CPRB_OK;
  k_gather_s<<<eblk(n), 256, 0, (cudaStream_t)stream>>>(n, idx, src, stride, dst);
  return check_launch("gather");
}

int cprb_unpad(int32_t nranks, int64_t cap, const int64_t* offs, const double* src, double* dst,
               void* stream) {
  const int64_t n = (int64_t)nranks * cap;
  if (n <= 0) return CPRB_OK;
  k_unpad<<<eblk(n), 256, 0, (cudaStream_t)stream>>>(nranks, cap, offs, src, dst);
  return check_launch("unpad");
}

int cprb_cpr_combine(int64_t ncells, int32_t b, const double* zp, const double* y, double* z,
                     void* stream) {
  if (ncells <= 0) return CPRB_OK;
  k_cpr_combine<<<eblk(ncells * b), 256, 0, (cudaStream_t)stream>>>(ncells, b, zp, y, z);
  return check_launch("cpr combine");
}

}  // extern "C"
