// K9/K10 + CPR orchestration: deterministic reductions, the fused Arnoldi
// modified Gram-Schmidt step (src/cpr.py:276-284), the GMRES update and the
// CPR application (src/cpr.py:178-186).
#include <cmath>
#include <mutex>
#include <string>

#include "device.cuh"
#include "engine.h"
#include "nvtx.h"

namespace cprb {

static thread_local std::string g_err;

int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(CPRB_EDEVICE, std::string(what) + ": " + cudaGetErrorString(e));
  return CPRB_OK;
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

constexpr int RED_THREADS = 256;

// fixed-order block reduction (shuffle xor tree, then warps in order)
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(CPRB_FULL, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s = s + sh[k];
  return s;  // valid in thread 0
}

// after every block stored its partial, the last block sums them in order
__device__ __forceinline__ bool last_block(int32_t* ticket) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int t = atomicAdd(ticket, 1);
    is_last = (t == (int)gridDim.x - 1);
    if (is_last) *ticket = 0;
  }
  __syncthreads();
  return is_last;
}

__device__ __forceinline__ double sum_partials(const double* partials, int np, double* sh) {
  double v = 0.0;
  for (int k = threadIdx.x; k < np; k += blockDim.x) v = v + ld_relaxed(partials + k);
  return block_sum(v, sh);
}

// one MGS stage: optionally w -= (*hprev) * vprev, then partial (w, vdot);
// finalize: *hout = sum (or sqrt(sum) when SQRT).  vdot == nullptr -> (w, w).
template <int SQRT>
__global__ void __launch_bounds__(RED_THREADS)
    k_mgs_stage(int64_t n, double* w, const double* __restrict__ vprev,
                const double* __restrict__ hprev, const double* __restrict__ vdot,
                double* partials, int32_t* ticket, double* hout) {
  __shared__ double sh[RED_THREADS / 32];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  const double h = vprev ? *hprev : 0.0;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double wi = w[i];
    if (vprev) {
      wi = wi - h * vprev[i];
      w[i] = wi;
    }
    const double d = vdot ? vdot[i] : wi;
    acc = acc + wi * d;
  }
  const double bs = block_sum(acc, sh);
  if (threadIdx.x == 0) st_relaxed(partials + blockIdx.x, bs);
  if (last_block(ticket)) {
    const double s = sum_partials(partials, gridDim.x, sh);
    if (threadIdx.x == 0) *hout = SQRT ? sqrt(s) : s;
  }
}

// V_{j+1} = w / h unless h == 0 (src/cpr.py:281-284)
__global__ void k_div_if_nonzero(int64_t n, double* w, const double* __restrict__ h) {
  const double hv = *h;
  if (hv == 0.0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = w[i] / hv;
}

__global__ void k_div(int64_t n, const double* __restrict__ x, const double* __restrict__ h,
                      double* __restrict__ out) {
  const double hv = *h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] / hv;
}

// u = y @ V[:k]  (sequential in i)
__global__ void k_gemv_t(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                         const double* __restrict__ y, double* __restrict__ u) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < k; ++i) s = s + y[i] * V[i * ldv + e];
    u[e] = s;
  }
}

__global__ void k_add(int64_t n, const double* __restrict__ x, const double* __restrict__ s,
                      double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = x[e] + s[e];
}

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x,
                       const double* __restrict__ y, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = a * x[e] + y[e];
}

__global__ void k_fill(double* p, int64_t n, unsigned long long bits) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    p[e] = __longlong_as_double((long long)bits);
}

static inline int red_blocks(int64_t n) {
  int64_t g = (n + RED_THREADS * 4 - 1) / (RED_THREADS * 4);
  if (g < 1) g = 1;
  if (g > CPRB_RED_BLOCKS) g = CPRB_RED_BLOCKS;
  return (int)g;
}

static inline int ew_blocks(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

int fill_sentinel(double* p, int64_t n, cudaStream_t st) {
  k_fill<<<ew_blocks(n), 256, 0, st>>>(p, n, CPRB_SENTINEL);
  return check_launch("fill sentinel");
}

}  // namespace cprb

using namespace cprb;

extern "C" {

const char* cprb_last_error(void) { return g_err.c_str(); }
int cprb_version(void) { return 1; }

int cprb_dot(int64_t n, const double* x, const double* y, double* out, double* partials,
             int32_t* ticket, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) {
    cudaMemsetAsync(out, 0, sizeof(double), st);
    return check_launch("dot");
  }
  // (x, y): reuse the MGS stage with w = x (read only: vprev == nullptr)
  k_mgs_stage<0><<<red_blocks(n), RED_THREADS, 0, st>>>(n, const_cast<double*>(x), nullptr,
                                                          nullptr, y, partials, ticket, out);
  return check_launch("dot");
}

// *out = sqrt((x, x)) on the device: the same partition, tree and sqrt as
// cprb_dot followed by a host sqrt (src/sparse.py:361-369), no host round trip
int cprb_norm2(int64_t n, const double* x, double* out, double* partials, int32_t* ticket,
               void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) {
    cudaMemsetAsync(out, 0, sizeof(double), st);
    return check_launch("norm2");
  }
  k_mgs_stage<1><<<red_blocks(n), RED_THREADS, 0, st>>>(n, const_cast<double*>(x), nullptr,
                                                          nullptr, nullptr, partials, ticket, out);
  return check_launch("norm2");
}

int cprb_arnoldi_mgs(int64_t n, int32_t j, double* V, int64_t ldv, double* Hcol,
                     double* partials, int32_t* ticket, void* stream) {
  NvtxRange nv("arnoldi_mgs");
  cudaStream_t st = (cudaStream_t)stream;
  double* w = V + (int64_t)(j + 1) * ldv;
  const int g = red_blocks(n);
  for (int i = 0; i <= j + 1; ++i) {
    const double* vprev = i > 0 ? V + (int64_t)(i - 1) * ldv : nullptr;
    const double* hprev = i > 0 ? Hcol + (i - 1) : nullptr;
    if (i <= j)
      k_mgs_stage<0><<<g, RED_THREADS, 0, st>>>(n, w, vprev, hprev, V + (int64_t)i * ldv,
                                                 partials, ticket, Hcol + i);
    else
      k_mgs_stage<1><<<g, RED_THREADS, 0, st>>>(n, w, vprev, hprev, nullptr, partials, ticket,
                                                 Hcol + i);
  }
  k_div_if_nonzero<<<ew_blocks(n), 256, 0, st>>>(n, w, Hcol + j + 1);
  return check_launch("arnoldi mgs");
}

int cprb_gemv_t(int64_t n, int32_t k, const double* V, int64_t ldv, const double* y, double* u,
                void* stream) {
  k_gemv_t<<<ew_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, k, V, ldv, y, u);
  return check_launch("gemv_t");
}

int cprb_add(int64_t n, const double* x, const double* s, double* out, void* stream) {
  k_add<<<ew_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, x, s, out);
  return check_launch("add");
}

int cprb_axpy(int64_t n, double alpha, const double* x, const double* y, double* out,
              void* stream) {
  k_axpy<<<ew_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, alpha, x, y, out);
  return check_launch("axpy");
}

int cprb_div_scalar(int64_t n, const double* x, const double* h_dev, double* out, void* stream) {
  k_div<<<ew_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, x, h_dev, out);
  return check_launch("div");
}

// src/cpr.py:184-186 given zp in P->zp:  r2 = r - A Pi zp;  z = Pi zp + BILU(r2)
int cprb_cpr_finish(const cprb_cpr* P, const double* r, double* z, void* stream) {
  NvtxRange nv("cpr_stage2_bilu");
  cudaStream_t st = (cudaStream_t)stream;
  const cprb_bilu& F = P->bilu;
  if (F.use_wave) {
    // stage-2 residual written straight into the L plan's step order; it
    // also arms the step-ordered outputs the L and U solves poll
    int rc;
    if (F.use_wave == 2) {
      // stencil solves: arm only the planes a round polls (csrc/stencil.cu)
      rc = bsr_op(2, P->A, P->b, P->zp, r, F.rhs_l, nullptr, nullptr, st, F.l_slot);
      if (!rc) rc = stencil_arm(F, st);
    } else {
      rc = bsr_op(2, P->A, P->b, P->zp, r, F.rhs_l, nullptr, F.zl_step, st, F.l_slot, F.y_step,
                  F.l_slot, F.u_slot);
    }
    if (rc) return rc;
    // the solves publish in step order (coalesced); z = Pi zp + y is one
    // gather pass afterwards
    rc = F.use_wave == 2 ? stencil_solve(F, F.rhs_l, st) : wave_solve(F, F.rhs_l, st);
    if (rc) return rc;
    return wave_combine(F, P->zp, z, st);
  }
  int rc = bsr_op(2, P->A, P->b, P->zp, r, P->r2, nullptr, P->zl, st);  // also arms zl
  if (rc) return rc;
  return bilu_solve(P->bilu, P->r2, P->zl, P->y, P->zp, z, st);
}

// src/cpr.py:178-186:  zp = AMG(Pi^T r);  r2 = r - A Pi zp;  z = Pi zp + BILU(r2)
int cprb_cpr_apply(const cprb_cpr* P, const double* r, double* z, void* stream) {
  NvtxRange nv("cpr_apply");
  int rc = P->amg.cycle != 0 ? kcycle_apply(P->amg, r, P->zp, (cudaStream_t)stream)
                             : amg_vcycle(P->amg, r, P->zp, (cudaStream_t)stream);
  if (rc) return rc;
  return cprb_cpr_finish(P, r, z, stream);
}

__global__ void k_div_host(int64_t n, const double* __restrict__ x, double h,
                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] / h;
}

int cprb_div_host(int64_t n, const double* x, double h, double* out, void* stream) {
  k_div_host<<<ew_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, x, h, out);
  return check_launch("div_host");
}

}  // extern "C"
