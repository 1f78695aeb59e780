// SETUP on the device: BILU(0) factorization (src/ilu.py:150-193) and the
// structured-grid ("stencil") packing of the factors for csrc/stencil.cu.
//
// The factorization is the IKJ loop of csrc/setup.cpp (bilu0_rows<3>) run
// level by level: rows of one level of the lower-triangular dependency
// schedule (src/ilu.py:38-59) only read rows of earlier levels, so a level
// is one launch with one thread per row.  Every 3x3 product, subtraction and
// Gauss-Jordan pivot inversion is the host loop's, operation for operation
// (-fmad=false), so the device factors are bitwise the host C++ factors
// (which match the reference's OpenBLAS-ordered products to ~1e-15).
// A singular pivot with a nonzero Frobenius norm is perturbed by
// 1e-8 ||B||_F I exactly as on the host (src/ilu.py:134-147); the perturbed
// rows are reported, and a zero pivot block reports its row (the lowest
// such row, which is the one the sequential host loop stops at).
#include <cmath>

#include "device.cuh"
#include "engine.h"
#include "nvtx.h"

namespace cprb {

__device__ __forceinline__ void mm3(const double* x, const double* y, double* out) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) s = s + x[i * 3 + j] * y[j * 3 + l];
      out[i * 3 + l] = s;
    }
}

// csrc/setup.cpp gj_invert, b = 3
__device__ bool gj3(const double* blk, double* inv) {
  double a[9], v[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    a[i] = blk[i];
    v[i] = (i % 4 == 0) ? 1.0 : 0.0;
  }
  for (int col = 0; col < 3; ++col) {
    int p = col;
    double best = fabs(a[col * 3 + col]);
    for (int r = col + 1; r < 3; ++r)
      if (fabs(a[r * 3 + col]) > best) {
        best = fabs(a[r * 3 + col]);
        p = r;
      }
    if (a[p * 3 + col] == 0.0) return false;
    if (p != col)
      for (int c = 0; c < 3; ++c) {
        double t = a[col * 3 + c];
        a[col * 3 + c] = a[p * 3 + c];
        a[p * 3 + c] = t;
        t = v[col * 3 + c];
        v[col * 3 + c] = v[p * 3 + c];
        v[p * 3 + c] = t;
      }
    const double piv = a[col * 3 + col];
    for (int c = 0; c < 3; ++c) {
      a[col * 3 + c] /= piv;
      v[col * 3 + c] /= piv;
    }
    for (int r = 0; r < 3; ++r) {
      if (r == col) continue;
      const double f = a[r * 3 + col];
      if (f != 0.0)
        for (int c = 0; c < 3; ++c) {
          a[r * 3 + c] = a[r * 3 + c] - f * a[col * 3 + c];
          v[r * 3 + c] = v[r * 3 + c] - f * v[col * 3 + c];
        }
    }
  }
#pragma unroll
  for (int i = 0; i < 9; ++i) inv[i] = v[i];
  return true;
}

// numpy pairwise sum of the 9 squared entries (csrc/setup.cpp pairwise_sum, n = 9)
__device__ __forceinline__ double pairwise9(const double* a) {
  const double s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  return s + a[8];
}

// err[0]: lowest row with a zero pivot block (INT32_MAX = none)
// err[1]: lowest row with a missing diagonal block; err[2]: perturbed count
__global__ void k_bilu_level(const int32_t* __restrict__ rows, int nrows, const int64_t* __restrict__ ptr,
                             const int64_t* __restrict__ cols, double* vals, double* uinv,
                             int32_t* err, int64_t* perturbed) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int64_t i = rows[t];
  const int64_t lo = ptr[i], hi = ptr[i + 1];
  int64_t dk = lo;
  while (dk < hi && cols[dk] < i) ++dk;
  if (dk >= hi || cols[dk] != i) {
    atomicMin(err + 1, (int)i);
    return;
  }
  double tmp[9];
  for (int64_t p = lo; p < dk; ++p) {
    const int64_t k = cols[p];
    double lik[9];
    mm3(vals + p * 9, uinv + k * 9, lik);
#pragma unroll
    for (int e = 0; e < 9; ++e) vals[p * 9 + e] = lik[e];
    const int64_t khi = ptr[k + 1];
    int64_t pos = ptr[k];
    for (int64_t q = p + 1; q < hi; ++q) {
      const int64_t j = cols[q];
      while (pos < khi && cols[pos] < j) ++pos;
      if (pos < khi && cols[pos] == j) {
        mm3(lik, vals + pos * 9, tmp);
#pragma unroll
        for (int e = 0; e < 9; ++e) vals[q * 9 + e] = vals[q * 9 + e] - tmp[e];
      }
    }
  }
  const double* piv = vals + dk * 9;
  double* ui = uinv + i * 9;
  if (!gj3(piv, ui)) {
    double sq[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) sq[e] = piv[e] * piv[e];
    const double fro = sqrt(pairwise9(sq));
    bool ok = fro != 0.0;
    if (ok) {
      const double tt = 1e-8 * fro;
      double bumped[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) bumped[e] = piv[e] + ((e % 4 == 0) ? tt * 1.0 : tt * 0.0);
      ok = gj3(bumped, ui);
    }
    if (!ok) {
      atomicMin(err, (int)i);
    } else {
      const int slot = atomicAdd(err + 2, 1);
      perturbed[slot] = i;
    }
  }
}

// factored CSR (A's pattern, L\U in place) -> stencil records (ilu.py
// stencil_plan): row (ix, iy, iz) at position pos = iz*P + doff[ix+iy] +
// ix - lo(ix+iy); L record 27 doubles (m: -z, -y, -x), U record 37 doubles
// (m: +x, +y, +z, then inv(U_ii), one pad word); absent neighbours stay 0
__global__ void k_stencil_pack(int64_t n, int nx, int ny, int P, const int32_t* __restrict__ doff,
                               const int64_t* __restrict__ ptr, const int64_t* __restrict__ cols,
                               const double* __restrict__ vals, const double* __restrict__ uinv,
                               double* __restrict__ lrec, double* __restrict__ urec,
                               int32_t* __restrict__ slot) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t nxy = (int64_t)nx * ny;
  const int ix = (int)(i % nx), iy = (int)((i / nx) % ny);
  const int64_t iz = i / nxy;
  const int d = ix + iy;
  const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
  const int64_t pos = iz * P + doff[d] + (ix - lo);
  slot[i] = (int32_t)(3 * pos);
  double* L = lrec + pos * 27;
  double* U = urec + pos * 37;
  for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) {
    const int64_t off = cols[p] - i;
    int m;
    double* dst;
    if (off == 0) continue;
    if (off < 0) {
      m = off == -nxy ? 0 : (off == -(int64_t)nx ? 1 : 2);
      dst = L + m * 9;
    } else {
      m = off == 1 ? 0 : (off == (int64_t)nx ? 1 : 2);
      dst = U + m * 9;
    }
#pragma unroll
    for (int e = 0; e < 9; ++e) dst[e] = vals[p * 9 + e];
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) U[27 + e] = uinv[i * 9 + e];
}

}  // namespace cprb

using namespace cprb;

// level_rows: dev, rows grouped by level; level_ptr: HOST, nlevels+1.
// err: dev int32[4] (initialised here); perturbed: dev, capacity n.
extern "C" int cprb_bilu0_factorize_device(int64_t n, int32_t b, const int64_t* ptr,
                                           const int64_t* cols, double* vals, double* uinv,
                                           const int32_t* level_rows, const int64_t* level_ptr,
                                           int64_t nlevels, int32_t* err, int64_t* perturbed,
                                           void* stream) {
  if (b != 3) return set_error(CPRB_EUNSUPPORTED, "device BILU(0) factorization needs 3x3 blocks");
  NvtxRange nv("bilu0_factorize_device");
  cudaStream_t st = (cudaStream_t)stream;
  const int32_t init[4] = {0x7fffffff, 0x7fffffff, 0, 0};
  cudaMemcpyAsync(err, init, sizeof(init), cudaMemcpyHostToDevice, st);
  for (int64_t l = 0; l < nlevels; ++l) {
    const int64_t a = level_ptr[l], m = level_ptr[l + 1] - a;
    if (m <= 0) continue;
    k_bilu_level<<<(int)((m + 127) / 128), 128, 0, st>>>(level_rows + a, (int)m, ptr, cols, vals,
                                                          uinv, err, perturbed);
  }
  return check_launch("bilu0 factorize (device)");
}

extern "C" int cprb_stencil_pack(int64_t n, int32_t nx, int32_t ny, int32_t P, const int32_t* doff,
                                 const int64_t* ptr, const int64_t* cols, const double* vals,
                                 const double* uinv, double* lrec, double* urec, int32_t* slot,
                                 void* stream) {
  if (n <= 0) return CPRB_OK;
  k_stencil_pack<<<(int)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      n, nx, ny, P, doff, ptr, cols, vals, uinv, lrec, urec, slot);
  return check_launch("stencil pack");
}
