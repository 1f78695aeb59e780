// K1/K2: BSR (b = 1 or 3) SpMV, residual and CPR stage-2 residual over the
// SELL-32 layout.  One thread per block row; each of the b*b value planes of a
// slot is one coalesced 256-byte warp load.  The expanded scalar row
// (block column m ascending, then c) is summed in numpy's reduceat order
// (src/sparse.py:322-351 via src/_kernels.py:17-45).
#include "device.cuh"
#include "engine.h"

namespace cprb {

// MODE 0: out = A x
// MODE 1: out = rhs - A x
// MODE 2: out = rhs - A (Pi x)  with Pi scattering x (nb) into block slot 0
//         (src/cpr.py:184-185); only the c = 0 value planes are read.
template <int B, int MODE, int K>
__device__ __forceinline__ void bsr_row_fixed(const cprb_sell& A, int64_t base, int lane,
                                              const double* __restrict__ x, double* res) {
  int col[K];
#pragma unroll
  for (int m = 0; m < K; ++m) col[m] = __ldg(A.cols + base + (int64_t)m * 32 + lane);
  double xv[B * K];
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int c = 0; c < B; ++c) {
      if constexpr (MODE == 2)
        xv[B * m + c] = (c == 0) ? __ldg(x + col[m]) : 0.0;
      else
        xv[B * m + c] = __ldg(x + (int64_t)B * col[m] + c);
    }
#pragma unroll
  for (int r = 0; r < B; ++r) {
    double e[B * K];
#pragma unroll
    for (int m = 0; m < K; ++m)
#pragma unroll
      for (int c = 0; c < B; ++c) {
        if (MODE == 2 && c != 0) {
          e[B * m + c] = 0.0;
        } else {
          const double v = __ldg(A.vals + (base + (int64_t)m * 32) * (B * B) +
                                 (int64_t)(r * B + c) * 32 + lane);
          e[B * m + c] = v * xv[B * m + c];
        }
      }
    res[r] = segsum_fixed<B * K>(e);
  }
}

template <int B, int MODE>
__device__ __forceinline__ void bsr_row_generic(const cprb_sell& A, int64_t base, int lane,
                                                int len, const double* __restrict__ x,
                                                double* res) {
#pragma unroll
  for (int r = 0; r < B; ++r) {
    auto f = [&](int t) -> double {
      const int m = t / B, c = t - m * B;
      if (MODE == 2 && c != 0) return 0.0;
      const int64_t e = base + (int64_t)m * 32 + lane;
      const int j = A.cols[e];
      const double xv = (MODE == 2) ? x[j] : x[(int64_t)B * j + c];
      return A.vals[(base + (int64_t)m * 32) * (B * B) + (int64_t)(r * B + c) * 32 + lane] * xv;
    };
    res[r] = segsum_rt(f, B * len);
  }
}

template <int B, int MODE>
__global__ void __launch_bounds__(256) k_bsr(const cprb_sell A, const double* __restrict__ x,
                                             const double* __restrict__ rhs,
                                             double* __restrict__ out, int32_t* flag,
                                             double* __restrict__ sent,
                                             const int32_t* __restrict__ out_idx) {
  pdl_trigger();
  pdl_wait();
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= A.nslices) return;
  const int lid = w * 32 + lane;
  const int row = A.lane_row[lid];
  if (row < 0) return;
  const int len = A.lane_len[lid];
  const int64_t base = A.slice_ptr[w];
  double res[B];
  switch (len) {
    case 0:
#pragma unroll
      for (int r = 0; r < B; ++r) res[r] = 0.0;
      break;
    case 1: bsr_row_fixed<B, MODE, 1>(A, base, lane, x, res); break;
    case 2: bsr_row_fixed<B, MODE, 2>(A, base, lane, x, res); break;
    case 3: bsr_row_fixed<B, MODE, 3>(A, base, lane, x, res); break;
    case 4: bsr_row_fixed<B, MODE, 4>(A, base, lane, x, res); break;
    case 5: bsr_row_fixed<B, MODE, 5>(A, base, lane, x, res); break;
    case 6: bsr_row_fixed<B, MODE, 6>(A, base, lane, x, res); break;
    case 7: bsr_row_fixed<B, MODE, 7>(A, base, lane, x, res); break;
    default: bsr_row_generic<B, MODE>(A, base, lane, len, x, res); break;
  }
  bool bad = false;
  const int64_t ob = out_idx ? (int64_t)out_idx[row] : (int64_t)B * row;
#pragma unroll
  for (int r = 0; r < B; ++r) {
    const int64_t o = (int64_t)B * row + r;
    const double v = (MODE == 0) ? res[r] : rhs[o] - res[r];
    out[ob + r] = v;
    bad |= !isfinite(v);
    if (MODE == 2 && sent) sent[o] = sentinel();
  }
  flag_nonfinite(flag, bad);
}

template <int B, int MODE>
static void launch_bsr(const cprb_sell& A, const double* x, const double* rhs, double* out,
                       int32_t* flag, double* sent, cudaStream_t st, const int32_t* oi) {
  if (A.nslices <= 0) return;
  const int threads = 256;
  const int blocks = (A.nslices * 32 + threads - 1) / threads;
  launch_pdl(k_bsr<B, MODE>, blocks, threads, 0, st, A, x, rhs, out, flag, sent, oi);
}

int bsr_op(int mode, const cprb_sell& A, int b, const double* x, const double* rhs, double* out,
           int32_t* flag, double* sent, cudaStream_t st, const int32_t* oi) {
  if (b == 3) {
    if (mode == 0) launch_bsr<3, 0>(A, x, rhs, out, flag, sent, st, oi);
    else if (mode == 1) launch_bsr<3, 1>(A, x, rhs, out, flag, sent, st, oi);
    else launch_bsr<3, 2>(A, x, rhs, out, flag, sent, st, oi);
  } else if (b == 1) {
    if (mode == 0) launch_bsr<1, 0>(A, x, rhs, out, flag, sent, st, oi);
    else if (mode == 1) launch_bsr<1, 1>(A, x, rhs, out, flag, sent, st, oi);
    else launch_bsr<1, 2>(A, x, rhs, out, flag, sent, st, oi);
  } else {
    return set_error(CPRB_EUNSUPPORTED, "block size " + std::to_string(b) + " not supported on device");
  }
  return check_launch("bsr_op");
}

}  // namespace cprb

using namespace cprb;

extern "C" int cprb_spmv(const cprb_sell* A, int32_t b, const double* x, double* y, int32_t* flag,
                         void* stream) {
  return bsr_op(0, *A, b, x, nullptr, y, flag, nullptr, (cudaStream_t)stream);
}

extern "C" int cprb_residual(const cprb_sell* A, int32_t b, const double* rhs, const double* x,
                             double* r, int32_t* flag, void* stream) {
  return bsr_op(1, *A, b, x, rhs, r, flag, nullptr, (cudaStream_t)stream);
}
