// K1/K2: BSR (b = 1 or 3) SpMV, residual and CPR stage-2 residual over the
// SELL-32 layout.  One thread per block row; each of the b*b value planes of a
// slot is one coalesced 256-byte warp load.  The expanded scalar row
// (block column m ascending, then c) is summed in numpy's reduceat order
// (src/sparse.py:322-351 via src/_kernels.py:17-45).
#include "device.cuh"
#include "engine.h"
#include "nvtx.h"

namespace cprb {

// MODE 0: out = A x
// MODE 1: out = rhs - A x
// MODE 2: out = rhs - A (Pi x)  with Pi scattering x (nb) into block slot 0
//         (src/cpr.py:184-185); only the c = 0 value planes are read.
//
// Work split: B warps per SELL slice, warp r computes scalar output row r of
// the slice's 32 block rows (so each thread holds one expanded row: 3K values,
// K columns, 3K x entries -> ~60 registers, 4x the occupancy of a thread per
// block row).  The slice width (max blocks per row) is warp-uniform; every
// lane walks it with predication and sums with segsum_masked, so lanes with
// shorter rows (grid boundaries) never split the warp.  Value planes (r, c)
// of a slot are 256-byte coalesced warp loads; the x gathers of the B warps
// of a slice hit the same L1 lines.
constexpr int BSR_WARPS = 6;  // warps per CTA (2 slices of a 3x3 BSR)

template <int B, int MODE, int K>
__device__ __forceinline__ double bsr_row_k(const cprb_sell& A, int64_t base, int lane, int r,
                                            int len, const double* __restrict__ x) {
  int col[K];
#pragma unroll
  for (int m = 0; m < K; ++m) col[m] = (m < len) ? __ldg(A.cols + base + (int64_t)m * 32 + lane) : 0;
  double e[B * K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    const double* vp = A.vals + (base + (int64_t)m * 32) * (B * B) + (int64_t)(r * B) * 32 + lane;
#pragma unroll
    for (int c = 0; c < B; ++c) {
      if (MODE == 2 && c != 0) {
        e[B * m + c] = 0.0;
      } else if (m < len) {
        const double xv = (MODE == 2) ? __ldg(x + col[m]) : __ldg(x + (int64_t)B * col[m] + c);
        e[B * m + c] = __ldg(vp + c * 32) * xv;
      } else {
        e[B * m + c] = 0.0;
      }
    }
  }
  return segsum_masked<B * K>(e, B * len);
}

template <int B, int MODE>
__device__ __forceinline__ double bsr_row_long(const cprb_sell& A, int64_t base, int lane, int r,
                                               int len, const double* __restrict__ x) {
  auto f = [&](int t) -> double {
    const int m = t / B, c = t - m * B;
    if (MODE == 2 && c != 0) return 0.0;
    const int64_t e = base + (int64_t)m * 32 + lane;
    const int j = __ldg(A.cols + e);
    const double xv = (MODE == 2) ? __ldg(x + j) : __ldg(x + (int64_t)B * j + c);
    return __ldg(A.vals + (base + (int64_t)m * 32) * (B * B) + (int64_t)(r * B + c) * 32 + lane) * xv;
  };
  return segsum_rt(f, B * len);
}

// resident CTAs per SM: the full products keep 5 (more spills their
// register prefetch: 139 -> 145 / 180 us at 6 / 8); the stage-2 residual
// (one value plane per block) is latency bound and gains from 8 (CPR
// application 1268 -> 1241 us at C3)
template <int B, int MODE>
__global__ void __launch_bounds__(BSR_WARPS * 32, MODE == 2 ? 8 : 5)
    k_bsr(const cprb_sell A, const double* __restrict__ x, const double* __restrict__ rhs,
          double* __restrict__ out, int32_t* flag, double* __restrict__ sent,
          double* __restrict__ sent2, const int32_t* __restrict__ out_idx,
          const int32_t* __restrict__ sent_idx, const int32_t* __restrict__ sent2_idx) {
  pdl_trigger();
  const int gw = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int s = gw / B;
  const int r = gw - s * B;
  if (s >= A.nslices) return;
  const int lid = s * 32 + lane;
  const int64_t base = __ldg(A.slice_ptr + s);
  const int width = (int)((__ldg(A.slice_ptr + s + 1) - base) >> 5);
  const int row = __ldg(A.lane_row + lid);
  const int len = row >= 0 ? __ldg(A.lane_len + lid) : 0;
  pdl_wait();
  double v;
  switch (width) {
    case 0: v = 0.0; break;
    case 1: v = bsr_row_k<B, MODE, 1>(A, base, lane, r, len, x); break;
    case 2: v = bsr_row_k<B, MODE, 2>(A, base, lane, r, len, x); break;
    case 3: v = bsr_row_k<B, MODE, 3>(A, base, lane, r, len, x); break;
    case 4: v = bsr_row_k<B, MODE, 4>(A, base, lane, r, len, x); break;
    case 5: v = bsr_row_k<B, MODE, 5>(A, base, lane, r, len, x); break;
    case 6: v = bsr_row_k<B, MODE, 6>(A, base, lane, r, len, x); break;
    case 7: v = bsr_row_k<B, MODE, 7>(A, base, lane, r, len, x); break;
    case 8: v = bsr_row_k<B, MODE, 8>(A, base, lane, r, len, x); break;
    default: v = bsr_row_long<B, MODE>(A, base, lane, r, len, x); break;
  }
  if (row < 0) return;
  const int64_t o = (int64_t)B * row + r;
  if (MODE != 0) v = rhs[o] - v;
  const int64_t ob = out_idx ? (int64_t)out_idx[row] + r : o;
  out[ob] = v;
  if (MODE == 2 && sent) sent[sent_idx ? (int64_t)sent_idx[row] + r : o] = sentinel();
  if (MODE == 2 && sent2) sent2[sent2_idx ? (int64_t)sent2_idx[row] + r : o] = sentinel();
  flag_nonfinite(flag, !isfinite(v));
}

template <int B, int MODE>
static void launch_bsr(const cprb_sell& A, const double* x, const double* rhs, double* out,
                       int32_t* flag, double* sent, double* sent2, cudaStream_t st,
                       const int32_t* oi, const int32_t* si, const int32_t* si2) {
  if (A.nslices <= 0) return;
  const int threads = BSR_WARPS * 32;
  const int64_t warps = (int64_t)A.nslices * B;
  const int blocks = (int)((warps + BSR_WARPS - 1) / BSR_WARPS);
  launch_pdl(k_bsr<B, MODE>, blocks, threads, 0, st, A, x, rhs, out, flag, sent, sent2, oi, si,
             si2);
}

int bsr_op(int mode, const cprb_sell& A, int b, const double* x, const double* rhs, double* out,
           int32_t* flag, double* sent, cudaStream_t st, const int32_t* oi, double* sent2,
           const int32_t* si, const int32_t* si2) {
  NvtxRange nv(mode == 0 ? "bsr_spmv" : (mode == 1 ? "bsr_residual" : "bsr_stage2_residual"));
  if (b == 3) {
    if (mode == 0) launch_bsr<3, 0>(A, x, rhs, out, flag, sent, sent2, st, oi, si, si2);
    else if (mode == 1) launch_bsr<3, 1>(A, x, rhs, out, flag, sent, sent2, st, oi, si, si2);
    else launch_bsr<3, 2>(A, x, rhs, out, flag, sent, sent2, st, oi, si, si2);
  } else if (b == 1) {
    if (mode == 0) launch_bsr<1, 0>(A, x, rhs, out, flag, sent, sent2, st, oi, si, si2);
    else if (mode == 1) launch_bsr<1, 1>(A, x, rhs, out, flag, sent, sent2, st, oi, si, si2);
    else launch_bsr<1, 2>(A, x, rhs, out, flag, sent, sent2, st, oi, si, si2);
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

// src/cpr.py:185  r2 = r - A (Pi zp), reading only block column 0 (zp holds
// the pressure values, one per block column)
extern "C" int cprb_stage2_residual(const cprb_sell* A, int32_t b, const double* zp,
                                    const double* r, double* r2, void* stream) {
  return bsr_op(2, *A, b, zp, r, r2, nullptr, nullptr, (cudaStream_t)stream);
}

// device SELL-32 packing of a BSR matrix in natural row order (the layout of
// device.sell_rows / pack_sell): entry m of row i lands at slot
// slice_ptr[i/32] + 32 m + i%32; values verbatim, padding left as zeros
__global__ void k_pack_bsr_sell(int64_t nrows, int bb, const int64_t* __restrict__ rp,
                                const int64_t* __restrict__ ci, const double* __restrict__ v,
                                const int64_t* __restrict__ slice_ptr, int32_t* __restrict__ cols,
                                double* __restrict__ vals) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= nrows) return;
  const int64_t e0 = rp[row], e1 = rp[row + 1];
  const int64_t sb = slice_ptr[row >> 5];
  const int l = (int)(row & 31);
  for (int64_t e = e0; e < e1; ++e) {
    const int64_t slot = sb + (e - e0) * 32 + l;
    if (lane == 0) cols[slot] = (int32_t)ci[e];
    for (int q = lane; q < bb; q += 32)
      vals[(slot - l) * bb + (int64_t)q * 32 + l] = v[e * bb + q];
  }
}

extern "C" int cprb_pack_bsr_sell(int64_t nrows, int32_t b, const int64_t* row_ptr,
                                  const int64_t* col_idx, const double* values,
                                  const int64_t* slice_ptr, int32_t* cols, double* vals,
                                  void* stream) {
  if (nrows <= 0) return CPRB_OK;
  const int per = 8;  // rows (warps) per CTA
  const int64_t grid = (nrows + per - 1) / per;
  k_pack_bsr_sell<<<(unsigned)grid, per * 32, 0, (cudaStream_t)stream>>>(
      nrows, b * b, row_ptr, col_idx, values, slice_ptr, cols, vals);
  return check_launch("pack bsr sell");
}
