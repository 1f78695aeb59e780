// K3-K7, K11: AMG V-cycle on the pressure hierarchy (src/amg.py:228-267).
//
// Every level lives in its colour-permuted order (src/smoothers.py:257-271),
// so a colour is a contiguous run of SELL-32 slices and one launch per
// colour implements the PGS-SCM barrier between colours.  The restriction
// operator stores each aggregate's (<= 2) member rows in adjacent lanes, in
// the level's ORIGINAL column order, so the fused residual + bincount kernel
// reproduces `r - spmv(A_l, x)` and `np.bincount` bitwise.
#include <vector>

#include "device.cuh"
#include "engine.h"

namespace cprb {

// PGS-SCM colour update (src/smoothers.py:106-115):
//   x_i = (b_i - sum_{stored off-diagonals, ascending permuted col} a_ij x_j) / d_i
// ZG: zero initial guess -> only the prefix of entries whose columns precede
//     the colour (earlier colours) can be nonzero; later entries are exact
//     zeros and skipping them is bitwise neutral.
// GATHER: b_i = src[stride * perm[i]] (level-0 CPR restriction, src/cpr.py:132)
//         and it is stored into b for the rest of the cycle.
// SCATTER: final value also written to out[perm[i]] (natural order).
constexpr int SWEEP_PRE = 8;  // entries held in registers across the PDL wait

template <int ZG, int GATHER, int SCATTER>
__global__ void __launch_bounds__(256)
    k_sweep(const cprb_sell S, int s0, int s1, int r0, int r1, const double* __restrict__ diag,
            double* b, const double* __restrict__ gsrc, int gstride,
            const int32_t* __restrict__ perm, const double* xin, double* xout,
            double* __restrict__ sout) {
  pdl_trigger();
  const int w = s0 + (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  // colours are contiguous row ranges padded to whole slices: the row is
  // implied by the lane.  Everything before pdl_wait() is static matrix data.
  const int row = r0 + (w - s0) * 32 + lane;
  const bool active = (w < s1) && (row < r1);
  int len = 0;
  int64_t base = 0;
  double d = 1.0;
  int colr[SWEEP_PRE];
  double valr[SWEEP_PRE];
  int pidx = 0;
  if (active) {
    const int lid = w * 32 + lane;
    len = ZG ? __ldg(S.lane_len_lo + lid) : __ldg(S.lane_len + lid);
    base = __ldg(S.slice_ptr + w) + lane;
    d = __ldg(diag + row);
    if (GATHER || SCATTER) pidx = __ldg(perm + row);
#pragma unroll
    for (int m = 0; m < SWEEP_PRE; ++m)
      if (m < len) {
        colr[m] = __ldg(S.cols + base + (int64_t)m * 32);
        valr[m] = __ldg(S.vals + base + (int64_t)m * 32);
      }
  }
  pdl_wait();
  if (!active) return;
  double bi;
  if (GATHER) {
    bi = gsrc[(int64_t)gstride * pidx];
    b[row] = bi;
  } else {
    bi = b[row];
  }
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < SWEEP_PRE; ++m)
    if (m < len) acc = acc + valr[m] * xin[colr[m]];
  for (int m = SWEEP_PRE; m < len; ++m) {
    const int64_t e = base + (int64_t)m * 32;
    acc = acc + __ldg(S.vals + e) * xin[__ldg(S.cols + e)];
  }
  const double xn = (bi - acc) / d;
  xout[row] = xn;
  if (SCATTER) sout[pidx] = xn;
}

__global__ void k_copy_rows(const cprb_sell S, int s0, int s1, const double* src, double* dst) {
  const int w = s0 + (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= s1) return;
  const int row = S.lane_row[w * 32 + lane];
  if (row >= 0) dst[row] = src[row];
}

// single-colour level: classic sequential GS on the permuted matrix
// (src/smoothers.py:296-299).  One thread: the recurrence is sequential.
__global__ void k_gs_sequential(const cprb_sell S, int n, const double* diag, const double* b,
                                double* x, int reverse) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int t = 0; t < n; ++t) {
    const int i = reverse ? n - 1 - t : t;
    const int w = i >> 5, lane = i & 31;
    const int len = S.lane_len[w * 32 + lane];
    const int64_t base = S.slice_ptr[w] + lane;
    double acc = 0.0;
    for (int m = 0; m < len; ++m) {
      const int64_t e = base + (int64_t)m * 32;
      acc = acc + S.vals[e] * x[S.cols[e]];
    }
    x[i] = (b[i] - acc) / diag[i];
  }
}

// residual r_i = b_i - A_l x (row in original column order, reduceat sum)
// fused with restriction rc[I] = (0 + r_{i1}) + r_{i2}  (np.bincount order).
constexpr int RR_PRE = 16;

template <int K>
__device__ __forceinline__ double rr_sum_fixed(const int* colr, const double* valr,
                                               const double* x) {
  double e[K];
#pragma unroll
  for (int m = 0; m < K; ++m) e[m] = valr[m] * x[colr[m]];
  return segsum_fixed<K>(e);
}

__global__ void __launch_bounds__(256)
    k_resid_restrict(const cprb_sell R, const double* __restrict__ b,
                     const double* __restrict__ x, double* __restrict__ bc) {
  pdl_trigger();
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const bool wok = w < R.nslices;  // warp-uniform
  const int lid = w * 32 + lane;
  int row = -1, len = 0, out = -1;
  int64_t base = 0;
  int colr[RR_PRE];
  double valr[RR_PRE];
  if (wok) {
    row = __ldg(R.lane_row + lid);
    len = __ldg(R.lane_len + lid);
    base = __ldg(R.slice_ptr + w) + lane;
    if ((lane & 1) == 0) out = __ldg(R.agg_out + w * 16 + (lane >> 1));
#pragma unroll
    for (int m = 0; m < RR_PRE; ++m)
      if (m < len) {
        colr[m] = __ldg(R.cols + base + (int64_t)m * 32);
        valr[m] = __ldg(R.vals + base + (int64_t)m * 32);
      }
  }
  pdl_wait();
  if (!wok) return;
  double res = 0.0;
  if (row >= 0) {
    double t;
    switch (len) {
      case 0: t = 0.0; break;
      case 1: t = rr_sum_fixed<1>(colr, valr, x); break;
      case 2: t = rr_sum_fixed<2>(colr, valr, x); break;
      case 3: t = rr_sum_fixed<3>(colr, valr, x); break;
      case 4: t = rr_sum_fixed<4>(colr, valr, x); break;
      case 5: t = rr_sum_fixed<5>(colr, valr, x); break;
      case 6: t = rr_sum_fixed<6>(colr, valr, x); break;
      case 7: t = rr_sum_fixed<7>(colr, valr, x); break;
      case 8: t = rr_sum_fixed<8>(colr, valr, x); break;
      case 9: t = rr_sum_fixed<9>(colr, valr, x); break;
      case 10: t = rr_sum_fixed<10>(colr, valr, x); break;
      case 11: t = rr_sum_fixed<11>(colr, valr, x); break;
      case 12: t = rr_sum_fixed<12>(colr, valr, x); break;
      case 13: t = rr_sum_fixed<13>(colr, valr, x); break;
      case 14: t = rr_sum_fixed<14>(colr, valr, x); break;
      case 15: t = rr_sum_fixed<15>(colr, valr, x); break;
      case 16: t = rr_sum_fixed<16>(colr, valr, x); break;
      default: {
        auto f = [&](int m) -> double {
          const int64_t e = base + (int64_t)m * 32;
          return __ldg(R.vals + e) * x[__ldg(R.cols + e)];
        };
        t = segsum_rt(f, len);
      }
    }
    res = b[row] - t;
  }
  const double other = __shfl_down_sync(CPRB_FULL, res, 1);
  if ((lane & 1) == 0 && out >= 0) bc[out] = (0.0 + res) + other;
}

// prolongation-correct x += ec[agg]  (src/amg.py:264)
__global__ void k_prolong(int n, const int32_t* __restrict__ aggp, const double* __restrict__ xc,
                          double* __restrict__ x) {
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = i < n ? __ldg(aggp + i) : 0;
  pdl_wait();
  if (i < n) x[i] = x[i] + xc[a];
}

// coarsest solve: x = inv(A_L) b, one warp per row, fixed lane/shuffle order
__global__ void k_dense_mv(int n, const double* __restrict__ inv, const double* __restrict__ b,
                           double* __restrict__ x, const int32_t* __restrict__ out_idx) {
  pdl_trigger();
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  constexpr int PRE = 8;
  double a[PRE];
  const double* row = inv + (int64_t)(w < n ? w : 0) * n;
#pragma unroll
  for (int k = 0; k < PRE; ++k) {
    const int c = lane + 32 * k;
    a[k] = (w < n && c < n) ? __ldg(row + c) : 0.0;
  }
  pdl_wait();
  if (w >= n) return;
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < PRE; ++k) {
    const int c = lane + 32 * k;
    if (c < n) s = s + a[k] * b[c];
  }
  for (int c = lane + 32 * PRE; c < n; c += 32) s = s + row[c] * b[c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = s + __shfl_xor_sync(CPRB_FULL, s, o);
  if (lane == 0) x[out_idx ? out_idx[w] : w] = s;
}

__global__ void k_gather(int n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                         int stride, double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[(int64_t)stride * (idx ? idx[i] : i)];
}

__global__ void k_scatter(int n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                          double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx ? idx[i] : i] = src[i];
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

template <int ZG, int G, int SC>
static void launch_sweep(const cprb_amg_level& L, int k, double* b, const double* gsrc,
                         int gstride, const int32_t* perm, const double* xin, double* xout,
                         double* sout, cudaStream_t st) {
  const int s0 = L.color_slices[k], s1 = L.color_slices[k + 1];
  if (s1 <= s0) return;
  const int threads = (s1 - s0) * 32 >= 256 ? 256 : 128;
  launch_pdl(k_sweep<ZG, G, SC>, nblk((int64_t)(s1 - s0) * 32, threads), threads, 0, st,
             L.smoother, s0, s1, L.color_rows[k], L.color_rows[k + 1], L.diag, b, gsrc, gstride,
             perm, xin, xout, sout);
}

int pgs_pass(const cprb_amg_level& L, const double* b_in, double* x, int dir, int zero_guess,
             const double* gsrc, int gstride, const int32_t* perm, double* sout,
             cudaStream_t st) {
  double* b = const_cast<double*>(b_in);
  const int c = L.ncolors;
  if (c == 1) {
    if (gsrc) k_gather<<<nblk(L.n, 256), 256, 0, st>>>(L.n, perm, gsrc, gstride, b);
    if (zero_guess) cudaMemsetAsync(x, 0, sizeof(double) * L.n, st);
    k_gs_sequential<<<1, 1, 0, st>>>(L.smoother, L.n, L.diag, b, x, dir);
    if (sout) k_scatter<<<nblk(L.n, 256), 256, 0, st>>>(L.n, perm, x, sout);
    return check_launch("pgs sequential");
  }
  for (int t = 0; t < c; ++t) {
    const int k = dir ? c - 1 - t : t;
    const int s0 = L.color_slices[k], s1 = L.color_slices[k + 1];
    const bool snap = L.color_snapshot && L.color_snapshot[k];
    double* xout = snap ? L.tmp : x;
    const int zg = zero_guess ? 1 : 0, g = gsrc ? 1 : 0, sc = sout ? 1 : 0;
    const int code = zg * 4 + g * 2 + sc;
    switch (code) {
      case 0: launch_sweep<0, 0, 0>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
      case 1: launch_sweep<0, 0, 1>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
      case 2: launch_sweep<0, 1, 0>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
      case 3: launch_sweep<0, 1, 1>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
      case 4: launch_sweep<1, 0, 0>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
      case 5: launch_sweep<1, 0, 1>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
      case 6: launch_sweep<1, 1, 0>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
      default: launch_sweep<1, 1, 1>(L, k, b, gsrc, gstride, perm, x, xout, sout, st); break;
    }
    if (snap && s1 > s0)
      k_copy_rows<<<nblk((int64_t)(s1 - s0) * 32, 256), 256, 0, st>>>(L.smoother, s0, s1, L.tmp, x);
  }
  return check_launch("pgs pass");
}

int amg_vcycle(const cprb_amg& h, const double* r, double* z, cudaStream_t st) {
  const int nl = h.nlevels;
  if (nl <= 1) {
    k_gather<<<nblk(h.n_coarse, 256), 256, 0, st>>>(h.n_coarse, nullptr, r, h.in_stride, h.coarse_b);
    k_dense_mv<<<nblk((int64_t)h.n_coarse * 32, 256), 256, 0, st>>>(h.n_coarse, h.coarse_inv,
                                                                     h.coarse_b, z, nullptr);
    return check_launch("coarse-only cycle");
  }
  for (int l = 0; l < nl - 1; ++l) {
    const cprb_amg_level& L = h.levels[l];
    int rc = pgs_pass(L, L.b, L.x, 0, 1, l == 0 ? r : nullptr, h.in_stride, h.perm0, nullptr, st);
    if (rc) return rc;
    double* bc = (l + 1 < nl - 1) ? h.levels[l + 1].b : h.coarse_b;
    if (L.restrict_op.nslices > 0)
      launch_pdl(k_resid_restrict, nblk((int64_t)L.restrict_op.nslices * 32, 256), 256, 0, st,
                 L.restrict_op, (const double*)L.b, (const double*)L.x, bc);
  }
  launch_pdl(k_dense_mv, nblk((int64_t)h.n_coarse * 32, 256), 256, 0, st, h.n_coarse,
             h.coarse_inv, (const double*)h.coarse_b, h.coarse_x, (const int32_t*)nullptr);
  for (int l = nl - 2; l >= 0; --l) {
    const cprb_amg_level& L = h.levels[l];
    const double* xc = (l + 1 < nl - 1) ? h.levels[l + 1].x : h.coarse_x;
    launch_pdl(k_prolong, nblk(L.n, 256), 256, 0, st, L.n, L.aggp, xc, L.x);
    int rc = pgs_pass(L, L.b, L.x, 1, 0, nullptr, 0, h.perm0, l == 0 ? z : nullptr, st);
    if (rc) return rc;
  }
  return check_launch("amg v-cycle");
}

}  // namespace cprb

using namespace cprb;

extern "C" int cprb_pgs_scm_pass(const cprb_amg_level* lvl, const double* b, double* x,
                                 int32_t direction, int32_t zero_guess, void* stream) {
  return pgs_pass(*lvl, b, x, direction, zero_guess, nullptr, 0, nullptr, nullptr,
                  (cudaStream_t)stream);
}

extern "C" int cprb_coarse_solve(const cprb_amg* h, const double* b, double* x, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  k_dense_mv<<<nblk((int64_t)h->n_coarse * 32, 256), 256, 0, st>>>(h->n_coarse, h->coarse_inv, b, x,
                                                                    nullptr);
  return check_launch("coarse solve");
}

extern "C" int cprb_resid_restrict(const cprb_amg_level* L, const double* b, const double* x,
                                   double* bc, void* stream) {
  if (L->restrict_op.nslices <= 0) return CPRB_OK;
  k_resid_restrict<<<nblk((int64_t)L->restrict_op.nslices * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      L->restrict_op, b, x, bc);
  return check_launch("resid restrict");
}

extern "C" int cprb_prolong(const cprb_amg_level* L, const double* xc, double* x, void* stream) {
  k_prolong<<<nblk(L->n, 256), 256, 0, (cudaStream_t)stream>>>(L->n, L->aggp, xc, x);
  return check_launch("prolong");
}

extern "C" int cprb_amg_cycle(const cprb_amg* h, const double* r, double* z, void* stream) {
  if (h->cycle != 0) return set_error(CPRB_EUNSUPPORTED, "K-cycle is driven from the host layer");
  return amg_vcycle(*h, r, z, (cudaStream_t)stream);
}
