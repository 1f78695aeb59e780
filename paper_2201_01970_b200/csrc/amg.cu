// K3-K7, K11: AMG V-cycle on the pressure hierarchy (src/amg.py:228-267).
//
// Every level lives in its colour-permuted order (src/smoothers.py:257-271),
// so a colour is a contiguous run of SELL-32 slices and one launch per
// colour implements the PGS-SCM barrier between colours.  The restriction
// operator stores each aggregate's (<= 2) member rows in adjacent lanes, in
// the level's ORIGINAL column order, so the fused residual + bincount kernel
// reproduces `r - spmv(A_l, x)` and `np.bincount` bitwise.
#include <cstdio>
#include <string>
#include <vector>

#include "device.cuh"
#include "engine.h"
#include "nvtx.h"

namespace cprb {

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// where the V-cycle kernels let the next launch start (PDL): at entry
// (default) or after their own dependency wait (-DPDL_LATE)
#ifdef PDL_LATE
#define PDL_EARLY_TRIGGER()
#define PDL_LATE_TRIGGER() pdl_trigger()
#else
#define PDL_EARLY_TRIGGER() pdl_trigger()
#define PDL_LATE_TRIGGER()
#endif
// widest register-prefetch template of a colour sweep (rows longer than it
// stream the rest of the row, same summation order)
#ifndef SWEEP_PRE_MAX
#define SWEEP_PRE_MAX 32
#endif

// PGS-SCM colour update (src/smoothers.py:106-115):
//   x_i = (b_i - sum_{stored off-diagonals, ascending permuted col} a_ij x_j) / d_i
// ZG: zero initial guess -> only the prefix of entries whose columns precede
//     the colour (earlier colours) can be nonzero; later entries are exact
//     zeros and skipping them is bitwise neutral.
// GATHER: b_i = src[stride * perm[i]] (level-0 CPR restriction, src/cpr.py:132)
//         and it is stored into b for the rest of the cycle.
// SCATTER: final value also written to out[perm[i]] (natural order).
// SWEEP_PRE (template): entries held in registers across the PDL wait,
// chosen per colour from its widest row so the whole static part of a row is
// fetched while the previous kernel still runs.

// diagnostic V-cycle timeline (cprb_amg_set_log): per launch, block 0 thread 0
// records {kind, start, after pdl_wait, end} as %globaltimer; nullptr = off
__device__ unsigned long long* g_amg_log = nullptr;
__device__ int g_amg_log_n = 0;
constexpr int AMG_LOG_CAP = 4096;

struct AmgMark {
  int idx = -1;
  __device__ __forceinline__ static unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
  }
  __device__ __forceinline__ void start(int kind) {
    if (g_amg_log && blockIdx.x == 0 && threadIdx.x == 0) {
      idx = atomicAdd(&g_amg_log_n, 1);
      if (idx < AMG_LOG_CAP) {
        g_amg_log[4 * idx] = (unsigned long long)kind;
        g_amg_log[4 * idx + 1] = now();
      }
    }
  }
  __device__ __forceinline__ void waited() {
    if (idx >= 0 && idx < AMG_LOG_CAP) g_amg_log[4 * idx + 2] = now();
  }
  __device__ __forceinline__ void end() {
    if (idx >= 0 && idx < AMG_LOG_CAP) g_amg_log[4 * idx + 3] = now();
  }
};

// continue a GS row sum acc += sum_{m0 <= m < len} a_m x[c_m] in storage
// order; entries are fetched CH at a time (all loads of a chunk in flight
// before the first use) so a long coarse-level row costs len/CH dependent
// round trips instead of len.  x is read through L2 (__ldcg): in the
// persistent tail it is rewritten between phases by other CTAs.
template <int CH>
__device__ __forceinline__ double gs_acc_from(const cprb_sell& S, int64_t base, int m0, int len,
                                              const double* x, double acc) {
  for (; m0 < len; m0 += CH) {
    int c[CH];
    double v[CH], xv[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (m0 + k < len) {
        c[k] = __ldg(S.cols + base + (int64_t)(m0 + k) * 32);
        v[k] = __ldg(S.vals + base + (int64_t)(m0 + k) * 32);
      }
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (m0 + k < len) xv[k] = __ldcg(x + c[k]);
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (m0 + k < len) acc = acc + v[k] * xv[k];
  }
  return acc;
}

#ifndef SWEEP_MINB
#define SWEEP_MINB 1
#endif
template <int ZG, int GATHER, int SCATTER, int SWEEP_PRE>
__global__ void __launch_bounds__(256, SWEEP_MINB)
    k_sweep(const cprb_sell S, int s0, int s1, int r0, int r1, const double* __restrict__ diag,
            double* b, const double* __restrict__ gsrc, int gstride,
            const int32_t* __restrict__ perm, const double* xin, double* xout,
            double* __restrict__ sout) {
  PDL_EARLY_TRIGGER();
  AmgMark mk;
  mk.start(1 + ZG);
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
  PDL_LATE_TRIGGER();
  mk.waited();
  if (!active) return;
  double bi;
  if (GATHER) {
    bi = gsrc[(int64_t)gstride * pidx];
    b[row] = bi;
  } else {
    bi = b[row];
  }
  double xv[SWEEP_PRE];
#pragma unroll
  for (int m = 0; m < SWEEP_PRE; ++m) xv[m] = (m < len) ? xin[colr[m]] : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < SWEEP_PRE; ++m)
    if (m < len) acc = acc + valr[m] * xv[m];
  if (len > SWEEP_PRE) acc = gs_acc_from<8>(S, base, SWEEP_PRE, len, xin, acc);
  const double xn = (bi - acc) / d;
  xout[row] = xn;
  if (SCATTER) sout[pidx] = xn;
  mk.end();
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
// The slice width is warp-uniform; lanes walk it predicated and sum with
// segsum_masked, so rows of different length keep the warp converged.
// Streaming form of the reduceat order: a0 + pairwise8(a[1:len]).  Entries are
// fetched CH (a multiple of 8) at a time; the eight pairwise accumulators are
// updated group by group, the tree is formed once the complete groups are
// consumed and the tail is added sequentially, so only r[8] + one chunk are
// live.  Bit-identical to np.add.reduceat for len <= 129 (no >128 split).
template <int CH>
__device__ __forceinline__ double rr_row_stream(const cprb_sell& R, int64_t base, int len,
                                                const double* x) {
  static_assert(CH % 8 == 0, "chunk must hold whole groups of 8");
  if (len <= 0) return 0.0;
  const int n = len - 1;
  const int nf = n >= 8 ? (n & ~7) : 0;
  double a0 = 0.0, s = -0.0, r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = 0.0;
  for (int p0 = 0; p0 < len; p0 += CH) {  // p = storage position, q = p - 1
    int c[CH];
    double v[CH], e[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (p0 + k < len) {
        c[k] = __ldg(R.cols + base + (int64_t)(p0 + k) * 32);
        v[k] = __ldg(R.vals + base + (int64_t)(p0 + k) * 32);
      }
#pragma unroll
    for (int k = 0; k < CH; ++k) e[k] = (p0 + k < len) ? v[k] * __ldcg(x + c[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int p = p0 + k;
      if (p >= len) break;
      if (p == 0) {
        a0 = e[k];
        continue;
      }
      const int q = p - 1;
      if (q < nf) {
        if (q < 8) r[q & 7] = e[k];
        else r[q & 7] = r[q & 7] + e[k];
        if (q == nf - 1) s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      } else {
        s = s + e[k];
      }
    }
  }
  return a0 + s;
}

__device__ __forceinline__ double rr_row(const cprb_sell& R, int64_t base, int width, int len,
                                         const double* x) {
  if (len <= 129) return rr_row_stream<8>(R, base, len, x);
  auto f = [&](int m) -> double {
    const int64_t e = base + (int64_t)m * 32;
    return __ldg(R.vals + e) * __ldcg(x + __ldg(R.cols + e));
  };
  return segsum_rt(f, len);
}

// one warp = one restriction slice (16 aggregates); returns nothing, writes bc
__device__ __forceinline__ void rr_slice(const cprb_sell& R, int w, int lane, const double* b,
                                         const double* x, double* bc) {
  const int lid = w * 32 + lane;
  const int row = __ldg(R.lane_row + lid);
  const int len = row >= 0 ? __ldg(R.lane_len + lid) : 0;
  const int64_t sb = __ldg(R.slice_ptr + w);
  const int width = (int)((__ldg(R.slice_ptr + w + 1) - sb) >> 5);
  const int out = ((lane & 1) == 0) ? __ldg(R.agg_out + w * 16 + (lane >> 1)) : -1;
  double res = 0.0;
  if (width > 0) {
    const double t = rr_row(R, sb + lane, width, len, x);
    if (row >= 0) res = __ldcg(b + row) - t;
  } else if (row >= 0) {
    res = __ldcg(b + row) - 0.0;
  }
  const double other = __shfl_down_sync(CPRB_FULL, res, 1);
  if ((lane & 1) == 0 && out >= 0) bc[out] = (0.0 + res) + other;
}

// standalone launch: the static part of the slice (columns, values, output
// slots) is fetched before the PDL wait; rows longer than PRE fall back to
// the streaming sum.
// long rows (> PRE entries) leave the register path: kept out of line so the
// common case is not charged the fallback's registers
__device__ __noinline__ double rr_row_far(const cprb_sell& R, int64_t base, int len,
                                          const double* x) {
  return rr_row(R, base, 0, len, x);
}

template <int PRE>
__global__ void __launch_bounds__(256, PRE <= 8 ? 6 : (PRE <= 16 ? 4 : 2))
    k_resid_restrict(const cprb_sell R, const double* __restrict__ b,
                     const double* __restrict__ x, double* __restrict__ bc,
                     double* __restrict__ xn, const double* __restrict__ dn, int c0_rows) {
  PDL_EARLY_TRIGGER();
  AmgMark mk;
  mk.start(3);
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const bool wok = w < R.nslices;  // warp-uniform
  int row = -1, len = 0, out = -1;
  int64_t base = 0;
  int c[PRE];
  double v[PRE];
  if (wok) {
    const int lid = w * 32 + lane;
    row = __ldg(R.lane_row + lid);
    len = row >= 0 ? __ldg(R.lane_len + lid) : 0;
    base = __ldg(R.slice_ptr + w) + lane;
    if ((lane & 1) == 0) out = __ldg(R.agg_out + w * 16 + (lane >> 1));
#pragma unroll
    for (int m = 0; m < PRE; ++m)
      if (m < len) {
        c[m] = __ldg(R.cols + base + (int64_t)m * 32);
        v[m] = __ldg(R.vals + base + (int64_t)m * 32);
      }
  }
  pdl_wait();
  PDL_LATE_TRIGGER();
  mk.waited();
  if (!wok) return;
  double res = 0.0;
  if (row >= 0) {
    double t;
    if (len <= PRE) {
      double e[PRE];
#pragma unroll
      for (int m = 0; m < PRE; ++m) e[m] = (m < len) ? v[m] * __ldg(x + c[m]) : 0.0;
      t = segsum_masked<PRE>(e, len);
    } else {
      t = rr_row_far(R, base, len, x);
    }
    res = __ldg(b + row) - t;
  }
  const double other = __shfl_down_sync(CPRB_FULL, res, 1);
  if ((lane & 1) == 0 && out >= 0) {
    const double bcv = (0.0 + res) + other;
    bc[out] = bcv;
    // fused first colour of the next level's zero-guess forward sweep: its
    // rows read no x (no earlier colour), so x = (b - 0.0) / d exactly as
    // k_sweep computes it (src/smoothers.py:106-115)
    if (xn && out < c0_rows) xn[out] = (bcv - 0.0) / dn[out];
  }
  mk.end();
}

// `next` (optional): the next (smoothed, multi-colour) level whose zero-guess
// first colour is computed by this kernel
static void launch_rr(const cprb_amg_level& L, const double* b, const double* x, double* bc,
                      cudaStream_t st, const cprb_amg_level* next = nullptr) {
  const cprb_sell& R = L.restrict_op;
  if (R.nslices <= 0) return;
  const int grid = nblk((int64_t)R.nslices * 32, 256);
  const int wdt = L.restrict_width > 0 ? L.restrict_width : 32;
  double* xn = next ? next->x : nullptr;
  const double* dn = next ? next->diag : nullptr;
  const int c0 = next ? next->color_rows[1] : 0;
  if (wdt <= 8) launch_pdl(k_resid_restrict<8>, grid, 256, 0, st, R, b, x, bc, xn, dn, c0);
  else if (wdt <= 16) launch_pdl(k_resid_restrict<16>, grid, 256, 0, st, R, b, x, bc, xn, dn, c0);
  else launch_pdl(k_resid_restrict<32>, grid, 256, 0, st, R, b, x, bc, xn, dn, c0);
}

// prolongation-correct x += ec[agg]  (src/amg.py:264)
__global__ void k_prolong(int n, const int32_t* __restrict__ aggp, const double* __restrict__ xc,
                          double* __restrict__ x) {
  PDL_EARLY_TRIGGER();
  AmgMark mk;
  mk.start(4);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = i < n ? __ldg(aggp + i) : 0;
  pdl_wait();
  PDL_LATE_TRIGGER();
  mk.waited();
  if (i < n) x[i] = x[i] + xc[a];
  mk.end();
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

template <int ZG, int G, int SC>
static void launch_sweep(const cprb_amg_level& L, int k, double* b, const double* gsrc,
                         int gstride, const int32_t* perm, const double* xin, double* xout,
                         double* sout, cudaStream_t st) {
  const int s0 = L.color_slices[k], s1 = L.color_slices[k + 1];
  if (s1 <= s0) return;
  // rows wider than 8 take the register-heavy templates: small blocks let
  // more warps share an SM (measured at C3: V-cycle 703 -> 673 us)
  const int wq = L.color_width ? L.color_width[2 * k + (ZG ? 1 : 0)] : 8;
  const int threads = wq > 8 ? 64 : ((s1 - s0) * 32 >= 256 ? 256 : 128);
  int width = L.color_width ? L.color_width[2 * k + (ZG ? 1 : 0)] : 8;
  if (width > SWEEP_PRE_MAX) width = SWEEP_PRE_MAX;
  const int grid = nblk((int64_t)(s1 - s0) * 32, threads);
  auto go = [&](auto kern) {
    launch_pdl(kern, grid, threads, 0, st, L.smoother, s0, s1, L.color_rows[k],
               L.color_rows[k + 1], L.diag, b, gsrc, gstride, perm, xin, xout, sout);
  };
  if (width <= 4) go(k_sweep<ZG, G, SC, 4>);
  else if (width <= 8) go(k_sweep<ZG, G, SC, 8>);
  else if (width <= 16) go(k_sweep<ZG, G, SC, 16>);
  else go(k_sweep<ZG, G, SC, 32>);
}

int pgs_pass(const cprb_amg_level& L, const double* b_in, double* x, int dir, int zero_guess,
             const double* gsrc, int gstride, const int32_t* perm, double* sout,
             cudaStream_t st, int skip_first) {
  double* b = const_cast<double*>(b_in);
  const int c = L.ncolors;
  if (c == 1) {
    if (gsrc) k_gather<<<nblk(L.n, 256), 256, 0, st>>>(L.n, perm, gsrc, gstride, b);
    if (zero_guess) cudaMemsetAsync(x, 0, sizeof(double) * L.n, st);
    k_gs_sequential<<<1, 1, 0, st>>>(L.smoother, L.n, L.diag, b, x, dir);
    if (sout) k_scatter<<<nblk(L.n, 256), 256, 0, st>>>(L.n, perm, x, sout);
    return check_launch("pgs sequential");
  }
  for (int t = skip_first; t < c; ++t) {
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
  NvtxRange nv("amg_vcycle");
  const int nl = h.nlevels;
  if (nl <= 1) {
    k_gather<<<nblk(h.n_coarse, 256), 256, 0, st>>>(h.n_coarse, nullptr, r, h.in_stride, h.coarse_b);
    k_dense_mv<<<nblk((int64_t)h.n_coarse * 32, 256), 256, 0, st>>>(h.n_coarse, h.coarse_inv,
                                                                     h.coarse_b, z, nullptr);
    return check_launch("coarse-only cycle");
  }
  // levels >= ts (and the coarse solve) run in the persistent tail
  const bool tail = h.tail_start >= 1 && h.tail_start < nl - 1 && h.tail_nphases > 0 &&
                    h.tail_stream && h.tail_phases && h.tail_chunks && h.tail_vec;
  const int ts = tail ? h.tail_start : nl - 1;
  int fused = 0;  // colour 0 of this level was computed by the previous restriction
  for (int l = 0; l < ts; ++l) {
    const cprb_amg_level& L = h.levels[l];
    int rc = pgs_pass(L, L.b, L.x, 0, 1, l == 0 ? r : nullptr, h.in_stride, h.perm0, nullptr, st,
                      fused);
    if (rc) return rc;
    double* bc = (l + 1 < nl - 1) ? h.levels[l + 1].b : h.coarse_b;
    const cprb_amg_level* next = (l + 1 < ts && h.levels[l + 1].ncolors > 1) ? &h.levels[l + 1] : nullptr;
    launch_rr(L, L.b, L.x, bc, st, next);
    fused = next ? 1 : 0;
  }
  if (tail) {
    int rc = launch_vtail(h, st);
    if (rc) return rc;
  } else {
    launch_pdl(k_dense_mv, nblk((int64_t)h.n_coarse * 32, 256), 256, 0, st, h.n_coarse,
               h.coarse_inv, (const double*)h.coarse_b, h.coarse_x, (const int32_t*)nullptr);
  }
  for (int l = ts - 1; l >= 0; --l) {
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

extern "C" int cprb_amg_set_log(uint64_t* dev_log) {
  unsigned long long* p = (unsigned long long*)dev_log;
  int zero = 0;
  cudaMemcpyToSymbol(cprb::g_amg_log, &p, sizeof(p));
  cudaMemcpyToSymbol(cprb::g_amg_log_n, &zero, sizeof(zero));
  return check_launch("amg log");
}

extern "C" int cprb_pgs_scm_pass(const cprb_amg_level* lvl, const double* b, double* x,
                                 int32_t direction, int32_t zero_guess, void* stream) {
  return pgs_pass(*lvl, b, x, direction, zero_guess, nullptr, 0, nullptr, nullptr,
                  (cudaStream_t)stream);
}

// one colour of a PGS-SCM pass (slab-partitioned path: the host exchanges
// halo values between colours); no snapshot colours (theta_amg = 0 levels)
extern "C" int cprb_pgs_scm_color(const cprb_amg_level* lvl, int32_t k, double* b, double* x,
                                  int32_t zero_guess, const double* gsrc, int32_t gstride,
                                  const int32_t* perm, double* sout, void* stream) {
  const cprb_amg_level& L = *lvl;
  cudaStream_t st = (cudaStream_t)stream;
  if (k < 0 || k >= L.ncolors) return set_error(CPRB_EINVAL, "colour index out of range");
  // a colour with intra-colour couplings reads the snapshot of x taken at
  // the colour's start (src/smoothers.py:301-308): write to tmp, copy back
  const bool snap = L.color_snapshot && L.color_snapshot[k];
  double* xo = snap ? L.tmp : x;
  const int code = (zero_guess ? 4 : 0) + (gsrc ? 2 : 0) + (sout ? 1 : 0);
  switch (code) {
    case 0: launch_sweep<0, 0, 0>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
    case 1: launch_sweep<0, 0, 1>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
    case 2: launch_sweep<0, 1, 0>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
    case 3: launch_sweep<0, 1, 1>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
    case 4: launch_sweep<1, 0, 0>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
    case 5: launch_sweep<1, 0, 1>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
    case 6: launch_sweep<1, 1, 0>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
    default: launch_sweep<1, 1, 1>(L, k, b, gsrc, gstride, perm, x, xo, sout, st); break;
  }
  const int s0 = L.color_slices[k], s1 = L.color_slices[k + 1];
  if (snap && s1 > s0)
    k_copy_rows<<<nblk((int64_t)(s1 - s0) * 32, 256), 256, 0, st>>>(L.smoother, s0, s1, L.tmp, x);
  return check_launch("pgs colour");
}

extern "C" int cprb_coarse_solve(const cprb_amg* h, const double* b, double* x, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  k_dense_mv<<<nblk((int64_t)h->n_coarse * 32, 256), 256, 0, st>>>(h->n_coarse, h->coarse_inv, b, x,
                                                                    nullptr);
  return check_launch("coarse solve");
}

extern "C" int cprb_resid_restrict(const cprb_amg_level* L, const double* b, const double* x,
                                   double* bc, void* stream) {
  launch_rr(*L, b, x, bc, (cudaStream_t)stream);
  return check_launch("resid restrict");
}

extern "C" int cprb_prolong(const cprb_amg_level* L, const double* xc, double* x, void* stream) {
  k_prolong<<<nblk(L->n, 256), 256, 0, (cudaStream_t)stream>>>(L->n, L->aggp, xc, x);
  return check_launch("prolong");
}

extern "C" int cprb_amg_cycle(const cprb_amg* h, const double* r, double* z, void* stream) {
  if (h->cycle != 0) return kcycle_apply(*h, r, z, (cudaStream_t)stream);
  return amg_vcycle(*h, r, z, (cudaStream_t)stream);
}
