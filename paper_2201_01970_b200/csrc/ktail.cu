// Persistent K-cycle tail (src/amg.py:177-225, :245-267).
//
// The K-cycle wraps every coarse recursion in two Krylov steps, so level l is
// visited 2^l times per application: 8,191 level visits and ~35 dependent
// phases each at C3 (14 levels).  Launched kernel by kernel that is ~290k
// dependent launches per application.  Below a size threshold the whole
// remaining recursion -- FCG (or FGMRES) at level `start`, the PGS-SCM colour
// sweeps, residual + restriction, prolongation, the coarse dense solve and
// every Krylov scalar -- runs inside ONE CTA: a phase is a __syncthreads, the
// recursion is ordinary (compile-time unrolled) control flow on block-uniform
// shared-memory scalars, and the coarse levels' vectors stay in the SM's L1.
//
// Arithmetic is the launched K-cycle's (csrc/kcycle.cu) operation for
// operation: the sweep rows of k_sweep, the reduceat rows of
// k_resid_restrict / k_bsr<1,0>, the fixed-partition tree of cprb_dot
// (red_blocks(n) virtual CTAs of 256 threads, xor-shuffle tree, warps in
// order, partials in order), k_kdense's lane-strided coarse rows, and the
// same separately rounded axpys -- so the tail is bitwise equal to it.
// "norm2(r) == 0" (src/amg.py:182) is evaluated as "every r_i * r_i == 0",
// which is exactly when the fixed-order sum of squares is zero.
#include <cmath>
#include <vector>

#include "device.cuh"
#include "engine.h"
#include "nvtx.h"
#include "ktail.h"

namespace cprb {

__shared__ KTDesc kt;                 // block-uniform plan (copied at entry)
__shared__ double kt_ws[2 * KT_MAXVB * 8];  // per-(virtual block, warp) dot partials
__shared__ double kt_dot_out[2];


// ---- row sums (summation orders of the launched kernels) -------------------

// a0 + pairwise(a[1:len]) for len <= 129, the n < 8 part from `z`
// (-0.0: segsum_masked / rr_row_stream; 0.0: pairwise_leaf).  Entries are
// fetched 8 at a time, all loads of a chunk in flight before the first use.
__device__ __forceinline__ double kt_seg(const cprb_sell& S, int64_t base, int len,
                                         const double* x, double z) {
  if (len <= 0) return 0.0;
  const int n = len - 1;
  const int nf = n >= 8 ? (n & ~7) : 0;
  double a0 = 0.0, s = z, r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = 0.0;
  for (int p0 = 0; p0 < len; p0 += 8) {
    int c[8];
    double v[8], e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (p0 + k < len) {
        c[k] = __ldg(S.cols + base + (int64_t)(p0 + k) * 32);
        v[k] = __ldg(S.vals + base + (int64_t)(p0 + k) * 32);
      }
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = (p0 + k < len) ? v[k] * x[c[k]] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
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

// reduceat row of any length (segsum_rt for len > 129)
__device__ __forceinline__ double kt_row(const cprb_sell& S, int64_t base, int len,
                                         const double* x, double z) {
  if (len <= 129) return kt_seg(S, base, len, x, z);
  auto f = [&](int m) -> double {
    const int64_t e = base + (int64_t)m * 32;
    return __ldg(S.vals + e) * x[__ldg(S.cols + e)];
  };
  return segsum_rt(f, len);
}

// ---- phases (every thread of the CTA calls; each ends with a barrier) ----

// one colour of a PGS-SCM pass (k_sweep): x_i = (b_i - sum a_ij x_j) / d_i,
// sequential from 0.0 in stored order; ZG reads only the earlier colours
template <int NT>
__device__ __noinline__ void kt_colour(int l, int k, int zg, const double* b, double* x) {
  const KTLevel& L = kt.lv[l];
  const int s0 = L.cs[k], s1 = L.cs[k + 1], r0 = L.cr[k], r1 = L.cr[k + 1];
  const bool snap = (L.snap >> k) & 1u;
  double* xo = snap ? L.tmp : x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int s = s0 + warp; s < s1; s += NT / 32) {
    const int row = r0 + (s - s0) * 32 + lane;
    if (row < r1) {
      const int lid = s * 32 + lane;
      const int len = zg ? __ldg(L.sm.lane_len_lo + lid) : __ldg(L.sm.lane_len + lid);
      const int64_t base = __ldg(L.sm.slice_ptr + s) + lane;
      double acc = 0.0;
      for (int m0 = 0; m0 < len; m0 += 8) {
        int c[8];
        double v[8], xv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (m0 + q < len) {
            c[q] = __ldg(L.sm.cols + base + (int64_t)(m0 + q) * 32);
            v[q] = __ldg(L.sm.vals + base + (int64_t)(m0 + q) * 32);
          }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (m0 + q < len) xv[q] = x[c[q]];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (m0 + q < len) acc = acc + v[q] * xv[q];
      }
      xo[row] = (b[row] - acc) / __ldg(L.diag + row);
    }
  }
  __syncthreads();
  if (snap) {
    for (int i = r0 + (int)threadIdx.x; i < r1; i += NT) x[i] = L.tmp[i];
    __syncthreads();
  }
}

// one PGS-SCM pass (pgs_pass): colours in order (dir 0) or reverse (dir 1);
// a single-colour level is classic sequential GS (k_gs_sequential)
template <int NT>
__device__ __noinline__ void kt_pass(int l, const double* b, double* x, int dir, int zg) {
  const KTLevel& L = kt.lv[l];
  if (L.nc == 1) {
    if (zg) {
      for (int i = threadIdx.x; i < L.n; i += NT) x[i] = 0.0;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      for (int t = 0; t < L.n; ++t) {
        const int i = dir ? L.n - 1 - t : t;
        const int w = i >> 5, lane = i & 31;
        const int len = __ldg(L.sm.lane_len + w * 32 + lane);
        const int64_t base = __ldg(L.sm.slice_ptr + w) + lane;
        double acc = 0.0;
        for (int m = 0; m < len; ++m) {
          const int64_t e = base + (int64_t)m * 32;
          acc = acc + __ldg(L.sm.vals + e) * x[__ldg(L.sm.cols + e)];
        }
        x[i] = (b[i] - acc) / __ldg(L.diag + i);
      }
    }
    __syncthreads();
    return;
  }
  for (int t = 0; t < L.nc; ++t) kt_colour<NT>(l, dir ? L.nc - 1 - t : t, zg, b, x);
}

// residual + restriction (k_resid_restrict): bc[I] = (0 + r_a) + r_b with
// r = b - A_l x in the level's original column order; optionally zeroes
// xz[0..nz) (the next frame's Krylov iterate).  Returns "some bc_I^2 != 0".
template <int NT>
__device__ __noinline__ int kt_rr(int l, const double* b, const double* x, double* bc,
                                  double* xz, int nz) {
  const cprb_sell& R = kt.lv[l].rop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int nonzero = 0;
  for (int w = warp; w < R.nslices; w += NT / 32) {
    const int lid = w * 32 + lane;
    const int row = __ldg(R.lane_row + lid);
    const int len = row >= 0 ? __ldg(R.lane_len + lid) : 0;
    const int out = ((lane & 1) == 0) ? __ldg(R.agg_out + w * 16 + (lane >> 1)) : -1;
    double res = 0.0;
    if (row >= 0) res = b[row] - kt_row(R, __ldg(R.slice_ptr + w) + lane, len, x, -0.0);
    const double other = __shfl_down_sync(CPRB_FULL, res, 1);
    if ((lane & 1) == 0 && out >= 0) {
      const double v = (0.0 + res) + other;
      bc[out] = v;
      nonzero |= (v * v != 0.0);
    }
  }
  if (xz)
    for (int i = threadIdx.x; i < nz; i += NT) xz[i] = 0.0;
  return __syncthreads_or(nonzero);
}

// y = A_l x (k_bsr<1,0>): slices of width <= 8 sum with segsum_masked
// (-0.0 identity), wider slices with segsum_rt
template <int NT>
__device__ __noinline__ void kt_spmv(int l, const double* x, double* y) {
  const cprb_sell& A = kt.lv[l].A;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int s = warp; s < A.nslices; s += NT / 32) {
    const int lid = s * 32 + lane;
    const int64_t base = __ldg(A.slice_ptr + s);
    const int width = (int)((__ldg(A.slice_ptr + s + 1) - base) >> 5);
    const int row = __ldg(A.lane_row + lid);
    const int len = row >= 0 ? __ldg(A.lane_len + lid) : 0;
    double v = 0.0;
    if (width > 0) v = kt_row(A, base + lane, len, x, width <= 8 ? -0.0 : 0.0);
    if (row >= 0) y[row] = v;
  }
  __syncthreads();
}

__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(CPRB_FULL, v, o);
  return v;
}

__device__ __forceinline__ int kt_red_blocks(int n) {
  int g = (n + 1023) / 1024;
  if (g < 1) g = 1;
  if (g > CPRB_RED_BLOCKS) g = CPRB_RED_BLOCKS;
  return g;
}

// cprb_dot's arithmetic for one or two products at once: virtual CTA vb of
// 256 threads sums x[i] * y[i] over its chunk (stride 256), xor tree per
// warp, warps in order -> partial[vb]; the partials in order through the
// same tree.  Results in kt_dot_out[0..1], read by every thread right after
// the call (the next write is at least one barrier later).
template <int NT>
__device__ __noinline__ void kt_dots(int n, int nd, const double* x0, const double* y0,
                                     const double* x1, const double* y1) {
  const int g = kt_red_blocks(n);
  const int chunk = (n + g - 1) / g;
  const int vt = threadIdx.x & 255, lane = threadIdx.x & 31;
  for (int vb = threadIdx.x >> 8; vb < g; vb += NT / 256) {
    const int lo = vb * chunk;
    const int hi = lo + chunk < n ? lo + chunk : n;
    double a0 = 0.0, a1 = 0.0;
    for (int i = lo + vt; i < hi; i += 256) {
      a0 = a0 + x0[i] * y0[i];
      if (nd > 1) a1 = a1 + x1[i] * y1[i];
    }
    a0 = warp_tree(a0);
    if (nd > 1) a1 = warp_tree(a1);
    if (lane == 0) {
      kt_ws[vb * 8 + (vt >> 5)] = a0;
      if (nd > 1) kt_ws[KT_MAXVB * 8 + vb * 8 + (vt >> 5)] = a1;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    for (int d = 0; d < nd; ++d) {
      const double* ws = kt_ws + d * KT_MAXVB * 8;
      // final CTA, virtual thread t = lane + 32 vw: v = 0 + sum_k partial[t + 256 k]
      double s = 0.0;
      for (int vw = 0; vw < 8; ++vw) {
        double v = 0.0;
        for (int t = lane + 32 * vw; t < g; t += 256) {
          double p = 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k) p = p + ws[t * 8 + k];
          v = v + p;
        }
        if (32 * vw < g) v = warp_tree(v);  // a virtual warp without partials sums to +0.0
        s = s + v;
      }
      if (lane == 0) kt_dot_out[d] = s;
    }
  }
  __syncthreads();
}

// coarsest level: x = inv(A_L) b (k_kdense: warp per row, lane-strided, xor tree)
template <int NT>
__device__ __noinline__ void kt_dense(const double* b, double* x) {
  const int n = kt.n_coarse;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int w = warp; w < n; w += NT / 32) {
    const double* row = kt.coarse_inv + (int64_t)w * n;
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s = s + __ldg(row + c) * b[c];
    s = warp_tree(s);
    if (lane == 0) x[w] = s;
  }
  __syncthreads();
}

template <int NT>
__device__ __noinline__ void kt_prolong(int l, const double* xc, double* x) {
  const KTLevel& L = kt.lv[l];
  for (int i = threadIdx.x; i < L.n; i += NT) x[i] = x[i] + xc[__ldg(L.aggp + i)];
  __syncthreads();
}

// out = a x + y (and "some out_i^2 != 0" when asked)
template <int NT>
__device__ __noinline__ int kt_axpy(int n, double a, const double* x, const double* y, double* out,
                                    int want_nz) {
  int nz = 0;
  for (int i = threadIdx.x; i < n; i += NT) {
    const double v = a * x[i] + y[i];
    out[i] = v;
    nz |= (v * v != 0.0);
  }
  if (want_nz) return __syncthreads_or(nz);
  __syncthreads();
  return 0;
}

// x = a0 x0 + y, r = a1 x1 + r (the two FCG updates), returns "some r_i^2 != 0"
template <int NT>
__device__ __noinline__ int kt_axpy2(int n, double a0, const double* x0, double* y0, double a1,
                                     const double* x1, double* y1) {
  int nz = 0;
  for (int i = threadIdx.x; i < n; i += NT) {
    y0[i] = a0 * x0[i] + y0[i];
    const double v = a1 * x1[i] + y1[i];
    y1[i] = v;
    nz |= (v * v != 0.0);
  }
  return __syncthreads_or(nz);
}

template <int NT>
__device__ __noinline__ void kt_div(int n, const double* x, double h, double* out) {
  for (int i = threadIdx.x; i < n; i += NT) out[i] = x[i] / h;
  __syncthreads();
}

// ---- the recursion ---------------------------------------------------------

template <int NT, int D>
__device__ void kt_krylov(int l, int nz);

// src/amg.py:245-267 (K): x = cycle_l(b) from a zero guess
template <int NT, int D>
__device__ __noinline__ void kt_visit(int l, const double* b, double* x) {
  if (l == kt.L - 1) {
    kt_dense<NT>(b, x);
    return;
  }
  const KTLevel& Lv = kt.lv[l];
  if (kt.pre == 0) {
    for (int i = threadIdx.x; i < Lv.n; i += NT) x[i] = 0.0;
    __syncthreads();
  }
  for (int sw = 0; sw < kt.pre; ++sw) kt_pass<NT>(l, b, x, 0, sw == 0 ? 1 : 0);
  const double* ec;
  if (l + 1 == kt.L - 1) {
    kt_rr<NT>(l, b, x, Lv.rc, nullptr, 0);
    kt_dense<NT>(Lv.rc, kt.coarse_x);
    ec = kt.coarse_x;
  } else {
    const KTLevel& Ln = kt.lv[l + 1];
    // FCG: the restriction is the frame's r (x = 0); FGMRES keeps rhs in rc
    const int nz = kt.use_fcg ? kt_rr<NT>(l, b, x, Ln.r, Ln.x, Ln.n)
                              : kt_rr<NT>(l, b, x, Lv.rc, nullptr, 0);
    kt_krylov<NT, D + 1>(l + 1, nz);
    ec = Ln.x;
  }
  kt_prolong<NT>(l, ec, x);
  for (int sw = 0; sw < kt.post; ++sw) kt_pass<NT>(l, b, x, 1, 0);
}

// two flexible-CG steps at level l (src/amg.py:177-196; csrc/kcycle.cu fcg_at):
// on entry r = rhs, x = 0 and nz = "norm2(r) != 0"; result in x
template <int NT, int D>
__device__ __noinline__ void kt_fcg(int l, int nz) {
  const KTLevel& L = kt.lv[l];
  const int n = L.n;
  if (!nz) return;
  // step 1 (no stored direction: p = z)
  kt_visit<NT, D>(l, L.r, L.z1);
  kt_spmv<NT>(l, L.z1, L.ap1);
  kt_dots<NT>(n, 2, L.z1, L.ap1, L.z1, L.r);
  const double pap1 = kt_dot_out[0], pr1 = kt_dot_out[1];
  if (pap1 <= 0.0 || !isfinite(pap1)) return;
  const double a1 = pr1 / pap1;
  nz = kt_axpy2<NT>(n, 1.0 * a1, L.z1, L.x, -1.0 * a1, L.ap1, L.r);
  if (!nz) return;
  // step 2 (one stored direction): p = z - (z, Ap1) / pap1 p1
  kt_visit<NT, D>(l, L.r, L.z2);
  kt_dots<NT>(n, 1, L.z2, L.ap1, nullptr, nullptr);
  const double coef = -(kt_dot_out[0] / pap1);
  kt_axpy<NT>(n, coef, L.z1, L.z2, L.p2, 0);
  kt_spmv<NT>(l, L.p2, L.ap2);
  kt_dots<NT>(n, 2, L.p2, L.ap2, L.p2, L.r);
  const double pap2 = kt_dot_out[0], pr2 = kt_dot_out[1];
  if (pap2 <= 0.0 || !isfinite(pap2)) return;
  kt_axpy<NT>(n, 1.0 * (pr2 / pap2), L.p2, L.x, L.x, 0);
}

// two flexible-GMRES steps at level l (src/amg.py:199-225; kcycle.cu
// fgmres_at): rhs in kt.lv[l-1].rc; result in x
template <int NT, int D>
__device__ __noinline__ void kt_fgmres(int l) {
  const KTLevel& L = kt.lv[l];
  const int n = L.n;
  const double* rhs = kt.lv[l - 1].rc;
  double *x = L.x, *v0 = L.r, *z0 = L.z1, *w = L.ap1, *z1 = L.z2, *v1 = L.p2, *w1 = L.ap2;
  for (int i = threadIdx.x; i < n; i += NT) x[i] = 0.0;
  kt_dots<NT>(n, 1, rhs, rhs, nullptr, nullptr);
  const double beta = sqrt(kt_dot_out[0]);
  if (!(beta != 0.0)) return;  // x = 0
  kt_div<NT>(n, rhs, beta, v0);
  kt_visit<NT, D>(l, v0, z0);
  kt_spmv<NT>(l, z0, w);
  kt_dots<NT>(n, 1, w, v0, nullptr, nullptr);
  const double h00 = kt_dot_out[0];
  kt_axpy<NT>(n, -1.0 * h00, v0, w, w, 0);
  kt_dots<NT>(n, 1, w, w, nullptr, nullptr);
  const double h10 = sqrt(kt_dot_out[0]);
  const bool cont = h10 != 0.0;
  double h01 = 0.0, h11 = 0.0, h21 = 0.0;
  if (cont) {
    kt_div<NT>(n, w, h10, v1);
    kt_visit<NT, D>(l, v1, z1);
    kt_spmv<NT>(l, z1, w1);
    kt_dots<NT>(n, 1, w1, v0, nullptr, nullptr);
    h01 = kt_dot_out[0];
    kt_axpy<NT>(n, -1.0 * h01, v0, w1, w1, 0);
    kt_dots<NT>(n, 1, w1, v1, nullptr, nullptr);
    h11 = kt_dot_out[0];
    kt_axpy<NT>(n, -1.0 * h11, v1, w1, w1, 0);
    kt_dots<NT>(n, 1, w1, w1, nullptr, nullptr);
    h21 = sqrt(kt_dot_out[0]);
  }
  // least squares (k_fg_lstsq: Givens QR of the (m+1) x m Hessenberg matrix)
  double y0 = 0.0, y1 = 0.0;
  {
    const int m = cont ? 2 : 1;
    double r00 = h00, r10 = h10, r01 = h01, r11 = h11, r21 = h21;
    double g0 = beta, g1 = 0.0;
    double d = hypot(r00, r10);
    if (d != 0.0) {
      double c = r00 / d, sn = r10 / d;
      r00 = d;
      const double t01 = c * r01 + sn * r11;
      r11 = -sn * r01 + c * r11;
      r01 = t01;
      g1 = -sn * g0;
      g0 = c * g0;
      if (m == 1) {
        y0 = g0 / r00;
      } else {
        d = hypot(r11, r21);
        if (d == 0.0) {
          y0 = g0 / r00;
        } else {
          c = r11 / d;
          r11 = d;
          g1 = c * g1;
          y1 = g1 / r11;
          y0 = (g0 - r01 * y1) / r00;
        }
      }
    }
  }
  kt_axpy<NT>(n, 1.0 * y0, z0, x, x, 0);
  if (cont) kt_axpy<NT>(n, 1.0 * y1, z1, x, x, 0);
}

template <int NT, int D>
__device__ void kt_krylov(int l, int nz) {
  if constexpr (D >= KT_MAXD) {
    __trap();
  } else {
    if (kt.use_fcg) kt_fcg<NT, D>(l, nz);
    else kt_fgmres<NT, D>(l);
  }
}

// the Krylov-wrapped recursion from level l (>= start): rhs (level-permuted
// order) -> kt.lv[l].x
template <int NT>
__global__ void __launch_bounds__(NT, 1) k_ktail(const KTDesc* __restrict__ desc, int l,
                                                  const double* __restrict__ rhs) {
  {
    const int* src = reinterpret_cast<const int*>(desc);
    int* dst = reinterpret_cast<int*>(&kt);
    for (int i = threadIdx.x; i < (int)(sizeof(KTDesc) / sizeof(int)); i += NT) dst[i] = src[i];
  }
  __syncthreads();
  const KTLevel& L = kt.lv[l];
  int nz = 0;
  if (kt.use_fcg) {
    for (int i = threadIdx.x; i < L.n; i += NT) {
      const double v = rhs[i];
      L.r[i] = v;
      L.x[i] = 0.0;
      nz |= (v * v != 0.0);
    }
  } else {
    double* rc = kt.lv[l - 1].rc;
    if (rc != rhs)
      for (int i = threadIdx.x; i < L.n; i += NT) rc[i] = rhs[i];
  }
  nz = __syncthreads_or(nz);
  kt_krylov<NT, 0>(l, nz);
}

int ktail_launch(const KTDesc* dev_desc, int threads, int l, const double* rhs, cudaStream_t st) {
  NvtxRange nv("amg_kcycle_tail");
  if (threads == 512) k_ktail<512><<<1, 512, 0, st>>>(dev_desc, l, rhs);
  else k_ktail<1024><<<1, 1024, 0, st>>>(dev_desc, l, rhs);
  return check_launch("k-cycle tail");
}

}  // namespace cprb
