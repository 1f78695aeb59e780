// K-cycle (nonlinear AMLI, src/amg.py:245-267) driven from C++ with every
// Krylov scalar on the device: the coarse recursion of each level is wrapped
// in two flexible-CG steps (src/amg.py:177-196) whose early exits
// ("norm2(r) == 0", "pap <= 0 or non-finite") become a device flag that
// predicates the updates, so an application needs no host synchronisation
// and can be captured whole into a CUDA graph.  The arithmetic is the host
// K-cycle's (amg.py DeviceAmg._fcg): the same deterministic dot products
// (cprb_dot), IEEE scalar divisions and separately rounded axpys, so the
// device and host K-cycles agree bitwise.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "device.cuh"
#include "engine.h"
#include "ktail.h"
#include "nvtx.h"

namespace cprb {

// scalar slots of one FCG frame
enum { S_ACTIVE = 0, S_RR = 1, S_ZAP = 2, S_PAP1 = 3, S_PAP2 = 4, S_PR = 5, S_ALPHA = 6, S_NS = 8 };

__global__ void k_fcg_init(double* s) { s[S_ACTIVE] = 1.0; }

// if norm2(r) == 0: break
__global__ void k_fcg_check_rr(double* s) {
  if (!(sqrt(s[S_RR]) != 0.0)) s[S_ACTIVE] = 0.0;
}

// pap = s[ip]; if pap <= 0 or non-finite: break; alpha = (p, r) / pap
__global__ void k_fcg_alpha(double* s, int ip) {
  const double pap = s[ip];
  if (s[S_ACTIVE] == 0.0) return;
  if (pap <= 0.0 || !isfinite(pap)) {
    s[S_ACTIVE] = 0.0;
    return;
  }
  s[S_ALPHA] = s[S_PR] / pap;
}

// out = (sign * alpha) * x + y  while the frame is active
__global__ void k_axpy_alpha(int n, const double* __restrict__ s, double sign,
                             const double* __restrict__ x, const double* y, double* out) {
  if (s[S_ACTIVE] == 0.0) return;
  const double a = sign * s[S_ALPHA];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a * x[i] + y[i];
}

// start of an FCG frame: active = 1, r = rhs, x = 0 (one launch instead of
// a flag kernel, a memset and a copy)
__global__ void k_fcg_start(int n, double* s, const double* __restrict__ rhs,
                            double* __restrict__ r, double* __restrict__ x) {
  if (blockIdx.x == 0 && threadIdx.x == 0) s[S_ACTIVE] = 1.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    r[i] = rhs[i];
    x[i] = 0.0;
  }
}

// k_fcg_alpha + k_axpy_alpha(+1: x += alpha p) [+ k_axpy_alpha(-1: r -= alpha ap)]
// in one launch: every thread evaluates the same predicate and quotient
// (bitwise those of k_fcg_alpha); block 0 thread 0 records them in s
__global__ void k_fcg_update(int n, double* s, int ip, const double* __restrict__ p,
                             double* x, const double* __restrict__ ap, double* r) {
  if (s[S_ACTIVE] == 0.0) return;
  const double pap = s[ip];
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  if (pap <= 0.0 || !isfinite(pap)) {
    if (lead) s[S_ACTIVE] = 0.0;
    return;
  }
  const double alpha = s[S_PR] / pap;
  if (lead) s[S_ALPHA] = alpha;
  const double na = -1.0 * alpha;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    x[i] = (1.0 * alpha) * p[i] + x[i];
    if (ap) r[i] = na * ap[i] + r[i];
  }
}

// p = p - (dot(z, ap_j) / pap_j) p_j  ==  (-coef) * p_j + z
__global__ void k_axpy_coef(int n, const double* __restrict__ s, const double* __restrict__ pj,
                            const double* __restrict__ z, double* __restrict__ out) {
  if (s[S_ACTIVE] == 0.0) return;
  const double a = -(s[S_ZAP] / s[S_PAP1]);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a * pj[i] + z[i];
}

__global__ void k_kgather(int n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                          int stride, double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[(int64_t)stride * idx[i]];
}

__global__ void k_kscatter(int n, const int32_t* __restrict__ idx, const double* __restrict__ src,
                           double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
}

__global__ void k_kprolong(int n, const int32_t* __restrict__ aggp, const double* __restrict__ xc,
                           double* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] + xc[aggp[i]];
}

__global__ void k_kdense(int n, const double* __restrict__ inv, const double* __restrict__ b,
                         double* __restrict__ x) {
  const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const double* row = inv + (int64_t)w * n;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s = s + row[c] * b[c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = s + __shfl_xor_sync(CPRB_FULL, s, o);
  if (lane == 0) x[w] = s;
}

// grid for the grid-stride kernels (axpys)
// ---- flexible GMRES flavour (src/amg.py:199-225), two steps ----------------
enum { G_ACTIVE = 0, G_BETA = 1, G_H00 = 2, G_H10 = 3, G_H01 = 4, G_H11 = 5, G_H21 = 6,
       G_CONT = 7, G_Y0 = 8, G_Y1 = 9, G_MEFF = 10, G_T = 11, G_NS = 16 };

// beta = sqrt(s[G_T]); active = beta != 0
__global__ void k_fg_beta(double* s) {
  s[G_BETA] = sqrt(s[G_T]);
  s[G_ACTIVE] = (s[G_BETA] != 0.0) ? 1.0 : 0.0;
}

// s[dst] = sqrt(s[G_T]); the next Arnoldi step runs iff it is nonzero
__global__ void k_fg_norm(double* s, int dst) {
  s[dst] = sqrt(s[G_T]);
  s[G_CONT] = (s[G_ACTIVE] != 0.0 && s[dst] != 0.0) ? 1.0 : 0.0;
}

// out = x / s[idx]  while s[flag] != 0
__global__ void k_div_pred(int n, const double* __restrict__ s, int idx, int flag,
                           const double* __restrict__ x, double* __restrict__ out) {
  if (s[flag] == 0.0) return;
  const double h = s[idx];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = x[i] / h;
}

// out = (sign * s[idx]) * x + y  while s[flag] != 0
__global__ void k_axpy_s(int n, const double* __restrict__ s, int idx, int flag, double sign,
                         const double* __restrict__ x, const double* y, double* out) {
  if (s[flag] == 0.0) return;
  const double a = sign * s[idx];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a * x[i] + y[i];
}

__global__ void k_fg_restore(double* s) {
  s[G_CONT] = (s[G_ACTIVE] != 0.0 && s[G_H10] != 0.0) ? 1.0 : 0.0;
}

// least squares min || H y - beta e1 || for m_eff = 1 or 2 (Givens QR of the
// (m_eff+1) x m_eff Hessenberg matrix; np.linalg.lstsq in the reference,
// equal up to rounding for full column rank)
__global__ void k_fg_lstsq(double* s) {
  s[G_Y0] = 0.0;
  s[G_Y1] = 0.0;
  if (s[G_ACTIVE] == 0.0) {
    s[G_MEFF] = 0.0;
    return;
  }
  const int m = s[G_CONT] != 0.0 ? 2 : 1;
  s[G_MEFF] = m;
  double r00 = s[G_H00], r10 = s[G_H10], r01 = s[G_H01], r11 = s[G_H11], r21 = s[G_H21];
  double g0 = s[G_BETA], g1 = 0.0, g2 = 0.0;
  double d = hypot(r00, r10);
  if (d == 0.0) return;
  double c = r00 / d, sn = r10 / d;
  r00 = d;
  const double t01 = c * r01 + sn * r11;
  r11 = -sn * r01 + c * r11;
  r01 = t01;
  g1 = -sn * g0;
  g0 = c * g0;
  if (m == 1) {
    s[G_Y0] = g0 / r00;
    return;
  }
  d = hypot(r11, r21);
  if (d == 0.0) {
    s[G_Y0] = g0 / r00;
    return;
  }
  c = r11 / d;
  sn = r21 / d;
  r11 = d;
  g2 = -sn * g1;
  g1 = c * g1;
  (void)g2;
  const double y1 = g1 / r11;
  s[G_Y1] = y1;
  s[G_Y0] = (g0 - r01 * y1) / r00;
}

static inline int kb(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}
// grid covering n threads (one element per thread: gather, scatter,
// prolongation, dense rows)
static inline int kfull(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 1 ? 1 : g);
}

struct KPlan {
  int nl = 0;
  std::vector<cprb_sell> spmv;  // level matrices (permuted rows, original column order)
  std::vector<int> n;
  std::vector<double*> x, r, z1, ap1, z2, p2, ap2, s, rc, b0, x0;
  double* coarse_x = nullptr;
  double* partials = nullptr;
  int32_t* ticket = nullptr;
  std::vector<void*> allocs;
  int pre = 1, post = 1;
  // persistent tail (csrc/ktail.cu): Krylov frames at levels >= kt_start run
  // in one CTA; kt_start >= nl - 1 disables it
  KTDesc* kt_dev = nullptr;
  int kt_start = 1 << 30;
  int kt_threads = 1024;

  double* alloc(size_t n_) {
    void* p = nullptr;
    if (cudaMalloc(&p, sizeof(double) * (n_ > 0 ? n_ : 1)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, sizeof(double) * (n_ > 0 ? n_ : 1));
    allocs.push_back(p);
    return (double*)p;
  }
  ~KPlan() {
    for (void* p : allocs) cudaFree(p);
  }
};

static int kdot(const KPlan& P, int n, const double* x, const double* y, double* out,
                cudaStream_t st) {
  return cprb_dot(n, x, y, out, P.partials, P.ticket, st);
}

static int kcycle_at(const KPlan& P, const cprb_amg& h, int l, const double* b, double* x,
                     cudaStream_t st);
static int fgmres_at(const KPlan& P, const cprb_amg& h, int l, const double* rhs,
                     cudaStream_t st);

// two flexible-CG steps at level l with the cycle at l as preconditioner;
// the result is P.x[l]
static int fcg_at(const KPlan& P, const cprb_amg& h, int l, const double* rhs, cudaStream_t st) {
  const int n = P.n[l];
  double* s = P.s[l];
  double *x = P.x[l], *r = P.r[l], *z1 = P.z1[l], *ap1 = P.ap1[l], *z2 = P.z2[l];
  double *p2 = P.p2[l], *ap2 = P.ap2[l];
  k_fcg_start<<<kb(n), 256, 0, st>>>(n, s, rhs, r, x);
  int rc;
  // step 1 (no stored directions: p = z)
  if ((rc = kdot(P, n, r, r, s + S_RR, st))) return rc;
  k_fcg_check_rr<<<1, 1, 0, st>>>(s);
  if ((rc = kcycle_at(P, h, l, r, z1, st))) return rc;
  if ((rc = bsr_op(0, P.spmv[l], 1, z1, nullptr, ap1, nullptr, nullptr, st))) return rc;
  if ((rc = kdot(P, n, z1, ap1, s + S_PAP1, st))) return rc;
  if ((rc = kdot(P, n, z1, r, s + S_PR, st))) return rc;
  k_fcg_update<<<kb(n), 256, 0, st>>>(n, s, S_PAP1, z1, x, ap1, r);
  // step 2 (one stored direction)
  if ((rc = kdot(P, n, r, r, s + S_RR, st))) return rc;
  k_fcg_check_rr<<<1, 1, 0, st>>>(s);
  if ((rc = kcycle_at(P, h, l, r, z2, st))) return rc;
  if ((rc = kdot(P, n, z2, ap1, s + S_ZAP, st))) return rc;
  k_axpy_coef<<<kb(n), 256, 0, st>>>(n, s, z1, z2, p2);
  if ((rc = bsr_op(0, P.spmv[l], 1, p2, nullptr, ap2, nullptr, nullptr, st))) return rc;
  if ((rc = kdot(P, n, p2, ap2, s + S_PAP2, st))) return rc;
  if ((rc = kdot(P, n, p2, r, s + S_PR, st))) return rc;
  k_fcg_update<<<kb(n), 256, 0, st>>>(n, s, S_PAP2, p2, x, (const double*)nullptr,
                                      (double*)nullptr);
  return check_launch("fcg");
}

// two flexible-GMRES steps at level l (src/amg.py:199-225); result P.x[l]
static int fgmres_at(const KPlan& P, const cprb_amg& h, int l, const double* rhs,
                     cudaStream_t st) {
  const int n = P.n[l];
  double* s = P.s[l];
  double *x = P.x[l], *v0 = P.r[l], *z0 = P.z1[l], *w = P.ap1[l], *z1 = P.z2[l];
  double *v1 = P.p2[l], *w1 = P.ap2[l];
  int rc;
  cudaMemsetAsync(x, 0, sizeof(double) * n, st);
  if ((rc = kdot(P, n, rhs, rhs, s + G_T, st))) return rc;
  k_fg_beta<<<1, 1, 0, st>>>(s);
  k_div_pred<<<kb(n), 256, 0, st>>>(n, s, G_BETA, G_ACTIVE, rhs, v0);
  // j = 0
  if ((rc = kcycle_at(P, h, l, v0, z0, st))) return rc;
  if ((rc = bsr_op(0, P.spmv[l], 1, z0, nullptr, w, nullptr, nullptr, st))) return rc;
  if ((rc = kdot(P, n, w, v0, s + G_H00, st))) return rc;
  k_axpy_s<<<kb(n), 256, 0, st>>>(n, s, G_H00, G_ACTIVE, -1.0, v0, w, w);
  if ((rc = kdot(P, n, w, w, s + G_T, st))) return rc;
  k_fg_norm<<<1, 1, 0, st>>>(s, G_H10);
  k_div_pred<<<kb(n), 256, 0, st>>>(n, s, G_H10, G_CONT, w, v1);
  // j = 1 (skipped by predicate after a happy breakdown)
  if ((rc = kcycle_at(P, h, l, v1, z1, st))) return rc;
  if ((rc = bsr_op(0, P.spmv[l], 1, z1, nullptr, w1, nullptr, nullptr, st))) return rc;
  if ((rc = kdot(P, n, w1, v0, s + G_H01, st))) return rc;
  k_axpy_s<<<kb(n), 256, 0, st>>>(n, s, G_H01, G_CONT, -1.0, v0, w1, w1);
  if ((rc = kdot(P, n, w1, v1, s + G_H11, st))) return rc;
  k_axpy_s<<<kb(n), 256, 0, st>>>(n, s, G_H11, G_CONT, -1.0, v1, w1, w1);
  if ((rc = kdot(P, n, w1, w1, s + G_T, st))) return rc;
  k_fg_norm<<<1, 1, 0, st>>>(s, G_H21);
  // k_fg_norm cleared G_CONT when H21 == 0; m_eff is 2 either way
  // (src/amg.py:216-218), so restore it from H10 before the solve
  k_fg_restore<<<1, 1, 0, st>>>(s);
  k_fg_lstsq<<<1, 1, 0, st>>>(s);
  k_axpy_s<<<kb(n), 256, 0, st>>>(n, s, G_Y0, G_ACTIVE, 1.0, z0, x, x);
  k_axpy_s<<<kb(n), 256, 0, st>>>(n, s, G_Y1, G_CONT, 1.0, z1, x, x);
  return check_launch("fgmres");
}

// src/amg.py:245-267 (K): x = cycle_l(b) from a zero guess
static int kcycle_at(const KPlan& P, const cprb_amg& h, int l, const double* b, double* x,
                     cudaStream_t st) {
  const int L = h.nlevels;
  if (l == L - 1) {
    k_kdense<<<kfull((int64_t)h.n_coarse * 32), 256, 0, st>>>(h.n_coarse, h.coarse_inv, b, x);
    return check_launch("k coarse");
  }
  const cprb_amg_level& Lv = h.levels[l];
  int rc;
  // zero guess (src/amg.py:250): with no pre-sweep nothing overwrites x, and
  // x is a persistent plan buffer that still holds the previous visit
  if (P.pre == 0 && cudaMemsetAsync(x, 0, sizeof(double) * (size_t)Lv.n, st) != cudaSuccess)
    return check_launch("k zero guess");
  for (int sw = 0; sw < P.pre; ++sw)
    if ((rc = pgs_pass(Lv, b, x, 0, sw == 0 ? 1 : 0, nullptr, 0, nullptr, nullptr, st))) return rc;
  double* bc = P.rc[l];
  if ((rc = cprb_resid_restrict(&Lv, b, x, bc, st))) return rc;
  const double* ec;
  if (l + 1 == L - 1) {
    k_kdense<<<kfull((int64_t)h.n_coarse * 32), 256, 0, st>>>(h.n_coarse, h.coarse_inv, bc,
                                                           P.coarse_x);
    ec = P.coarse_x;
  } else {
    if (l + 1 >= P.kt_start) rc = ktail_launch(P.kt_dev, P.kt_threads, l + 1, bc, st);
    else rc = h.use_fcg ? fcg_at(P, h, l + 1, bc, st) : fgmres_at(P, h, l + 1, bc, st);
    if (rc) return rc;
    ec = P.x[l + 1];
  }
  k_kprolong<<<kfull(Lv.n), 256, 0, st>>>(Lv.n, Lv.aggp, ec, x);
  for (int sw = 0; sw < P.post; ++sw)
    if ((rc = pgs_pass(Lv, b, x, 1, 0, nullptr, 0, nullptr, nullptr, st))) return rc;
  return check_launch("k cycle");
}

int kcycle_apply(const cprb_amg& h, const double* r, double* z, cudaStream_t st) {
  NvtxRange nv("amg_kcycle");
  const KPlan* P = static_cast<const KPlan*>((void*)h.kwork);
  if (!P) return set_error(CPRB_EINVAL, "K-cycle plan missing (cprb_kcycle_create)");
  if (h.nlevels <= 1) {
    k_kgather<<<kfull(h.n_coarse), 256, 0, st>>>(h.n_coarse, h.perm0, r, h.in_stride, P->b0[0]);
    k_kdense<<<kfull((int64_t)h.n_coarse * 32), 256, 0, st>>>(h.n_coarse, h.coarse_inv, P->b0[0], z);
    return check_launch("k coarse only");
  }
  const int n0 = P->n[0];
  k_kgather<<<kfull(n0), 256, 0, st>>>(n0, h.perm0, r, h.in_stride, P->b0[0]);
  int rc = kcycle_at(*P, h, 0, P->b0[0], P->x0[0], st);
  if (rc) return rc;
  k_kscatter<<<kfull(n0), 256, 0, st>>>(n0, h.perm0, P->x0[0], z);
  return check_launch("k cycle apply");
}

// Persistent tail plan: the first level l >= 1 with at most CPRB_KTAIL_ROWS
// rows (default 0 = off) such that every level from l on fits the
// tail's limits.  CPRB_KTAIL_THREADS = 512 | 1024 (default) sizes the CTA.
static int ktail_plan(KPlan& P, const cprb_amg& h) {
  const int L = h.nlevels;
  long thr = 0;
  if (const char* e = getenv("CPRB_KTAIL_ROWS")) thr = atol(e);
  if (const char* e = getenv("CPRB_KTAIL_THREADS")) P.kt_threads = atoi(e) == 512 ? 512 : 1024;
  if (thr <= 0 || L < 3 || L - 1 > KT_MAXL) return CPRB_OK;
  int start = -1;
  for (int l = L - 2; l >= 1; --l) {
    const cprb_amg_level& Lv = h.levels[l];
    if (Lv.n > thr || Lv.n > KT_MAXVB * 1024 || Lv.ncolors > KT_MAXC || Lv.ncolors < 1) break;
    start = l;
  }
  if (start < 1 || L - 1 - start > KT_MAXD) return CPRB_OK;
  KTDesc d;
  memset(&d, 0, sizeof(d));
  d.L = L;
  d.start = start;
  d.pre = P.pre;
  d.post = P.post;
  d.use_fcg = h.use_fcg;
  d.n_coarse = h.n_coarse;
  d.coarse_inv = h.coarse_inv;
  d.coarse_x = P.coarse_x;
  for (int l = start - 1; l < L - 1; ++l) {
    const cprb_amg_level& Lv = h.levels[l];
    KTLevel& t = d.lv[l];
    t.sm = Lv.smoother;
    t.rop = Lv.restrict_op;
    if (l >= 1) t.A = P.spmv[l];
    t.diag = Lv.diag;
    t.aggp = Lv.aggp;
    t.x = P.x[l]; t.r = P.r[l]; t.z1 = P.z1[l]; t.ap1 = P.ap1[l];
    t.z2 = P.z2[l]; t.p2 = P.p2[l]; t.ap2 = P.ap2[l];
    t.tmp = Lv.tmp;
    t.rc = P.rc[l];
    t.n = Lv.n;
    t.nc = Lv.ncolors;
    t.snap = 0;
    if (l >= start) {
      for (int k = 0; k <= Lv.ncolors; ++k) {
        t.cr[k] = Lv.color_rows[k];
        t.cs[k] = Lv.color_slices[k];
      }
      for (int k = 0; k < Lv.ncolors; ++k)
        if (Lv.color_snapshot && Lv.color_snapshot[k]) t.snap |= 1u << k;
    }
  }
  void* dd = nullptr;
  if (cudaMalloc(&dd, sizeof(KTDesc)) != cudaSuccess)
    return set_error(CPRB_EDEVICE, "K-cycle tail plan allocation");
  P.allocs.push_back(dd);
  if (cudaMemcpy(dd, &d, sizeof(KTDesc), cudaMemcpyHostToDevice) != cudaSuccess)
    return set_error(CPRB_EDEVICE, "K-cycle tail plan upload");
  P.kt_dev = (KTDesc*)dd;
  P.kt_start = start;
  return CPRB_OK;
}

}  // namespace cprb

using namespace cprb;

extern "C" {

int cprb_kcycle_create(const cprb_amg* h, const cprb_sell* level_spmv, int32_t pre_sweeps,
                       int32_t post_sweeps, void** out) {
  if (!h || !out) return set_error(CPRB_EINVAL, "null argument");
  auto* P = new KPlan();
  const int L = h->nlevels;
  P->nl = L;
  P->pre = pre_sweeps;
  P->post = post_sweeps;
  P->n.resize(L);
  for (int l = 0; l < L - 1; ++l) P->n[l] = h->levels[l].n;
  P->n[L - 1] = h->n_coarse;
  P->spmv.assign(level_spmv, level_spmv + (L > 1 ? L - 1 : 0));
  auto vec = [&](std::vector<double*>& v) { v.assign(L, nullptr); };
  vec(P->x); vec(P->r); vec(P->z1); vec(P->ap1); vec(P->z2); vec(P->p2); vec(P->ap2);
  vec(P->s); vec(P->rc); vec(P->b0); vec(P->x0);
  for (int l = 0; l < L; ++l) {
    const size_t n = (size_t)P->n[l];
    if (l >= 1 && l < L - 1) {
      P->x[l] = P->alloc(n); P->r[l] = P->alloc(n); P->z1[l] = P->alloc(n);
      P->ap1[l] = P->alloc(n); P->z2[l] = P->alloc(n); P->p2[l] = P->alloc(n);
      P->ap2[l] = P->alloc(n); P->s[l] = P->alloc(G_NS);
    }
    if (l < L - 1) P->rc[l] = P->alloc((size_t)P->n[l + 1]);
  }
  P->b0[0] = P->alloc((size_t)P->n[0]);
  P->x0[0] = P->alloc((size_t)P->n[0]);
  P->coarse_x = P->alloc((size_t)h->n_coarse);
  P->partials = P->alloc(CPRB_RED_BLOCKS);
  {
    void* t = nullptr;
    if (cudaMalloc(&t, 64) != cudaSuccess) {
      delete P;
      return set_error(CPRB_EDEVICE, "K-cycle ticket allocation");
    }
    cudaMemset(t, 0, 64);
    P->allocs.push_back(t);
    P->ticket = (int32_t*)t;
  }
  for (void* p : P->allocs)
    if (!p) {
      delete P;
      return set_error(CPRB_EDEVICE, "K-cycle workspace allocation");
    }
  if (int rc = ktail_plan(*P, *h)) {
    delete P;
    return rc;
  }
  cudaDeviceSynchronize();
  *out = P;
  return check_launch("kcycle create");
}

// K-cycle coarse correction from level l (src/amg.py:256-263): two Krylov
// steps at level l preconditioned by the cycle at l, or the coarse solve when
// l is the coarsest level.  rhs / out are in the level's natural order
// (perm: level-permuted row -> natural index).  Used by the slab-partitioned
// solve, whose level 0 is distributed while levels >= 1 live on rank 0.
int cprb_kcycle_correction(const cprb_amg* h, int32_t l, const int32_t* perm, const double* rhs,
                           double* out, void* stream) {
  const KPlan* P = static_cast<const KPlan*>(h->kwork);
  if (!P) return set_error(CPRB_EINVAL, "K-cycle plan missing (cprb_kcycle_create)");
  if (l < 1 || l >= h->nlevels) return set_error(CPRB_EINVAL, "level out of range");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = P->n[l];
  double* bl = P->rc[l - 1];  // level-l right-hand side buffer (permuted order)
  k_kgather<<<kfull(n), 256, 0, st>>>(n, perm, rhs, 1, bl);
  const double* xl;
  if (l == h->nlevels - 1) {
    k_kdense<<<kfull((int64_t)h->n_coarse * 32), 256, 0, st>>>(h->n_coarse, h->coarse_inv, bl,
                                                              P->coarse_x);
    xl = P->coarse_x;
  } else {
    const int rc = l >= P->kt_start ? ktail_launch(P->kt_dev, P->kt_threads, l, bl, st)
                   : h->use_fcg     ? fcg_at(*P, *h, l, bl, st)
                                    : fgmres_at(*P, *h, l, bl, st);
    if (rc) return rc;
    xl = P->x[l];
  }
  k_kscatter<<<kfull(n), 256, 0, st>>>(n, perm, xl, out);
  return check_launch("kcycle correction");
}

int cprb_kcycle_destroy(void* plan) {
  delete static_cast<KPlan*>(plan);
  return CPRB_OK;
}

}  // extern "C"
