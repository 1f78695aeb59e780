// Restarted right-preconditioned GMRES (src/cpr.py:231-316) driven from C++
// for hosts that bind the C ABI directly (no Python): the same device steps
// as the Python driver (cpr.py:gmres_solve) -- explicit residual, CPR
// application (graph-replayed when a cache is given), BSR product, fused MGS
// column, correction and explicit residual -- and the reference's host
// arithmetic for the Givens rotations (hypot from libm, as numpy's) and the
// upper-triangular solve.  The back substitution is the column-oriented
// textbook order, so y (and x) agree with the Python driver (which calls
// LAPACK trtrs) to rounding; iteration counts and the convergence decision
// follow the same rules.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "engine.h"

namespace {

using cprb::set_error;

struct HostSync {
  cudaStream_t st;
  int copy(void* dst, const void* src, size_t bytes) {
    if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return cprb::check_launch("gmres host copy");
    return CPRB_OK;
  }
};

}  // namespace

extern "C" {

int cprb_gmres_solve(const cprb_sell* A, int32_t b, const cprb_cpr* P, void* graphs, int64_t n,
                     const double* rhs, double* x, int32_t m, int32_t max_restarts, double tol,
                     double* work, int32_t* iwork, double* result, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!A || !rhs || !x || !work || !iwork || !result || n <= 0 || m < 1 || max_restarts < 0)
    return set_error(CPRB_EINVAL, "cprb_gmres_solve: invalid arguments");
  if ((int64_t)A->nrows * b != n)
    return set_error(CPRB_EINVAL, "dimension mismatch: matrix rows x block size != rhs length");
  // device workspace: V (m+1) x n | z | r | u | hcol (m+2) | y (m) | dot out | partials
  double* V = work;
  double* z = V + (int64_t)(m + 1) * n;
  double* r = z + n;
  double* u = r + n;
  double* hcol = u + n;
  double* ydev = hcol + (m + 2);
  double* dout = ydev + m;
  double* partials = dout + 1;
  int32_t* flags = iwork;       // [0] Krylov vector, [1] residual
  int32_t* ticket = iwork + 2;  // dot ticket
  HostSync hs{st};
  int rc;
  if (cudaMemsetAsync(iwork, 0, 4 * sizeof(int32_t), st) != cudaSuccess)
    return cprb::check_launch("gmres flags");
  auto norm = [&](const double* v, double& out) -> int {
    int e = cprb_dot(n, v, v, dout, partials, ticket, st);
    if (e) return e;
    double s = 0.0;
    if ((e = hs.copy(&s, dout, sizeof(double)))) return e;
    out = std::sqrt(s);
    return CPRB_OK;
  };
  auto apply = [&](const double* in, double* out) -> int {
    return graphs ? cprb_cpr_apply_graph(graphs, P, in, out, st) : cprb_cpr_apply(P, in, out, st);
  };
  if ((rc = cprb_residual(A, b, rhs, x, r, nullptr, st))) return rc;
  double beta0 = 0.0;
  if ((rc = norm(r, beta0))) return rc;
  result[0] = result[1] = 0.0;
  result[2] = 0.0;
  result[3] = 1.0;
  if (!std::isfinite(beta0))
    return set_error(CPRB_ENONFINITE, "non-finite initial residual in gmres_solve");
  if (beta0 == 0.0) {
    result[2] = 1.0;
    result[3] = 0.0;
    return CPRB_OK;
  }
  int inner_total = 0, outer = 0;
  bool converged = false;
  double rel = 1.0;
  std::vector<double> H, cs, sn, g, y, hc(m + 2);
  for (outer = 1; outer <= max_restarts; ++outer) {
    double beta = beta0;
    if (outer > 1 && (rc = norm(r, beta))) return rc;
    if (beta == 0.0) {
      converged = true;
      break;
    }
    if ((rc = cprb_div_host(n, r, beta, V, st))) return rc;
    H.assign((size_t)(m + 1) * m, 0.0);  // row-major (m+1) x m
    cs.assign(m, 0.0);
    sn.assign(m, 0.0);
    g.assign(m + 1, 0.0);
    g[0] = beta;
    auto h = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };
    int j_used = 0, shrink = 0;
    for (int j = 0; j < m; ++j) {
      double* vj = V + (int64_t)j * n;
      const double* zj = vj;
      if (P) {
        if ((rc = apply(vj, z))) return rc;
        zj = z;
      }
      if ((rc = cprb_spmv(A, b, zj, V + (int64_t)(j + 1) * n, flags, st))) return rc;
      if ((rc = cprb_arnoldi_mgs(n, j, V, n, hcol, partials, ticket, st))) return rc;
      int32_t fl[1] = {0};
      if (cudaMemcpyAsync(hc.data(), hcol, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess)
        return cprb::check_launch("gmres hcol");
      if ((rc = hs.copy(fl, flags, sizeof(int32_t)))) return rc;
      if (fl[0]) return set_error(CPRB_ENONFINITE, "non-finite Krylov vector in gmres_solve");
      for (int i = 0; i < j + 2; ++i) h(i, j) = hc[i];
      j_used = j + 1;
      ++inner_total;
      const bool breakdown = h(j + 1, j) == 0.0;
      for (int i = 0; i < j; ++i) {  // previous rotations (reference arithmetic)
        const double tt = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
        h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
        h(i, j) = tt;
      }
      const double denom = std::hypot(h(j, j), h(j + 1, j));
      if (denom == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = h(j, j) / denom;
        sn[j] = h(j + 1, j) / denom;
      }
      h(j, j) = denom;
      h(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      if (breakdown) {
        shrink = j + 1;
        break;
      }
      if (std::fabs(g[j + 1]) < tol * beta0) break;
    }
    // y = R^{-1} g (src/cpr.py:224-228); a zero pivot takes the reference's
    // least-squares branch, which this driver does not restate
    y.assign(j_used, 0.0);
    for (int i = 0; i < j_used; ++i)
      if (!(std::fabs(h(i, i)) > 0.0))
        return set_error(CPRB_EUNSUPPORTED,
                         "cprb_gmres_solve: singular Hessenberg (the reference's lstsq branch); "
                         "use the Python driver");
    for (int i = 0; i < j_used; ++i) y[i] = g[i];
    for (int jj = j_used - 1; jj >= 0; --jj) {
      y[jj] = y[jj] / h(jj, jj);
      for (int i = 0; i < jj; ++i) y[i] = y[i] - y[jj] * h(i, jj);
    }
    if (cudaMemcpyAsync(ydev, y.data(), sizeof(double) * j_used, cudaMemcpyHostToDevice, st) !=
        cudaSuccess)
      return cprb::check_launch("gmres y");
    if ((rc = cprb_gemv_t(n, j_used, V, n, ydev, u, st))) return rc;
    if (P) {
      if ((rc = apply(u, z))) return rc;
      if ((rc = cprb_add(n, x, z, x, st))) return rc;
    } else if ((rc = cprb_add(n, x, u, x, st))) {
      return rc;
    }
    if ((rc = cprb_residual(A, b, rhs, x, r, flags + 1, st))) return rc;
    if ((rc = norm(r, rel))) return rc;
    rel /= beta0;
    int32_t fl1 = 0;
    if ((rc = hs.copy(&fl1, flags + 1, sizeof(int32_t)))) return rc;
    if (fl1) return set_error(CPRB_ENONFINITE, "non-finite residual in gmres_solve (divergence)");
    if (shrink) m = shrink;
    if (rel < tol) {
      converged = true;
      break;
    }
  }
  if (outer > max_restarts) outer = max_restarts;
  result[0] = outer;
  result[1] = inner_total;
  result[2] = converged ? 1.0 : 0.0;
  result[3] = rel;
  return CPRB_OK;
}

}  // extern "C"
