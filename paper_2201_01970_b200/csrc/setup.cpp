// Host-side SETUP of the CPR preconditioner: strong connections, colour
// grouping, pairwise aggregation, Galerkin products, BILU(0), level
// schedules, coarsest inverse.  Structural outputs are bit-exact to the
// reference (cprkit); floating-point sums follow numpy's reduceat order.
// Compiled with -ffp-contract=off (no FMA contraction).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <queue>
#include <string>
#include <vector>

#include "common.h"

namespace cprb {

// numpy pairwise summation of a contiguous float64 run (the order of
// np.add.reduce / the reduceat tail).
double pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i];
    return s;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int64_t i = 8;
    for (; i + 8 <= n; i += 8)
      for (int k = 0; k < 8; ++k) r[k] += a[i + k];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) s += a[i];
    return s;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

// one np.add.reduceat segment: a[0] + pairwise(a[1:])
double segment_sum(const double* a, int64_t n) {
  if (n <= 0) return 0.0;
  return a[0] + pairwise_sum(a + 1, n - 1);
}

}  // namespace cprb

using namespace cprb;

extern "C" {

// src/coloring.py:79-114
int cprb_strong_connections(int64_t n, const int64_t* ptr, const int64_t* cols,
                            const double* vals, double theta, int64_t* s_ptr,
                            int64_t* s_cols) {
  if (!(theta >= 0.0 && theta <= 1.0))
    return set_error(CPRB_EINVAL, "theta must lie in [0, 1], got " + std::to_string(theta));
  std::vector<double> absrow;
  int64_t k = 0;
  s_ptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = ptr[i], hi = ptr[i + 1];
    absrow.resize(hi - lo);
    for (int64_t p = lo; p < hi; ++p) absrow[p - lo] = std::fabs(vals[p]);
    const double thr = theta * segment_sum(absrow.data(), hi - lo);
    for (int64_t p = lo; p < hi; ++p)
      if (cols[p] != i && absrow[p - lo] > thr) s_cols[k++] = cols[p];
    s_ptr[i + 1] = k;
  }
  return CPRB_OK;
}

// src/coloring.py:238-256, vertices_splitting :171-235.
int cprb_vertices_grouping(int64_t n, const int64_t* s_ptr, const int64_t* s_cols,
                           int64_t* perm, int64_t* group_sizes, int64_t* ncolors) {
  // symmetrised pattern S ∪ S^T (src/coloring.py:58-71), sorted & deduplicated
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = s_ptr[i]; p < s_ptr[i + 1]; ++p) {
      cnt[i + 1]++;
      cnt[s_cols[p] + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int64_t> adj(cnt[n]);
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = s_ptr[i]; p < s_ptr[i + 1]; ++p) {
      adj[fill[i]++] = s_cols[p];
      adj[fill[s_cols[p]]++] = i;
    }
  std::vector<int64_t> nptr(n + 1, 0);
  std::vector<int32_t> nadj;  // 32-bit: half the cache footprint of the walks below
  nadj.reserve(adj.size());
  for (int64_t i = 0; i < n; ++i) {
    auto b = adj.begin() + cnt[i], e = adj.begin() + cnt[i + 1];
    std::sort(b, e);
    auto u = std::unique(b, e);
    for (auto it = b; it != u; ++it) nadj.push_back((int32_t)*it);
    nptr[i + 1] = (int64_t)nadj.size();
  }
  std::vector<int64_t> infl(n);
  int64_t maxinfl = 0;
  for (int64_t i = 0; i < n; ++i) {
    infl[i] = nptr[i + 1] - nptr[i];
    maxinfl = std::max(maxinfl, infl[i]);
  }
  // priority key: (-influence, index) ascending  <=>  (maxinfl-infl, index)
  auto key = [&](int64_t v) -> uint64_t {
    return ((uint64_t)(maxinfl - infl[v]) << 32) | (uint64_t)v;
  };
  using MinHeap = std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>>;

  std::vector<uint8_t> und(n), deferred(n), in_front(n), in_w(n);
  std::vector<int64_t> vertices(n);
  std::iota(vertices.begin(), vertices.end(), 0);
  int64_t out = 0, ng = 0;
  while (!vertices.empty()) {
    std::fill(und.begin(), und.end(), 0);
    std::fill(deferred.begin(), deferred.end(), 0);
    std::fill(in_front.begin(), in_front.end(), 0);
    std::fill(in_w.begin(), in_w.end(), 0);
    // V candidates by (influence desc, index asc): the keys never change
    // within a round, so the heap of the reference is a bucket-sorted list
    // consumed front to back (entries no longer undetermined are skipped)
    std::vector<int64_t> vorder(vertices.size());
    {
      std::vector<int64_t> bstart(maxinfl + 2, 0);
      for (int64_t v : vertices) {
        und[v] = 1;
        ++bstart[maxinfl - infl[v] + 1];
      }
      for (int64_t b = 0; b <= maxinfl; ++b) bstart[b + 1] += bstart[b];
      for (int64_t v : vertices) vorder[bstart[maxinfl - infl[v]]++] = v;  // vertices ascending
    }
    size_t vpos = 0;
    // frontier by (influence desc, index asc): one index min-heap per
    // influence bucket -- the same pop order as one heap on the pair
    std::vector<std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>>> fb(
        maxinfl + 1);
    int64_t ftop = maxinfl + 1, fsize = 0;
    std::vector<int64_t> w;
    int64_t remaining = (int64_t)vertices.size();
    while (remaining > 0) {
      int64_t v = -1;
      while (fsize > 0) {
        while (fb[ftop].empty()) ++ftop;
        const int64_t c = fb[ftop].top();
        fb[ftop].pop();
        --fsize;
        if (in_front[c] && und[c]) {
          in_front[c] = 0;
          v = c;
          break;
        }
        in_front[c] = 0;
      }
      if (v < 0) {
        while (vpos < vorder.size()) {
          const int64_t c = vorder[vpos++];
          if (und[c]) {
            v = c;
            break;
          }
        }
        if (v < 0) break;
      }
      bool touches = false;
      for (int64_t p = nptr[v]; p < nptr[v + 1]; ++p)
        if (in_w[nadj[p]]) { touches = true; break; }
      if (touches) {
        deferred[v] = 1;
        und[v] = 0;
        --remaining;
        continue;
      }
      in_w[v] = 1;
      w.push_back(v);
      und[v] = 0;
      --remaining;
      for (int64_t p = nptr[v]; p < nptr[v + 1]; ++p) {
        int64_t k = nadj[p];
        if (und[k]) {
          deferred[k] = 1;
          und[k] = 0;
          --remaining;
        }
      }
      for (int64_t p = nptr[v]; p < nptr[v + 1]; ++p) {
        int64_t k = nadj[p];
        for (int64_t q = nptr[k]; q < nptr[k + 1]; ++q) {
          int64_t j = nadj[q];
          if (und[j] && !in_front[j] && j != v) {
            in_front[j] = 1;
            const int64_t bkt = maxinfl - infl[j];
            fb[bkt].push(j);
            ++fsize;
            if (bkt < ftop) ftop = bkt;
          }
        }
      }
    }
    if (w.empty()) return set_error(CPRB_ERUNTIME, "vertices_splitting returned an empty group");
    std::sort(w.begin(), w.end());
    for (int64_t v : w) perm[out++] = v;
    group_sizes[ng++] = (int64_t)w.size();
    std::vector<int64_t> wbar;
    for (int64_t v = 0; v < n; ++v)
      if (deferred[v]) wbar.push_back(v);
    vertices.swap(wbar);
  }
  *ncolors = ng;
  return CPRB_OK;
}

// src/amg.py:89-119
int cprb_pairwise_aggregate(int64_t n, const int64_t* ptr, const int64_t* cols,
                            const double* vals, double theta_amg, int64_t* agg,
                            int64_t* n_agg) {
  std::vector<int64_t> sptr(n + 1), scols(ptr[n] > 0 ? ptr[n] : 1);
  int rc = cprb_strong_connections(n, ptr, cols, vals, theta_amg, sptr.data(), scols.data());
  if (rc) return rc;
  auto find = [&](int64_t row, int64_t col) -> int64_t {
    const int64_t* b = cols + ptr[row];
    const int64_t* e = cols + ptr[row + 1];
    const int64_t* it = std::lower_bound(b, e, col);
    return (it != e && *it == col) ? (int64_t)(it - cols) : -1;
  };
  for (int64_t i = 0; i < n; ++i) agg[i] = -1;
  int64_t na = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    int64_t best = -1;
    double bw = 0.0;
    for (int64_t p = sptr[i]; p < sptr[i + 1]; ++p) {
      int64_t j = scols[p];
      if (agg[j] >= 0) continue;
      // W = |A| + |A|^T via duplicate-summing COO: |a_ij| first, then |a_ji|
      int64_t pij = find(i, j), pji = find(j, i);
      double wgt = std::fabs(vals[pij]);
      if (pji >= 0) wgt = wgt + (0.0 + std::fabs(vals[pji]));
      if (best < 0 || wgt > bw) {
        best = j;
        bw = wgt;
      }
    }
    if (best >= 0) agg[best] = na;
    agg[i] = na;
    ++na;
  }
  *n_agg = na;
  return CPRB_OK;
}

// src/amg.py:127-132 via CsrMatrix.from_coo(sum_duplicates=True)
// (src/sparse.py:88-110): stable order = fine row-major inside each (I, J).
int cprb_galerkin(int64_t n, const int64_t* ptr, const int64_t* cols, const double* vals,
                  const int64_t* agg, int64_t n_agg, int64_t* c_ptr, int64_t* c_cols,
                  double* c_vals, int64_t* c_nnz) {
  const int64_t nnz = ptr[n];
  // stable counting sort of entries by coarse row I
  std::vector<int64_t> rcnt(n_agg + 1, 0);
  for (int64_t i = 0; i < n; ++i) rcnt[agg[i] + 1] += ptr[i + 1] - ptr[i];
  for (int64_t I = 0; I < n_agg; ++I) rcnt[I + 1] += rcnt[I];
  std::vector<int64_t> order(nnz);
  {
    std::vector<int64_t> fill(rcnt.begin(), rcnt.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) order[fill[agg[i]]++] = p;
  }
  std::vector<double> run;
  std::vector<int64_t> key;
  int64_t k = 0;
  c_ptr[0] = 0;
  for (int64_t I = 0; I < n_agg; ++I) {
    int64_t* ob = order.data() + rcnt[I];
    const int64_t m = rcnt[I + 1] - rcnt[I];
    // stable insertion sort by coarse column J (the lexsort order; rows are short)
    key.resize(m > 0 ? m : 1);
    for (int64_t t = 0; t < m; ++t) {
      const int64_t x = ob[t], kx = agg[cols[x]];
      int64_t u = t;
      while (u > 0 && key[u - 1] > kx) {
        key[u] = key[u - 1];
        ob[u] = ob[u - 1];
        --u;
      }
      key[u] = kx;
      ob[u] = x;
    }
    for (int64_t t = 0; t < m;) {
      const int64_t J = key[t];
      run.clear();
      int64_t u = t;
      while (u < m && key[u] == J) run.push_back(vals[ob[u++]]);
      c_cols[k] = J;
      c_vals[k] = segment_sum(run.data(), (int64_t)run.size());
      ++k;
      t = u;
    }
    c_ptr[I + 1] = k;
  }
  *c_nnz = k;
  return CPRB_OK;
}

// src/amg.py:135-140
int cprb_is_symmetric(int64_t n, const int64_t* ptr, const int64_t* cols, const double* vals,
                      double tol, int32_t* out) {
  double scale = 0.0, diff = 0.0;
  bool nan = false;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) {
      const int64_t j = cols[p];
      const int64_t* b = cols + ptr[j];
      const int64_t* e = cols + ptr[j + 1];
      const int64_t* it = std::lower_bound(b, e, i);
      if (it == e || *it != i) {
        *out = 0;
        return CPRB_OK;
      }
      const double a = vals[p], t = vals[it - cols];
      if (std::isnan(a) || std::isnan(t)) nan = true;
      scale = std::max(scale, std::fabs(a));
      diff = std::max(diff, std::fabs(a - t));
    }
  *out = (!nan && diff <= tol * std::max(scale, 1.0)) ? 1 : 0;
  return CPRB_OK;
}

}  // extern "C"

namespace {

// src/sparse.py:372-396 (Gauss-Jordan with partial pivoting; same elementwise
// operation sequence, so bitwise equal).  Returns false on an exact zero pivot.
bool gj_invert(int b, const double* blk, double* inv) {
  double a[64], v[64];
  for (int i = 0; i < b * b; ++i) a[i] = blk[i];
  for (int r = 0; r < b; ++r)
    for (int c = 0; c < b; ++c) v[r * b + c] = (r == c) ? 1.0 : 0.0;
  for (int col = 0; col < b; ++col) {
    int p = col;
    double best = std::fabs(a[col * b + col]);
    for (int r = col + 1; r < b; ++r)
      if (std::fabs(a[r * b + col]) > best) {
        best = std::fabs(a[r * b + col]);
        p = r;
      }
    if (a[p * b + col] == 0.0) return false;
    if (p != col)
      for (int c = 0; c < b; ++c) {
        std::swap(a[col * b + c], a[p * b + c]);
        std::swap(v[col * b + c], v[p * b + c]);
      }
    const double piv = a[col * b + col];
    for (int c = 0; c < b; ++c) {
      a[col * b + c] /= piv;
      v[col * b + c] /= piv;
    }
    for (int r = 0; r < b; ++r) {
      if (r == col) continue;
      const double f = a[r * b + col];
      if (f != 0.0)
        for (int c = 0; c < b; ++c) {
          a[r * b + c] = a[r * b + c] - f * a[col * b + c];
          v[r * b + c] = v[r * b + c] - f * v[col * b + c];
        }
    }
  }
  for (int i = 0; i < b * b; ++i) inv[i] = v[i];
  return true;
}

inline void matmul(int b, const double* x, const double* y, double* out) {
  for (int i = 0; i < b; ++i)
    for (int l = 0; l < b; ++l) {
      double s = 0.0;
      for (int j = 0; j < b; ++j) s = s + x[i * b + j] * y[j * b + l];
      out[i * b + l] = s;
    }
}

// BILU(0) rows with a compile-time block size: the generic loop below with
// matmul/gj_invert unrolled -- the same operations in the same order, so the
// factors are bitwise those of the runtime-b path
template <int B>
inline void matmul_t(const double* x, const double* y, double* out) {
  for (int i = 0; i < B; ++i)
    for (int l = 0; l < B; ++l) {
      double s = 0.0;
      for (int j = 0; j < B; ++j) s = s + x[i * B + j] * y[j * B + l];
      out[i * B + l] = s;
    }
}

template <int B>
int bilu0_rows(int64_t n, const int64_t* ptr, const int64_t* cols, double* vals, double* uinv,
               int64_t* perturbed, int64_t* n_perturbed) {
  constexpr int BB = B * B;
  int64_t npert = 0;
  double tmp[BB];
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = ptr[i], hi = ptr[i + 1];
    const int64_t* rb = cols + lo;
    const int64_t dk = std::lower_bound(rb, cols + hi, i) - rb;
    if (lo + dk >= hi || cols[lo + dk] != i)
      return set_error(CPRB_EINVAL, "diagonal block missing in row " + std::to_string(i));
    for (int64_t p = lo; p < lo + dk; ++p) {
      const int64_t k = cols[p];
      matmul_t<B>(vals + p * BB, uinv + k * BB, tmp);
      std::memcpy(vals + p * BB, tmp, sizeof(double) * BB);
      const int64_t klo = ptr[k], khi = ptr[k + 1];
      int64_t pos = klo;
      for (int64_t q = p + 1; q < hi; ++q) {
        const int64_t j = cols[q];
        while (pos < khi && cols[pos] < j) ++pos;
        if (pos < khi && cols[pos] == j) {
          matmul_t<B>(vals + p * BB, vals + pos * BB, tmp);
          for (int e = 0; e < BB; ++e) vals[q * BB + e] = vals[q * BB + e] - tmp[e];
        }
      }
    }
    const double* piv = vals + (lo + dk) * BB;
    if (!gj_invert(B, piv, uinv + i * BB)) {
      double sq[BB];
      for (int e = 0; e < BB; ++e) sq[e] = piv[e] * piv[e];
      const double fro = std::sqrt(pairwise_sum(sq, BB));
      if (fro == 0.0)
        return set_error(CPRB_ESINGULAR, "singular pivot block at row " + std::to_string(i));
      const double t = 1e-8 * fro;
      double bumped[BB];
      for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) bumped[r * B + c] = piv[r * B + c] + (r == c ? t * 1.0 : t * 0.0);
      if (!gj_invert(B, bumped, uinv + i * BB))
        return set_error(CPRB_ESINGULAR, "singular pivot block at row " + std::to_string(i));
      perturbed[npert++] = i;
    }
  }
  *n_perturbed = npert;
  return CPRB_OK;
}

}  // namespace

extern "C" {

int cprb_invert_small_blocks(int64_t m, int32_t b, const double* blocks, double* out) {
  if (b < 1 || b > 8) return set_error(CPRB_EINVAL, "block size must be 1..8");
  for (int64_t k = 0; k < m; ++k)
    if (!gj_invert(b, blocks + k * b * b, out + k * b * b))
      return set_error(CPRB_ESINGULAR, "singular diagonal block at row " + std::to_string(k));
  return CPRB_OK;
}

// src/ilu.py:150-193 (+ _invert_pivot :134-147)
int cprb_bilu0_factorize(int64_t n, int32_t b, const int64_t* ptr, const int64_t* cols,
                         double* vals, double* uinv, int64_t* perturbed,
                         int64_t* n_perturbed) {
  if (b < 1 || b > 8) return set_error(CPRB_EINVAL, "block size must be 1..8");
  if (b == 3) return bilu0_rows<3>(n, ptr, cols, vals, uinv, perturbed, n_perturbed);
  const int bb = b * b;
  int64_t npert = 0;
  double tmp[64];
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = ptr[i], hi = ptr[i + 1];
    const int64_t* rb = cols + lo;
    const int64_t dk = std::lower_bound(rb, cols + hi, i) - rb;
    if (lo + dk >= hi || cols[lo + dk] != i)
      return set_error(CPRB_EINVAL, "diagonal block missing in row " + std::to_string(i));
    for (int64_t p = lo; p < lo + dk; ++p) {
      const int64_t k = cols[p];
      matmul(b, vals + p * bb, uinv + k * bb, tmp);
      std::memcpy(vals + p * bb, tmp, sizeof(double) * bb);
      const int64_t klo = ptr[k], khi = ptr[k + 1];
      int64_t pos = klo;
      for (int64_t q = p + 1; q < hi; ++q) {
        const int64_t j = cols[q];
        while (pos < khi && cols[pos] < j) ++pos;
        if (pos < khi && cols[pos] == j) {
          matmul(b, vals + p * bb, vals + pos * bb, tmp);
          for (int e = 0; e < bb; ++e) vals[q * bb + e] = vals[q * bb + e] - tmp[e];
        }
      }
    }
    const double* piv = vals + (lo + dk) * bb;
    if (!gj_invert(b, piv, uinv + i * bb)) {
      double sq[64];
      for (int e = 0; e < bb; ++e) sq[e] = piv[e] * piv[e];
      const double fro = std::sqrt(pairwise_sum(sq, bb));
      if (fro == 0.0)
        return set_error(CPRB_ESINGULAR, "singular pivot block at row " + std::to_string(i));
      const double t = 1e-8 * fro;
      double bumped[64];
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c)
          bumped[r * b + c] = piv[r * b + c] + (r == c ? t * 1.0 : t * 0.0);
      if (!gj_invert(b, bumped, uinv + i * bb))
        return set_error(CPRB_ESINGULAR, "singular pivot block at row " + std::to_string(i));
      perturbed[npert++] = i;
    }
  }
  *n_perturbed = npert;
  return CPRB_OK;
}

// src/ilu.py:38-59
int cprb_level_schedule(int64_t n, const int64_t* ptr, const int64_t* cols, int64_t* level,
                        int64_t* nlevels) {
  bool any_below = false, any_above = false;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p) {
      if (cols[p] < i) any_below = true;
      if (cols[p] > i) any_above = true;
    }
  if (any_below && any_above)
    return set_error(CPRB_EINVAL, "pattern is neither lower nor upper triangular");
  const bool lower = !any_above;
  int64_t maxl = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = lower ? t : n - 1 - t;
    int64_t m = 0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p)
      if (cols[p] != i) m = std::max(m, level[cols[p]]);
    level[i] = 1 + m;
    maxl = std::max(maxl, level[i]);
  }
  *nlevels = n > 0 ? maxl : 1;
  return CPRB_OK;
}

// Level schedule of the STRICT LOWER part of a pattern that may hold both
// triangles (A's own pattern): level(i) = 1 + max level(j), j < i in row i.
// The BILU(0) factorization's row dependencies (src/ilu.py:150-193); equal
// to cprb_level_schedule on the factor L's pattern.
int cprb_lower_level_schedule(int64_t n, const int64_t* ptr, const int64_t* cols, int64_t* level,
                              int64_t* nlevels) {
  int64_t maxl = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t m = 0;
    for (int64_t p = ptr[i]; p < ptr[i + 1]; ++p)
      if (cols[p] < i) m = std::max(m, level[cols[p]]);
    level[i] = 1 + m;
    maxl = std::max(maxl, level[i]);
  }
  *nlevels = n > 0 ? maxl : 1;
  return CPRB_OK;
}

// Colour-permuted diagonal / off-diagonal split (smoothers.ScalarSplit,
// src/smoothers.py:257-271 A.permuted(perm)): permuted row pr = inv[r]
// holds the entries (inv[c], v), c != r, sorted by inv[c]; diag[pr] = a_rr.
// off_ptr[n+1]; off_cols/off_vals capacity nnz.  Returns CPRB_ESINGULAR
// naming the first permuted row with a zero (or missing) diagonal.
int cprb_scalar_split(int64_t n, const int64_t* ptr, const int64_t* cols, const double* vals,
                      const int64_t* perm, const int64_t* inv, int64_t* off_ptr,
                      int64_t* off_cols, double* off_vals, double* diag) {
  off_ptr[0] = 0;
  for (int64_t pr = 0; pr < n; ++pr) {
    const int64_t r = perm[pr];
    int64_t cnt = 0;
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) cnt += cols[e] != r;
    off_ptr[pr + 1] = off_ptr[pr] + cnt;
  }
  for (int64_t pr = 0; pr < n; ++pr) {
    const int64_t r = perm[pr];
    int64_t* oc = off_cols + off_ptr[pr];
    double* ov = off_vals + off_ptr[pr];
    int64_t k = 0;
    double d = 0.0;
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
      if (cols[e] == r) {
        d = vals[e];
        continue;
      }
      // insertion by permuted column (rows are short)
      const int64_t pc = inv[cols[e]];
      int64_t t = k++;
      while (t > 0 && oc[t - 1] > pc) {
        oc[t] = oc[t - 1];
        ov[t] = ov[t - 1];
        --t;
      }
      oc[t] = pc;
      ov[t] = vals[e];
    }
    diag[pr] = d;
  }
  for (int64_t pr = 0; pr < n; ++pr)
    if (diag[pr] == 0.0) return set_error(CPRB_ESINGULAR, "zero diagonal at row " + std::to_string(pr));
  return CPRB_OK;
}

// SELL-32 fills (device.pack_sell layout: entry m of lane l of slice s at
// slice_ptr[s] + 32 m + l; b x b block value e at (slice_ptr[s] + 32 m) * bb +
// e * 32 + l).  The output arrays are zero-initialised by the caller.
// Lanes take their entries from a per-lane list (lane_ptr into ent_*):
int cprb_sell_fill_lanes(int64_t L, const int64_t* lane_ptr, const int64_t* slice_ptr,
                         const int64_t* ent_cols, const double* ent_vals, int32_t bs,
                         int32_t* out_cols, double* out_vals) {
  const int bb = bs * bs;
  for (int64_t l = 0; l < L; ++l) {
    const int64_t s = l >> 5, lane = l & 31;
    const int64_t a = lane_ptr[l], n = lane_ptr[l + 1] - a;
    for (int64_t m = 0; m < n; ++m) {
      const int64_t d = slice_ptr[s] + 32 * m + lane;
      out_cols[d] = (int32_t)ent_cols[a + m];
      if (bb == 1) {
        out_vals[d] = ent_vals[a + m];
      } else {
        const int64_t base = (slice_ptr[s] + 32 * m) * bb + lane;
        for (int e = 0; e < bb; ++e) out_vals[base + (int64_t)e * 32] = ent_vals[(a + m) * bb + e];
      }
    }
  }
  return CPRB_OK;
}

// ... or straight from the rows of a scalar CSR (lane_src[l] = source row,
// -1 = padding), entries in the row's stored order, columns optionally
// renumbered through colmap
int cprb_sell_fill_rows(int64_t L, const int64_t* lane_src, const int64_t* slice_ptr,
                        const int64_t* ptr, const int64_t* cols, const double* vals,
                        const int64_t* colmap, int32_t* out_cols, double* out_vals) {
  for (int64_t l = 0; l < L; ++l) {
    const int64_t r = lane_src[l];
    if (r < 0) continue;
    const int64_t d0 = slice_ptr[l >> 5] + (l & 31);
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
      const int64_t d = d0 + 32 * (e - ptr[r]);
      out_cols[d] = (int32_t)(colmap ? colmap[cols[e]] : cols[e]);
      out_vals[d] = vals[e];
    }
  }
  return CPRB_OK;
}

// Structured-grid detection for the stencil BILU plan (ilu.py stencil_plan):
// n = nx*ny*nz with x fastest and every row's block columns exactly the
// in-range 7-point neighbours, ascending (-z, -y, -x, i, +x, +y, +z).
// dims[0..2] = nx, ny, nz on success; returns 0 when the pattern is not such
// a grid (dims untouched), 1 when it is.
int cprb_detect_stencil(int64_t n, const int64_t* ptr, const int64_t* cols, int64_t* dims) {
  if (n < 8) return 0;
  // nx = distance to the first +y neighbour of row 0 = (col of the third
  // upper entry of row 0 when all three exist) -- derive from row 0: cols
  // 0, 1, nx, nxy
  if (ptr[1] - ptr[0] != 4) return 0;
  const int64_t nx = cols[ptr[0] + 2], nxy = cols[ptr[0] + 3];
  if (cols[ptr[0]] != 0 || cols[ptr[0] + 1] != 1 || nx < 2 || nxy <= nx || nxy % nx || n % nxy)
    return 0;
  const int64_t ny = nxy / nx, nz = n / nxy;
  if (ny < 2 || nz < 2) return 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t ix = i % nx, iy = (i / nx) % ny, iz = i / nxy;
    int64_t want[7];
    int k = 0;
    if (iz > 0) want[k++] = i - nxy;
    if (iy > 0) want[k++] = i - nx;
    if (ix > 0) want[k++] = i - 1;
    want[k++] = i;
    if (ix + 1 < nx) want[k++] = i + 1;
    if (iy + 1 < ny) want[k++] = i + nx;
    if (iz + 1 < nz) want[k++] = i + nxy;
    if (ptr[i + 1] - ptr[i] != k) return 0;
    for (int t = 0; t < k; ++t)
      if (cols[ptr[i] + t] != want[t]) return 0;
  }
  dims[0] = nx;
  dims[1] = ny;
  dims[2] = nz;
  return 1;
}

// Coarsest solve operator: inverse of a dense n x n matrix via LU with
// partial pivoting (first max |pivot|, the LAPACK getrf rule), then
// forward/back substitution of the identity columns.
int cprb_dense_inverse(int64_t n, const double* a_in, double* inv) {
  std::vector<double> a(a_in, a_in + n * n);
  std::vector<int64_t> piv(n);
  for (int64_t k = 0; k < n; ++k) {
    int64_t p = k;
    double best = std::fabs(a[k * n + k]);
    for (int64_t r = k + 1; r < n; ++r)
      if (std::fabs(a[r * n + k]) > best) {
        best = std::fabs(a[r * n + k]);
        p = r;
      }
    if (!std::isfinite(best))
      return set_error(CPRB_ERUNTIME, "coarsest-level dense factorization failed: non-finite entries");
    if (best == 0.0)
      return set_error(CPRB_ERUNTIME, "coarsest-level dense factorization failed: singular matrix");
    piv[k] = p;
    if (p != k)
      for (int64_t c = 0; c < n; ++c) std::swap(a[k * n + c], a[p * n + c]);
    const double d = a[k * n + k];
    for (int64_t r = k + 1; r < n; ++r) {
      const double l = a[r * n + k] / d;
      a[r * n + k] = l;
      if (l != 0.0)
        for (int64_t c = k + 1; c < n; ++c) a[r * n + c] -= l * a[k * n + c];
    }
  }
  std::vector<double> col(n);
  for (int64_t e = 0; e < n; ++e) {
    std::fill(col.begin(), col.end(), 0.0);
    col[e] = 1.0;
    for (int64_t k = 0; k < n; ++k)
      if (piv[k] != k) std::swap(col[k], col[piv[k]]);
    for (int64_t r = 0; r < n; ++r) {
      double s = col[r];
      for (int64_t c = 0; c < r; ++c) s -= a[r * n + c] * col[c];
      col[r] = s;
    }
    for (int64_t r = n - 1; r >= 0; --r) {
      double s = col[r];
      for (int64_t c = r + 1; c < n; ++c) s -= a[r * n + c] * col[c];
      col[r] = s / a[r * n + r];
    }
    for (int64_t r = 0; r < n; ++r) inv[r * n + e] = col[r];
  }
  return CPRB_OK;
}

}  // extern "C"
