// Device helpers shared by the cprb kernels.
//
// Summation orders reproduce numpy exactly:
//   reduceat segment = e[0] + pairwise(e[1:]);  pairwise(n<8) = sequential
//   from 0.0; 8<=n<=128: 8 accumulators, then ((r0+r1)+(r2+r3))+((r4+r5)+
//   (r6+r7)), then the tail; n>128 splits at n2 = n/2 - (n/2)%8.
// All kernels are compiled with -fmad=false so products and sums round
// separately, as numpy does.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cpr_b200.h"

#define CPRB_FULL 0xffffffffu
// sentinel for sync-free triangular solves: a signalling-NaN payload that
// GPU arithmetic never produces (results are canonical quiet NaNs)
#define CPRB_SENTINEL 0x7FF4C0FFEE5EED01ull

namespace cprb {

__device__ __forceinline__ double ld_relaxed(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return __longlong_as_double((long long)v);
}

__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v))
               : "memory");
}

__device__ __forceinline__ double sentinel() { return __longlong_as_double((long long)CPRB_SENTINEL); }

// wait until *p holds a published value (anything but the sentinel)
__device__ __forceinline__ double wait_value(const double* p) {
  double v = ld_relaxed(p);
  int spins = 0;
  while ((unsigned long long)__double_as_longlong(v) == CPRB_SENTINEL) {
    if (++spins > 4) __nanosleep(32);
    v = ld_relaxed(p);
  }
  return v;
}

// ---- exact numpy pairwise summation, compile-time length ------------------
template <int N>
__device__ __forceinline__ double pairwise_fixed(const double* a) {
  if constexpr (N < 8) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < N; ++t) s = s + a[t];
    return s;
  } else if constexpr (N <= 128) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    constexpr int nf = N & ~7;
#pragma unroll
    for (int g = 8; g < nf; g += 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = r[k] + a[g + k];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
    for (int t = nf; t < N; ++t) s = s + a[t];
    return s;
  } else {
    constexpr int h = N / 2;
    constexpr int n2 = h - h % 8;
    return pairwise_fixed<n2>(a) + pairwise_fixed<N - n2>(a + n2);
  }
}

// reduceat segment of compile-time length N: a[0] + pairwise(a[1:])
template <int N>
__device__ __forceinline__ double segsum_fixed(const double* a) {
  if constexpr (N == 0) {
    return 0.0;
  } else {
    return a[0] + pairwise_fixed<N - 1>(a + 1);
  }
}

// ---- runtime length, elements produced by a functor f(t) -------------------
template <class F>
__device__ __forceinline__ double pairwise_leaf(const F& f, int off, int n) {
  if (n < 8) {
    double s = 0.0;
    for (int t = 0; t < n; ++t) s = s + f(off + t);
    return s;
  }
  double r0 = f(off + 0), r1 = f(off + 1), r2 = f(off + 2), r3 = f(off + 3);
  double r4 = f(off + 4), r5 = f(off + 5), r6 = f(off + 6), r7 = f(off + 7);
  const int nf = n & ~7;
  for (int g = 8; g < nf; g += 8) {
    r0 = r0 + f(off + g + 0);
    r1 = r1 + f(off + g + 1);
    r2 = r2 + f(off + g + 2);
    r3 = r3 + f(off + g + 3);
    r4 = r4 + f(off + g + 4);
    r5 = r5 + f(off + g + 5);
    r6 = r6 + f(off + g + 6);
    r7 = r7 + f(off + g + 7);
  }
  double s = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (int t = nf; t < n; ++t) s = s + f(off + t);
  return s;
}

template <class F>
__device__ __noinline__ double pairwise_rec(const F f, int off, int n) {
  if (n <= 128) return pairwise_leaf(f, off, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_rec(f, off, n2) + pairwise_rec(f, off + n2, n - n2);
}

template <class F>
__device__ __forceinline__ double segsum_rt(const F& f, int L) {
  if (L <= 0) return 0.0;
  const double a0 = f(0);
  const int n = L - 1;
  if (n <= 128) return a0 + pairwise_leaf(f, 1, n);
  return a0 + pairwise_rec(f, 1, n);
}

// reduceat segment of runtime length L <= N held in registers e[0..N-1]
// (entries >= L are ignored): e[0] + pairwise(e[1:L]) with predicated,
// branch-free accumulation so that lanes of different length stay converged.
// The n < 8 sequential part starts from -0.0, the exact additive identity.
template <int N>
__device__ __forceinline__ double segsum_masked(const double* e, int L) {
  static_assert(N <= 129, "segsum_masked handles rows of at most 129 entries");
  if constexpr (N == 0) {
    return 0.0;
  } else {
    const int n = L - 1;  // entries in the pairwise part
    double s = -0.0;
    if constexpr (N - 1 < 8) {
#pragma unroll
      for (int t = 0; t < N - 1; ++t)
        if (t < n) s = s + e[1 + t];
    } else {
      if (n < 8) {
#pragma unroll
        for (int t = 0; t < 7; ++t)
          if (t < n) s = s + e[1 + t];
      } else {
        const int nf = n & ~7;
        double r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = e[1 + k];
#pragma unroll
        for (int g = 8; g + 8 <= N - 1; g += 8)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (g < nf) r[k] = r[k] + e[1 + g + k];
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
        for (int t = 8; t < N - 1; ++t)
          if (t >= nf && t < n) s = s + e[1 + t];
      }
    }
    return L > 0 ? e[0] + s : 0.0;
  }
}

// np.einsum('kij,kj->ki') row r of a b x b block times a b-vector
// (b = 3: (p0 + p2) + p1; b = 1: p0)
template <int B>
__device__ __forceinline__ double block_row_dot(const double* m, const double* v) {
  if constexpr (B == 1) {
    return m[0] * v[0];
  } else if constexpr (B == 3) {
    return (m[0] * v[0] + m[2] * v[2]) + m[1] * v[1];
  } else {
    static_assert(B == 1 || B == 3, "block size");
    return 0.0;
  }
}

// Programmatic Dependent Launch: let the next grid start its prologue now;
// wait until every prerequisite grid finished (and its writes are visible).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void flag_nonfinite(int32_t* flag, bool bad) {
  if (flag && bad) atomicOr(flag, 1);
}

}  // namespace cprb
