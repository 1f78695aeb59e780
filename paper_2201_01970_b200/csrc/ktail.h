// Plan of the persistent K-cycle tail (csrc/ktail.cu), built by
// cprb_kcycle_create (csrc/kcycle.cu) and copied to the device once.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cpr_b200.h"

namespace cprb {

constexpr int KT_MAXL = 24;   // levels addressable by the tail
constexpr int KT_MAXD = 12;   // Krylov frames nested inside one tail launch
constexpr int KT_MAXC = 32;   // colours per level
constexpr int KT_MAXVB = 32;  // cprb_dot virtual CTAs (tail levels <= 32768 rows)

struct KTLevel {
  cprb_sell sm;          // smoother: off-diagonals, ascending permuted columns
  cprb_sell rop;         // residual + restriction (aggregate lane pairs)
  cprb_sell A;           // Krylov operator (permuted rows, original column order)
  const double* diag;
  const int32_t* aggp;
  // Krylov frame at this level (csrc/kcycle.cu KPlan) and the restriction buffer
  double *x, *r, *z1, *ap1, *z2, *p2, *ap2, *tmp, *rc;
  int32_t n, nc;
  uint32_t snap;         // bit k: colour k has intra-colour couplings
  int32_t cr[KT_MAXC + 1];
  int32_t cs[KT_MAXC + 1];
};

struct KTDesc {
  int32_t L;             // levels including the coarsest
  int32_t start;         // first level whose Krylov frame runs in the tail
  int32_t pre, post;
  int32_t use_fcg;
  int32_t n_coarse;
  const double* coarse_inv;
  double* coarse_x;
  KTLevel lv[KT_MAXL];
};

int ktail_launch(const KTDesc* dev_desc, int threads, int l, const double* rhs, cudaStream_t st);

}  // namespace cprb
