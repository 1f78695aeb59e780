// Internal declarations shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/cpr_b200.h"

#include <utility>

namespace cprb {

// launch with programmatic stream serialization (PDL); kernels call
// pdl_trigger() early and pdl_wait() before touching data of earlier grids
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int set_error(int code, const std::string& msg);
int check_launch(const char* what);

int bsr_op(int mode, const cprb_sell& A, int b, const double* x, const double* rhs, double* out,
           int32_t* flag, double* sent, cudaStream_t st, const int32_t* out_idx = nullptr,
           double* sent2 = nullptr, const int32_t* sent_idx = nullptr,
           const int32_t* sent2_idx = nullptr);
int wave_solve(const cprb_bilu& F, const double* rhsL, cudaStream_t st);
int stencil_solve(const cprb_bilu& F, const double* rhsL, cudaStream_t st);
int stencil_arm(const cprb_bilu& F, cudaStream_t st);
int wave_combine(const cprb_bilu& F, const double* zp, double* z, cudaStream_t st);
int wave_scatter_rhs(const cprb_bilu& F, const double* r, double* rhsL, cudaStream_t st);
int amg_vcycle(const cprb_amg& h, const double* r, double* z, cudaStream_t st);
int launch_vtail(const cprb_amg& h, cudaStream_t st);
int kcycle_apply(const cprb_amg& h, const double* r, double* z, cudaStream_t st);
int bilu_solve(const cprb_bilu& F, const double* r, double* zl, double* y, const double* zp,
               double* zout, cudaStream_t st);
int fill_sentinel(double* p, int64_t n, cudaStream_t st);
int pgs_pass(const cprb_amg_level& L, const double* b, double* x, int dir, int zero_guess,
             const double* gather_src, int gather_stride, const int32_t* perm,
             double* scatter_out, cudaStream_t st, int skip_first = 0);
}  // namespace cprb
