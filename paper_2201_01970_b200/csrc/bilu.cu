// K8: BILU(0) triangular solves (src/ilu.py:196-223), sync-free.
//
// Lanes are laid out in level order (src/ilu.py:38-59) with every level
// padded to whole warps, so a warp never waits on itself.  Warps take slices
// through a global ticket (so every slice a warp waits on belongs to a warp
// that already started), prefetch their blocks, then spin on the
// dependencies' solution values: an output slot holds a sentinel NaN until
// its producer stores the value, so the value itself is the ready flag (one
// L2 round trip per dependency, no fences).
//
// Arithmetic matches the reference bitwise: block products in np.einsum
// order ((p0 + p2) + p1), per-component row sums in reduceat order.
#include "device.cuh"
#include "engine.h"

namespace cprb {

template <int B, int K>
__device__ __forceinline__ void tri_rowsum_fixed(const cprb_sell& T, int64_t base, int lane,
                                                 const double* dep, double* t) {
  int col[K];
  double mv[K][B * B];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    col[m] = __ldg(T.cols + base + (int64_t)m * 32 + lane);
#pragma unroll
    for (int e = 0; e < B * B; ++e)
      mv[m][e] = __ldg(T.vals + (base + (int64_t)m * 32) * (B * B) + (int64_t)e * 32 + lane);
  }
  double v[K][B];
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int c = 0; c < B; ++c) v[m][c] = wait_value(dep + (int64_t)B * col[m] + c);
#pragma unroll
  for (int r = 0; r < B; ++r) {
    double p[K];
#pragma unroll
    for (int m = 0; m < K; ++m) p[m] = block_row_dot<B>(&mv[m][r * B], v[m]);
    t[r] = segsum_fixed<K>(p);
  }
}

template <int B>
__device__ __forceinline__ void tri_rowsum_generic(const cprb_sell& T, int64_t base, int lane,
                                                   int len, const double* dep, double* t) {
#pragma unroll
  for (int r = 0; r < B; ++r) {
    auto f = [&](int m) -> double {
      const int64_t e = base + (int64_t)m * 32 + lane;
      const int j = T.cols[e];
      double mr[B], v[B];
#pragma unroll
      for (int c = 0; c < B; ++c) {
        mr[c] = T.vals[(base + (int64_t)m * 32) * (B * B) + (int64_t)(r * B + c) * 32 + lane];
        v[c] = wait_value(dep + (int64_t)B * j + c);
      }
      return block_row_dot<B>(mr, v);
    };
    t[r] = segsum_rt(f, len);
  }
}

template <int B>
__device__ __forceinline__ void tri_rowsum(const cprb_sell& T, int64_t base, int lane, int len,
                                           const double* dep, double* t) {
  switch (len) {
    case 0:
#pragma unroll
      for (int r = 0; r < B; ++r) t[r] = 0.0;
      break;
    case 1: tri_rowsum_fixed<B, 1>(T, base, lane, dep, t); break;
    case 2: tri_rowsum_fixed<B, 2>(T, base, lane, dep, t); break;
    case 3: tri_rowsum_fixed<B, 3>(T, base, lane, dep, t); break;
    case 4: tri_rowsum_fixed<B, 4>(T, base, lane, dep, t); break;
    default: tri_rowsum_generic<B>(T, base, lane, len, dep, t); break;
  }
}

__device__ __forceinline__ int take_ticket(int32_t* ticket) {
  const int lane = threadIdx.x & 31;
  int w = 0;
  if (lane == 0) {
    w = atomicAdd(ticket, 1);
    const int total = (int)(gridDim.x * (blockDim.x >> 5));
    if (w == total - 1) atomicExch(ticket, 0);  // last warp re-arms the ticket
  }
  return __shfl_sync(CPRB_FULL, w, 0);
}

// z_i = r_i - sum_{k<i} L_ik z_k ; also arms y (U-solve output) with the sentinel
template <int B>
__global__ void __launch_bounds__(256)
    k_bilu_lower(const cprb_sell L, int32_t* ticket, const double* __restrict__ r, double* z,
                 double* __restrict__ yarm) {
  const int w = take_ticket(ticket);
  const int lane = threadIdx.x & 31;
  if (w >= L.nslices) return;
  const int lid = w * 32 + lane;
  const int row = L.lane_row[lid];
  if (row < 0) return;
  const int len = L.lane_len[lid];
  double t[B];
  tri_rowsum<B>(L, L.slice_ptr[w], lane, len, z, t);
#pragma unroll
  for (int c = 0; c < B; ++c) {
    const int64_t o = (int64_t)B * row + c;
    st_relaxed(z + o, r[o] - t[c]);
    if (yarm) yarm[o] = sentinel();
  }
}

// y_i = Uinv_i (z_i - sum_{k>i} U_ik y_k);  zout = z1 + y  (src/cpr.py:186)
// with z1 = Pi zp (zp in block slot 0) when zp != NULL, else zout = y.
template <int B>
__global__ void __launch_bounds__(256)
    k_bilu_upper(const cprb_sell U, const double* __restrict__ uinv, int32_t* ticket,
                 const double* __restrict__ z, double* y, const double* __restrict__ zp,
                 double* __restrict__ zout) {
  const int w = take_ticket(ticket);
  const int lane = threadIdx.x & 31;
  if (w >= U.nslices) return;
  const int lid = w * 32 + lane;
  const int row = U.lane_row[lid];
  if (row < 0) return;
  const int len = U.lane_len[lid];
  double ui[B * B];
#pragma unroll
  for (int e = 0; e < B * B; ++e)
    ui[e] = __ldg(uinv + ((int64_t)w * (B * B) + e) * 32 + lane);
  double zi[B];
#pragma unroll
  for (int c = 0; c < B; ++c) zi[c] = z[(int64_t)B * row + c];
  double t[B];
  tri_rowsum<B>(U, U.slice_ptr[w], lane, len, y, t);
  double d[B];
#pragma unroll
  for (int c = 0; c < B; ++c) d[c] = zi[c] - t[c];
#pragma unroll
  for (int r = 0; r < B; ++r) {
    const double yr = block_row_dot<B>(&ui[r * B], d);
    const int64_t o = (int64_t)B * row + r;
    st_relaxed(y + o, yr);
    if (zout) {
      const double z1 = (zp && r == 0) ? zp[row] : 0.0;
      zout[o] = zp ? z1 + yr : yr;
    }
  }
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

int bilu_solve(const cprb_bilu& F, const double* r, double* zl, double* y, const double* zp,
               double* zout, cudaStream_t st) {
  // y must hold the sentinel before the U solve starts: the L kernel arms it.
  if (F.b == 3) {
    if (F.L.nslices > 0)
      k_bilu_lower<3><<<nblk((int64_t)F.L.nslices * 32, 256), 256, 0, st>>>(F.L, F.tickets, r, zl, y);
    if (F.U.nslices > 0)
      k_bilu_upper<3><<<nblk((int64_t)F.U.nslices * 32, 256), 256, 0, st>>>(F.U, F.uinv, F.tickets + 1,
                                                                            zl, y, zp, zout);
  } else if (F.b == 1) {
    if (F.L.nslices > 0)
      k_bilu_lower<1><<<nblk((int64_t)F.L.nslices * 32, 256), 256, 0, st>>>(F.L, F.tickets, r, zl, y);
    if (F.U.nslices > 0)
      k_bilu_upper<1><<<nblk((int64_t)F.U.nslices * 32, 256), 256, 0, st>>>(F.U, F.uinv, F.tickets + 1,
                                                                            zl, y, zp, zout);
  } else {
    return set_error(CPRB_EUNSUPPORTED, "BILU block size " + std::to_string(F.b) + " not supported on device");
  }
  return check_launch("bilu solve");
}

}  // namespace cprb

using namespace cprb;

// standalone bilu_apply: z = U^{-1} L^{-1} r.  work_l: n*b doubles; z doubles as y.
extern "C" int cprb_bilu_apply(const cprb_bilu* F, const double* r, double* z, double* work_l,
                               void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  // arm the L output with the sentinel (the stage-2 kernel does this inside CPR)
  const int64_t n = (int64_t)F->n * F->b;
  if (n == 0) return CPRB_OK;
  int rc;
  if (F->use_wave) {
    // the solves poll their own step-ordered outputs (the stencil solves
    // only the planes a round reads from global memory)
    if (F->use_wave == 2) {
      rc = stencil_arm(*F, st);
    } else {
      rc = fill_sentinel(F->zl_step, F->len_l, st);
      if (!rc) rc = fill_sentinel(F->y_step, F->len_u, st);
    }
    if (rc) return rc;
    rc = wave_scatter_rhs(*F, r, F->rhs_l, st);
    if (rc) return rc;
    rc = F->use_wave == 2 ? stencil_solve(*F, F->rhs_l, st) : wave_solve(*F, F->rhs_l, st);
    if (rc) return rc;
    return wave_combine(*F, nullptr, z, st);
  }
  rc = fill_sentinel(work_l, n, st);
  if (rc) return rc;
  return bilu_solve(*F, r, work_l, z, nullptr, nullptr, st);
}
