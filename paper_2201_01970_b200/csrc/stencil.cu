// K8 (structured-grid path): BILU(0) triangular solves of a natural-ordered
// 7-point nx x ny x nz grid (src/ilu.py:196-223), the SPE10-shaped Jacobians
// of every BASELINE config.
//
// Dependency structure: row (ix, iy, iz) of L needs (ix-1, iy, iz),
// (ix, iy-1, iz) and (ix, iy, iz-1); U the mirrored +x, +y, +z rows.
//
// Mapping.  One CTA owns one xy-plane and sweeps its anti-diagonals
// d = ix + iy (L ascending, U descending); warp s of the CTA holds the rows
// ix = 32 s + lane, so at diagonal d
//   * the -y neighbour is the lane's own result of diagonal d-1 (register),
//   * the -x neighbour is lane-1's result of diagonal d-1 (shuffle; lane 0
//     takes warp s-1's lane 31 from a shared-memory hand-off, the segment
//     warps step together on a named barrier),
//   * the -z neighbour is the previous plane's row at the same position.
// Planes are processed by thread-block clusters of C consecutive planes:
// inside a cluster, a plane's warp PUSHES each diagonal's results into the
// next plane's shared memory (st.async, completing the consumer's mbarrier:
// no polling, ~200-cycle DSMEM latency per hand-off); the first plane of a
// cluster polls the previous cluster's last plane in global memory
// (sentinel NaN = not yet published), after first letting that plane run
// STENCIL_LAG diagonals ahead so that the polls then succeed at once.
// The critical path is nx + ny - 1 diagonals plus one hand-off per plane.
//
// Streaming.  The factor records of a diagonal (27 doubles per L row, 37 per
// U row, one record per row) and its right-hand side are streamed into a
// shared-memory ring by a producer warp with cp.async.bulk (TMA), R
// diagonals ahead (full / empty mbarriers per slot).
//
// Arithmetic is the reference's: einsum block products ((p0 + p2) + p1) and
// reduceat row sums over the present neighbours in ascending column order,
// e0 + (e1 + e2), with absent neighbours as -0.0 (the exact additive
// identity, so the sum of the present terms is unchanged bit for bit) and
// 0.0 for a row without neighbours.
#include <cooperative_groups.h>
#include <cstdlib>

#include "device.cuh"
#include "engine.h"
#include "nvtx.h"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace cprb {

constexpr int STENCIL_SMEM = 210 * 1024;
// planes per thread-block cluster (DSMEM hand-offs): 16 (non-portable; the
// B200 places ~7 such clusters) when the device can co-schedule them, else
// 8.  Measured at C3: 8 / LAG 8 0.614 ms, 16 / LAG 4 0.528 ms per apply.
#ifndef STENCIL_CLUSTER
#define STENCIL_CLUSTER 16
#endif
#ifndef STENCIL_RZ
#define STENCIL_RZ 8                 // pushed diagonals in flight per segment
#endif
#ifndef STENCIL_LAG
#define STENCIL_LAG 4                // diagonals a cluster's first plane lets its producer lead
#endif
constexpr int STENCIL_DMAX = 1024;   // anti-diagonals per plane (nx + ny - 1) held in smem

// diagnostic (cprb_stencil_set_log): per plane [UPPER][z] x 8 u64:
// {start ns, end ns, cycles in TMA waits, cycles in plane waits, total
//  cycles, diagonals, cycles in compute, cycles in segment barriers};
// nullptr = off
__device__ unsigned long long* g_stencil_log = nullptr;
static bool g_stencil_log_on = false;  // host mirror: launch the TL variant

// doubles per row record: L 27 (-z, -y, -x blocks), U 36 + 1 pad (+x, +y, +z
// blocks, inv(U_ii)); the odd word strides keep the 16 lanes of an LDS.64
// phase on distinct bank pairs
template <bool UPPER>
__host__ __device__ constexpr int stencil_nf() { return UPPER ? 37 : 27; }

// shared-memory layout (bytes): [ring R x SLOT][zbuf S x RZ x 32 x 3 doubles]
// [mbarriers: full 16, empty 16, zfull 4*RZ, zempty 4*RZ][xh S x 2 x 3 doubles]
// [ticket 16][doff DMAX + 1 ints]
__host__ __device__ constexpr int stencil_rec_bytes(int nf, int S) { return nf * 8 * 32 * S; }
__host__ __device__ constexpr int stencil_slot_bytes(int nf, int S) {
  return ((stencil_rec_bytes(nf, S) + 24 * 32 * S) + 127) / 128 * 128;
}
__host__ __device__ constexpr int stencil_fixed_bytes(int S) {
  return S * STENCIL_RZ * 768 + 8 * (2 * 16 + 2 * 4 * STENCIL_RZ) + S * 48 + 16 +
         4 * (STENCIL_DMAX + 1);
}
__host__ __device__ constexpr int stencil_ring(int nf, int S) {
  return (STENCIL_SMEM - stencil_fixed_bytes(S)) / stencil_slot_bytes(nf, S) > 16
             ? 16
             : (STENCIL_SMEM - stencil_fixed_bytes(S)) / stencil_slot_bytes(nf, S);
}

__device__ __forceinline__ double lds_f64s(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// store 8 bytes into another CTA's shared memory, completing tx bytes on its mbarrier
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                   raddr),
               "d"(v), "r"(rbar)
               : "memory");
}
// relaxed: the slot's values were consumed (used in arithmetic) before this
// arrive, and a release here would wait for the thread's global stores
__device__ __forceinline__ void mbar_arrive_remote(uint32_t rbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_relaxed(uint32_t bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ bool stencil_is_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == CPRB_SENTINEL;
}

// poll the 3 components of a published row until none is the sentinel
__device__ __forceinline__ void stencil_wait3(const double* g, double* v) {
  int spins = 0;
  while (stencil_is_sentinel(v[0]) || stencil_is_sentinel(v[1]) || stencil_is_sentinel(v[2])) {
    if (++spins > 8) __nanosleep(20);
#ifdef STENCIL_DIAG
    if (spins > (1 << 22)) __trap();
#endif
    if (spins > (1 << 27)) __trap();  // a producer that never publishes: fail, do not hang
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (stencil_is_sentinel(v[c])) v[c] = ld_relaxed(g + c);
  }
}

#ifdef STENCIL_DIAG
// diagnostic build only (tools/build_variant.py ... -DSTENCIL_DIAG): per-warp
// progress marks in host-mapped memory and bounded waits that trap
__device__ int* g_sdiag = nullptr;
__device__ __forceinline__ void sd_mark(int kr, int t, int m, int x) {
  if (g_sdiag && blockIdx.x < 512 && (threadIdx.x & 31) == 0) {
    volatile int* e = g_sdiag + (blockIdx.x * 8 + (threadIdx.x >> 5)) * 8;
    e[0] = kr;
    e[1] = t;
    e[2] = m;
    e[3] = x;
  }
}
__device__ __forceinline__ void st_wait(uint32_t bar, uint32_t parity) {
  for (long long k = 0;; ++k) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (k == (1ll << 20) && g_sdiag && blockIdx.x < 512) {
      unsigned long long raw;
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(bar) : "memory");
      volatile int* e = g_sdiag + (blockIdx.x * 8 + (threadIdx.x >> 5)) * 8;
      e[4] = (int)(raw & 0xffffffffu);
      e[5] = (int)(raw >> 32);
      e[6] = (int)parity;
      e[7] = (int)(bar & 0xffff);
    }
    if (k > (1ll << 22)) __trap();
  }
}
#define SD_MARK(kr, t, m, x) sd_mark((kr), (t), (m), (int)(x))
#define ST_WAIT(b, p) st_wait((b), (p))
#else
#define SD_MARK(kr, t, m, x) \
  do {                       \
  } while (0)
#define ST_WAIT(b, p) mbar_wait((b), (p))
#endif

// UPPER = false: z = r - sum_{-z,-y,-x} L z             (rhs = r, out = z)
// UPPER = true : y = inv(U_ii) (z - sum_{+x,+y,+z} U y)  (rhs = z, out = y)
// rhs / out in stencil order (3 doubles per position); out must hold the
// sentinel wherever a row is polled (a cluster's first plane reads it).
// Block: S segment warps + 1 producer warp; cluster: C CTAs.
template <bool UPPER, int S, bool TL>
__global__ void __launch_bounds__(32 * (S + 1), 1)
    k_stencil(const cprb_stencil T, const double* __restrict__ rhs, double* out, int32_t* ticket) {
  constexpr int NF = stencil_nf<UPPER>();
  constexpr int R = stencil_ring(NF, S);
  static_assert(R >= 3, "stencil ring too small");
  constexpr uint32_t SLOT = stencil_slot_bytes(NF, S);
  constexpr uint32_t REC = stencil_rec_bytes(NF, S);
  constexpr int RZ = STENCIL_RZ;
  extern __shared__ __align__(128) uint8_t smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;  // 0..S-1: segment warps (the solve), S: producer (TMA)
  const int D = T.D, nx = T.nx, ny = T.ny, nz = T.nz;
  if (D > STENCIL_DMAX) __trap();
  const uint32_t s_ring = smem_u32(smem);
  const uint32_t s_zbuf = s_ring + (uint32_t)R * SLOT;
  const uint32_t s_bars = s_zbuf + (uint32_t)(S * RZ * 768);
  const uint32_t b_full = s_bars, b_empty = s_bars + 8u * 16;
  const uint32_t b_zfull = s_bars + 8u * 32, b_zempty = b_zfull + 8u * 4 * RZ;
  double* xh = reinterpret_cast<double*>(smem + (s_bars - s_ring) + 8 * (2 * 16 + 2 * 4 * RZ));
  int* s_ticket = reinterpret_cast<int*>(xh + S * 6);
  int* s_doff = s_ticket + 4;
  for (int k = threadIdx.x; k <= D; k += blockDim.x) s_doff[k] = T.doff[k];
  if (threadIdx.x == 0) {
    for (int k = 0; k < R; ++k) {
      mbar_init(b_full + 8u * k, 1);
      mbar_init(b_empty + 8u * k, S);
    }
    for (int k = 0; k < S * RZ; ++k) {
      mbar_init(b_zfull + 8u * k, 2);  // the receiver's arming + the sender's arrival
      mbar_init(b_zempty + 8u * k, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();
  pdl_wait();  // rhs comes from the previous kernel
  const double* rec_g = UPPER ? T.urec : T.lrec;
  unsigned long long* const tlog = TL ? g_stencil_log : nullptr;  // diagnostic variant only
  uint32_t g = 0;   // TMA ring uses (slot g % R, phase (g / R) & 1)
  uint32_t gz = 0;  // pushed / received diagonals (slot gz % RZ, phase (gz / RZ) & 1)
  // one round = C consecutive planes, one per rank; rounds are taken in
  // ticket order.  Persistent clusters: the grid holds only as many clusters as can be
  // resident at once (launch_stencil_s), and each takes rounds of C planes
  // until all are done, so a round only waits on an earlier round held by a
  // running cluster.  (With more clusters than fit, the hardware's placement
  // of the waiting ones does not follow ticket order: measured to deadlock.)
  int kr_last = -1;
  for (;;) {
    SD_MARK(kr_last, -1, 5, 0);
    if (threadIdx.x == 0 && rank == 0) s_ticket[0] = atomicAdd(ticket, 1);
    cluster.sync();
    const int kround = *cluster.map_shared_rank(s_ticket, 0);
    cluster.sync();                    // every rank read the ticket before the next one is taken
    if (kround * C >= nz) break;       // cluster-uniform: no rounds left
    kr_last = kround;
    const int zt = kround * C + rank;  // plane in processing order
    if (zt >= nz) continue;            // idle rank of the last round
    const int z = UPPER ? nz - 1 - zt : zt;
    const int64_t pbase = (int64_t)z * T.P;
    if (warp == S) {
      // producer: stream the records + rhs of every diagonal, R ahead
      if (lane == 0) {
        for (int t = 0; t < D; ++t, ++g) {
          const int d = UPPER ? D - 1 - t : t;
          const int o = s_doff[d], wp = s_doff[d + 1] - o;
          const uint32_t slot = g % (uint32_t)R;
          SD_MARK(kround, t, 6, g);
          if (g >= (uint32_t)R) ST_WAIT(b_empty + 8u * slot, ((g / (uint32_t)R) - 1u) & 1u);
          const uint32_t bar = b_full + 8u * slot;
          const uint32_t rb = (uint32_t)(NF * 8 * wp), hb = (uint32_t)(24 * wp);
          mbar_expect_tx(bar, rb + hb);
          bulk_g2s(s_ring + slot * SLOT, rec_g + (pbase + o) * NF, rb, bar);
          bulk_g2s(s_ring + slot * SLOT + REC, rhs + (pbase + o) * 3, hb, bar);
        }
      }
      __syncwarp();  // the warp reaches the next cluster barrier converged
      continue;
    }
    const int s = warp;
    const int ix = 32 * s + lane;
    const bool has_z = zt > 0;
    const bool z_push = rank > 0;             // -z values arrive by DSMEM push
    const bool push_next = rank + 1 < C && zt + 1 < nz;
    // the neighbouring plane this one reads (-z for L, +z for U), global copy
    const double* zplane = out + (UPPER ? pbase + T.P : pbase - T.P) * 3;
    double* oplane = out + pbase * 3;
    const uint32_t my_zbuf = s_zbuf + (uint32_t)(s * RZ * 768);
    const uint32_t my_zfull = b_zfull + 8u * (uint32_t)(s * RZ);
    const uint32_t my_zempty = b_zempty + 8u * (uint32_t)(s * RZ);
    // remote addresses: the next plane's receive ring, the previous plane's empty barriers
    const uint32_t nx_zbuf = push_next ? mapa_u32(my_zbuf, rank + 1) : 0;
    const uint32_t nx_zfull = push_next ? mapa_u32(my_zfull, rank + 1) : 0;
    const uint32_t pv_zempty = z_push ? mapa_u32(my_zempty, rank - 1) : 0;
    // rows of this warp's segment on the t-th processed diagonal, and the
    // first of them (the receive ring stores them from offset 0)
    auto seg_lo = [&](int t, int& first) -> int {
      const int d = UPPER ? D - 1 - t : t;
      const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
      const int hi = d < nx - 1 ? d : nx - 1;
      const int a = lo > 32 * s ? lo : 32 * s, e = hi < 32 * s + 31 ? hi : 32 * s + 31;
      first = a;
      return e >= a ? e - a + 1 : 0;
    };
    long long c_mbar = 0, c_z = 0, c_t0 = TL ? clock64() : 0, c_comp = 0, c_bar = 0;
    unsigned long long ns0 = 0;
    if (tlog) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0));
    // receive ring: arm the first RZ diagonals of this plane (24 bytes per row)
    if (z_push && lane == 0)
      for (int k = 0; k < RZ && k < D; ++k) {
        int f;
        mbar_expect_tx(my_zfull + 8u * ((gz + k) % RZ), (uint32_t)(24 * seg_lo(k, f)));
      }
    // a cluster's first plane: let the previous plane lead by STENCIL_LAG diagonals
    if (has_z && !z_push) {
      const int tl = STENCIL_LAG < D ? STENCIL_LAG : D - 1;
      const int d = UPPER ? D - 1 - tl : tl;
      const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
      const int hi = d < nx - 1 ? d : nx - 1;
      SD_MARK(kround, -1, 7, 0);
      if (ix >= lo && ix <= hi) {
        double v[3];
        const double* gq = zplane + 3 * (s_doff[d] + ix - lo);
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = ld_relaxed(gq + c);
        stencil_wait3(gq, v);
      }
      __syncwarp();
    }
    // first plane of a cluster: its -z values come from global memory,
    // loaded two diagonals ahead (the lag above makes them ready by then)
    const bool z_glob = has_z && !z_push;
    auto zload = [&](int t, double* v) {
      v[0] = v[1] = v[2] = 0.0;
      if (!z_glob || t >= D) return;
      const int d = UPPER ? D - 1 - t : t;
      const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
      const int hi = d < nx - 1 ? d : nx - 1;
      if (ix < lo || ix > hi) return;
      const double* gq = zplane + 3 * (s_doff[d] + ix - lo);
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = ld_relaxed(gq + c);
    };
    double zq0[3], zq1[3];
    zload(0, zq0);
    zload(1, zq1);
    double prev[3] = {0.0, 0.0, 0.0};
    for (int t = 0; t < D; ++t, ++g, ++gz) {
      const int d = UPPER ? D - 1 - t : t;
      const int lo = d - (ny - 1) > 0 ? d - (ny - 1) : 0;
      const int hi = d < nx - 1 ? d : nx - 1;
      const int o = s_doff[d];
      const bool ok = ix >= lo && ix <= hi;
      const int j = ok ? ix - lo : 0;
      const int iy = d - ix;
      const int first = lo > 32 * s ? lo : 32 * s;   // first row of this segment
      // x-neighbour of the previous diagonal: shuffle inside the warp, the
      // segment boundary from the neighbouring warp's hand-off slot
      double xv[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xv[c] = __shfl_sync(CPRB_FULL, prev[c], UPPER ? ((lane + 1) & 31) : ((lane + 31) & 31));
        if constexpr (S > 1) {
          if constexpr (UPPER) {
            if (lane == 31 && s + 1 < S) xv[c] = xh[((s + 1) * 2 + ((t - 1) & 1)) * 3 + c];
          } else {
            if (lane == 0 && s > 0) xv[c] = xh[((s - 1) * 2 + ((t - 1) & 1)) * 3 + c];
          }
        }
      }
      // neighbouring-plane values
      double zv[3] = {0.0, 0.0, 0.0};
      const uint32_t zslot = gz % (uint32_t)RZ;
      if (has_z) {
        long long tz0 = tlog ? clock64() : 0;
        if (z_push) {
          SD_MARK(kround, t, 1, gz);
          ST_WAIT(my_zfull + 8u * zslot, (gz / (uint32_t)RZ) & 1u);
          if (ok) {
            const uint32_t a = my_zbuf + zslot * 768u + 24u * (uint32_t)(ix - first);
#pragma unroll
            for (int c = 0; c < 3; ++c) zv[c] = lds_f64s(a + 8u * c);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            zv[c] = zq0[c];
            zq0[c] = zq1[c];
          }
          zload(t + 2, zq1);
          SD_MARK(kround, t, 8, 0);
          if (ok) stencil_wait3(zplane + 3 * (o + j), zv);
        }
        if (tlog) c_z += clock64() - tz0;
      }
      const uint32_t slot = g % (uint32_t)R;
      long long tw0 = tlog ? clock64() : 0;
      SD_MARK(kround, t, 2, g);
      ST_WAIT(b_full + 8u * slot, (g / (uint32_t)R) & 1u);
      if (tlog) c_mbar += clock64() - tw0;
      long long tc0 = tlog ? clock64() : 0;
      const uint32_t srec = s_ring + slot * SLOT;
      const uint32_t srhs = srec + REC;
      // neighbour presence (the plan guarantees the full in-range stencil)
      bool hx, hy;
      if constexpr (UPPER) {
        hx = ix + 1 < nx;
        hy = iy + 1 < ny;
      } else {
        hx = ix > 0;
        hy = iy > 0;
      }
      // neighbour values in ascending column order
      //   L: m0 = -z, m1 = -y, m2 = -x     U: m0 = +x, m1 = +y, m2 = +z
      const double* v0 = UPPER ? xv : zv;
      const double* v1 = prev;
      const double* v2 = UPPER ? zv : xv;
      const bool h0 = UPPER ? hx : has_z, h1 = hy, h2 = UPPER ? has_z : hx;
      const bool any = h0 || h1 || h2;
      const uint32_t rrow = srec + 8u * (uint32_t)(j * NF);
      double dd[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        double m[3][3];
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int c = 0; c < 3; ++c) m[q][c] = lds_f64s(rrow + 8u * (q * 9 + r * 3 + c));
        const double p0 = h0 ? block_row_dot<3>(m[0], v0) : -0.0;
        const double p1 = h1 ? block_row_dot<3>(m[1], v1) : -0.0;
        const double p2 = h2 ? block_row_dot<3>(m[2], v2) : -0.0;
        const double sum = any ? p0 + (p1 + p2) : 0.0;
        dd[r] = lds_f64s(srhs + 8u * (uint32_t)(j * 3 + r)) - sum;
      }
      double res[3];
      if constexpr (UPPER) {
        double ui[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) ui[e] = lds_f64s(rrow + 8u * (27 + e));
#pragma unroll
        for (int r = 0; r < 3; ++r) res[r] = block_row_dot<3>(&ui[r * 3], dd);
      } else {
#pragma unroll
        for (int r = 0; r < 3; ++r) res[r] = dd[r];
      }
      // push this diagonal to the next plane's CTA (its slot is free once
      // that CTA consumed the diagonal RZ before), publish it globally
      if (push_next) {
        if (gz >= (uint32_t)RZ) {
          SD_MARK(kround, t, 3, gz);
          ST_WAIT(my_zempty + 8u * zslot, ((gz / (uint32_t)RZ) - 1u) & 1u);
        }
        if (ok) {
          const uint32_t a = nx_zbuf + zslot * 768u + 24u * (uint32_t)(ix - first);
#pragma unroll
          for (int c = 0; c < 3; ++c) st_async_f64(a + 8u * c, res[c], nx_zfull + 8u * zslot);
        }
        // the receiver's slot phase also waits for this arrival, so a warp
        // whose segment is empty on this diagonal cannot run a phase ahead of
        // the sender's empty-wait above (which would alias its parity)
        if (lane == 0) mbar_arrive_remote(nx_zfull + 8u * zslot);
      }
      if (ok) {
        double* go = oplane + 3 * (o + j);
#pragma unroll
        for (int c = 0; c < 3; ++c) st_relaxed(go + c, res[c]);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) prev[c] = res[c];
      if constexpr (S > 1) {
        // segment-boundary hand-off for the neighbouring warp's next diagonal
        if (UPPER ? lane == 0 : lane == 31)
#pragma unroll
          for (int c = 0; c < 3; ++c) xh[(s * 2 + (t & 1)) * 3 + c] = res[c];
      }
      if (tlog) c_comp += clock64() - tc0;
      // TMA slot and received slot are free once every lane read them
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_relaxed(b_empty + 8u * slot);
        if (z_push) {
          mbar_arrive_remote(pv_zempty + 8u * zslot);
          if (t + RZ < D) {
            int f;
            mbar_expect_tx(my_zfull + 8u * zslot, (uint32_t)(24 * seg_lo(t + RZ, f)));
          }
        }
      }
      if constexpr (S > 1) {
        long long tb0 = tlog ? clock64() : 0;
        SD_MARK(kround, t, 4, 0);
        named_bar(1, 32 * S);
        if (tlog) c_bar += clock64() - tb0;
      }
    }
#ifdef STENCIL_LIGHTLOG
    // diagnostic build: plane end times only, from the production kernel
    if (!TL && g_stencil_log && lane == 0 && s == 0) {
      unsigned long long ns1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
      unsigned long long* e = g_stencil_log + ((UPPER ? 1 : 0) * 1024 + z) * 8;
      e[0] = ns1;
      e[1] = ns1;
      e[5] = (unsigned long long)D;
    }
#endif
    if (tlog && lane == 0 && s == 0) {
      unsigned long long ns1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
      unsigned long long* e = tlog + ((UPPER ? 1 : 0) * 1024 + z) * 8;
      e[0] = ns0;
      e[1] = ns1;
      e[2] = (unsigned long long)c_mbar;
      e[3] = (unsigned long long)c_z;
      e[4] = (unsigned long long)(clock64() - c_t0);
      e[5] = (unsigned long long)D;
      e[6] = (unsigned long long)c_comp;
      e[7] = (unsigned long long)c_bar;
    }
  }
  SD_MARK(kr_last, -1, 9, 0);
  cluster.sync();  // no CTA leaves while a neighbour may still push into it
}

// Per device and kernel: dynamic shared memory opt-in, the cluster size
// (16 when the device co-schedules such clusters, else 8, 4, 2) and the
// number of clusters that can be resident together.  Returns 0 on failure.
struct StencilShape {
  int C = 0, maxc = 0;
  size_t smem = 0;
};
template <bool UPPER, int S>
static StencilShape stencil_shape() {
  constexpr int NF = stencil_nf<UPPER>();
  constexpr int R = stencil_ring(NF, S);
  const size_t smem = (size_t)R * stencil_slot_bytes(NF, S) + stencil_fixed_bytes(S);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  static StencilShape cache[64];
  StencilShape& sh = cache[dev];
  if (sh.C) return sh;
  cudaFuncSetAttribute(k_stencil<UPPER, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  cudaFuncSetAttribute(k_stencil<UPPER, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  if (STENCIL_CLUSTER > 8) {
    cudaFuncSetAttribute(k_stencil<UPPER, S, false>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                         1);
    cudaFuncSetAttribute(k_stencil<UPPER, S, true>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                         1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(32 * (S + 1));
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int want = STENCIL_CLUSTER;
  if (const char* e = std::getenv("CPRB_STENCIL_CLUSTER")) want = std::atoi(e);  // test hook
  for (int c = want; c >= 2 && sh.C == 0; c /= 2) {
    at[0].val.clusterDim.x = c;
    cfg.gridDim = dim3(c);
    int m = 0;
    if (cudaOccupancyMaxActiveClusters(&m, (void*)k_stencil<UPPER, S, false>, &cfg) ==
            cudaSuccess &&
        m >= 1) {
      sh.C = c;
      sh.maxc = m;
    } else {
      cudaGetLastError();
    }
  }
  sh.smem = smem;
  return sh;
}

template <bool UPPER>
static int stencil_cluster_size(int S) {
  switch (S) {
    case 1: return stencil_shape<UPPER, 1>().C;
    case 2: return stencil_shape<UPPER, 2>().C;
    case 3: return stencil_shape<UPPER, 3>().C;
    case 4: return stencil_shape<UPPER, 4>().C;
    default: return 0;
  }
}

template <bool UPPER, int S>
static int launch_stencil_s(const cprb_stencil& T, const double* rhs, double* out, int32_t* ticket,
                            cudaStream_t st) {
  if (T.D > STENCIL_DMAX) return set_error(CPRB_EUNSUPPORTED, "stencil BILU: nx + ny too large");
  const StencilShape sh = stencil_shape<UPPER, S>();
  if (sh.C == 0) return set_error(CPRB_EDEVICE, "stencil BILU: no cluster shape fits the device");
  const int C = sh.C;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(32 * (S + 1));
  cfg.dynamicSmemBytes = sh.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  // persistent grid: at most the clusters that can be resident together
  int nclus = (T.nz + C - 1) / C;
  if (nclus > sh.maxc) nclus = sh.maxc;
  // test hook: fewer clusters, so each takes several rounds
  if (const char* e = std::getenv("CPRB_STENCIL_MAXCLUS")) {
    const int cap = std::atoi(e);
    if (cap > 0 && nclus > cap) nclus = cap;
  }
  cfg.gridDim = dim3(nclus * C);
#ifdef STENCIL_LIGHTLOG
  if (false)
#else
  if (g_stencil_log_on)
#endif
    cudaLaunchKernelEx(&cfg, k_stencil<UPPER, S, true>, T, rhs, out, ticket);
  else
    cudaLaunchKernelEx(&cfg, k_stencil<UPPER, S, false>, T, rhs, out, ticket);
  return check_launch("stencil bilu");
}

// The only rows the solves poll are those of the plane a round's first
// plane reads from global memory: the last plane of every earlier round
// (processing order zt = kC - 1).  Arm just those planes with the sentinel
// instead of the whole L / U outputs (2 x 27 MB at C3).
__global__ void k_arm_planes(double* zl, double* yu, int64_t P3, int nz, int CL, int CU,
                             int nl, int nu) {
  const int k = blockIdx.y;  // plane ordinal
  const bool upper = k >= nl;
  const int i = upper ? k - nl : k;
  const int zt = (i + 1) * (upper ? CU : CL) - 1;
  const int z = upper ? nz - 1 - zt : zt;
  double* base = (upper ? yu : zl) + (int64_t)z * P3;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < P3;
       e += (int64_t)gridDim.x * blockDim.x)
    base[e] = __longlong_as_double((long long)CPRB_SENTINEL);
}

int stencil_arm(const cprb_bilu& F, cudaStream_t st) {
  const cprb_stencil& T = F.St;
  const int CL = stencil_cluster_size<false>(T.S), CU = stencil_cluster_size<true>(T.S);
  if (CL == 0 || CU == 0) return set_error(CPRB_EDEVICE, "stencil BILU: no cluster shape fits the device");
  // round k >= 1 reads plane kC - 1 (processing order); rounds exist while kC < nz
  const int nl = (T.nz + CL - 1) / CL - 1, nu = (T.nz + CU - 1) / CU - 1;
  const int tot = nl + nu;
  if (tot <= 0) return CPRB_OK;
  const int64_t P3 = (int64_t)T.P * 3;
  const int bx = (int)((P3 + 255) / 256 < 64 ? (P3 + 255) / 256 : 64);
  k_arm_planes<<<dim3(bx, tot), 256, 0, st>>>(F.zl_step, F.y_step, P3, T.nz, CL, CU, nl, nu);
  return check_launch("stencil arm");
}

template <bool UPPER>
static int launch_stencil(const cprb_stencil& T, const double* rhs, double* out, int32_t* ticket,
                          cudaStream_t st) {
  switch (T.S) {
    case 1: return launch_stencil_s<UPPER, 1>(T, rhs, out, ticket, st);
    case 2: return launch_stencil_s<UPPER, 2>(T, rhs, out, ticket, st);
    case 3: return launch_stencil_s<UPPER, 3>(T, rhs, out, ticket, st);
    case 4: return launch_stencil_s<UPPER, 4>(T, rhs, out, ticket, st);
    default: return set_error(CPRB_EUNSUPPORTED, "stencil BILU supports nx <= 128");
  }
}

// L solve then U solve of a stencil plan.  rhsL: r in stencil order;
// F.zl_step and F.y_step must be sentinel-armed; y is left in stencil
// order in F.y_step (z = Pi zp + y gathers it through F.u_slot).
int stencil_solve(const cprb_bilu& F, const double* rhsL, cudaStream_t st) {
  NvtxRange nv("bilu_stencil_solve");
  if (F.b != 3) return set_error(CPRB_EUNSUPPORTED, "stencil BILU needs 3x3 blocks");
  if (cudaMemsetAsync(F.tickets + 4, 0, 2 * sizeof(int32_t), st) != cudaSuccess)
    return check_launch("stencil tickets");
  int rc = launch_stencil<false>(F.St, rhsL, F.zl_step, F.tickets + 4, st);
  if (rc) return rc;
  return launch_stencil<true>(F.St, F.zl_step, F.y_step, F.tickets + 5, st);
}

}  // namespace cprb

#ifdef STENCIL_DIAG
extern "C" int cprb_stencil_set_diag(int* p) {
  cudaMemcpyToSymbol(cprb::g_sdiag, &p, sizeof(p));
  return cprb::check_launch("stencil diag");
}
#endif

extern "C" int cprb_stencil_set_log(uint64_t* dev_log) {
  unsigned long long* p = (unsigned long long*)dev_log;
  cudaMemcpyToSymbol(cprb::g_stencil_log, &p, sizeof(p));
  cprb::g_stencil_log_on = p != nullptr;
  return cprb::check_launch("stencil log");
}
