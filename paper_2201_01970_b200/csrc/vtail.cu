// Persistent single-CTA V-cycle tail (src/amg.py:245-267 below level
// `tail_start`).
//
// Every coarse V-cycle level costs ~24 dependent phases (the colour sweeps
// down and up, residual + restriction, prolongation); launched one kernel per
// phase each costs a grid hand-off (~2.6 us on B200), although a coarse
// phase touches only a few hundred rows.  Here the levels >= tail_start and
// the coarse solve run in ONE CTA:
//   * the levels' vectors (b and x of every tail level, coarse b and x) live
//     in shared memory for the whole launch;
//   * the static data (row lengths, diagonals, columns, values, aggregate
//     maps, coarse-inverse rows) is packed on the host into one stream of
//     <= slot-sized chunks in phase order, and a producer warp streams it with
//     bulk-async (TMA) copies into a 4-deep shared-memory ring, ahead of the
//     consumers (mbarrier full/empty hand-off) -- from the very start of the
//     launch, overlapping the previous kernel through PDL;
//   * a phase is shared-memory reads, FP64 arithmetic and one named barrier
//     over the consumer warps.
// Arithmetic is the launched kernels' (k_sweep, k_resid_restrict,
// k_prolong, k_dense_mv) operation for operation: bitwise equal.
#include <cstdlib>

#include "device.cuh"
#include "engine.h"
#include "nvtx.h"
#include "tma.cuh"

namespace cprb {

constexpr int VT_CONSUMER_WARPS = 8;
constexpr int VT_THREADS = 32 * (VT_CONSUMER_WARPS + 1);
constexpr int VT_NSLOT = 4;
enum { VT_SWEEP = 1, VT_RR = 3, VT_COARSE = 4, VT_PROLONG = 5 };

__device__ __forceinline__ const uint8_t* al16(const uint8_t* p) {
  return reinterpret_cast<const uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
}

// GS row (k_sweep): acc = sum_m a_m x[c_m] sequentially from 0.0; entries
// are fetched 8 at a time (all shared-memory loads of a group in flight
// before the first product)
__device__ __forceinline__ double vt_gsrow(const uint16_t* cols, const double* vals, int stride,
                                           int t, int len, const double* x) {
  double acc = 0.0;
  for (int m0 = 0; m0 < len; m0 += 8) {
    int c[8];
    double v[8], xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (m0 + k < len) {
        c[k] = cols[(m0 + k) * stride + t];
        v[k] = vals[(m0 + k) * stride + t];
      }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (m0 + k < len) xv[k] = x[c[k]];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (m0 + k < len) acc = acc + v[k] * xv[k];
  }
  return acc;
}

// reduceat row (k_resid_restrict): a0 + pairwise(rest), the n < 8 part from
// -0.0 (segsum_masked / rr_row_stream) for len <= 129, segsum_rt beyond;
// entries fetched 8 at a time
__device__ __forceinline__ double vt_rrow(const uint16_t* cols, const double* vals, int stride, int t,
                                          int len, const double* x) {
  if (len <= 0) return 0.0;
  if (len > 129) {
    auto e = [&](int m) -> double { return vals[m * stride + t] * x[cols[m * stride + t]]; };
    return segsum_rt(e, len);
  }
  const int n = len - 1;
  const int nf = n >= 8 ? (n & ~7) : 0;
  double a0 = 0.0, s = -0.0, r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = 0.0;
  for (int p0 = 0; p0 < len; p0 += 8) {
    int c[8];
    double v[8], e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (p0 + k < len) {
        c[k] = cols[(p0 + k) * stride + t];
        v[k] = vals[(p0 + k) * stride + t];
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

__device__ unsigned long long* g_vtail_log = nullptr;  // diagnostic: per-phase end times

__device__ __forceinline__ unsigned long long vt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct VtArgs {
  int32_t nl;                   // levels including the coarsest
  int32_t start, nphases, nchunks, slot;
  const int4* phases;           // {type, level, colour/zg, first chunk}, nphases + 1
  const int4* chunks;           // {phase, byte offset, bytes, rows}
  const uint8_t* stream;
  const int32_t* vec;           // smem double offsets: b_l = vec[2l], x_l = vec[2l+1]
  const double* b_in;           // global b of level `start` (written by the launched restriction)
  double* x_out;                // global x of level `start` (read by the launched prolongation)
  int32_t n_start, n_coarse, vec_len;
};

constexpr int VT_NCT = VT_CONSUMER_WARPS * 32;

// the launch's dynamic shared memory, addressed by OFFSETS from this symbol
// so that every access compiles to LDS/STS (pointers carried through
// integer address arithmetic otherwise degrade to generic loads)
extern __shared__ __align__(128) uint8_t vt_smem[];

// one chunk of phase ph (all consumer threads)
__device__ __forceinline__ void vt_chunk(const int4 ph, uint32_t rec_off, const int* svec, int nl,
                                         int tid) {
  double* vec = reinterpret_cast<double*>(vt_smem);
  const int warp = tid >> 5, lane = tid & 31;
  const int4 hdr = *reinterpret_cast<const int4*>(vt_smem + rec_off);
  const int cnt = hdr.x, W = hdr.y, first = hdr.z;
  const uint32_t o = rec_off + 16;
  auto A16 = [](uint32_t v) -> uint32_t { return (v + 15u) & ~15u; };
  const int l = ph.y;
  if (ph.x == VT_SWEEP) {
    double* x = vec + svec[2 * l + 1];
    const double* b = vec + svec[2 * l];
    const uint32_t o_diag = A16(o + 4u * cnt);
    const uint32_t o_cols = A16(o_diag + 8u * cnt);
    const uint32_t o_vals = A16(o_cols + 2u * W * cnt);
    const int* lens = reinterpret_cast<const int*>(vt_smem + o);
    const double* diag = reinterpret_cast<const double*>(vt_smem + o_diag);
    const uint16_t* cols = reinterpret_cast<const uint16_t*>(vt_smem + o_cols);
    const double* vals = reinterpret_cast<const double*>(vt_smem + o_vals);
    for (int t = tid; t < cnt; t += VT_NCT) {
      const double acc = vt_gsrow(cols, vals, cnt, t, lens[t], x);
      x[first + t] = (b[first + t] - acc) / diag[t];
    }
  } else if (ph.x == VT_RR) {
    const double* x = vec + svec[2 * l + 1];
    const double* b = vec + svec[2 * l];
    double* bc = vec + svec[2 * (l + 1)];
    const uint32_t o_lens = A16(o + 4u * cnt);
    const uint32_t o_outs = A16(o_lens + 4u * cnt);
    const uint32_t o_cols = A16(o_outs + 4u * (cnt / 2));
    const uint32_t o_vals = A16(o_cols + 2u * W * cnt);
    const int* rows = reinterpret_cast<const int*>(vt_smem + o);
    const int* lens = reinterpret_cast<const int*>(vt_smem + o_lens);
    const int* outs = reinterpret_cast<const int*>(vt_smem + o_outs);
    const uint16_t* cols = reinterpret_cast<const uint16_t*>(vt_smem + o_cols);
    const double* vals = reinterpret_cast<const double*>(vt_smem + o_vals);
    for (int t0 = 0; t0 < cnt; t0 += VT_NCT) {  // lanes 2I, 2I+1 are neighbours in a warp
      const int t = t0 + tid;
      double res = 0.0;
      if (t < cnt) {
        const int row = rows[t];
        if (row >= 0) res = b[row] - vt_rrow(cols, vals, cnt, t, lens[t], x);
      }
      const double other = __shfl_down_sync(CPRB_FULL, res, 1);
      if (t < cnt && (t & 1) == 0) {
        const int out = outs[t >> 1];
        if (out >= 0) bc[out] = (0.0 + res) + other;
      }
    }
  } else if (ph.x == VT_PROLONG) {
    double* x = vec + svec[2 * l + 1];
    const double* xc = vec + svec[2 * (l + 1) + 1];
    const int* aggp = reinterpret_cast<const int*>(vt_smem + o);
    for (int t = tid; t < cnt; t += VT_NCT) x[first + t] = x[first + t] + xc[aggp[t]];
  } else {  // VT_COARSE: rows of inv(A_L) times the coarse b (k_dense_mv order)
    const double* cb = vec + svec[2 * (nl - 1)];
    double* cx = vec + svec[2 * (nl - 1) + 1];
    const double* rowsd = reinterpret_cast<const double*>(vt_smem + o);
    for (int r = warp; r < cnt; r += VT_CONSUMER_WARPS) {
      const double* row = rowsd + (size_t)r * W;
      double sacc = 0.0;
      for (int cc = lane; cc < W; cc += 32) sacc = sacc + row[cc] * cb[cc];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sacc = sacc + __shfl_xor_sync(CPRB_FULL, sacc, o);
      if (lane == 0) cx[first + r] = sacc;
    }
  }
}

__device__ __forceinline__ void vt_bar() { asm volatile("bar.sync 1, %0;" ::"r"(VT_NCT) : "memory"); }

// the prologue shared by both streaming modes: phase table / offsets into
// shared memory, PDL wait, b of the first tail level in
__device__ __forceinline__ void vt_prologue(const VtArgs& a, double* vec, int4* sph, int* svec,
                                            int tid) {
  for (int i = tid; i <= a.nphases; i += VT_NCT) sph[i] = __ldg(a.phases + i);
  for (int i = tid; i < 2 * a.nl; i += VT_NCT) svec[i] = __ldg(a.vec + i);
  unsigned long long* const tlog = g_vtail_log;
  if (tlog && tid == 0) tlog[0] = vt_now();
  pdl_wait();
  if (tlog && tid == 0) tlog[1] = vt_now();
  vt_bar();
  double* b0 = vec + svec[2 * a.start];
  for (int i = tid; i < a.n_start; i += VT_NCT) b0[i] = a.b_in[i];
  vt_bar();
}

__device__ __forceinline__ void vt_epilogue(const VtArgs& a, const double* vec, const int* svec,
                                            int tid) {
  const double* x0 = vec + svec[2 * a.start + 1];
  for (int i = tid; i < a.n_start; i += VT_NCT) a.x_out[i] = x0[i];
}

// MODE 0: a producer warp streams chunks with cp.async.bulk into a 4-slot
// mbarrier ring.  MODE 1: the consumer threads themselves copy chunk c + 2
// with 16-byte cp.async while chunk c is processed (3 buffers, one barrier
// per chunk) -- many small requests in flight instead of one bulk copy.
template <int MODE>
__global__ void __launch_bounds__(VT_THREADS, 1) k_vtail(const VtArgs a) {
  double* vec = reinterpret_cast<double*>(vt_smem);
  const uint32_t ring_off = (uint32_t)(((a.vec_len * 8) + 127) & ~127);
  const uint32_t bars_off = ring_off + (uint32_t)(VT_NSLOT * a.slot);
  const uint32_t ring = smem_u32(vt_smem) + ring_off;
  const uint32_t bars = smem_u32(vt_smem) + bars_off;
  const uint32_t b_full = bars, b_empty = bars + 8u * VT_NSLOT;
  int4* sph = reinterpret_cast<int4*>(vt_smem + bars_off + 8 * 2 * VT_NSLOT);
  int* svec = reinterpret_cast<int*>(sph + a.nphases + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  unsigned long long* const tlog = g_vtail_log;
  if constexpr (MODE == 0) {
    if (threadIdx.x == 0) {
      for (int k = 0; k < VT_NSLOT; ++k) {
        mbar_init(b_full + 8u * k, 1);
        mbar_init(b_empty + 8u * k, VT_CONSUMER_WARPS);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_trigger();
    if (warp == VT_CONSUMER_WARPS) {
      // producer: the static stream does not depend on earlier kernels, so
      // it starts before the PDL wait
      if (lane == 0) {
        for (int c = 0; c < a.nchunks; ++c) {
          const uint32_t s = (uint32_t)(c % VT_NSLOT);
          if (c >= VT_NSLOT) mbar_wait(b_empty + 8u * s, (uint32_t)((c / VT_NSLOT) - 1) & 1u);
          const int4 ch = __ldg(a.chunks + c);
          mbar_expect_tx(b_full + 8u * s, (uint32_t)ch.z);
          bulk_g2s(ring + s * (uint32_t)a.slot, a.stream + (int64_t)ch.y * 16, (uint32_t)ch.z,
                   b_full + 8u * s);
        }
      }
      return;
    }
    vt_prologue(a, vec, sph, svec, tid);
    int c = 0;
    for (int p = 0; p < a.nphases; ++p) {
      const int4 ph = sph[p];
      const int c1 = sph[p + 1].w;
      for (; c < c1; ++c) {
        const uint32_t s = (uint32_t)(c % VT_NSLOT);
        if (tlog && tid == 0) tlog[2 + a.nphases + 3 * c] = vt_now();
        mbar_wait(b_full + 8u * s, (uint32_t)(c / VT_NSLOT) & 1u);
        if (tlog && tid == 0) tlog[3 + a.nphases + 3 * c] = vt_now();
        vt_chunk(ph, ring_off + s * (uint32_t)a.slot, svec, a.nl, tid);
        if (tlog && tid == 0) tlog[4 + a.nphases + 3 * c] = vt_now();
        __syncwarp();
        if (lane == 0) mbar_arrive(b_empty + 8u * s);
      }
      vt_bar();
      if (tlog && tid == 0) tlog[2 + p] = vt_now();
    }
    vt_epilogue(a, vec, svec, tid);
  } else {
    pdl_trigger();
    if (warp == VT_CONSUMER_WARPS) return;
    constexpr int NB = 3;  // chunk buffers (uses 3 of the ring's slots)
    auto issue = [&](int c) {
      if (c >= a.nchunks) {
        asm volatile("cp.async.commit_group;" ::: "memory");
        return;
      }
      const int4 ch = __ldg(a.chunks + c);
      const uint32_t dst = ring + (uint32_t)(c % NB) * (uint32_t)a.slot;
      const uint8_t* src = a.stream + (int64_t)ch.y * 16;
      for (int i = tid; i < ch.z / 16; i += VT_NCT)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * i),
                     "l"(src + 16 * (int64_t)i)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // static chunks do not depend on earlier kernels: start before the PDL wait
    issue(0);
    issue(1);
    vt_prologue(a, vec, sph, svec, tid);
    int c = 0;
    for (int p = 0; p < a.nphases; ++p) {
      const int4 ph = sph[p];
      const int c1 = sph[p + 1].w;
      for (; c < c1; ++c) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        vt_bar();  // chunk c visible to all; everyone is done with chunk c - 1
        issue(c + 2);
        vt_chunk(ph, ring_off + (uint32_t)(c % NB) * (uint32_t)a.slot, svec, a.nl, tid);
      }
      if (tlog && tid == 0) tlog[2 + p] = vt_now();
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    vt_bar();
    vt_epilogue(a, vec, svec, tid);
  }
}

static int vt_attr_done[64];

int launch_vtail(const cprb_amg& h, cudaStream_t st) {
  NvtxRange nv("amg_vcycle_tail");
  VtArgs a;
  a.nl = h.nlevels;
  a.start = h.tail_start;
  a.nphases = h.tail_nphases;
  a.nchunks = h.tail_nchunks;
  a.slot = h.tail_slot;
  a.phases = reinterpret_cast<const int4*>(h.tail_phases);
  a.chunks = reinterpret_cast<const int4*>(h.tail_chunks);
  a.stream = h.tail_stream;
  a.vec = h.tail_vec;
  const cprb_amg_level& L = h.levels[h.tail_start];
  a.b_in = L.b;
  a.x_out = L.x;
  a.n_start = L.n;
  a.n_coarse = h.n_coarse;
  a.vec_len = h.tail_vec_len;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !vt_attr_done[dev]) {
    cudaFuncSetAttribute(k_vtail<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_vtail<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    vt_attr_done[dev] = 1;
  }
  // the stream is read once per V-cycle: keep it resident in the persisting
  // L2 carve-out so the level-0 traffic of the next cycle does not evict it
  if (dev >= 0 && dev < 64 && vt_attr_done[dev] == 1) {
    int maxp = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    size_t want = (size_t)h.tail_stream_bytes;
    if (maxp > 0) {
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want < (size_t)maxp ? want : (size_t)maxp);
    }
    cudaGetLastError();
    vt_attr_done[dev] = 2;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(VT_THREADS);
  cfg.dynamicSmemBytes = (size_t)h.tail_smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeAccessPolicyWindow;
  at[1].val.accessPolicyWindow.base_ptr = (void*)h.tail_stream;
  at[1].val.accessPolicyWindow.num_bytes = (size_t)h.tail_stream_bytes;
  at[1].val.accessPolicyWindow.hitRatio = 1.0f;
  at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = getenv("CPRB_TAIL_NOPERSIST") ? 1 : 2;
  static const int mode = getenv("CPRB_TAIL_MODE") ? atoi(getenv("CPRB_TAIL_MODE")) : 1;
  if (mode == 0) cudaLaunchKernelEx(&cfg, k_vtail<0>, a);
  else cudaLaunchKernelEx(&cfg, k_vtail<1>, a);
  return check_launch("v-cycle tail");
}

}  // namespace cprb

extern "C" int cprb_vtail_set_log(uint64_t* dev_log) {
  unsigned long long* p = (unsigned long long*)dev_log;
  cudaMemcpyToSymbol(cprb::g_vtail_log, &p, sizeof(p));
  return cprb::check_launch("vtail log");
}
