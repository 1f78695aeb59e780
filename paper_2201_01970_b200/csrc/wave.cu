// K8 (fast path): chunked-wavefront BILU(0) triangular solves.
//
// Rows are split into contiguous chunks of two dependency bandwidths (two
// xy-planes for the natural-ordered 7-point grid), so a chunk only depends on
// the chunk before it (L) / after it (U).  One persistent CTA owns a chunk
// (ticket order = dependency order, so waiting is deadlock free) and walks
// its rows level by level ("steps", <= 128 rows, one row per thread).
//   * Step records are warp-sliced (ilu.wave_plan): each consumer warp
//     streams only its own 32-row slice of every step with cp.async.bulk
//     (TMA) into its private DEPTH-slot shared-memory ring, refilled by the
//     warp itself as soon as it is done with a slot.  No warp waits for
//     another warp's staging, so the natural skew between warps of a
//     wavefront does not eat the lookahead.
//   * There is no barrier per step: a dependency computed <= DINT steps ago
//     in this chunk is read from a shared-memory result ring guarded by a
//     per-slot step flag (release/acquire at CTA scope); a warp-progress
//     word bounds the skew so that no ring slot is overwritten early.
//   * Anything else (the previous chunk, older rows) is polled from global
//     memory, where exported results are published with a relaxed store
//     (sentinel NaN = not ready).
// Arithmetic is the reference's: einsum block products ((p0 + p2) + p1),
// reduceat row sums (src/ilu.py:97-107, :216-222).
#include <cstdlib>

#include "device.cuh"
#include "tma.cuh"
#include "engine.h"
#include "nvtx.h"

namespace cprb {

constexpr int WAVE_THREADS = 128;  // == ilu.WAVE_WMAX: rows per step == threads per CTA
constexpr int WAVE_NWARPS = WAVE_THREADS / 32;
constexpr int WAVE_DEPTH = 2;      // per-warp stage ring (steps in flight)
constexpr int WAVE_DINT = 3;       // == ilu.WAVE_DINT: ring-served dependency distance
constexpr int WAVE_RING = 32;      // result ring (steps)
// a warp may write step k only when every warp finished step k - SKEW, so a
// ring slot is never overwritten while a reader of its previous occupant
// (at most DINT steps younger) is pending
constexpr int WAVE_SKEW = WAVE_RING - WAVE_DINT;
constexpr int WAVE_KMAX = 3;       // == ilu.WAVE_KMAX: streamed (register) path
constexpr int WAVE_META = 320;     // step metadata staged in shared memory per chunk
// lens[] word: low 16 bits = dependency count; bit 30 = the row's value must be
// published to global memory (another chunk or an older-than-DINT row reads it)
constexpr int WAVE_LEN_MASK = 0xFFFF;
constexpr int WAVE_EXPORT = 1 << 30;
// bit 29 = a row of another rank's slab reads this row (slab-partitioned
// solve): its value is also stored into that rank's output array (peer
// memory over NVLink, same offset)
constexpr int WAVE_REMOTE = 1 << 29;

__device__ __forceinline__ void st_relaxed_sys(double* p, double v) {
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v))
               : "memory");
}

// diagnostic timeline (cprb_wave_set_log): [UPPER][chunk][local step] ->
// %globaltimer when row position 0 of the step finished; nullptr = off
__device__ unsigned long long* g_wave_log = nullptr;

static bool g_wave_log_on = false;  // host mirror of g_wave_log != nullptr

constexpr int WAVE_LOG_STEPS = 512;
constexpr int WAVE_LOG_CHUNKS = 256;

struct StepMeta {
  int64_t off;      // stream byte offset of the step (warp slice q at off + q * bytes)
  int64_t rhs_off;  // rhs double offset (row position p at rhs_off + p * b)
  int32_t bytes;    // bytes of one warp slice
  int32_t rhs_bytes;
  int32_t w;
  int32_t k;
};

__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int lds_acquire_s32(uint32_t a) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_release_s32(uint32_t a, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ bool is_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == CPRB_SENTINEL;
}

// Global dependencies may have been published by a peer GPU (slab path:
// st.relaxed.sys into this rank's buffer), so they are read at system scope;
// on one GPU this is the same L2 access as a gpu-scope relaxed load.
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return __longlong_as_double((long long)v);
}

// all B components polled concurrently until none is the sentinel
template <int B>
__device__ __forceinline__ void wait_block(const double* g, double* v) {
  int spins = 0;
  while (true) {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < B; ++c) ok &= !is_sentinel(v[c]);
    if (ok) return;
    if (++spins > 8) __nanosleep(20);
    if (spins > (1 << 27)) __trap();  // a producer that never publishes: fail, do not hang
#pragma unroll
    for (int c = 0; c < B; ++c)
      if (is_sentinel(v[c])) v[c] = ld_relaxed_sys(g + c);
  }
}

struct Ring {
  uint32_t vals;  // smem: RING * WAVE_THREADS * B doubles
  uint32_t flag;  // smem: RING * WAVE_THREADS ints (global step index held)
};

__device__ __forceinline__ int lds_relaxed_s32(uint32_t a) {
  int v;
  asm volatile("ld.relaxed.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// ring slot of an in-chunk dependency (code q = (diff-1) * THREADS + position)
__device__ __forceinline__ uint32_t ring_slot(int k, int q, int& dstep) {
  const int diff = q / WAVE_THREADS + 1;
  const int pos = q - (diff - 1) * WAVE_THREADS;
  dstep = k - diff;
  return (uint32_t)((dstep % WAVE_RING) * WAVE_THREADS + pos);
}

// value of an in-chunk dependency (code q = (diff-1) * THREADS + position)
template <int B>
__device__ __forceinline__ void ring_value(const Ring ring, int k, int q, double* v) {
  const int diff = q / WAVE_THREADS + 1;
  const int pos = q - (diff - 1) * WAVE_THREADS;
  const int dstep = k - diff;
  const uint32_t slot = (uint32_t)((dstep % WAVE_RING) * WAVE_THREADS + pos);
  while (lds_acquire_s32(ring.flag + 4u * slot) != dstep) {
  }
#pragma unroll
  for (int c = 0; c < B; ++c) v[c] = lds_f64(ring.vals + 8u * (slot * B + c));
}

// Field addresses of lane l in a warp slice (layout: ilu.wave_plan):
//   int32 rows[32], lens[32], aux[32], codes[K][32]; f64 vals[K][BB][32], uinv[BB][32]
// `base` is a shared (space = 1) or generic (space = 0) address.
template <int B, bool UPPER, int K>
__device__ __forceinline__ void row_fast(uint32_t sblk, uint32_t srhs, int l, int len,
                                         const Ring ring, int k, const double* glob,
                                         double* res, int kr) {
  // K: register extent (the largest dependency count served); kr: the
  // step's record layout (its K); rows with len < K are predicated, and the
  // reduceat order of segsum_masked depends on len only
  constexpr int BB = B * B;
  constexpr int KA = K > 0 ? K : 1;
  int code[KA];
  double mv[KA][BB];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    code[m] = (m < len) ? lds_s32(sblk + 4u * (96 + 32 * m + l)) : 0;
#pragma unroll
    for (int e = 0; e < BB; ++e)
      mv[m][e] = (m < len) ? lds_f64(sblk + 4u * (96 + 32 * kr) + 8u * ((m * BB + e) * 32 + l)) : 0.0;
  }
  double rh[B];
#pragma unroll
  for (int r = 0; r < B; ++r) rh[r] = lds_f64(srhs + 8u * (l * B + r));
  double dv[KA][B];
  // global dependencies: issue all loads first, then take the ring values,
  // then finish the polls
#pragma unroll
  for (int m = 0; m < K; ++m)
    if (m < len && code[m] >= 0)
#pragma unroll
      for (int c = 0; c < B; ++c) dv[m][c] = ld_relaxed_sys(glob + (int64_t)code[m] + c);
  // in-chunk dependencies: poll all flags with relaxed loads, then one
  // acquire fence before reading the values (instead of one acquire each)
  uint32_t rslot[KA];
#pragma unroll
  for (int m = 0; m < K; ++m)
    if (m < len && code[m] < 0) {
      int dstep;
      rslot[m] = ring_slot(k, -code[m] - 1, dstep);
      while (lds_relaxed_s32(ring.flag + 4u * rslot[m]) != dstep) {
      }
    }
  asm volatile("fence.acq_rel.cta;" ::: "memory");
#pragma unroll
  for (int m = 0; m < K; ++m) {
    if (m < len) {
      if (code[m] < 0) {
#pragma unroll
        for (int c = 0; c < B; ++c) dv[m][c] = lds_f64(ring.vals + 8u * (rslot[m] * B + c));
      } else {
        wait_block<B>(glob + (int64_t)code[m], dv[m]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < B; ++c) dv[m][c] = 0.0;
    }
  }
  double d[B];
#pragma unroll
  for (int r = 0; r < B; ++r) {
    if constexpr (K > 0) {
      double p[K];
#pragma unroll
      for (int m = 0; m < K; ++m) p[m] = block_row_dot<B>(&mv[m][r * B], dv[m]);
      d[r] = rh[r] - segsum_masked<K>(p, len);
    } else {
      d[r] = rh[r] - 0.0;
    }
  }
  if constexpr (UPPER) {
    const uint32_t a_ui = sblk + 4u * (96 + 32 * kr) + 8u * (kr * BB * 32);
    double ui[BB];
#pragma unroll
    for (int e = 0; e < BB; ++e) ui[e] = lds_f64(a_ui + 8u * (e * 32 + l));
#pragma unroll
    for (int r = 0; r < B; ++r) res[r] = block_row_dot<B>(&ui[r * B], d);
  } else {
#pragma unroll
    for (int r = 0; r < B; ++r) res[r] = d[r];
  }
}

// general path (rows with more than KMAX dependencies; random test matrices):
// reads the warp slice straight from global memory
template <int B, bool UPPER>
__device__ __noinline__ void row_general(const uint8_t* blk, int K, const double* rhs, int l,
                                         int len, const Ring ring, int k, const double* glob,
                                         double* res) {
  constexpr int BB = B * B;
  const int32_t* codes = reinterpret_cast<const int32_t*>(blk) + 96;
  const double* vals = reinterpret_cast<const double*>(blk + 4 * (96 + 32 * K));
  double d[B];
#pragma unroll
  for (int r = 0; r < B; ++r) {
    auto f = [&](int m) -> double {
      const int code = codes[32 * m + l];
      double dv[B];
      if (code < 0) {
        ring_value<B>(ring, k, -code - 1, dv);
      } else {
#pragma unroll
        for (int c = 0; c < B; ++c) dv[c] = ld_relaxed_sys(glob + (int64_t)code + c);
        wait_block<B>(glob + (int64_t)code, dv);
      }
      double mr[B];
#pragma unroll
      for (int c = 0; c < B; ++c) mr[c] = vals[(size_t)(m * BB + r * B + c) * 32 + l];
      return block_row_dot<B>(mr, dv);
    };
    d[r] = rhs[l * B + r] - segsum_rt(f, len);
  }
  if constexpr (UPPER) {
    const double* uinv = vals + (size_t)K * BB * 32;
    double ui[BB];
#pragma unroll
    for (int e = 0; e < BB; ++e) ui[e] = uinv[(size_t)e * 32 + l];
#pragma unroll
    for (int r = 0; r < B; ++r) res[r] = block_row_dot<B>(&ui[r * B], d);
  } else {
#pragma unroll
    for (int r = 0; r < B; ++r) res[r] = d[r];
  }
}

// UPPER = false: z = r - sum L z         (z published in L-step order)
// UPPER = true : y = Uinv (z - sum U y)   (y published in U-step order)
// out_step must hold the sentinel (armed by the caller) wherever it is polled.
template <int B, bool UPPER, bool STG, bool TL>
__global__ void __launch_bounds__(WAVE_THREADS, 1)
    k_wave(const cprb_wave W, const double* __restrict__ rhs_steps, double* out_step,
           int32_t* ticket, double* peer_out) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // diagnostic timeline, compiled in only for the TL variant
  unsigned long long* const tlog = TL ? g_wave_log : nullptr;
  __shared__ StepMeta s_meta[WAVE_META];
  __shared__ __align__(8) uint64_t s_full[WAVE_NWARPS][WAVE_DEPTH];
  __shared__ int s_prog[WAVE_NWARPS];
  __shared__ int s_chunk;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int slot_bytes = W.stage_max + W.rhs_max;  // one warp slice + its rhs block
  const uint32_t my_stage = smem_u32(smem_raw) + (uint32_t)(warp * WAVE_DEPTH * slot_bytes);
  const uint32_t my_full = smem_u32(&s_full[warp][0]);
  // dynamic smem: per-warp stage rings | result ring | ring flags
  double* s_ring = reinterpret_cast<double*>(smem_raw + (size_t)WAVE_NWARPS * WAVE_DEPTH * slot_bytes);
  int* s_flag = reinterpret_cast<int*>(s_ring + WAVE_RING * WAVE_THREADS * B);
  for (int i = tid; i < WAVE_RING * WAVE_THREADS; i += blockDim.x) s_flag[i] = -1;
  if (lane == 0) {
    for (int d = 0; d < WAVE_DEPTH; ++d) mbar_init(my_full + 8u * d, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const Ring ring{smem_u32(s_ring), smem_u32(s_flag)};
  const uint32_t sprog = smem_u32(s_prog);
  uint32_t nis = 0, ncons = 0;  // this warp's slices issued / consumed (all chunks)

  while (true) {
    __syncthreads();  // previous chunk fully consumed (ring, meta, progress)
    if (tid == 0) {
      const int c = atomicAdd(ticket, 1);
      if (c == W.nchunks + (int)gridDim.x - 1) atomicExch(ticket, 0);
      s_chunk = c;
    }
    __syncthreads();
    const int c = s_chunk;
    if (c >= W.nchunks) break;
    const int s0 = W.chunk_step[c];
    const int s1 = W.chunk_step[c + 1];
    // STG: every chunk's step metadata fits in shared memory (checked by the
    // host), so the per-step global fallback is compiled out
    const bool staged = STG || (s1 - s0) <= WAVE_META;
    if (staged) {
      for (int k = s0 + tid; k < s1; k += blockDim.x) {
        StepMeta m;
        m.off = W.step_off[k];
        m.rhs_off = W.rhs_off[k];
        m.bytes = W.step_bytes[k];
        m.rhs_bytes = W.rhs_bytes[k];
        m.w = W.step_w[k];
        m.k = W.step_k[k];
        s_meta[k - s0] = m;
      }
    }
    if (tid < WAVE_NWARPS) s_prog[tid] = s0 - 1;
    __syncthreads();
    auto meta = [&](int k) -> StepMeta {
      if (STG || staged) return s_meta[k - s0];
      StepMeta m;
      m.off = W.step_off[k];
      m.rhs_off = W.rhs_off[k];
      m.bytes = W.step_bytes[k];
      m.rhs_bytes = W.rhs_bytes[k];
      m.w = W.step_w[k];
      m.k = W.step_k[k];
      return m;
    };
    // this warp streams its slice of a step iff it has rows there and the
    // step is on the register path
    auto streamed = [&](const StepMeta& m) { return m.w > warp * 32 && m.k <= WAVE_KMAX; };
    int ik = s0;  // next step to consider for issue
    auto top_up = [&]() {
      if (lane == 0) {
        while (ik < s1 && nis - ncons < (uint32_t)WAVE_DEPTH) {
          const StepMeta m = meta(ik);
          if (streamed(m)) {
            const int sl = nis % WAVE_DEPTH;
            const uint32_t dst = my_stage + (uint32_t)(sl * slot_bytes);
            const int rows_here = min(32, m.w - warp * 32);
            const uint32_t rb = (uint32_t)((rows_here * B * 8 + 15) & ~15);
            mbar_expect_tx(my_full + 8u * sl, (uint32_t)m.bytes + rb);
            bulk_g2s(dst, W.stream + m.off + (int64_t)warp * m.bytes, (uint32_t)m.bytes,
                     my_full + 8u * sl);
            bulk_g2s(dst + (uint32_t)W.stage_max, rhs_steps + m.rhs_off + warp * 32 * B, rb,
                     my_full + 8u * sl);
            ++nis;
          }
          ++ik;
        }
      }
      // no __syncwarp: the other lanes only need the mbarrier, not lane 0
    };
    top_up();
    for (int k = s0; k < s1; ++k) {
      const StepMeta mk = meta(k);
      // skew bound (see WAVE_SKEW), checked every 16th step for the next 16
      if (((k - s0) & 15) == 0 && k + 15 - WAVE_SKEW >= s0) {
        const int need = k + 15 - WAVE_SKEW;
#pragma unroll
        for (int q = 0; q < WAVE_NWARPS; ++q)
          while (lds_acquire_s32(sprog + 4u * q) < need) {
            __nanosleep(100);  // a throttled lead warp is off the critical path
          }
      }
      const int pos = warp * 32 + lane;
      if (mk.w > warp * 32) {
        const bool fast = mk.k <= WAVE_KMAX;
        uint32_t sblk = 0, srhs = 0;
        if (fast) {
          const int sl = ncons % WAVE_DEPTH;
          mbar_wait(my_full + 8u * sl, (ncons / WAVE_DEPTH) & 1);
          sblk = my_stage + (uint32_t)(sl * slot_bytes);
          srhs = sblk + (uint32_t)W.stage_max;
        }
        if (pos < mk.w) {
          const uint8_t* gblk = W.stream + mk.off + (int64_t)warp * mk.bytes;
          const double* grhs = rhs_steps + mk.rhs_off + warp * 32 * B;
          const int lenw = fast ? lds_s32(sblk + 4u * (32 + lane))
                                : reinterpret_cast<const int32_t*>(gblk)[32 + lane];
          const int len = lenw & WAVE_LEN_MASK;
          double res[B];
          if (fast) {
            // one instantiation for every streamed step (smaller hot loop)
            row_fast<B, UPPER, WAVE_KMAX>(sblk, srhs, lane, len, ring, k, out_step, res, mk.k);
          } else {
            // the out-of-line path gets its own buffer so that res itself
            // never needs an address (stays in registers on the fast path)
            double rg[B];
            row_general<B, UPPER>(gblk, mk.k, grhs, lane, len, ring, k, out_step, rg);
#pragma unroll
            for (int r = 0; r < B; ++r) res[r] = rg[r];
          }
          const uint32_t slot = (uint32_t)((k % WAVE_RING) * WAVE_THREADS + pos);
#pragma unroll
          for (int r = 0; r < B; ++r) sts_f64(ring.vals + 8u * (slot * B + r), res[r]);
          sts_release_s32(ring.flag + 4u * slot, k);
          // publish in step order: one contiguous, coalesced row block per
          // warp (the next chunk's polls, the U solve's input and the final
          // combine all read this array)
          {
            double* o = out_step + mk.rhs_off + (int64_t)pos * B;
#pragma unroll
            for (int r = 0; r < B; ++r) st_relaxed(o + r, res[r]);
            if (peer_out && (lenw & WAVE_REMOTE)) {
              double* q = peer_out + mk.rhs_off + (int64_t)pos * B;
#pragma unroll
              for (int r = 0; r < B; ++r) st_relaxed_sys(q + r, res[r]);
            }
          }
          if (TL && pos == 0 && tlog && c < WAVE_LOG_CHUNKS && k - s0 < WAVE_LOG_STEPS) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tt));
            tlog[((UPPER ? 1 : 0) * WAVE_LOG_CHUNKS + c) * WAVE_LOG_STEPS + (k - s0)] = tt;
          }
        }
        __syncwarp();
        if (fast) {
          ++ncons;
          top_up();  // refill the slot just released
        }
      }
      // progress is published per group of 4 steps (the skew check reads it
      // every 4th step with a 3-step margin)
      if (((k - s0) & 3) == 3 || k + 1 == s1) {  // (read every 16th step with margin)
        __syncwarp();
        if (lane == 0) sts_release_s32(sprog + 4u * warp, k);
      }
    }
  }
}

// scatter r into the L plan's step order (slots) for standalone applies
__global__ void k_scatter_slots(int n, int b, const int32_t* __restrict__ slot,
                                const double* __restrict__ r, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < b; ++c) out[slot[i] + c] = r[(int64_t)b * i + c];
}

static size_t wave_smem(const cprb_wave& W, int b) {
  return (size_t)WAVE_NWARPS * WAVE_DEPTH * (size_t)(W.stage_max + W.rhs_max) +
         (size_t)WAVE_RING * WAVE_THREADS * (8 * b + 4);
}

template <int B, bool UPPER>
static int launch_wave(const cprb_wave& W, const double* rhs_steps, double* out_step,
                       int32_t* ticket, cudaStream_t st, double* peer_out = nullptr) {
  // per-device caches: the SM count and the dynamic-smem opt-in are
  // properties of the device the launch goes to
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  static int num_sms_dev[64] = {0};
  if (!num_sms_dev[dev])
    cudaDeviceGetAttribute(&num_sms_dev[dev], cudaDevAttrMultiProcessorCount, dev);
  const int num_sms = num_sms_dev[dev];
  if (W.nchunks <= 0) return CPRB_OK;
  const int grid = W.nchunks < num_sms ? W.nchunks : num_sms;
  const size_t smem = wave_smem(W, B);
  // set once per instantiation (the attribute call can serialise against
  // running work; concurrent slab solves on other streams must not wait)
  static size_t smem_set_dev[64] = {0};
  size_t& smem_set = smem_set_dev[dev];
  if (smem > smem_set) {
    cudaFuncSetAttribute(k_wave<B, UPPER, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_wave<B, UPPER, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_wave<B, UPPER, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_wave<B, UPPER, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set = smem;
  }
  const bool stg = W.max_chunk_steps > 0 && W.max_chunk_steps <= WAVE_META;
  if (g_wave_log_on) {
    if (stg) k_wave<B, UPPER, true, true><<<grid, WAVE_THREADS, smem, st>>>(W, rhs_steps, out_step, ticket, peer_out);
    else k_wave<B, UPPER, false, true><<<grid, WAVE_THREADS, smem, st>>>(W, rhs_steps, out_step, ticket, peer_out);
  } else {
    if (stg) k_wave<B, UPPER, true, false><<<grid, WAVE_THREADS, smem, st>>>(W, rhs_steps, out_step, ticket, peer_out);
    else k_wave<B, UPPER, false, false><<<grid, WAVE_THREADS, smem, st>>>(W, rhs_steps, out_step, ticket, peer_out);
  }
  return check_launch("wave solve");
}

// U-plan rhs from the L solve's step-ordered output: rhs_u[u_slot[i] + c] =
// zl_step[l_slot[i] + c] (one coalesced gather pass between the solves)
__global__ void k_l_to_u(int n, int b, const int32_t* __restrict__ ls, const int32_t* __restrict__ us,
                         const double* __restrict__ z, double* __restrict__ rhs_u) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int a = __ldg(ls + i), d = __ldg(us + i);
    for (int c = 0; c < b; ++c) rhs_u[d + c] = z[a + c];
  }
}

// L solve -> permute -> U solve.  rhsL: r in L-step order; F.zl_step and
// F.y_step must be sentinel-armed; y is left in U-step order in F.y_step.
int wave_solve(const cprb_bilu& F, const double* rhsL, cudaStream_t st) {
  NvtxRange nv("bilu_wave_solve");
  int rc;
  const int blocks = (F.n + 255) / 256 < 4 * 148 ? (F.n + 255) / 256 : 4 * 148;
  if (F.b == 3) {
    rc = launch_wave<3, false>(F.Lw, rhsL, F.zl_step, F.tickets + 2, st);
    if (rc) return rc;
    launch_pdl(k_l_to_u, blocks, 256, 0, st, F.n, 3, F.l_slot, F.u_slot, (const double*)F.zl_step,
               F.rhs_u);
    rc = launch_wave<3, true>(F.Uw, F.rhs_u, F.y_step, F.tickets + 3, st);
  } else if (F.b == 1) {
    rc = launch_wave<1, false>(F.Lw, rhsL, F.zl_step, F.tickets + 2, st);
    if (rc) return rc;
    launch_pdl(k_l_to_u, blocks, 256, 0, st, F.n, 1, F.l_slot, F.u_slot, (const double*)F.zl_step,
               F.rhs_u);
    rc = launch_wave<1, true>(F.Uw, F.rhs_u, F.y_step, F.tickets + 3, st);
  } else {
    return set_error(CPRB_EUNSUPPORTED, "wave BILU supports block sizes 1 and 3");
  }
  return rc;
}

// z = Pi zp + y (zp == nullptr: z = y), y gathered from U-step order
__global__ void k_wave_combine(int n, int b, const int32_t* __restrict__ us,
                               const double* __restrict__ y_step, const double* __restrict__ zp,
                               double* __restrict__ z) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int d = __ldg(us + i);
    for (int c = 0; c < b; ++c) {
      const double y = y_step[d + c];
      // src/cpr.py:184-186: prolong(zp) has zeros off the pressure slot
      z[(int64_t)b * i + c] = zp ? ((c == 0 ? zp[i] : 0.0) + y) : y;
    }
  }
}

int wave_combine(const cprb_bilu& F, const double* zp, double* z, cudaStream_t st) {
  const int blocks = (F.n + 255) / 256 < 4 * 148 ? (F.n + 255) / 256 : 4 * 148;
  launch_pdl(k_wave_combine, blocks, 256, 0, st, F.n, F.b, F.u_slot, (const double*)F.y_step, zp,
             z);
  return check_launch("wave combine");
}

}  // namespace cprb

extern "C" int cprb_wave_set_log(uint64_t* dev_log) {
  unsigned long long* p = (unsigned long long*)dev_log;
  cudaMemcpyToSymbol(cprb::g_wave_log, &p, sizeof(p));
  cprb::g_wave_log_on = p != nullptr;

  return cprb::check_launch("wave log");
}

namespace cprb {

int wave_scatter_rhs(const cprb_bilu& F, const double* r, double* rhsL, cudaStream_t st) {
  k_scatter_slots<<<(F.n + 255) / 256, 256, 0, st>>>(F.n, F.b, F.l_slot, r, rhsL);
  return check_launch("scatter slots");
}

}  // namespace cprb

// ---- slab-partitioned BILU (paper_2201_01970_b200/partition.py SlabBilu) ----
__global__ void k_fill_sentinel_idx(int n, int b, const int32_t* __restrict__ idx, double* base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int c = 0; c < b; ++c) base[(int64_t)idx[i] + c] = cprb::sentinel();
}

using namespace cprb;

extern "C" {

int cprb_wave_solve_part(const cprb_bilu* F, int32_t upper, int32_t chunk0, int32_t nchunks,
                         const double* rhs_steps, double* out_step, double* peer_out,
                         int32_t* ticket, void* stream) {
  cprb_wave W = upper ? F->Uw : F->Lw;
  if (chunk0 < 0 || nchunks < 0 || chunk0 + nchunks > W.nchunks)
    return set_error(CPRB_EINVAL, "chunk range out of bounds");
  W.chunk_step += chunk0;
  W.nchunks = nchunks;
  cudaStream_t st = (cudaStream_t)stream;
  if (F->b == 3)
    return upper ? launch_wave<3, true>(W, rhs_steps, out_step, ticket, st, peer_out)
                 : launch_wave<3, false>(W, rhs_steps, out_step, ticket, st, peer_out);
  if (F->b == 1)
    return upper ? launch_wave<1, true>(W, rhs_steps, out_step, ticket, st, peer_out)
                 : launch_wave<1, false>(W, rhs_steps, out_step, ticket, st, peer_out);
  return set_error(CPRB_EUNSUPPORTED, "wave BILU supports block sizes 1 and 3");
}

int cprb_l_to_u_rows(const cprb_bilu* F, int32_t row0, int32_t nrows, const double* zl_step,
                     double* rhs_u, void* stream) {
  if (nrows <= 0) return CPRB_OK;
  const int blocks = (nrows + 255) / 256 < 4 * 148 ? (nrows + 255) / 256 : 4 * 148;
  k_l_to_u<<<blocks, 256, 0, (cudaStream_t)stream>>>(nrows, F->b, F->l_slot + row0,
                                                     F->u_slot + row0, zl_step, rhs_u);
  return check_launch("l to u rows");
}

int cprb_wave_combine_rows(const cprb_bilu* F, int32_t row0, int32_t nrows, const double* y_step,
                           const double* zp, double* z, void* stream) {
  if (nrows <= 0) return CPRB_OK;
  const int blocks = (nrows + 255) / 256 < 4 * 148 ? (nrows + 255) / 256 : 4 * 148;
  k_wave_combine<<<blocks, 256, 0, (cudaStream_t)stream>>>(nrows, F->b, F->u_slot + row0, y_step,
                                                           zp, z);
  return check_launch("wave combine rows");
}

int cprb_fill_sentinel_idx(int64_t n, int32_t b, const int32_t* idx, double* base, void* stream) {
  if (n <= 0) return CPRB_OK;
  k_fill_sentinel_idx<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>((int)n, b,
                                                                                   idx, base);
  return check_launch("fill sentinel idx");
}

// stage-2 residual of this rank's rows written straight into the L plan's
// step order, arming the rows' L and U output slots (cprb_cpr_finish's
// fused kernel for a row range: slots are the plan's, offset by row0)
int cprb_stage2_residual_steps(const cprb_sell* A, const cprb_bilu* F, int32_t row0,
                               const double* zp, const double* r, double* rhs_l, double* zl_step,
                               double* y_step, void* stream) {
  return bsr_op(2, *A, F->b, zp, r, rhs_l, nullptr, zl_step, (cudaStream_t)stream,
                F->l_slot + row0, y_step, F->l_slot + row0, F->u_slot + row0);
}

}  // extern "C"
