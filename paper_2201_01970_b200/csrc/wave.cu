// K8 (fast path): chunked-wavefront BILU(0) triangular solves.
//
// Rows are split into contiguous chunks of two dependency bandwidths (two
// xy-planes for the natural-ordered 7-point grid), so a chunk only depends on
// the chunk before it (L) / after it (U).  One persistent CTA owns a chunk
// (ticket order = dependency order, so waiting is deadlock free) and walks
// its rows level by level ("steps", <= 128 rows):
//   * a producer warp streams every step's record (blocks, column codes) and
//     right-hand side into a shared-memory stage ring with cp.async.bulk (TMA)
//     on full/empty mbarrier pairs, DEPTH steps ahead of the consumers;
//   * consumer thread t owns row position t of every step.  There is NO
//     barrier per step: a dependency computed <= DINT steps ago in this chunk
//     is read from a shared-memory result ring guarded by a per-slot step
//     flag (release/acquire at CTA scope), so a row starts as soon as its own
//     inputs exist and neighbouring positions pipeline across steps;
//   * anything else (the previous chunk, older rows) is polled from global
//     memory, where every result is published with a relaxed store
//     (sentinel NaN = not ready).
// Critical path ~ (#levels x one smem hand-off) + (#chunks x one L2 hop).
// Arithmetic is the reference's: einsum block products ((p0 + p2) + p1),
// reduceat row sums (src/ilu.py:97-107, :216-222).
#include "device.cuh"
#include "engine.h"

namespace cprb {

constexpr int WAVE_THREADS = 128;  // consumers == wmax of the plan (rows per step)
constexpr int WAVE_BLOCK = WAVE_THREADS + 32;  // + one producer warp
constexpr int WAVE_DEPTH = 4;      // stage ring (steps in flight)
constexpr int WAVE_DINT = 3;       // == ilu.WAVE_DINT: ring-served dependency distance
constexpr int WAVE_RING = 8;       // result ring; >= DEPTH + DINT (no overwrite while read)
constexpr int WAVE_KPRE = 3;       // external dependencies prefetched per row
constexpr int WAVE_META = 1024;    // step metadata staged in shared memory per chunk
// lens[] word: low 16 bits = dependency count; bit 30 = the row's value must be
// published to global memory (another chunk or an older-than-DINT row reads it)
constexpr int WAVE_LEN_MASK = 0xFFFF;
constexpr int WAVE_EXPORT = 1 << 30;
static_assert(WAVE_RING >= WAVE_DEPTH + WAVE_DINT, "result ring too small");

// diagnostic timeline (cprb_wave_set_log): [UPPER][chunk][local step] ->
// %globaltimer when row position 0 of the step finished; nullptr = off
__device__ unsigned long long* g_wave_log = nullptr;
constexpr int WAVE_LOG_STEPS = 512;
constexpr int WAVE_LOG_CHUNKS = 256;

struct StepMeta {
  int64_t off;      // stream byte offset
  int64_t rhs_off;  // rhs double offset
  int32_t bytes;
  int32_t rhs_bytes;
  int32_t w;
  int32_t k;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_s32(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct WaveSmem {
  uint8_t* stage;     // DEPTH * stage_max
  double* rhs;        // DEPTH * rhs_max/8
  double* ring;       // RING * WAVE_THREADS * B
  int* flag;          // RING * WAVE_THREADS: global step index held by the ring slot
  StepMeta* meta;     // WAVE_META
  uint64_t* full;     // DEPTH (TMA landed)
  uint64_t* empty;    // DEPTH (all consumer warps done with the slot)
  int* chunk;         // 1
};

template <int B>
struct Pre {
  double v[WAVE_KPRE][B];
};

__device__ __forceinline__ bool is_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == CPRB_SENTINEL;
}

// issue (do not wait for) the loads of a row's cross-chunk dependencies
template <int B>
__device__ __forceinline__ void wave_prefetch(const int32_t* codes, int Wp, int t, int len,
                                              const double* glob, Pre<B>& p) {
#pragma unroll
  for (int m = 0; m < WAVE_KPRE; ++m) {
    if (m < len) {
      const int code = codes[m * Wp + t];
      if (code >= 0) {
#pragma unroll
        for (int c = 0; c < B; ++c) p.v[m][c] = ld_relaxed(glob + (int64_t)B * code + c);
      }
    }
  }
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
#pragma unroll
    for (int c = 0; c < B; ++c)
      if (is_sentinel(v[c])) v[c] = ld_relaxed(g + c);
  }
}

struct RingRef {
  const double* vals;  // RING * WAVE_THREADS * B
  const int* flag;     // RING * WAVE_THREADS
  int k;               // global step index of the row being computed
};

template <int B>
__device__ __forceinline__ void dep_value(int code, int m, const RingRef& ring, const double* glob,
                                          const Pre<B>& p, double* v) {
  if (code < 0) {
    const int q = -code - 1;
    const int diff = q / WAVE_THREADS + 1;
    const int pos = q - (diff - 1) * WAVE_THREADS;
    const int dstep = ring.k - diff;
    const int slot = (dstep % WAVE_RING) * WAVE_THREADS + pos;
    int spins = 0;
    while (ld_acquire_s32(ring.flag + slot) != dstep) {
      if (++spins > 64) __nanosleep(8);
    }
    const double* s = ring.vals + (int64_t)slot * B;
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = s[c];
    return;
  }
  const double* g = glob + (int64_t)B * code;
  if (m < WAVE_KPRE) {
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = p.v[m][c];
  } else {
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = ld_relaxed(g + c);
  }
  wait_block<B>(g, v);
}

template <int B, int K>
__device__ __forceinline__ void wave_rowsum_fixed(const int32_t* codes, const double* vals, int Wp,
                                                  int t, const RingRef& ring, const double* glob,
                                                  const Pre<B>& pre, double* tsum) {
  double v[K][B];
#pragma unroll
  for (int m = 0; m < K; ++m) dep_value<B>(codes[m * Wp + t], m, ring, glob, pre, v[m]);
#pragma unroll
  for (int r = 0; r < B; ++r) {
    double p[K];
#pragma unroll
    for (int m = 0; m < K; ++m) {
      double mr[B];
#pragma unroll
      for (int c = 0; c < B; ++c) mr[c] = vals[(int64_t)(m * B * B + r * B + c) * Wp + t];
      p[m] = block_row_dot<B>(mr, v[m]);
    }
    tsum[r] = segsum_fixed<K>(p);
  }
}

template <int B>
__device__ __forceinline__ void wave_rowsum_generic(const int32_t* codes, const double* vals,
                                                    int Wp, int t, int len, const RingRef& ring,
                                                    const double* glob, const Pre<B>& pre,
                                                    double* tsum) {
#pragma unroll
  for (int r = 0; r < B; ++r) {
    auto f = [&](int m) -> double {
      double v[B], mr[B];
      dep_value<B>(codes[m * Wp + t], m, ring, glob, pre, v);
#pragma unroll
      for (int c = 0; c < B; ++c) mr[c] = vals[(int64_t)(m * B * B + r * B + c) * Wp + t];
      return block_row_dot<B>(mr, v);
    };
    tsum[r] = segsum_rt(f, len);
  }
}

__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
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

// One row of a step with at most K (<= WAVE_KPRE) dependencies, all operands
// addressed explicitly in shared memory (no generic loads, no local memory).
// Returns the row's result in res[B].
template <int B, bool UPPER, int K>
__device__ __forceinline__ void lean_row(uint32_t sblk, uint32_t srhs, uint32_t sring,
                                         uint32_t sflag, int Wp, int t, int k, int len,
                                         const double* glob, const Pre<B>& pre, double* res) {
  constexpr int BB = B * B;
  constexpr int KA = K > 0 ? K : 1;  // array extent
  const uint32_t a_codes = sblk + 12u * Wp;
  const uint32_t a_vals = sblk + (uint32_t)(12 + 4 * K) * Wp;
  int code[KA];
  double mv[KA][BB];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    code[m] = (m < len) ? lds_s32(a_codes + 4u * (m * Wp + t)) : 0;
#pragma unroll
    for (int e = 0; e < BB; ++e)
      mv[m][e] = (m < len) ? lds_f64(a_vals + 8u * ((m * BB + e) * Wp + t)) : 0.0;
  }
  double rh[B];
#pragma unroll
  for (int r = 0; r < B; ++r) rh[r] = lds_f64(srhs + 8u * (t * B + r));
  double ui[UPPER ? BB : 1];
  if constexpr (UPPER) {
    const uint32_t a_ui = a_vals + 8u * (K * BB * Wp);
#pragma unroll
    for (int e = 0; e < BB; ++e) ui[e] = lds_f64(a_ui + 8u * (e * Wp + t));
  }
  double dv[KA][B];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    if (m < len) {
      const int cd = code[m];
      if (cd < 0) {
        const int q = -cd - 1;
        const int diff = q / WAVE_THREADS + 1;
        const int pos = q - (diff - 1) * WAVE_THREADS;
        const int dstep = k - diff;
        const uint32_t slot = (uint32_t)((dstep % WAVE_RING) * WAVE_THREADS + pos);
        while (lds_acquire_s32(sflag + 4u * slot) != dstep) {
        }
#pragma unroll
        for (int c = 0; c < B; ++c) dv[m][c] = lds_f64(sring + 8u * (slot * B + c));
      } else {
#pragma unroll
        for (int c = 0; c < B; ++c) dv[m][c] = pre.v[m][c];
        wait_block<B>(glob + (int64_t)B * cd, dv[m]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < B; ++c) dv[m][c] = 0.0;
    }
  }
  if constexpr (K > 0) {
#pragma unroll
    for (int r = 0; r < B; ++r) {
      double p[K];
#pragma unroll
      for (int m = 0; m < K; ++m) p[m] = block_row_dot<B>(&mv[m][r * B], dv[m]);
      const double ts = segsum_masked<K>(p, len);
      rh[r] = rh[r] - ts;
    }
  } else {
#pragma unroll
    for (int r = 0; r < B; ++r) rh[r] = rh[r] - 0.0;
  }
  if constexpr (UPPER) {
#pragma unroll
    for (int r = 0; r < B; ++r) res[r] = block_row_dot<B>(&ui[r * B], rh);
  } else {
#pragma unroll
    for (int r = 0; r < B; ++r) res[r] = rh[r];
  }
}

// UPPER = false: z = r - sum L z   (publishes exported z rows, copies z into
//                the U plan's rhs order via aux slots; y must be armed with
//                the sentinel by the caller)
// UPPER = true : y = Uinv (z - sum U y); final = z1 + y
template <int B, bool UPPER>
__global__ void __launch_bounds__(WAVE_BLOCK, 1)
    k_wave(const cprb_wave W, const double* __restrict__ rhs_steps, double* out_nat,
           double* __restrict__ next_rhs, double* __restrict__ arm, const double* __restrict__ zp,
           double* __restrict__ final_out, int32_t* ticket) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int BB = B * B;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const bool producer = warp == WAVE_THREADS / 32;
  const int stage_max = W.stage_max, rhs_max = W.rhs_max;
  WaveSmem S;
  S.stage = smem_raw;
  S.rhs = reinterpret_cast<double*>(smem_raw + (size_t)WAVE_DEPTH * stage_max);
  S.ring = S.rhs + (size_t)WAVE_DEPTH * (rhs_max / 8);
  S.flag = reinterpret_cast<int*>(S.ring + (size_t)WAVE_RING * WAVE_THREADS * B);
  S.meta = reinterpret_cast<StepMeta*>(S.flag + WAVE_RING * WAVE_THREADS);
  S.full = reinterpret_cast<uint64_t*>(S.meta + WAVE_META);
  S.empty = S.full + WAVE_DEPTH;
  S.chunk = reinterpret_cast<int*>(S.empty + WAVE_DEPTH);
  if (tid == 0) {
    for (int d = 0; d < WAVE_DEPTH; ++d) {
      mbar_init(&S.full[d], 1);
      mbar_init(&S.empty[d], WAVE_THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < WAVE_RING * WAVE_THREADS; i += blockDim.x) S.flag[i] = -1;
  __syncthreads();
  uint32_t g = 0;  // steps consumed by this CTA (slot = g % DEPTH, phase = (g / DEPTH) & 1)
  const RingRef ring0{S.ring, S.flag, 0};
  const uint32_t sring = smem_u32(S.ring);
  const uint32_t sflag = smem_u32(S.flag);

  while (true) {
    if (tid == 0) {
      const int c = atomicAdd(ticket, 1);
      if (c == W.nchunks + (int)gridDim.x - 1) atomicExch(ticket, 0);
      *S.chunk = c;
    }
    __syncthreads();
    const int c = *S.chunk;
    if (c >= W.nchunks) break;
    const int s0 = W.chunk_step[c];
    const int s1 = W.chunk_step[c + 1];
    const bool staged = (s1 - s0) <= WAVE_META;
    if (staged) {
      for (int k = s0 + tid; k < s1; k += blockDim.x) {
        StepMeta m;
        m.off = W.step_off[k];
        m.rhs_off = W.rhs_off[k];
        m.bytes = W.step_bytes[k];
        m.rhs_bytes = W.rhs_bytes[k];
        m.w = W.step_w[k];
        m.k = W.step_k[k];
        S.meta[k - s0] = m;
      }
    }
    __syncthreads();  // metadata visible; previous chunk fully consumed
    auto meta = [&](int k) -> StepMeta {
      if (staged) return S.meta[k - s0];
      StepMeta m;
      m.off = W.step_off[k];
      m.rhs_off = W.rhs_off[k];
      m.bytes = W.step_bytes[k];
      m.rhs_bytes = W.rhs_bytes[k];
      m.w = W.step_w[k];
      m.k = W.step_k[k];
      return m;
    };
    if (producer) {
      if ((tid & 31) == 0) {
        for (int k = s0; k < s1; ++k) {
          const uint32_t gg = g + (uint32_t)(k - s0);
          const int st = gg % WAVE_DEPTH;
          const long long t_pw = clock64();
          if (gg >= WAVE_DEPTH) mbar_wait(&S.empty[st], ((gg / WAVE_DEPTH) - 1) & 1);
          if (g_wave_log && c == 0 && k - s0 < WAVE_LOG_STEPS) {
            const long long t_is = clock64();
            g_wave_log[((UPPER ? 1 : 0) * WAVE_LOG_CHUNKS + 206) * WAVE_LOG_STEPS + (k - s0)] = (unsigned long long)t_is;
            g_wave_log[((UPPER ? 1 : 0) * WAVE_LOG_CHUNKS + 208) * WAVE_LOG_STEPS + (k - s0)] = (unsigned long long)(t_is - t_pw);
          }
          const StepMeta m = meta(k);
          mbar_expect_tx(&S.full[st], (uint32_t)(m.bytes + m.rhs_bytes));
          bulk_g2s(S.stage + (size_t)st * stage_max, W.stream + m.off, m.bytes, &S.full[st]);
          bulk_g2s(S.rhs + (size_t)st * (rhs_max / 8), rhs_steps + m.rhs_off, m.rhs_bytes,
                   &S.full[st]);
        }
      }
      __syncwarp();
    } else {
      const int pos = tid;  // row position of every step handled by this thread
      long long cyc[5] = {0, 0, 0, 0, 0};
      long long tlast = clock64();
      Pre<B> pre;
      {
        const int st = g % WAVE_DEPTH;
        mbar_wait(&S.full[st], (g / WAVE_DEPTH) & 1);
        const int w = meta(s0).w;
        const int Wp = (w + 3) & ~3;
        const int32_t* rows = reinterpret_cast<const int32_t*>(S.stage + (size_t)st * stage_max);
        if (pos < w) wave_prefetch<B>(rows + 3 * Wp, Wp, pos, rows[Wp + pos] & WAVE_LEN_MASK, out_nat, pre);
      }
      for (int k = s0; k < s1; ++k) {
        const uint32_t gk = g + (uint32_t)(k - s0);
        const int st = gk % WAVE_DEPTH;
        const bool tl = g_wave_log != nullptr;
        auto tmark = [&](int which) {
          if (tl) {
            const long long now = clock64();
            if (which > 0) cyc[which - 1] += now - tlast;
            tlast = now;
          }
        };
        tmark(0);
        mbar_wait(&S.full[st], (gk / WAVE_DEPTH) & 1);
        if (tid == 0 && g_wave_log && c == 0 && k - s0 < WAVE_LOG_STEPS)
          g_wave_log[((UPPER ? 1 : 0) * WAVE_LOG_CHUNKS + 207) * WAVE_LOG_STEPS + (k - s0)] = (unsigned long long)clock64();
        tmark(1);
        const uint8_t* blk = S.stage + (size_t)st * stage_max;
        const StepMeta mk = meta(k);
        const int w = mk.w, K = mk.k;
        const int Wp = (w + 3) & ~3;
        const int32_t* rows = reinterpret_cast<const int32_t*>(blk);
        const int32_t* lens = rows + Wp;
        const int32_t* aux = lens + Wp;
        const int32_t* codes = aux + Wp;
        const double* vals = reinterpret_cast<const double*>(blk + (size_t)(12 + 4 * K) * Wp);
        const double* uinv = vals + (size_t)K * BB * Wp;
        const double* rhs = S.rhs + (size_t)st * (rhs_max / 8);
        Pre<B> nxt;
        tmark(2);
        if (pos < w && K <= WAVE_KPRE) {
          // lean path (all rows of 7-point-type factors)
          const uint32_t sblk = smem_u32(blk);
          const uint32_t srhs = smem_u32(rhs);
          const int row = lds_s32(sblk + 4u * pos);
          const int lenw = lds_s32(sblk + 4u * (Wp + pos));
          const int len = lenw & WAVE_LEN_MASK;
          const bool publish = (lenw & WAVE_EXPORT) || (UPPER && !final_out);
          const int ns = UPPER ? 0 : lds_s32(sblk + 4u * (2 * Wp + pos));
          double z1 = 0.0;
          if (UPPER && zp) z1 = zp[row];
          double res[B];
          switch (K) {
            case 0: lean_row<B, UPPER, 0>(sblk, srhs, sring, sflag, Wp, pos, k, len, out_nat, pre, res); break;
            case 1: lean_row<B, UPPER, 1>(sblk, srhs, sring, sflag, Wp, pos, k, len, out_nat, pre, res); break;
            case 2: lean_row<B, UPPER, 2>(sblk, srhs, sring, sflag, Wp, pos, k, len, out_nat, pre, res); break;
            default: lean_row<B, UPPER, 3>(sblk, srhs, sring, sflag, Wp, pos, k, len, out_nat, pre, res); break;
          }
          tmark(3);
          const uint32_t slot = (uint32_t)((k % WAVE_RING) * WAVE_THREADS + pos);
#pragma unroll
          for (int r = 0; r < B; ++r) sts_f64(sring + 8u * (slot * B + r), res[r]);
          sts_release_s32(sflag + 4u * slot, k);
          if (publish) {
#pragma unroll
            for (int r = 0; r < B; ++r) st_relaxed(out_nat + (int64_t)B * row + r, res[r]);
          }
          if constexpr (!UPPER) {
#pragma unroll
            for (int r = 0; r < B; ++r) next_rhs[(int64_t)ns + r] = res[r];
          } else {
            if (final_out) {
#pragma unroll
              for (int r = 0; r < B; ++r)
                final_out[(int64_t)B * row + r] = zp ? ((r == 0 ? z1 : 0.0) + res[r]) : res[r];
            }
          }
        } else if (pos < w) {
          RingRef ring = ring0;
          ring.k = k;
          const int row = rows[pos];
          const int lenw = lens[pos];
          const int len = lenw & WAVE_LEN_MASK;
          const bool publish = (lenw & WAVE_EXPORT) || (UPPER && !final_out);
          double z1 = 0.0;
          if (UPPER && zp) z1 = zp[row];
          double ts[B];
          switch (len) {
            case 0:
#pragma unroll
              for (int r = 0; r < B; ++r) ts[r] = 0.0;
              break;
            case 1: wave_rowsum_fixed<B, 1>(codes, vals, Wp, pos, ring, out_nat, pre, ts); break;
            case 2: wave_rowsum_fixed<B, 2>(codes, vals, Wp, pos, ring, out_nat, pre, ts); break;
            case 3: wave_rowsum_fixed<B, 3>(codes, vals, Wp, pos, ring, out_nat, pre, ts); break;
            default: wave_rowsum_generic<B>(codes, vals, Wp, pos, len, ring, out_nat, pre, ts); break;
          }
          double res[B];
          if constexpr (!UPPER) {
#pragma unroll
            for (int r = 0; r < B; ++r) res[r] = rhs[pos * B + r] - ts[r];
          } else {
            double d[B], ui[BB];
#pragma unroll
            for (int r = 0; r < B; ++r) d[r] = rhs[pos * B + r] - ts[r];
#pragma unroll
            for (int e = 0; e < BB; ++e) ui[e] = uinv[(size_t)e * Wp + pos];
#pragma unroll
            for (int r = 0; r < B; ++r) res[r] = block_row_dot<B>(&ui[r * B], d);
          }
          tmark(3);
          const int slot = (k % WAVE_RING) * WAVE_THREADS + pos;
          double* ring_slot = S.ring + (size_t)slot * B;
#pragma unroll
          for (int r = 0; r < B; ++r) ring_slot[r] = res[r];
          st_release_s32(S.flag + slot, k);
          if (publish) {
#pragma unroll
            for (int r = 0; r < B; ++r) st_relaxed(out_nat + (int64_t)B * row + r, res[r]);
          }
          if constexpr (!UPPER) {
            const int ns = aux[pos];
#pragma unroll
            for (int r = 0; r < B; ++r) next_rhs[(int64_t)ns + r] = res[r];
          } else {
            if (final_out) {
#pragma unroll
              for (int r = 0; r < B; ++r)
                final_out[(int64_t)B * row + r] = zp ? ((r == 0 ? z1 : 0.0) + res[r]) : res[r];
            }
          }
        }
        if (tid == 0 && g_wave_log && c < WAVE_LOG_CHUNKS && k - s0 < WAVE_LOG_STEPS) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tt));
          g_wave_log[((UPPER ? 1 : 0) * WAVE_LOG_CHUNKS + c) * WAVE_LOG_STEPS + (k - s0)] = tt;
        }
        // after this step's row is published: issue the next step's
        // cross-chunk dependency loads (if its record has landed), so their
        // L2 round trip overlaps the global stores and the step hand-off
        if (k + 1 < s1) {
          const uint32_t g1 = gk + 1;
          const int st1 = g1 % WAVE_DEPTH;
          mbar_wait(&S.full[st1], (g1 / WAVE_DEPTH) & 1);
          const int w1 = meta(k + 1).w;
          const int Wp1 = (w1 + 3) & ~3;
          const int32_t* r1 = reinterpret_cast<const int32_t*>(S.stage + (size_t)st1 * stage_max);
          if (pos < w1) wave_prefetch<B>(r1 + 3 * Wp1, Wp1, pos, r1[Wp1 + pos] & WAVE_LEN_MASK, out_nat, nxt);
        }
        tmark(4);
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&S.empty[st]);  // this warp is done with the slot
        pre = nxt;
        tmark(5);
      }
      if (g_wave_log && c < WAVE_LOG_CHUNKS && tid < 128) {
        // cycles per phase summed over the chunk, slot [UPPER][200 + phase][chunk*... ] pos-major
        for (int q = 0; q < 5; ++q)
          g_wave_log[((UPPER ? 1 : 0) * WAVE_LOG_CHUNKS + 200 + q) * WAVE_LOG_STEPS + (c % 4) * 128 + tid] =
              (unsigned long long)cyc[q];
      }
    }
    g += (uint32_t)(s1 - s0);
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
  return (size_t)WAVE_DEPTH * (W.stage_max + W.rhs_max) + (size_t)WAVE_RING * WAVE_THREADS * b * 8 +
         (size_t)WAVE_RING * WAVE_THREADS * 4 + sizeof(StepMeta) * WAVE_META +
         2 * WAVE_DEPTH * 8 + 16;
}

template <int B, bool UPPER>
static int launch_wave(const cprb_wave& W, const double* rhs_steps, double* out_nat, double* next_rhs,
                       double* arm, const double* zp, double* final_out, int32_t* ticket,
                       cudaStream_t st) {
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t smem = wave_smem(W, B);
  cudaFuncSetAttribute(k_wave<B, UPPER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = W.nchunks < num_sms ? W.nchunks : num_sms;
  k_wave<B, UPPER><<<grid, WAVE_BLOCK, smem, st>>>(W, rhs_steps, out_nat, next_rhs, arm, zp,
                                                   final_out, ticket);
  return check_launch("wave solve");
}

// L then U; rhsL: r in L-step order; zl: natural z (sentinel-armed by caller);
// zu_rhs: z in U-step order (written by L); y: natural y; zout = Pi zp + y.
int wave_solve(const cprb_bilu& F, const double* rhsL, double* zl, double* zu_rhs, double* y,
               const double* zp, double* zout, cudaStream_t st) {
  int rc;
  if (F.b == 3) {
    rc = launch_wave<3, false>(F.Lw, rhsL, zl, zu_rhs, y, nullptr, nullptr, F.tickets + 2, st);
    if (rc) return rc;
    rc = launch_wave<3, true>(F.Uw, zu_rhs, y, nullptr, nullptr, zp, zout, F.tickets + 3, st);
  } else if (F.b == 1) {
    rc = launch_wave<1, false>(F.Lw, rhsL, zl, zu_rhs, y, nullptr, nullptr, F.tickets + 2, st);
    if (rc) return rc;
    rc = launch_wave<1, true>(F.Uw, zu_rhs, y, nullptr, nullptr, zp, zout, F.tickets + 3, st);
  } else {
    return set_error(CPRB_EUNSUPPORTED, "wave BILU supports block sizes 1 and 3");
  }
  return rc;
}

}  // namespace cprb

extern "C" int cprb_wave_set_log(uint64_t* dev_log) {
  unsigned long long* p = (unsigned long long*)dev_log;
  cudaMemcpyToSymbol(cprb::g_wave_log, &p, sizeof(p));
  return cprb::check_launch("wave log");
}

namespace cprb {

int wave_scatter_rhs(const cprb_bilu& F, const double* r, double* rhsL, cudaStream_t st) {
  k_scatter_slots<<<(F.n + 255) / 256, 256, 0, st>>>(F.n, F.b, F.l_slot, r, rhsL);
  return check_launch("scatter slots");
}

}  // namespace cprb
