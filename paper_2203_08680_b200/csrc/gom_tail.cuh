// gom_tail.cuh — the end of a per-group GOM launch, shared by the
// lane-per-solution kernels (gom_group_kernel in gom.cu, gom_univ_f64_kernel
// in gom_univ_f64.cu): per-CTA counters, the CTA's per-solution fitness and
// Zobrist deltas (teams combined, then fixed-point atomics), then the group epilogue
// (engine_parallel.hpp:221-247, :305-310) in the last CTA to finish.
#pragma once

#include "gom_common.cuh"

namespace gomix_b200 {

// acc / dh1 / dh2: this thread's deltas of its solutions (wit + tw * j) * 32 + lane;
// smem: at least teams_per_cta * Wp * 32 * 24 bytes when teams_per_cta > 1.
template <int WPT>
__device__ __forceinline__ void gom_group_tail(const GomArgs& a, const EpiArgs& epi, uint32_t* smem,
                                               uint32_t teams_per_cta, uint32_t team, uint32_t wit, uint32_t tw,
                                               uint32_t lane, const long long (&acc)[WPT], const unsigned long long (&dh1)[WPT],
                                               const unsigned long long (&dh2)[WPT], uint32_t steps,
                                               unsigned long long calls) {
  const uint32_t Wp = a.Wp, n = a.n;
  // ---- per-CTA reductions: counters, fitness deltas, elitist distances ----
  __syncthreads();
  __shared__ unsigned long long s_steps, s_calls;
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    s_steps = 0;
    s_calls = 0;
  }
  __syncthreads();
  {
    const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, steps);
    unsigned long long wc = calls;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wc += __shfl_xor_sync(0xFFFFFFFFu, wc, o);
    if (lane == 0 && (ws | wc)) {
      atomicAdd(&s_steps, (unsigned long long)ws);
      atomicAdd(&s_calls, wc);
    }
  }
  // fitness deltas are fixed-point integers (every delta rounded before any
  // sum, GomArgs::fix_scale): order-free atomics, deterministic for any grid
  unsigned long long* dfit = reinterpret_cast<unsigned long long*>(a.dfit);
  if (teams_per_cta > 1) {
    // several teams per CTA: combine them first (one global atomic per solution)
    long long* sacc = reinterpret_cast<long long*>(smem);
    unsigned long long* sh1 = reinterpret_cast<unsigned long long*>(sacc + (size_t)teams_per_cta * Wp * 32u);
    unsigned long long* sh2 = sh1 + (size_t)teams_per_cta * Wp * 32u;
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      const uint32_t s = (wit + tw * (uint32_t)j) * 32u + lane;
      sacc[(size_t)team * Wp * 32u + s] = acc[j];
      sh1[(size_t)team * Wp * 32u + s] = dh1[j];
      sh2[(size_t)team * Wp * 32u + s] = dh2[j];
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < Wp * 32u; s += blockDim.x) {
      long long v = 0;
      unsigned long long x1 = 0, x2 = 0;
      for (uint32_t t = 0; t < teams_per_cta; ++t) {
        v += sacc[(size_t)t * Wp * 32u + s];
        x1 ^= sh1[(size_t)t * Wp * 32u + s];
        x2 ^= sh2[(size_t)t * Wp * 32u + s];
      }
      if (s < n) {
        if (v) atomicAdd(dfit + s, (unsigned long long)v);
        if (x1 | x2) {
          atomicXor(&a.dh1[s], x1);
          atomicXor(&a.dh2[s], x2);
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      const uint32_t s = (wit + tw * (uint32_t)j) * 32u + lane;
      if (s < n) {
        if (acc[j]) atomicAdd(dfit + s, (unsigned long long)acc[j]);
        if (dh1[j] | dh2[j]) {
          atomicXor(&a.dh1[s], dh1[j]);
          atomicXor(&a.dh2[s], dh2[j]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && (s_steps | s_calls)) {
    atomicAdd(&a.ctl->grp_steps, s_steps);
    atomicAdd(&a.ctl->grp_calls, s_calls);
  }
  const uint32_t parties = gridDim.x;
  if (threadIdx.x == 0) {
    // last-party ticket: everything above is visible to the last one
    __threadfence();
    s_last = atomicAdd(&a.ctl->done, 1u) == parties - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  epilogue_body(epi);
  if (threadIdx.x == 0) a.ctl->done = 0;
}

}  // namespace gomix_b200
