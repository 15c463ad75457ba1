// gom_gen.cu — a whole Philox generation (engine_parallel.hpp:283-316) in ONE
// persistent kernel, for general linkage sets on integer weights with small
// populations (n <= 256, the C2 shape: 10^4 sets of 5 variables, n = 64).
//
// Why: at that size a colour group is ~1250 (set, 64-solution) teams that
// all fit in one wave, and the per-group kernel boundary plus its serial
// last-CTA epilogue cost more than the GOM work itself (measured on C2: an
// empty-bodied group kernel still takes 9.5 us of the 16 us per group).
// Here the CTAs stay resident for all k groups:
//
//   for each group g (order = device Fisher-Yates on Philox, :291):
//     work   : phases 1-4 for the group's sets (gom_general_set, shared with
//              the per-group kernel), per-CTA sums -> global atomics into
//              triple-buffered accumulators D[g % 3] (fitness / hash deltas,
//              steps, calls)
//     barrier: grid-wide (all CTAs co-resident: cooperative launch)
//     epilogue, REDUNDANTLY in every CTA from D[g % 3]: fitness + hashes of
//              all n members (kept in shared memory), evaluator-call
//              accounting + budget stop (runtime.hpp:75-80), the chained
//              elitist scan + target stop (:305-310) -> every CTA takes the
//              same decisions without a second barrier.  CTA 0 alone writes
//              the results back (fitness, hashes, counters, improvement log)
//              and zeroes the accumulator of group g-1 (last read before the
//              barrier of g, next written after the barrier of g+1).
//
// LEAN kernels (C2) differ in three ways: the barrier is the flat one
// (grid_barrier_flat); the epilogue of group g runs in one warp per CTA while
// the other warps already run group g+1's units, which wait for it only at
// their accept step; and a unit's sibling warps (one per population word)
// are adjacent warps of one CTA and meet at a named barrier.
//
// Results are bit-identical to the per-group path with the same device group
// order (tests/test_gen_kernel.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include "gom_general.cuh"
#include "gom_lean.cuh"

namespace gomix_b200 {

namespace {

constexpr uint32_t kTagOrderGen = 0x4F524400u;
__device__ unsigned long long g_cta_probe[8192];  // latency study: per-CTA arrival time and SM id  // same stream as begin_generation_kernel ("ORD")

// Launch timeline of the persistent generation kernel (probes builds only):
// point i = [2i] first / [2i+1] last arrival (%globaltimer ns) over every
// caller; point 0 = CTA start, then per slot s points 1 + 6s + {0: unit
// start, 1: unit done (warp 0 of every CTA with a unit), 2: CTA flushed,
// 3: barrier passed, 4: epilogue done (thread 0 of every CTA)}.
__device__ unsigned long long g_gen_tl[128];
__device__ __forceinline__ void gen_mark(uint32_t i, bool who) {
#ifdef GOMIX_PROBES
  if (who && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : : "memory");
    atomicMin(&g_gen_tl[2 * i], t);
    atomicMax(&g_gen_tl[2 * i + 1], t);
  }
#endif
}

// Two-level grid barrier.  ~1,250 single-team CTAs arriving on one counter
// serialise in one L2 slice (measured ~4 us per barrier on C2), so CTAs
// arrive on kBarSub counters (one 128-byte line each), the last arriver of
// each sub-group arrives on the top counter, and the last of those bumps the
// generation word every CTA polls.  Layout (uint32): [0] generation,
// [32] top arrivals, [64 + 32 g] arrivals of sub-group g.  The gpu-scope
// fences order each CTA's writes before its arrival and, on the way out,
// invalidate the SM's L1 so later loads see other CTAs' writes.
constexpr uint32_t kBarSub = 32;

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = bar;
    const unsigned int g = *vgen;
    __threadfence();
    const uint32_t subs = min(kBarSub, nblocks);
    const uint32_t grp = blockIdx.x % subs;
    const uint32_t members = nblocks / subs + (grp < nblocks % subs ? 1u : 0u);
    bool released = false;
    if (atomicAdd(bar + 64 + 32 * grp, 1u) == members - 1) {
      *(volatile unsigned int*)(bar + 64 + 32 * grp) = 0u;
      __threadfence();
      if (atomicAdd(bar + 32, 1u) == subs - 1) {
        *(volatile unsigned int*)(bar + 32) = 0u;
        __threadfence();
        atomicAdd(bar, 1u);
        released = true;
      }
    }
    if (!released)
      while (*vgen == g) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

// Flat grid barrier on a monotonic 64-bit counter (bar word 1536, never
// reset): every CTA adds 1 with acq_rel semantics and waits until the
// counter reaches the next multiple of the grid size — the last arrival
// releases everyone with no further hop (the two-level barrier above needs
// two more dependent atomics and a generation store after the last arrival).
__device__ __forceinline__ void grid_barrier_flat(unsigned int* bar, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(bar + 1536);
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
    const unsigned long long target = (old / nblocks + 1ull) * nblocks;
    if (old + 1ull != target) {
      unsigned long long v;
      do {
        __nanosleep(32);
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      } while (v < target);
    }
#ifdef GOMIX_GEN_BAR_FENCE
    __threadfence();
#endif
  }
  __syncthreads();  // the acquire above orders every thread's later loads (the CTA shares the SM's L1)
}

#ifdef GOMIX_GEN_TWO_LEVEL
#define GOMIX_GEN_BARRIER grid_barrier
#else
#define GOMIX_GEN_BARRIER grid_barrier_flat
#endif

}  // namespace

// Every set of a group should get its own team in ONE wave (a second set per
// team doubles the group's critical path), so team kernels are register-
// capped for that: 2-warp teams (n <= 64) at 11 CTAs per SM = 1,628 teams.
constexpr int gen_min_blocks(bool team, int tw) { return team ? (tw == 2 ? 11 : (tw == 4 ? 5 : 2)) : 2; }

// LEAN: every warp owns one population word of the sets it processes
// (gom_lean_unit, |F| <= 32); otherwise teams run gom_general_set.
template <int WPT, bool TEAM, int TW, bool LEAN>
__global__ void __launch_bounds__(LEAN ? 256 : (TEAM ? 32 * TW : 256), LEAN ? 3 : gen_min_blocks(TEAM, TW))
    gom_generation_kernel(const GomArgs a, const GenArgs ga) {
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ double s_fit[kGenMaxN];
  __shared__ unsigned long long s_h1[kGenMaxN], s_h2[kGenMaxN];
  __shared__ uint32_t s_order[kGenMaxK];
  __shared__ double s_chunkmax[kGenMaxN / 32];
  __shared__ unsigned long long s_steps, s_calls;
  // run state, identical in every CTA
  __shared__ double s_elit_fit;
  __shared__ int32_t s_elit_src, s_stop, s_stop_reason;
  __shared__ unsigned long long s_eh1, s_eh2, s_calls_total, s_run_steps, s_run_calls, s_groups, s_nimpr;
  __shared__ uint32_t s_ver;

  using Acc = long long;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t tw = TEAM ? (uint32_t)TW : 1u;
  const uint32_t teams_per_cta = TEAM ? 1u : (blockDim.x >> 5);
  const uint32_t team = TEAM ? 0u : warp, wit = TEAM ? warp : 0u;
  const uint32_t tid_team = wit * 32u + lane, team_threads = tw * 32u;
  const uint32_t Wp = a.Wp, n = a.n;
  uint32_t* stage = smem + (size_t)team * a.stage_words;
  // LEAN units go to warps in warp-major order (slot w of every CTA before
  // slot w + 1), so every SM gets the same number of busy warps
  // LEAN: the Wp sibling warps of a unit (one per population word) are
  // adjacent warps of one CTA (they meet at a named barrier before
  // committing), and units go to sibling groups warp-major (group g of every
  // CTA before group g + 1), so every SM gets the same number of busy warps:
  // unit p = (warp / Wp) * gridDim + blockIdx, word = warp % Wp
  const uint32_t gwarp = LEAN ? (warp / Wp) * (gridDim.x * Wp) + blockIdx.x * Wp + warp % Wp
                              : blockIdx.x * (blockDim.x >> 5) + warp;
  const uint32_t lean_w = LEAN ? gwarp % Wp : 0u;  // Wp divides the CTA's 8 warps
  // solution of this thread's word j
  auto sol = [&](int j) -> uint32_t { return LEAN ? lean_w * 32u + lane : (wit + tw * (uint32_t)j) * 32u + lane; };
  const BeginArgs& b = ga.begin;
  DevCtl* c = a.ctl;
  const uint32_t gen = *(volatile unsigned int*)&c->gen_counter;
  const uint32_t buf0 = *(volatile unsigned int*)&c->gen_buf;
  const bool lead = blockIdx.x == 0;

  if (threadIdx.x == 0) {
    s_elit_fit = c->elit_fit;
    s_elit_src = c->elit_src;
    s_eh1 = c->eh1;
    s_eh2 = c->eh2;
    s_ver = c->elit_ver;
    s_stop = 0;
    s_stop_reason = GOMIX_STOP_NONE;
    s_calls_total = b.calls_before;
    s_run_steps = s_run_calls = s_groups = s_nimpr = 0;
    // this generation's group order (Fisher-Yates, engine_parallel.hpp:291)
    const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
    for (uint32_t i = 0; i < ga.k; ++i) s_order[i] = i;
    for (uint32_t i = ga.k; i > 1; --i) {
      const uint4 r = philox4x32_10(make_uint4(i, gen, 0u, kTagOrderGen), key);
      const uint32_t j = bounded(lo64(r), i);
      const uint32_t t = s_order[i - 1];
      s_order[i - 1] = s_order[j];
      s_order[j] = t;
    }
  }
  for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
    s_fit[s] = a.fit[s];
    s_h1[s] = a.h1[s];
    s_h2[s] = a.h2[s];
  }
  __syncthreads();
  gen_mark(0, threadIdx.x == 0);

  uint32_t slot = 0;
  uint32_t ran = 0;   // groups whose epilogue ran (the accumulator rotation advances by this)
  LeanPre pre{};     // LEAN: the next group's first unit, prefetched before the barrier
  GroupDesc dnext{};  // the next group's descriptor, loaded before the barrier
  if constexpr (LEAN) {
    // LEAN: the epilogue of group t runs in ONE warp per CTA (the last one)
    // while the other warps already work on group t + 1: a unit's donor draw
    // and partial evaluation read only the rows committed before the barrier,
    // so only its accept / commit waits for the epilogue (the gate: s_gate
    // counts the epilogues done in this CTA; group t + 1's units pass at t + 1).
    __shared__ uint32_t s_gate;
    if (threadIdx.x == 0) s_gate = 0;
    __syncthreads();
    const uint32_t epi_warp = (blockDim.x >> 5) - 1u;
    uint32_t* wsm = smem + (size_t)warp * kLeanSmemWords;
    const uint32_t per_round = (gridDim.x * (blockDim.x >> 5)) / Wp;
    // the epilogue of slot t: commit, accounting, chained scan (one warp)
    auto epilogue = [&](uint32_t t) {
      const uint32_t gi_t = s_order[t];
      const uint32_t bt = (buf0 + t) % 3u;
      const long long* Dt = ga.dfit + (size_t)bt * n * kAccStride;
      const unsigned long long* DH1t = ga.dh + (size_t)bt * 2 * n * kAccStride;
      const unsigned long long* DH2t = DH1t + (size_t)n * kAccStride;
      const unsigned long long* CNTt = ga.cnt + 2 * bt;
      const uint32_t zb = (bt + 2u) % 3u;  // group t - 1's accumulators: every CTA read them before barrier t
      unsigned long long cnt_st = 0, cnt_ca = 0;
      if (lane == 0) {
        cnt_st = __ldcg(CNTt);
        cnt_ca = __ldcg(CNTt + 1);
      }
#pragma unroll 4
      for (uint32_t s = lane; s < n; s += 32u) {
        const double f = s_fit[s] + (double)__ldcg(Dt + s * kAccStride);
        const unsigned long long x1 = s_h1[s] ^ __ldcg(DH1t + s * kAccStride);
        const unsigned long long x2 = s_h2[s] ^ __ldcg(DH2t + s * kAccStride);
        s_fit[s] = f;
        s_h1[s] = x1;
        s_h2[s] = x2;
        if (lead) {
          a.epi.fit[s] = f;
          a.epi.h1[s] = x1;
          a.epi.h2[s] = x2;
          ga.dfit[((size_t)zb * n + s) * kAccStride] = 0;
          ga.dh[((size_t)zb * 2 * n + s) * kAccStride] = 0;
          ga.dh[((size_t)zb * 2 * n + n + s) * kAccStride] = 0;
        }
      }
      if (lead) {
        if (lane == 0) {
          ga.cnt[2 * zb] = 0;
          ga.cnt[2 * zb + 1] = 0;
        }
      }
      if (lane == 0) {
        s_calls_total += cnt_ca;
        s_run_steps += cnt_st;
        s_run_calls += cnt_ca;
        s_groups += 1;
        if (lead) {
          a.epi.gsteps[gi_t] += cnt_st;
          a.epi.gcalls[gi_t] += cnt_ca;
        }
        if (b.has_budget && (double)s_calls_total / b.q >= b.max_evals && !s_stop) {
          s_stop = 1;
          s_stop_reason = GOMIX_STOP_BUDGET;
        }
      }
      __syncwarp();
      for (uint32_t ch = 0; ch * 32u < n; ++ch) {
        const uint32_t s = ch * 32u + lane;
        double f = s < n ? s_fit[s] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) f = fmax(f, __shfl_xor_sync(0xFFFFFFFFu, f, o));
        if (lane == 0) s_chunkmax[ch] = f;
      }
      __syncwarp();
      // chained elitist scan over all members in index order (:305-310)
      double cur = s_elit_fit;
      int32_t best = -1;
      bool hit = false;
      unsigned long long ni = s_nimpr;
      const unsigned long long calls_now = s_calls_total;
      for (uint32_t base = 0; base < n; base += 32u) {
        if (!(s_chunkmax[base >> 5] > cur)) continue;  // better() implies >
        const uint32_t s = base + lane;
        const double f = s < n ? s_fit[s] : -INFINITY;
        uint32_t m = __ballot_sync(0xFFFFFFFFu, s < n && f > cur);
        while (m) {
          const uint32_t l = __ffs(m) - 1;
          cur = __shfl_sync(0xFFFFFFFFu, f, l);
          best = (int32_t)(base + l);
          if (lead && lane == 0 && ni < a.epi.impr_cap) {
            a.epi.impr[ni].fit = cur;
            a.epi.impr[ni].calls = calls_now;
          }
          ++ni;
          hit |= b.has_target && cur >= b.target;
          m = __ballot_sync(0xFFFFFFFFu, s < n && lane > l && f > cur);
        }
      }
      __syncwarp();
      if (lane == 0) {
        s_nimpr = ni;
        if (hit && !s_stop) {
          s_stop = 1;
          s_stop_reason = GOMIX_STOP_TARGET;
        }
        if (best >= 0) {  // new elitist: member `best` (snapshot taken copy-on-write)
          s_elit_fit = cur;
          s_elit_src = best;
          s_eh1 = s_h1[best];
          s_eh2 = s_h2[best];
          s_ver += 1;
        }
        __threadfence_block();
        *(volatile uint32_t*)&s_gate = t + 1u;  // group t + 1's units may accept / commit
      }
      __syncwarp();
    };
    bool aborted = false;
    for (; slot < ga.k; ++slot) {
      const uint32_t gi = s_order[slot];
      const GroupDesc d = slot == 0 ? a.groups[gi] : dnext;
      const uint4* gmeta = a.gmeta + d.g0;
      const uint32_t bi = (buf0 + slot) % 3u;
      long long* D = ga.dfit + (size_t)bi * n * kAccStride;
      unsigned long long* DH1 = ga.dh + (size_t)bi * 2 * n * kAccStride;
      unsigned long long* DH2 = DH1 + (size_t)n * kAccStride;
      unsigned long long* CNT = ga.cnt + 2 * bi;
      if (warp == epi_warp && slot > 0) epilogue(slot - 1u);
      // group-start state of this slot, read once the gate opens
      auto gate = [&](uint32_t s) -> LeanGate {
        if (lane == 0)
          while (*(volatile uint32_t*)&s_gate < slot) __nanosleep(20);
        __syncwarp();
        __threadfence_block();
        LeanGate g;
        g.stop = *(volatile int32_t*)&s_stop != 0;
        const unsigned long long e1 = *(volatile unsigned long long*)&s_eh1;
        const unsigned long long e2 = *(volatile unsigned long long*)&s_eh2;
        g.is_elit = s < n && ((volatile unsigned long long*)s_h1)[s] == e1 &&
                    ((volatile unsigned long long*)s_h2)[s] == e2;
        g.esrc = *(volatile int32_t*)&s_elit_src;
        g.ever_cur = *(volatile uint32_t*)&s_ver;
        return g;
      };
      long long acc = 0;
      unsigned long long dh1 = 0, dh2 = 0, calls = 0;
      uint32_t steps = 0;
      for (uint32_t p = gwarp / Wp; p < d.G; p += per_round) {
        const LeanPre cur = (p == gwarp / Wp && slot > 0) ? pre : lean_prefetch(a, gmeta, p, lane);
        gen_mark(1 + 6 * slot, lane == 0 && warp == 0);
        gom_lean_unit<(uint32_t)WPT>(a, p, cur, lean_w, gen, wsm, lane, gate, false, acc, dh1, dh2, steps, calls,
                      1u + warp / Wp);
        gen_mark(2 + 6 * slot, lane == 0 && warp == 0);
      }
      // the next group's first unit: plan inputs in flight during the barrier
      if (slot + 1 < ga.k) {
        dnext = a.groups[s_order[slot + 1]];
        if (gwarp / Wp < dnext.G) pre = lean_prefetch(a, a.gmeta + dnext.g0, gwarp / Wp, lane);
      }
      if (threadIdx.x == 0) {
        s_steps = 0;
        s_calls = 0;
      }
      __syncthreads();  // this CTA's units and the epilogue of slot - 1 are done
      if (s_stop) {     // stopped by the epilogue of slot - 1: nothing of this slot was committed
        aborted = true;
        break;
      }
      {
        const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, steps);
        const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)calls);
        if (lane == 0 && (ws | wc)) {
          atomicAdd(reinterpret_cast<unsigned int*>(&s_steps), ws);
          atomicAdd(reinterpret_cast<unsigned int*>(&s_calls), wc);
        }
      }
      const uint32_t s0 = lean_w * 32u + lane;
      if (s0 < n) {
        if (acc) atomicAdd(reinterpret_cast<unsigned long long*>(D + s0 * kAccStride), (unsigned long long)acc);
        if (dh1 | dh2) {
          atomicXor(DH1 + s0 * kAccStride, dh1);
          atomicXor(DH2 + s0 * kAccStride, dh2);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && (s_steps | s_calls)) {
        atomicAdd(CNT, s_steps);
        atomicAdd(CNT + 1, s_calls);
      }
      gen_mark(3 + 6 * slot, threadIdx.x == 0);
      GOMIX_GEN_BARRIER(ga.bar, gridDim.x);
      gen_mark(4 + 6 * slot, threadIdx.x == 0);
    }
    if (!aborted) {
      if (warp == epi_warp) epilogue(ga.k - 1u);
      __syncthreads();
      ran = ga.k;
    } else {
      ran = slot;  // stopped by the epilogue of slot - 1
    }
  } else {
  for (; slot < ga.k; ++slot) {
    const uint32_t gi = s_order[slot];
    const GroupDesc d = slot == 0 ? a.groups[gi] : dnext;
    const uint4* gmeta = a.gmeta + d.g0;
    const uint32_t bi = (buf0 + slot) % 3u;
    // accumulators spread one per 256-byte line: ~1,250 CTAs add into the same
    // n solutions, so neighbouring solutions must not share an L2 line
    long long* D = ga.dfit + (size_t)bi * n * kAccStride;
    unsigned long long* DH1 = ga.dh + (size_t)bi * 2 * n * kAccStride;
    unsigned long long* DH2 = DH1 + (size_t)n * kAccStride;
    unsigned long long* CNT = ga.cnt + 2 * bi;

    // ---- work: phases 1-4 over this CTA's sets ------------------------------
    const unsigned long long eh1 = s_eh1, eh2 = s_eh2;
    const int32_t esrc = s_elit_src;
    const uint32_t ever_cur = s_ver;
    bool is_elit[WPT];
    double pfit[WPT];
    Acc acc[WPT];
    unsigned long long dh1[WPT], dh2[WPT];
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      const uint32_t s = sol(j);
      is_elit[j] = s < n && s_h1[s] == eh1 && s_h2[s] == eh2;
      pfit[j] = 0.0;
      acc[j] = 0;
      dh1[j] = 0;
      dh2[j] = 0;
    }
    uint32_t steps = 0;
    unsigned long long calls = 0;
    {  // teams (the LEAN kernel runs the overlapped loop above)
      for (uint32_t p = blockIdx.x * teams_per_cta + team; p < d.G; p += gridDim.x * teams_per_cta)
        gom_general_set<WPT, true, TEAM>(a, p, gmeta, gen, stage, lane, tw, wit, tid_team, team_threads,
                                         teams_per_cta, team, true, false, false, is_elit, pfit, esrc, ever_cur,
                                         acc, dh1, dh2, steps, calls);
      if (slot + 1 < ga.k) dnext = a.groups[s_order[slot + 1]];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_steps = 0;
      s_calls = 0;
    }
    __syncthreads();
    {
      // per-CTA group counts fit 32 bits (units per CTA x n x footprint):
      // native 32-bit shared atomics (64-bit ones are compare-and-swap loops)
      const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, steps);
      const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)calls);
      if (lane == 0 && (ws | wc)) {
        atomicAdd(reinterpret_cast<unsigned int*>(&s_steps), ws);
        atomicAdd(reinterpret_cast<unsigned int*>(&s_calls), wc);
      }
    }
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      const uint32_t s = sol(j);
      if (s < n) {
        if (acc[j]) atomicAdd(reinterpret_cast<unsigned long long*>(D + s * kAccStride), (unsigned long long)acc[j]);
        if (dh1[j] | dh2[j]) {
          atomicXor(DH1 + s * kAccStride, dh1[j]);
          atomicXor(DH2 + s * kAccStride, dh2[j]);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && (s_steps | s_calls)) {
      atomicAdd(CNT, s_steps);
      atomicAdd(CNT + 1, s_calls);
    }
    probe(a.exp_flags, 16 + 4 * slot);
#ifdef GOMIX_PROBES
    if ((a.exp_flags & 32u) && slot == 0 && threadIdx.x == 0 && blockIdx.x < 4096) {
      unsigned long long t;
      uint32_t smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_cta_probe[2 * blockIdx.x] = t;
      g_cta_probe[2 * blockIdx.x + 1] = smid;
    }
#endif
    gen_mark(3 + 6 * slot, threadIdx.x == 0);
    GOMIX_GEN_BARRIER(ga.bar, gridDim.x);
    gen_mark(4 + 6 * slot, threadIdx.x == 0);
    probe(a.exp_flags, 17 + 4 * slot);

    // ---- epilogue (every CTA): fitness / hash commit ------------------------
    unsigned long long cnt_st = 0, cnt_ca = 0;
    if (threadIdx.x == 0) {  // issued with the accumulator loads below (one round trip)
      cnt_st = __ldcg(CNT);
      cnt_ca = __ldcg(CNT + 1);
    }
    for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
      const double f = s_fit[s] + (double)__ldcg(D + s * kAccStride);
      const unsigned long long x1 = s_h1[s] ^ __ldcg(DH1 + s * kAccStride), x2 = s_h2[s] ^ __ldcg(DH2 + s * kAccStride);
      s_fit[s] = f;
      s_h1[s] = x1;
      s_h2[s] = x2;
      if (lead) {
        a.epi.fit[s] = f;
        a.epi.h1[s] = x1;
        a.epi.h2[s] = x2;
        // accumulator of the previous group: read by every CTA before this
        // group's barrier, written again only after the next one
        const uint32_t zb = (bi + 2u) % 3u;
        ga.dfit[((size_t)zb * n + s) * kAccStride] = 0;
        ga.dh[((size_t)zb * 2 * n + s) * kAccStride] = 0;
        ga.dh[((size_t)zb * 2 * n + n + s) * kAccStride] = 0;
      }
    }
    if (lead && threadIdx.x == 0) {
      const uint32_t zb = (bi + 2u) % 3u;
      ga.cnt[2 * zb] = 0;
      ga.cnt[2 * zb + 1] = 0;
    }
    if (threadIdx.x == 0) {
      const unsigned long long st = cnt_st, ca = cnt_ca;
      s_calls_total += ca;
      s_run_steps += st;
      s_run_calls += ca;
      s_groups += 1;
      if (lead) {
        a.epi.gsteps[gi] += st;
        a.epi.gcalls[gi] += ca;
      }
      if (b.has_budget && (double)s_calls_total / b.q >= b.max_evals && !s_stop) {
        s_stop = 1;
        s_stop_reason = GOMIX_STOP_BUDGET;
      }
    }
    __syncthreads();
    // chained elitist scan over all members in index order (:305-310)
    for (uint32_t ch = warp; ch * 32u < n; ch += blockDim.x >> 5) {
      const uint32_t s = ch * 32u + lane;
      double f = s < n ? s_fit[s] : -INFINITY;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) f = fmax(f, __shfl_xor_sync(0xFFFFFFFFu, f, o));
      if (lane == 0) s_chunkmax[ch] = f;
    }
    __syncthreads();
    if (warp == 0) {
      double cur = s_elit_fit;
      int32_t best = -1;
      bool hit = false;
      unsigned long long ni = s_nimpr;
      const unsigned long long calls_now = s_calls_total;
      for (uint32_t base = 0; base < n; base += 32u) {
        if (!(s_chunkmax[base >> 5] > cur)) continue;  // better() implies >
        const uint32_t s = base + lane;
        const double f = s < n ? s_fit[s] : -INFINITY;
        uint32_t m = __ballot_sync(0xFFFFFFFFu, s < n && f > cur);
        while (m) {
          const uint32_t l = __ffs(m) - 1;
          cur = __shfl_sync(0xFFFFFFFFu, f, l);
          best = (int32_t)(base + l);
          if (lead && lane == 0 && ni < a.epi.impr_cap) {
            a.epi.impr[ni].fit = cur;
            a.epi.impr[ni].calls = calls_now;
          }
          ++ni;
          hit |= b.has_target && cur >= b.target;
          m = __ballot_sync(0xFFFFFFFFu, s < n && lane > l && f > cur);
        }
      }
      __syncwarp();  // every lane read s_elit_fit / s_nimpr above before lane 0 rewrites them
      if (lane == 0) {
        s_nimpr = ni;
        if (hit && !s_stop) {
          s_stop = 1;
          s_stop_reason = GOMIX_STOP_TARGET;
        }
        if (best >= 0) {  // new elitist: member `best` (snapshot taken copy-on-write)
          s_elit_fit = cur;
          s_elit_src = best;
          s_eh1 = s_h1[best];
          s_eh2 = s_h2[best];
          s_ver += 1;
        }
      }
    }
    __syncthreads();
    gen_mark(5 + 6 * slot, threadIdx.x == 0);
    probe(a.exp_flags, 18 + 4 * slot);
    if (s_stop) break;
  }
  ran = slot < ga.k ? slot + 1 : ga.k;
  }

  if (lead && threadIdx.x == 0) {
    c->elit_fit = s_elit_fit;
    c->elit_src = s_elit_src;
    c->eh1 = s_eh1;
    c->eh2 = s_eh2;
    c->elit_ver = s_ver;
    c->stop = s_stop;
    c->stop_reason = s_stop_reason;
    c->has_budget = b.has_budget;
    c->has_target = b.has_target;
    c->max_evals = b.max_evals;
    c->target = b.target;
    c->calls_total = s_calls_total;
    c->run_steps = s_run_steps;
    c->run_calls = s_run_calls;
    c->groups_run = s_groups;
    c->n_impr = s_nimpr;
    c->grp_steps = c->grp_calls = 0;
    c->done = 0;
    c->cur_gen = gen;
    c->gen_counter = gen + 1;
    // the accumulator index itself (mod 3), not a running count: a count
    // would wrap at 2^32, where 2^32 = 1 (mod 3) breaks the rotation
    c->gen_buf = (buf0 + ran) % 3u;
    for (uint32_t i = 0; i < ga.k; ++i) ga.order[i] = s_order[i];
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {
void* gen_kernel(int wpt, bool team, int tw, bool lean) {
  if (lean) {  // wpt = the population's words per row (Wp)
    switch (wpt) {
      case 1: return (void*)gom_generation_kernel<1, false, 1, true>;
      case 2: return (void*)gom_generation_kernel<2, false, 1, true>;
      case 4: return (void*)gom_generation_kernel<4, false, 1, true>;
      case 8: return (void*)gom_generation_kernel<8, false, 1, true>;
    }
    return nullptr;
  }
  if (team) {
    if (wpt != 1) return nullptr;
    switch (tw) {
      case 2: return (void*)gom_generation_kernel<1, true, 2, false>;
      case 4: return (void*)gom_generation_kernel<1, true, 4, false>;
      case 8: return (void*)gom_generation_kernel<1, true, 8, false>;
    }
  } else {
    switch (wpt) {
      case 1: return (void*)gom_generation_kernel<1, false, 1, false>;
      case 2: return (void*)gom_generation_kernel<2, false, 1, false>;
      case 4: return (void*)gom_generation_kernel<4, false, 1, false>;
      case 8: return (void*)gom_generation_kernel<8, false, 1, false>;
    }
  }
  return nullptr;
}
}  // namespace

void debug_cta_probes(unsigned long long* out) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_cta_probe, sizeof(unsigned long long) * 8192));
}

// the generation kernel's timeline (probes builds): 128 words, then reset
void debug_gen_timeline(unsigned long long* out) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_gen_tl, sizeof(unsigned long long) * 128));
  unsigned long long z[128];
  for (int i = 0; i < 64; ++i) {
    z[2 * i] = ~0ull;
    z[2 * i + 1] = 0ull;
  }
  GOMIX_CUDA(cudaMemcpyToSymbol(g_gen_tl, z, sizeof(z)));
}

void debug_probes_gen(unsigned long long* out, bool reset) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_probe, sizeof(unsigned long long) * 64));
  if (reset) {
    unsigned long long z[64] = {};
    GOMIX_CUDA(cudaMemcpyToSymbol(g_probe, z, sizeof(z)));
  }
}

int gen_lean_smem() { return 8 * (int)kLeanSmemWords * 4; }

int gen_kernel_max_blocks(int wpt, bool team, int block, size_t smem, bool lean) {
  void* fn = gen_kernel(wpt, team, team ? block / 32 : 1, lean);
  if (!fn) return 0;
  GOMIX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = 0;
  GOMIX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, block, smem));
  return blocks;
}

void launch_generation_kernel(const GomArgs& a, const GenArgs& ga, int wpt, bool team, int grid, int block,
                              size_t smem, cudaStream_t s, bool lean) {
  void* fn = gen_kernel(wpt, team, team ? block / 32 : 1, lean);
  void* args[] = {(void*)&a, (void*)&ga};
  GOMIX_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, smem, s));
}

}  // namespace gomix_b200
