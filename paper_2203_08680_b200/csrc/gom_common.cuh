// gom_common.cuh — device helpers shared by the GOM kernels (gom.cu,
// gom_univ.cu): Philox4x32-10, the reference's FitnessComparator, Zobrist
// keys, the copy-on-write elitist capture, bit tricks, and the group epilogue
// (fitness commit, evaluator-call accounting, elitist scan) run by the last
// CTA of a GOM launch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"
#include "gom_peer.cuh"

namespace gomix_b200 {

constexpr uint32_t kEpiSmemFit = 256;  // fitness values the epilogue keeps in shared memory

// Timing probes for latency studies: CTA 0 / thread 0 records %globaltimer at
// numbered points.  Compiled in only with -DGOMIX_PROBES (and then enabled at
// run time by GOMIX_EXP bit 32); production builds carry no probe code.
static __device__ unsigned long long g_probe[64];  // one copy per translation unit
__device__ __forceinline__ void probe(uint32_t flags, uint32_t i) {
#ifdef GOMIX_PROBES
  if ((flags & 32u) && blockIdx.x == 0 && threadIdx.x == 0 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (g_probe[i] == 0) g_probe[i] = t;
  }
#endif
}
// the same from thread 0 of whichever CTA calls it (the last-CTA epilogue)
__device__ __forceinline__ void probe_last(uint32_t flags, uint32_t i) {
#ifdef GOMIX_PROBES
  if ((flags & 32u) && threadIdx.x == 0 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (g_probe[i] == 0) g_probe[i] = t;
  }
#endif
}

// Last-CTA ticket with release / acquire semantics in one instruction (the
// CTA's earlier writes are visible to whoever draws the last ticket, and the
// last one sees everyone's): replaces __threadfence() + atomicAdd.
__device__ __forceinline__ unsigned int ticket_acq_rel(unsigned int* p) {
  unsigned int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

// Launch timeline (probes builds only): for point i of launch row r (the
// graph slot + 1; 0 = a direct launch), the earliest and latest CTA to reach
// it (thread 0), as %globaltimer ns; read and reset through
// gomix_debug_timeline.
constexpr int kTimelineRows = 4;
static __device__ unsigned long long g_timeline[kTimelineRows * 32];  // one copy per translation unit
#ifdef GOMIX_PROBES
static __shared__ int32_t s_tl_row;  // the launch's row, for marks in shared device code (row -1)
#endif
__device__ __forceinline__ void timeline_set_row(int32_t row) {
#ifdef GOMIX_PROBES
  if (threadIdx.x == 0) s_tl_row = row;
#endif
}
// SM cycle stamps of the epilogue CTA (probes builds): point i, thread 0
static __device__ long long g_epiclk[16];
__device__ __forceinline__ void epi_clock(uint32_t i) {
#ifdef GOMIX_PROBES
  if (threadIdx.x == 0 && i < 16) {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : : "memory");
    g_epiclk[i] = t;
  }
#endif
}
__device__ __forceinline__ void timeline_mark(uint32_t i, int32_t row = 0) {
  epi_clock(i);
#ifdef GOMIX_PROBES
  if (row == -1) row = s_tl_row;
  if (threadIdx.x == 0 && i < 16) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : : "memory");  // memory: no load/store moves across
    const int32_t r = row < 0 ? 0 : (row >= kTimelineRows ? kTimelineRows - 1 : row);
    atomicMin(&g_timeline[r * 32 + 2 * i], t);
    atomicMax(&g_timeline[r * 32 + 2 * i + 1], t);
  }
#endif
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11), counter-based: every (generation, set,
// solution, call) has its own counter, so draws need no state and no order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ uint64_t lo64(uint4 r) { return (uint64_t)r.x | ((uint64_t)r.y << 32); }
__device__ __forceinline__ uint64_t hi64(uint4 r) { return (uint64_t)r.z | ((uint64_t)r.w << 32); }
// uniform in [0, n): high 64 bits of r*n (bias <= n / 2^64).
__device__ __forceinline__ uint32_t bounded(uint64_t r, uint32_t n) {
  return (uint32_t)__umul64hi(r, (uint64_t)n);
}

constexpr uint32_t kTagGom = 0x474F4D00u;   // "GOM"
constexpr uint32_t kTagInit = 0x494E4900u;  // "INI"

// FitnessComparator (graybox.hpp:22-35).
__device__ __forceinline__ double cmp_scale(double a, double b) {
  return 1e-9 * fmax(1.0, fmax(fabs(a), fabs(b)));
}
__device__ __forceinline__ bool cmp_better(bool exact, double a, double b) {
  return exact ? a > b : a - b > cmp_scale(a, b);
}
__device__ __forceinline__ bool cmp_equal(bool exact, double a, double b) {
  return exact ? a == b : fabs(a - b) <= cmp_scale(a, b);
}

// 128-bit Zobrist key of variable v (two independent splitmix64 streams).
// A genotype's hash is the XOR of the keys of its variables set to 1, so a
// flip of v toggles key(v): "parent == elitist" (engine_parallel.hpp:202) is
// hash equality, maintained incrementally instead of recounted per group.
__device__ __forceinline__ unsigned long long smix(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ void zobrist(uint32_t v, unsigned long long& z1, unsigned long long& z2) {
  z1 = smix(0x5A0B0000000000ull ^ (unsigned long long)v);
  z2 = smix(0xC3A5C85C97CB3127ull + 0x9E37ull * (unsigned long long)v);
}

// Copy-on-write elitist snapshot: before solution elit_src changes variable v
// for the first time since it became the elitist, record its old bit.
__device__ __forceinline__ void capture_row(uint32_t* elit, uint32_t* ever, uint32_t ver, uint32_t v,
                                            uint32_t old_bit) {
  if (ever[v] == ver) return;
  if (old_bit)
    atomicOr(&elit[v >> 5], 1u << (v & 31u));
  else
    atomicAnd(&elit[v >> 5], ~(1u << (v & 31u)));
  ever[v] = ver;
}

__device__ __forceinline__ uint32_t valid_mask(uint32_t w, uint32_t n) {
  const uint32_t lo = w * 32u;
  if (lo + 32u <= n) return 0xFFFFFFFFu;
  if (lo >= n) return 0u;
  return (1u << (n - lo)) - 1u;
}

// A team is one warp (several per CTA) or a whole CTA (tw > 1); the host
// never builds multi-warp teams that share a CTA, so no named barriers are
// needed (dynamic barrier ids would reserve all 16 and cap CTAs per SM).
__device__ __forceinline__ void team_sync(uint32_t tw, uint32_t, uint32_t) {
  if (tw == 1)
    __syncwarp();
  else
    __syncthreads();
}

// Members of word w2 that differ from pattern m somewhere on F.
// word wg of the staged pool (stride RW per row; Wp words per rank's shard of
// n members).
__device__ __forceinline__ uint32_t differ_word(const uint32_t* rowsF, uint32_t f, uint32_t RW,
                                                uint32_t wg, uint64_t m, uint32_t n, uint32_t Wp) {
  uint32_t dw = 0;
  for (uint32_t jv = 0; jv < f; ++jv)
    dw |= rowsF[jv * RW + wg] ^ (((m >> jv) & 1ull) ? 0xFFFFFFFFu : 0u);
  return dw & valid_mask(wg & (Wp - 1u), n);  // Wp is a power of two
}

// 32x32 bit-matrix transpose across a warp: lane r holds row r on entry;
// on exit lane c holds column c (bit r = bit c of the old row r).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, uint32_t lane) {
  constexpr uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const uint32_t j = 16u >> st, m = masks[st];
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, j);
#ifdef GOMIX_TRANSPOSE_ROT
    // lower lane: keep the m blocks of x, take y's m blocks moved up by j;
    // upper lane: keep the ~m blocks, take y's ~m blocks moved down by j —
    // one rotate (funnel shift by j or 32 - j) and one 3-input select
    // (measured: no faster — the lane-dependent constants are rematerialised)
    const bool up = (lane & j) != 0u;
    const uint32_t keep = up ? ~m : m;
    const uint32_t r = __funnelshift_l(y, y, up ? 32u - j : j);
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x) : "r"(x), "r"(r), "r"(keep));  // (x & keep) | (r & ~keep)
#else
    x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
#endif
  }
  return x;
}

__device__ __forceinline__ double shfl_d(double x, int src) {
  return __shfl_sync(0xFFFFFFFFu, x, src);
}

// Position of the k-th (0-based) set bit of x; k < popc(x).
__device__ __forceinline__ uint32_t select_bit(uint32_t x, uint32_t k) {
  uint32_t pos = 0;
#pragma unroll
  for (uint32_t sh = 16; sh >= 1; sh >>= 1) {
    const uint32_t c = __popc(x & ((1u << sh) - 1u));
    if (k >= c) {
      k -= c;
      x >>= sh;
      pos += sh;
    }
  }
  return pos;
}

// ---------------------------------------------------------------------------
// epilogue (run by the last CTA of the GOM kernel to finish): commit the
// group's fitness deltas, account the evaluator calls (budget stop first,
// runtime.hpp:75-80), then the elitist scan of engine_parallel.hpp:305-310 —
// the first member strictly better than the running elitist replaces it and
// the scan continues against the new value — logging every improvement with
// the call count at that moment and latching the target stop
// (runtime.hpp:88-93,136-143).
// ---------------------------------------------------------------------------
static __device__ void request_stop(DevCtl* c, int reason) {
  if (!c->stop) {
    c->stop = 1;
    c->stop_reason = reason;
  }
}

static __device__ void note_improvement(const EpiArgs& a, double f) {
  DevCtl* c = a.ctl;
  const unsigned long long i = c->n_impr++;
  if (i < a.impr_cap) {
    a.impr[i].fit = f;
    a.impr[i].calls = c->calls_total;
  }
  if (c->has_target && (cmp_better(c->exact, f, c->target) || cmp_equal(c->exact, f, c->target)))
    request_stop(c, GOMIX_STOP_TARGET);
}

// Commit this rank's group deltas: fitness (fixed-point sums of the accepted
// deltas / reference-ordered recorded deltas) and Zobrist hashes of its n
// solutions.  Fixed point: every delta is rounded to a multiple of
// 1 / fix_scale (1 for integer weights: exact) before any summation, so the
// integer sums do not depend on which thread or CTA added what — the
// float path is deterministic for any grid, within 1e-9 relative of the
// reference's sums (north star).
static __device__ void commit_range(const EpiArgs& a, uint32_t s0, uint32_t s1, double* s_fit,
                                    unsigned long long* s_h) {
  const uint32_t n = a.n;
#pragma unroll 4
  for (uint32_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    double f = a.fit[s];
    if (a.mode == 2) {
      for (uint32_t p = 0; p < a.G; ++p)
        if (a.rec_accept[(size_t)p * n + s]) f += a.rec_delta[(size_t)p * n + s];
    } else {
      f += (double)a.dfit[s] * a.fix_inv;
      a.dfit[s] = 0;
    }
    a.fit[s] = f;
    if (s_fit && s < kEpiSmemFit) s_fit[s] = f;
    const unsigned long long x1 = a.h1[s] ^ a.dh1[s], x2 = a.h2[s] ^ a.dh2[s];
    a.h1[s] = x1;
    a.h2[s] = x2;
    if (s_h && s < kEpiSmemFit) {  // the scan takes a new elitist's hash from here
      s_h[2 * s] = x1;
      s_h[2 * s + 1] = x2;
    }
    a.dh1[s] = 0;
    a.dh2[s] = 0;
  }
}



// Evaluator-call accounting (budget stop first, runtime.hpp:75-80), then the
// elitist scan of engine_parallel.hpp:305-310 over all n_global members in
// index order — the first member strictly better than the running elitist
// replaces it and the scan continues against the new value — logging every
// improvement with the call count at that moment and latching the target stop
// (runtime.hpp:88-93,136-143).  Sharded runs execute it on every rank from the
// gathered state, so all ranks take identical decisions.
// The control-block fields the scan reads, loaded by thread 0 in one memory
// round trip — issued before the group's commit where the caller can, so the
// two round trips overlap.
struct CtlSnap {
  unsigned long long st, ca, calls_total, run_steps, run_calls, groups_run, n_impr, gst, gca;
  int32_t has_budget, has_target, exact, stop;
  uint32_t ver;
  double max_evals, q, target, elit_fit;
};

static __device__ __forceinline__ CtlSnap load_ctl_snap(const EpiArgs& a) {
  const DevCtl* c = a.ctl;
  CtlSnap k;
  k.st = 0;
  k.ca = 0;
  if (a.R > 1) {
    for (uint32_t r = 0; r < a.R; ++r) {
      k.st += a.rank_cnt[2 * r];
      k.ca += a.rank_cnt[2 * r + 1];
    }
  } else {
    k.st = c->grp_steps;
    k.ca = c->grp_calls;
  }
  k.calls_total = c->calls_total;
  k.run_steps = c->run_steps;
  k.run_calls = c->run_calls;
  k.groups_run = c->groups_run;
  k.n_impr = c->n_impr;
  k.gst = a.gsteps[a.group];
  k.gca = a.gcalls[a.group];
  k.has_budget = c->has_budget;
  k.has_target = c->has_target;
  k.exact = c->exact;
  k.stop = c->stop;
  k.ver = c->elit_ver;
  k.max_evals = c->max_evals;
  k.q = c->q;
  k.target = c->target;
  k.elit_fit = c->elit_fit;
  return k;
}

static __device__ void elitist_scan(const EpiArgs& a, const double* s_fit,
                                    const unsigned long long* s_h = nullptr, const CtlSnap* pre = nullptr) {
  DevCtl* c = a.ctl;
  const uint32_t n = a.n_global;
  const uint32_t nchunks = (n + 31u) / 32u;  // <= 128 (populations up to 4096)
  __shared__ double s_chunkmax[128];
  __shared__ double s_cur, s_target;
  __shared__ unsigned long long s_ni, s_calls_now;
  __shared__ int32_t s_exact, s_has_target, s_stopped;
  __shared__ uint32_t s_ver;
  if (threadIdx.x == 0) {
    // every control-block load first (independent of each other: one memory
    // round trip, or none when the caller loaded them), then the updates
    const CtlSnap k = pre ? *pre : load_ctl_snap(a);
    int32_t stop = k.stop;
    if (a.R == 1) {
      c->grp_steps = 0;
      c->grp_calls = 0;
    }
    const unsigned long long ct = k.calls_total + k.ca;
    c->calls_total = ct;
    c->run_steps = k.run_steps + k.st;
    c->run_calls = k.run_calls + k.ca;
    c->groups_run = k.groups_run + 1;
    a.gsteps[a.group] = k.gst + k.st;
    a.gcalls[a.group] = k.gca + k.ca;
    if (k.has_budget && (double)ct / k.q >= k.max_evals && !stop) {  // request_stop(budget)
      c->stop = 1;
      c->stop_reason = GOMIX_STOP_BUDGET;
      stop = 1;
    }
    s_stopped = stop;
    s_ver = k.ver;
    s_cur = k.elit_fit;
    s_target = k.target;
    s_ni = k.n_impr;
    s_calls_now = ct;
    s_exact = k.exact;
    s_has_target = k.has_target;
  }
  timeline_mark(9, -1);  // scan: control block accounted
  __syncthreads();
  // chunk maxima let the serial scan skip chunks that cannot hold a record:
  // precomputed by the CTAs that committed the chunks (a.word_max), else
  // one warp per chunk
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, nwarps = blockDim.x >> 5;
  auto fit_at = [&](uint32_t s) { return (s_fit && s < kEpiSmemFit) ? s_fit[s] : a.fit_all[s]; };
  if (a.word_max != nullptr && a.R == 1) {
    for (uint32_t chunk = threadIdx.x; chunk < nchunks; chunk += blockDim.x) s_chunkmax[chunk] = __ldcg(a.word_max + chunk);
  } else {
#pragma unroll 4
    for (uint32_t chunk = warp; chunk < nchunks; chunk += nwarps) {
      const uint32_t s = chunk * 32u + lane;
      double f = s < n ? fit_at(s) : -INFINITY;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) f = fmax(f, __shfl_xor_sync(0xFFFFFFFFu, f, o));
      if (lane == 0) s_chunkmax[chunk] = f;
    }
  }
  __syncthreads();
  timeline_mark(10, -1);  // scan: chunk maxima
  if (warp == 0) {
    const bool exact = s_exact != 0;
    const int32_t has_target = s_has_target;
    const double target = s_target;
    unsigned long long ni = s_ni;
    const unsigned long long calls_now = s_calls_now;
    double cur = s_cur;
    int32_t best = -1;
    bool hit = false;
    // the chunks that can hold a record, found 32 at a time: the running
    // elitist only rises, so a chunk whose maximum does not beat its value
    // at scan start never will (steady state: none qualifies — the serial
    // walk over all chunks cost ~150 cycles each, 10 us at n = 4096)
    const double cur0 = cur;
    for (uint32_t q = 0; q * 32u < nchunks; ++q) {
     uint32_t cand = __ballot_sync(0xFFFFFFFFu, q * 32u + lane < nchunks && s_chunkmax[q * 32u + lane] > cur0);
     while (cand) {
      const uint32_t chunk = q * 32u + (uint32_t)(__ffs(cand) - 1);
      cand &= cand - 1u;
      if (!(s_chunkmax[chunk] > cur)) continue;  // better() implies >
      const uint32_t base = chunk * 32u;
      const uint32_t s = base + lane;
      const double f = s < n ? fit_at(s) : -INFINITY;
      uint32_t m = __ballot_sync(0xFFFFFFFFu, s < n && cmp_better(exact, f, cur));
      while (m) {
        const uint32_t l = __ffs(m) - 1;
        cur = __shfl_sync(0xFFFFFFFFu, f, l);
        best = (int32_t)(base + l);
        if (lane == 0 && ni < a.impr_cap) {
          a.impr[ni].fit = cur;
          a.impr[ni].calls = calls_now;
        }
        ++ni;
        hit |= has_target && (cmp_better(exact, cur, target) || cmp_equal(exact, cur, target));
        m = __ballot_sync(0xFFFFFFFFu, s < n && lane > l && cmp_better(exact, f, cur));
      }
     }
    }
    if (lane == 0) {
      c->n_impr = ni;
      if (hit && !s_stopped) {  // request_stop(target): the budget stop, if any, came first
        c->stop = 1;
        c->stop_reason = GOMIX_STOP_TARGET;
      }
      if (best >= 0) {  // new elitist: member `best` (snapshot taken copy-on-write)
        c->elit_fit = cur;
        c->elit_src = best;
        if (s_h && (uint32_t)best < kEpiSmemFit) {
          c->eh1 = s_h[2 * best];
          c->eh2 = s_h[2 * best + 1];
        } else {
          c->eh1 = a.h1_all[best];
          c->eh2 = a.h2_all[best];
        }
        c->elit_ver = s_ver + 1;
      }
    }
  }
  timeline_mark(11, -1);  // scan: done (warp 0)
  __syncthreads();
}

// After this rank's members are committed: the elitist scan (one GPU), or
// the rank's counters for the exchange and — with the peer transport — the
// exchange and the global scan in the same kernel (gom_peer.cuh; with NCCL
// they follow the launch).
static __device__ void epilogue_global(const EpiArgs& a, const double* s_fit, const unsigned long long* s_h,
                                       const CtlSnap* pre = nullptr) {
  if (a.R == 1) {
    elitist_scan(a, s_fit, s_h, pre);
    return;
  }
  if (threadIdx.x == 0) {  // this rank's counters, all-gathered next
    DevCtl* c = a.ctl;
    a.rank_cnt[2 * a.rank] = c->grp_steps;
    a.rank_cnt[2 * a.rank + 1] = c->grp_calls;
    c->grp_steps = 0;
    c->grp_calls = 0;
  }
  __syncthreads();
  if (a.peer != nullptr && peer_exchange(a)) elitist_scan(a, nullptr);
}

static __device__ void epilogue_body(const EpiArgs& a) {
  __shared__ double s_fit[kEpiSmemFit];              // this group's fitness, scanned without global loads
  __shared__ unsigned long long s_h[2 * kEpiSmemFit];  // ... and hashes (a new elitist's)
  __shared__ CtlSnap s_snap;
  // one CTA: the scan's control-block loads in flight with the commit's —
  // issued by the last thread, parked in registers until its commit share
  // is done (a thread that stored them right away would wait for them first)
  const bool loader = a.R == 1 && threadIdx.x == blockDim.x - 1;
  CtlSnap pre;
  if (loader) pre = load_ctl_snap(a);
  commit_range(a, 0, a.n, a.R == 1 ? s_fit : nullptr, a.R == 1 ? s_h : nullptr);
  if (loader) s_snap = pre;
  __syncthreads();
  timeline_mark(8, -1);  // epilogue: committed
  epilogue_global(a, s_fit, s_h, a.R == 1 ? &s_snap : nullptr);
}

}  // namespace gomix_b200
