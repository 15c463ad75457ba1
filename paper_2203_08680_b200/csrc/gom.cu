// gom.cu — the hot path: one batched GOM step per colour class with its fused
// epilogue (fitness commit, elitist scan, stop criteria), the elitist
// snapshot / hashing kernels, and the population init / full-evaluation kernels.
//
// Reference semantics (proj/include/gomix/engine_parallel.hpp):
//   phase 1 insert_donor_genes        :104-121  -> donor per (s, set): replay tape
//                                                  or counter-based Philox draw
//   phase 2 parallel_partial_evals    :130-187  -> delta = sum_new - sum_old over the
//                                                  set's footprint, ascending edge id
//   phase 3 determine_improvements    :194-214  -> accept iff better, or equal and the
//                                                  parent is not the elitist
//   phase 4 apply_acceptance          :221-247  -> commit bits / fitness in place
//   elitist scan                      :305-310  -> epilogue_kernel
// all fused into gom_group_kernel: nothing per pair is materialised in HBM.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

#include "gom_common.cuh"
#include "gom_general.cuh"
#include "gom_tail.cuh"

namespace gomix_b200 {

// Sharded runs: after the all-gather of populations, fitness, hashes and
// counters, every rank runs the same scan.
__global__ void global_epilogue_kernel(const EpiArgs a) {
  if (*(volatile int32_t*)&a.ctl->stop) return;
  elitist_scan(a, nullptr);
}

// ---------------------------------------------------------------------------
// hashes and the elitist snapshot
// ---------------------------------------------------------------------------
// h[s] = XOR of key(v) over the variables of solution s set to 1.  A warp takes
// 32 rows of one word column; lane k accumulates solution 32w+k.
__global__ void hash_population_kernel(const SnapArgs a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t Wp = a.Wp;
  const uint64_t blocks = (a.nv + 31) / 32;
  for (uint64_t unit = gwarp; unit < blocks * Wp; unit += nwarps) {
    const uint32_t w = (uint32_t)(unit % Wp);
    if (w * 32u >= a.n) continue;
    const uint64_t v = (unit / Wp) * 32u + lane;
    const uint32_t x = v < a.nv ? a.pop[v * Wp + w] : 0u;
    unsigned long long z1 = 0, z2 = 0;
    if (v < a.nv) zobrist((uint32_t)v, z1, z2);
    unsigned long long h1 = 0, h2 = 0;
    for (int r = 0; r < 32; ++r) {
      const uint32_t xr = __shfl_sync(0xFFFFFFFFu, x, r);
      const unsigned long long a1 = __shfl_sync(0xFFFFFFFFu, z1, r), a2 = __shfl_sync(0xFFFFFFFFu, z2, r);
      if ((xr >> lane) & 1u) {
        h1 ^= a1;
        h2 ^= a2;
      }
    }
    const uint32_t s = w * 32u + lane;
    if (s < a.n && (h1 | h2)) {
      atomicXor(&a.h1[s], h1);
      atomicXor(&a.h2[s], h2);
    }
  }
}

// Complete the copy-on-write snapshot: rows not captured since the elitist was
// chosen still hold its bit in population column elit_src.
__global__ void finalize_elitist_kernel(const SnapArgs a) {
  const DevCtl* c = a.ctl;
  const int32_t src = c->elit_src;
  if (src < 0) return;
  // column of global member src: shard src / n, local index src % n
  const uint32_t owner = (uint32_t)src / a.n, loc = (uint32_t)src % a.n;
  const uint32_t ver = c->elit_ver, sw = loc >> 5, sb = loc & 31u;
  const uint32_t* rows = a.pool + (uint64_t)owner * a.nv * a.Wp;
  const uint64_t words = (a.nv + 31) / 32;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < words;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t word = a.elit[t];
    for (uint32_t k = 0; k < 32 && t * 32 + k < a.nv; ++k) {
      const uint64_t v = t * 32 + k;
      if (a.ever[v] != ver) {
        const uint32_t b = (rows[v * a.Wp + sw] >> sb) & 1u;
        word = (word & ~(1u << k)) | (b << k);
        a.ever[v] = ver;
      }
    }
    a.elit[t] = word;
  }
}

// offer_elitist (engine_parallel.hpp:320-322): the elitist bits were uploaded;
// recompute its hash, mark the snapshot complete.
__global__ void external_elitist_reset_kernel(DevCtl* c, double fitness) {
  c->elit_fit = fitness;
  c->elit_src = -2;
  c->eh1 = 0;
  c->eh2 = 0;
  c->elit_ver += 1;
}

__global__ void external_elitist_hash_kernel(const SnapArgs a) {
  unsigned long long h1 = 0, h2 = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if ((a.elit[v >> 5] >> (v & 31u)) & 1u) {
      unsigned long long z1, z2;
      zobrist((uint32_t)v, z1, z2);
      h1 ^= z1;
      h2 ^= z2;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    h1 ^= __shfl_xor_sync(0xFFFFFFFFu, h1, o);
    h2 ^= __shfl_xor_sync(0xFFFFFFFFu, h2, o);
  }
  if ((threadIdx.x & 31u) == 0 && (h1 | h2)) {
    atomicXor(&a.ctl->eh1, h1);
    atomicXor(&a.ctl->eh2, h2);
  }
}

// ---------------------------------------------------------------------------
// IMS elitist exchange on the device (ImsDriver::collect / offer_elitist,
// ims.hpp:77-95, engine_parallel.hpp:320-322): the decision is taken by one
// thread, the ℓ-bit copy by the grid, so no host round trip is needed.
// ---------------------------------------------------------------------------
__global__ void ims_collect_decide_kernel(const DevCtl* c, ImsBestDev* b, int exact) {
  const bool take = c->elit_src != -1 && (!b->valid || cmp_better(exact != 0, c->elit_fit, b->fit));
  b->flag = take;
  if (take) b->pending = c->elit_fit;
}

// best bits = the engine's elitist genotype (copy-on-write snapshot rows where
// captured, otherwise population column elit_src; elit_src == -2: given bits)
__global__ void ims_collect_copy_kernel(const SnapArgs a, ImsBestDev* b, uint32_t* bits) {
  if (!*(volatile int32_t*)&b->flag) return;
  const DevCtl* c = a.ctl;
  const int32_t src = c->elit_src;
  const uint32_t ver = c->elit_ver;
  const uint64_t words = (a.nv + 31) / 32;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < words;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t word = a.elit[t];
    if (src >= 0) {
      const uint32_t sw = (uint32_t)src >> 5, sb = (uint32_t)src & 31u;
      for (uint32_t k = 0; k < 32 && t * 32 + k < a.nv; ++k) {
        const uint64_t v = t * 32 + k;
        if (a.ever[v] != ver) word = (word & ~(1u << k)) | (((a.pop[v * a.Wp + sw] >> sb) & 1u) << k);
      }
    }
    bits[t] = word;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    b->fit = b->pending;
    b->valid = 1;
  }
}

__global__ void ims_offer_decide_kernel(DevCtl* c, ImsBestDev* b, int exact) {
  const bool take = b->valid && cmp_better(exact != 0, b->fit, c->elit_fit);
  b->flag = take;
  if (take) {
    c->elit_fit = b->fit;
    c->elit_src = -2;
    c->eh1 = 0;
    c->eh2 = 0;
    c->elit_ver += 1;
  }
}

__global__ void ims_offer_copy_kernel(const SnapArgs a, const ImsBestDev* b, const uint32_t* bits) {
  if (!*(volatile const int32_t*)&b->flag) return;
  unsigned long long h1 = 0, h2 = 0;
  const uint64_t words = (a.nv + 31) / 32;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < words;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t word = bits[t];
    a.elit[t] = word;
    for (uint32_t m = word; m; m &= m - 1) {
      unsigned long long z1, z2;
      zobrist((uint32_t)(t * 32 + (__ffs(m) - 1)), z1, z2);
      h1 ^= z1;
      h2 ^= z2;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    h1 ^= __shfl_xor_sync(0xFFFFFFFFu, h1, o);
    h2 ^= __shfl_xor_sync(0xFFFFFFFFu, h2, o);
  }
  if ((threadIdx.x & 31u) == 0 && (h1 | h2)) {
    atomicXor(&a.ctl->eh1, h1);
    atomicXor(&a.ctl->eh2, h2);
  }
}

// A row's words owned by this thread: all WPT words (vector loads) for a
// one-warp team, every tw-th word otherwise.
template <int WPT, bool TEAM>
__device__ __forceinline__ void load_words(const uint32_t* row, uint32_t wit, uint32_t tw, uint32_t (&o)[WPT]) {
  if constexpr (!TEAM && WPT == 4) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(row));
    o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
  } else if constexpr (!TEAM && WPT == 8) {
    const uint4 t0 = __ldg(reinterpret_cast<const uint4*>(row));
    const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(row) + 1);
    o[0] = t0.x; o[1] = t0.y; o[2] = t0.z; o[3] = t0.w;
    o[4] = t1.x; o[5] = t1.y; o[6] = t1.z; o[7] = t1.w;
  } else if constexpr (!TEAM && WPT == 2) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(row));
    o[0] = t.x; o[1] = t.y;
  } else {
#pragma unroll
    for (int j = 0; j < WPT; ++j) o[j] = row[wit + tw * j];
  }
}

// Write back the words of a row that changed (one vector store for a
// one-warp team).
template <int WPT, bool TEAM>
__device__ __forceinline__ void store_words(uint32_t* row, uint32_t wit, uint32_t tw, const uint32_t (&old)[WPT],
                                            const uint32_t (&nw)[WPT]) {
  if constexpr (!TEAM && WPT == 4) {
    *reinterpret_cast<uint4*>(row) = make_uint4(nw[0], nw[1], nw[2], nw[3]);
  } else if constexpr (!TEAM && WPT == 2) {
    *reinterpret_cast<uint2*>(row) = make_uint2(nw[0], nw[1]);
  } else {
#pragma unroll
    for (int j = 0; j < WPT; ++j)
      if (nw[j] != old[j]) row[wit + tw * j] = nw[j];
  }
}


// ---------------------------------------------------------------------------
// gom_group_kernel
//
// Work decomposition: a *team* (one warp, or the whole CTA when n > 256)
// owns one linkage set at a time; inside the team, lane b of the warp that
// holds word w is solution 32w+b, and each thread carries WPT words.  Teams
// stride over the group's sets (persistent grid sized to the SM count), so
// per-solution fitness / elitist-distance deltas accumulate in registers and
// reach HBM once per CTA.  Same-colour sets share no variable and no
// interaction edge (scheduling.hpp:22-27), so teams update their rows in place
// without races and without a shadow copy.  A set's footprint (its CSR row,
// or its FpEntry list) and the neighbour rows it needs are fetched by the
// lanes in parallel — one coalesced round of loads per 32 entries — then
// broadcast with shuffles, so the sums below run without dependent loads.
// The last CTA to finish runs the epilogue, so a group is one launch.
// ---------------------------------------------------------------------------
template <int WPT, bool UNIV, bool I32, bool TEAM>
// univariate launches with WPT <= 4 always use <= 256 threads: allow 3 CTAs/SM
__global__ void __launch_bounds__((UNIV && WPT <= 4) ? 256 : 512, (UNIV && WPT <= 4) ? 3 : 1)
    gom_group_kernel(const GomArgs a) {
  extern __shared__ __align__(16) uint32_t smem[];
  if (*(volatile int32_t*)&a.ctl->stop) return;

  using Acc = long long;  // fixed-point fitness deltas (GomArgs::fix_scale)
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  // TEAM: the CTA is one team of tw warps; otherwise every warp is a team
  // holding all Wp == WPT words of its solutions (compile-time index math)
  const uint32_t tw = TEAM ? a.team_warps : 1u;
  const uint32_t teams_per_cta = TEAM ? 1u : (blockDim.x >> 5);
  const uint32_t team = TEAM ? 0u : warp, wit = TEAM ? warp : 0u;
  const uint32_t tid_team = wit * 32u + lane, team_threads = tw * 32u;
  const uint32_t Wp = a.Wp, n = a.n;
  const bool exact = I32 || a.exact != 0;  // integer-weight instances only take the I32 path
  const bool replay = a.tape != nullptr;
  const bool record = a.rec_present != nullptr;
  uint32_t* stage = smem + (size_t)team * a.stage_words;
  uint32_t G = a.G, generation = a.generation;
  const uint32_t* gsets = a.gsets;
  const uint32_t* gvars = a.gvars;
  const uint4* gmeta = a.gmeta;
  EpiArgs epi = a.epi;
  if (a.slot >= 0) {  // graph path: this launch's group comes from the device-side order
    const uint32_t gi = a.order[a.slot];
    const GroupDesc d = a.groups[gi];
    G = d.G;
    gsets += d.g0;
    if (gvars) gvars += d.g0;
    if (gmeta) gmeta += d.g0;
    generation = *(volatile unsigned int*)&a.ctl->cur_gen;
    epi.group = gi;
    epi.G = G;
  }

  // group-start state of this thread's solutions: "parent == elitist"
  // (engine_parallel.hpp:202) and the parent fitness, read once per launch
  const unsigned long long eh1 = a.ctl->eh1, eh2 = a.ctl->eh2;
  const int32_t esrc = a.ctl->elit_src;        // copy-on-write snapshot source
  const uint32_t ever_cur = a.ctl->elit_ver;
  bool is_elit[WPT];
  double pfit[WPT];
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    const uint32_t s = (wit + tw * (uint32_t)j) * 32u + lane;
    is_elit[j] = s < n && a.h1[s] == eh1 && a.h2[s] == eh2;
    pfit[j] = (!exact && s < n) ? a.fit[s] : 0.0;
  }
  Acc acc[WPT];
  unsigned long long dh1[WPT], dh2[WPT];
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    acc[j] = 0;
    dh1[j] = 0;
    dh2[j] = 0;
  }
  uint32_t steps = 0;
  unsigned long long calls = 0;

  for (uint32_t p = blockIdx.x * teams_per_cta + team; p < G; p += gridDim.x * teams_per_cta) {
    if constexpr (UNIV) {
      // ---- univariate set {v}: a donor differing on v holds !x_v, so the
      // pair is present iff some member holds the other value and the move
      // is the flip of v; in Philox mode the draw cannot change the outcome
      // and is skipped.
      const uint32_t v = gvars[p];
      const uint32_t* row = a.pop + (size_t)v * Wp;
      uint32_t pw[WPT];
#pragma unroll
      for (int j = 0; j < WPT; ++j) pw[j] = 0;
      load_words<WPT, TEAM>(row, wit, tw, pw);
      const int32_t rs = a.row_ptr[v], re = a.row_ptr[v + 1];
      uint32_t ones = 0;  // members holding 1 at v, over every rank's shard
      if (!replay) {
        if (a.ones) {
          ones = a.ones[v];  // sharded, variable-once FOS: counted at generation start
        } else if (a.R > 1) {
          for (uint32_t wg = lane; wg < a.R * Wp; wg += 32)
            ones += __popc(a.pool[((size_t)(wg / Wp) * a.nv + v) * Wp + (wg % Wp)]);
          ones = __reduce_add_sync(0xFFFFFFFFu, ones);
        } else if (tw == 1) {
#pragma unroll
          for (int j = 0; j < WPT; ++j) ones += __popc(pw[j]);
        } else {
          for (uint32_t w = lane; w < Wp; w += 32) ones += __popc(row[w]);
          ones = __reduce_add_sync(0xFFFFFFFFu, ones);
        }
      }
      const uint32_t deg = (uint32_t)(re - rs);
      int32_t di[WPT];
      double sn[WPT], so[WPT];
#pragma unroll
      for (int j = 0; j < WPT; ++j) {
        di[j] = 0;
        sn[j] = 0.0;
        so[j] = 0.0;
      }
      for (int32_t base = rs; base < re; base += 32) {
        const int32_t e = base + (int32_t)lane;
        const bool has = e < re;
        const uint32_t u = has ? (uint32_t)a.col[e] : v;
        int32_t wti = 0;
        double wtd = 0.0;
        if constexpr (I32) wti = has ? a.wi[e] : 0;
        else wtd = has ? a.w[e] : 0.0;
        uint32_t nb[WPT];
#pragma unroll
        for (int j = 0; j < WPT; ++j) nb[j] = 0;
        load_words<WPT, TEAM>(a.pop + (size_t)u * Wp, wit, tw, nb);
        const int cnt = min(32, re - base);
        for (int t = 0; t < cnt; ++t) {
          if constexpr (I32) {
            const int32_t wt = __shfl_sync(0xFFFFFFFFu, wti, t);
#pragma unroll
            for (int j = 0; j < WPT; ++j) {
              const uint32_t x = __shfl_sync(0xFFFFFFFFu, nb[j], t);
              di[j] += (((pw[j] ^ x) >> lane) & 1u) ? -wt : wt;
            }
          } else {
            const double wt = shfl_d(wtd, t);
#pragma unroll
            for (int j = 0; j < WPT; ++j) {
              const uint32_t cut_old = (((pw[j] ^ __shfl_sync(0xFFFFFFFFu, nb[j], t)) >> lane) & 1u);
              sn[j] += cut_old ? 0.0 : wt;  // reference adds every value, 0.0 included
              so[j] += cut_old ? wt : 0.0;
            }
          }
        }
      }
      // phases 3 + 4.  Philox mode: a singleton pair is present iff the row
      // holds both values among the members (per set, all or nothing).
      const bool set_present = ones > 0u && ones < a.n_global;
      uint32_t accb = 0;  // bit j: this lane accepted in word j
      uint32_t nw[WPT];
#pragma unroll
      for (int j = 0; j < WPT; ++j) {
        const uint32_t w = wit + tw * j;
        const uint32_t s = w * 32u + lane;
        const bool valid = s < n;
        const uint32_t pv = (pw[j] >> lane) & 1u;
        bool present;
        int32_t dn = -1;
        if (replay) {
          dn = valid ? a.tape[(size_t)p * n + s] : -1;
          present = dn >= 0;
        } else {
          present = valid && set_present;
          dn = present ? (int32_t)n : -1;  // donor identity is not materialised
        }
        bool accept = false;
        double delta;
        if constexpr (I32) {
          const int32_t d = di[j];
          delta = (double)d;
          accept = present && (d > 0 || (d == 0 && !is_elit[j]));
          if (accept) acc[j] += (Acc)d;
        } else {
          delta = sn[j] - so[j];
          if (present) {
            const double pf = pfit[j];
            const double cand = pf + delta;
            accept = exact ? (delta > 0.0 || (delta == 0.0 && !is_elit[j]))
                           : (cmp_better(false, cand, pf) || (cmp_equal(false, cand, pf) && !is_elit[j]));
          }
          if (accept) acc[j] += __double2ll_rn(delta * a.fix_scale);
        }
        nw[j] = pw[j] ^ __ballot_sync(0xFFFFFFFFu, accept);  // accepted members flip v
        accb |= accept ? (1u << j) : 0u;
        if (accept && (int32_t)(a.rank * n + s) == esrc) capture_row(a.elit, a.ever, ever_cur, v, pv);
        steps += present ? 1u : 0u;
        calls += present ? deg : 0u;
        if (record && valid) {
          const size_t at = (size_t)p * n + s;
          a.rec_donor[at] = dn;
          a.rec_delta[at] = present ? delta : 0.0;
          a.rec_present[at] = present;
          a.rec_accept[at] = accept;
        }
      }
      if (__any_sync(0xFFFFFFFFu, accb != 0)) {
        unsigned long long zv1, zv2;
        zobrist(v, zv1, zv2);
#pragma unroll
        for (int j = 0; j < WPT; ++j)
          if (accb & (1u << j)) {
            dh1[j] ^= zv1;
            dh2[j] ^= zv2;
          }
        if (lane == 0) store_words<WPT, TEAM>(a.pop + (size_t)v * Wp, wit, tw, pw, nw);
      }
    } else {
      gom_general_set<WPT, I32, TEAM>(a, p, gmeta, generation, stage, lane, tw, wit, tid_team, team_threads,
                                      teams_per_cta, team, exact, replay, record, is_elit, pfit, esrc, ever_cur,
                                      acc, dh1, dh2, steps, calls);
    }
  }

  gom_group_tail<WPT>(a, epi, smem, teams_per_cta, team, wit, tw, lane, acc, dh1, dh2, steps, calls);
}

__global__ void begin_call_kernel(const BeginArgs b) {
  DevCtl* c = b.ctl;
  c->stop = 0;
  c->stop_reason = GOMIX_STOP_NONE;
  c->has_budget = b.has_budget;
  c->has_target = b.has_target;
  c->exact = b.exact;
  c->max_evals = b.max_evals;
  c->q = b.q;
  c->target = b.target;
  c->calls_total = b.calls_before;
  c->grp_steps = c->grp_calls = 0;
  c->run_steps = c->run_calls = c->groups_run = 0;
  c->n_impr = 0;
  c->done = 0;
  c->cur_gen = b.gen;
  c->gen_counter = b.gen + 1;
}

constexpr uint32_t kTagOrder = 0x4F524400u;  // "ORD"

// Graph path: reset the per-call block and draw this generation's group
// order (Fisher-Yates, engine_parallel.hpp:291) from the counter-based stream.
__global__ void begin_generation_kernel(const BeginArgs* bp, const OrderArgs o) {
  // the first group's launch may start now: it waits for this kernel's
  // completion before reading the order or the control block
  asm volatile("griddepcontrol.launch_dependents;");
  timeline_mark(0);
  // the criteria (mapped host memory, staged before the launch was issued)
  // cross the bus while the previous kernel on the stream finishes: this
  // launch is programmatic, everything after the wait touches the control
  // block that kernel may still write
  const BeginArgs b = *bp;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  DevCtl* c = b.ctl;
  c->stop = 0;
  c->stop_reason = GOMIX_STOP_NONE;
  c->has_budget = b.has_budget;
  c->has_target = b.has_target;
  c->exact = b.exact;
  c->max_evals = b.max_evals;
  c->q = b.q;
  c->target = b.target;
  c->calls_total = b.calls_before;
  c->grp_steps = c->grp_calls = 0;
  c->run_steps = c->run_calls = c->groups_run = 0;
  c->n_impr = 0;
  c->done = 0;
  const uint32_t gen = c->gen_counter++;
  c->cur_gen = gen;
  const uint2 key = make_uint2((uint32_t)o.seed, (uint32_t)(o.seed >> 32));
  for (uint32_t i = 0; i < o.k; ++i) o.order[i] = i;
  for (uint32_t i = o.k; i > 1; --i) {
    const uint4 r = philox4x32_10(make_uint4(i, gen, 0u, kTagOrder), key);
    const uint32_t j = bounded(lo64(r), i);
    const uint32_t t = o.order[i - 1];
    o.order[i - 1] = o.order[j];
    o.order[j] = t;
  }
  timeline_mark(1);
}

// After init_population (engine_parallel.hpp:331-346): one add_evaluator_calls(q)
// per solution and "i == 0 || better" elitist updates, interleaved in order.
__global__ void init_epilogue_kernel(const EpiArgs a) {
  DevCtl* c = a.ctl;
  if (threadIdx.x == 0) {
    const bool exact = c->exact != 0;
    double cur = 0.0;
    int32_t best = -1;
    for (uint32_t i = 0; i < a.n_global; ++i) {
      c->calls_total += (unsigned long long)c->q;
      c->run_calls += (unsigned long long)c->q;
      if (c->has_budget && (double)c->calls_total / c->q >= c->max_evals)
        request_stop(c, GOMIX_STOP_BUDGET);
      const double f = a.fit_all[i];
      if (i == 0 || cmp_better(exact, f, cur)) {
        cur = f;
        best = (int32_t)i;
        note_improvement(a, f);
      }
    }
    c->elit_fit = cur;
    c->elit_src = best;
    c->eh1 = a.h1_all[best];
    c->eh2 = a.h2_all[best];
    c->elit_ver += 1;
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < a.n; s += blockDim.x) {
    a.dh1[s] = 0;
    a.dh2[s] = 0;
    a.dfit[s] = 0;
  }
}

// ---------------------------------------------------------------------------
// init / full evaluation / layout conversion
// ---------------------------------------------------------------------------
// Initial alleles: bit (v, g) of global member g is bit g%32 of Philox block
// (v, g/32), so a shard of the population draws exactly the bits the same
// members get in a single-GPU run.
// Members holding 1, per row (sharded univariate runs: summed over the ranks
// once per generation instead of all-gathering every row after every group).
__global__ void count_ones_kernel(const uint32_t* pop, uint64_t nv, uint32_t Wp, uint32_t* ones) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (uint32_t w = 0; w < Wp; ++w) c += __popc(pop[v * Wp + w]);
    ones[v] = c;
  }
}

__global__ void sum_ones_kernel(const uint32_t* stage, uint32_t R, uint64_t nv, uint32_t* ones) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (uint32_t r = 0; r < R; ++r) c += stage[(uint64_t)r * nv + v];
    ones[v] = c;
  }
}

__global__ void philox_init_kernel(uint32_t* pop, uint64_t nv, uint32_t n, uint32_t Wp,
                                   uint64_t seed, uint32_t rank) {
  const uint64_t total = nv * Wp;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = (uint32_t)(i % Wp);
    const uint64_t v = i / Wp;
    const uint64_t g0 = (uint64_t)rank * n + 32ull * w;  // global index of bit 0
    const uint64_t blk = g0 >> 5;
    const uint32_t off = (uint32_t)(g0 & 31u);
    uint32_t word = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)blk, kTagInit), key).x;
    if (off) {
      const uint32_t hi = philox4x32_10(make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(blk + 1), kTagInit), key).x;
      word = (word >> off) | (hi << (32u - off));
    }
    pop[i] = word & valid_mask(w, n);
  }
}

// Exact (integer) fitness: any summation order is exact -> parallel over edges.
__global__ void full_eval_parallel_kernel(const uint32_t* eu, const uint32_t* ev,
                                          const double* ew, uint64_t q, const uint32_t* pop,
                                          double* fit, uint32_t n, uint32_t Wp,
                                          uint64_t edges_per_chunk) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gwarp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t chunks = (q + edges_per_chunk - 1) / edges_per_chunk;
  for (uint64_t unit = gwarp; unit < chunks * Wp; unit += nwarps) {
    const uint32_t w = (uint32_t)(unit % Wp);
    if (w * 32u >= n) continue;
    const uint64_t e0 = (unit / Wp) * edges_per_chunk, e1 = min(e0 + edges_per_chunk, q);
    double sum = 0.0;
    for (uint64_t e = e0; e < e1; ++e) {
      const uint32_t x = pop[(uint64_t)eu[e] * Wp + w] ^ pop[(uint64_t)ev[e] * Wp + w];
      sum += ((x >> lane) & 1u) ? ew[e] : 0.0;
    }
    const uint32_t s = w * 32u + lane;
    if (s < n && sum != 0.0) atomicAdd(&fit[s], sum);
  }
}

// Float fitness, deterministic and parallel (production mode): a warp per
// solution, lane-strided partial sums combined by an xor butterfly.
__global__ void full_eval_warp_kernel(const uint32_t* eu, const uint32_t* ev, const double* ew, uint64_t q,
                                      const uint32_t* pop, double* fit, uint32_t n, uint32_t Wp) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n) return;
  const uint32_t w = s >> 5, b = s & 31u;
  double sum = 0.0;
  for (uint64_t e = lane; e < q; e += 32) {
    const uint32_t x = pop[(uint64_t)eu[e] * Wp + w] ^ pop[(uint64_t)ev[e] * Wp + w];
    sum += ((x >> b) & 1u) ? ew[e] : 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
  if (lane == 0) fit[s] = sum;
}

// Float fitness in the reference's left-to-right edge order (graybox.hpp:139-144).
__global__ void full_eval_ordered_kernel(const uint32_t* eu, const uint32_t* ev,
                                         const double* ew, uint64_t q, const uint32_t* pop,
                                         double* fit, uint32_t n, uint32_t Wp) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t w = s >> 5, b = s & 31u;
  double sum = 0.0;
  for (uint64_t e = 0; e < q; ++e) {
    const uint32_t x = pop[(uint64_t)eu[e] * Wp + w] ^ pop[(uint64_t)ev[e] * Wp + w];
    sum += ((x >> b) & 1u) ? ew[e] : 0.0;
  }
  fit[s] = sum;
}

__global__ void unpack_kernel(const uint32_t* pop, uint8_t* out, uint64_t nv, uint32_t n,
                              uint32_t Wp) {
  const uint64_t total = (uint64_t)n * nv;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = i / nv, v = i - s * nv;
    out[i] = (pop[v * Wp + (s >> 5)] >> (s & 31u)) & 1u;
  }
}

__global__ void pack_kernel(const uint8_t* in, uint32_t* pop, uint64_t nv, uint32_t n,
                            uint32_t Wp) {
  const uint64_t total = nv * Wp;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = i / Wp;
    const uint32_t w = (uint32_t)(i - v * Wp);
    uint32_t word = 0;
    for (uint32_t b = 0; b < 32; ++b) {
      const uint32_t s = w * 32u + b;
      if (s < n && in[(uint64_t)s * nv + v]) word |= 1u << b;
    }
    pop[i] = word;
  }
}

__global__ void pack_elitist_kernel(const uint8_t* in, uint32_t* elit, uint64_t nv) {
  const uint64_t nw = (nv + 31) / 32;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nw;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
    for (uint32_t k = 0; k < 32 && t * 32 + k < nv; ++k)
      if (in[t * 32 + k]) word |= 1u << k;
    elit[t] = word;
  }
}

__global__ void unpack_elitist_kernel(const uint32_t* elit, uint8_t* out, uint64_t nv) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv;
       v += (uint64_t)gridDim.x * blockDim.x)
    out[v] = (elit[v >> 5] >> (v & 31u)) & 1u;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {
template <int WPT, bool TEAM>
void* gom_kernel_ptr(bool univariate, bool i32) {
  if (univariate)
    return i32 ? (void*)gom_group_kernel<WPT, true, true, TEAM> : (void*)gom_group_kernel<WPT, true, false, TEAM>;
  return i32 ? (void*)gom_group_kernel<WPT, false, true, TEAM> : (void*)gom_group_kernel<WPT, false, false, TEAM>;
}

// instantiated shapes: one-warp teams with all words per lane (WPT = Wp <= 8),
// and CTA teams with WPT 1 (few sets), 4 or 8 words per thread (large n)
void* gom_kernel(bool univariate, bool i32, int wpt, bool team) {
  if (team) {
    switch (wpt) {
      case 1: return gom_kernel_ptr<1, true>(univariate, i32);
      case 4: return gom_kernel_ptr<4, true>(univariate, i32);
      case 8: return gom_kernel_ptr<8, true>(univariate, i32);
    }
  } else {
    switch (wpt) {
      case 1: return gom_kernel_ptr<1, false>(univariate, i32);
      case 2: return gom_kernel_ptr<2, false>(univariate, i32);
      case 4: return gom_kernel_ptr<4, false>(univariate, i32);
      case 8: return gom_kernel_ptr<8, false>(univariate, i32);
    }
  }
  throw GomixError(GOMIX_E_INVALID, "unsupported words-per-thread");
}

int grid_for(uint64_t work, int block, uint64_t cap) {
  uint64_t g = (work + block - 1) / block;
  if (g > cap) g = cap;
  return (int)(g ? g : 1);
}
}  // namespace

void prepare_gom(bool univariate, bool i32, int wpt, bool team, size_t smem) {
  void* fn = gom_kernel(univariate, i32, wpt, team);
  // opt in whenever dynamic + static shared memory may exceed the 48 KB default
  GOMIX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

void launch_gom(const GomArgs& a, bool univariate, bool i32, int wpt, bool team, int grid, int block,
                size_t smem, cudaStream_t s) {
  void* fn = gom_kernel(univariate, i32, wpt, team);
  void* args[] = {(void*)&a};
  GOMIX_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(block), args, smem, s));
}

int gom_max_blocks_per_sm(bool univariate, bool i32, int wpt, bool team, int block, size_t smem) {
  void* fn = gom_kernel(univariate, i32, wpt, team);
  GOMIX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = 0;
  GOMIX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, block, smem));
  return blocks;
}

void launch_begin(const BeginArgs& b, cudaStream_t s) {
  begin_call_kernel<<<1, 1, 0, s>>>(b);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_order(const BeginArgs* d_b, const OrderArgs& o, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GOMIX_CUDA(cudaLaunchKernelEx(&cfg, begin_generation_kernel, d_b, o));
}

// The control block and the first improvement-log entries, written straight
// into mapped pinned host memory, then a sequence number (system-scope
// release): a synchronous call spins on that number instead of a device-to-
// host copy plus a stream synchronisation.
__global__ void publish_ctl_kernel(const uint4* src, uint4* dst, uint32_t words, unsigned long long* seq_dst,
                                   unsigned long long seq) {
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(seq_dst), "l"(seq) : "memory");
}

void debug_timeline_gom(unsigned long long* out) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_timeline, sizeof(unsigned long long) * 32));
  unsigned long long z[32 * kTimelineRows];
  for (int i = 0; i < 32 * kTimelineRows; ++i) z[i] = (i & 1) ? 0ull : ~0ull;
  GOMIX_CUDA(cudaMemcpyToSymbol(g_timeline, z, sizeof(z)));
}

void launch_publish_ctl(const void* ctl, void* host_dst, size_t bytes, unsigned long long* host_seq,
                        unsigned long long seq, cudaStream_t s) {
  publish_ctl_kernel<<<1, 128, 0, s>>>(static_cast<const uint4*>(ctl), static_cast<uint4*>(host_dst),
                                       (uint32_t)(bytes / 16), host_seq, seq);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_global_epilogue(const EpiArgs& a, cudaStream_t s) {
  global_epilogue_kernel<<<1, 256, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_init_epilogue(const EpiArgs& a, cudaStream_t s) {
  init_epilogue_kernel<<<1, 256, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_hash_population(const SnapArgs& a, cudaStream_t s) {
  GOMIX_CUDA(cudaMemsetAsync(a.h1, 0, a.n * sizeof(unsigned long long), s));
  GOMIX_CUDA(cudaMemsetAsync(a.h2, 0, a.n * sizeof(unsigned long long), s));
  const uint64_t units = ((a.nv + 31) / 32) * a.Wp;
  hash_population_kernel<<<grid_for(units * 32, 256, 148 * 16), 256, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_finalize_elitist(const SnapArgs& a, cudaStream_t s) {
  finalize_elitist_kernel<<<grid_for((a.nv + 31) / 32, 256, 148 * 16), 256, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_external_elitist(const SnapArgs& a, double fitness, cudaStream_t s) {
  external_elitist_reset_kernel<<<1, 1, 0, s>>>(a.ctl, fitness);
  external_elitist_hash_kernel<<<grid_for(a.nv, 256, 148 * 8), 256, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_ims_collect(const SnapArgs& a, ImsBestDev* b, uint32_t* bits, int exact, cudaStream_t s) {
  ims_collect_decide_kernel<<<1, 1, 0, s>>>(a.ctl, b, exact);
  ims_collect_copy_kernel<<<grid_for((a.nv + 31) / 32, 256, 148 * 4), 256, 0, s>>>(a, b, bits);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_ims_offer(const SnapArgs& a, ImsBestDev* b, const uint32_t* bits, int exact, cudaStream_t s) {
  ims_offer_decide_kernel<<<1, 1, 0, s>>>(a.ctl, b, exact);
  ims_offer_copy_kernel<<<grid_for((a.nv + 31) / 32, 256, 148 * 4), 256, 0, s>>>(a, b, bits);
  GOMIX_CUDA(cudaGetLastError());
}

// Rows of Wp >= 4 words: Wp / 4 lanes per row, one 16-byte load each
// (a warp reads 512 contiguous bytes), counts summed across the row's lanes.
__global__ void count_ones_wide_kernel(const uint32_t* pop, uint64_t nv, uint32_t Wp, uint32_t* ones) {
  const uint32_t L = Wp >> 2;  // lanes per row (1 .. 32)
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t rows_per_warp = 32u / min(L, 32u);
  for (uint64_t base = warp * rows_per_warp; base < nv; base += nwarps * rows_per_warp) {
    uint32_t c = 0;
    for (uint32_t part = 0; part < max(1u, L / 32u); ++part) {  // rows wider than 128 words: several loads
      const uint64_t v = base + lane / min(L, 32u);
      const uint32_t q = (lane % min(L, 32u)) + part * 32u;
      if (v < nv) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(pop + v * Wp) + q);
        c += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
      }
    }
    for (uint32_t o = min(L, 32u) >> 1; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    const uint64_t v = base + lane / min(L, 32u);
    if (lane % min(L, 32u) == 0 && v < nv) ones[v] = c;
  }
}

void launch_count_ones(const uint32_t* pop, uint64_t nv, uint32_t Wp, uint32_t* ones, cudaStream_t s) {
  if (Wp >= 4)
    count_ones_wide_kernel<<<148 * 8, 256, 0, s>>>(pop, nv, Wp, ones);
  else
    count_ones_kernel<<<grid_for(nv, 256, 148 * 8), 256, 0, s>>>(pop, nv, Wp, ones);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_sum_ones(const uint32_t* stage, uint32_t R, uint64_t nv, uint32_t* ones, cudaStream_t s) {
  sum_ones_kernel<<<grid_for(nv, 256, 148 * 8), 256, 0, s>>>(stage, R, nv, ones);
  GOMIX_CUDA(cudaGetLastError());
}

void debug_probes(unsigned long long* out, bool reset) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_probe, sizeof(unsigned long long) * 64));
  if (reset) {
    unsigned long long z[64] = {};
    GOMIX_CUDA(cudaMemcpyToSymbol(g_probe, z, sizeof(z)));
  }
}

void launch_philox_init(uint32_t* pop, uint64_t nv, uint32_t n, uint32_t Wp, uint64_t seed,
                        uint32_t rank, cudaStream_t s) {
  philox_init_kernel<<<grid_for(nv * Wp, 256, 4096), 256, 0, s>>>(pop, nv, n, Wp, seed, rank);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_full_eval(const Problem& P, const uint32_t* pop, double* fit, uint32_t n,
                      uint32_t Wp, bool ordered, cudaStream_t s) {
  if (ordered) {
    full_eval_ordered_kernel<<<(n + 127) / 128, 128, 0, s>>>(P.eu, P.ev, P.ew, P.q, pop, fit, n, Wp);
  } else if (!P.exact) {
    full_eval_warp_kernel<<<(n + 7) / 8, 256, 0, s>>>(P.eu, P.ev, P.ew, P.q, pop, fit, n, Wp);
  } else {
    GOMIX_CUDA(cudaMemsetAsync(fit, 0, n * sizeof(double), s));
    const uint64_t chunk = 1024;
    const uint64_t units = ((P.q + chunk - 1) / chunk) * Wp;
    full_eval_parallel_kernel<<<grid_for(units * 32, 256, 4096), 256, 0, s>>>(
        P.eu, P.ev, P.ew, P.q, pop, fit, n, Wp, chunk);
  }
  GOMIX_CUDA(cudaGetLastError());
}

void launch_unpack(const uint32_t* pop, uint8_t* out, uint64_t nv, uint32_t n, uint32_t Wp,
                   cudaStream_t s) {
  unpack_kernel<<<grid_for(nv * n, 256, 8192), 256, 0, s>>>(pop, out, nv, n, Wp);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_pack(const uint8_t* in, uint32_t* pop, uint64_t nv, uint32_t n, uint32_t Wp,
                 cudaStream_t s) {
  pack_kernel<<<grid_for(nv * Wp, 256, 8192), 256, 0, s>>>(in, pop, nv, n, Wp);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_pack_elitist(const uint8_t* in, uint32_t* elit, uint64_t nv, cudaStream_t s) {
  pack_elitist_kernel<<<grid_for((nv + 31) / 32, 256, 4096), 256, 0, s>>>(in, elit, nv);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_unpack_elitist(const uint32_t* elit, uint8_t* out, uint64_t nv, cudaStream_t s) {
  unpack_elitist_kernel<<<grid_for(nv, 256, 4096), 256, 0, s>>>(elit, out, nv);
  GOMIX_CUDA(cudaGetLastError());
}

}  // namespace gomix_b200
