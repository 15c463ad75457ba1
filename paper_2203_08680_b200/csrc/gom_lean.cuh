// gom_lean.cuh — one (linkage set, population word) unit of a colour group,
// executed by ONE warp with no block-level synchronisation: phases 1-4 of
// engine_parallel.hpp:104-247 for the 32 solutions of word w.  Philox mode,
// one population shard, integer weights, |F| <= 32.
//
// Same donors, deltas and decisions as gom_general_set (same Philox counters
// and the same candidate / k-th-differing-member draw), bit for bit, but with
// the set's data moved between "lane = variable" and "lane = solution" views
// by 32x32 ballot transposes instead of shared-memory staging passes:
//   * the rows of F (every pool word) are staged once per warp; a transpose
//     per word turns them into every member's pattern on F;
//   * the donors' patterns, transposed back, are the donor-inserted row words
//     (lane jv = variable jv) — the evaluation reads them with shuffles;
//   * the commit is one ballot of the accept bits and one masked merge per
//     variable lane.
// A warp owns a fixed word w of every set it processes, so warps never share
// rows and need no barrier; per-warp shared memory holds F's rows, the
// members' patterns and F's Zobrist keys.
#pragma once

#include "gom_common.cuh"

namespace gomix_b200 {

constexpr uint32_t kLeanMaxF = 32;       // set size (variables per lane view)
constexpr uint32_t kLeanMaxWords = 8;    // pool words (n <= 256)
constexpr uint32_t kLeanSmemWords = kLeanMaxF * kLeanMaxWords + kLeanMaxWords * 32 + 2 * 2 * kLeanMaxF;

// The unit's population-independent inputs (plan record, F's variables, its
// first footprint chunk): loaded ahead, e.g. during the grid barrier before
// the unit's group, so the group's critical path starts at the row loads.
struct LeanPre {
  uint4 gm;    // {set id, vars offset, footprint offset, f << 24 | footprint}
  uint32_t vj; // lane jv: variable jv of F
  FpEntry e0;  // lane t: footprint entry t
};

__device__ __forceinline__ LeanPre lean_prefetch(const GomArgs& a, const uint4* gmeta, uint32_t p, uint32_t lane) {
  LeanPre r;
  r.gm = gmeta[p];
  const uint32_t f = r.gm.w >> 24;
  r.vj = lane < f ? a.set_vars[r.gm.y + lane] : 0u;
  const uint32_t e = r.gm.z + lane, e1 = r.gm.z + (r.gm.w & 0xFFFFFFu);
  if (e < e1) {
    r.e0 = a.fp[e];
  } else {
    r.e0.a = kInSet;
    r.e0.b = kInSet;
    r.e0.w = 0.0;
  }
  return r;
}

// What the accept / commit step needs from the previous colour group's
// epilogue: whether it stopped the run, and this lane's group-start
// "parent == elitist" with the elitist's column and snapshot version.
struct LeanGate {
  bool stop;
  bool is_elit;
  int32_t esrc;
  uint32_t ever_cur;
};

// gate(s) is called once per unit by every lane (s = its solution) right
// before the accept decision: everything up to there (donor draw, partial
// evaluation) depends only on the group-start rows, so it overlaps the
// previous group's epilogue when the caller runs that concurrently.  A gate
// that reports stop ends the unit with nothing committed or counted.
// MW: the population words the kernel was built for (>= Wp; the donor
// search's per-word masks are unrolled over MW).
template <uint32_t MW, class Gate>
__device__ __forceinline__ void gom_lean_unit(const GomArgs& a, uint32_t p, const LeanPre& pre, uint32_t w,
                                              uint32_t generation, uint32_t* wsm, uint32_t lane, Gate&& gate,
                                              bool record, long long& acc, unsigned long long& dh1,
                                              unsigned long long& dh2, uint32_t& steps, unsigned long long& calls,
                                              uint32_t sib_bar = 0u) {
  constexpr uint32_t FULL = 0xFFFFFFFFu;
  constexpr uint32_t Wp = MW;  // the kernel is instantiated for the population's row width (a.Wp)
  const uint32_t n = a.n, lwp = 31u - __clz(Wp);
  const uint4 gm = pre.gm;
  const uint32_t sid = gm.x, f = gm.w >> 24;
  const uint32_t* vars = a.set_vars + gm.y;
  const uint32_t e0 = gm.z, e1 = gm.z + (gm.w & 0xFFFFFFu);
  uint32_t* rowsW = wsm;                                         // [jv * Wp + wg]
  uint32_t* pattW = wsm + kLeanMaxF * kLeanMaxWords;             // [member]
  unsigned long long* zW = reinterpret_cast<unsigned long long*>(pattW + kLeanMaxWords * 32);  // [2 jv + {0,1}]
  const uint32_t vj = pre.vj;  // lane jv: variable jv of F
  // ---- F's rows at group start (the donor pool, engine_parallel.hpp:100-103)
  for (uint32_t base = 0; base < f * Wp; base += 32) {
    const uint32_t idx = base + lane;
    const uint32_t jv = min(idx >> lwp, 31u);
    const uint32_t v = __shfl_sync(FULL, vj, jv);
    if (idx < f * Wp) rowsW[idx] = a.pop[(size_t)v * Wp + (idx & (Wp - 1u))];
  }
  // first footprint chunk: entry per lane (prefetched) and its outside row word (word w)
  const FpEntry E0 = pre.e0;
  const uint32_t v0 = __shfl_sync(FULL, vj, 0);
  uint32_t xo0;
  {
    const uint32_t ext = !(E0.a & kInSet) ? E0.a : (!(E0.b & kInSet) ? E0.b : v0);
    xo0 = a.pop[(size_t)ext * Wp + w];
  }
  if (lane < f) zobrist(vj, zW[2 * lane], zW[2 * lane + 1]);
  __syncwarp();
  // The Wp warps of this set (one per population word, warps of one CTA)
  // each read ALL words of F's rows as the group-start donor pool and each
  // commits its own word: they meet at named barrier sib_bar (1 + their
  // index, 32 Wp threads) before committing, so no sibling reads a word
  // already committed.  The siblings walk the same unit sequence and take
  // the same gate decision, so every barrier is reached by all of them.
  // ---- every member's pattern on F: lane jv holds row jv, one transpose per word
  for (uint32_t wg = 0; wg < Wp; ++wg) {
    const uint32_t r = lane < f ? rowsW[lane * Wp + wg] : 0u;
    pattW[wg * 32u + lane] = transpose32(r, lane);
  }
  __syncwarp();
  const uint32_t s = w * 32u + lane;
  const bool valid = s < n;
  const uint32_t m = pattW[s];
  const uint32_t oldT = lane < f ? rowsW[lane * Wp + w] : 0u;  // lane jv: its row word w

  // ---- phase 1: donor (engine_serial.hpp:30-46 law; same draw as gom_general_set)
  int32_t d = -1;
  uint32_t x = m;
  if (valid) {
    const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
    const uint4 rr = philox4x32_10(make_uint4(s, sid, generation, kTagGom), key);
    const uint32_t c0 = bounded(lo64(rr), a.n_global);
    const uint32_t x0 = pattW[c0];
    if (x0 != m) {
      d = (int32_t)c0;
      x = x0;
    } else {
      // k-th member (k uniform) among those differing from m on F, in one
      // pass over F's rows: dwa[wg] = members of pool word wg that differ
      uint32_t dwa[MW];
#pragma unroll
      for (uint32_t wg = 0; wg < MW; ++wg) dwa[wg] = 0;
      for (uint32_t jv = 0; jv < f; ++jv) {
        const uint32_t mk = 0u - ((m >> jv) & 1u);
#pragma unroll
        for (uint32_t wg = 0; wg < MW; ++wg)
          if (wg < Wp) dwa[wg] |= rowsW[jv * Wp + wg] ^ mk;
      }
      uint32_t total = 0;
#pragma unroll
      for (uint32_t wg = 0; wg < MW; ++wg) {
        if (wg < Wp) dwa[wg] &= valid_mask(wg, n);
        total += __popc(dwa[wg]);
      }
      if (total > 0) {
        uint32_t kth = bounded(hi64(rr), total);
#pragma unroll
        for (uint32_t wg = 0; wg < MW; ++wg) {
          const uint32_t c = __popc(dwa[wg]);
          if (d < 0) {
            if (kth < c)
              d = (int32_t)(wg * 32u + select_bit(dwa[wg], kth));
            else
              kth -= c;
          }
        }
        x = pattW[d];
      }
    }
  }
  const bool present = d >= 0;
  const uint32_t xT = transpose32(x, lane);  // lane jv: donor-inserted row word of variable jv

  // ---- phase 2: delta over the footprint, ascending edge id (:164-173);
  // lane t = entry t: old / new cut words of the 32 solutions, transposed to
  // lane = solution, weighted popcounts over the weight bit-planes (exact)
  int32_t di = 0;
  for (uint32_t base = e0; base < e1; base += 32) {
    FpEntry E;
    uint32_t xo;
    if (base == e0) {
      E = E0;
      xo = xo0;
    } else {
      const uint32_t e = base + lane;
      if (e < e1) {
        E = a.fp[e];
      } else {
        E.a = kInSet;
        E.b = kInSet;
        E.w = 0.0;
      }
      const uint32_t ext = !(E.a & kInSet) ? E.a : (!(E.b & kInSet) ? E.b : v0);
      xo = a.pop[(size_t)ext * Wp + w];
    }
    const bool ina = E.a & kInSet, inb = E.b & kInSet;
    const uint32_t pa = E.a & 31u, pb = E.b & 31u;  // in-set positions (< 32)
    const uint32_t oA = __shfl_sync(FULL, oldT, pa), nA = __shfl_sync(FULL, xT, pa);
    const uint32_t oB = __shfl_sync(FULL, oldT, pb), nB = __shfl_sync(FULL, xT, pb);
    const uint32_t aO = ina ? oA : xo, aN = ina ? nA : xo;
    const uint32_t bO = inb ? oB : xo, bN = inb ? nB : xo;
    const uint32_t nz = E.w != 0.0 ? FULL : 0u;
    const uint32_t mo = transpose32((aO ^ bO) & nz, lane);
    const uint32_t mn = transpose32((aN ^ bN) & nz, lane);
    const int32_t wt = (int32_t)E.w;
    const uint32_t aw = wt < 0 ? (uint32_t)(-wt) : (uint32_t)wt;
    for (uint32_t k = 0; k < a.wbits; ++k) {
      const uint32_t bp = __ballot_sync(FULL, wt > 0 && ((aw >> k) & 1u));
      const uint32_t bn = __ballot_sync(FULL, wt < 0 && ((aw >> k) & 1u));
      di += ((int32_t)(__popc(mn & bp) - __popc(mo & bp)) - (int32_t)(__popc(mn & bn) - __popc(mo & bn))) << k;
    }
  }
  const int32_t delta = (e1 == e0) ? 0 : di;

  // ---- phases 3 + 4: accept (:194-214, exact comparator) and commit (:221-247)
  const LeanGate gt = gate(s);
  if (gt.stop) {
    __syncwarp();
    return;
  }
  const bool is_elit = gt.is_elit;
  const int32_t esrc = gt.esrc;
  const uint32_t ever_cur = gt.ever_cur;
  const bool accept = present && (delta > 0 || (delta == 0 && !is_elit));
  const uint32_t accw = __ballot_sync(FULL, accept);
  if (Wp > 1 && sib_bar != 0u) asm volatile("bar.sync %0, %1;" ::"r"(sib_bar), "r"(32u * Wp) : "memory");
  if (lane < f) {
    const uint32_t nw = (oldT & ~accw) | (xT & accw);
    if (nw != oldT) a.pop[(size_t)vj * Wp + w] = nw;
  }
  if (accept) {
    acc += delta;
    uint32_t changed = (x ^ m) & (f >= 32 ? FULL : ((1u << f) - 1u));
    const bool cap = (int32_t)s == esrc;
    while (changed) {
      const uint32_t jv = (uint32_t)(__ffs(changed) - 1);
      changed &= changed - 1;
      dh1 ^= zW[2 * jv];
      dh2 ^= zW[2 * jv + 1];
      if (cap) capture_row(a.elit, a.ever, ever_cur, vars[jv], (m >> jv) & 1u);
    }
  }
  steps += present ? 1u : 0u;
  calls += present ? (e1 - e0) : 0u;
  if (record && valid) {
    const size_t at = (size_t)p * n + s;
    a.rec_donor[at] = d;
    a.rec_delta[at] = (double)delta;
    a.rec_present[at] = present;
    a.rec_accept[at] = accept;
  }
  __syncwarp();  // the next unit overwrites this warp's shared rows / patterns / keys
}

}  // namespace gomix_b200
