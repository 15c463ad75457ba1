// gom_general.cuh — one general linkage set F (|F| <= 64) of a colour class:
// phases 1-4 of engine_parallel.hpp:104-247 for every solution of this rank,
// executed by a team (one warp, or the whole CTA).  Shared by the per-group
// kernel (gom.cu) and the persistent generation kernel (gom_gen.cu).
#pragma once

#include <type_traits>

#include "gom_common.cuh"

namespace gomix_b200 {

template <int WPT, bool I32, bool TEAM>
__device__ __forceinline__ void gom_general_set(
    const GomArgs& a, uint32_t p, const uint4* gmeta, uint32_t generation, uint32_t* stage, uint32_t lane,
    uint32_t tw, uint32_t wit, uint32_t tid_team, uint32_t team_threads, uint32_t teams_per_cta, uint32_t team,
    bool exact, bool replay, bool record, const bool (&is_elit)[WPT], const double (&pfit)[WPT], int32_t esrc,
    uint32_t ever_cur, long long (&acc)[WPT],
    unsigned long long (&dh1)[WPT], unsigned long long (&dh2)[WPT], uint32_t& steps, unsigned long long& calls) {
  using Acc = long long;  // fixed-point fitness deltas (GomArgs::fix_scale)
  const uint32_t Wp = a.Wp, n = a.n;
  // ---- general set F (|F| <= 64).  Shared memory per team holds the F
  // rows at group start (the donor pool, engine_parallel.hpp:100-103),
  // every solution's pattern on F (so a donor test is one load), the
  // donor-inserted rows and the committed rows.
  probe(a.exp_flags, 0);
  const uint4 gm = gmeta[p];
  const uint32_t sid = gm.x;
  const uint32_t f = gm.w >> 24;
  const uint32_t* vars = a.set_vars + gm.y;
  const uint32_t e0 = gm.z, e1 = gm.z + (gm.w & 0xFFFFFFu);
  // pool words: RW = R*Wp per row (every rank's shard; R == 1: the population)
  const uint32_t RW = a.R * Wp, own = a.rank * Wp;
  probe(a.exp_flags, 1);
  uint64_t* patt = reinterpret_cast<uint64_t*>(stage);  // pattern of every member (padded index)
  uint32_t* rowsF = stage + 64u * RW;                    // F rows at group start, stride RW
  uint32_t* newD = rowsF + f * RW;                       // own donor-inserted rows, stride Wp
  uint32_t* newF = newD + f * Wp;                        // own committed rows, stride Wp
  const uint32_t lwp = 31u - __clz(Wp);  // Wp is a power of two
  for (uint32_t jv = 0; jv < f; ++jv) {
    const size_t v = vars[jv];
    for (uint32_t wg = tid_team; wg < RW; wg += team_threads)
      rowsF[jv * RW + wg] = a.pool[((size_t)(wg >> lwp) * a.nv + v) * Wp + (wg & (Wp - 1u))];
  }
  // first footprint chunk: entry per lane and its outside row, fetched
  // now so the loads overlap the staging above
  FpEntry E0;
  uint32_t xw0[WPT];
  {
    const uint32_t e = e0 + lane;
    if (e < e1) {
      E0 = a.fp[e];
    } else {
      E0.a = kInSet;
      E0.b = kInSet;
      E0.w = 0.0;
    }
    const uint32_t ext = !(E0.a & kInSet) ? E0.a : (!(E0.b & kInSet) ? E0.b : vars[0]);
#pragma unroll
    for (int j = 0; j < WPT; ++j) xw0[j] = a.pop[(size_t)ext * Wp + wit + tw * j];
  }
  // Zobrist keys of F, 8-byte aligned: offset from the (aligned) stage is
  // 64*RW + f*RW + 2*f*Wp, so pad by the parity of f*RW
  unsigned long long* zF = reinterpret_cast<unsigned long long*>(newF + f * Wp + ((f * RW) & 1u));
  for (uint32_t jv = tid_team; jv < f; jv += team_threads) zobrist(vars[jv], zF[2 * jv], zF[2 * jv + 1]);
  const uint64_t fm = f >= 64 ? ~0ull : ((1ull << f) - 1ull);
  team_sync(tw, teams_per_cta, team);
  probe(a.exp_flags, 2);
  for (uint32_t wg = wit; wg < RW; wg += tw) {
    uint64_t m = 0;
    for (uint32_t jv = 0; jv < f; ++jv) m |= (uint64_t)((rowsF[jv * RW + wg] >> lane) & 1u) << jv;
    patt[wg * 32u + lane] = m;
  }
  team_sync(tw, teams_per_cta, team);
  probe(a.exp_flags, 3);
  uint64_t pm[WPT];
#pragma unroll
  for (int j = 0; j < WPT; ++j) pm[j] = patt[(own + wit + tw * j) * 32u + lane];

  // phase 1: donors
  uint64_t dm[WPT];
  bool present[WPT];
  int32_t dsel[WPT];
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    const uint32_t w = wit + tw * j;
    const uint32_t s = w * 32u + lane;
    const uint32_t sg = a.rank * n + s;  // global member index (Philox counter, donors)
    const uint64_t m = pm[j];
    int32_t d = -1;
    uint64_t x = m;
    if (s < n) {
      if (replay) {
        d = a.tape[(size_t)p * n + s];
        if (d >= 0) x = patt[d];
      } else {
        // uniform over the members that differ on F — the distribution of
        // the lazy Fisher-Yates scan of engine_serial.hpp:30-46 — from ONE
        // Philox call: candidate c0 uniform over all members is taken when it
        // differs; otherwise the k-th differing member, k uniform from the
        // call's other 64 bits.  P(d) = 1/n + (n_same/n)(1/n_diff) = 1/n_diff
        // for every differing d, and a warp diverges for at most one
        // count-and-select (instead of more draws).
        const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
        const uint32_t ng = a.n_global;
        const uint4 r = philox4x32_10(make_uint4(sg, sid, generation, kTagGom), key);
        const uint32_t c0 = bounded(lo64(r), ng);
        const uint32_t i0 = a.R == 1 ? c0 : (c0 / n) * (32u * Wp) + c0 % n;
        const uint64_t x0 = patt[i0];
        if (x0 != m) {
          d = (int32_t)c0;
          x = x0;
        } else {
          uint32_t total = 0;
          for (uint32_t wg = 0; wg < RW; ++wg) total += __popc(differ_word(rowsF, f, RW, wg, m, n, Wp));
          if (total > 0) {
            uint32_t kth = bounded(hi64(r), total);
            for (uint32_t wg = 0; wg < RW; ++wg) {
              const uint32_t dw = differ_word(rowsF, f, RW, wg, m, n, Wp);
              const uint32_t c = __popc(dw);
              if (kth < c) {
                const uint32_t b = select_bit(dw, kth);
                d = (int32_t)((wg >> lwp) * n + (wg & (Wp - 1u)) * 32u + b);
                x = patt[wg * 32u + b];
                break;
              }
              kth -= c;
            }
          }
        }
      }
    }
    dm[j] = x;
    present[j] = d >= 0;
    dsel[j] = d;
    uint32_t mine = 0, mine2 = 0;  // lane jv keeps the donor-inserted word of F's jv-th row
    for (uint32_t jv = 0; jv < f; ++jv) {
      const uint32_t word = __ballot_sync(0xFFFFFFFFu, (uint32_t)(x >> jv) & 1u);
      if (lane == (jv & 31u)) {
        if (jv < 32) mine = word; else mine2 = word;
      }
    }
    if (lane < f) newD[lane * Wp + w] = mine;
    if (lane + 32u < f) newD[(lane + 32u) * Wp + w] = mine2;
  }
  team_sync(tw, teams_per_cta, team);
  probe(a.exp_flags, 4);

  // phase 2: footprint sums, ascending edge id (engine_parallel.hpp:164-173)
  int32_t di[WPT];
  double sn[WPT], so[WPT];
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    di[j] = 0;
    sn[j] = 0.0;
    so[j] = 0.0;
  }
  for (uint32_t base = e0; base < e1; base += 32) {
    FpEntry E;
    uint32_t xw[WPT];
    if (base == e0) {
      E = E0;
#pragma unroll
      for (int j = 0; j < WPT; ++j) xw[j] = xw0[j];
    } else {
      const uint32_t e = base + lane;
      if (e < e1) {
        E = a.fp[e];
      } else {
        E.a = kInSet;
        E.b = kInSet;
        E.w = 0.0;
      }
      const uint32_t ext = !(E.a & kInSet) ? E.a : (!(E.b & kInSet) ? E.b : vars[0]);
#pragma unroll
      for (int j = 0; j < WPT; ++j) xw[j] = a.pop[(size_t)ext * Wp + wit + tw * j];
    }
    const bool ina = E.a & kInSet, inb = E.b & kInSet;
    const uint32_t ja = (E.a & ~kInSet) * Wp, jb = (E.b & ~kInSet) * Wp;            // newD rows
    const uint32_t jaR = (E.a & ~kInSet) * RW + own, jbR = (E.b & ~kInSet) * RW + own;  // own old rows
    if constexpr (I32) {
      // lane t = entry t: old / new cut words for 32 solutions at once,
      // transposed so lane s holds its solution's entry masks, then delta
      // = weighted popcounts over the weight bit-planes (exact integers).
      const int32_t wt = (int32_t)E.w;
      const uint32_t aw = wt < 0 ? (uint32_t)(-wt) : (uint32_t)wt;
#pragma unroll
      for (int j = 0; j < WPT; ++j) {
        const uint32_t w = wit + tw * j;
        const uint32_t aO = ina ? rowsF[jaR + w] : xw[j], aN = ina ? newD[ja + w] : xw[j];
        const uint32_t bO = inb ? rowsF[jbR + w] : xw[j], bN = inb ? newD[jb + w] : xw[j];
        const uint32_t mo = transpose32((aO ^ bO) & (E.w != 0.0 ? 0xFFFFFFFFu : 0u), lane);
        const uint32_t mn = transpose32((aN ^ bN) & (E.w != 0.0 ? 0xFFFFFFFFu : 0u), lane);
        int32_t d = 0;
        for (uint32_t k = 0; k < a.wbits; ++k) {
          const uint32_t bp = __ballot_sync(0xFFFFFFFFu, wt > 0 && ((aw >> k) & 1u));
          const uint32_t bn = __ballot_sync(0xFFFFFFFFu, wt < 0 && ((aw >> k) & 1u));
          d += ((int32_t)(__popc(mn & bp) - __popc(mo & bp)) - (int32_t)(__popc(mn & bn) - __popc(mo & bn))) << k;
        }
        di[j] += d;
      }
    } else {
      const int cnt = (int)(e1 - base < 32 ? e1 - base : 32);
      for (int t = 0; t < cnt; ++t) {
        const uint32_t ca = __shfl_sync(0xFFFFFFFFu, E.a, t);
        const uint32_t cb = __shfl_sync(0xFFFFFFFFu, E.b, t);
        const bool ina_t = ca & kInSet, inb_t = cb & kInSet;
        const uint32_t ja_t = (ca & ~kInSet) * Wp, jb_t = (cb & ~kInSet) * Wp;
        const uint32_t jaR_t = (ca & ~kInSet) * RW + own, jbR_t = (cb & ~kInSet) * RW + own;
        const double wt = shfl_d(E.w, t);
#pragma unroll
        for (int j = 0; j < WPT; ++j) {
          const uint32_t w = wit + tw * j;
          const uint32_t xo = (ina_t && inb_t) ? 0u : __shfl_sync(0xFFFFFFFFu, xw[j], t);
          const uint32_t aO = ina_t ? rowsF[jaR_t + w] : xo, aN = ina_t ? newD[ja_t + w] : xo;
          const uint32_t bO = inb_t ? rowsF[jbR_t + w] : xo, bN = inb_t ? newD[jb_t + w] : xo;
          sn[j] += (((aN ^ bN) >> lane) & 1u) ? wt : 0.0;
          so[j] += (((aO ^ bO) >> lane) & 1u) ? wt : 0.0;
        }
      }
    }
  }
  const uint32_t fpl = e1 - e0;

  // phases 3 + 4
  probe(a.exp_flags, 5);
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    const uint32_t w = wit + tw * j;
    const uint32_t s = w * 32u + lane;
    const bool valid = s < n;
    const double delta = (e1 == e0) ? 0.0 : (I32 ? (double)di[j] : sn[j] - so[j]);
    bool accept = false;
    if (present[j]) {
      const bool elit = is_elit[j];
      if (exact) {
        accept = delta > 0.0 || (delta == 0.0 && !elit);
      } else {
        const double pf = pfit[j];
        const double cand = pf + delta;
        accept = cmp_better(false, cand, pf) || (cmp_equal(false, cand, pf) && !elit);
      }
    }
    const uint32_t acc_w = __ballot_sync(0xFFFFFFFFu, accept);
    for (uint32_t jv = lane; jv < f; jv += 32)
      newF[jv * Wp + w] = (rowsF[jv * RW + own + w] & ~acc_w) | (newD[jv * Wp + w] & acc_w);
    if (accept) {
      acc[j] += I32 ? (Acc)di[j] : __double2ll_rn(delta * a.fix_scale);
      uint64_t changed = (dm[j] ^ pm[j]) & fm;
      const bool cap = (int32_t)(a.rank * n + s) == esrc;
      while (changed) {
        const uint32_t jv = (uint32_t)(__ffsll((long long)changed) - 1);
        changed &= changed - 1;
        dh1[j] ^= zF[2 * jv];
        dh2[j] ^= zF[2 * jv + 1];
        if (cap) capture_row(a.elit, a.ever, ever_cur, vars[jv], (uint32_t)(pm[j] >> jv) & 1u);
      }
    }
    steps += present[j] ? 1u : 0u;
    calls += present[j] ? fpl : 0u;
    if (record && valid) {
      const size_t at = (size_t)p * n + s;
      a.rec_donor[at] = dsel[j];
      a.rec_delta[at] = delta;
      a.rec_present[at] = present[j];
      a.rec_accept[at] = accept;
    }
  }
  team_sync(tw, teams_per_cta, team);
  probe(a.exp_flags, 6);
  for (uint32_t idx = tid_team; idx < f * Wp; idx += team_threads) {
    const uint32_t jv = idx / Wp, w = idx - jv * Wp;
    const uint32_t nw = newF[idx];
    if (nw != rowsF[jv * RW + own + w]) a.pop[(size_t)vars[jv] * Wp + w] = nw;
  }
  team_sync(tw, teams_per_cta, team);
  probe(a.exp_flags, 7);
}

}  // namespace gomix_b200
