// gom_tt.cuh — the truth-table univariate GOM step (degree <= 4, Philox,
// rows of WC <= 4 words) as a device function: the batch loop of
// gom_univ_tt_kernel (gom_univ.cu; a persistent whole-generation variant was
// measured and not kept).  Semantics and layout: gom_univ.cu's
// header and DESIGN.md §4.
#pragma once

#include "gom_common.cuh"

namespace gomix_b200 {

constexpr int kUnivWarps = 8;        // warps per CTA of the univariate kernels

// Path counters of the batch loop (builds with -DGOMIX_PROBES
// -DGOMIX_PROBE_COUNTS only — the same-address atomics distort timing;
// lane 0 adds v): read with gomix_debug_cta_stats after the per-CTA records.
static __device__ unsigned long long g_ttcount[16];
__device__ __forceinline__ void tt_count(uint32_t i, uint32_t v, uint32_t lane) {
#ifdef GOMIX_PROBE_COUNTS
  if (lane == 0 && v) atomicAdd(&g_ttcount[i], (unsigned long long)v);
#endif
}
constexpr uint32_t kSparseKeys = 6;  // hash deltas key by key up to this many accepted sets per solution

template <int WP>
__device__ __forceinline__ void load_row(const uint32_t* row, uint32_t (&x)[WP]) {
  if constexpr (WP == 4) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(row));
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
  } else if constexpr (WP == 2) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(row));
    x[0] = t.x; x[1] = t.y;
  } else {
    x[0] = __ldg(row);
  }
}

// neighbour rows are written by no lane of this launch (same-colour sets are
// not adjacent), so the read-only path is safe for them too
template <int WP>
__device__ __forceinline__ void store_row(uint32_t* row, const uint32_t (&x)[WP]) {
  if constexpr (WP == 4) {
    *reinterpret_cast<uint4*>(row) = make_uint4(x[0], x[1], x[2], x[3]);
  } else if constexpr (WP == 2) {
    *reinterpret_cast<uint2*>(row) = make_uint2(x[0], x[1]);
  } else {
    row[0] = x[0];
  }
}

// 64-bit XOR into shared memory as two native 32-bit atomics (a 64-bit
// shared atomic XOR compiles to a compare-and-swap loop)
__device__ __forceinline__ void xor_shared64(unsigned long long* p, unsigned long long v) {
  unsigned int* q = reinterpret_cast<unsigned int*>(p);
  const unsigned int lo = (unsigned int)v, hi = (unsigned int)(v >> 32);
  if (lo) atomicXor(q, lo);
  if (hi) atomicXor(q + 1, hi);
}

// 64-bit add into shared memory as two native 32-bit atomics (the 64-bit
// shared atomicAdd compiles to a compare-and-swap loop): the low word's
// carry, read from the returned old value, goes into the high word
__device__ __forceinline__ void add_shared64(long long* p, long long v) {
  unsigned int* q = reinterpret_cast<unsigned int*>(p);
  const unsigned int lo = (unsigned int)v;
  const unsigned int old = atomicAdd(q, lo);
  const unsigned int hi = (unsigned int)((unsigned long long)v >> 32) + ((old + lo) < old ? 1u : 0u);
  if (hi) atomicAdd(q + 1, hi);
}
#ifndef GOMIX_TT_SPARSE_IMP
#define GOMIX_TT_SPARSE_IMP 2
#endif
constexpr uint32_t kSparseImp = GOMIX_TT_SPARSE_IMP;  // strict improvements pair by pair up to this many per set and word

// leaf masks of a 16-entry table held in bits [16*half, 16*half + 16) of tt
__device__ __forceinline__ void tt_masks(uint32_t tt, int half, uint32_t (&m)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = (uint32_t)((int32_t)(tt << (31 - (16 * half + i))) >> 31);
}

// bit-sliced lookup: bit s of the result = table[p_s], p_s = b0_s | b1_s<<1 | b2_s<<2 | b3_s<<3
__device__ __forceinline__ uint32_t tt_mux(const uint32_t (&m)[16], uint32_t b0, uint32_t b1, uint32_t b2,
                                           uint32_t b3) {
  uint32_t l0[8], l1[4], l2[2];
#pragma unroll
  for (int q = 0; q < 8; ++q) l0[q] = (b0 & m[2 * q + 1]) | (~b0 & m[2 * q]);
#pragma unroll
  for (int q = 0; q < 4; ++q) l1[q] = (b1 & l0[2 * q + 1]) | (~b1 & l0[2 * q]);
#pragma unroll
  for (int q = 0; q < 2; ++q) l2[q] = (b2 & l1[2 * q + 1]) | (~b2 & l1[2 * q]);
  return (b3 & l2[1]) | (~b3 & l2[0]);
}

// the same lookup at the complemented pattern: bit s = table[~p_s & 15]
// (complementing every input swaps the two leaves of every multiplexer)
__device__ __forceinline__ uint32_t tt_mux_not(const uint32_t (&m)[16], uint32_t b0, uint32_t b1, uint32_t b2,
                                               uint32_t b3) {
  uint32_t l0[8], l1[4], l2[2];
#pragma unroll
  for (int q = 0; q < 8; ++q) l0[q] = (b0 & m[2 * q]) | (~b0 & m[2 * q + 1]);
#pragma unroll
  for (int q = 0; q < 4; ++q) l1[q] = (b1 & l0[2 * q]) | (~b1 & l0[2 * q + 1]);
#pragma unroll
  for (int q = 0; q < 2; ++q) l2[q] = (b2 & l1[2 * q]) | (~b2 & l1[2 * q + 1]);
  return (b3 & l2[0]) | (~b3 & l2[1]);
}

__device__ __forceinline__ int32_t w16(uint32_t packed, int hi) {
  return hi ? ((int32_t)packed >> 16) : ((int32_t)(packed << 16) >> 16);
}

// per-CTA scratch of the batch loop
struct TtShared {
  unsigned long long key[kUnivWarps][32][2];      // the warp's sets' Zobrist keys
  unsigned long long tbl[kUnivWarps][8][16][2];   // 4-bit-chunk key XOR tables
  ulonglong2 wh[kUnivWarps][4 * 32];              // per-warp hash deltas of the CTA's solutions
};

// The plan records of a warp's next batch, in flight while a batch computes.
struct TtNext {
  uint4 ra, rc;
  ulonglong2 zk;
};

__device__ __forceinline__ TtNext tt_fetch(const uint4* urec, const ulonglong2* ukey, uint32_t G, uint32_t p) {
  TtNext r;
  r.ra = make_uint4(0, 0, 0, 0);
  r.rc = make_uint4(0, 0, 0, 0);
  r.zk = make_ulonglong2(0ull, 0ull);
  if (p < G) {
    r.ra = __ldg(urec + 2u * (size_t)p);
    r.rc = __ldg(urec + 2u * (size_t)p + 1u);
    r.zk = __ldg(ukey + p);
  }
  return r;
}

// Which part of the population a CTA works on.  Rows of up to WC words
// (n <= 32 WC): every CTA takes whole rows.  Wider rows (n > 128): the row is
// cut into chunks of WC words and CTA i takes chunk i % chunks of the sets
// assigned to CTA slot i / chunks; a CTA's per-solution accumulators then
// cover only its chunk's 32 WC solutions.  The grid is a whole number of
// CTAs per SM (every SM equally loaded), so chunks may differ by one CTA.
struct TtPart {
  uint32_t chunk;   // this CTA's chunk of every row
  uint32_t cta;     // this CTA's slot among the CTAs of its chunk
  uint32_t ctas;    // CTAs per chunk (gridDim.x / chunks)
  uint32_t cbase;   // first solution of the chunk
  uint32_t n_chunk; // solutions in the chunk
};

template <int WC>
__device__ __forceinline__ TtPart tt_part(const GomArgs& a) {
  TtPart t;
  const uint32_t chunks = a.Wp / (uint32_t)WC;
  t.chunk = blockIdx.x % chunks;
  t.cta = blockIdx.x / chunks;
  t.ctas = (gridDim.x - t.chunk + chunks - 1) / chunks;  // the grid need not be a multiple of chunks
  t.cbase = t.chunk * (uint32_t)WC * 32u;
  t.n_chunk = min((uint32_t)WC * 32u, a.n - min(a.n, t.cbase));
  return t;
}

// The batches of one colour group handled by this warp: warp-major batch
// order (bt = warp * ctas + cta, then + ctas * kUnivWarps), `nx` = the first
// batch's records (fetched by the caller).  Commits the accepted flips in
// place, records the elitist's old bits copy-on-write, accumulates fitness
// deltas into s_dfit (per chunk solution, shared atomics) and hash deltas
// into sh.wh[warp] (this warp's own slice), counts steps/calls.  s_elit:
// group-start "parent == elitist" mask per word of the chunk.  Chunked rows
// take the presence test from a.ones (every row's count of 1s at group
// start, counted per generation: a univariate, variable-once FOS changes a
// row only in its own group).
template <int B, int WC>
__device__ __forceinline__ uint32_t tt_batches(const GomArgs& a, const TtPart& part, const uint4* urec,
                                           const ulonglong2* ukey, uint32_t G, TtNext nx, const uint32_t* s_elit,
                                           long long* s_dfit, TtShared& sh, int32_t esrc, uint32_t ever_cur,
                                           uint32_t lane, uint32_t warp, unsigned long long& steps,
                                           unsigned long long& calls) {
  const uint32_t Wp = a.Wp;  // row stride (words)
  const uint32_t cw = part.chunk * (uint32_t)WC;  // first word of the chunk
  const uint32_t n = a.n;
  const uint32_t batches = (G + 31u) / 32u;
  const uint32_t bstride = part.ctas * kUnivWarps;
  // Every warp takes the same number of batches statically (warp-major, so
  // every SM gets the same mix); the remainder — less than one batch per
  // warp — goes to whichever warps finish first, claimed from kTailCounters
  // counters (counter c hands out batches dyn0 + c + kTailCounters * i to
  // the warps with slot % kTailCounters == c): the CTAs that run slow (memory
  // latency, accept-heavy sets) no longer set the launch's tail.
  const uint32_t nstatic = batches / bstride;
  const uint32_t dyn0 = nstatic * bstride;
  const uint32_t slot = warp * part.ctas + part.cta;
  const uint32_t tc = slot % kTailCounters;
  unsigned int* tail = a.tail + ((a.tail_per_chunk ? part.chunk : 0u) * kTailCounters + tc) * kTailStride;
  const uint32_t dyn = dyn0 + tc;
  uint32_t k = 0;
  uint32_t np = 0, dsum = 0;  // this lane's present sets and their degrees
  uint32_t bt = slot;  // the caller prefetched this batch's records
  if (nstatic == 0) {  // fewer batches than warps: every batch is claimed
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(tail, 1u);
    bt = dyn + kTailCounters * __shfl_sync(0xFFFFFFFFu, c, 0);
    nx = tt_fetch(urec, ukey, G, bt * 32u + lane);
  }
  while (bt < batches) {
    const uint32_t p = bt * 32u + lane;
    const bool live = p < G;
    const uint4 ra = nx.ra, rc = nx.rc;
    const ulonglong2 zk = nx.zk;
    uint32_t bt_next;
    if (++k < nstatic) {
      bt_next = bt + bstride;
    } else {
      uint32_t c = 0;
      if (lane == 0) c = atomicAdd(tail, 1u);
      bt_next = dyn + kTailCounters * __shfl_sync(0xFFFFFFFFu, c, 0);
    }
    nx = tt_fetch(urec, ukey, G, bt_next * 32u + lane);
    const uint32_t v = ra.x;
    const uint32_t u[4] = {rc.x, rc.y, rc.z, rc.w};
    uint32_t x[WC], nb[4][WC];
#pragma unroll
    for (int j = 0; j < WC; ++j) {
      x[j] = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) nb[t][j] = 0;
    }
    if (live) {
      load_row<WC>(a.pop + (size_t)v * Wp + cw, x);
#pragma unroll
      for (int t = 0; t < 4; ++t) load_row<WC>(a.pop + (size_t)u[t] * Wp + cw, nb[t]);
    }
    int32_t w[4];
    w[0] = w16(ra.z, 0);
    w[1] = w16(ra.z, 1);
    w[2] = w16(ra.w, 0);
    w[3] = w16(ra.w, 1);
    uint32_t neg[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) neg[t] = w[t] < 0 ? 0xFFFFFFFFu : 0u;
    const uint32_t deg = (uint32_t)(u[0] != v) + (uint32_t)(u[1] != v) + (uint32_t)(u[2] != v) + (uint32_t)(u[3] != v);
    // ---- presence: some member (over every rank's shard) holds the other value
    uint32_t ones = 0;
    if (live) {
      if (a.ones) {
        ones = a.ones[v];
      } else if (a.R == 1) {
#pragma unroll
        for (int j = 0; j < WC; ++j) ones += __popc(x[j]);
      } else {
        for (uint32_t r = 0; r < a.R; ++r) {
          uint32_t y[WC];
          load_row<WC>(a.pool + ((size_t)r * a.nv + v) * Wp, y);
#pragma unroll
          for (int j = 0; j < WC; ++j) ones += __popc(y[j]);
        }
      }
    }
    const bool present = live && ones > 0u && ones < a.n_global;
    if (present) {  // (x n_chunk at the end)
      ++np;
      dsum += deg;
    }
    const uint32_t pmask = present ? 0xFFFFFFFFu : 0u;
    // ---- b words (edge "uncut-gain" bits), then accept via the LE table
    // (LT | LE & ~elitist where the group-start elitist lives)
    uint32_t bw[4][WC], acc[WC];
    bool any = false;
#pragma unroll
    for (int j = 0; j < WC; ++j)
#pragma unroll
      for (int t = 0; t < 4; ++t) bw[t][j] = x[j] ^ nb[t][j] ^ neg[t];
    uint32_t mle[16];
    tt_masks(ra.y, 1, mle);
    {
#pragma unroll
      for (int j = 0; j < WC; ++j) {
        uint32_t ac = tt_mux(mle, bw[0][j], bw[1][j], bw[2][j], bw[3][j]);
        const uint32_t ew = s_elit[j];
        if (ew) {  // warp-uniform: group-start elitist copies take strict improvements only
          uint32_t e = ew, keep = 0xFFFFFFFFu;
          while (e) {
            const uint32_t b = (uint32_t)(__ffs(e) - 1);
            e &= e - 1u;
            const uint32_t pat = ((bw[0][j] >> b) & 1u) | (((bw[1][j] >> b) & 1u) << 1) |
                                 (((bw[2][j] >> b) & 1u) << 2) | (((bw[3][j] >> b) & 1u) << 3);
            if (!((ra.y >> pat) & 1u)) keep &= ~(1u << b);  // LT[p] bit of the table
          }
          ac &= keep;
        }
        acc[j] = ac & pmask & valid_mask(cw + (uint32_t)j, n);
        any |= acc[j] != 0u;
      }
    }
#ifdef GOMIX_PROBE_COUNTS
    tt_count(0, 1, lane);
    tt_count(6, __any_sync(0xFFFFFFFFu, any) ? 1u : 0u, lane);
#pragma unroll
    for (int j = 0; j < WC; ++j) {
      tt_count(1, __any_sync(0xFFFFFFFFu, acc[j] != 0u) ? 1u : 0u, lane);
      tt_count(7, s_elit[j] ? 1u : 0u, lane);
      tt_count(8, __reduce_add_sync(0xFFFFFFFFu, (uint32_t)__popc(acc[j])), lane);
      tt_count(9, __popc(__ballot_sync(0xFFFFFFFFu, acc[j] != 0u)), lane);
    }
#endif
    // ---- commit: accepted solutions flip v (apply_acceptance, :221-247)
    if (any) {
      uint32_t nw[WC];
#pragma unroll
      for (int j = 0; j < WC; ++j) nw[j] = x[j] ^ acc[j];
      store_row<WC>(a.pop + (size_t)v * Wp + cw, nw);
      if (esrc >= 0) {  // (esrc is relative to the chunk: -1 when the elitist lives elsewhere)
        const uint32_t ew = (uint32_t)esrc >> 5, eb = (uint32_t)esrc & 31u;
        uint32_t aw = 0, xw = 0;
#pragma unroll
        for (int j = 0; j < WC; ++j)
          if ((uint32_t)j == ew) {
            aw = acc[j];
            xw = x[j];
          }
        if ((aw >> eb) & 1u) capture_row(a.elit, a.ever, ever_cur, v, (xw >> eb) & 1u);
      }
    }
    // ---- per-solution reductions over the warp's 32 sets ----------------
    if (__any_sync(0xFFFFFFFFu, any)) {
      sh.key[warp][lane][0] = zk.x;
      sh.key[warp][lane][1] = zk.y;
      __syncwarp();
      bool tbl = false;
#pragma unroll
      for (int j = 0; j < WC; ++j) {
        if (!__any_sync(0xFFFFFFFFu, acc[j] != 0u)) continue;
        const uint32_t accT = transpose32(acc[j], lane);  // lane b: sets l accepted by solution 32j+b
        const uint32_t b0 = bw[0][j], b1 = bw[1][j], b2 = bw[2][j], b3 = bw[3][j];
        long long d = 0;
        // strict improvements: T(p) < A/2  <=>  T(~p) = A - T(p) > A/2  <=>
        // ~p is not in LE — the LE table at the complemented pattern, no LT masks
        const uint32_t imp = acc[j] & ~tt_mux_not(mle, b0, b1, b2, b3);
        tt_count(2, __any_sync(0xFFFFFFFFu, imp != 0u) ? 1u : 0u, lane);
#ifndef GOMIX_TT_IMP_PLANES_ONLY
        const uint32_t imax = __reduce_max_sync(0xFFFFFFFFu, (uint32_t)__popc(imp));
        if (imax != 0u && imax <= kSparseImp) {
          // few strict improvements per set (generations after the first):
          // each set adds its delta A - 2T(p) to the solutions it improves,
          // pair by pair, instead of transposing every T plane
          const int32_t m0 = abs(w[0]), m1 = abs(w[1]), m2 = abs(w[2]), m3 = abs(w[3]);
          const int32_t A = m0 + m1 + m2 + m3;
          uint32_t r = imp;
          while (r) {
            const uint32_t b = (uint32_t)(__ffs(r) - 1);
            r &= r - 1u;
            const int32_t T = (((b0 >> b) & 1u) ? m0 : 0) + (((b1 >> b) & 1u) ? m1 : 0) +
                              (((b2 >> b) & 1u) ? m2 : 0) + (((b3 >> b) & 1u) ? m3 : 0);
            add_shared64(&s_dfit[(uint32_t)j * 32u + b], (long long)(A - 2 * T));
          }
        } else if (imax != 0u) {
#else
        if (__any_sync(0xFFFFFFFFu, imp != 0u)) {
#endif
          // T planes of this word (only words with a strictly improving pair)
          uint32_t T[B];
#pragma unroll
          for (int k = 0; k < B; ++k) T[k] = 0;
          const uint32_t bb[4] = {b0, b1, b2, b3};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t mg = (uint32_t)abs(w[t]);
            uint32_t cy = 0;
#pragma unroll
            for (int k = 0; k < B; ++k) {
              const uint32_t xb = ((mg >> k) & 1u) ? bb[t] : 0u;
              const uint32_t tk = T[k];
              T[k] = tk ^ xb ^ cy;
              cy = (tk & xb) | (tk & cy) | (xb & cy);
            }
          }
          const uint32_t impT = transpose32(imp, lane);
          const uint32_t A = (uint32_t)(abs(w[0]) + abs(w[1]) + abs(w[2]) + abs(w[3]));
#pragma unroll
          for (int k = 0; k < B; ++k) d += (long long)__popc(impT & __ballot_sync(0xFFFFFFFFu, (A >> k) & 1u)) << k;
#pragma unroll
          for (int k = 0; k < B - 1; ++k) d -= (long long)__popc(transpose32(T[k] & imp, lane)) << (k + 1);
        }
        const uint32_t sj = (uint32_t)j * 32u + lane;
        if (d) add_shared64(&s_dfit[sj], d);
        // hash delta of solution 32j+lane: XOR of the keys of its accepted
        // sets — key by key when every solution of the word accepted few
        // sets (the steady state: neutral flips are sparse), else through the
        // 4-bit-chunk table of key XORs.  (Walking the accepting sets
        // instead — ~2.5 of 32 per word at C3 — each set's accept word
        // broadcast from its lane, saves the transpose but measured 11%
        // slower: registers spill; so did LT muxes for the elitist copies.)
        unsigned long long x1 = 0, x2 = 0;
#ifdef GOMIX_PROBE_COUNTS
        {
          const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, (uint32_t)__popc(accT));
          tt_count(mx <= kSparseKeys ? 3 : 4, 1, lane);
          tt_count(5, mx, lane);
        }
#endif
        if (__reduce_max_sync(0xFFFFFFFFu, (uint32_t)__popc(accT)) <= kSparseKeys) {
          uint32_t r = accT;
          while (r) {
            const uint32_t l = (uint32_t)(__ffs(r) - 1);
            r &= r - 1u;
            const ulonglong2 k = *reinterpret_cast<const ulonglong2*>(sh.key[warp][l]);
            x1 ^= k.x;
            x2 ^= k.y;
          }
        } else {
          if (!tbl) {
            tbl = true;
            const uint32_t q = lane >> 2, sub = lane & 3u;
            const ulonglong2 k0 = *reinterpret_cast<const ulonglong2*>(sh.key[warp][4 * q + 0]);
            const ulonglong2 k1 = *reinterpret_cast<const ulonglong2*>(sh.key[warp][4 * q + 1]);
            const ulonglong2 k2 = *reinterpret_cast<const ulonglong2*>(sh.key[warp][4 * q + 2]);
            const ulonglong2 k3 = *reinterpret_cast<const ulonglong2*>(sh.key[warp][4 * q + 3]);
            const unsigned long long l1 = ((sub & 1u) ? k0.x : 0ull) ^ ((sub & 2u) ? k1.x : 0ull);
            const unsigned long long l2 = ((sub & 1u) ? k0.y : 0ull) ^ ((sub & 2u) ? k1.y : 0ull);
            ulonglong2* tb = reinterpret_cast<ulonglong2*>(sh.tbl[warp][q]);
            tb[sub] = make_ulonglong2(l1, l2);
            tb[sub + 4] = make_ulonglong2(l1 ^ k2.x, l2 ^ k2.y);
            tb[sub + 8] = make_ulonglong2(l1 ^ k3.x, l2 ^ k3.y);
            tb[sub + 12] = make_ulonglong2(l1 ^ k2.x ^ k3.x, l2 ^ k2.y ^ k3.y);
            __syncwarp();
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t m = (accT >> (4 * q)) & 15u;
            const ulonglong2 tq = *reinterpret_cast<const ulonglong2*>(sh.tbl[warp][q][m]);
            x1 ^= tq.x;
            x2 ^= tq.y;
          }
        }
        if (x1 | x2) {  // the warp's own running hash deltas: no atomics
          ulonglong2* q = &sh.wh[warp][j * 32 + lane];
          ulonglong2 o = *q;
          o.x ^= x1;
          o.y ^= x2;
          *q = o;
        }
      }
    }
    __syncwarp();
    bt = bt_next;
  }
  steps += (unsigned long long)np * part.n_chunk;
  calls += (unsigned long long)dsum * part.n_chunk;
  return k;  // batches this warp processed (+1 when it claimed past the end)
}

}  // namespace gomix_b200
