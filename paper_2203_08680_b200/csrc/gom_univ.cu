// gom_univ.cu — the batched GOM step for a univariate FOS on integer weights
// in Philox mode, bit-sliced: one linkage set {v} per LANE, the solutions of
// that set as the bits of its packed row.
//
// Same semantics as gom_group_kernel's univariate path (engine_parallel.hpp:
// 104-247): for F = {v} every donor that differs on F holds !x_v, so the pair
// (s, {v}) is present iff some member holds the other value, and the GOM move
// is the flip of v.  Its partial-evaluation delta over v's edges e = (v, u_e)
// (the set's footprint, engine_parallel.hpp:48-55) is
//     delta_s = sum_e w_e (1 - 2 c_e,s),   c_e,s = x_v,s xor x_u,s (edge cut now)
//             = A - 2 T_s,   A = sum_e |w_e|,   T_s = sum_e |w_e| b_e,s
// with b_e = c_e for w_e > 0 and !c_e for w_e < 0.  T is accumulated for all
// solutions of the row at once as a B-plane bit-sliced counter (full adders
// on 32-bit words: bit b of plane k = bit k of T for solution 32j+b), the
// accept rule (determine_improvements, :194-214; exact comparator)
//     delta > 0  or  (delta == 0 and parent != elitist)
// becomes  T < h  or  (T == h and A even and not elitist),  h = (A+1)/2,
// one bit-sliced comparison.  Accepted solutions flip v: one XOR per word.
//
// Per-solution results (fitness delta sum, Zobrist hash delta) are reduced
// over the 32 sets of a warp by 32x32 bit transposes (bit l of lane b's word
// = set l, solution b): fitness += sum_l acc (A_l - 2 T_l) = popcounts of the
// transposed planes against ballots of the A_l bits; hash ^= XOR of key(v_l)
// over accepted l via a 4-bit-chunk table of key XORs in shared memory.
//
// Why: the lane-per-solution path walks one set per warp with a chain of
// dependent loads (set -> CSR row -> neighbour rows) and shuffles every
// neighbour word to every lane; here the 32 sets of a warp load in parallel,
// no neighbour data crosses lanes, and an edge costs ~3B+2 logic ops per 32
// solutions.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "gom_common.cuh"
#include "gom_tt.cuh"

namespace gomix_b200 {

namespace {
constexpr int kNbChunk = 4;  // neighbour (col, w) pairs fetched per round
}  // namespace

template <int B, int WC, bool MULTI>
__global__ void __launch_bounds__(kUnivWarps * 32, 3) gom_univ_sliced_kernel(const GomArgs a) {
  // WC words of a row per pass ("chunk"); MULTI: rows of Wp = a.Wp > WC words
  // take Wp / WC passes, otherwise Wp == WC and the row is loaded once
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ __align__(16) unsigned long long s_key[kUnivWarps][32][2];
  __shared__ __align__(16) unsigned long long s_tbl[kUnivWarps][8][16][2];
  __shared__ unsigned long long s_steps, s_calls;
  __shared__ int s_last;
  if (*(volatile int32_t*)&a.ctl->stop) return;

  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t n = a.n, Wp = MULTI ? a.Wp : (uint32_t)WC, chunks = MULTI ? Wp / WC : 1u;
  // per-solution fitness / hash deltas (shared-memory atomics per batch) and
  // the group-start "parent == elitist" word masks
  long long* s_dfit = reinterpret_cast<long long*>(dyn);
  unsigned long long* s_dh1 = reinterpret_cast<unsigned long long*>(s_dfit + Wp * 32u);
  unsigned long long* s_dh2 = s_dh1 + Wp * 32u;
  uint32_t* s_elit = reinterpret_cast<uint32_t*>(s_dh2 + Wp * 32u);
  uint32_t G = a.G;
  const uint32_t* gvars = a.gvars;
  EpiArgs epi = a.epi;
  if (a.slot >= 0) {  // graph path: this launch's group comes from the device-side order
    const uint32_t gi = a.order[a.slot];
    const GroupDesc d = a.groups[gi];
    G = d.G;
    gvars += d.g0;
    epi.group = gi;
    epi.G = G;
  }
  // group-start "parent == elitist" (engine_parallel.hpp:202) as word masks
  const unsigned long long eh1 = a.ctl->eh1, eh2 = a.ctl->eh2;
  const int32_t esrc_g = a.ctl->elit_src;
  const uint32_t ever_cur = a.ctl->elit_ver;
  const int32_t esrc = (esrc_g >= 0 && (uint32_t)esrc_g / n == a.rank) ? (int32_t)((uint32_t)esrc_g % n) : -1;
  for (uint32_t j = warp; j < Wp; j += kUnivWarps) {
    const uint32_t s = j * 32u + lane;
    const bool e = s < n && a.h1[s] == eh1 && a.h2[s] == eh2;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, e);
    if (lane == 0) s_elit[j] = m;
  }
  for (uint32_t i = threadIdx.x; i < Wp * 32u; i += blockDim.x) {
    s_dfit[i] = 0;
    s_dh1[i] = 0;
    s_dh2[i] = 0;
  }
  if (threadIdx.x == 0) {
    s_steps = 0;
    s_calls = 0;
  }
  __syncthreads();
  unsigned long long steps = 0, calls = 0;

  const uint32_t batches = (G + 31u) / 32u;
  for (uint32_t bt = blockIdx.x * kUnivWarps + warp; bt < batches; bt += gridDim.x * kUnivWarps) {
    const uint32_t p = bt * 32u + lane;
    const bool live = p < G;
    const uint32_t v = live ? gvars[p] : 0u;
    const uint32_t* row = a.pop + (size_t)v * Wp;
    int32_t rs = 0, re = 0;
    if (live) {
      rs = a.row_ptr[v];
      re = a.row_ptr[v + 1];
    }
    uint32_t x0[WC];
#pragma unroll
    for (int j = 0; j < WC; ++j) x0[j] = 0;
    if (!MULTI && live) load_row<WC>(row, x0);
    // ---- presence: some member (over every rank's shard) holds the other value
    uint32_t ones = 0;
    if (live) {
      if (a.ones) {
        ones = a.ones[v];  // sharded, variable-once FOS: counted at generation start
      } else if (!MULTI && a.R == 1) {
#pragma unroll
        for (int j = 0; j < WC; ++j) ones += __popc(x0[j]);
      } else {
        for (uint32_t r = 0; r < a.R; ++r) {
          const uint32_t* pr = a.R > 1 ? a.pool + ((size_t)r * a.nv + v) * Wp : row;
          for (uint32_t c = 0; c < chunks; ++c) {
            uint32_t y[WC];
            load_row<WC>(pr + c * WC, y);
#pragma unroll
            for (int j = 0; j < WC; ++j) ones += __popc(y[j]);
          }
        }
      }
    }
    const bool present = live && ones > 0u && ones < a.n_global;
    if (present) {
      steps += n;
      calls += (unsigned long long)n * (uint32_t)(re - rs);
    }
    uint32_t A = 0, h = 0, aeven = 0;
    bool table = false;
    uint32_t Ab[B];
    for (uint32_t c = 0; c < chunks; ++c) {
      uint32_t x[WC];
#pragma unroll
      for (int j = 0; j < WC; ++j) x[j] = x0[j];
      if (MULTI && live) load_row<WC>(row + c * WC, x);
      // ---- T = sum_e |w_e| b_e (bit-sliced over the chunk's solutions) ------
      uint32_t T[B][WC];
#pragma unroll
      for (int k = 0; k < B; ++k)
#pragma unroll
        for (int j = 0; j < WC; ++j) T[k][j] = 0;
      for (int32_t base = rs; base < re; base += kNbChunk) {
        uint32_t u[kNbChunk];
        int32_t w[kNbChunk];
#pragma unroll
        for (int t = 0; t < kNbChunk; ++t) {
          const bool has = base + t < re;
          u[t] = has ? (uint32_t)__ldg(a.col + base + t) : v;
          w[t] = has ? __ldg(a.wi + base + t) : 0;
        }
        uint32_t nb[kNbChunk][WC];
#pragma unroll
        for (int t = 0; t < kNbChunk; ++t) load_row<WC>(a.pop + (size_t)u[t] * Wp + c * WC, nb[t]);
#pragma unroll
        for (int t = 0; t < kNbChunk; ++t) {
          const uint32_t m = (uint32_t)(w[t] < 0 ? -w[t] : w[t]);
          const uint32_t neg = w[t] < 0 ? 0xFFFFFFFFu : 0u;
          if (c == 0) A += m;
#pragma unroll
          for (int j = 0; j < WC; ++j) {
            const uint32_t b = (x[j] ^ nb[t][j]) ^ neg;
            uint32_t cy = 0;
#pragma unroll
            for (int k = 0; k < B; ++k) {
              const uint32_t xb = ((m >> k) & 1u) ? b : 0u;
              const uint32_t tk = T[k][j];
              T[k][j] = tk ^ xb ^ cy;
              cy = (tk & xb) | (tk & cy) | (xb & cy);
            }
          }
        }
      }
      if (c == 0) {
        h = (A + 1u) >> 1;
        aeven = (A & 1u) ? 0u : 0xFFFFFFFFu;
      }
      // ---- accept: T < h, or T == h with A even and the parent not the elitist
      uint32_t acc[WC], ltw[WC];
      bool any = false;
#pragma unroll
      for (int j = 0; j < WC; ++j) {
        const uint32_t wj = c * WC + (uint32_t)j;
        uint32_t lt = 0, eq = 0xFFFFFFFFu;
#pragma unroll
        for (int k = B - 1; k >= 0; --k) {
          const uint32_t hk = ((h >> k) & 1u) ? 0xFFFFFFFFu : 0u;
          lt |= eq & ~T[k][j] & hk;
          eq &= ~(T[k][j] ^ hk);
        }
        acc[j] = present ? ((lt | (eq & aeven & ~s_elit[wj])) & valid_mask(wj, n)) : 0u;
        ltw[j] = lt;
        any |= acc[j] != 0u;
      }
      // ---- commit: accepted solutions flip v (apply_acceptance, :221-247)
      if (any) {
        uint32_t nx[WC];
#pragma unroll
        for (int j = 0; j < WC; ++j) nx[j] = x[j] ^ acc[j];
        store_row<WC>(a.pop + (size_t)v * Wp + c * WC, nx);
        if (esrc >= 0 && ((uint32_t)esrc >> 5) / WC == c) {
          const uint32_t ew = ((uint32_t)esrc >> 5) - c * WC, eb = (uint32_t)esrc & 31u;
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
      if (!__any_sync(0xFFFFFFFFu, any)) continue;
      if (!table) {  // first accepting chunk of this batch (warp-uniform)
        table = true;
#pragma unroll
        for (int k = 0; k < B; ++k) Ab[k] = __ballot_sync(0xFFFFFFFFu, (A >> k) & 1u);
        // Zobrist key XOR table: s_tbl[c][m] = XOR of key(v_{4c+i}) over bits i of m
        unsigned long long z1 = 0, z2 = 0;
        if (present) zobrist(v, z1, z2);
        s_key[warp][lane][0] = z1;
        s_key[warp][lane][1] = z2;
        __syncwarp();
        {
          // lane = (chunk q, low bits sub): entries sub, sub+4, sub+8, sub+12 of
          // chunk q share the XOR of keys 4q, 4q+1 selected by sub
          const uint32_t q = lane >> 2, sub = lane & 3u;
          const ulonglong2 k0 = *reinterpret_cast<const ulonglong2*>(s_key[warp][4 * q + 0]);
          const ulonglong2 k1 = *reinterpret_cast<const ulonglong2*>(s_key[warp][4 * q + 1]);
          const ulonglong2 k2 = *reinterpret_cast<const ulonglong2*>(s_key[warp][4 * q + 2]);
          const ulonglong2 k3 = *reinterpret_cast<const ulonglong2*>(s_key[warp][4 * q + 3]);
          const unsigned long long l1 = ((sub & 1u) ? k0.x : 0ull) ^ ((sub & 2u) ? k1.x : 0ull);
          const unsigned long long l2 = ((sub & 1u) ? k0.y : 0ull) ^ ((sub & 2u) ? k1.y : 0ull);
          ulonglong2* t = reinterpret_cast<ulonglong2*>(s_tbl[warp][q]);
          t[sub] = make_ulonglong2(l1, l2);
          t[sub + 4] = make_ulonglong2(l1 ^ k2.x, l2 ^ k2.y);
          t[sub + 8] = make_ulonglong2(l1 ^ k3.x, l2 ^ k3.y);
          t[sub + 12] = make_ulonglong2(l1 ^ k2.x ^ k3.x, l2 ^ k2.y ^ k3.y);
        }
        __syncwarp();
      }
#pragma unroll
      for (int j = 0; j < WC; ++j) {
        const uint32_t accT = transpose32(acc[j], lane);  // lane b: sets l accepted by solution 32j+b
        // fitness: only strictly improving pairs (T < h) change it; neutral
        // accepts (delta 0) do not.  Late in a run improving moves are rare,
        // so the plane transposes are skipped for most words.
        long long d = 0;
        const uint32_t imp = acc[j] & ltw[j];
        if (__any_sync(0xFFFFFFFFu, imp != 0u)) {
          const uint32_t impT = transpose32(imp, lane);
#pragma unroll
          for (int k = 0; k < B; ++k) d += (long long)__popc(impT & Ab[k]) << k;
          // improving pairs have T < A/2 < 2^(B-1): the top plane is zero
#pragma unroll
          for (int k = 0; k < B - 1; ++k) d -= (long long)__popc(transpose32(T[k][j] & imp, lane)) << (k + 1);
        }
        const uint32_t sj = (c * WC + (uint32_t)j) * 32u + lane;
        if (d) atomicAdd(reinterpret_cast<unsigned long long*>(&s_dfit[sj]), (unsigned long long)d);
        unsigned long long x1 = 0, x2 = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t m = (accT >> (4 * q)) & 15u;
          const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(s_tbl[warp][q][m]);
          x1 ^= t.x;
          x2 ^= t.y;
        }
        if (x1 | x2) {
          xor_shared64(&s_dh1[sj], x1);
          xor_shared64(&s_dh2[sj], x2);
        }
      }
    }
    __syncwarp();
  }

  // ---- per-CTA reductions, then the group epilogue in the last CTA -------
  {
    unsigned long long ws = steps, wc = calls;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ws += __shfl_xor_sync(0xFFFFFFFFu, ws, o);
      wc += __shfl_xor_sync(0xFFFFFFFFu, wc, o);
    }
    if (lane == 0 && (ws | wc)) {
      atomicAdd(&s_steps, ws);
      atomicAdd(&s_calls, wc);
    }
  }
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < n && s < Wp * 32u; s += blockDim.x) {
    if (s_dfit[s]) atomicAdd(reinterpret_cast<unsigned long long*>(&a.dfit[s]), (unsigned long long)s_dfit[s]);
    if (s_dh1[s] | s_dh2[s]) {
      atomicXor(&a.dh1[s], s_dh1[s]);
      atomicXor(&a.dh2[s], s_dh2[s]);
    }
  }
  if (threadIdx.x == 0) {
    if (s_steps | s_calls) {
      atomicAdd(&a.ctl->grp_steps, s_steps);
      atomicAdd(&a.ctl->grp_calls, s_calls);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&a.ctl->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  epilogue_body(epi);
  if (threadIdx.x == 0) a.ctl->done = 0;
}

// ---------------------------------------------------------------------------
// Truth-table variant for sets whose variable has at most 4 edges (every
// torus): the accept decision of (s, {v}) depends only on the 4-bit pattern
// p_s = (b_0,s .. b_3,s) of v's edges, so the group plan stores, per
// position, the 16-entry tables LT[p] = [T(p) < h] (strict improvement) and
// LE[p] = LT[p] | [2T(p) == A] (improvement or neutral), built once from the
// weights (build_univ_records_kernel).  The decision for 32 solutions is then
// a 4-level multiplexer tree over the b words (15 LOP3s) instead of the
// B-plane adder + comparator; words holding no group-start elitist take
// accept = LE directly.  T planes are only formed for words that hold a
// strictly improving pair (their fitness deltas).  The plan record also
// carries the neighbour ids and weights, so a set costs two coalesced
// 16-byte loads before its rows (no gvars -> row_ptr -> col chain).
// ---------------------------------------------------------------------------


// One record pair per group position: r[2p] = {v, LT | LE << 16, w0 | w1 << 16,
// w2 | w3 << 16} (int16 weights in CSR order = ascending neighbour), r[2p+1] =
// the neighbours (padding: v itself with weight 0, whose b word is 0);
// key[p] = Zobrist key of v.
__global__ void build_univ_records_kernel(const uint32_t* gvars, const int32_t* row_ptr, const int32_t* col,
                                          const int32_t* wi, uint64_t m, uint4* rec, ulonglong2* key) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m) return;
  const uint32_t v = gvars[p];
  const int32_t rs = row_ptr[v], deg = row_ptr[v + 1] - rs;
  uint32_t c[4] = {v, v, v, v}, mag[4] = {0, 0, 0, 0};
  int32_t w[4] = {0, 0, 0, 0};
  for (int t = 0; t < deg && t < 4; ++t) {
    c[t] = (uint32_t)col[rs + t];
    w[t] = wi[rs + t];
    mag[t] = (uint32_t)(w[t] < 0 ? -w[t] : w[t]);
  }
  const uint32_t A = mag[0] + mag[1] + mag[2] + mag[3], h = (A + 1u) >> 1;
  uint32_t lt = 0, le = 0;
  for (uint32_t pat = 0; pat < 16; ++pat) {
    uint32_t T = 0;
    for (int t = 0; t < 4; ++t)
      if ((pat >> t) & 1u) T += mag[t];
    if (T < h) lt |= 1u << pat;
    if (T < h || 2u * T == A) le |= 1u << pat;
  }
  rec[2 * p] = make_uint4(v, lt | (le << 16), ((uint32_t)w[0] & 0xFFFFu) | ((uint32_t)w[1] << 16),
                          ((uint32_t)w[2] & 0xFFFFu) | ((uint32_t)w[3] << 16));
  rec[2 * p + 1] = make_uint4(c[0], c[1], c[2], c[3]);
  unsigned long long z1, z2;
  zobrist(v, z1, z2);
  key[p] = make_ulonglong2(z1, z2);
}

// Per-CTA record of the truth-table launches (probes builds only): SM id,
// start and batches-done %globaltimer, batches processed; per launch row
// (graph slot + 1) and CTA; read through gomix_debug_cta_stats.
constexpr int kCtaStatMax = 1024;
static __device__ unsigned long long g_ctastat[kTimelineRows][kCtaStatMax][4];
#ifdef GOMIX_PROBES
static __shared__ unsigned long long s_stat_t0;
static __shared__ unsigned int s_stat_nb;
#endif
__device__ __forceinline__ void cta_stat_start() {
#ifdef GOMIX_PROBES
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_stat_t0));
    s_stat_nb = 0;
  }
#endif
}
__device__ __forceinline__ void cta_stat_batches(uint32_t nb, uint32_t lane) {
#ifdef GOMIX_PROBES
  if (lane == 0) atomicAdd(&s_stat_nb, nb);
#endif
}
__device__ __forceinline__ void cta_stat_done(int32_t row) {
#ifdef GOMIX_PROBES
  if (threadIdx.x == 0 && blockIdx.x < kCtaStatMax) {
    const int32_t r = row < 0 ? 0 : (row >= kTimelineRows ? kTimelineRows - 1 : row);
    unsigned long long t, sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    sm = smid;
    g_ctastat[r][blockIdx.x][0] = sm;
    g_ctastat[r][blockIdx.x][1] = s_stat_t0;
    g_ctastat[r][blockIdx.x][2] = t;
    g_ctastat[r][blockIdx.x][3] = s_stat_nb;
  }
#endif
}

template <int B, int WC, int MINB = 3>
__global__ void __launch_bounds__(kUnivWarps * 32, MINB) gom_univ_tt_kernel(const GomArgs a) {
  __shared__ __align__(16) TtShared sh;
  __shared__ long long s_dfit[WC * 32];
  __shared__ unsigned long long s_dh1[WC * 32], s_dh2[WC * 32];
  __shared__ uint32_t s_elit[WC];
  __shared__ unsigned long long s_steps, s_calls;
  __shared__ int s_last;
  probe(a.exp_flags, 40);
  timeline_mark(0, a.slot + 1);  // CTA start
  timeline_set_row(a.slot + 1);
  cta_stat_start();

  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  constexpr uint32_t Wp = (uint32_t)WC;  // words of this CTA's chunk (whole rows when a.Wp == WC)
  const uint32_t n = a.n;
  const TtPart part = tt_part<WC>(a);
  uint32_t G = a.G;
  const uint4* urec = a.urec;
  const ulonglong2* ukey = a.ukey;
  EpiArgs epi = a.epi;
  // this CTA's accumulators: shared memory only, before any dependency wait
  for (uint32_t i = threadIdx.x; i < Wp * 32u; i += blockDim.x) {
    s_dfit[i] = 0;
#pragma unroll
    for (int q = 0; q < kUnivWarps; ++q) sh.wh[q][i] = make_ulonglong2(0ull, 0ull);
  }
  if (threadIdx.x == 0) {
    s_steps = 0;
    s_calls = 0;
  }
  // Programmatic dependent launches (graph path): the first group's launch
  // follows the begin kernel, which writes this generation's group order, so
  // it waits before reading it; later groups' launches read the order (written
  // before the previous launch could start) and prefetch their first batch's
  // plan records before waiting for the previous group.
  if (a.slot == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.slot >= 0) {  // graph path: this launch's group comes from the device-side order
    const uint32_t gi = a.order[a.slot];
    const GroupDesc d = a.groups[gi];
    G = d.G;
    urec += 2u * (size_t)d.g0;
    ukey += d.g0;
    epi.group = gi;
    epi.G = G;
  }
  const TtNext first = tt_fetch(urec, ukey, G, (warp * part.ctas + part.cta) * 32u + lane);
  // everything below reads what the previous group's launch wrote
  // (population, control block, hashes)
  if (a.slot != 0) asm volatile("griddepcontrol.wait;" ::: "memory");
  timeline_mark(7, a.slot + 1);  // dependency wait over
  // the control block and this warp's hashes in one round trip, then the stop check
  const int32_t stopped = *(volatile int32_t*)&a.ctl->stop;
  const unsigned long long eh1 = a.ctl->eh1, eh2 = a.ctl->eh2;
  const int32_t esrc_g = a.ctl->elit_src;
  const uint32_t ever_cur = a.ctl->elit_ver;
  const uint32_t sw = part.cbase + warp * 32u + lane;
  unsigned long long hs1 = 0, hs2 = 0;
  if (warp < Wp && sw < n) {
    hs1 = a.h1[sw];
    hs2 = a.h2[sw];
  }
  if (stopped) return;
  // the elitist's column relative to this CTA's chunk (-1: not here)
  int32_t esrc = (esrc_g >= 0 && (uint32_t)esrc_g / n == a.rank) ? (int32_t)((uint32_t)esrc_g % n) : -1;
  esrc = (esrc >= (int32_t)part.cbase && esrc < (int32_t)(part.cbase + Wp * 32u)) ? esrc - (int32_t)part.cbase : -1;
  if (warp < Wp) {  // group-start "parent == elitist" (engine_parallel.hpp:202) as word masks
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, sw < n && hs1 == eh1 && hs2 == eh2);
    if (lane == 0) s_elit[warp] = m;
  }
  timeline_mark(12, a.slot + 1);  // prologue: control block and hashes back
  __syncthreads();
  probe(a.exp_flags, 41);
  timeline_mark(1, a.slot + 1);  // prologue done
  unsigned long long steps = 0, calls = 0;
  const uint32_t nbt =
      tt_batches<B, WC>(a, part, urec, ukey, G, first, s_elit, s_dfit, sh, esrc, ever_cur, lane, warp, steps, calls);
  cta_stat_batches(nbt, lane);

  probe(a.exp_flags, 42);
  timeline_mark(2, a.slot + 1);  // warp 0's batches done
  // the next group's launch may start its prologue (it waits for this grid's
  // completion before touching anything written here)
  asm volatile("griddepcontrol.launch_dependents;");
  {
    unsigned long long ws = steps, wc = calls;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ws += __shfl_xor_sync(0xFFFFFFFFu, ws, o);
      wc += __shfl_xor_sync(0xFFFFFFFFu, wc, o);
    }
    if (lane == 0 && (ws | wc)) {
      atomicAdd(&s_steps, ws);
      atomicAdd(&s_calls, wc);
    }
  }
  __syncthreads();
  timeline_mark(6, a.slot + 1);  // every warp of the CTA done with its batches
  cta_stat_done(a.slot + 1);
  for (uint32_t s = threadIdx.x; s < part.n_chunk; s += blockDim.x) {
    unsigned long long x1 = 0, x2 = 0;
#pragma unroll
    for (int q = 0; q < kUnivWarps; ++q) {
      x1 ^= sh.wh[q][s].x;
      x2 ^= sh.wh[q][s].y;
    }
    s_dh1[s] = x1;
    s_dh2[s] = x2;
    const uint32_t g = part.cbase + s;
    if (s_dfit[s]) atomicAdd(reinterpret_cast<unsigned long long*>(&a.dfit[g]), (unsigned long long)s_dfit[s]);
    if (x1 | x2) {
      atomicXor(&a.dh1[g], x1);
      atomicXor(&a.dh2[g], x2);
    }
  }
  if (threadIdx.x == 0) {
    if (s_steps | s_calls) {
      atomicAdd(&a.ctl->grp_steps, s_steps);
      atomicAdd(&a.ctl->grp_calls, s_calls);
    }
  }
  __syncthreads();
  timeline_mark(3, a.slot + 1);  // CTA flushed
  const uint32_t chunks = a.Wp / (uint32_t)WC;
  if (chunks > 1) {
    // Rows in chunks (n > 128): the last CTA of every chunk commits that
    // chunk's solutions and their per-word fitness maxima, so the group's
    // last CTA only scans (the commit of up to 4096 solutions no longer
    // runs serially in one CTA after the grid)
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(&a.chunk_done[part.chunk], 1u) == part.ctas - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    commit_range(epi, part.cbase, part.cbase + part.n_chunk, nullptr, nullptr);
    __syncthreads();
    if (warp < Wp) {
      const uint32_t s = part.cbase + warp * 32u + lane;
      double f = s < n ? __ldcg(epi.fit + s) : -INFINITY;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) f = fmax(f, __shfl_xor_sync(0xFFFFFFFFu, f, o));
      if (lane == 0 && part.cbase + warp * 32u < n) a.word_max[part.cbase / 32u + warp] = f;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      a.chunk_done[part.chunk] = 0;
      for (uint32_t c = 0; c < kTailCounters; ++c)  // every CTA of the chunk is done claiming
        a.tail[(part.chunk * kTailCounters + c) * kTailStride] = 0;
      __threadfence();
      s_last = atomicAdd(&a.ctl->done, 1u) == chunks - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    timeline_mark(4, a.slot + 1);  // epilogue start (last chunk CTA)
    epi.word_max = a.word_max;
    epilogue_global(epi, nullptr, nullptr);
    timeline_mark(5, a.slot + 1);  // epilogue end
    if (threadIdx.x == 0) a.ctl->done = 0;
    return;
  }
  if (threadIdx.x == 0) s_last = ticket_acq_rel(&a.ctl->done) == gridDim.x - 1;
  __syncthreads();
  probe(a.exp_flags, 43);
  if (!s_last) return;
#ifdef GOMIX_TT_LAST_FENCE
  __threadfence();
#endif
  // (no fence: thread 0's acq_rel ticket and the barrier order this CTA's
  // loads after every other CTA's flush)
  probe_last(a.exp_flags, 44);
  timeline_mark(4, a.slot + 1);  // epilogue start (last CTA)
  epilogue_body(epi);
  probe_last(a.exp_flags, 45);
  timeline_mark(5, a.slot + 1);  // epilogue end
  if (threadIdx.x == 0) {
    a.ctl->done = 0;
    for (uint32_t c = 0; c < kTailCounters; ++c) a.tail[c * kTailStride] = 0;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {
// CTAs per SM the truth-table kernel is register-capped for (GOMIX_TT_OCC=4:
// 64 registers, for A/B measurements; default 3: 80 registers)
int tt_occupancy() {
  static const int occ = [] {
    const char* e = std::getenv("GOMIX_TT_OCC");
#ifdef GOMIX_TT_OCC2  // A/B builds: 2 CTAs per SM, 128 registers
    if (e && std::atoi(e) == 2) return 2;
#endif
    return (e && std::atoi(e) == 4) ? 4 : 3;
  }();
  return occ;
}

template <int b, int WC>
void* tt_kernel_for_occupancy() {
#ifdef GOMIX_TT_OCC2
  if (tt_occupancy() == 2) return (void*)gom_univ_tt_kernel<b, WC, 2>;
#endif
  return tt_occupancy() == 4 ? (void*)gom_univ_tt_kernel<b, WC, 4> : (void*)gom_univ_tt_kernel<b, WC, 3>;
}

template <int WC, bool MULTI>
void* univ_kernel_wc(int planes, bool tt) {
#define GOMIX_UNIV_CASE(b)                                                                            \
  case b:                                                                                             \
    return tt ? tt_kernel_for_occupancy<b, WC>() : (void*)gom_univ_sliced_kernel<b, WC, MULTI>;
  switch (planes) {
    GOMIX_UNIV_CASE(4)
    GOMIX_UNIV_CASE(6)
    GOMIX_UNIV_CASE(8)
    GOMIX_UNIV_CASE(12)
    GOMIX_UNIV_CASE(16)
  }
#undef GOMIX_UNIV_CASE
  throw GomixError(GOMIX_E_INVALID, "univariate sliced kernel: unsupported plane count");
}

// rows of up to 4 words in one pass, wider rows in passes of 4 words
int words_per_chunk(int wp) { return wp >= 4 ? 4 : wp; }

void* univ_kernel(int planes, int wp, bool tt) {
  if (tt) {  // truth tables: 1, 2 or 4 words per row, wider rows in 4-word chunks (one chunk per CTA)
    switch (words_per_chunk(wp)) {
      case 1: return univ_kernel_wc<1, false>(planes, true);
      case 2: return univ_kernel_wc<2, false>(planes, true);
      case 4: return univ_kernel_wc<4, false>(planes, true);
    }
  }
  // 12/16-plane counters for 4-word chunks do not fit the register budget
  // (T alone is 48/64 registers): 2-word passes instead
  if (planes >= 12 && wp >= 4 && !(tt && wp == 4)) return univ_kernel_wc<2, true>(planes, false);
  if (wp > 4) return univ_kernel_wc<4, true>(planes, tt);
  switch (words_per_chunk(wp)) {
    case 1: return univ_kernel_wc<1, false>(planes, tt);
    case 2: return univ_kernel_wc<2, false>(planes, tt);
    case 4: return univ_kernel_wc<4, false>(planes, tt);
  }
  throw GomixError(GOMIX_E_INVALID, "univariate sliced kernel: unsupported row width");
}

// dynamic shared memory of the adder kernel (the truth-table kernel's is static)
size_t univ_smem(int wp, bool tt) { return tt ? 0 : (size_t)wp * 32 * 24 + (size_t)wp * 4; }
}  // namespace

int univ_sliced_planes(uint64_t max_abs_row_sum) {
  // T <= A <= max_abs_row_sum must fit in B planes
  for (int b : {4, 6, 8, 12, 16})
    if (max_abs_row_sum < (1ull << b)) return b;
  return 0;
}

int univ_sliced_block() { return kUnivWarps * 32; }

int univ_sliced_sets_per_cta() { return kUnivWarps * 32; }

int univ_sliced_max_blocks_per_sm(int planes, int wp, bool tt) {
  void* fn = univ_kernel(planes, wp, tt);
  GOMIX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)univ_smem(wp, tt)));
  int blocks = 0;
  GOMIX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kUnivWarps * 32, univ_smem(wp, tt)));
  return blocks;
}

void launch_univ_sliced(const GomArgs& a, int planes, int wp, bool tt, int grid, cudaStream_t s, bool pdl) {
  void* fn = univ_kernel(planes, wp, tt);
  void* args[] = {(void*)&a};
  if (!pdl) {
    GOMIX_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kUnivWarps * 32), args, univ_smem(wp, tt), s));
    return;
  }
  // programmatic dependent launch: may begin while the previous kernel on the
  // stream finishes (the kernel waits with griddepcontrol.wait)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kUnivWarps * 32);
  cfg.dynamicSmemBytes = univ_smem(wp, tt);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GOMIX_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
}

void debug_timeline_univ(unsigned long long* out) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_timeline, sizeof(unsigned long long) * 32 * kTimelineRows));
  unsigned long long z[32 * kTimelineRows];
  for (int i = 0; i < 32 * kTimelineRows; ++i) z[i] = (i & 1) ? 0ull : ~0ull;
  GOMIX_CUDA(cudaMemcpyToSymbol(g_timeline, z, sizeof(z)));
}

void debug_cta_stats_univ(unsigned long long* out) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_ctastat, sizeof(unsigned long long) * kTimelineRows * kCtaStatMax * 4));
  GOMIX_CUDA(cudaMemcpyFromSymbol(out + kTimelineRows * kCtaStatMax * 4, g_ttcount, sizeof(unsigned long long) * 16));
  GOMIX_CUDA(cudaMemcpyFromSymbol(out + kTimelineRows * kCtaStatMax * 4 + 16, g_epiclk, sizeof(long long) * 16));
  unsigned long long z[16] = {};
  GOMIX_CUDA(cudaMemcpyToSymbol(g_ttcount, z, sizeof(z)));
}

void debug_probes_univ(unsigned long long* out, bool reset) {
  GOMIX_CUDA(cudaDeviceSynchronize());
  GOMIX_CUDA(cudaMemcpyFromSymbol(out, g_probe, sizeof(unsigned long long) * 64));
  if (reset) {
    unsigned long long z[64] = {};
    GOMIX_CUDA(cudaMemcpyToSymbol(g_probe, z, sizeof(z)));
  }
}

void build_univ_records(Problem& P) {
  const uint64_t m = P.m;
  P.urec = dev_alloc<uint4>(P.allocations, 2 * m);
  P.ukey = dev_alloc<ulonglong2>(P.allocations, m);
  build_univ_records_kernel<<<(unsigned)((m + 255) / 256), 256>>>(P.gvars, P.row_ptr, P.col, P.wi, m, P.urec,
                                                                  P.ukey);
  GOMIX_CUDA(cudaGetLastError());
}

}  // namespace gomix_b200
