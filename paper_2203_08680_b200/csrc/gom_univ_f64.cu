// gom_univ_f64.cu — the batched GOM step for a univariate FOS on float
// weights (BASELINE C4: random d-regular graphs, fp64 weights) in Philox
// mode: one warp per linkage set {v}, lane = solution, every word of the
// population row in registers (n <= 128).
//
// Semantics (engine_parallel.hpp:104-247, as gom_group_kernel's univariate
// path): the pair (s, {v}) is present iff some member holds the other value
// of v (every differing donor then holds !x_v, so the move is the flip and
// the draw is skipped); Δ = Σnew − Σold with both sums taken left to right
// over v's edges in ascending edge id (:164-186) — Σold over the cut edges,
// Σnew over the uncut ones, every term added, zeros included, exactly as the
// reference's reduce_by_key does; accept iff better(parent + Δ, parent) or
// equal and the parent is not the group-start elitist (graybox.hpp:22-35,
// relative 1e-9); accepted pairs flip v.  Decisions, populations and the
// fixed-point fitness sums are therefore bit-identical to gom_group_kernel
// (within 1e-9 relative of the reference's position-order sums, north star).
//
// Why a second kernel: the group kernel walks set -> row_ptr -> CSR ->
// neighbour rows as a dependent chain per set and broadcasts every edge with
// shuffles.  Here the plan record {v, row start, row end} and v's Zobrist key
// come from one per-position table, the next set's record is in flight while
// the current set computes, the edge weights are staged in shared memory
// (one broadcast load per edge instead of two 32-bit shuffles), and the
// neighbour rows are read once per set as 16-byte loads.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "gom_common.cuh"
#include "gom_tail.cuh"

namespace gomix_b200 {

namespace {
constexpr int kF64Warps = 8;
constexpr int kF64MaxDeg = 32;  // edges per set handled in one pass (one per lane)
}  // namespace

template <int WPT>
__device__ __forceinline__ void load_row_f64(const uint32_t* row, uint32_t (&x)[WPT]) {
  if constexpr (WPT == 4) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(row));
    x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
  } else if constexpr (WPT == 2) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(row));
    x[0] = t.x; x[1] = t.y;
  } else {
    x[0] = __ldg(row);
  }
}

// One set's loads that do not depend on this launch's writes to the
// population rows of its own group: the plan record, v's row (written only
// by this warp, after it is read), v's key and lane t's edge.
template <int WPT>
struct F64Next {
  uint4 rec;
  uint32_t x[WPT];
  ulonglong2 key;
  uint32_t u;
  double w;
};

template <int WPT>
__device__ __forceinline__ F64Next<WPT> f64_fetch(const GomArgs& a, const uint4* uvr, const ulonglong2* ukey,
                                                  uint32_t G, uint32_t p, uint32_t lane) {
  F64Next<WPT> r;
#pragma unroll
  for (int j = 0; j < WPT; ++j) r.x[j] = 0;
  r.u = 0;
  r.w = 0.0;
  r.key = make_ulonglong2(0ull, 0ull);
  r.rec = make_uint4(0, 0, 0, 0);
  if (p >= G) return r;
  r.rec = __ldg(uvr + p);
  r.key = __ldg(ukey + p);
  load_row_f64<WPT>(a.pop + (size_t)r.rec.x * WPT, r.x);
  const int32_t e = (int32_t)r.rec.y + (int32_t)lane;
  if (e < (int32_t)r.rec.z) {
    r.u = (uint32_t)__ldg(a.col + e);
    r.w = __ldg(a.w + e);
  }
  return r;
}

template <int WPT, int MINB>
__global__ void __launch_bounds__(kF64Warps * 32, MINB) gom_univ_f64_kernel(const GomArgs a) {
  __shared__ __align__(16) uint32_t s_tail[kF64Warps * WPT * 32 * 6];  // gom_group_tail's team combine
  __shared__ double s_w[kF64Warps][kF64MaxDeg];
  __shared__ uint32_t s_nb[kF64Warps][kF64MaxDeg][WPT];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  // programmatic dependent launch (graph path): everything below reads what
  // the previous group's launch wrote (population, control block, hashes)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (*(volatile int32_t*)&a.ctl->stop) return;
  const uint32_t n = a.n;
  constexpr uint32_t Wp = (uint32_t)WPT;
  uint32_t G = a.G;
  const uint4* uvr = a.uvr;
  const ulonglong2* ukey = a.ukey;
  EpiArgs epi = a.epi;
  if (a.slot >= 0) {  // graph path: this launch's group comes from the device-side order
    const uint32_t gi = a.order[a.slot];
    const GroupDesc d = a.groups[gi];
    G = d.G;
    uvr += d.g0;
    ukey += d.g0;
    epi.group = gi;
    epi.G = G;
  }
  // group-start "parent == elitist" (engine_parallel.hpp:202) and parent
  // fitness of this lane's solutions, read once per launch
  const unsigned long long eh1 = a.ctl->eh1, eh2 = a.ctl->eh2;
  const int32_t esrc = a.ctl->elit_src;
  const uint32_t ever_cur = a.ctl->elit_ver;
  const bool exact = a.exact != 0;
  bool is_elit[WPT];
  double pfit[WPT];
  long long acc[WPT];  // fixed-point fitness deltas (GomArgs::fix_scale)
  unsigned long long dh1[WPT], dh2[WPT];
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    const uint32_t s = (uint32_t)j * 32u + lane;
    is_elit[j] = s < n && a.h1[s] == eh1 && a.h2[s] == eh2;
    pfit[j] = s < n ? a.fit[s] : 0.0;
    acc[j] = 0;
    dh1[j] = 0;
    dh2[j] = 0;
  }
  uint32_t steps = 0;
  unsigned long long calls = 0;

  const uint32_t stride = gridDim.x * kF64Warps;
  uint32_t p = blockIdx.x * kF64Warps + warp;
  // Software pipeline over this warp's sets (every set has at most
  // kF64MaxDeg edges: one edge per lane).  While set p computes, the loads
  // of set p + stride that do not depend on the population in flight:
  // its record, then v's row, key, and lane t's edge (neighbour id, weight);
  // only the neighbour rows are loaded at the top of an iteration.
  F64Next<WPT> cur = f64_fetch<WPT>(a, uvr, ukey, G, p, lane);
  for (; p < G; p += stride) {
    const uint32_t v = cur.rec.x;
    const int32_t deg = (int32_t)(cur.rec.z - cur.rec.y);
    uint32_t nb[WPT];
#pragma unroll
    for (int j = 0; j < WPT; ++j) nb[j] = 0;
    if ((int32_t)lane < deg) load_row_f64<WPT>(a.pop + (size_t)cur.u * Wp, nb);
    const F64Next<WPT> nxt = f64_fetch<WPT>(a, uvr, ukey, G, p + stride, lane);
    s_w[warp][lane] = cur.w;
#pragma unroll
    for (int j = 0; j < WPT; ++j) s_nb[warp][lane][j] = nb[j];
    __syncwarp();
    double sn[WPT], so[WPT];
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      sn[j] = 0.0;
      so[j] = 0.0;
    }
    for (int32_t t = 0; t < deg; ++t) {
      const double wt = s_w[warp][t];
#pragma unroll
      for (int j = 0; j < WPT; ++j) {
        const uint32_t cut = ((cur.x[j] ^ s_nb[warp][t][j]) >> lane) & 1u;
        sn[j] += cut ? 0.0 : wt;  // the reference adds every value, 0.0 included
        so[j] += cut ? wt : 0.0;
      }
    }
    __syncwarp();
    uint32_t ones = 0;
#pragma unroll
    for (int j = 0; j < WPT; ++j) ones += __popc(cur.x[j]);
    const bool set_present = ones > 0u && ones < a.n_global;
    uint32_t accb = 0;
    uint32_t nw[WPT];
    bool any = false;
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      const uint32_t s = (uint32_t)j * 32u + lane;
      const bool present = s < n && set_present;
      bool accept = false;
      const double delta = sn[j] - so[j];
      if (present) {
        const double pf = pfit[j];
        const double cand = pf + delta;
        accept = exact ? (delta > 0.0 || (delta == 0.0 && !is_elit[j]))
                       : (cmp_better(false, cand, pf) || (cmp_equal(false, cand, pf) && !is_elit[j]));
      }
      if (accept) acc[j] += __double2ll_rn(delta * a.fix_scale);
      const uint32_t aw = __ballot_sync(0xFFFFFFFFu, accept);
      nw[j] = cur.x[j] ^ aw;
      any |= aw != 0u;
      accb |= accept ? (1u << j) : 0u;
      if (accept && (int32_t)s == esrc) capture_row(a.elit, a.ever, ever_cur, v, (cur.x[j] >> lane) & 1u);
      steps += present ? 1u : 0u;
      calls += present ? (uint32_t)deg : 0u;
    }
    if (any) {  // warp-uniform (ballots)
#pragma unroll
      for (int j = 0; j < WPT; ++j)
        if (accb & (1u << j)) {
          dh1[j] ^= cur.key.x;
          dh2[j] ^= cur.key.y;
        }
      if (lane == 0) {
        uint32_t* row = a.pop + (size_t)v * Wp;
#pragma unroll
        for (int j = 0; j < WPT; ++j)
          if (nw[j] != cur.x[j]) row[j] = nw[j];
      }
    }
    cur = nxt;
  }
  // the next group's launch may start its prologue (it waits for this
  // grid's completion before touching anything written here)
  asm volatile("griddepcontrol.launch_dependents;");
  gom_group_tail<WPT>(a, epi, s_tail, kF64Warps, warp, 0u, 1u, lane, acc, dh1, dh2, steps, calls);
}

// Plan of a univariate FOS, per group position: {v, row start, row end, 0}
// and v's Zobrist key (shared with the truth-table plan when that exists).
__global__ void build_univ_plan_kernel(const uint32_t* gvars, const int32_t* row_ptr, uint64_t m, uint4* uvr,
                                       ulonglong2* key) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m) return;
  const uint32_t v = gvars[p];
  uvr[p] = make_uint4(v, (uint32_t)row_ptr[v], (uint32_t)row_ptr[v + 1], 0u);
  if (key) {
    unsigned long long z1, z2;
    zobrist(v, z1, z2);
    key[p] = make_ulonglong2(z1, z2);
  }
}

namespace {
// CTAs per SM the kernel is register-capped for: 3 (80 registers, some
// spills of the prefetch state) or 2 (no spills); GOMIX_F64_OCC for A/B
int f64_occupancy() {
  static const int occ = [] {
    const char* e = std::getenv("GOMIX_F64_OCC");
    return (e && std::atoi(e) == 2) ? 2 : 3;
  }();
  return occ;
}

void* f64_kernel(int wp) {
  const bool two = f64_occupancy() == 2;
  switch (wp) {
    case 1: return two ? (void*)gom_univ_f64_kernel<1, 2> : (void*)gom_univ_f64_kernel<1, 3>;
    case 2: return two ? (void*)gom_univ_f64_kernel<2, 2> : (void*)gom_univ_f64_kernel<2, 3>;
    case 4: return two ? (void*)gom_univ_f64_kernel<4, 2> : (void*)gom_univ_f64_kernel<4, 3>;
  }
  throw GomixError(GOMIX_E_INVALID, "univariate f64 kernel: unsupported row width");
}
}  // namespace

int univ_f64_max_blocks_per_sm(int wp) {
  int blocks = 0;
  GOMIX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, f64_kernel(wp), kF64Warps * 32, 0));
  return blocks;
}

int univ_f64_sets_per_cta() { return kF64Warps; }

int univ_f64_max_degree() { return kF64MaxDeg; }

void launch_univ_f64(const GomArgs& a, int wp, int grid, cudaStream_t s, bool pdl) {
  void* args[] = {(void*)&a};
  if (!pdl) {
    GOMIX_CUDA(cudaLaunchKernel(f64_kernel(wp), dim3(grid), dim3(kF64Warps * 32), args, 0, s));
    return;
  }
  // programmatic dependent launch: may begin while the previous group's
  // kernel finishes (this kernel waits with griddepcontrol.wait)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kF64Warps * 32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GOMIX_CUDA(cudaLaunchKernelExC(&cfg, f64_kernel(wp), args));
}

void build_univ_plan(Problem& P) {
  const uint64_t m = P.m;
  P.uvr = dev_alloc<uint4>(P.allocations, m);
  const bool need_key = P.ukey == nullptr;
  if (need_key) P.ukey = dev_alloc<ulonglong2>(P.allocations, m);
  build_univ_plan_kernel<<<(unsigned)((m + 255) / 256), 256>>>(P.gvars, P.row_ptr, m, P.uvr,
                                                              need_key ? P.ukey : nullptr);
  GOMIX_CUDA(cudaGetLastError());
}

}  // namespace gomix_b200
