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
// relative 1e-9); accepted pairs flip v.  Decisions and populations are
// therefore bit-identical to gom_group_kernel; fitness commits through the
// same deterministic per-CTA partials (within 1e-9 relative of the
// reference's position-order sums, north star).
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

template <int WPT>
__global__ void __launch_bounds__(kF64Warps * 32, 3) gom_univ_f64_kernel(const GomArgs a) {
  __shared__ __align__(16) uint32_t s_tail[kF64Warps * WPT * 32 * 6];  // gom_group_tail's team combine
  __shared__ double s_w[kF64Warps][kF64MaxDeg];
  __shared__ uint32_t s_nb[kF64Warps][kF64MaxDeg][WPT];
  if (*(volatile int32_t*)&a.ctl->stop) return;

  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
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
  double pfit[WPT], acc[WPT];
  unsigned long long dh1[WPT], dh2[WPT];
#pragma unroll
  for (int j = 0; j < WPT; ++j) {
    const uint32_t s = (uint32_t)j * 32u + lane;
    is_elit[j] = s < n && a.h1[s] == eh1 && a.h2[s] == eh2;
    pfit[j] = s < n ? a.fit[s] : 0.0;
    acc[j] = 0.0;
    dh1[j] = 0;
    dh2[j] = 0;
  }
  uint32_t steps = 0;
  unsigned long long calls = 0;

  const uint32_t stride = gridDim.x * kF64Warps;
  uint32_t p = blockIdx.x * kF64Warps + warp;
  uint4 rec = p < G ? __ldg(uvr + p) : make_uint4(0, 0, 0, 0);
  for (; p < G; p += stride) {
    // the next set's plan record: in flight while this one computes
    const uint32_t pn = p + stride;
    const uint4 rec_next = pn < G ? __ldg(uvr + pn) : make_uint4(0, 0, 0, 0);
    const uint32_t v = rec.x;
    const int32_t rs = (int32_t)rec.y, re = (int32_t)rec.z;
    const int32_t deg = re - rs;
    // v's row (every lane: the same 16 bytes) and, lane t, edge t's
    // neighbour row and weight, staged for the broadcast reads below
    uint32_t x[WPT];
    load_row_f64<WPT>(a.pop + (size_t)v * Wp, x);
    const ulonglong2 key = __ldg(ukey + p);
    double sn[WPT], so[WPT];
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      sn[j] = 0.0;
      so[j] = 0.0;
    }
    for (int32_t base = rs; base < re; base += kF64MaxDeg) {
      const int32_t cnt = min(kF64MaxDeg, re - base);
      if ((int32_t)lane < cnt) {
        const uint32_t u = (uint32_t)__ldg(a.col + base + (int32_t)lane);
        s_w[warp][lane] = __ldg(a.w + base + (int32_t)lane);
        uint32_t nb[WPT];
        load_row_f64<WPT>(a.pop + (size_t)u * Wp, nb);
#pragma unroll
        for (int j = 0; j < WPT; ++j) s_nb[warp][lane][j] = nb[j];
      }
      __syncwarp();
      for (int32_t t = 0; t < cnt; ++t) {
        const double wt = s_w[warp][t];
#pragma unroll
        for (int j = 0; j < WPT; ++j) {
          const uint32_t cut = ((x[j] ^ s_nb[warp][t][j]) >> lane) & 1u;
          sn[j] += cut ? 0.0 : wt;  // the reference adds every value, 0.0 included
          so[j] += cut ? wt : 0.0;
        }
      }
      __syncwarp();
    }
    uint32_t ones = 0;
#pragma unroll
    for (int j = 0; j < WPT; ++j) ones += __popc(x[j]);
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
      if (accept) acc[j] += delta;
      const uint32_t aw = __ballot_sync(0xFFFFFFFFu, accept);
      nw[j] = x[j] ^ aw;
      any |= aw != 0u;
      accb |= accept ? (1u << j) : 0u;
      if (accept && (int32_t)s == esrc) capture_row(a.elit, a.ever, ever_cur, v, (x[j] >> lane) & 1u);
      steps += present ? 1u : 0u;
      calls += present ? (uint32_t)deg : 0u;
    }
    if (any) {  // warp-uniform (ballots)
#pragma unroll
      for (int j = 0; j < WPT; ++j)
        if (accb & (1u << j)) {
          dh1[j] ^= key.x;
          dh2[j] ^= key.y;
        }
      if (lane == 0) {
        uint32_t* row = a.pop + (size_t)v * Wp;
#pragma unroll
        for (int j = 0; j < WPT; ++j)
          if (nw[j] != x[j]) row[j] = nw[j];
      }
    }
    rec = rec_next;
  }
  gom_group_tail<WPT, double>(a, epi, s_tail, kF64Warps, warp, 0u, 1u, lane, acc, dh1, dh2, steps, calls);
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
void* f64_kernel(int wp) {
  switch (wp) {
    case 1: return (void*)gom_univ_f64_kernel<1>;
    case 2: return (void*)gom_univ_f64_kernel<2>;
    case 4: return (void*)gom_univ_f64_kernel<4>;
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

void launch_univ_f64(const GomArgs& a, int wp, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  GOMIX_CUDA(cudaLaunchKernel(f64_kernel(wp), dim3(grid), dim3(kF64Warps * 32), args, 0, s));
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
