// gom_fi.cu — a parallel-friendly Forced Improvement (FI) phase: the paper's
// future work (§5.4: "the design of a procedure akin to FI that is
// more amenable to parallelization"), SURVEY.md §8(f) row 4.
//
// The reference's FI (engine_serial.hpp:98-128, SerialEngine only) walks the
// FOS of ONE stagnating solution o in a fresh random order with the elitist
// as donor (gom_step with the elitist tie rule), halts at the first strict
// improvement, and replaces o by the elitist when a whole pass brings none.
// Its trigger (engine_serial.hpp:176-186): o accepted no GOM move in the
// generation, or o has not strictly improved for more than
// 1 + floor(log10 n) generations.
//
// Parallel-friendly restatement (what these kernels and the engine do):
//   * trigger, per solution at the end of a generation: "accepted no move" is
//     "genotype unchanged since the generation started" (Zobrist hash
//     equality; every accepted GOM move copies differing donor genes), and
//     the stagnation counter is kept per solution as in SerialEngine;
//   * the FI pass walks the colour GROUPS in a fresh random order; in a group
//     every triggered solution that has not yet strictly improved takes the
//     elitist as donor on every set of the group at once (sets of a group
//     are independent, engine_parallel.hpp:22-25) — one batched GOM step with
//     the donor tape {elitist where it differs on the set, else none}, run by
//     the ordinary group kernel and epilogue (accept rule, fitness, hashes,
//     evaluator calls, elitist scan, stop criteria);
//   * "halt at the first strict improvement" becomes: a solution leaves the
//     pass after the first GROUP that left it strictly better than at the
//     start of the pass;
//   * solutions still not strictly better after every group become copies of
//     the elitist (fitness, hash and genotype).
// The elitist is a population column at every group boundary (the chained
// scan always ends on the current member it copied), so the donor tape names
// that column; an elitist adopted from outside (IMS offer, elit_src < 0)
// skips FI for that generation.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "gom_common.cuh"

namespace gomix_b200 {

namespace {
constexpr int kFiBlock = 256;
unsigned fi_blocks(uint64_t work) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 1u << 20)); }

__device__ __forceinline__ uint32_t pop_bit(const FiArgs& a, uint64_t v, uint32_t s) {
  return (a.pop[v * a.Wp + (s >> 5)] >> (s & 31u)) & 1u;
}

// still in the pass: triggered and not yet strictly better than at its start
__device__ __forceinline__ bool fi_active(const FiArgs& a, uint32_t s) {
  return a.flag[s] && !cmp_better(a.ctl->exact != 0, a.fit[s], a.fit0[s]);
}
}  // namespace

// generation start: fitness and genotype hashes the trigger compares against
__global__ void fi_snapshot_kernel(const FiArgs a) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  a.fit_start[s] = a.fit[s];
  a.h1s[s] = a.h1[s];
  a.h2s[s] = a.h2[s];
}

// generation end: the trigger (engine_serial.hpp:176-186) -> flag, pass start fitness
__global__ void fi_flags_kernel(const FiArgs a) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  const DevCtl* c = a.ctl;
  const bool improved = cmp_better(c->exact != 0, a.fit[s], a.fit_start[s]);
  const bool changed = a.h1[s] != a.h1s[s] || a.h2[s] != a.h2s[s];
  const int32_t pending = improved ? 0 : a.stag[s] + 1;
  const bool run = !c->stop && c->elit_src >= 0;
  a.flag[s] = run && (!changed || pending > a.threshold) ? 1 : 0;
  a.fit0[s] = a.fit[s];
}

// explicit flags (gomix_gpu_forced_improvement): pass start fitness
__global__ void fi_given_flags_kernel(const FiArgs a) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  const DevCtl* c = a.ctl;
  if (c->stop || c->elit_src < 0) a.flag[s] = 0;
  a.fit0[s] = a.fit[s];
}

// donor tape of one group, p-major [p * n + s]: the elitist column where it
// differs from s on the set and s is still in the pass, else -1
__global__ void fi_tape_kernel(const FiArgs a, uint64_t g0, uint64_t G, int32_t* tape) {
  const DevCtl* c = a.ctl;
  const int32_t src = c->elit_src;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < G * a.n;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = t / a.n;
    const uint32_t s = (uint32_t)(t % a.n);
    int32_t d = -1;
    if (src >= 0 && !c->stop && fi_active(a, s)) {
      const uint32_t sid = a.gsets[g0 + p];
      for (int64_t k = a.set_off[sid]; k < a.set_off[sid + 1]; ++k) {
        const uint32_t v = a.set_vars[k];
        if (pop_bit(a, v, s) != pop_bit(a, v, (uint32_t)src)) {
          d = src;
          break;
        }
      }
    }
    tape[p * a.n + s] = d;
  }
}

// solutions still in the pass after every group, as word masks
__global__ void fi_mask_kernel(const FiArgs a) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t w = s >> 5;
  if (w >= a.Wp) return;
  const bool take = s < a.n && !a.ctl->stop && a.ctl->elit_src >= 0 && fi_active(a, s);
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, take);
  if ((threadIdx.x & 31u) == 0) a.mask[w] = m;
}

// ... become copies of the elitist column: genotype rows
__global__ void fi_copy_rows_kernel(const FiArgs a) {
  const int32_t src = a.ctl->elit_src;
  if (src < 0) return;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < a.nv * a.Wp;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t m = a.mask[t % a.Wp];
    if (!m) continue;
    const uint64_t v = t / a.Wp;
    const uint32_t e = pop_bit(a, v, (uint32_t)src) ? m : 0u;
    a.pop[t] = (a.pop[t] & ~m) | e;
  }
}

// ... fitness and hashes; then the stagnation counters (engine_serial.hpp:187)
__global__ void fi_finish_kernel(const FiArgs a, int32_t update_stag) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.n) return;
  const DevCtl* c = a.ctl;
  if ((a.mask[s >> 5] >> (s & 31u)) & 1u) {
    a.fit[s] = c->elit_fit;
    a.h1[s] = c->eh1;
    a.h2[s] = c->eh2;
  }
  if (update_stag) a.stag[s] = cmp_better(c->exact != 0, a.fit[s], a.fit_start[s]) ? 0 : a.stag[s] + 1;
}

void launch_fi_snapshot(const FiArgs& a, cudaStream_t s) {
  fi_snapshot_kernel<<<fi_blocks(a.n), kFiBlock, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_fi_flags(const FiArgs& a, bool given, cudaStream_t s) {
  if (given)
    fi_given_flags_kernel<<<fi_blocks(a.n), kFiBlock, 0, s>>>(a);
  else
    fi_flags_kernel<<<fi_blocks(a.n), kFiBlock, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_fi_tape(const FiArgs& a, uint64_t g0, uint64_t G, int32_t* tape, cudaStream_t s) {
  fi_tape_kernel<<<fi_blocks(G * a.n), kFiBlock, 0, s>>>(a, g0, G, tape);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_fi_finish(const FiArgs& a, bool update_stag, cudaStream_t s) {
  fi_mask_kernel<<<(unsigned)((a.Wp * 32 + kFiBlock - 1) / kFiBlock), kFiBlock, 0, s>>>(a);
  fi_copy_rows_kernel<<<fi_blocks(a.nv * a.Wp), kFiBlock, 0, s>>>(a);
  fi_finish_kernel<<<fi_blocks(a.n), kFiBlock, 0, s>>>(a, update_stag ? 1 : 0);
  GOMIX_CUDA(cudaGetLastError());
}

}  // namespace gomix_b200
