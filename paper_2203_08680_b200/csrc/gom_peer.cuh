// gom_peer.cuh — the sharded engine's exchanges over peer memory (NVLink P2P
// mappings of every rank's exchange block, CUDA IPC across processes),
// executed by the GOM kernels themselves instead of NCCL calls between
// launches.
//
// One population sharded over R GPUs needs, after every
// colour group, every rank's fitness, hashes and counters of its members
// (engine_parallel.hpp:305-310: the elitist scan runs over all n), and, once
// per generation for a univariate variable-once FOS, which rows hold both
// values anywhere (the presence test; rows themselves never cross ranks).
// With the peer transport the last CTA of a rank's GOM launch commits its
// members, writes them into slot `rank` of EVERY rank's exchange block,
// raises its flag there, waits for all R flags in its own block and runs the
// global elitist scan — compute, collective and epilogue in one kernel.
//
// Protocol.  Exchanges are numbered (epochs, kept in each rank's control
// block; every rank runs the same sequence, so the numbers agree).  Slots are
// double-buffered by epoch parity: a rank can publish epoch e + 1 while a
// slower one still reads epoch e, and cannot reach e + 2 before every rank
// has published e + 1, which each does only after reading e.  Writes go out
// before the flag (__threadfence_system, then a release store); readers
// acquire the flags.  A wait that exceeds PeerArgs::timeout_ns latches a
// fault in the control block instead of hanging the GPU.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace gomix_b200 {

constexpr uint32_t kMaxRanks = 16;

// Every rank's exchange block, mapped into this process (own included).
struct PeerArgs {
  char* blocks[kMaxRanks];
  uint32_t R, rank, n, w32;  // ranks, this rank, members per rank, 32-row words of a presence map
  unsigned long long timeout_ns;
};

// Byte offsets inside one exchange block (R ranks, n members each, w32 words).
struct PeerLayout {
  size_t flags, pflags, eflags, fit, h1, h2, cnt, any0, any1, ebits, bytes;
  __host__ __device__ PeerLayout(uint32_t R, uint32_t n, uint32_t w32) {
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    flags = 0;                                  // u64 [2][R]  group exchanges
    pflags = flags + 16 * (size_t)R;            // u64 [2][R]  presence maps
    eflags = pflags + 16 * (size_t)R;           // u64 [2]     elitist broadcast
    fit = up(eflags + 16);                      // f64 [2][R][n]
    h1 = up(fit + 16 * (size_t)R * n);          // u64 [2][R][n]
    h2 = up(h1 + 16 * (size_t)R * n);           // u64 [2][R][n]
    cnt = up(h2 + 16 * (size_t)R * n);          // u64 [2][R][2]  steps, calls
    any0 = up(cnt + 32 * (size_t)R);            // u32 [2][R][w32]  rows with a member holding 0
    any1 = up(any0 + 8 * (size_t)R * w32);      // u32 [2][R][w32]  ... holding 1
    ebits = up(any1 + 8 * (size_t)R * w32);     // u32 [2][w32]     the elitist genotype
    bytes = up(ebits + 8 * (size_t)w32);
  }
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread 0: wait until flags[0 .. count) >= epoch (acquire); false on timeout.
__device__ __forceinline__ bool peer_wait(const unsigned long long* flags, uint32_t count, unsigned long long epoch,
                                          unsigned long long timeout_ns) {
  const unsigned long long t0 = global_ns();
  for (uint32_t r = 0; r < count; ++r) {
    while (ld_acquire_sys(flags + r) < epoch) {
      if (global_ns() - t0 > timeout_ns) return false;
      __nanosleep(256);
    }
  }
  return true;
}

// The group exchange, run by ONE whole CTA after this rank committed its
// members (commit_local): publish fitness, hashes and counters to every
// rank, wait for every rank, gather into fit_all / h1_all / h2_all /
// rank_cnt (what the global elitist scan reads).  Returns false on a timeout
// (the control block's peer_fault is set and the run stopped).
static __device__ bool peer_exchange(const EpiArgs& a) {
  const PeerArgs& pa = *a.peer;
  const PeerLayout L(pa.R, pa.n, pa.w32);
  const uint32_t R = pa.R, n = pa.n, me = pa.rank;
  __shared__ unsigned long long s_epoch;
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    s_epoch = a.ctl->xg_epoch + 1;
    a.ctl->xg_epoch = s_epoch;
  }
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const size_t par = epoch & 1ull;
  const double* fit = a.fit_all + (size_t)me * n;
  const unsigned long long* h1 = a.h1_all + (size_t)me * n;
  const unsigned long long* h2 = a.h2_all + (size_t)me * n;
  for (uint32_t p = 0; p < R; ++p) {
    char* b = pa.blocks[p];
    double* dfit = reinterpret_cast<double*>(b + L.fit) + (par * R + me) * n;
    unsigned long long* dh1 = reinterpret_cast<unsigned long long*>(b + L.h1) + (par * R + me) * n;
    unsigned long long* dh2 = reinterpret_cast<unsigned long long*>(b + L.h2) + (par * R + me) * n;
    for (uint32_t s = threadIdx.x; s < n; s += blockDim.x) {
      dfit[s] = fit[s];
      dh1[s] = h1[s];
      dh2[s] = h2[s];
    }
    if (threadIdx.x < 2) {
      unsigned long long* dc = reinterpret_cast<unsigned long long*>(b + L.cnt) + (par * R + me) * 2;
      dc[threadIdx.x] = a.rank_cnt[2 * me + threadIdx.x];
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t p = 0; p < R; ++p)
      st_release_sys(reinterpret_cast<unsigned long long*>(pa.blocks[p] + L.flags) + par * R + me, epoch);
    s_ok = peer_wait(reinterpret_cast<const unsigned long long*>(pa.blocks[me] + L.flags) + par * R, R, epoch,
                     pa.timeout_ns);
  }
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) {
      a.ctl->peer_fault = 1;
      a.ctl->stop = 1;
      a.ctl->stop_reason = GOMIX_STOP_NONE;
    }
    return false;
  }
  const char* own = pa.blocks[me];
  for (uint32_t i = threadIdx.x; i < R * n; i += blockDim.x) {
    const size_t at = par * R * n + i;
    const_cast<double*>(a.fit_all)[i] = reinterpret_cast<const double*>(own + L.fit)[at];
    const_cast<unsigned long long*>(a.h1_all)[i] = reinterpret_cast<const unsigned long long*>(own + L.h1)[at];
    const_cast<unsigned long long*>(a.h2_all)[i] = reinterpret_cast<const unsigned long long*>(own + L.h2)[at];
  }
  for (uint32_t i = threadIdx.x; i < 2 * R; i += blockDim.x)
    a.rank_cnt[i] = reinterpret_cast<const unsigned long long*>(own + L.cnt)[par * R * 2 + i];
  __syncthreads();
  return true;
}

}  // namespace gomix_b200
