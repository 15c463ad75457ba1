// gom_peer.cu — the peer-transport kernels outside the GOM launches
// (protocol: gom_peer.cuh): the member exchange after init / load, the
// per-generation presence maps of a univariate FOS, and the elitist
// genotype broadcast.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gom_common.cuh"
#include "gom_peer.cuh"

namespace gomix_b200 {

namespace {

// Init / load_population: the member exchange alone (one CTA).
__global__ void peer_exchange_kernel(const EpiArgs a) { peer_exchange(a); }

// Presence maps of this rank's rows: bit v of any1 = some local member holds
// 1 at v, of any0 = some local member holds 0; written into slot `rank` of
// every rank's block.  The last CTA raises this rank's flag everywhere.
__global__ void presence_publish_kernel(const PeerArgs* pap, DevCtl* ctl, const uint32_t* pop, uint64_t nv,
                                        uint32_t Wp, uint32_t n_local) {
  const PeerArgs& pa = *pap;
  // the epoch lives in the control block (the kernel may sit in a CUDA
  // graph): every CTA reads it here; only the last CTA, after every CTA's
  // ticket, advances it
  const unsigned long long epoch = *(volatile unsigned long long*)&ctl->xp_epoch + 1;
  const PeerLayout L(pa.R, pa.n, pa.w32);
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const size_t par = epoch & 1ull;
  for (uint64_t w = warp; w < pa.w32; w += nwarps) {
    const uint64_t v = w * 32u + lane;
    uint32_t ones = 0;
    if (v < nv)
      for (uint32_t j = 0; j < Wp; ++j) ones += __popc(pop[v * Wp + j]);
    const uint32_t a1 = __ballot_sync(0xFFFFFFFFu, v < nv && ones > 0u);
    const uint32_t a0 = __ballot_sync(0xFFFFFFFFu, v < nv && ones < n_local);
    if (lane < pa.R) {  // lane p writes this word into rank p's block
      char* b = pa.blocks[lane];
      reinterpret_cast<uint32_t*>(b + L.any1)[(par * pa.R + pa.rank) * pa.w32 + w] = a1;
      reinterpret_cast<uint32_t*>(b + L.any0)[(par * pa.R + pa.rank) * pa.w32 + w] = a0;
    }
  }
  __threadfence_system();
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(&ctl->xp_ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  ctl->xp_ticket = 0;
  ctl->xp_epoch = epoch;
  __threadfence_system();
  for (uint32_t p = 0; p < pa.R; ++p)
    st_release_sys(reinterpret_cast<unsigned long long*>(pa.blocks[p] + L.pflags) + par * pa.R + pa.rank, epoch);
}

// Every rank's maps in this rank's block -> ones[v] in the form the GOM
// kernels' presence test reads (present iff 0 < ones < n_global): 1 when some
// member anywhere holds 0 and some holds 1, 0 when all hold 0, n_global when
// all hold 1.  Few CTAs: on one GPU the peers' publish kernels must still
// find room while these wait.
__global__ void presence_combine_kernel(const PeerArgs* pap, DevCtl* ctl, uint32_t* ones, uint64_t nv,
                                        uint32_t n_global) {
  const PeerArgs& pa = *pap;
  const unsigned long long epoch = *(volatile unsigned long long*)&ctl->xp_epoch;  // advanced by the publish
  const PeerLayout L(pa.R, pa.n, pa.w32);
  const size_t par = epoch & 1ull;
  __shared__ int s_ok;
  if (threadIdx.x == 0)
    s_ok = peer_wait(reinterpret_cast<const unsigned long long*>(pa.blocks[pa.rank] + L.pflags) + par * pa.R, pa.R,
                     epoch, pa.timeout_ns);
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) {
      ctl->peer_fault = 1;
      ctl->stop = 1;
    }
    return;
  }
  const char* own = pa.blocks[pa.rank];
  const uint32_t* any0 = reinterpret_cast<const uint32_t*>(own + L.any0) + par * pa.R * pa.w32;
  const uint32_t* any1 = reinterpret_cast<const uint32_t*>(own + L.any1) + par * pa.R * pa.w32;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w = v >> 5;
    uint32_t a0 = 0, a1 = 0;
    for (uint32_t r = 0; r < pa.R; ++r) {
      a0 |= __ldcg(any0 + (size_t)r * pa.w32 + w);
      a1 |= __ldcg(any1 + (size_t)r * pa.w32 + w);
    }
    const uint32_t b = 1u << (v & 31u);
    ones[v] = (a0 & a1 & b) ? 1u : ((a1 & b) ? n_global : 0u);
  }
}

// The elitist's owner writes its snapshot bits into every other rank's block.
__global__ void peer_elitist_send_kernel(const PeerArgs* pap, DevCtl* ctl, const uint32_t* elit,
                                         unsigned long long epoch) {
  const PeerArgs& pa = *pap;
  const PeerLayout L(pa.R, pa.n, pa.w32);
  const size_t par = epoch & 1ull;
  for (uint32_t p = 0; p < pa.R; ++p) {
    if (p == pa.rank) continue;
    uint32_t* dst = reinterpret_cast<uint32_t*>(pa.blocks[p] + L.ebits) + par * pa.w32;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < pa.w32; w += (uint64_t)gridDim.x * blockDim.x)
      dst[w] = elit[w];
  }
  __threadfence_system();
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) s_last = atomicAdd(&ctl->xp_ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  ctl->xp_ticket = 0;
  __threadfence_system();
  for (uint32_t p = 0; p < pa.R; ++p)
    if (p != pa.rank) st_release_sys(reinterpret_cast<unsigned long long*>(pa.blocks[p] + L.eflags) + par, epoch);
}

// ... and every other rank waits for them and takes them as its snapshot.
__global__ void peer_elitist_recv_kernel(const PeerArgs* pap, DevCtl* ctl, uint32_t* elit, unsigned long long epoch) {
  const PeerArgs& pa = *pap;
  const PeerLayout L(pa.R, pa.n, pa.w32);
  const size_t par = epoch & 1ull;
  __shared__ int s_ok;
  if (threadIdx.x == 0)
    s_ok = peer_wait(reinterpret_cast<const unsigned long long*>(pa.blocks[pa.rank] + L.eflags) + par, 1, epoch,
                     pa.timeout_ns);
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) ctl->peer_fault = 1;
    return;
  }
  const uint32_t* src = reinterpret_cast<const uint32_t*>(pa.blocks[pa.rank] + L.ebits) + par * pa.w32;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < pa.w32; w += (uint64_t)gridDim.x * blockDim.x)
    elit[w] = __ldcg(src + w);
}

}  // namespace

size_t peer_block_bytes(uint32_t R, uint32_t n, uint32_t w32) { return PeerLayout(R, n, w32).bytes; }

void launch_peer_exchange(const EpiArgs& a, cudaStream_t s) {
  peer_exchange_kernel<<<1, 256, 0, s>>>(a);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_presence(const PeerArgs* d_peer, DevCtl* ctl, const uint32_t* pop, uint64_t nv, uint32_t Wp,
                     uint32_t n_local, uint32_t n_global, uint32_t* ones, cudaStream_t s) {
  const uint64_t w32 = (nv + 31) / 32;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((w32 + 7) / 8, 148 * 4));
  presence_publish_kernel<<<grid, 256, 0, s>>>(d_peer, ctl, pop, nv, Wp, n_local);
  GOMIX_CUDA(cudaGetLastError());
  presence_combine_kernel<<<32, 256, 0, s>>>(d_peer, ctl, ones, nv, n_global);
  GOMIX_CUDA(cudaGetLastError());
}

void launch_peer_elitist(const PeerArgs* d_peer, DevCtl* ctl, uint32_t* elit, uint64_t nv, bool owner,
                         unsigned long long epoch, cudaStream_t s) {
  const uint64_t w32 = (nv + 31) / 32;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((w32 + 255) / 256, 148));
  if (owner)
    peer_elitist_send_kernel<<<grid, 256, 0, s>>>(d_peer, ctl, elit, epoch);
  else
    peer_elitist_recv_kernel<<<std::min(grid, 32u), 256, 0, s>>>(d_peer, ctl, elit, epoch);
  GOMIX_CUDA(cudaGetLastError());
}

}  // namespace gomix_b200
