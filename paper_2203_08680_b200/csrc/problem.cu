// problem.cu — the shared, immutable model of a run (ModelArtifacts,
// model.hpp:25-29): validated Max-Cut instance as a device CSR graph, the FOS,
// its linkage-set interaction graph (LMIG, scheduling.hpp:35-68) and an exact
// GPU reproduction of the reference's Welsh-Powell colouring
// (scheduling.hpp:85-114), the colour groups and every set's footprint plan
// (make_group_plan, engine_parallel.hpp:37-59).
//
// Colouring: Welsh-Powell is greedy colouring in the order (degree desc,
// index asc).  Colouring every set as soon as all its higher-priority
// neighbours are coloured, with the smallest colour they do not use, is the
// same function computed in parallel (Jones-Plassmann with that priority);
// here it runs as a dataflow kernel (wp_dataflow_kernel).  So the groups, and
// with them replay parity, are identical to the reference's.
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>

#include <map>
#include <mutex>
#include <unordered_map>

#include "internal.cuh"

namespace gomix_b200 {
namespace cg = cooperative_groups;

// ---- device allocator (internal.cuh) -------------------------------------------
// Stream-ordered allocation from each device's default memory pool, with a
// release threshold so freed memory stays in the pool (cudaFree-free
// rebuilds: IMS creates and drops populations, bench / tests rebuild
// problems).  Allocations and frees go through one internal stream per
// device; an allocation is complete before cached_malloc returns, so any
// stream may use it.  Frees: callers synchronise the streams that used the
// block first (engine and problem destructors do), which makes the
// stream-ordered free safe.  The pool hands a freed block to the next
// allocation on the same internal stream; nothing is cleared, exactly like
// cudaMalloc.
namespace {
constexpr uint64_t kPoolKeep = 8ull << 30;  // bytes the pool keeps reserved across frees
struct DevicePool {
  std::once_flag once;
  cudaStream_t stream = nullptr;
};
DevicePool& pool_of(int dev) {
  static std::mutex mu;
  static std::map<int, DevicePool*> pools;  // never destroyed: frees may run during process exit
  std::lock_guard<std::mutex> lk(mu);
  DevicePool*& p = pools[dev];
  if (!p) p = new DevicePool;
  return *p;
}
DevicePool& current_pool() {
  int dev = 0;
  GOMIX_CUDA(cudaGetDevice(&dev));
  DevicePool& p = pool_of(dev);
  std::call_once(p.once, [&] {
    cudaMemPool_t mp = nullptr;
    GOMIX_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
    uint64_t keep = kPoolKeep;
    GOMIX_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep));
    GOMIX_CUDA(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
  });
  return p;
}
}  // namespace

void* cached_malloc(size_t bytes) {
  DevicePool& p = current_pool();
  void* ptr = nullptr;
  GOMIX_CUDA(cudaMallocAsync(&ptr, std::max<size_t>(bytes, 1), p.stream));
  GOMIX_CUDA(cudaStreamSynchronize(p.stream));
  return ptr;
}

void cached_free(void* ptr) {
  if (!ptr) return;
  cudaPointerAttributes at{};
  int dev = 0;
  if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess) dev = at.device;
  cudaGetLastError();
  int cur = 0;
  cudaGetDevice(&cur);
  if (dev != cur) cudaSetDevice(dev);
  DevicePool& p = current_pool();
  cudaFreeAsync(ptr, p.stream);
  if (dev != cur) cudaSetDevice(cur);
}

void cached_free_all(std::vector<void*>& blocks) {
  for (void* p : blocks) cached_free(p);
  blocks.clear();
}

Problem::~Problem() {
  cudaSetDevice(device);
  cudaDeviceSynchronize();  // engines' streams may still read the problem
  cached_free_all(allocations);
}

namespace {

int blocks_for(uint64_t n, int block = 256) {
  uint64_t g = (n + block - 1) / block;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(g, 65535ull * 16));
}

// entry -> owning set id, for a CSR of sets
__global__ void entry_owner_kernel(const int64_t* off, uint64_t m, uint32_t* owner) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    for (int64_t k = off[i]; k < off[i + 1]; ++k) owner[k] = (uint32_t)i;
}

__global__ void count_kernel(const uint32_t* keys, uint64_t cnt, int64_t* hist) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&hist[keys[i]], 1ull);
}

// LMIG candidate bound of set i: shared-variable sets plus sets of every
// interaction neighbour (scheduling.hpp:369-373).
__global__ void lmig_bound_kernel(const int64_t* set_off, const uint32_t* set_vars,
                                  const int64_t* vs_off, const int32_t* row_ptr,
                                  const int32_t* col, uint64_t m, int64_t* bound) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t b = 0;
    for (int64_t k = set_off[i]; k < set_off[i + 1]; ++k) {
      const uint32_t u = set_vars[k];
      b += vs_off[u + 1] - vs_off[u];
      for (int32_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
        const uint32_t x = (uint32_t)col[e];
        b += vs_off[x + 1] - vs_off[x];
      }
    }
    bound[i] = b;
  }
}

__global__ void lmig_fill_kernel(const int64_t* set_off, const uint32_t* set_vars,
                                 const int64_t* vs_off, const uint32_t* vs_sets,
                                 const int32_t* row_ptr, const int32_t* col, uint64_t m,
                                 const int64_t* cand_off, uint32_t* cand) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t at = cand_off[i];
    const uint32_t self = (uint32_t)i;
    for (int64_t k = set_off[i]; k < set_off[i + 1]; ++k) {
      const uint32_t u = set_vars[k];
      for (int64_t t = vs_off[u]; t < vs_off[u + 1]; ++t) cand[at++] = vs_sets[t];
      for (int32_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
        const uint32_t x = (uint32_t)col[e];
        for (int64_t t = vs_off[x]; t < vs_off[x + 1]; ++t) cand[at++] = vs_sets[t];
      }
    }
    // self appears at least once (shared variable); marked for removal below
    for (int64_t t = cand_off[i]; t < at; ++t)
      if (cand[t] == self) cand[t] = 0xFFFFFFFFu;
  }
}

// distinct values of a sorted segment, ignoring the 0xFFFFFFFF "self" marker
__global__ void unique_count_kernel(const uint32_t* keys, const int64_t* off, uint64_t m,
                                    int64_t* cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
      if (keys[t] != 0xFFFFFFFFu && (t == off[i] || keys[t] != keys[t - 1])) ++c;
    cnt[i] = c;
  }
}

__global__ void unique_fill_kernel(const uint32_t* keys, const int64_t* off, uint64_t m,
                                   const int64_t* out_off, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t at = out_off[i];
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
      if (keys[t] != 0xFFFFFFFFu && (t == off[i] || keys[t] != keys[t - 1])) out[at++] = keys[t];
  }
}

__global__ void wp_key_kernel(const int64_t* deg_off, uint64_t m, uint64_t maxdeg,
                              uint64_t* key) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = (uint64_t)(deg_off[i + 1] - deg_off[i]);
    key[i] = ((maxdeg - d) << 32) | i;  // degree desc, index asc (scheduling.hpp:89-93)
  }
}

__global__ void rank_kernel(const uint64_t* sorted_key, uint64_t m, uint32_t* rank) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < m;
       t += (uint64_t)gridDim.x * blockDim.x)
    rank[sorted_key[t] & 0xFFFFFFFFull] = (uint32_t)t;
}

// One Jones-Plassmann round in Welsh-Powell priority.  Colours are final once
// written, so reading a colour set earlier in the same round is safe.
__global__ void jp_round_kernel(const int64_t* off, const uint32_t* adj, const uint32_t* rank,
                                int32_t* colour, uint64_t m, unsigned long long* coloured) {
  unsigned long long mine = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    volatile int32_t* vc = colour;
    if (vc[i] >= 0) continue;
    const uint32_t ri = rank[i];
    bool ready = true;
    for (int64_t t = off[i]; t < off[i + 1]; ++t) {
      const uint32_t j = adj[t];
      if (rank[j] < ri && vc[j] < 0) {
        ready = false;
        break;
      }
    }
    if (!ready) continue;
    int32_t c = -1;
    for (int32_t base = 0; c < 0; base += 64) {
      uint64_t used = 0;
      for (int64_t t = off[i]; t < off[i + 1]; ++t) {
        const uint32_t j = adj[t];
        if (rank[j] < ri) {
          const int32_t cj = vc[j];
          if (cj >= base && cj < base + 64) used |= 1ull << (cj - base);
        }
      }
      if (~used) c = base + __ffsll((long long)~used) - 1;
    }
    vc[i] = c;
    __threadfence();
    ++mine;
  }
  if (mine) atomicAdd(coloured, mine);
}

// Welsh-Powell level by level (Kahn's order on the "lower-ranked neighbour"
// DAG): a vertex's colour depends only on its lower-ranked neighbours', so
// any topological order gives exactly the sequential greedy's colouring
// (scheduling.hpp:85-114).  pending[v] = lower-ranked neighbours not yet
// coloured; level 0 = the vertices with none.
__global__ void kahn_init_kernel(const int64_t* off, const uint32_t* adj, const uint32_t* rank, uint64_t m,
                                 uint32_t* pending, uint32_t* frontier, unsigned int* count) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < m; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t rv = rank[v];
    uint32_t c = 0;
    for (int64_t t = off[v]; t < off[v + 1]; ++t) c += rank[adj[t]] < rv ? 1u : 0u;
    pending[v] = c;
    if (c == 0) frontier[atomicAdd(count, 1u)] = (uint32_t)v;
  }
}

// One cooperative grid walks the levels: colour every vertex of the current
// level (smallest colour its lower-ranked neighbours leave free), release its
// higher-ranked neighbours into the next level, grid barrier.  Level counts
// rotate over three slots (read at L, appended at L + 1, cleared at L + 2).
// Stops after max_levels; whatever is left (long chains) goes to the
// dataflow kernel.  count[3] = levels run, count[4] = vertices coloured.
__global__ void kahn_levels_kernel(const int64_t* off, const uint32_t* adj, const uint32_t* rank, int32_t* colour,
                                   uint32_t* pending, uint32_t* fr0, uint32_t* fr1, uint32_t* fr2,
                                   unsigned int* count, uint32_t max_levels) {
  cg::grid_group grid = cg::this_grid();
  uint32_t* fr[3] = {fr0, fr1, fr2};
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t gsize = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long coloured = 0;
  uint32_t level = 0;
  for (; level < max_levels; ++level) {
    const uint32_t cur = level % 3u, nxt = (level + 1u) % 3u, old = (level + 2u) % 3u;
    const uint32_t n_cur = *(volatile unsigned int*)&count[cur];
    if (n_cur == 0) break;
    if (gtid == 0) count[old] = 0;
    for (uint64_t i = gtid; i < n_cur; i += gsize) {
      const uint32_t v = fr[cur][i];
      const uint32_t rv = rank[v];
      int32_t c = -1;
      for (int32_t base = 0; c < 0; base += 64) {
        uint64_t used = 0;
        for (int64_t t = off[v]; t < off[v + 1]; ++t) {
          const uint32_t j = adj[t];
          if (rank[j] < rv) {
            const int32_t cj = __ldcg(colour + j);
            if (cj >= base && cj < base + 64) used |= 1ull << (cj - base);
          }
        }
        if (~used) c = base + __ffsll((long long)~used) - 1;
      }
      colour[v] = c;
      ++coloured;
      for (int64_t t = off[v]; t < off[v + 1]; ++t) {
        const uint32_t u = adj[t];
        if (rank[u] > rv && atomicSub(&pending[u], 1u) == 1u) fr[nxt][atomicAdd(&count[nxt], 1u)] = u;
      }
    }
    __threadfence();
    grid.sync();
  }
  if (coloured) atomicAdd(reinterpret_cast<unsigned long long*>(count + 4), coloured);
  if (gtid == 0) count[3] = level;
}

// Welsh-Powell as a dataflow: the warp holding the vertex of rank r colours
// it as soon as every lower-ranked neighbour is coloured, with the smallest
// colour none of them uses — exactly the sequential greedy (scheduling.hpp:
// 85-114), but a chain link costs one shared-memory (or L2) hand-off instead
// of a kernel launch per Jones-Plassmann round.  Warps take ranks gw, gw+W,
// ... in increasing order, and the lowest uncoloured rank never waits, so a
// co-resident grid cannot deadlock.  SMEM: one CTA, colours as uint16 in
// shared memory (m <= kWpSmemMax); otherwise colours in global memory.
constexpr uint64_t kWpSmemMax = 100000;
constexpr int kJpBatches = 256;  // x 16 rounds before switching to the dataflow kernel
constexpr uint32_t kKahnMaxLevels = 8192;  // levels before the dataflow kernel takes the rest
constexpr uint32_t kWpUncoloured = 0xFFFFu;

// Welsh-Powell as a dataflow: a vertex's warp spins (volatile loads) until
// every lower-ranked neighbour has its colour, then writes its own.  The
// volatile read / write pairs on the colour array are the synchronisation
// itself: compute-sanitizer racecheck reports them as shared-memory hazards
// (it does not model spin-wait handoffs); every colour is written once, and
// the result equals the reference's sequential Welsh-Powell
// (tests/test_gpu_parity.py colouring cases).
template <bool SMEM>
__global__ void wp_dataflow_kernel(const int64_t* off, const uint32_t* adj, const uint32_t* rank,
                                   const uint64_t* sorted_key, uint64_t m, int32_t* colour) {
  extern __shared__ uint16_t scol[];
  if constexpr (SMEM) {
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) scol[i] = (uint16_t)kWpUncoloured;
    __syncthreads();
  }
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  auto load_colour = [&](uint32_t j) -> uint32_t {
    if constexpr (SMEM)
      return *(volatile uint16_t*)&scol[j];
    else
      return (uint32_t)*(volatile int32_t*)&colour[j];
  };
  for (uint64_t r = gw; r < m; r += nw) {
    const uint32_t v = (uint32_t)(sorted_key[r] & 0xFFFFFFFFull);
    if constexpr (!SMEM) {
      if (*(volatile int32_t*)&colour[v] >= 0) continue;  // coloured by the Jones-Plassmann rounds
    }
    const int64_t b = off[v], e = off[v + 1];
    // the mex of the lower-ranked neighbours' colours, 32 candidates at a time
    uint32_t c = 0xFFFFFFFFu;
    for (uint32_t base = 0; c == 0xFFFFFFFFu; base += 32) {
      uint32_t used = 0;
      for (int64_t t0 = b; t0 < e; t0 += 32) {
        const int64_t t = t0 + lane;
        uint32_t bit = 0;
        if (t < e) {
          const uint32_t j = adj[t];
          if (rank[j] < r) {
            uint32_t cj;
            const uint32_t unc = SMEM ? kWpUncoloured : 0xFFFFFFFFu;
            while ((cj = load_colour(j)) == unc) {
              if constexpr (!SMEM) __nanosleep(64);  // back off: keep L2 free for the writers
            }
            if (cj >= base && cj < base + 32) bit = 1u << (cj - base);
          }
        }
        used |= __reduce_or_sync(0xFFFFFFFFu, bit);
      }
      if (~used) c = base + (uint32_t)__ffs(~used) - 1;
    }
    if (lane == 0) {
      if constexpr (SMEM)
        *(volatile uint16_t*)&scol[v] = (uint16_t)c;
      else
        *(volatile int32_t*)&colour[v] = (int32_t)c;
    }
    __syncwarp();
  }
  if constexpr (SMEM) {
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) colour[i] = (int32_t)scol[i];
  }
}

__global__ void check_colouring_kernel(const int64_t* off, const uint32_t* adj,
                                       const int32_t* colour, uint64_t m, int32_t k,
                                       int* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (colour[i] < 0 || colour[i] >= k) {
      atomicExch(bad, 1);
      continue;
    }
    for (int64_t t = off[i]; t < off[i + 1]; ++t)
      if (colour[adj[t]] == colour[i]) atomicExch(bad, 1);
  }
}

__global__ void max_colour_kernel(const int32_t* colour, uint64_t m, int* mx) {
  int c = -1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    c = max(c, colour[i]);
  atomicMax(mx, c);
}

// footprint candidates: every subfunction (edge id) touching a variable of the set
__global__ void fp_bound_kernel(const int64_t* set_off, const uint32_t* set_vars,
                                const int32_t* row_ptr, uint64_t m, int64_t* bound) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t b = 0;
    for (int64_t k = set_off[i]; k < set_off[i + 1]; ++k)
      b += row_ptr[set_vars[k] + 1] - row_ptr[set_vars[k]];
    bound[i] = b;
  }
}

__global__ void fp_fill_kernel(const int64_t* set_off, const uint32_t* set_vars,
                               const int32_t* row_ptr, const int32_t* eid, uint64_t m,
                               const int64_t* cand_off, uint32_t* cand) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t at = cand_off[i];
    for (int64_t k = set_off[i]; k < set_off[i + 1]; ++k) {
      const uint32_t v = set_vars[k];
      for (int32_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) cand[at++] = (uint32_t)eid[e];
    }
  }
}

__device__ uint32_t encode_endpoint(uint32_t x, const uint32_t* vars, int64_t f) {
  int64_t lo = 0, hi = f;  // sets are sorted: binary search
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (vars[mid] < x) lo = mid + 1; else hi = mid;
  }
  return (lo < f && vars[lo] == x) ? (kInSet | (uint32_t)lo) : x;
}

__global__ void fp_entries_kernel(const int64_t* set_off, const uint32_t* set_vars,
                                  const uint32_t* eu, const uint32_t* ev, const double* ew,
                                  uint64_t m, const int64_t* fp_off, const uint32_t* fp_eid,
                                  FpEntry* fp) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* vars = set_vars + set_off[i];
    const int64_t f = set_off[i + 1] - set_off[i];
    for (int64_t t = fp_off[i]; t < fp_off[i + 1]; ++t) {
      const uint32_t e = fp_eid[t];
      FpEntry x;
      x.a = encode_endpoint(eu[e], vars, f);
      x.b = encode_endpoint(ev[e], vars, f);
      x.w = ew[e];
      fp[t] = x;
    }
  }
}

struct Scratch {
  std::vector<void*> bufs;
  template <typename T>
  T* get(size_t count) {
    void* p = cached_malloc(std::max<size_t>(count, 1) * sizeof(T));
    bufs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    cudaDeviceSynchronize();
    cached_free_all(bufs);
  }
};

void exclusive_scan(Scratch& S, const int64_t* in, int64_t* out, uint64_t cnt) {
  size_t bytes = 0;
  GOMIX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int64_t)cnt));
  void* tmp = S.get<char>(bytes);
  GOMIX_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int64_t)cnt));
}

int64_t read_back(const int64_t* p) {
  int64_t v = 0;
  GOMIX_CUDA(cudaMemcpy(&v, p, sizeof(v), cudaMemcpyDeviceToHost));
  return v;
}

// CSR of per-set candidate lists -> sorted, unique lists (seg sort + compaction)
void seg_sort_unique(Scratch& S, uint32_t* cand, const int64_t* cand_off, uint64_t m,
                     uint64_t total, int64_t** out_off, uint32_t** out_vals,
                     std::vector<void*>* keep) {
  uint32_t* sorted = S.get<uint32_t>(total);
  if (total > 0) {
    size_t bytes = 0;
    GOMIX_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, cand, sorted, (int64_t)total,
                                                  (int64_t)m, cand_off, cand_off + 1));
    void* tmp = S.get<char>(bytes);
    GOMIX_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, cand, sorted, (int64_t)total,
                                                  (int64_t)m, cand_off, cand_off + 1));
  }
  int64_t* cnt = S.get<int64_t>(m + 1);
  GOMIX_CUDA(cudaMemset(cnt, 0, (m + 1) * sizeof(int64_t)));
  unique_count_kernel<<<blocks_for(m), 256>>>(sorted, cand_off, m, cnt);
  GOMIX_CUDA(cudaGetLastError());
  int64_t* off = keep ? dev_alloc<int64_t>(*keep, m + 1) : S.get<int64_t>(m + 1);
  exclusive_scan(S, cnt, off, m + 1);
  const int64_t uniq = read_back(off + m);
  uint32_t* vals = keep ? dev_alloc<uint32_t>(*keep, (size_t)uniq) : S.get<uint32_t>((size_t)uniq);
  unique_fill_kernel<<<blocks_for(m), 256>>>(sorted, cand_off, m, off, vals);
  GOMIX_CUDA(cudaGetLastError());
  *out_off = off;
  *out_vals = vals;
}

}  // namespace

// ---- CSR from the edge list (create_problem) ---------------------------------
namespace {
__global__ void csr_count_kernel(const uint32_t* eu, const uint32_t* ev, uint64_t q, int32_t* cnt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (uint64_t)gridDim.x * blockDim.x) {
    atomicAdd(&cnt[eu[i] + 1], 1);
    atomicAdd(&cnt[ev[i] + 1], 1);
  }
}
// key = (row << 32) | neighbour: sorting makes every row contiguous and ascending
__global__ void csr_keys_kernel(const uint32_t* eu, const uint32_t* ev, uint64_t q, unsigned long long* key,
                                int32_t* val) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long u = eu[i], v = ev[i];
    key[2 * i] = (u << 32) | v;
    key[2 * i + 1] = (v << 32) | u;
    val[2 * i] = val[2 * i + 1] = (int32_t)i;
  }
}
__global__ void csr_fill_kernel(const unsigned long long* key, const int32_t* eidv, const double* ew, uint64_t cnt,
                                int32_t exact, int32_t* col, int32_t* eid, double* w, int32_t* wi) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t e = eidv[j];
    const double x = ew[e];
    col[j] = (int32_t)(uint32_t)(key[j] & 0xFFFFFFFFull);
    eid[j] = e;
    w[j] = x;
    wi[j] = exact && fabs(x) < 2147483648.0 ? (int32_t)x : 0;
  }
}
// max over rows of sum |wi| (the univariate kernels' plane count)
__global__ void csr_row_abs_kernel(const int32_t* row_ptr, const int32_t* wi, uint64_t nv, unsigned long long* mx) {
  unsigned long long best = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long a = 0;
    for (int32_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) a += (unsigned long long)llabs((long long)wi[e]);
    best = a > best ? a : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // one atomic per warp, not per row
    const unsigned long long y = __shfl_xor_sync(0xFFFFFFFFu, best, o);
    best = y > best ? y : best;
  }
  if ((threadIdx.x & 31u) == 0 && best) atomicMax(mx, best);
}
unsigned grid_for(uint64_t work) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 65535)); }
}  // namespace

void build_csr_device(Problem& P, bool exact, int32_t* d_eid, uint64_t* max_abs_row) {
  Scratch S;
  const uint64_t nv = P.nv, q = P.q, cnt2 = 2 * q;
  int32_t* cnt = S.get<int32_t>(nv + 1);
  GOMIX_CUDA(cudaMemset(cnt, 0, (nv + 1) * sizeof(int32_t)));
  if (q) csr_count_kernel<<<grid_for(q), 256>>>(P.eu, P.ev, q, cnt);
  GOMIX_CUDA(cudaGetLastError());
  {
    size_t bytes = 0;
    GOMIX_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, cnt, P.row_ptr, (int64_t)(nv + 1)));
    void* tmp = S.get<char>(bytes);
    GOMIX_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, cnt, P.row_ptr, (int64_t)(nv + 1)));
  }
  if (q) {
    unsigned long long* key = S.get<unsigned long long>(cnt2);
    unsigned long long* key_s = S.get<unsigned long long>(cnt2);
    int32_t* val = S.get<int32_t>(cnt2);
    int32_t* val_s = S.get<int32_t>(cnt2);
    csr_keys_kernel<<<grid_for(q), 256>>>(P.eu, P.ev, q, key, val);
    GOMIX_CUDA(cudaGetLastError());
    int end_bit = 64;  // only the bits a vertex id can occupy
    while (end_bit > 33 && !((nv - 1) >> (end_bit - 33))) --end_bit;
    size_t bytes = 0;
    GOMIX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key_s, val, val_s, (int64_t)cnt2, 0, end_bit));
    void* tmp = S.get<char>(bytes);
    GOMIX_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, key, key_s, val, val_s, (int64_t)cnt2, 0, end_bit));
    csr_fill_kernel<<<grid_for(cnt2), 256>>>(key_s, val_s, P.ew, cnt2, exact ? 1 : 0, P.col, d_eid, P.w, P.wi);
    GOMIX_CUDA(cudaGetLastError());
  }
  unsigned long long* mx = S.get<unsigned long long>(1);
  GOMIX_CUDA(cudaMemset(mx, 0, sizeof(unsigned long long)));
  csr_row_abs_kernel<<<grid_for(nv), 256>>>(P.row_ptr, P.wi, nv, mx);
  GOMIX_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  GOMIX_CUDA(cudaMemcpy(&h, mx, sizeof(h), cudaMemcpyDeviceToHost));
  *max_abs_row = h;
}

// Device part of problem construction.  Expects P's CSR, edge list and FOS
// already uploaded (row_ptr, col, eu, ev, ew, set_off, set_vars) and eid in
// `eid` (CSR entry -> edge id).
// GOMIX_TRACE_BUILD=1: per-phase wall times of the device build on stderr
struct PhaseClock {
  bool on = std::getenv("GOMIX_TRACE_BUILD") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[build] %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

void build_problem_device_impl(Problem& P, const int32_t* given_colour, const int32_t* eid) {
  Scratch S;
  PhaseClock clk;
  const uint64_t m = P.m, nv = P.nv, entries = P.h_set_off[m];
  // 1. inverse FOS: variable -> sets (ascending set id)
  uint32_t* owner = S.get<uint32_t>(entries);
  entry_owner_kernel<<<blocks_for(m), 256>>>(P.set_off, m, owner);
  GOMIX_CUDA(cudaGetLastError());
  uint32_t* vs_var = S.get<uint32_t>(entries);
  uint32_t* vs_sets = S.get<uint32_t>(entries);
  {
    size_t bytes = 0;
    GOMIX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, P.set_vars, vs_var, owner, vs_sets,
                                               (int64_t)entries));
    void* tmp = S.get<char>(bytes);
    GOMIX_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, P.set_vars, vs_var, owner, vs_sets,
                                               (int64_t)entries));
  }
  int64_t* vs_cnt = S.get<int64_t>(nv + 1);
  GOMIX_CUDA(cudaMemset(vs_cnt, 0, (nv + 1) * sizeof(int64_t)));
  count_kernel<<<blocks_for(entries), 256>>>(vs_var, entries, vs_cnt);
  GOMIX_CUDA(cudaGetLastError());
  int64_t* vs_off = S.get<int64_t>(nv + 1);
  exclusive_scan(S, vs_cnt, vs_off, nv + 1);

  clk.mark("fos-inverse");
  // 2. LMIG: sorted unique adjacency per set
  int64_t* bound = S.get<int64_t>(m + 1);
  GOMIX_CUDA(cudaMemset(bound, 0, (m + 1) * sizeof(int64_t)));
  lmig_bound_kernel<<<blocks_for(m), 256>>>(P.set_off, P.set_vars, vs_off, P.row_ptr, P.col, m, bound);
  GOMIX_CUDA(cudaGetLastError());
  int64_t* cand_off = S.get<int64_t>(m + 1);
  exclusive_scan(S, bound, cand_off, m + 1);
  const int64_t total = read_back(cand_off + m);
  uint32_t* cand = S.get<uint32_t>((size_t)total);
  lmig_fill_kernel<<<blocks_for(m), 256>>>(P.set_off, P.set_vars, vs_off, vs_sets, P.row_ptr,
                                           P.col, m, cand_off, cand);
  GOMIX_CUDA(cudaGetLastError());
  int64_t* lmig_off = nullptr;
  uint32_t* lmig_adj = nullptr;
  seg_sort_unique(S, cand, cand_off, m, (uint64_t)total, &lmig_off, &lmig_adj, nullptr);
  std::vector<int64_t> h_lmig_off(m + 1);
  GOMIX_CUDA(cudaMemcpy(h_lmig_off.data(), lmig_off, (m + 1) * sizeof(int64_t),
                        cudaMemcpyDeviceToHost));
  P.lmig_edges = (uint64_t)h_lmig_off[m] / 2;
  uint64_t maxdeg = 0;
  for (uint64_t i = 0; i < m; ++i)
    maxdeg = std::max<uint64_t>(maxdeg, (uint64_t)(h_lmig_off[i + 1] - h_lmig_off[i]));

  clk.mark("lmig");
  // 3. colouring
  int32_t* colour = S.get<int32_t>(m);
  if (given_colour) {
    GOMIX_CUDA(cudaMemcpy(colour, given_colour, m * sizeof(int32_t), cudaMemcpyHostToDevice));
  } else {
    uint64_t* key = S.get<uint64_t>(m);
    uint64_t* key_sorted = S.get<uint64_t>(m);
    wp_key_kernel<<<blocks_for(m), 256>>>(lmig_off, m, maxdeg, key);
    GOMIX_CUDA(cudaGetLastError());
    size_t bytes = 0;
    GOMIX_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, key, key_sorted, (int64_t)m));
    void* tmp = S.get<char>(bytes);
    GOMIX_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, key, key_sorted, (int64_t)m));
    uint32_t* rank = S.get<uint32_t>(m);
    rank_kernel<<<blocks_for(m), 256>>>(key_sorted, m, rank);
    GOMIX_CUDA(cudaGetLastError());
    GOMIX_CUDA(cudaMemset(colour, 0xFF, m * sizeof(int32_t)));
    unsigned long long done = 0;
    if (m <= kWpSmemMax && maxdeg < kWpUncoloured) {
      // one CTA, colours in shared memory: a chain link is a shared-memory hand-off
      const size_t sm = m * sizeof(uint16_t);
      GOMIX_CUDA(cudaFuncSetAttribute(wp_dataflow_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      wp_dataflow_kernel<true><<<1, 1024, sm>>>(lmig_off, lmig_adj, rank, key_sorted, m, colour);
      GOMIX_CUDA(cudaGetLastError());
    } else {
      // Kahn levels in one cooperative grid while the levels are wide
      // (grids, univariate: ~2W levels), then the dataflow kernel for
      // whatever long chains are left (e.g. neighbourhood sets in index
      // order: one chain of m links).  GOMIX_COLOUR=jp: Jones-Plassmann
      // rounds instead (round 1's scheme, A/B measurements).
      static const bool use_jp = [] {
        const char* e = std::getenv("GOMIX_COLOUR");
        return e && std::string(e) == "jp";
      }();
      if (!use_jp) {
        uint32_t* pending = S.get<uint32_t>(m);
        uint32_t* fr0 = S.get<uint32_t>(m);
        uint32_t* fr1 = S.get<uint32_t>(m);
        uint32_t* fr2 = S.get<uint32_t>(m);
        unsigned int* count = S.get<unsigned int>(6);  // 3 level slots, levels, coloured (u64)
        GOMIX_CUDA(cudaMemset(count, 0, 6 * sizeof(unsigned int)));
        kahn_init_kernel<<<blocks_for(m), 256>>>(lmig_off, lmig_adj, rank, m, pending, fr0, count);
        GOMIX_CUDA(cudaGetLastError());
        int dev = 0, sms = 0, per = 0;
        GOMIX_CUDA(cudaGetDevice(&dev));
        GOMIX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        GOMIX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kahn_levels_kernel, 256, 0));
        static const int kahn_grid = [] {  // GOMIX_KAHN_GRID: CTAs of the level walk (A/B)
          const char* e = std::getenv("GOMIX_KAHN_GRID");
          return e ? std::atoi(e) : 0;
        }();
        // one CTA per SM: a level costs its dependent memory round trips, not
        // threads (measured: 18 ms at C3 for 148 CTAs as for 4, 21 ms for 296)
        const int grid = std::max(1, std::min(kahn_grid > 0 ? kahn_grid : sms, per * sms));
        uint32_t max_levels = kKahnMaxLevels;
        void* args[] = {(void*)&lmig_off, (void*)&lmig_adj, (void*)&rank, (void*)&colour, (void*)&pending,
                        (void*)&fr0, (void*)&fr1, (void*)&fr2, (void*)&count, (void*)&max_levels};
        GOMIX_CUDA(cudaLaunchCooperativeKernel((void*)kahn_levels_kernel, dim3(grid), dim3(256), args, 0, nullptr));
        unsigned long long got = 0;
        GOMIX_CUDA(cudaMemcpy(&got, count + 4, sizeof(got), cudaMemcpyDeviceToHost));
        done = got;
      } else {
        unsigned long long* coloured = S.get<unsigned long long>(1);
        GOMIX_CUDA(cudaMemset(coloured, 0, sizeof(unsigned long long)));
        for (int batch = 0; batch < kJpBatches && done < m; ++batch) {
          for (int r = 0; r < 16; ++r)
            jp_round_kernel<<<blocks_for(m), 256>>>(lmig_off, lmig_adj, rank, colour, m, coloured);
          GOMIX_CUDA(cudaGetLastError());
          GOMIX_CUDA(cudaMemcpy(&done, coloured, sizeof(done), cudaMemcpyDeviceToHost));
        }
      }
    }
    if ((m > kWpSmemMax || maxdeg >= kWpUncoloured) && done < m) {
      // co-resident grid (cooperative launch), colours in global memory; a
      // warp whose vertex is already coloured moves on
      int dev = 0, sms = 0, per = 0;
      GOMIX_CUDA(cudaGetDevice(&dev));
      GOMIX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      GOMIX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wp_dataflow_kernel<false>, 256, 0));
      const int grid = std::max(1, std::min(per * sms, blocks_for(m * 32)));
      void* args[] = {(void*)&lmig_off, (void*)&lmig_adj, (void*)&rank, (void*)&key_sorted, (void*)&m,
                      (void*)&colour};
      GOMIX_CUDA(cudaLaunchCooperativeKernel((void*)wp_dataflow_kernel<false>, dim3(grid), dim3(256), args, 0,
                                             nullptr));
    }
  }
  int* mx = S.get<int>(2);
  const int init[2] = {-1, 0};
  GOMIX_CUDA(cudaMemcpy(mx, init, sizeof(init), cudaMemcpyHostToDevice));
  max_colour_kernel<<<blocks_for(m), 256>>>(colour, m, mx);
  GOMIX_CUDA(cudaGetLastError());
  int kmax = 0;
  GOMIX_CUDA(cudaMemcpy(&kmax, mx, sizeof(int), cudaMemcpyDeviceToHost));
  P.k = (uint64_t)(kmax + 1);
  check_colouring_kernel<<<blocks_for(m), 256>>>(lmig_off, lmig_adj, colour, m, (int32_t)P.k, mx + 1);
  GOMIX_CUDA(cudaGetLastError());
  int bad = 0;
  GOMIX_CUDA(cudaMemcpy(&bad, mx + 1, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad) invalid("colouring: adjacent linkage sets share a colour (groups must be independent)");

  clk.mark("colouring");
  // 4. groups: sets by colour, ascending set id inside a colour (scheduling.hpp:418-422)
  {
    uint32_t* ids = S.get<uint32_t>(m);
    std::vector<uint32_t> h_ids(m);
    std::iota(h_ids.begin(), h_ids.end(), 0u);
    GOMIX_CUDA(cudaMemcpy(ids, h_ids.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice));
    int32_t* col_sorted = S.get<int32_t>(m);
    P.gsets = dev_alloc<uint32_t>(P.allocations, m);
    size_t bytes = 0;
    GOMIX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, colour, col_sorted, ids, P.gsets,
                                               (int64_t)m));
    void* tmp = S.get<char>(bytes);
    GOMIX_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, colour, col_sorted, ids, P.gsets,
                                               (int64_t)m));
    std::vector<int32_t> h_col(m);
    std::vector<uint32_t> h_gs(m);
    GOMIX_CUDA(cudaMemcpy(h_col.data(), col_sorted, m * sizeof(int32_t), cudaMemcpyDeviceToHost));
    GOMIX_CUDA(cudaMemcpy(h_gs.data(), P.gsets, m * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    P.group_off.assign(P.k + 1, 0);
    for (uint64_t i = 0; i < m; ++i) P.group_off[(size_t)h_col[i] + 1]++;
    for (uint64_t c = 0; c < P.k; ++c) P.group_off[c + 1] += P.group_off[c];
    P.group_sets.assign(h_gs.begin(), h_gs.end());
    if (P.univariate) {  // variable of each member, in group order
      std::vector<uint32_t> gv(m);
      for (uint64_t i = 0; i < m; ++i) gv[i] = P.h_set_vars[P.h_set_off[h_gs[i]]];
      P.gvars = dev_alloc<uint32_t>(P.allocations, m);
      GOMIX_CUDA(cudaMemcpy(P.gvars, gv.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
  }

  clk.mark("groups");
  // 5. footprint plans (multi-variable sets only; singletons read the CSR row)
  P.footprint.assign(m, 0);
  if (!P.univariate) {
    int64_t* fb = S.get<int64_t>(m + 1);
    GOMIX_CUDA(cudaMemset(fb, 0, (m + 1) * sizeof(int64_t)));
    fp_bound_kernel<<<blocks_for(m), 256>>>(P.set_off, P.set_vars, P.row_ptr, m, fb);
    GOMIX_CUDA(cudaGetLastError());
    int64_t* fc_off = S.get<int64_t>(m + 1);
    exclusive_scan(S, fb, fc_off, m + 1);
    const int64_t ftotal = read_back(fc_off + m);
    uint32_t* fcand = S.get<uint32_t>((size_t)ftotal);
    fp_fill_kernel<<<blocks_for(m), 256>>>(P.set_off, P.set_vars, P.row_ptr, eid, m, fc_off, fcand);
    GOMIX_CUDA(cudaGetLastError());
    uint32_t* fp_eid = nullptr;
    seg_sort_unique(S, fcand, fc_off, m, (uint64_t)ftotal, &P.fp_off, &fp_eid, &P.allocations);
    std::vector<int64_t> h_fp_off(m + 1);
    GOMIX_CUDA(cudaMemcpy(h_fp_off.data(), P.fp_off, (m + 1) * sizeof(int64_t),
                          cudaMemcpyDeviceToHost));
    P.fp = dev_alloc<FpEntry>(P.allocations, (size_t)h_fp_off[m]);
    fp_entries_kernel<<<blocks_for(m), 256>>>(P.set_off, P.set_vars, P.eu, P.ev, P.ew, m, P.fp_off,
                                              fp_eid, P.fp);
    GOMIX_CUDA(cudaGetLastError());
    for (uint64_t i = 0; i < m; ++i) {
      P.footprint[i] = (uint64_t)(h_fp_off[i + 1] - h_fp_off[i]);
      P.max_fp = std::max(P.max_fp, P.footprint[i]);
    }
    if ((uint64_t)h_fp_off[m] >= (1ull << 32) || P.h_set_off[m] >= (1ull << 32) || P.max_fp >= (1u << 24))
      invalid("fos: footprint plans exceed 32-bit offsets");
    // per group position: {set id, vars offset, footprint offset, f << 24 | footprint}
    std::vector<uint4> gm(m);
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t sid = P.group_sets[i];
      const uint64_t f = P.h_set_off[sid + 1] - P.h_set_off[sid];
      gm[i] = make_uint4((uint32_t)sid, (uint32_t)P.h_set_off[sid], (uint32_t)h_fp_off[sid],
                         (uint32_t)((f << 24) | P.footprint[sid]));
    }
    P.gmeta = dev_alloc<uint4>(P.allocations, m);
    GOMIX_CUDA(cudaMemcpy(P.gmeta, gm.data(), m * sizeof(uint4), cudaMemcpyHostToDevice));
  }
  GOMIX_CUDA(cudaDeviceSynchronize());
  clk.mark("plans");
}

}  // namespace gomix_b200
