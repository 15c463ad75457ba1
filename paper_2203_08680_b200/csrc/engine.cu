// engine.cu — host side of libgomix_b200: problem construction (validation,
// CSR build), the per-population engine (ParallelEngine,
// engine_parallel.hpp:255-368) and the C-ABI of include/gomix_gpu.h.
//
// Host work per generation is O(k) launches in Philox mode and one stream
// sync; the device keeps population, fitness, elitist and the run-control
// block resident across generations.  Replay mode additionally brings the
// packed population back once per group to draw donors exactly like the
// reference's sequential RngStream (engine_parallel.hpp:104-121).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is resolved at run time with dlopen

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "gomix_gpu.h"
#include "internal.cuh"
#include "gom_peer.cuh"

namespace gomix_b200 {
void build_problem_device_impl(Problem& P, const int32_t* given_colour, const int32_t* eid);
}

using namespace gomix_b200;

namespace {

thread_local std::string g_last_error;

// latency-study instrumentation switch (GOMIX_EXP at load, gomix_debug_set_flags)
std::atomic<uint32_t> g_exp_flags{[] {
  const char* ex = std::getenv("GOMIX_EXP");
  return ex ? (uint32_t)std::atoi(ex) : 0u;
}()};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return GOMIX_OK;
  } catch (const GomixError& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return GOMIX_E_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return GOMIX_E_STATE;
  }
}

uint32_t next_pow2(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

// ===========================================================================
// problem
// ===========================================================================
struct gomix_gpu_problem {
  std::unique_ptr<Problem> P;
};

namespace {

// validate_instance (maxcut.hpp:39-54) + Fos sanity (linkage.hpp:279-309) and
// the CSR build: row v = edges (a, v), a < v, then (v, b), b > v, both in edge
// order -> ascending neighbour = ascending edge id (the reference's order).
std::unique_ptr<Problem> create_problem(const gomix_maxcut* inst, const gomix_fos* fos,
                                        const int32_t* colour, int32_t device) {
  const bool trace = std::getenv("GOMIX_TRACE_BUILD") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[host ] %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_start).count());
    t_start = now;
  };
  if (!inst || !fos) invalid("problem: instance and fos are required");
  const uint64_t nv = inst->num_vertices, q = inst->num_edges, m = fos->num_sets;
  if (nv == 0) invalid("maxcut: instance needs at least one vertex");
  if (nv >= (1ull << 31)) invalid("maxcut: at most 2^31-1 vertices");
  if (q >= (1ull << 30)) invalid("maxcut: at most 2^30-1 edges");
  if (q && (!inst->edge_u || !inst->edge_v || !inst->edge_w)) invalid("maxcut: missing edge arrays");
  bool exact = true;
  double maxw = 0.0, sum_abs_w = 0.0;
  for (uint64_t i = 0; i < q; ++i) {
    const uint32_t u = inst->edge_u[i], v = inst->edge_v[i];
    const double w = inst->edge_w[i];
    if (u >= v) invalid("maxcut: edge endpoints must satisfy u < v");
    if (v >= nv) invalid("maxcut: edge endpoint out of range");
    if (!std::isfinite(w)) invalid("maxcut: non-finite edge weight");
    if (i > 0) {
      const uint32_t pu = inst->edge_u[i - 1], pv = inst->edge_v[i - 1];
      if (pu > u || (pu == u && pv >= v)) invalid("maxcut: edges must be sorted and unique");
    }
    if (w != std::floor(w) || std::fabs(w) > 9e15) exact = false;
    maxw = std::max(maxw, std::fabs(w));
    sum_abs_w += std::fabs(w);
  }
  if (m == 0) invalid("fos: needs at least one linkage set");
  if (!fos->set_offset || !fos->set_vars) invalid("fos: missing arrays");
  if (fos->set_offset[0] != 0) invalid("fos: set_offset[0] must be 0");

  auto P = std::make_unique<Problem>();
  P->nv = nv;
  P->q = q;
  P->m = m;
  P->exact = exact;
  P->sum_abs_w = sum_abs_w;
  P->h_set_off.assign(fos->set_offset, fos->set_offset + m + 1);
  const uint64_t entries = P->h_set_off[m];
  P->h_set_vars.assign(fos->set_vars, fos->set_vars + entries);
  P->univariate = true;
  for (uint64_t i = 0; i < m; ++i) {
    const uint64_t a = P->h_set_off[i], b = P->h_set_off[i + 1];
    if (b <= a) invalid("fos: set " + std::to_string(i) + " is empty");
    if (b - a > (uint64_t)kMaxSetSize)
      invalid("fos: set " + std::to_string(i) + " has more than 64 variables (unsupported)");
    for (uint64_t t = a; t < b; ++t) {
      if (P->h_set_vars[t] >= nv) invalid("scheduling: linkage set references unknown variable");
      if (t > a && P->h_set_vars[t] <= P->h_set_vars[t - 1])
        invalid("fos: set " + std::to_string(i) + " is not sorted and unique");
    }
    P->max_f = std::max<uint64_t>(P->max_f, b - a);
    if (b - a != 1) P->univariate = false;
  }
  {
    std::vector<uint8_t> seen(nv, 0);
    for (uint64_t t = 0; t < entries && P->var_once; ++t) {
      if (seen[P->h_set_vars[t]]) P->var_once = false;
      seen[P->h_set_vars[t]] = 1;
    }
  }
  if (colour) {
    for (uint64_t i = 0; i < m; ++i)
      if (colour[i] < 0) invalid("colouring: negative colour");
  }

  mark("validate");
  if (device >= 0) GOMIX_CUDA(cudaSetDevice(device));
  GOMIX_CUDA(cudaGetDevice(&P->device));

  // CSR, built on the device from the uploaded edge list (build_csr_device):
  // row v = v's neighbours ascending = its edges in ascending edge id (the
  // reference's summation order for sorted edge lists)
  auto& A = P->allocations;
  P->row_ptr = dev_alloc<int32_t>(A, nv + 1);
  P->col = dev_alloc<int32_t>(A, 2 * q);
  P->w = dev_alloc<double>(A, 2 * q);
  P->wi = dev_alloc<int32_t>(A, 2 * q);
  P->eu = dev_alloc<uint32_t>(A, q);
  P->ev = dev_alloc<uint32_t>(A, q);
  P->ew = dev_alloc<double>(A, q);
  P->set_off = dev_alloc<int64_t>(A, m + 1);
  P->set_vars = dev_alloc<uint32_t>(A, entries);
  int32_t* d_eid = dev_alloc<int32_t>(A, 2 * q);
  auto up = [](void* dst, const void* src, size_t bytes) {
    if (bytes) GOMIX_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  };
  up(P->eu, inst->edge_u, q * 4);
  up(P->ev, inst->edge_v, q * 4);
  up(P->ew, inst->edge_w, q * 8);
  std::vector<int64_t> so(P->h_set_off.begin(), P->h_set_off.end());
  up(P->set_off, so.data(), (m + 1) * 8);
  up(P->set_vars, P->h_set_vars.data(), entries * 4);
  uint64_t max_abs_row = 0;
  build_csr_device(*P, exact, d_eid, &max_abs_row);
  std::vector<int32_t> row_ptr(nv + 1);
  GOMIX_CUDA(cudaMemcpy(row_ptr.data(), P->row_ptr, (nv + 1) * 4, cudaMemcpyDeviceToHost));
  uint64_t max_deg_sum = 0;
  for (uint64_t i = 0; i < m; ++i) {
    uint64_t s = 0;
    for (uint64_t t = P->h_set_off[i]; t < P->h_set_off[i + 1]; ++t)
      s += (uint64_t)(row_ptr[P->h_set_vars[t] + 1] - row_ptr[P->h_set_vars[t]]);
    max_deg_sum = std::max(max_deg_sum, s);
  }
  // int32 per-pair arithmetic is exact when |delta| <= max|w| * footprint < 2^30
  P->i32 = exact && maxw * (double)std::max<uint64_t>(max_deg_sum, 1) < 1073741824.0;
  P->wbits = 1;
  while (P->i32 && P->wbits < 31 && (double)(1u << P->wbits) <= maxw) ++P->wbits;
  if (P->univariate) {
    for (uint64_t i = 0; i < m; ++i) {
      const uint32_t v = P->h_set_vars[i];
      P->max_fp = std::max<uint64_t>(P->max_fp, (uint64_t)(row_ptr[v + 1] - row_ptr[v]));
    }
    P->max_abs_row = max_abs_row;  // over every vertex: univariate sets cover a subset of them
  }
  mark("csr+upload");
  build_problem_device_impl(*P, colour, d_eid);
  // truth-table plan of the bit-sliced univariate kernel (every variable of
  // degree <= 4, int16 weights)
  if (P->univariate && P->i32 && P->max_fp <= 4 && maxw < 32768.0 && univ_sliced_planes(P->max_abs_row) > 0)
    build_univ_records(*P);
  if (P->univariate) build_univ_plan(*P);  // {v, row} records + keys of every position (gom_univ_f64.cu)
  GOMIX_CUDA(cudaDeviceSynchronize());  // engines read the problem from their own (non-blocking) streams
  mark("device");
  if (P->univariate) {
    for (uint64_t i = 0; i < m; ++i) {
      const uint32_t v = P->h_set_vars[i];
      P->footprint[i] = (uint64_t)(row_ptr[v + 1] - row_ptr[v]);
    }
  }
  return P;
}

}  // namespace

// ===========================================================================
// NCCL, resolved at run time (the process's already-loaded libnccl.so.2, e.g.
// PyTorch's, or the system one), so the library has no link-time dependency.
// ===========================================================================
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
#define GOMIX_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
    GOMIX_SYM(GetUniqueId, "ncclGetUniqueId");
    GOMIX_SYM(CommInitRank, "ncclCommInitRank");
    GOMIX_SYM(CommDestroy, "ncclCommDestroy");
    GOMIX_SYM(AllGather, "ncclAllGather");
    GOMIX_SYM(Broadcast, "ncclBroadcast");
    GOMIX_SYM(AllReduce, "ncclAllReduce");
    GOMIX_SYM(GroupStart, "ncclGroupStart");
    GOMIX_SYM(GroupEnd, "ncclGroupEnd");
    GOMIX_SYM(GetErrorString, "ncclGetErrorString");
#undef GOMIX_SYM
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.Broadcast && a.AllReduce &&
           a.GroupStart && a.GroupEnd && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks required symbols";
    return a;
  }();
  return api;
}

const NcclApi& nccl_or_throw() {
  const NcclApi& a = nccl_api();
  if (!a.ok) throw GomixError(GOMIX_E_NCCL, a.why);
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw GomixError(GOMIX_E_NCCL, std::string(what) + ": " + nccl_api().GetErrorString(r));
}
}  // namespace

struct NcclComm {
  ncclComm_t comm = nullptr;
  ~NcclComm() {
    if (comm) nccl_api().CommDestroy(comm);
  }
};

// ===========================================================================
// engine
// ===========================================================================

struct gomix_gpu_engine {
  Problem* P = nullptr;
  uint64_t n = 0;          // this rank's solutions
  uint64_t n_global = 0;   // population size
  uint32_t R = 1, rank = 0;
  std::unique_ptr<NcclComm> nccl;    // one process per GPU
  // peer transport (GOMIX_FLAG_PEER_TRANSPORT, gom_peer.cuh): this rank's
  // exchange block (cudaMalloc: IPC-exportable), every rank's mapped block
  bool peer_on = false;
  char* xblock = nullptr;
  size_t xbytes = 0;
  std::vector<void*> peer_opened;  // cudaIpcOpenMemHandle mappings to close
  PeerArgs* d_peer = nullptr;
  unsigned long long xe_epoch = 0;  // elitist broadcasts (host-driven; group / presence epochs live in DevCtl)
  gomix_gpu_local_group* local = nullptr;  // several shards in one process
  uint32_t W = 0, Wp = 0, wpt = 1, tw = 1, block = 256, teams = 8, stage_words = 0;
  size_t smem = 0;
  int grid_cap = 1;
  int univ_planes = 0;     // > 0: Philox groups run the bit-sliced lane-per-set kernel
  bool univ_tt = false;    // ... its truth-table variant (degree <= 4 plan records)
  uint32_t tt_chunks = 1;  // > 1: n > 128, rows processed in 4-word chunks (counted rows in `ones`)
  unsigned int* chunk_done = nullptr;  // ... per-chunk CTA tickets of a launch
  double* word_max = nullptr;          // ... per-word fitness maxima after the chunk commits
  unsigned int* tail_ctr = nullptr;    // truth-table kernel: dynamic batch counters (kTailCounters per chunk)
  bool univ_f64 = false;   // univariate, non-int32 weights, Philox: gom_univ_f64_kernel
  int f64_grid_cap = 1;
  int univ_grid_cap = 1;
  // Sharded univariate runs on a variable-once FOS: a row changes only in its
  // own group, so its count of 1s over all ranks (the presence test) is
  // exchanged once per generation and the per-group exchange drops the rows.
  bool lite = false;
  uint32_t* ones = nullptr;        // [nv] all ranks
  uint32_t* ones_local = nullptr;  // [nv] this rank
  uint32_t* ones_stage = nullptr;  // [R][nv] (in-process shards)
  bool gen_ok = false;     // Philox generations run as one persistent kernel (gom_gen.cu)
  bool gen_lean = false;   // ... with one warp per (set, population word)
  int gen_grid = 0;
  long long* gen_dfit = nullptr;
  unsigned long long* gen_dh = nullptr;
  unsigned long long* gen_cnt = nullptr;
  unsigned int* gen_bar = nullptr;
  int sms = 148;
  uint32_t mode = GOMIX_MODE_PHILOX, flags = 0;
  int32_t pop_id = 1;
  int epi_mode = 0;  // 0 exact atomics, 1 float partials, 2 ordered
  bool record = false;
  uint64_t seed = 1;

  std::vector<void*> allocs;
  uint32_t* pool = nullptr;  // [R][nv][Wp]: every rank's rows (R == 1: the population)
  uint32_t* pop = nullptr;   // this rank's slot of the pool
  double* fit_all = nullptr;  // [n_global], this rank's slice at rank*n
  unsigned long long* h1_all = nullptr;
  unsigned long long* h2_all = nullptr;
  unsigned long long* rank_cnt = nullptr;  // [R][steps, calls]
  double* fit = nullptr;
  long long* dfit = nullptr;  // fixed-point fitness deltas of the current group
  double fix_scale = 1.0;     // 1 (integer weights) or 2^S (float weights), see setup
  unsigned long long* h1 = nullptr;  // per-solution Zobrist hashes
  unsigned long long* h2 = nullptr;
  unsigned long long* dh1 = nullptr;
  unsigned long long* dh2 = nullptr;
  uint32_t* ever = nullptr;  // per-row elitist snapshot version
  uint32_t* elit = nullptr;
  DevCtl* ctl = nullptr;
  DevCtl* h_ctl = nullptr;  // pinned
  BeginArgs* d_begin = nullptr;  // per-call criteria read by the graph's begin kernel: the device
  BeginArgs* h_begin = nullptr;  // view of h_begin, mapped pinned host memory read in place
  static constexpr uint64_t kImprInline = 64;  // improvements copied back with every read_ctl
  static constexpr size_t kCtlBytes = (sizeof(DevCtl) + 63) / 64 * 64;  // control block, then the log
  ImprRec* h_impr = nullptr;                   // pinned [kImprInline], right after *h_ctl
  DevCtl* d_hctl = nullptr;                    // device view of h_ctl (mapped)
  volatile unsigned long long* h_seq = nullptr;  // publish sequence, after the inline log
  unsigned long long pub_seq = 0;
  unsigned long long* gsteps = nullptr;
  unsigned long long* gcalls = nullptr;
  ImprRec* impr = nullptr;  // right after *ctl
  uint64_t impr_cap = 0;
  int32_t* tape = nullptr;
  int32_t* h_tape_pinned = nullptr;
  // forced improvement (GOMIX_FLAG_FORCED_IMPROVEMENT / gomix_gpu_forced_improvement, gom_fi.cu)
  bool fi_on = false;
  double* fi_fit_start = nullptr;
  unsigned long long* fi_h1s = nullptr;
  unsigned long long* fi_h2s = nullptr;
  int32_t* fi_stag = nullptr;
  uint8_t* fi_flag = nullptr;
  double* fi_fit0 = nullptr;
  uint32_t* fi_mask = nullptr;
  int32_t* rec_donor = nullptr;
  double* rec_delta = nullptr;
  uint8_t* rec_present = nullptr;
  uint8_t* rec_accept = nullptr;
  uint64_t max_group = 0;
  uint8_t* d_bytes = nullptr;  // n x nv genotype staging for host transfers
  uint32_t* d_order = nullptr;
  GroupDesc* d_groups = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  uint64_t graph_launches = 0;
  static constexpr int kGraphAfter = 4;  // generations issued directly before the graph is captured
  // Generations of large groups go launch by launch: every launch is
  // programmatic, so the next generation's begin kernel fetches its criteria
  // and the first group's CTAs become resident while this generation's last
  // launch drains — across graph launches nothing overlaps (C3: 55.9 vs
  // 57.5 us per generation).  Small groups, where the host's launch cost
  // would show, keep the captured graph.  GOMIX_GRAPH=0/1 forces either.
  static constexpr uint64_t kDirectPairs = 1ull << 22;  // solution-set pairs per launch
  bool use_graph() const {
    static const int force = [] {
      const char* e = std::getenv("GOMIX_GRAPH");
      return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    if (force >= 0) return force == 1;
    return max_group * n < kDirectPairs;
  }
  int graph_warm = 0;

  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ReplayStream rng{1};
  int64_t generation = 0;
  bool initialized = false;
  double elit_fit = 0.0;
  bool ctl_stale = false;  // a device-side IMS offer may have changed the elitist since read_ctl()
  std::vector<uint32_t> h_pop;
  std::vector<uint64_t> perm, perm_touched;  // replay donor scans (draw_replay_tape)
  int64_t last_group = -1;
  uint64_t launches = 0;
  std::vector<cudaEvent_t> ev_free;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending;

  ~gomix_gpu_engine() {
    if (stream) cudaStreamSynchronize(stream);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (auto& pr : ev_pending) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    for (auto e : ev_free) cudaEventDestroy(e);
    cudaDeviceSynchronize();
    for (void* p : peer_opened) cudaIpcCloseMemHandle(p);
    if (xblock) cudaFree(xblock);
    cached_free_all(allocs);
    if (h_ctl) cudaFreeHost(h_ctl);
    if (h_begin) cudaFreeHost(h_begin);
    if (h_tape_pinned) cudaFreeHost(h_tape_pinned);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  bool exact() const { return P->exact; }

  bool better(double a, double b) const {
    if (exact()) return a > b;
    return a - b > 1e-9 * std::max({1.0, std::fabs(a), std::fabs(b)});
  }

  void setup(const gomix_engine_config& cfg) {
    n_global = cfg.population_size;
    if (n_global == 0) invalid("engine: population must be non-empty");
    if (cfg.mode != GOMIX_MODE_REPLAY && cfg.mode != GOMIX_MODE_PHILOX) invalid("engine: unknown mode");
    R = cfg.world_size > 1 ? (uint32_t)cfg.world_size : 1u;
    rank = R > 1 ? (uint32_t)cfg.rank : 0u;
    if (R > 1) {
      if (cfg.rank < 0 || (uint32_t)cfg.rank >= R) invalid("engine: rank out of range");
      if (cfg.mode != GOMIX_MODE_PHILOX) invalid("engine: sharded populations need GOMIX_MODE_PHILOX");
      if (n_global % R) invalid("engine: population size must be divisible by world_size");
      if (cfg.flags & GOMIX_FLAG_RECORD_BATCH) invalid("engine: batch recording is single-GPU only");
    }
    n = n_global / R;
    mode = cfg.mode;
    flags = cfg.flags;
    seed = cfg.seed;
    pop_id = cfg.population_id ? cfg.population_id : 1;
    rng = ReplayStream(seed);
    W = (uint32_t)((n + 31) / 32);
    GOMIX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device));
    if (W <= 8) {
      Wp = next_pow2(W);
      // few sets per group (small instances / big sets): one word per warp and
      // Wp warps per set, for parallelism; otherwise a warp per set with every
      // word in registers.
      const uint64_t avg_group = (P->m + P->k - 1) / P->k;
      if (Wp > 1 && avg_group * Wp <= (uint64_t)sms * 32) {
        wpt = 1;
        tw = Wp;
        block = 32 * tw;  // one team per CTA: the whole group fits in one wave
      } else {
        wpt = Wp;
        tw = 1;
        block = 256;
      }
    } else if (W <= 32) {
      Wp = next_pow2(W);
      wpt = 4;
      tw = Wp / 4;
      block = 32 * tw;
    } else if (W <= 128) {
      Wp = next_pow2(W);
      wpt = 8;
      tw = Wp / 8;
      block = 32 * tw;
    } else {
      invalid("engine: population sizes above 4096 are not supported");
    }
    teams = block / 32 / tw;
    if (tw > 1 && teams != 1) invalid("engine: internal team layout error");
    if (!P->univariate) {
      // patterns (64-bit per pool member), F pool rows, own donor rows, own new
      // rows, Zobrist keys of F
      const uint64_t RW = (uint64_t)R * Wp;
      stage_words = (uint32_t)(64 * RW + P->max_f * RW + 2 * P->max_f * Wp + 1 + 4 * P->max_f);
      stage_words += stage_words & 1u;  // keep the next team's patterns 8-byte aligned
    }
    const size_t stage = (size_t)teams * stage_words * 4;
    const size_t red = teams > 1 ? (size_t)teams * Wp * 32 * 24 : 0;  // fitness + 2 hash deltas
    smem = std::max(stage, red);
    if (smem > 227 * 1024) invalid("engine: set size x population too large for shared-memory staging");
    record = (flags & GOMIX_FLAG_RECORD_BATCH) != 0;
    // Float fitness deltas are summed as fixed-point integers: each delta is
    // rounded to a multiple of 2^-S before any addition, so the sums are
    // order-free (deterministic on any grid) and exact in int64 as long as a
    // group's total stays below 2^62: |sum| <= 2 * sum|w| bounds it, which
    // fixes S.  Resolution 2^-S per accepted delta (C4: S = 44, 6e-14).
    if (!P->exact) {
      const int e = (int)std::ceil(std::log2(2.0 * P->sum_abs_w + 1.0));
      fix_scale = std::ldexp(1.0, std::max(0, std::min(60, 62 - e)));
    }
    const bool ordered = !P->exact && (mode == GOMIX_MODE_REPLAY || (flags & GOMIX_FLAG_ORDERED_FLOAT));
    epi_mode = P->exact ? 0 : (ordered ? 2 : 1);

    GOMIX_CUDA(cudaSetDevice(P->device));
    GOMIX_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    own_stream = true;
    if (R > 1 && cfg.nccl_unique_id) {  // one process per GPU: collective communicator
      const NcclApi& api = nccl_or_throw();
      ncclUniqueId id;
      std::memcpy(&id, cfg.nccl_unique_id, sizeof(id));
      nccl = std::make_unique<NcclComm>();
      nccl_check(api.CommInitRank(&nccl->comm, (int)R, id, (int)rank), "ncclCommInitRank");
    }
    const int per_sm = gom_max_blocks_per_sm(P->univariate, P->i32, (int)wpt, tw > 1, (int)block, smem);
    if (per_sm < 1) invalid("engine: GOM kernel does not fit on an SM with this configuration");
    grid_cap = per_sm * sms;
    // The bit-sliced univariate kernels draw no donor: for F = {v} every
    // member that differs on F holds !x_v, so the step is the same whatever
    // donor the reference's scan picks (engine_serial.hpp:30-46) and only its
    // presence (some member differs) matters.  They therefore serve REPLAY
    // as well: the host walks the reference's RngStream through the same
    // donor scans to stay in step (walk_replay_rng) and the kernel computes
    // presence from the group-start row.
    if (P->univariate && P->i32 && !(flags & GOMIX_FLAG_RECORD_BATCH) && !(flags & GOMIX_FLAG_LANE_PER_SOLUTION)) {
      univ_planes = univ_sliced_planes(P->max_abs_row);
      // rows wider than 4 words run in 4-word chunks, one per CTA; their
      // presence test reads per-row counts of 1s taken at generation start,
      // valid when every variable sits in one set (a row then changes only
      // in its own group)
      univ_tt = P->urec != nullptr && (Wp <= 4 || P->var_once) && !(flags & GOMIX_FLAG_NO_TRUTH_TABLE);
      tt_chunks = univ_tt && Wp > 4 ? Wp / 4 : 1;
      if (univ_planes) univ_grid_cap = univ_sliced_max_blocks_per_sm(univ_planes, (int)Wp, univ_tt) * sms;
      if (univ_grid_cap < 1) univ_planes = 0;
    }
    // float weights on a univariate FOS (BASELINE C4): one warp per set with
    // its record / weights staged (gom_univ_f64.cu); the lane-per-solution
    // group kernel stays the A/B reference (GOMIX_FLAG_LANE_PER_SOLUTION)
    if (P->univariate && !P->i32 && P->uvr && mode == GOMIX_MODE_PHILOX && R == 1 && epi_mode != 2 && !record &&
        Wp <= 4 && P->max_fp <= (uint64_t)univ_f64_max_degree() && !(flags & GOMIX_FLAG_LANE_PER_SOLUTION)) {
      f64_grid_cap = univ_f64_max_blocks_per_sm((int)Wp) * sms;
      univ_f64 = f64_grid_cap >= 1;
    }
    for (uint64_t c = 0; c < P->k; ++c)
      max_group = std::max(max_group, P->group_off[c + 1] - P->group_off[c]);
    if (mode == GOMIX_MODE_PHILOX && P->i32 && !P->univariate && R == 1 && n <= kGenMaxN && P->k <= kGenMaxK &&
        !(flags & GOMIX_FLAG_RECORD_BATCH) && !(flags & GOMIX_FLAG_PER_GROUP_KERNELS)) {
      // lean layout (one warp per set and population word, gom_lean.cuh) for sets of <= 32 variables
      gen_lean = P->max_f <= 32 && !(flags & GOMIX_FLAG_LANE_PER_SOLUTION);
      const int gblock = gen_lean ? 256 : (int)block;
      const size_t gsmem = gen_lean ? (size_t)gen_lean_smem() : smem;
      const int per = gen_kernel_max_blocks(gen_lean ? (int)Wp : (int)wpt, tw > 1, gblock, gsmem, gen_lean);
      const uint64_t want = gen_lean ? std::max<uint64_t>(1, (max_group * Wp + 7) / 8)
                                     : std::max<uint64_t>(1, (max_group + teams - 1) / teams);
      if (per >= 1) {
        gen_grid = (int)std::min<uint64_t>(want, (uint64_t)per * sms);
        // lean units: whole waves of CTAs per SM (every SM holds the same
        // number of CTAs; units spread warp-major over them)
        if (gen_lean && want > (uint64_t)sms)
          gen_grid = (int)std::min<uint64_t>((uint64_t)sms * ((want + sms - 1) / sms), (uint64_t)per * sms);
        gen_ok = true;
        gen_dfit = dev_alloc<long long>(allocs, 3 * n * kAccStride);
        gen_dh = dev_alloc<unsigned long long>(allocs, 6 * n * kAccStride);
        gen_cnt = dev_alloc<unsigned long long>(allocs, 6);
        gen_bar = dev_alloc<unsigned int>(allocs, 2048);  // two-level barrier (gom_gen.cu)
        GOMIX_CUDA(cudaMemset(gen_dfit, 0, 3 * n * kAccStride * 8));
        GOMIX_CUDA(cudaMemset(gen_dh, 0, 6 * n * kAccStride * 8));
        GOMIX_CUDA(cudaMemset(gen_cnt, 0, 6 * 8));
        GOMIX_CUDA(cudaMemset(gen_bar, 0, 2048 * 4));
      }
    }

    const uint64_t nv = P->nv;
    pool = dev_alloc<uint32_t>(allocs, (uint64_t)R * nv * Wp);
    pop = pool + (uint64_t)rank * nv * Wp;
    fit_all = dev_alloc<double>(allocs, n_global);
    h1_all = dev_alloc<unsigned long long>(allocs, n_global);
    h2_all = dev_alloc<unsigned long long>(allocs, n_global);
    rank_cnt = dev_alloc<unsigned long long>(allocs, 2 * (uint64_t)R);
    fit = fit_all + (uint64_t)rank * n;
    h1 = h1_all + (uint64_t)rank * n;
    h2 = h2_all + (uint64_t)rank * n;
    dfit = dev_alloc<long long>(allocs, n);
    dh1 = dev_alloc<unsigned long long>(allocs, n);
    dh2 = dev_alloc<unsigned long long>(allocs, n);
    ever = dev_alloc<uint32_t>(allocs, nv);
    elit = dev_alloc<uint32_t>(allocs, (nv + 31) / 32);
    impr_cap = std::min<uint64_t>(std::max<uint64_t>(4096, n_global * (P->k + 1)), 1ull << 22);
    {  // control block + improvement log in one block (read back with one copy)
      char* blk = dev_alloc<char>(allocs, kCtlBytes + impr_cap * sizeof(ImprRec));
      ctl = reinterpret_cast<DevCtl*>(blk);
      impr = reinterpret_cast<ImprRec*>(blk + kCtlBytes);
    }
    gsteps = dev_alloc<unsigned long long>(allocs, P->k);
    gcalls = dev_alloc<unsigned long long>(allocs, P->k);
    fi_on = (flags & GOMIX_FLAG_FORCED_IMPROVEMENT) != 0;
    if (fi_on && R > 1) invalid("engine: forced improvement needs a single-GPU engine");
    d_order = dev_alloc<uint32_t>(allocs, P->k);
    d_groups = dev_alloc<GroupDesc>(allocs, P->k);
    {
      std::vector<GroupDesc> gd(P->k);
      for (uint64_t c = 0; c < P->k; ++c)
        gd[c] = GroupDesc{(uint32_t)P->group_off[c], (uint32_t)(P->group_off[c + 1] - P->group_off[c])};
      GOMIX_CUDA(cudaMemcpy(d_groups, gd.data(), P->k * sizeof(GroupDesc), cudaMemcpyHostToDevice));
    }
    prepare_gom(P->univariate, P->i32, (int)wpt, tw > 1, smem);
    if (record || epi_mode == 2) {
      rec_donor = dev_alloc<int32_t>(allocs, max_group * n);
      rec_delta = dev_alloc<double>(allocs, max_group * n);
      rec_present = dev_alloc<uint8_t>(allocs, max_group * n);
      rec_accept = dev_alloc<uint8_t>(allocs, max_group * n);
    }
    lite = R > 1 && P->univariate && P->var_once && mode == GOMIX_MODE_PHILOX;
    if ((flags & GOMIX_FLAG_PEER_TRANSPORT) && R > 1 && !lite)
      invalid("engine: the peer transport needs a univariate FOS with every variable in one set (use NCCL)");
    if (tt_chunks > 1 && R > 1 && !lite) invalid("engine: internal: chunked rows need the sharded row counts");
    if (lite || tt_chunks > 1) ones = dev_alloc<uint32_t>(allocs, nv);
    tail_ctr = dev_alloc<unsigned int>(allocs, tt_chunks * kTailCounters * kTailStride);
    GOMIX_CUDA(cudaMemset(tail_ctr, 0, tt_chunks * kTailCounters * kTailStride * sizeof(unsigned int)));
    if (tt_chunks > 1) {
      chunk_done = dev_alloc<unsigned int>(allocs, tt_chunks);
      word_max = dev_alloc<double>(allocs, Wp);
      GOMIX_CUDA(cudaMemset(chunk_done, 0, tt_chunks * sizeof(unsigned int)));
    }
    if (lite) {
      ones_local = dev_alloc<uint32_t>(allocs, nv);
      if (!cfg.nccl_unique_id) ones_stage = dev_alloc<uint32_t>(allocs, (uint64_t)R * nv);
    }
    // mapped: the synchronous generation path has the device write it in place (publish_ctl)
    GOMIX_CUDA(cudaHostAlloc(&h_ctl, kCtlBytes + kImprInline * sizeof(ImprRec) + 64, cudaHostAllocMapped));
    GOMIX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hctl), h_ctl, 0));
    h_seq = reinterpret_cast<volatile unsigned long long*>(reinterpret_cast<char*>(h_ctl) + kCtlBytes +
                                                          kImprInline * sizeof(ImprRec));
    *h_seq = 0;
    h_impr = reinterpret_cast<ImprRec*>(reinterpret_cast<char*>(h_ctl) + kCtlBytes);
    GOMIX_CUDA(cudaHostAlloc(&h_begin, sizeof(BeginArgs), cudaHostAllocMapped));
    GOMIX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_begin), h_begin, 0));
    *h_begin = make_begin(nullptr);
    std::memset(h_ctl, 0, sizeof(DevCtl));
    h_ctl->elit_src = -1;
    h_ctl->exact = P->exact;
    h_ctl->q = (double)P->q;
    GOMIX_CUDA(cudaMemcpy(ctl, h_ctl, sizeof(DevCtl), cudaMemcpyHostToDevice));
    // the log entries read_ctl copies back with the control block (only the
    // first n_impr are meaningful; defined bytes keep initcheck quiet)
    GOMIX_CUDA(cudaMemset(reinterpret_cast<char*>(ctl) + sizeof(DevCtl), 0,
                          kCtlBytes - sizeof(DevCtl) + std::min(kImprInline, impr_cap) * sizeof(ImprRec)));
    GOMIX_CUDA(cudaMemset(pool, 0, (uint64_t)R * nv * Wp * 4));
    GOMIX_CUDA(cudaMemset(gsteps, 0, P->k * 8));
    GOMIX_CUDA(cudaMemset(rank_cnt, 0, 2 * (uint64_t)R * 8));  // gathered at init before any group ran
    GOMIX_CUDA(cudaMemset(gcalls, 0, P->k * 8));
    GOMIX_CUDA(cudaMemset(dfit, 0, n * 8));
    GOMIX_CUDA(cudaMemset(dh1, 0, n * 8));
    GOMIX_CUDA(cudaMemset(dh2, 0, n * 8));
    GOMIX_CUDA(cudaMemset(ever, 0, nv * 4));
    GOMIX_CUDA(cudaMemset(elit, 0, ((nv + 31) / 32) * 4));
    // the memsets above run on the legacy stream, which the engine's
    // non-blocking stream does not wait for (recycled blocks hold old data)
    GOMIX_CUDA(cudaDeviceSynchronize());
  }

  uint8_t* staging() {
    if (!d_bytes) d_bytes = dev_alloc<uint8_t>(allocs, n * P->nv);
    return d_bytes;
  }

  // ---- per-call control ------------------------------------------------------
  BeginArgs make_begin(const gomix_stop_criteria* stop) const {
    BeginArgs b{};
    b.ctl = ctl;
    b.has_budget = stop && stop->has_max_evaluations;
    b.has_target = stop && stop->has_target;
    b.exact = P->exact;
    b.max_evals = stop ? stop->max_evaluations : 0.0;
    b.q = (double)P->q;
    b.target = stop ? stop->target_fitness : 0.0;
    b.calls_before = stop ? stop->evaluator_calls_before : 0;
    b.gen = (uint32_t)generation;
    return b;
  }

  void begin_call(const gomix_stop_criteria* stop) {
    BeginArgs b;
    b.ctl = ctl;
    b.has_budget = stop && stop->has_max_evaluations;
    b.has_target = stop && stop->has_target;
    b.exact = P->exact;
    b.max_evals = stop ? stop->max_evaluations : 0.0;
    b.q = (double)P->q;
    b.target = stop ? stop->target_fitness : 0.0;
    b.calls_before = stop ? stop->evaluator_calls_before : 0;
    b.gen = (uint32_t)generation;
    launch_begin(b, stream);
    ++launches;
  }

  // A whole Philox generation as one persistent kernel (gom_gen.cu).
  void launch_generation_persistent() {
    GomArgs a = gom_args(0, max_group, false, -1);
    a.epi = epi_args(0, 0, 0);
    GenArgs ga{*h_begin, (uint32_t)P->k, d_order, gen_dfit, gen_dh, gen_cnt, gen_bar};
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (flags & GOMIX_FLAG_TIME_KERNELS) {
      e0 = take_event();
      e1 = take_event();
      GOMIX_CUDA(cudaEventRecord(e0, stream));
    }
    launch_generation_kernel(a, ga, gen_lean ? (int)Wp : (int)wpt, tw > 1, gen_grid, gen_lean ? 256 : (int)block,
                             gen_lean ? (size_t)gen_lean_smem() : smem, stream, gen_lean);
    ++launches;
    if (e1) {
      GOMIX_CUDA(cudaEventRecord(e1, stream));
      ev_pending.push_back({e0, e1});
    }
  }

  // One CUDA graph per engine for a whole Philox generation: the order
  // kernel, then k GOM launches that find their group through
  // the device-side order.  Replaces ~2k launches by one graph launch.
  void launch_generation_graph() {
    // The first generations of an engine (IMS creates short-lived ones) are
    // issued launch by launch — the same kernels in the same order as the
    // captured graph — so a population that reaches the target early never
    // pays the capture and instantiation.
    if (!graph_exec && (graph_warm < kGraphAfter || !use_graph())) {
      ++graph_warm;
      count_rows(stream);
      OrderArgs o{ctl, d_order, (uint32_t)P->k, seed};
      launch_order(d_begin, o, stream);
      for (uint64_t slot = 0; slot < P->k; ++slot) launch_group(0, false, (int32_t)slot, stream);
      ++launches;
      return;
    }
    if (!graph_exec) {
      cudaStream_t cap = nullptr;
      GOMIX_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
      GOMIX_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      const uint64_t saved = launches;
      count_rows(cap);
      OrderArgs o{ctl, d_order, (uint32_t)P->k, seed};
      launch_order(d_begin, o, cap);
      for (uint64_t slot = 0; slot < P->k; ++slot) launch_group(0, false, (int32_t)slot, cap);
      graph_launches = launches - saved + 1;
      launches = saved;
      cudaGraph_t g = nullptr;
      GOMIX_CUDA(cudaStreamEndCapture(cap, &g));
      GOMIX_CUDA(cudaGraphInstantiate(&graph_exec, g, 0));
      GOMIX_CUDA(cudaGraphDestroy(g));
      GOMIX_CUDA(cudaStreamDestroy(cap));
    }
    GOMIX_CUDA(cudaGraphLaunch(graph_exec, stream));
    launches += graph_launches;
  }

  // Chunked truth-table rows (n > 128): every row's count of 1s at
  // generation start, the presence test of its set (the FOS is univariate and
  // variable-once: a row changes only in its own group).
  void count_rows(cudaStream_t st) {
    if (R > 1 && peer_on) {  // sharded over peer memory: every rank's presence maps (graph path)
      launch_presence(d_peer, ctl, pop, P->nv, Wp, (uint32_t)n, (uint32_t)n_global, ones, st);
      launches += 2;
      return;
    }
    if (tt_chunks <= 1 || R > 1) return;  // sharded NCCL runs count (and all-reduce) in run_generation_sharded
    launch_count_ones(pop, P->nv, Wp, ones, st);
    ++launches;
  }

  // Stage this call's stop criteria for the graph's begin kernel.  The pinned
  // staging buffer is only rewritten when no earlier copy from it can be
  // pending (sync calls wait first; async calls always stage "no criteria").
  void stage_criteria(const gomix_stop_criteria* stop, bool sync_first) {
    if (sync_first) GOMIX_CUDA(cudaStreamSynchronize(stream));
    // the begin kernel reads the criteria in place over the bus: no copy to
    // queue.  Async calls stage "no criteria" every time, so a generation
    // still queued reads the same values (the generation number is the
    // device's own counter, begin_generation_kernel)
    BeginArgs b = make_begin(stop);
    if (!sync_first) b.gen = 0;  // (unused by the graph kernels; keeps queued reads byte-identical)
    *h_begin = b;
    std::atomic_thread_fence(std::memory_order_release);
  }

  // Synchronous read-back after a generation: the device writes the control
  // block and inline log into h_ctl (mapped) and then bumps the sequence;
  // the host spins on it (a device-to-host copy plus a stream synchronise
  // cost microseconds per generation).  A failed stream still surfaces: the
  // spin checks the stream every few thousand polls.
  void read_ctl_published() {
    const size_t bytes = kCtlBytes + std::min(kImprInline, impr_cap) * sizeof(ImprRec);
    launch_publish_ctl(ctl, d_hctl, (bytes + 15) / 16 * 16,
                       const_cast<unsigned long long*>(reinterpret_cast<volatile unsigned long long*>(
                           reinterpret_cast<char*>(d_hctl) + kCtlBytes + kImprInline * sizeof(ImprRec))),
                       ++pub_seq, stream);
    ++launches;
    for (uint64_t spins = 1; *h_seq < pub_seq; ++spins) {
      if ((spins & 4095u) == 0) {
        const cudaError_t e = cudaStreamQuery(stream);
        if (e != cudaSuccess && e != cudaErrorNotReady) GOMIX_CUDA(e);
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    ctl_stale = false;
  }

  void read_ctl() {
    // one copy: the control block and the first log entries behind it
    GOMIX_CUDA(cudaMemcpyAsync(h_ctl, ctl, kCtlBytes + std::min(kImprInline, impr_cap) * sizeof(ImprRec),
                               cudaMemcpyDeviceToHost, stream));
    GOMIX_CUDA(cudaStreamSynchronize(stream));
    ctl_stale = false;
  }

  // host copy of the elitist fitness, refreshed after device-side IMS offers
  double host_elit_fit() {
    if (ctl_stale) {
      read_ctl();
      elit_fit = h_ctl->elit_fit;
    }
    return elit_fit;
  }

  void fill_stats(gomix_run_stats* out) {
    elit_fit = h_ctl->elit_fit;
    if (!out) return;
    out->groups_run = h_ctl->groups_run;
    out->steps = h_ctl->run_steps;
    out->evaluator_calls = h_ctl->run_calls;
    out->stopped = h_ctl->stop;
    out->stop_reason = h_ctl->stop_reason;
    out->improvements = h_ctl->n_impr;
    out->elitist_fitness = h_ctl->elit_fit;
  }

  SnapArgs snap_args() const {
    SnapArgs r;
    r.pop = pop;
    r.pool = pool;
    r.elit = elit;
    r.ever = ever;
    r.ctl = ctl;
    r.h1 = h1;
    r.h2 = h2;
    r.nv = P->nv;
    r.n = (uint32_t)n;
    r.Wp = Wp;
    return r;
  }

  EpiArgs epi_args(uint64_t group, uint32_t G, uint32_t nparts) const {
    EpiArgs e;
    e.fit = fit;
    e.dfit = dfit;
    e.fix_inv = 1.0 / fix_scale;
    e.h1 = h1;
    e.h2 = h2;
    e.dh1 = dh1;
    e.dh2 = dh2;
    e.rec_delta = rec_delta;
    e.rec_accept = rec_accept;
    e.ctl = ctl;
    e.gsteps = gsteps;
    e.gcalls = gcalls;
    e.impr = impr;
    e.impr_cap = impr_cap;
    e.fit_all = fit_all;
    e.h1_all = h1_all;
    e.h2_all = h2_all;
    e.rank_cnt = rank_cnt;
    e.n_global = (uint32_t)n_global;
    e.R = R;
    e.rank = rank;
    e.peer = peer_on ? d_peer : nullptr;
    e.word_max = nullptr;  // set by the chunked truth-table kernel itself
    e.n = (uint32_t)n;
    e.G = G;
    e.nparts = nparts;
    e.group = (uint32_t)group;
    e.mode = epi_mode;
    return e;
  }

  // ---- one batched group step -----------------------------------------------
  GomArgs gom_args(uint64_t g0, uint64_t G, bool with_tape, int32_t slot) {
    GomArgs a;
    a.row_ptr = P->row_ptr;
    a.col = P->col;
    a.w = P->w;
    a.wi = P->wi;
    a.set_off = P->set_off;
    a.set_vars = P->set_vars;
    a.fp_off = P->fp_off;
    a.fp = P->fp;
    a.gsets = P->gsets + g0;
    a.gvars = P->gvars ? P->gvars + g0 : nullptr;
    a.urec = P->urec ? P->urec + 2 * g0 : nullptr;
    a.ukey = P->ukey ? P->ukey + g0 : nullptr;
    a.uvr = P->uvr ? P->uvr + g0 : nullptr;
    a.chunk_done = chunk_done;
    a.tail = tail_ctr;
    a.tail_per_chunk = tt_chunks > 1;
    a.word_max = word_max;
    a.gmeta = P->gmeta ? P->gmeta + g0 : nullptr;
    a.wbits = P->wbits;
    a.G = (uint32_t)G;
    a.pop = pop;
    a.fit = fit;
    a.h1 = h1;
    a.h2 = h2;
    a.ever = ever;
    a.elit = elit;
    a.dfit = dfit;
    a.fix_scale = fix_scale;
    a.dh1 = dh1;
    a.dh2 = dh2;
    a.ctl = ctl;
    a.tape = with_tape ? tape : nullptr;
    const bool rec = record || epi_mode == 2;
    a.rec_donor = rec ? rec_donor : nullptr;
    a.rec_delta = rec ? rec_delta : nullptr;
    a.rec_present = rec ? rec_present : nullptr;
    a.rec_accept = rec ? rec_accept : nullptr;
    a.n = (uint32_t)n;
    a.Wp = Wp;
    a.pool = pool;
    a.ones = (lite || tt_chunks > 1) ? ones : nullptr;
    a.nv = P->nv;
    a.R = R;
    a.rank = rank;
    a.n_global = (uint32_t)n_global;
    a.team_warps = tw;
    a.stage_words = stage_words;
    a.exact = P->exact;
    a.generation = (uint32_t)generation;
    a.seed = seed;
    a.slot = slot;
    a.exp_flags = g_exp_flags.load(std::memory_order_relaxed);
    a.order = d_order;
    a.groups = d_groups;
    return a;
  }

  void launch_group(uint64_t group, bool with_tape, int32_t slot = -1, cudaStream_t st = nullptr) {
    if (!st) st = stream;
    const uint64_t g0 = slot >= 0 ? 0 : P->group_off[group];
    const uint64_t G = slot >= 0 ? max_group : P->group_off[group + 1] - g0;
    GomArgs a = gom_args(g0, G, with_tape, slot);
    const uint64_t want = (G + teams - 1) / teams;
    const int grid = (int)std::min<uint64_t>(want, (uint64_t)grid_cap);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if ((flags & GOMIX_FLAG_TIME_KERNELS) && slot < 0) {
      e0 = take_event();
      e1 = take_event();
      GOMIX_CUDA(cudaEventRecord(e0, st));
    }
    if (univ_f64 && !with_tape) {
      const uint64_t per = (uint64_t)univ_f64_sets_per_cta();
      const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>((G + per - 1) / per, (uint64_t)f64_grid_cap));
      a.epi = epi_args(group, (uint32_t)G, (uint32_t)g);
      launch_univ_f64(a, (int)Wp, g, st, slot >= 0);  // graph path: PDL (the begin kernel or the previous group)
    } else if (univ_planes && !with_tape) {
      const uint64_t per = (uint64_t)univ_sliced_sets_per_cta();
      // chunked rows: tt_chunks CTAs per set range, one per chunk
      // chunked rows: every chunk's CTAs split its sets; the grid stays a
      // multiple of the SM count when the work fills it (chunks then differ
      // by at most one CTA), and covers every chunk at least once
      const uint64_t want = tt_chunks * ((G + per - 1) / per);
      const int g = (int)std::max<uint64_t>(tt_chunks, std::min<uint64_t>(std::max<uint64_t>(1, want),
                                                                          (uint64_t)univ_grid_cap));
      a.epi = epi_args(group, (uint32_t)G, (uint32_t)g);
      // graph path: programmatic dependent launches (the first group after
      // the begin kernel, later groups after the previous group)
      // (truth-table kernel only: it waits on griddepcontrol before reading
      // the previous group's results)
      launch_univ_sliced(a, univ_planes, (int)Wp, univ_tt, g, st, univ_tt && slot >= 0);
    } else {
      a.epi = epi_args(group, (uint32_t)G, (uint32_t)grid);
      launch_gom(a, P->univariate, P->i32, (int)wpt, tw > 1, grid, (int)block, smem, st);
    }
    ++launches;
    if (e1) {
      GOMIX_CUDA(cudaEventRecord(e1, st));
      ev_pending.push_back({e0, e1});
    }
    if (slot < 0) last_group = (int64_t)group;
  }

  cudaEvent_t take_event() {
    if (!ev_free.empty()) {
      cudaEvent_t e = ev_free.back();
      ev_free.pop_back();
      return e;
    }
    cudaEvent_t e;
    GOMIX_CUDA(cudaEventCreate(&e));
    return e;
  }

  // ---- replay: the reference's sequential donor draws ----------------------
  // insert_donor_genes (engine_parallel.hpp:110-120) + select_donor
  // (engine_serial.hpp:30-46) against the group-start population.
  // donor tapes (replay mode / explicit donors) are allocated on first use:
  // max_group * n entries is a gigabyte at 10^6 vertices and n = 512
  void ensure_tape(bool host = true) {
    if (!tape) tape = dev_alloc<int32_t>(allocs, max_group * n);
    if (host && !h_tape_pinned)
      GOMIX_CUDA(cudaMallocHost(&h_tape_pinned, std::max<uint64_t>(1, max_group * n) * sizeof(int32_t)));
  }

  // ---- forced improvement (gom_fi.cu) ----------------------------------------
  void ensure_fi() {
    if (fi_fit_start) return;
    fi_fit_start = dev_alloc<double>(allocs, n);
    fi_h1s = dev_alloc<unsigned long long>(allocs, n);
    fi_h2s = dev_alloc<unsigned long long>(allocs, n);
    fi_stag = dev_alloc<int32_t>(allocs, n);
    fi_flag = dev_alloc<uint8_t>(allocs, n);
    fi_fit0 = dev_alloc<double>(allocs, n);
    fi_mask = dev_alloc<uint32_t>(allocs, Wp);
    GOMIX_CUDA(cudaMemsetAsync(fi_stag, 0, n * sizeof(int32_t), stream));
    GOMIX_CUDA(cudaMemsetAsync(fi_flag, 0, n, stream));
  }

  FiArgs fi_args() {
    FiArgs a;
    a.pop = pop;
    a.fit = fit;
    a.h1 = h1;
    a.h2 = h2;
    a.fit_start = fi_fit_start;
    a.h1s = fi_h1s;
    a.h2s = fi_h2s;
    a.stag = fi_stag;
    a.flag = fi_flag;
    a.fit0 = fi_fit0;
    a.mask = fi_mask;
    a.ctl = ctl;
    a.gsets = P->gsets;
    a.set_off = P->set_off;
    a.set_vars = P->set_vars;
    a.nv = P->nv;
    a.n = (uint32_t)n;
    a.Wp = Wp;
    a.threshold = 1 + (int32_t)std::floor(std::log10((double)n));  // engine_serial.hpp:153-155
    return a;
  }

  // generation start (before its GOM groups)
  void fi_snapshot() {
    ensure_fi();
    launch_fi_snapshot(fi_args(), stream);
    ++launches;
  }

  // The pass itself: trigger (or given flags), then every colour group in
  // `order` as one batched GOM step with the elitist as donor, then the
  // elitist copies.  Runs after the generation's groups, on the same stream,
  // against the same control block (calls, stop criteria, elitist scan).
  void fi_pass(const uint8_t* given, const std::vector<uint64_t>& order, bool update_stag) {
    ensure_fi();
    ensure_tape(false);
    const FiArgs fa = fi_args();
    if (given) GOMIX_CUDA(cudaMemcpyAsync(fi_flag, given, n, cudaMemcpyHostToDevice, stream));
    launch_fi_flags(fa, given != nullptr, stream);
    ++launches;
    for (uint64_t gi : order) {
      const uint64_t g0 = P->group_off[gi], G = P->group_off[gi + 1] - g0;
      launch_fi_tape(fa, g0, G, tape, stream);
      launch_group(gi, true);
      ++launches;
    }
    launch_fi_finish(fa, update_stag, stream);
    launches += 3;
  }

  // the engine's own trigger after a generation, groups in a fresh order
  void fi_after_generation() {
    std::vector<uint64_t> order;
    rng.permutation(order, P->k);
    fi_pass(nullptr, order, true);
  }

  void forced_improvement(const uint8_t* flags_in, const uint32_t* group_order, const gomix_stop_criteria* stop,
                          gomix_run_stats* out) {
    if (!initialized) throw GomixError(GOMIX_E_STATE, "forced_improvement: population not initialised");
    if (R > 1) invalid("forced_improvement: single-GPU engines only");
    std::vector<uint64_t> order;
    if (group_order) {
      std::vector<uint8_t> seen(P->k, 0);
      for (uint64_t i = 0; i < P->k; ++i) {
        if (group_order[i] >= P->k || seen[group_order[i]]) invalid("forced_improvement: group_order is not a permutation");
        seen[group_order[i]] = 1;
        order.push_back(group_order[i]);
      }
    } else {
      rng.permutation(order, P->k);
    }
    if (!flags_in && !fi_fit_start) invalid("forced_improvement: no generation has set the trigger (pass flags)");
    begin_call(stop);
    fi_pass(flags_in, order, false);
    read_ctl();
    fill_stats(out);
  }

  // upload == false: only walk the stream (the bit-sliced univariate kernels
  // need no donors, see setup); the draws are the same either way.
  void draw_replay_tape(uint64_t group, bool upload = true) {
    if (upload) ensure_tape();
    const uint64_t nv = P->nv;
    h_pop.resize(nv * Wp);
    GOMIX_CUDA(cudaMemcpyAsync(h_pop.data(), pop, nv * Wp * 4, cudaMemcpyDeviceToHost, stream));
    GOMIX_CUDA(cudaStreamSynchronize(stream));
    const uint64_t g0 = P->group_off[group], G = P->group_off[group + 1] - g0;
    // perm is the identity between scans: each scan restores the entries it
    // swapped (a scan touches ~2 entries on average, not n)
    if (perm.size() != n) {
      perm.resize(n);
      for (uint64_t i = 0; i < n; ++i) perm[i] = i;
    }
    std::vector<uint64_t>& touched = perm_touched;
    auto bit = [&](uint32_t v, uint64_t s) { return (h_pop[(uint64_t)v * Wp + (s >> 5)] >> (s & 31)) & 1u; };
    for (uint64_t p = 0; p < G; ++p) {
      const uint64_t sid = P->group_sets[g0 + p];
      const uint32_t* vars = P->h_set_vars.data() + P->h_set_off[sid];
      const uint64_t f = P->h_set_off[sid + 1] - P->h_set_off[sid];
      for (uint64_t s = 0; s < n; ++s) {
        int32_t donor = -1;
        touched.clear();
        for (uint64_t i = 0; i < n && donor < 0; ++i) {
          const uint64_t j = i + rng.uniform_index(n - i);
          std::swap(perm[i], perm[j]);
          touched.push_back(i);
          touched.push_back(j);
          const uint64_t c = perm[i];
          for (uint64_t t = 0; t < f; ++t)
            if (bit(vars[t], c) != bit(vars[t], s)) {
              donor = (int32_t)c;
              break;
            }
        }
        for (uint64_t t : touched) perm[t] = t;
        if (upload) h_tape_pinned[p * n + s] = donor;
      }
    }
    if (upload) GOMIX_CUDA(cudaMemcpyAsync(tape, h_tape_pinned, G * n * 4, cudaMemcpyHostToDevice, stream));
  }

  void upload_tape(uint64_t group, const int32_t* donor_sp) {
    ensure_tape();
    const uint64_t g0 = P->group_off[group], G = P->group_off[group + 1] - g0;
    for (uint64_t s = 0; s < n; ++s)
      for (uint64_t p = 0; p < G; ++p) {
        const int32_t d = donor_sp[s * G + p];
        if (d >= (int64_t)n) invalid("run_group: donor index out of range");
        h_tape_pinned[p * n + s] = d < 0 ? -1 : d;
      }
    GOMIX_CUDA(cudaMemcpyAsync(tape, h_tape_pinned, G * n * 4, cudaMemcpyHostToDevice, stream));
  }

  // ---- peer transport -------------------------------------------------------
  // This rank's exchange block: plain cudaMalloc (pool memory cannot be
  // exported through a CUDA IPC handle), zeroed once; epochs start at 1.
  void peer_alloc() {
    if (R < 2 || !(flags & GOMIX_FLAG_PEER_TRANSPORT)) invalid("peer transport: needs world_size > 1 and GOMIX_FLAG_PEER_TRANSPORT");
    if (R > kMaxRanks) invalid("peer transport: at most 16 ranks");
    if (xblock) return;
    xbytes = peer_block_bytes(R, (uint32_t)n, (uint32_t)((P->nv + 31) / 32));
    GOMIX_CUDA(cudaSetDevice(P->device));
    GOMIX_CUDA(cudaMalloc(&xblock, xbytes));
    GOMIX_CUDA(cudaMemset(xblock, 0, xbytes));
    GOMIX_CUDA(cudaDeviceSynchronize());
  }

  // blocks[r]: rank r's block as mapped in this process (own = xblock)
  void peer_set_blocks(char* const* blocks) {
    PeerArgs h{};
    for (uint32_t r = 0; r < R; ++r) h.blocks[r] = r == rank ? xblock : blocks[r];
    h.R = R;
    h.rank = rank;
    h.n = (uint32_t)n;
    h.w32 = (uint32_t)((P->nv + 31) / 32);
    h.timeout_ns = 60ull * 1000000000ull;  // a rank that stopped calling: fault after a minute, never a hang
    if (!d_peer) d_peer = dev_alloc<PeerArgs>(allocs, 1);
    GOMIX_CUDA(cudaMemcpy(d_peer, &h, sizeof(PeerArgs), cudaMemcpyHostToDevice));
    peer_on = true;
  }

  void peer_export(uint8_t* handle) {
    peer_alloc();
    cudaIpcMemHandle_t h;
    GOMIX_CUDA(cudaIpcGetMemHandle(&h, xblock));
    static_assert(sizeof(cudaIpcMemHandle_t) == GOMIX_PEER_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
  }

  void peer_connect(const uint8_t* handles) {
    if (!xblock) invalid("peer_connect: export this rank's block first (gomix_gpu_peer_export)");
    if (initialized) throw GomixError(GOMIX_E_STATE, "peer_connect: call before init_population");
    GOMIX_CUDA(cudaSetDevice(P->device));
    std::vector<char*> blocks(R, nullptr);
    for (uint32_t r = 0; r < R; ++r) {
      if (r == rank) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + (size_t)r * GOMIX_PEER_HANDLE_BYTES, sizeof(h));
      void* p = nullptr;
      GOMIX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      peer_opened.push_back(p);
      blocks[r] = static_cast<char*>(p);
    }
    peer_set_blocks(blocks.data());
  }

  // ---- API operations ---------------------------------------------------------
  void init_population(const uint8_t* genotypes, const gomix_stop_criteria* stop,
                       gomix_run_stats* out) {
    if (initialized) throw GomixError(GOMIX_E_STATE, "init_population: already initialised");
    const uint64_t nv = P->nv;
    if (genotypes) {
      for (uint64_t i = 0; i < n * nv; ++i)
        if (genotypes[i] > 1) invalid("graybox: genotype value outside alphabet");
      uint8_t* d = staging();
      GOMIX_CUDA(cudaMemcpyAsync(d, genotypes, n * nv, cudaMemcpyHostToDevice, stream));
      launch_pack(d, pop, nv, (uint32_t)n, Wp, stream);
      ++launches;
    } else if (mode == GOMIX_MODE_REPLAY) {
      // n*l draws of uniform_index(2) = low bit of each output (rng.hpp:28-35,
      // threshold 0), solution-major (engine_parallel.hpp:334-336)
      std::vector<uint32_t> words(nv * Wp, 0);
      for (uint64_t s = 0; s < n; ++s)
        for (uint64_t v = 0; v < nv; ++v)
          if (rng.uniform_index(2)) words[v * Wp + (s >> 5)] |= 1u << (s & 31);
      GOMIX_CUDA(cudaMemcpyAsync(pop, words.data(), nv * Wp * 4, cudaMemcpyHostToDevice, stream));
      GOMIX_CUDA(cudaStreamSynchronize(stream));
    } else {
      launch_philox_init(pop, nv, (uint32_t)n, Wp, seed, rank, stream);
      ++launches;
    }
    launch_full_eval(*P, pop, fit, (uint32_t)n, Wp, epi_mode == 2, stream);
    launch_hash_population(snap_args(), stream);
    launches += 2;
    if (R > 1 && peer_on) {
      launch_peer_exchange(epi_args(0, 0, 0), stream);  // every rank's fitness and hashes
      ++launches;
    } else if (R > 1 && nccl) {
      exchange();
    }
    if (R == 1 || nccl || (peer_on && !local)) init_global(stop, out);
  }

  // the part of init after every rank's fitness and hashes are known
  void init_global(const gomix_stop_criteria* stop, gomix_run_stats* out) {
    begin_call(stop);
    launch_init_epilogue(epi_args(0, 0, 0), stream);
    ++launches;
    read_ctl();
    fill_stats(out);
    initialized = true;
  }

  // ---- sharding ---------------------------------------------------------------
  // Per-rank chunks exchanged after every group: rows (the donor pool of the
  // next group, engine_parallel.hpp:100-103), fitness, hashes, counters.
  struct Chunk {
    void* base;
    size_t bytes;  // rank r's chunk sits at base + r * bytes
  };
  std::vector<Chunk> shard_chunks(bool rows = true) const {
    std::vector<Chunk> c;
    if (rows) c.push_back({pool, P->nv * Wp * 4});
    c.push_back({fit_all, n * 8});
    c.push_back({h1_all, n * 8});
    c.push_back({h2_all, n * 8});
    c.push_back({rank_cnt, 16});
    return c;
  }

  // per-group exchange: rows only when the next group may read other ranks' rows
  std::vector<Chunk> group_chunks() const { return shard_chunks(!lite); }

  // all-gather over NCCL (in place), one grouped call
  void exchange(bool rows = true) {
    const NcclApi& api = nccl_or_throw();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const Chunk& c : shard_chunks(rows))
      nccl_check(api.AllGather(static_cast<char*>(c.base) + rank * c.bytes, c.base, c.bytes, ncclUint8,
                               nccl->comm, stream),
                 "ncclAllGather");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }

  void global_epilogue(uint64_t group) {
    const uint64_t G = P->group_off[group + 1] - P->group_off[group];
    launch_global_epilogue(epi_args(group, (uint32_t)G, 0), stream);
    ++launches;
  }

  // sharded generation (NCCL): local GOM step, exchange, global epilogue per group
  void run_generation_sharded(const gomix_stop_criteria* stop, gomix_run_stats* out) {
    begin_call(stop);
    std::vector<uint64_t> order;
    rng.permutation(order, P->k);  // same seed on every rank: same order
    if (peer_on) {
      // presence maps over peer memory, then per group ONE launch: the GOM
      // kernel's last CTA publishes, waits for every rank and runs the
      // global elitist scan (gom_peer.cuh) — no NCCL call, no extra launch
      launch_presence(d_peer, ctl, pop, P->nv, Wp, (uint32_t)n, (uint32_t)n_global, ones, stream);
      launches += 2;
      for (uint64_t gi : order) launch_group(gi, false);
      read_ctl();
      if (h_ctl->peer_fault) throw GomixError(GOMIX_E_NCCL, "peer exchange timed out (a rank stopped calling)");
      fill_stats(out);
      if (!h_ctl->stop) ++generation;
      return;
    }
    if (lite) {  // members holding 1 per row, summed over the ranks
      launch_count_ones(pop, P->nv, Wp, ones_local, stream);
      const NcclApi& api = nccl_or_throw();
      nccl_check(api.AllReduce(ones_local, ones, P->nv, ncclUint32, ncclSum, nccl->comm, stream), "ncclAllReduce");
      ++launches;
    }
    for (uint64_t gi : order) {
      launch_group(gi, false);
      exchange(!lite);
      global_epilogue(gi);
    }
    read_ctl();
    fill_stats(out);
    if (!h_ctl->stop) ++generation;
  }

  int32_t elitist_owner() const {
    return h_ctl->elit_src >= 0 ? (int32_t)((uint64_t)h_ctl->elit_src / n) : -1;
  }

  void run_generation(const gomix_stop_criteria* stop, gomix_run_stats* out) {
    if (!initialized) throw GomixError(GOMIX_E_STATE, "run_generation: population not initialised");
    if (R > 1) {
      if (!nccl && !peer_on)
        throw GomixError(GOMIX_E_STATE, "run_generation: in-process shards are driven by their local group");
      run_generation_sharded(stop, out);
      return;
    }
    if (mode == GOMIX_MODE_PHILOX && (gen_ok || !(flags & GOMIX_FLAG_TIME_KERNELS))) {
      stage_criteria(stop, true);
      if (fi_on) fi_snapshot();
      if (gen_ok)
        launch_generation_persistent();
      else
        launch_generation_graph();
      if (fi_on) fi_after_generation();
      read_ctl_published();
      fill_stats(out);
      if (!h_ctl->stop) ++generation;
      return;
    }
    begin_call(stop);
    if (fi_on) fi_snapshot();
    count_rows(stream);
    std::vector<uint64_t> order;
    rng.permutation(order, P->k);  // engine_parallel.hpp:291
    for (uint64_t gi : order) {
      if (mode == GOMIX_MODE_REPLAY) {
        if (gi != order.front()) {
          read_ctl();
          if (h_ctl->stop) break;
        }
        draw_replay_tape(gi, !univ_planes);  // the bit-sliced kernels take no donor tape
      }
      launch_group(gi, mode == GOMIX_MODE_REPLAY && !univ_planes);
    }
    if (fi_on) fi_after_generation();
    read_ctl();
    fill_stats(out);
    if (!h_ctl->stop) ++generation;  // engine_parallel.hpp:311-314
  }

  // Enqueue one generation without any host synchronisation (Philox mode,
  // no stop criteria); results are read by synchronize().
  void run_generation_async() {
    if (!initialized) throw GomixError(GOMIX_E_STATE, "run_generation: population not initialised");
    if (mode != GOMIX_MODE_PHILOX) invalid("run_generation_async: needs GOMIX_MODE_PHILOX");
    // sharded over peer memory (one process per GPU): the same CUDA graph
    // with the presence maps in front — every exchange runs inside the
    // kernels, the group order comes from the shared seed on the device
    if (R > 1 && (!peer_on || local)) invalid("run_generation_async: single-GPU or peer-transport engines only");
    if (gen_ok) {
      stage_criteria(nullptr, false);
      if (fi_on) fi_snapshot();
      launch_generation_persistent();
    } else if (flags & GOMIX_FLAG_TIME_KERNELS) {
      begin_call(nullptr);
      if (fi_on) fi_snapshot();
      count_rows(stream);
      std::vector<uint64_t> order;
      rng.permutation(order, P->k);
      for (uint64_t gi : order) launch_group(gi, false);
    } else {
      stage_criteria(nullptr, false);
      if (fi_on) fi_snapshot();
      launch_generation_graph();
    }
    if (fi_on) fi_after_generation();
    ++generation;
  }

  void synchronize(gomix_run_stats* out) {
    read_ctl();
    fill_stats(out);
  }

  // Replace the population (n x nv bytes, row per solution) and its fitness
  // (NULL = evaluate on the device); the elitist is kept.
  void load_population(const uint8_t* genotypes, const double* fitness) {
    if (!initialized) throw GomixError(GOMIX_E_STATE, "load_population: population not initialised");
    if (R > 1 && !nccl && !peer_on) invalid("load_population: in-process shards are driven by their local group");
    const uint64_t nv = P->nv;
    // the elitist snapshot may still point into the old population: finish it
    launch_finalize_elitist(snap_args(), stream);
    ++launches;
    uint8_t* d = staging();
    GOMIX_CUDA(cudaMemcpyAsync(d, genotypes, n * nv, cudaMemcpyHostToDevice, stream));
    launch_pack(d, pop, nv, (uint32_t)n, Wp, stream);
    ++launches;
    if (fitness) {
      GOMIX_CUDA(cudaMemcpyAsync(fit, fitness, n * 8, cudaMemcpyHostToDevice, stream));
    } else {
      launch_full_eval(*P, pop, fit, (uint32_t)n, Wp, epi_mode == 2, stream);
      ++launches;
    }
    launch_hash_population(snap_args(), stream);  // hashes of the new members
    ++launches;
    if (R > 1 && peer_on) {  // every rank's fitness and hashes (collective)
      launch_peer_exchange(epi_args(0, 0, 0), stream);
      ++launches;
    } else if (R > 1) {
      exchange();  // every rank's pool rows, fitness and hashes (collective)
    }
    GOMIX_CUDA(cudaStreamSynchronize(stream));
  }

  void run_group(uint64_t group, const int32_t* donor_tape, const gomix_stop_criteria* stop,
                 gomix_run_stats* out) {
    if (!initialized) throw GomixError(GOMIX_E_STATE, "run_group: population not initialised");
    if (R > 1) invalid("run_group: single-GPU engines only");
    if (group >= P->k) invalid("run_group: group index out of range");
    begin_call(stop);
    bool with_tape = true;
    if (donor_tape) {
      upload_tape(group, donor_tape);
    } else if (mode == GOMIX_MODE_REPLAY) {
      draw_replay_tape(group, !univ_planes);
      with_tape = !univ_planes;
    } else {
      with_tape = false;
    }
    if (!with_tape) count_rows(stream);
    launch_group(group, with_tape);
    read_ctl();
    fill_stats(out);
  }
};

// ===========================================================================
// In-process shards: R engines (one per device, or several on one device)
// driven in lock step by one host thread; the exchange is device-to-device
// copies ordered by events.  Same arithmetic as the NCCL path.
// ===========================================================================
struct gomix_gpu_local_group {
  std::vector<std::unique_ptr<gomix_gpu_engine>> eng;
  std::vector<cudaEvent_t> ev_step, ev_done;

  ~gomix_gpu_local_group() {
    for (auto& e : eng)
      if (e && e->stream) cudaStreamSynchronize(e->stream);
    for (auto e : ev_step) cudaEventDestroy(e);
    for (auto e : ev_done) cudaEventDestroy(e);
  }

  uint32_t R() const { return (uint32_t)eng.size(); }

  void set_device(uint32_t r) { GOMIX_CUDA(cudaSetDevice(eng[r]->P->device)); }

  // every engine finished its local step -> copy every rank's chunks everywhere
  void exchange(bool rows = true) {
    for (uint32_t r = 0; r < R(); ++r) {
      set_device(r);
      GOMIX_CUDA(cudaEventRecord(ev_step[r], eng[r]->stream));
    }
    for (uint32_t d = 0; d < R(); ++d) {
      set_device(d);
      gomix_gpu_engine& dst = *eng[d];
      const auto dchunks = dst.shard_chunks(rows);
      for (uint32_t r = 0; r < R(); ++r) {
        if (r == d) continue;
        GOMIX_CUDA(cudaStreamWaitEvent(dst.stream, ev_step[r], 0));
        const auto schunks = eng[r]->shard_chunks(rows);
        for (size_t c = 0; c < dchunks.size(); ++c)
          GOMIX_CUDA(cudaMemcpyAsync(static_cast<char*>(dchunks[c].base) + r * dchunks[c].bytes,
                                     static_cast<const char*>(schunks[c].base) + r * schunks[c].bytes,
                                     dchunks[c].bytes, cudaMemcpyDefault, dst.stream));
      }
      GOMIX_CUDA(cudaEventRecord(ev_done[d], dst.stream));
    }
    // nobody overwrites its rows before every copy out of them is done
    for (uint32_t r = 0; r < R(); ++r) {
      set_device(r);
      for (uint32_t d = 0; d < R(); ++d)
        if (d != r) GOMIX_CUDA(cudaStreamWaitEvent(eng[r]->stream, ev_done[d], 0));
    }
  }

  bool peer() const { return eng[0]->peer_on; }

  void init(const gomix_stop_criteria* stop, gomix_run_stats* out) {
    // every rank's work is queued before any rank synchronises: with the
    // peer transport the ranks' kernels wait for each other on the device
    for (uint32_t r = 0; r < R(); ++r) {
      set_device(r);
      eng[r]->init_population(nullptr, stop, nullptr);
    }
    if (!peer()) exchange();
    for (uint32_t r = 0; r < R(); ++r) {
      set_device(r);
      eng[r]->init_global(stop, r == 0 ? out : nullptr);
    }
  }

  void run_generation(const gomix_stop_criteria* stop, gomix_run_stats* out) {
    for (auto& e : eng)
      if (!e->initialized) throw GomixError(GOMIX_E_STATE, "run_generation: population not initialised");
    std::vector<uint64_t> order;
    for (uint32_t r = 0; r < R(); ++r) {
      set_device(r);
      eng[r]->begin_call(stop);
      std::vector<uint64_t> o;
      eng[r]->rng.permutation(o, eng[r]->P->k);
      if (r == 0) order = o;
    }
    if (peer()) {
      // presence maps, then per group one launch per rank whose last CTA
      // exchanges over peer memory and runs the global scan (gom_peer.cuh);
      // every rank's launches are queued before any rank synchronises
      for (uint32_t r = 0; r < R(); ++r) {
        set_device(r);
        gomix_gpu_engine& e = *eng[r];
        launch_presence(e.d_peer, e.ctl, e.pop, e.P->nv, e.Wp, (uint32_t)e.n, (uint32_t)e.n_global, e.ones,
                        e.stream);
        e.launches += 2;
      }
      for (uint64_t gi : order)
        for (uint32_t r = 0; r < R(); ++r) {
          set_device(r);
          eng[r]->launch_group(gi, false);
        }
      for (uint32_t r = 0; r < R(); ++r) {
        set_device(r);
        eng[r]->read_ctl();
        if (eng[r]->h_ctl->peer_fault) throw GomixError(GOMIX_E_NCCL, "peer exchange timed out");
        eng[r]->fill_stats(r == 0 ? out : nullptr);
        if (!eng[r]->h_ctl->stop) ++eng[r]->generation;
      }
      return;
    }
    const bool lite = eng[0]->lite;
    if (lite) {  // members holding 1 per row, summed over the ranks (the NCCL all-reduce)
      for (uint32_t r = 0; r < R(); ++r) {
        set_device(r);
        launch_count_ones(eng[r]->pop, eng[r]->P->nv, eng[r]->Wp, eng[r]->ones_local, eng[r]->stream);
        GOMIX_CUDA(cudaEventRecord(ev_step[r], eng[r]->stream));
      }
      for (uint32_t d = 0; d < R(); ++d) {
        set_device(d);
        gomix_gpu_engine& dst = *eng[d];
        const uint64_t nv = dst.P->nv;
        for (uint32_t r = 0; r < R(); ++r) {
          GOMIX_CUDA(cudaStreamWaitEvent(dst.stream, ev_step[r], 0));
          GOMIX_CUDA(cudaMemcpyAsync(dst.ones_stage + (uint64_t)r * nv, eng[r]->ones_local, nv * 4, cudaMemcpyDefault,
                                     dst.stream));
        }
        launch_sum_ones(dst.ones_stage, R(), nv, dst.ones, dst.stream);
        GOMIX_CUDA(cudaEventRecord(ev_done[d], dst.stream));
      }
      for (uint32_t r = 0; r < R(); ++r) {
        set_device(r);
        for (uint32_t d = 0; d < R(); ++d)
          if (d != r) GOMIX_CUDA(cudaStreamWaitEvent(eng[r]->stream, ev_done[d], 0));
      }
    }
    for (uint64_t gi : order) {
      for (uint32_t r = 0; r < R(); ++r) {
        set_device(r);
        eng[r]->launch_group(gi, false);
      }
      exchange(!lite);
      for (uint32_t r = 0; r < R(); ++r) {
        set_device(r);
        eng[r]->global_epilogue(gi);
      }
    }
    for (uint32_t r = 0; r < R(); ++r) {
      set_device(r);
      eng[r]->read_ctl();
      eng[r]->fill_stats(r == 0 ? out : nullptr);
      if (!eng[r]->h_ctl->stop) ++eng[r]->generation;
    }
  }
};

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int gomix_gpu_abi_version(void) { return GOMIX_GPU_ABI_VERSION; }

GOMIX_API int gomix_debug_cta_probes(unsigned long long* out) {
  return guarded([&] { debug_cta_probes(out); });
}

// latency-study probes (GOMIX_EXP bit 32), not part of the public header
GOMIX_API int gomix_debug_set_flags(uint32_t flags) {
  g_exp_flags.store(flags);
  return GOMIX_OK;
}

GOMIX_API int gomix_debug_probes(unsigned long long* out, int32_t reset) {
  return guarded([&] {
    unsigned long long b[64];
    debug_probes(out, reset != 0);
    debug_probes_gen(b, reset != 0);
    for (int i = 0; i < 64; ++i)
      if (!out[i]) out[i] = b[i];
    debug_probes_univ(b, reset != 0);
    for (int i = 0; i < 64; ++i)
      if (!out[i]) out[i] = b[i];
  });
}

// truth-table kernel launch timeline, probes builds (build.py --probes):
// out[32r + 2i] / out[32r + 2i + 1] = first / last CTA at point i of launch
// row r (graph slot + 1, 0 = direct), r < 4; out[128 + ...] the begin
// kernel (points 0, 1); %globaltimer ns, 160 words; resets
GOMIX_API int gomix_debug_timeline(unsigned long long* out) {
  return guarded([&] {
    debug_timeline_univ(out);
    debug_timeline_gom(out + 128);
  });
}

// the persistent generation kernel's timeline, probes builds (gom_gen.cu
// gen_mark): 128 words, first / last arrival per point; resets
GOMIX_API int gomix_debug_gen_timeline(unsigned long long* out) {
  return guarded([&] { debug_gen_timeline(out); });
}

// per-CTA record of the truth-table launches, probes builds: out[((r * 1024)
// + cta) * 4 + {0: SM, 1: start ns, 2: batches done ns, 3: batches}], row r =
// graph slot + 1 (0 = direct), 4 rows; then 16 batch-loop path counters
// (gom_tt.cuh tt_count, reset on read)
GOMIX_API int gomix_debug_cta_stats(unsigned long long* out) {
  return guarded([&] { debug_cta_stats_univ(out); });
}

const char* gomix_gpu_last_error(void) { return g_last_error.c_str(); }

int gomix_gpu_problem_create(const gomix_maxcut* instance, const gomix_fos* fos,
                             const int32_t* set_colour, int32_t device, gomix_gpu_problem** out) {
  return guarded([&] {
    if (!out) invalid("problem_create: out is NULL");
    *out = nullptr;
    auto h = std::make_unique<gomix_gpu_problem>();
    h->P = create_problem(instance, fos, set_colour, device);
    *out = h.release();
  });
}

int gomix_gpu_problem_destroy(gomix_gpu_problem* p) {
  return guarded([&] { delete p; });
}

int gomix_gpu_problem_info(const gomix_gpu_problem* p, gomix_problem_info* out) {
  return guarded([&] {
    if (!p || !out) invalid("problem_info: NULL argument");
    const Problem& P = *p->P;
    out->num_vertices = P.nv;
    out->num_edges = P.q;
    out->num_sets = P.m;
    out->num_groups = P.k;
    out->lmig_edges = P.lmig_edges;
    out->max_set_size = P.max_f;
    out->exact = P.exact;
    out->univariate = P.univariate;
  });
}

int gomix_gpu_problem_groups(const gomix_gpu_problem* p, uint64_t* group_offset,
                             uint64_t* group_sets) {
  return guarded([&] {
    if (!p) invalid("problem_groups: NULL problem");
    if (group_offset) std::copy(p->P->group_off.begin(), p->P->group_off.end(), group_offset);
    if (group_sets) std::copy(p->P->group_sets.begin(), p->P->group_sets.end(), group_sets);
  });
}

int gomix_gpu_problem_footprints(const gomix_gpu_problem* p, uint64_t* footprint) {
  return guarded([&] {
    if (!p || !footprint) invalid("problem_footprints: NULL argument");
    std::copy(p->P->footprint.begin(), p->P->footprint.end(), footprint);
  });
}

int gomix_gpu_engine_create(gomix_gpu_problem* p, const gomix_engine_config* cfg,
                            gomix_gpu_engine** out) {
  return guarded([&] {
    if (!p || !cfg || !out) invalid("engine_create: NULL argument");
    *out = nullptr;
    auto e = std::make_unique<gomix_gpu_engine>();
    e->P = p->P.get();
    e->setup(*cfg);
    *out = e.release();
  });
}

int gomix_gpu_engine_destroy(gomix_gpu_engine* e) {
  return guarded([&] { delete e; });
}

int gomix_gpu_set_stream(gomix_gpu_engine* e, void* cuda_stream) {
  return guarded([&] {
    if (!e) invalid("set_stream: NULL engine");
    GOMIX_CUDA(cudaStreamSynchronize(e->stream));
    if (e->own_stream) GOMIX_CUDA(cudaStreamDestroy(e->stream));
    if (cuda_stream) {
      e->stream = static_cast<cudaStream_t>(cuda_stream);
      e->own_stream = false;
    } else {
      GOMIX_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
      e->own_stream = true;
    }
  });
}

int gomix_gpu_init_population(gomix_gpu_engine* e, const uint8_t* genotypes,
                              const gomix_stop_criteria* stop, gomix_run_stats* out) {
  return guarded([&] {
    if (!e) invalid("init_population: NULL engine");
    e->init_population(genotypes, stop, out);
  });
}

int gomix_gpu_run_generation(gomix_gpu_engine* e, const gomix_stop_criteria* stop,
                             gomix_run_stats* out) {
  return guarded([&] {
    if (!e) invalid("run_generation: NULL engine");
    e->run_generation(stop, out);
  });
}

int gomix_gpu_run_generation_async(gomix_gpu_engine* e) {
  return guarded([&] {
    if (!e) invalid("run_generation_async: NULL engine");
    e->run_generation_async();
  });
}

int gomix_gpu_synchronize(gomix_gpu_engine* e, gomix_run_stats* out) {
  return guarded([&] {
    if (!e) invalid("synchronize: NULL engine");
    e->synchronize(out);
  });
}

int gomix_gpu_load_population(gomix_gpu_engine* e, const uint8_t* genotypes, const double* fitness) {
  return guarded([&] {
    if (!e || !genotypes) invalid("load_population: NULL argument");
    for (uint64_t i = 0; i < e->n * e->P->nv; ++i)
      if (genotypes[i] > 1) invalid("graybox: genotype value outside alphabet");
    e->load_population(genotypes, fitness);
  });
}

int gomix_gpu_run_group(gomix_gpu_engine* e, uint64_t group, const int32_t* donor_tape,
                        const gomix_stop_criteria* stop, gomix_run_stats* out) {
  return guarded([&] {
    if (!e) invalid("run_group: NULL engine");
    e->run_group(group, donor_tape, stop, out);
  });
}

int gomix_gpu_forced_improvement(gomix_gpu_engine* e, const uint8_t* flags, const uint32_t* group_order,
                                 const gomix_stop_criteria* stop, gomix_run_stats* out) {
  return guarded([&] {
    if (!e) invalid("forced_improvement: NULL engine");
    e->forced_improvement(flags, group_order, stop, out);
  });
}

int gomix_gpu_read_batch(gomix_gpu_engine* e, int32_t* donor, double* delta, uint8_t* present,
                         uint8_t* accept) {
  return guarded([&] {
    if (!e) invalid("read_batch: NULL engine");
    if (!e->record) throw GomixError(GOMIX_E_STATE, "read_batch: engine created without GOMIX_FLAG_RECORD_BATCH");
    if (e->last_group < 0) throw GomixError(GOMIX_E_STATE, "read_batch: no group has run");
    const uint64_t g = (uint64_t)e->last_group;
    const uint64_t G = e->P->group_off[g + 1] - e->P->group_off[g], n = e->n, pairs = G * n;
    std::vector<int32_t> d(pairs);
    std::vector<double> de(pairs);
    std::vector<uint8_t> pr(pairs), ac(pairs);
    GOMIX_CUDA(cudaMemcpyAsync(d.data(), e->rec_donor, pairs * 4, cudaMemcpyDeviceToHost, e->stream));
    GOMIX_CUDA(cudaMemcpyAsync(de.data(), e->rec_delta, pairs * 8, cudaMemcpyDeviceToHost, e->stream));
    GOMIX_CUDA(cudaMemcpyAsync(pr.data(), e->rec_present, pairs, cudaMemcpyDeviceToHost, e->stream));
    GOMIX_CUDA(cudaMemcpyAsync(ac.data(), e->rec_accept, pairs, cudaMemcpyDeviceToHost, e->stream));
    GOMIX_CUDA(cudaStreamSynchronize(e->stream));
    for (uint64_t p = 0; p < G; ++p)
      for (uint64_t s = 0; s < n; ++s) {
        const uint64_t src = p * n + s, dst = s * G + p;
        if (donor) donor[dst] = d[src];
        if (delta) delta[dst] = de[src];
        if (present) present[dst] = pr[src];
        if (accept) accept[dst] = ac[src];
      }
  });
}

int gomix_gpu_read_population(gomix_gpu_engine* e, uint8_t* genotypes, double* fitness) {
  return guarded([&] {
    if (!e) invalid("read_population: NULL engine");
    if (genotypes) {
      const uint64_t bytes = e->n * e->P->nv;
      uint8_t* d = e->staging();
      launch_unpack(e->pop, d, e->P->nv, (uint32_t)e->n, e->Wp, e->stream);
      ++e->launches;
      GOMIX_CUDA(cudaMemcpyAsync(genotypes, d, bytes, cudaMemcpyDeviceToHost, e->stream));
    }
    if (fitness)
      GOMIX_CUDA(cudaMemcpyAsync(fitness, e->fit, e->n * 8, cudaMemcpyDeviceToHost, e->stream));
    GOMIX_CUDA(cudaStreamSynchronize(e->stream));
  });
}

int gomix_gpu_read_population_packed(gomix_gpu_engine* e, uint32_t* words, uint64_t* words_per_var) {
  return guarded([&] {
    if (!e) invalid("read_population_packed: NULL engine");
    if (words_per_var) *words_per_var = e->Wp;
    if (words) {
      GOMIX_CUDA(cudaMemcpyAsync(words, e->pop, e->P->nv * e->Wp * 4, cudaMemcpyDeviceToHost, e->stream));
      GOMIX_CUDA(cudaStreamSynchronize(e->stream));
    }
  });
}

int gomix_gpu_read_elitist(gomix_gpu_engine* e, uint8_t* genotype, double* fitness) {
  return guarded([&] {
    if (!e) invalid("read_elitist: NULL engine");
    if (!e->initialized) throw GomixError(GOMIX_E_STATE, "read_elitist: population not initialised");
    if (genotype) {
      launch_finalize_elitist(e->snap_args(), e->stream);  // complete the copy-on-write snapshot
      ++e->launches;
      if (e->R > 1 && e->peer_on && !e->local) {
        // collective over the ranks over peer memory: the owner's snapshot
        const int32_t owner = e->elitist_owner();
        if (owner >= 0) {
          launch_peer_elitist(e->d_peer, e->ctl, e->elit, e->P->nv, (uint32_t)owner == e->rank, ++e->xe_epoch,
                              e->stream);
          ++e->launches;
        }
      } else if (e->R > 1) {
        // collective over the ranks: the owner's snapshot is the valid one
        if (!e->nccl) invalid("read_elitist: use gomix_gpu_local_group_read_elitist for in-process shards");
        const int32_t owner = e->elitist_owner();
        if (owner >= 0) {
          const NcclApi& api = nccl_or_throw();
          nccl_check(api.Broadcast(e->elit, e->elit, ((e->P->nv + 31) / 32) * 4, ncclUint8, owner,
                                   e->nccl->comm, e->stream),
                     "ncclBroadcast");
        }
      }
      uint8_t* d = e->staging();
      launch_unpack_elitist(e->elit, d, e->P->nv, e->stream);
      ++e->launches;
      GOMIX_CUDA(cudaMemcpyAsync(genotype, d, e->P->nv, cudaMemcpyDeviceToHost, e->stream));
    }
    GOMIX_CUDA(cudaStreamSynchronize(e->stream));
    if (fitness) *fitness = e->host_elit_fit();
  });
}

int gomix_gpu_offer_elitist(gomix_gpu_engine* e, const uint8_t* genotype, double fitness,
                            int32_t* adopted) {
  return guarded([&] {
    if (!e || !genotype) invalid("offer_elitist: NULL argument");
    if (!e->initialized) throw GomixError(GOMIX_E_STATE, "offer_elitist: population not initialised");
    const bool take = e->better(fitness, e->host_elit_fit());
    if (adopted) *adopted = take;
    if (!take) return;
    const uint64_t nv = e->P->nv;
    uint8_t* d = nullptr;
    GOMIX_CUDA(cudaMallocAsync(&d, nv, e->stream));
    GOMIX_CUDA(cudaMemcpyAsync(d, genotype, nv, cudaMemcpyHostToDevice, e->stream));
    launch_pack_elitist(d, e->elit, nv, e->stream);
    GOMIX_CUDA(cudaFreeAsync(d, e->stream));
    launch_external_elitist(e->snap_args(), fitness, e->stream);
    e->launches += 2;
    GOMIX_CUDA(cudaStreamSynchronize(e->stream));
    e->elit_fit = fitness;
  });
}

// ---- IMS on the device ---------------------------------------------------------
struct gomix_gpu_ims_best {
  Problem* P = nullptr;
  int device = 0;
  ImsBestDev* dev = nullptr;
  uint32_t* bits = nullptr;
  ImsBestDev* host = nullptr;  // pinned
  cudaEvent_t ev = nullptr;    // last queued exchange
  cudaStream_t last = nullptr;
  std::vector<void*> allocs;
  ~gomix_gpu_ims_best() {
    if (ev) cudaEventSynchronize(ev), cudaEventDestroy(ev);
    cudaDeviceSynchronize();
    cached_free_all(allocs);
    if (host) cudaFreeHost(host);
  }
  void order_before(gomix_gpu_engine* e) {
    if (e->P != P) invalid("ims: engine belongs to another problem");
    if (e->R > 1) invalid("ims: sharded engines are not supported");
    if (!e->initialized) throw GomixError(GOMIX_E_STATE, "ims: population not initialised");
    GOMIX_CUDA(cudaStreamWaitEvent(e->stream, ev, 0));
  }
  void order_after(gomix_gpu_engine* e) {
    GOMIX_CUDA(cudaEventRecord(ev, e->stream));
    last = e->stream;
  }
};

int gomix_gpu_ims_best_create(gomix_gpu_problem* p, gomix_gpu_ims_best** out) {
  return guarded([&] {
    if (!p || !out) invalid("ims_best_create: NULL argument");
    auto b = std::make_unique<gomix_gpu_ims_best>();
    b->P = p->P.get();
    b->device = b->P->device;
    GOMIX_CUDA(cudaSetDevice(b->device));
    b->dev = dev_alloc<ImsBestDev>(b->allocs, 1);
    b->bits = dev_alloc<uint32_t>(b->allocs, (b->P->nv + 31) / 32);
    GOMIX_CUDA(cudaMemset(b->dev, 0, sizeof(ImsBestDev)));
    GOMIX_CUDA(cudaMemset(b->bits, 0, ((b->P->nv + 31) / 32) * 4));
    GOMIX_CUDA(cudaMallocHost(&b->host, sizeof(ImsBestDev)));
    GOMIX_CUDA(cudaEventCreateWithFlags(&b->ev, cudaEventDisableTiming));
    GOMIX_CUDA(cudaDeviceSynchronize());
    *out = b.release();
  });
}

int gomix_gpu_ims_best_destroy(gomix_gpu_ims_best* b) {
  delete b;
  return GOMIX_OK;
}

int gomix_gpu_ims_collect(gomix_gpu_ims_best* b, gomix_gpu_engine* e) {
  return guarded([&] {
    if (!b || !e) invalid("ims_collect: NULL argument");
    b->order_before(e);
    launch_ims_collect(e->snap_args(), b->dev, b->bits, e->P->exact, e->stream);
    e->launches += 2;
    b->order_after(e);
  });
}

int gomix_gpu_ims_offer(gomix_gpu_ims_best* b, gomix_gpu_engine* e) {
  return guarded([&] {
    if (!b || !e) invalid("ims_offer: NULL argument");
    b->order_before(e);
    launch_ims_offer(e->snap_args(), b->dev, b->bits, e->P->exact, e->stream);
    e->launches += 2;
    e->ctl_stale = true;
    b->order_after(e);
  });
}

int gomix_gpu_ims_best_read(gomix_gpu_ims_best* b, uint8_t* genotype, double* fitness, int32_t* valid) {
  return guarded([&] {
    if (!b) invalid("ims_best_read: NULL argument");
    GOMIX_CUDA(cudaSetDevice(b->device));
    GOMIX_CUDA(cudaEventSynchronize(b->ev));
    GOMIX_CUDA(cudaMemcpy(b->host, b->dev, sizeof(ImsBestDev), cudaMemcpyDeviceToHost));
    if (fitness) *fitness = b->host->fit;
    if (valid) *valid = b->host->valid;
    if (genotype) {
      const uint64_t nv = b->P->nv;
      std::vector<uint32_t> w((nv + 31) / 32);
      GOMIX_CUDA(cudaMemcpy(w.data(), b->bits, w.size() * 4, cudaMemcpyDeviceToHost));
      for (uint64_t v = 0; v < nv; ++v) genotype[v] = (w[v >> 5] >> (v & 31)) & 1u;
    }
  });
}

int gomix_gpu_read_improvements(gomix_gpu_engine* e, double* fitness, uint64_t* evaluator_calls,
                                uint64_t capacity, uint64_t* count) {
  return guarded([&] {
    if (!e) invalid("read_improvements: NULL engine");
    const uint64_t avail = std::min<uint64_t>(e->h_ctl->n_impr, e->impr_cap);
    const bool any = fitness || evaluator_calls;
    const uint64_t take = any ? std::min(avail, capacity) : 0;
    std::vector<ImprRec> far;
    const ImprRec* src = e->h_impr;  // copied back with the control block
    if (take > gomix_gpu_engine::kImprInline) {
      far.resize(take);
      GOMIX_CUDA(cudaMemcpyAsync(far.data(), e->impr, take * sizeof(ImprRec), cudaMemcpyDeviceToHost, e->stream));
      GOMIX_CUDA(cudaStreamSynchronize(e->stream));
      src = far.data();
    }
    for (uint64_t i = 0; i < take; ++i) {
      if (fitness) fitness[i] = src[i].fit;
      if (evaluator_calls) evaluator_calls[i] = src[i].calls;
    }
    if (count) *count = any ? take : avail;
  });
}

int gomix_gpu_group_counters(gomix_gpu_engine* e, uint64_t* sets, uint64_t* steps,
                             uint64_t* evaluator_calls) {
  return guarded([&] {
    if (!e) invalid("group_counters: NULL engine");
    const uint64_t k = e->P->k;
    if (sets)
      for (uint64_t c = 0; c < k; ++c) sets[c] = e->P->group_off[c + 1] - e->P->group_off[c];
    if (steps) GOMIX_CUDA(cudaMemcpyAsync(steps, e->gsteps, k * 8, cudaMemcpyDeviceToHost, e->stream));
    if (evaluator_calls)
      GOMIX_CUDA(cudaMemcpyAsync(evaluator_calls, e->gcalls, k * 8, cudaMemcpyDeviceToHost, e->stream));
    GOMIX_CUDA(cudaStreamSynchronize(e->stream));
  });
}

int gomix_gpu_generation(gomix_gpu_engine* e, int64_t* generation) {
  return guarded([&] {
    if (!e || !generation) invalid("generation: NULL argument");
    *generation = e->generation;
  });
}

int gomix_gpu_kernel_times(gomix_gpu_engine* e, float* ms, uint64_t capacity, uint64_t* count) {
  return guarded([&] {
    if (!e) invalid("kernel_times: NULL engine");
    if (!ms) {  // query only
      if (count) *count = e->ev_pending.size();
      return;
    }
    GOMIX_CUDA(cudaStreamSynchronize(e->stream));
    uint64_t written = 0;
    for (auto& pr : e->ev_pending) {
      float t = 0.f;
      GOMIX_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second));
      if (written < capacity) ms[written] = t;
      ++written;
      e->ev_free.push_back(pr.first);
      e->ev_free.push_back(pr.second);
    }
    e->ev_pending.clear();
    if (count) *count = std::min(written, capacity);
  });
}

int gomix_gpu_set_timing(gomix_gpu_engine* e, int32_t enable) {
  return guarded([&] {
    if (!e) invalid("set_timing: NULL engine");
    if (enable)
      e->flags |= GOMIX_FLAG_TIME_KERNELS;
    else
      e->flags &= ~(uint32_t)GOMIX_FLAG_TIME_KERNELS;
  });
}

const char* gomix_gpu_engine_kernel_name(const gomix_gpu_engine* e) {
  if (!e) return "";
  if (e->univ_f64) return "gom_univ_f64_kernel";
  return e->univ_planes ? (e->univ_tt ? "gom_univ_tt_kernel" : "gom_univ_sliced_kernel") : e->gen_ok ? "gom_generation_kernel" : "gom_group_kernel";
}

int gomix_gpu_launch_count(gomix_gpu_engine* e, uint64_t* count) {
  return guarded([&] {
    if (!e || !count) invalid("launch_count: NULL argument");
    *count = e->launches;
  });
}

int gomix_gpu_color(const gomix_maxcut* instance, const gomix_fos* fos, int32_t device,
                    int32_t* set_colour, uint64_t* num_groups, uint64_t* lmig_edges) {
  return guarded([&] {
    auto P = create_problem(instance, fos, nullptr, device);
    if (set_colour)
      for (uint64_t c = 0; c < P->k; ++c)
        for (uint64_t t = P->group_off[c]; t < P->group_off[c + 1]; ++t)
          set_colour[P->group_sets[t]] = (int32_t)c;
    if (num_groups) *num_groups = P->k;
    if (lmig_edges) *lmig_edges = P->lmig_edges;
  });
}

int gomix_gpu_nccl_unique_id(uint8_t* id) {
  return guarded([&] {
    if (!id) invalid("nccl_unique_id: NULL buffer");
    const NcclApi& api = nccl_or_throw();
    ncclUniqueId u;
    nccl_check(api.GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int gomix_gpu_peer_export(gomix_gpu_engine* e, uint8_t* handle) {
  return guarded([&] {
    if (!e || !handle) invalid("peer_export: NULL argument");
    e->peer_export(handle);
  });
}

int gomix_gpu_peer_connect(gomix_gpu_engine* e, const uint8_t* handles) {
  return guarded([&] {
    if (!e || !handles) invalid("peer_connect: NULL argument");
    e->peer_connect(handles);
  });
}

int gomix_gpu_local_group_create(gomix_gpu_problem* const* problems, const gomix_engine_config* cfg,
                                 gomix_gpu_local_group** out) {
  return guarded([&] {
    if (!problems || !cfg || !out) invalid("local_group_create: NULL argument");
    if (cfg->world_size < 1) invalid("local_group_create: world_size must be >= 1");
    *out = nullptr;
    auto g = std::make_unique<gomix_gpu_local_group>();
    for (int32_t r = 0; r < cfg->world_size; ++r) {
      if (!problems[r]) invalid("local_group_create: NULL problem");
      gomix_engine_config c = *cfg;
      c.rank = r;
      c.nccl_unique_id = nullptr;
      auto e = std::make_unique<gomix_gpu_engine>();
      e->P = problems[r]->P.get();
      if (e->P->nv != problems[0]->P->nv || e->P->k != problems[0]->P->k)
        invalid("local_group_create: every rank needs the same problem");
      e->setup(c);
      e->local = g.get();
      cudaEvent_t a, b;
      GOMIX_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      GOMIX_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      g->ev_step.push_back(a);
      g->ev_done.push_back(b);
      g->eng.push_back(std::move(e));
    }
    if (cfg->flags & GOMIX_FLAG_PEER_TRANSPORT) {  // in process: every rank's block by its device pointer
      std::vector<char*> blocks;
      for (auto& e : g->eng) {
        e->peer_alloc();
        blocks.push_back(e->xblock);
      }
      for (auto& e : g->eng) e->peer_set_blocks(blocks.data());
    }
    *out = g.release();
  });
}

int gomix_gpu_local_group_destroy(gomix_gpu_local_group* g) {
  return guarded([&] { delete g; });
}

int gomix_gpu_local_group_engine(gomix_gpu_local_group* g, int32_t rank, gomix_gpu_engine** out) {
  return guarded([&] {
    if (!g || !out || rank < 0 || (uint32_t)rank >= g->R()) invalid("local_group_engine: bad argument");
    *out = g->eng[rank].get();
  });
}

int gomix_gpu_local_group_init_population(gomix_gpu_local_group* g, const gomix_stop_criteria* stop,
                                          gomix_run_stats* out) {
  return guarded([&] {
    if (!g) invalid("local_group_init_population: NULL group");
    g->init(stop, out);
  });
}

int gomix_gpu_local_group_run_generation(gomix_gpu_local_group* g, const gomix_stop_criteria* stop,
                                         gomix_run_stats* out) {
  return guarded([&] {
    if (!g) invalid("local_group_run_generation: NULL group");
    g->run_generation(stop, out);
  });
}

int gomix_gpu_local_group_read_elitist(gomix_gpu_local_group* g, uint8_t* genotype, double* fitness) {
  return guarded([&] {
    if (!g) invalid("local_group_read_elitist: NULL group");
    gomix_gpu_engine& e0 = *g->eng[0];
    const int32_t owner = e0.elitist_owner();
    gomix_gpu_engine& e = *g->eng[owner >= 0 ? owner : 0];
    GOMIX_CUDA(cudaSetDevice(e.P->device));
    if (genotype) {
      launch_finalize_elitist(e.snap_args(), e.stream);
      uint8_t* d = e.staging();
      launch_unpack_elitist(e.elit, d, e.P->nv, e.stream);
      GOMIX_CUDA(cudaMemcpyAsync(genotype, d, e.P->nv, cudaMemcpyDeviceToHost, e.stream));
      GOMIX_CUDA(cudaStreamSynchronize(e.stream));
    }
    if (fitness) *fitness = e0.elit_fit;
  });
}

}  // extern "C"
