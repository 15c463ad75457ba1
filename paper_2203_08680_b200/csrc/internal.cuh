// internal.cuh — device data layout and shared helpers of libgomix_b200.
//
// HBM layout:
//   population  : num_vertices rows x Wp uint32 words ("variable-major, bit-
//                 sliced"): bit b of word w of row v = allele of variable v in
//                 solution 32w+b.  One coalesced row gives a variable's value in
//                 every solution, so "does any member differ on F" is a few
//                 word ops and a group touches each row it needs once.
//   graph CSR   : row_ptr[nv+1], col[2q] (ascending neighbour = ascending edge
//                 id, the reference's summation order), w[2q] fp64 and, when the
//                 weights are small integers, wi[2q] int32.
//   footprints  : per linkage set, its dependent subfunctions (edges) sorted by
//                 edge id (make_group_plan, engine_parallel.hpp:37-59) as
//                 FpEntry {a, b, w}; endpoints inside the set are encoded as
//                 kInSet | position-in-set.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "gomix_gpu.h"

namespace gomix_b200 {

constexpr uint32_t kInSet = 0x80000000u;
constexpr int kMaxSetSize = 64;     // per-lane set patterns are uint64 masks
constexpr int kEpilogueThreads = 1024;

struct FpEntry {
  uint32_t a, b;  // endpoint vertex id, or kInSet | index within the set
  double w;
};

// Run-control block living in device memory; updated by the epilogue kernel
// after every group so stop criteria never need a host round trip.
struct DevCtl {
  double elit_fit;
  int32_t elit_src;     // >= 0: elitist = population column elit_src (copy-on-write); -2: bits given; -1: none
  int32_t stop;         // latched stop request (RunControl::request_stop, runtime.hpp:104-109)
  int32_t stop_reason;  // GOMIX_STOP_*
  int32_t has_budget;
  int32_t has_target;
  int32_t exact;
  double max_evals;
  double q;
  double target;
  unsigned long long calls_total;  // absolute evaluator calls (RunControl::calls_)
  unsigned long long grp_steps, grp_calls;
  unsigned long long run_steps, run_calls, groups_run;
  unsigned long long n_impr;
  unsigned int done;  // last-CTA-done ticket of the GOM kernel
  unsigned int gen_counter;  // device-side generation counter (graph path)
  unsigned int cur_gen;
  // device-owned elitist identity (never touched by the per-call reset)
  unsigned long long eh1, eh2;  // 128-bit Zobrist hash of the elitist genotype
  unsigned int elit_ver;        // snapshot version: row v is captured iff ever[v] == elit_ver
  unsigned int gen_buf;         // persistent generation kernel: running accumulator index
  // peer transport (gom_peer.cuh): exchange epochs, identical on every rank
  unsigned long long xg_epoch, xp_epoch, xe_epoch;
  unsigned int xp_ticket;       // last-CTA ticket of the presence publish
  unsigned int peer_fault;      // a peer exchange timed out
};

// One colour group as the device sees it (graph path: kernels look their
// group up through the per-generation order array).
struct GroupDesc {
  uint32_t g0;  // offset of the group's members in gsets / gvars
  uint32_t G;   // member count
};

struct Problem {
  int device = 0;
  uint64_t nv = 0, q = 0, m = 0, k = 0, lmig_edges = 0, max_f = 0, max_fp = 0;
  double sum_abs_w = 0.0;    // sum of |w| over the edges (fixed-point scale of float fitness deltas)
  uint64_t max_abs_row = 0;  // univariate: max over sets {v} of sum |w| on v's edges (integer weights)
  bool exact = true, univariate = true, i32 = false;
  bool var_once = true;  // every variable is in at most one linkage set
  // host mirrors (small)
  std::vector<uint64_t> h_set_off;
  std::vector<uint32_t> h_set_vars;
  std::vector<uint64_t> group_off;   // k + 1
  std::vector<uint64_t> group_sets;  // m, concatenated, ascending within a group
  std::vector<uint64_t> footprint;   // per set
  // device
  int32_t* row_ptr = nullptr;
  int32_t* col = nullptr;
  double* w = nullptr;
  int32_t* wi = nullptr;
  uint32_t* eu = nullptr;
  uint32_t* ev = nullptr;
  double* ew = nullptr;
  int64_t* set_off = nullptr;
  uint32_t* set_vars = nullptr;
  uint32_t* gsets = nullptr;
  uint32_t* gvars = nullptr;
  uint4* gmeta = nullptr;
  uint4* urec = nullptr;       // univariate, degree <= 4, |w| < 2^15: truth-table plan records (2 per position)
  ulonglong2* ukey = nullptr;  // ... and the Zobrist key of each position's variable (every univariate FOS)
  uint4* uvr = nullptr;        // univariate FOS: {v, row start, row end, 0} per group position
  uint32_t wbits = 1;
  int64_t* fp_off = nullptr;
  FpEntry* fp = nullptr;
  std::vector<void*> allocations;
  ~Problem();
};

// One elitist improvement (TraceSink::improvement, runtime.hpp:24-29); the log
// directly follows the control block in device memory, so one copy returns
// the control block and the first log entries.
struct ImprRec {
  double fit;
  unsigned long long calls;
};

struct PeerArgs;

struct EpiArgs {
  double* fit;
  long long* dfit;   // fixed-point fitness deltas of this group (fix_inv per unit)
  double fix_inv;    // 1 / GomArgs::fix_scale
  unsigned long long* h1;  // per-solution Zobrist hashes
  unsigned long long* h2;
  unsigned long long* dh1;  // this group's XOR deltas
  unsigned long long* dh2;
  const double* rec_delta;
  const uint8_t* rec_accept;
  DevCtl* ctl;
  unsigned long long* gsteps;
  unsigned long long* gcalls;
  ImprRec* impr;  // improvement log: fitness + RunControl call count when it was reported
  uint64_t impr_cap;
  uint32_t n, G, nparts, group;  // n: this rank's solutions
  int32_t mode;  // 0 integer weights, 1 float, 2 ordered (replay float: recorded deltas in position order)
  // sharding: fit/h1/h2 above are this rank's slices of the gathered arrays
  const double* fit_all;
  const unsigned long long* h1_all;
  const unsigned long long* h2_all;
  unsigned long long* rank_cnt;  // [R][steps, calls] of the current group
  uint32_t n_global, R, rank;
  const PeerArgs* peer;  // sharded, peer transport: the exchange runs inside the epilogue (gom_peer.cuh)
  const double* word_max;  // per 32-solution word: max fitness after the commit (nullptr: the scan computes it)
};

// elitist snapshot / hashing kernels
struct SnapArgs {
  const uint32_t* pop;   // this rank's rows
  const uint32_t* pool;  // every rank's rows [R][nv][Wp] (elitist column lookup)
  uint32_t* elit;
  uint32_t* ever;
  DevCtl* ctl;
  unsigned long long* h1;
  unsigned long long* h2;
  uint64_t nv;
  uint32_t n, Wp;
};

// The truth-table kernel's dynamically claimed batches are spread over
// kTailCounters counters, each on its own 128-byte line: one counter would
// serialise every warp's claim at the end of the static share (~1 ns per
// same-address atomic, thousands of warps).
constexpr uint32_t kTailCounters = 16;
constexpr uint32_t kTailStride = 32;

struct GomArgs {
  const int32_t* row_ptr;
  const int32_t* col;
  const double* w;
  const int32_t* wi;
  const int64_t* set_off;
  const uint32_t* set_vars;
  const int64_t* fp_off;
  const FpEntry* fp;
  const uint32_t* gsets;  // this group's members (ascending set ids)
  const uint32_t* gvars;  // singleton FOS: the variable of each member
  const uint4* gmeta;     // general FOS: {set id, vars offset, footprint offset, f << 24 | footprint}
  const uint4* urec;       // truth-table plan records of this group (gom_univ_tt_kernel)
  const ulonglong2* ukey;  // Zobrist keys of this group's variables
  const uint4* uvr;        // univariate plan records of this group (gom_univ_f64_kernel)
  uint32_t wbits;         // bit-planes of max |w| (integer path)
  uint32_t G;             // |G|
  uint32_t* pop;
  const double* fit;
  const unsigned long long* h1;
  const unsigned long long* h2;
  uint32_t* elit;  // copy-on-write snapshot of the elitist genotype
  uint32_t* ever;  // per-row snapshot version
  long long* dfit;       // fixed-point fitness deltas: round(delta * fix_scale), summed by atomics
  double fix_scale;      // 1 for integer weights, 2^S for float weights
  unsigned long long* dh1;
  unsigned long long* dh2;
  DevCtl* ctl;
  const int32_t* tape;  // replay donors, p-major [p*n + s]; nullptr -> Philox
  int32_t* rec_donor;   // optional GroupBatch recording, p-major
  double* rec_delta;
  uint8_t* rec_present;
  uint8_t* rec_accept;
  uint32_t n, Wp, team_warps, stage_words;  // n: this rank's solutions, Wp: words per row per rank
  const uint32_t* pool;  // all ranks' rows, rank-major [R][nv][Wp] (== pop when R == 1)
  const uint32_t* ones;  // sharded univariate runs: members holding 1 per row over all ranks (else nullptr)
  uint64_t nv;
  uint32_t R, rank, n_global;
  int32_t exact;
  uint32_t generation;
  uint64_t seed;
  EpiArgs epi;         // run by the last CTA
  unsigned int* chunk_done;  // truth-table rows in chunks: per-chunk CTA tickets
  unsigned int* tail;        // truth-table kernel: counters of the dynamically claimed batches,
                             // kTailCounters per set (kTailStride words apart)
  uint32_t tail_per_chunk;   // ... one set per chunk (rows in chunks) or one per launch
  double* word_max;          // ... and per-word maxima written by each chunk's last CTA
  int32_t slot;                 // >= 0: group = order[slot] (graph path)
  uint32_t exp_flags;           // latency studies only (GOMIX_EXP env): 32 = %globaltimer probes
  const uint32_t* order;
  const GroupDesc* groups;
};

// Forced-improvement phase (gom_fi.cu)
struct FiArgs {
  uint32_t* pop;
  double* fit;
  unsigned long long* h1;
  unsigned long long* h2;
  double* fit_start;  // generation start
  unsigned long long* h1s;
  unsigned long long* h2s;
  int32_t* stag;      // generations without strict improvement (SerialEngine::stagnation_)
  uint8_t* flag;      // triggered this generation
  double* fit0;       // fitness at the start of the pass
  uint32_t* mask;     // Wp words: still in the pass after every group
  const DevCtl* ctl;
  const uint32_t* gsets;
  const int64_t* set_off;
  const uint32_t* set_vars;
  uint64_t nv;
  uint32_t n, Wp;
  int32_t threshold;  // 1 + floor(log10 n) (engine_serial.hpp:153-155)
};

// Run-wide best of an IMS run (ImsDriver::best_, ims.hpp:98-99), device-resident.
struct ImsBestDev {
  double fit;
  double pending;
  int32_t valid;
  int32_t flag;  // decision of the last collect / offer (consumed by its copy kernel)
};

struct OrderArgs {
  DevCtl* ctl;
  uint32_t* order;
  uint32_t k;
  uint64_t seed;
};

// Persistent generation kernel (gom_gen.cu)
constexpr uint32_t kGenMaxN = 256;  // members kept in shared memory by every CTA
constexpr uint32_t kGenMaxK = 256;  // colour groups
constexpr uint32_t kAccStride = 32;  // persistent kernel accumulators: one per 256-byte line
struct BeginArgs {
  DevCtl* ctl;
  int32_t has_budget, has_target, exact;
  double max_evals, q, target;
  unsigned long long calls_before;
  uint32_t gen;  // host generation (direct path keeps the device counter in step)
};
struct GenArgs {
  BeginArgs begin;  // by value: the persistent kernel is launched directly, never captured
  uint32_t k;
  uint32_t* order;             // this generation's group order (written back for inspection)
  long long* dfit;             // [3][n] fitness deltas
  unsigned long long* dh;      // [3][2][n] Zobrist deltas
  unsigned long long* cnt;     // [3][2] steps, calls
  unsigned int* bar;           // grid barrier: flat monotonic counter at word 1536 (two-level layout below it for GOMIX_GEN_TWO_LEVEL A/B builds)
};

// BeginArgs (above): per-call control values, passed as kernel parameters
// (captured at launch, so host calls can be queued back to back without host
// syncs) or read in place from mapped host memory by the graph's begin kernel.

// -------------------------------------------------------------------------
// errors
// -------------------------------------------------------------------------
struct GomixError : std::runtime_error {
  int status;
  GomixError(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define GOMIX_CUDA(call)                                                              \
  do {                                                                                \
    cudaError_t err__ = (call);                                                       \
    if (err__ != cudaSuccess)                                                         \
      throw ::gomix_b200::GomixError(err__ == cudaErrorMemoryAllocation ? GOMIX_E_OOM \
                                                                        : GOMIX_E_CUDA, \
                                     std::string(#call) + ": " + cudaGetErrorString(err__)); \
  } while (0)

inline void invalid(const std::string& m) { throw GomixError(GOMIX_E_INVALID, m); }

// Process-wide caching device allocator (problem.cu): blocks go back to a
// per-device free list instead of cudaFree (which synchronises the device
// and, for large blocks, costs milliseconds), so repeated problem / engine
// builds of similar sizes reuse memory.  Callers synchronise before freeing
// (the cache does not track stream use).  Sizes are rounded up (1 MiB
// granules above 1 MiB, powers of two below); at most 8 GiB stay cached.
void* cached_malloc(size_t bytes);
void cached_free(void* p);
void cached_free_all(std::vector<void*>& blocks);

template <typename T>
T* dev_alloc(std::vector<void*>& owner, size_t count) {
  if (count == 0) count = 1;
  void* p = cached_malloc(count * sizeof(T));
  owner.push_back(p);
  return static_cast<T*>(p);
}

// -------------------------------------------------------------------------
// Host replay stream: the reference's RngStream = std::mt19937_64 seeded with
// mix64(seed) (rng.hpp:11-63).  std::mt19937_64 is pinned by the C++ standard.
// -------------------------------------------------------------------------
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

class ReplayStream {
 public:
  explicit ReplayStream(uint64_t seed) : gen_(mix64(seed)) {}
  uint64_t next() { return gen_(); }
  // Lemire-free rejection draw identical to rng.hpp:28-35.
  uint64_t uniform_index(uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
      const uint64_t r = gen_();
      if (r >= threshold) return r % n;
    }
  }
  void permutation(std::vector<uint64_t>& out, uint64_t n) {
    out.resize(n);
    for (uint64_t i = 0; i < n; ++i) out[i] = i;
    for (uint64_t i = n; i > 1; --i) std::swap(out[i - 1], out[uniform_index(i)]);
  }

 private:
  std::mt19937_64 gen_;
};

// kernel launchers (gom.cu)
void launch_gom(const GomArgs& a, bool univariate, bool i32, int wpt, bool team, int grid, int block,
                size_t smem, cudaStream_t s);
// persistent generation kernel (gom_gen.cu)
int gen_kernel_max_blocks(int wpt, bool team, int block, size_t smem, bool lean);
int gen_lean_smem();  // dynamic shared memory of a lean launch (8 warps)
void launch_generation_kernel(const GomArgs& a, const GenArgs& ga, int wpt, bool team, int grid, int block,
                              size_t smem, cudaStream_t s, bool lean);
// bit-sliced univariate kernel (gom_univ.cu)
int univ_sliced_planes(uint64_t max_abs_row_sum);  // 0: not representable
int univ_sliced_block();
int univ_sliced_sets_per_cta();
int univ_sliced_max_blocks_per_sm(int planes, int wp, bool tt);
void launch_univ_sliced(const GomArgs& a, int planes, int wp, bool tt, int grid, cudaStream_t s,
                        bool pdl = false);
void build_univ_records(Problem& P);
// float univariate kernel (gom_univ_f64.cu)
void build_univ_plan(Problem& P);
int univ_f64_max_blocks_per_sm(int wp);
int univ_f64_sets_per_cta();
int univ_f64_max_degree();
void launch_univ_f64(const GomArgs& a, int wp, int grid, cudaStream_t s, bool pdl = false);
void build_csr_device(Problem& P, bool exact, int32_t* d_eid, uint64_t* max_abs_row);  // problem.cu
void launch_fi_snapshot(const FiArgs& a, cudaStream_t s);
void launch_fi_flags(const FiArgs& a, bool given, cudaStream_t s);
void launch_fi_tape(const FiArgs& a, uint64_t g0, uint64_t G, int32_t* tape, cudaStream_t s);
void launch_fi_finish(const FiArgs& a, bool update_stag, cudaStream_t s);  // truth-table plan records (urec, ukey) of a degree <= 4 univariate FOS
int gom_max_blocks_per_sm(bool univariate, bool i32, int wpt, bool team, int block, size_t smem);
void launch_begin(const BeginArgs& b, cudaStream_t s);
void launch_order(const BeginArgs* d_b, const OrderArgs& o, cudaStream_t s);
void prepare_gom(bool univariate, bool i32, int wpt, bool team, size_t smem);
void launch_init_epilogue(const EpiArgs& a, cudaStream_t s);
void launch_global_epilogue(const EpiArgs& a, cudaStream_t s);
void launch_publish_ctl(const void* ctl, void* host_dst, size_t bytes, unsigned long long* host_seq,
                        unsigned long long seq, cudaStream_t s);
void launch_hash_population(const SnapArgs& a, cudaStream_t s);
void launch_finalize_elitist(const SnapArgs& a, cudaStream_t s);
void launch_external_elitist(const SnapArgs& a, double fitness, cudaStream_t s);
void launch_ims_collect(const SnapArgs& a, ImsBestDev* b, uint32_t* bits, int exact, cudaStream_t s);
void launch_ims_offer(const SnapArgs& a, ImsBestDev* b, const uint32_t* bits, int exact, cudaStream_t s);
void launch_count_ones(const uint32_t* pop, uint64_t nv, uint32_t Wp, uint32_t* ones, cudaStream_t s);
// peer transport (gom_peer.cu / gom_peer.cuh)
size_t peer_block_bytes(uint32_t R, uint32_t n, uint32_t w32);
void launch_peer_exchange(const EpiArgs& a, cudaStream_t s);
void launch_presence(const PeerArgs* d_peer, DevCtl* ctl, const uint32_t* pop, uint64_t nv, uint32_t Wp,
                     uint32_t n_local, uint32_t n_global, uint32_t* ones, cudaStream_t s);
void launch_peer_elitist(const PeerArgs* d_peer, DevCtl* ctl, uint32_t* elit, uint64_t nv, bool owner,
                        unsigned long long epoch, cudaStream_t s);
void launch_sum_ones(const uint32_t* stage, uint32_t R, uint64_t nv, uint32_t* ones, cudaStream_t s);
void debug_probes(unsigned long long* out, bool reset);
void debug_probes_gen(unsigned long long* out, bool reset);
void debug_gen_timeline(unsigned long long* out);
void debug_probes_univ(unsigned long long* out, bool reset);
void debug_timeline_univ(unsigned long long* out);  // gom_univ_tt_kernel launch timeline (probes builds), 4 x 32
void debug_timeline_gom(unsigned long long* out);   // begin_generation_kernel (points 0, 1), 32
void debug_cta_stats_univ(unsigned long long* out);  // per-CTA stats of the tt launches, 4 x 1024 x 4
void debug_cta_probes(unsigned long long* out);
void launch_philox_init(uint32_t* pop, uint64_t nv, uint32_t n, uint32_t Wp, uint64_t seed,
                        uint32_t rank, cudaStream_t s);
void launch_full_eval(const Problem& P, const uint32_t* pop, double* fit, uint32_t n,
                      uint32_t Wp, bool ordered, cudaStream_t s);
void launch_unpack(const uint32_t* pop, uint8_t* out, uint64_t nv, uint32_t n, uint32_t Wp,
                   cudaStream_t s);
void launch_pack(const uint8_t* in, uint32_t* pop, uint64_t nv, uint32_t n, uint32_t Wp,
                 cudaStream_t s);
void launch_pack_elitist(const uint8_t* in, uint32_t* elit, uint64_t nv, cudaStream_t s);
void launch_unpack_elitist(const uint32_t* elit, uint8_t* out, uint64_t nv, cudaStream_t s);


}  // namespace gomix_b200
