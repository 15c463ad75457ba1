/*
 * gomix_gpu.h — C-ABI of the B200-native parallel Gene-pool Optimal Mixing
 * engine (libgomix_b200.so).  Plain pointers and sizes only.
 *
 * It replaces the hot path of the reference's header-only C++ library
 * (`gomix`, proj/include/gomix/), split the way the reference splits it:
 *
 *   gomix_gpu_problem  ~ the immutable, shared model of a run:
 *                        MaxCutInstance + as_graybox   (maxcut.hpp:21-79)
 *                        Fos                            (linkage.hpp:124-131)
 *                        build_vig/build_lmig/welsh_powell -> ColorGroups
 *                                                       (graybox.hpp:305-323,
 *                                                        scheduling.hpp:35-114)
 *                        make_group_plan per group      (engine_parallel.hpp:37-59)
 *                        = ModelArtifacts shared by every population
 *                                                       (model.hpp:25-29, run.hpp:110)
 *   gomix_gpu_engine   ~ one population: ParallelEngine (engine_parallel.hpp:255-368)
 *                        with its GenerationRunner face (ims.hpp:14-22).
 *
 * Every entry point returns a gomix_status; on failure a message is available
 * from gomix_gpu_last_error() (thread-local).  Host arrays passed in are
 * caller-owned and copied during the call; read-backs write into caller
 * buffers.  All device work of a handle is ordered on that handle's stream.
 */
#ifndef GOMIX_GPU_H
#define GOMIX_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GOMIX_GPU_ABI_VERSION 1

#if defined(__GNUC__)
#define GOMIX_API __attribute__((visibility("default")))
#else
#define GOMIX_API
#endif

typedef enum {
  GOMIX_OK = 0,
  GOMIX_E_INVALID = 1, /* std::invalid_argument in the reference (engine_parallel.hpp:266-270) */
  GOMIX_E_CUDA = 2,
  GOMIX_E_NCCL = 3,
  GOMIX_E_OOM = 4,
  GOMIX_E_STATE = 5 /* std::logic_error: call out of order */
} gomix_status;

typedef enum {
  /* Deterministic replay: population init, group order and every donor are
   * drawn from the reference's own RngStream(seed) (rng.hpp:21-63) in the
   * reference's order, so populations match ParallelEngine bit for bit. */
  GOMIX_MODE_REPLAY = 0,
  /* Production: donors drawn on the device from a counter-based Philox4x32-10
   * stream keyed by the seed; same donor distribution (uniform over members
   * that differ on the set, engine_serial.hpp:26-46), no host round trips. */
  GOMIX_MODE_PHILOX = 1
} gomix_mode;

enum {
  /* Float weights: accumulate fitness in the reference's order (positions
   * ascending per solution, engine_parallel.hpp:230-236) instead of a
   * deterministic tree; bit-identical to the reference.  Default in REPLAY. */
  GOMIX_FLAG_ORDERED_FLOAT = 1u << 0,
  /* Keep each group's GroupBatch arrays (donor/delta/present/accept) for
   * gomix_gpu_read_batch (engine_parallel.hpp:64-97). */
  GOMIX_FLAG_RECORD_BATCH = 1u << 1,
  /* Time every GOM kernel launch with CUDA events (gomix_gpu_kernel_times). */
  GOMIX_FLAG_TIME_KERNELS = 1u << 2,
  /* Univariate FOS, integer weights, PHILOX: use the lane-per-solution kernel
   * instead of the bit-sliced lane-per-set kernel (same results; A/B tests). */
  GOMIX_FLAG_LANE_PER_SOLUTION = 1u << 3,
  /* General sets, integer weights, PHILOX, n <= 256: run one kernel launch
   * per colour group instead of the persistent whole-generation kernel
   * (same results; A/B tests). */
  GOMIX_FLAG_PER_GROUP_KERNELS = 1u << 4,
  /* Univariate FOS of degree <= 4: use the adder/comparator bit-sliced kernel
   * instead of the truth-table one (same results; A/B tests). */
  GOMIX_FLAG_NO_TRUTH_TABLE = 1u << 5,
  /* Parallel-friendly Forced Improvement after every generation (single GPU):
   * triggered solutions take the elitist as donor group by group, halt after
   * the first group that strictly improved them, else become elitist copies
   * (engine_serial.hpp:98-128 restated group-wise; see gom_fi.cu). */
  GOMIX_FLAG_FORCED_IMPROVEMENT = 1u << 6,
  /* Sharded engines (world_size > 1), univariate variable-once FOS: exchange
   * over peer memory instead of NCCL — the last CTA of every GOM launch
   * publishes its members into every rank's exchange block and runs the
   * global elitist scan itself (gom_peer.cuh).  Each rank exports its block
   * (gomix_gpu_peer_export) and maps everyone's (gomix_gpu_peer_connect)
   * before gomix_gpu_init_population; no NCCL id is needed. */
  GOMIX_FLAG_PEER_TRANSPORT = 1u << 7
};

enum { GOMIX_STOP_NONE = 0, GOMIX_STOP_BUDGET = 1, GOMIX_STOP_CLOCK = 2, GOMIX_STOP_TARGET = 3,
       GOMIX_STOP_GENERATION_LIMIT = 4 }; /* runtime.hpp:31-37 */

/* MaxCutInstance (maxcut.hpp:21-37): canonical edges u < v, sorted by (u, v),
 * unique; one subfunction per edge with value w*[x_u != x_v] (maxcut.hpp:67-79).
 * Integer weights (all w integral, |w| <= 9e15) select the exact comparator
 * (graybox.hpp:22-35, maxcut.hpp:32-36). */
typedef struct {
  uint64_t num_vertices;
  uint64_t num_edges;
  const uint32_t* edge_u;
  const uint32_t* edge_v;
  const double* edge_w;
} gomix_maxcut;

/* Fos::sets (linkage.hpp:124-131) in CSR form; each set sorted, unique. */
typedef struct {
  uint64_t num_sets;
  const uint64_t* set_offset; /* num_sets + 1 */
  const uint32_t* set_vars;
} gomix_fos;

typedef struct {
  uint64_t num_vertices, num_edges, num_sets, num_groups, lmig_edges, max_set_size;
  int32_t exact;      /* integer weights -> exact comparator */
  int32_t univariate; /* every set is a singleton */
} gomix_problem_info;

typedef struct gomix_gpu_problem gomix_gpu_problem;
typedef struct gomix_gpu_engine gomix_gpu_engine;
typedef struct gomix_gpu_local_group gomix_gpu_local_group;
typedef struct gomix_gpu_ims_best gomix_gpu_ims_best;

/* EngineConfig (engine_serial.hpp:18-24). */
typedef struct {
  uint64_t population_size;
  uint64_t seed;
  uint32_t mode;  /* gomix_mode */
  uint32_t flags; /* GOMIX_FLAG_* */
  int32_t population_id; /* reporting only (engine_parallel.hpp:258) */
  /* Sharding of the population over GPUs (Philox mode).  world_size 1 = one
   * GPU.  With world_size R > 1 rank r holds members [r*n/R, (r+1)*n/R)
   * (population_size is the GLOBAL n, divisible by R); after every group the
   * bit-packed rows (the next group's donor pool), fitness, hashes and
   * counters are all-gathered, and every rank takes the same elitist / stop
   * decisions.  Results equal a single-GPU run of the same n and seed.
   * One process per GPU: every rank passes the same 128-byte NCCL unique id
   * (gomix_gpu_nccl_unique_id on one rank, then broadcast by the caller).
   * Several shards in one process: gomix_gpu_local_group_*. */
  int32_t rank, world_size;
  const void* nccl_unique_id;
} gomix_engine_config;

/* Termination criteria evaluated after every group, in the reference's order:
 * evaluation budget first (RunControl::add_evaluator_calls, runtime.hpp:75-80),
 * then the target via each elitist improvement (runtime.hpp:88-93,136-143).
 * evaluator_calls_before is the shared run-wide count when the call starts. */
typedef struct {
  int32_t has_max_evaluations;
  double max_evaluations; /* gray-box units: calls / num_edges */
  uint64_t evaluator_calls_before;
  int32_t has_target;
  double target_fitness;
} gomix_stop_criteria;

typedef struct {
  uint64_t groups_run;
  uint64_t steps;           /* executed (solution, set) pairs = partial evaluations */
  uint64_t evaluator_calls; /* subfunction evaluations (GroupCounter, runtime.hpp:170-175) */
  int32_t stopped;
  int32_t stop_reason;
  uint64_t improvements;    /* elitist improvements recorded (read with read_improvements) */
  double elitist_fitness;
} gomix_run_stats;

/* ---- problem (shared model) ------------------------------------------------ */

/* Builds the device CSR graph, the FOS, the LMIG and its Welsh-Powell colouring
 * (on the GPU, exact), the colour groups and their footprint plans.
 * set_colour != NULL adopts a prebuilt ColorGroups (engine_parallel.hpp:271-272)
 * given as one colour per set. device < 0 uses the current device. */
GOMIX_API int gomix_gpu_problem_create(const gomix_maxcut* instance, const gomix_fos* fos,
                             const int32_t* set_colour, int32_t device,
                             gomix_gpu_problem** out);
GOMIX_API int gomix_gpu_problem_destroy(gomix_gpu_problem* p);
GOMIX_API int gomix_gpu_problem_info(const gomix_gpu_problem* p, gomix_problem_info* out);
/* ColorGroups (scheduling.hpp:72-81): group c = group_sets[group_offset[c] .. group_offset[c+1]),
 * members ascending.  group_offset has num_groups + 1 entries. */
GOMIX_API int gomix_gpu_problem_groups(const gomix_gpu_problem* p, uint64_t* group_offset,
                             uint64_t* group_sets);
/* Per set footprint size = number of dependent subfunctions (GroupPlan::footprint). */
GOMIX_API int gomix_gpu_problem_footprints(const gomix_gpu_problem* p, uint64_t* footprint);

/* ---- engine (one population) ----------------------------------------------- */

GOMIX_API int gomix_gpu_engine_create(gomix_gpu_problem* p, const gomix_engine_config* cfg,
                            gomix_gpu_engine** out);
GOMIX_API int gomix_gpu_engine_destroy(gomix_gpu_engine* e);
/* Use an external CUDA stream (cudaStream_t) for all later work; NULL = own stream. */
GOMIX_API int gomix_gpu_set_stream(gomix_gpu_engine* e, void* cuda_stream);

/* init_population (engine_parallel.hpp:331-346).  genotypes (n x num_vertices
 * bytes, row per solution) may be NULL: REPLAY draws them from RngStream(seed)
 * like the reference, PHILOX draws them on the device.  Reports n*q evaluator
 * calls and the initial elitist chain like the reference. */
GOMIX_API int gomix_gpu_init_population(gomix_gpu_engine* e, const uint8_t* genotypes,
                              const gomix_stop_criteria* stop, gomix_run_stats* out);

/* run_generation (engine_parallel.hpp:283-316): permutes the groups and runs one
 * batched GOM step per group, stopping after the first group at which a stop
 * criterion fires.  The generation counter advances only if every group ran. */
GOMIX_API int gomix_gpu_run_generation(gomix_gpu_engine* e, const gomix_stop_criteria* stop,
                             gomix_run_stats* out);

/* Philox mode, no stop criteria: enqueue one generation on the engine's
 * stream and return without synchronising (for back-to-back generations and
 * CUDA-event timing).  gomix_gpu_synchronize waits and returns the stats of
 * the last queued generation. */
GOMIX_API int gomix_gpu_run_generation_async(gomix_gpu_engine* e);
GOMIX_API int gomix_gpu_synchronize(gomix_gpu_engine* e, gomix_run_stats* out);

/* Replace the population with n x num_vertices genotype bytes and their
 * fitness (NULL = evaluate on the device); the elitist is kept. */
GOMIX_API int gomix_gpu_load_population(gomix_gpu_engine* e, const uint8_t* genotypes,
                                        const double* fitness);

/* One batched GOM step over colour group `group` (phases 1-4 of
 * engine_parallel.hpp:104-247 plus the elitist scan :305-310) with the donors
 * given as a GroupBatch::donor array (s*|G| + p order, -1 = no donor).
 * donor_tape == NULL draws donors with the engine's mode. */
GOMIX_API int gomix_gpu_run_group(gomix_gpu_engine* e, uint64_t group, const int32_t* donor_tape,
                        const gomix_stop_criteria* stop, gomix_run_stats* out);

/* One Forced-Improvement pass now (see GOMIX_FLAG_FORCED_IMPROVEMENT) over the
 * solutions with flags[s] != 0 (flags NULL: the engine's own trigger —
 * unchanged genotype or stagnation since the last generation started), the
 * colour groups in group_order (k entries; NULL: a fresh permutation from the
 * engine's stream).  Counts toward the run's evaluator calls and stop
 * criteria like a generation's groups.  Single-GPU engines. */
GOMIX_API int gomix_gpu_forced_improvement(gomix_gpu_engine* e, const uint8_t* flags, const uint32_t* group_order,
                                           const gomix_stop_criteria* stop, gomix_run_stats* out);

/* Last group's GroupBatch arrays, each n*|G| in s*|G| + p order (needs
 * GOMIX_FLAG_RECORD_BATCH).  Any pointer may be NULL. */
GOMIX_API int gomix_gpu_read_batch(gomix_gpu_engine* e, int32_t* donor, double* delta, uint8_t* present,
                         uint8_t* accept);

/* population() (engine_parallel.hpp:324): genotypes as n x num_vertices bytes. */
GOMIX_API int gomix_gpu_read_population(gomix_gpu_engine* e, uint8_t* genotypes, double* fitness);
/* Raw device layout: num_vertices rows of words_per_var uint32 words; bit b of
 * word w of row v is variable v of solution 32*w + b (local solutions). */
GOMIX_API int gomix_gpu_read_population_packed(gomix_gpu_engine* e, uint32_t* words,
                                     uint64_t* words_per_var);
GOMIX_API int gomix_gpu_read_elitist(gomix_gpu_engine* e, uint8_t* genotype, double* fitness);
/* offer_elitist (engine_parallel.hpp:320-322): adopt iff strictly better. */
GOMIX_API int gomix_gpu_offer_elitist(gomix_gpu_engine* e, const uint8_t* genotype, double fitness,
                            int32_t* adopted);
/* Elitist improvements of the last init/run call, in report order: fitness
 * and the run-wide evaluator-call count at the moment of the report (what the
 * reference's TraceSink row records, runtime.hpp:136-143).  Either array may
 * be NULL; with both NULL, count = number available. */
GOMIX_API int gomix_gpu_read_improvements(gomix_gpu_engine* e, double* fitness,
                                          uint64_t* evaluator_calls, uint64_t capacity,
                                          uint64_t* count);
/* group_counters() (engine_parallel.hpp:326-328). */
GOMIX_API int gomix_gpu_group_counters(gomix_gpu_engine* e, uint64_t* sets, uint64_t* steps,
                             uint64_t* evaluator_calls);
GOMIX_API int gomix_gpu_generation(gomix_gpu_engine* e, int64_t* generation);
/* Durations (ms) of the GOM kernel launches since the last call (needs
 * GOMIX_FLAG_TIME_KERNELS); count = number written. */
GOMIX_API int gomix_gpu_kernel_times(gomix_gpu_engine* e, float* ms, uint64_t capacity, uint64_t* count);
/* Turn GOMIX_FLAG_TIME_KERNELS on or off.  While on, generations are issued
 * launch by launch (events around every GOM kernel) instead of as one CUDA
 * graph. */
GOMIX_API int gomix_gpu_set_timing(gomix_gpu_engine* e, int32_t enable);
/* Name of the GOM kernel this engine's Philox generations launch
 * ("gom_univ_sliced_kernel" or "gom_group_kernel"); static storage. */
GOMIX_API const char* gomix_gpu_engine_kernel_name(const gomix_gpu_engine* e);
/* Number of device kernels this engine has launched so far. */
GOMIX_API int gomix_gpu_launch_count(gomix_gpu_engine* e, uint64_t* count);

/* ---- IMS on the device (ims.hpp:38-101) ---------------------------------------- */

/* The run-wide best solution of an interleaved multistart run
 * (ImsDriver::best_), resident on the problem's device. */
GOMIX_API int gomix_gpu_ims_best_create(gomix_gpu_problem* p, gomix_gpu_ims_best** out);
GOMIX_API int gomix_gpu_ims_best_destroy(gomix_gpu_ims_best* b);
/* ImsDriver::collect (ims.hpp:89-95): best = e's elitist if strictly better
 * (or no best yet).  Queued on e's stream, no host synchronisation; every
 * collect / offer on the same best is ordered after the previous one. */
GOMIX_API int gomix_gpu_ims_collect(gomix_gpu_ims_best* b, gomix_gpu_engine* e);
/* runner->offer_elitist(best_) (ims.hpp:83, engine_parallel.hpp:320-322): e
 * adopts the best iff strictly better than its elitist.  Queued, no sync. */
GOMIX_API int gomix_gpu_ims_offer(gomix_gpu_ims_best* b, gomix_gpu_engine* e);
/* Waits for the queued exchanges; genotype (num_vertices bytes) may be NULL. */
GOMIX_API int gomix_gpu_ims_best_read(gomix_gpu_ims_best* b, uint8_t* genotype, double* fitness,
                                      int32_t* valid);

/* ---- multi-GPU sharding ------------------------------------------------------ */

/* 128-byte NCCL unique id for gomix_engine_config.nccl_unique_id (NCCL is
 * loaded at run time: the process's libnccl.so.2, e.g. PyTorch's). */
GOMIX_API int gomix_gpu_nccl_unique_id(uint8_t* id);

#define GOMIX_PEER_HANDLE_BYTES 64
/* GOMIX_FLAG_PEER_TRANSPORT: allocate this rank's exchange block and return
 * its CUDA IPC handle (GOMIX_PEER_HANDLE_BYTES) for the other ranks. */
GOMIX_API int gomix_gpu_peer_export(gomix_gpu_engine* e, uint8_t* handle);
/* Map every rank's block (handles: world_size x GOMIX_PEER_HANDLE_BYTES in
 * rank order, this rank's own entry ignored); then init_population. */
GOMIX_API int gomix_gpu_peer_connect(gomix_gpu_engine* e, const uint8_t* handles);
/* In-process shards: world_size engines (problems[r] on the device of rank r;
 * the same problem may serve several ranks on one device) driven in lock step
 * by one host thread; the exchange is device-to-device copies. */
GOMIX_API int gomix_gpu_local_group_create(gomix_gpu_problem* const* problems,
                                           const gomix_engine_config* cfg,
                                           gomix_gpu_local_group** out);
GOMIX_API int gomix_gpu_local_group_destroy(gomix_gpu_local_group* g);
/* rank r's engine: read its shard with gomix_gpu_read_population / counters */
GOMIX_API int gomix_gpu_local_group_engine(gomix_gpu_local_group* g, int32_t rank,
                                           gomix_gpu_engine** out);
GOMIX_API int gomix_gpu_local_group_init_population(gomix_gpu_local_group* g,
                                                    const gomix_stop_criteria* stop,
                                                    gomix_run_stats* out);
GOMIX_API int gomix_gpu_local_group_run_generation(gomix_gpu_local_group* g,
                                                   const gomix_stop_criteria* stop,
                                                   gomix_run_stats* out);
GOMIX_API int gomix_gpu_local_group_read_elitist(gomix_gpu_local_group* g, uint8_t* genotype,
                                                 double* fitness);

/* ---- synthetic instances (host only) ------------------------------------------ */

/* generate_torus (maxcut.hpp:87-147): 2*width*height canonical edges written to
 * eu/ev/ew.  weight_kind 0 = unit, 1 = uniform_int[lo, hi]; same RngStream and
 * draw order as the reference, so the instance is identical. */
GOMIX_API int gomix_generate_torus(uint64_t width, uint64_t height, int32_t weight_kind, int64_t lo,
                         int64_t hi, uint64_t seed, uint32_t* eu, uint32_t* ev, double* ew);
/* Random simple d-regular graph, num_vertices*degree/2 canonical edges.
 * weight_kind 0 unit, 1 uniform_int[lo, hi], 2 uniform_real [0, 1). */
GOMIX_API int gomix_generate_regular(uint64_t num_vertices, uint32_t degree, int32_t weight_kind, int64_t lo,
                           int64_t hi, uint64_t seed, uint32_t* eu, uint32_t* ev, double* ew);

/* ---- linkage model (host only) -------------------------------------------------- */

/* build_fixed_model's FOS (model.hpp:31-52): learn_tree_upgma (linkage.hpp:
 * 133-264) over vig_similarity (weighted = 0: 1 per edge) or weight_similarity
 * (weighted != 0: |w| per edge), size bound `bound` (0 = unbounded FLT),
 * computed without the n x n matrix (sparse similarity, O((n+q) log n)).
 * Same sets in the same order as the reference: singletons in variable
 * order, then merged sets in merge order, the full set never emitted.
 * With set_offset or set_vars NULL only num_sets and total_vars are returned;
 * otherwise set_offset holds num_sets + 1 entries and set_vars total_vars. */
GOMIX_API int gomix_fos_bounded_flt(uint64_t num_vertices, uint64_t num_edges, const uint32_t* edge_u,
                                    const uint32_t* edge_v, const double* edge_w, uint64_t bound,
                                    int32_t weighted, uint64_t* num_sets, uint64_t* total_vars,
                                    uint64_t* set_offset, uint32_t* set_vars);

/* ---- misc ------------------------------------------------------------------- */

/* Standalone GPU colouring (the color-stats path, gomix_main.cpp:319-351). */
GOMIX_API int gomix_gpu_color(const gomix_maxcut* instance, const gomix_fos* fos, int32_t device,
                    int32_t* set_colour, uint64_t* num_groups, uint64_t* lmig_edges);
GOMIX_API const char* gomix_gpu_last_error(void);
GOMIX_API int gomix_gpu_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GOMIX_GPU_H */
