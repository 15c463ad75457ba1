/*
 * gomix_oracle.c — CPU restatement of the reference's parallel GOM path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * engine: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product path (libgomix_b200.so) never
 * links or calls it.
 *
 * It restates, in plain C11, the algorithm of the reference header-only C++
 * library `gomix` (read-only at /root/reference/proj/include/gomix/).  Every
 * function cites the reference file:line it follows.  Parity of this
 * restatement is pinned two ways (see tests/test_oracle.py):
 *   1. the reference's own known-answer tests (test_rng.cpp:13-24,
 *      test_scheduling.cpp:84-107, test_engine_parallel.cpp:40-56,163-202);
 *   2. byte-for-byte comparison with the reference itself, compiled from its
 *      headers into oracle/_ref/ref_driver (oracle/ref_driver.cpp), on the
 *      committed golden fixtures under tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))
#define ORC_NPOS ((uint64_t)-1)

/* ------------------------------------------------------------------------- */
/* RNG: mix64 (rng.hpp:11-16) and std::mt19937_64 (pinned by the C++ std,    */
/* rng.hpp:18-20); RngStream seeds it with mix64(seed) (rng.hpp:23).          */
/* ------------------------------------------------------------------------- */

ORC_API uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

enum { MT_N = 312, MT_M = 156 };

typedef struct {
  uint64_t s[MT_N];
  int i;
} orc_mt64;

ORC_API void orc_mt_seed(orc_mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int k = 1; k < MT_N; ++k)
    g->s[k] = 6364136223846793005ull * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
  g->i = MT_N;
}

static void mt_twist(orc_mt64* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
  for (int k = 0; k < MT_N; ++k) {
    const uint64_t y = (g->s[k] & upper) | (g->s[(k + 1) % MT_N] & lower);
    uint64_t v = g->s[(k + MT_M) % MT_N] ^ (y >> 1);
    if (y & 1) v ^= 0xB5026F5AA96619E9ull;
    g->s[k] = v;
  }
  g->i = 0;
}

ORC_API uint64_t orc_mt_next(orc_mt64* g) {
  if (g->i >= MT_N) mt_twist(g);
  uint64_t y = g->s[g->i++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* RngStream(seed): generator seeded with mix64(seed) (rng.hpp:23). */
ORC_API void orc_stream_init(orc_mt64* g, uint64_t seed) { orc_mt_seed(g, orc_mix64(seed)); }

/* Unbiased rejection draw in [0, n) (rng.hpp:28-35). */
ORC_API uint64_t orc_uniform_index(orc_mt64* g, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t r = orc_mt_next(g);
    if (r >= threshold) return r % n;
  }
}

/* Back-to-front Fisher-Yates over iota(n) (rng.hpp:49-59). */
ORC_API void orc_permutation(orc_mt64* g, uint64_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = i;
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = orc_uniform_index(g, i);
    const uint64_t t = out[i - 1];
    out[i - 1] = out[j];
    out[j] = t;
  }
}

ORC_API size_t orc_mt_state_size(void) { return sizeof(orc_mt64); }

/* ------------------------------------------------------------------------- */
/* Max-Cut torus generator (maxcut.hpp:87-147).                              */
/* weight kind 0 = unit (1.0), 1 = uniform_int[lo,hi] drawn per edge in      */
/* generation order (right edge, then down edge), then edges sorted (u,v).   */
/* ------------------------------------------------------------------------- */

typedef struct {
  uint32_t u, v;
  double w;
} orc_edge;

static int edge_cmp(const void* a, const void* b) {
  const orc_edge* x = (const orc_edge*)a;
  const orc_edge* y = (const orc_edge*)b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return 0;
}

ORC_API int orc_generate_torus(uint64_t width, uint64_t height, int weight_kind, int64_t lo,
                               int64_t hi, uint64_t seed, uint32_t* eu, uint32_t* ev,
                               double* ew) {
  if (width < 3 || height < 3) return -1;
  if (weight_kind == 1 && lo > hi) return -2;
  orc_mt64 rng;
  orc_stream_init(&rng, seed);
  const uint64_t nv = width * height, q = 2 * nv;
  orc_edge* e = (orc_edge*)malloc(q * sizeof(orc_edge));
  uint64_t k = 0;
  for (uint64_t r = 0; r < height; ++r) {
    for (uint64_t c = 0; c < width; ++c) {
      const uint64_t v = r * width + c;
      const uint64_t right = r * width + (c + 1) % width;
      const uint64_t down = ((r + 1) % height) * width + c;
      const uint64_t nb[2] = {right, down};
      for (int t = 0; t < 2; ++t) {
        double w = 1.0;
        if (weight_kind == 1)
          w = (double)(lo + (int64_t)orc_uniform_index(&rng, (uint64_t)(hi - lo) + 1));
        e[k].u = (uint32_t)(v < nb[t] ? v : nb[t]);
        e[k].v = (uint32_t)(v < nb[t] ? nb[t] : v);
        e[k].w = w;
        ++k;
      }
    }
  }
  qsort(e, q, sizeof(orc_edge), edge_cmp);
  for (uint64_t i = 0; i < q; ++i) {
    eu[i] = e[i].u;
    ev[i] = e[i].v;
    ew[i] = e[i].w;
  }
  free(e);
  return 0;
}

/* MaxCutInstance::integer_weights (maxcut.hpp:32-36). */
static int integer_weights(const double* w, uint64_t q) {
  for (uint64_t i = 0; i < q; ++i)
    if (w[i] != floor(w[i]) || fabs(w[i]) > 9e15) return 0;
  return 1;
}

/* ------------------------------------------------------------------------- */
/* Small growable uint64 vector.                                             */
/* ------------------------------------------------------------------------- */
typedef struct {
  uint64_t* a;
  uint64_t n, cap;
} vec64;

static void v_push(vec64* v, uint64_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 8;
    v->a = (uint64_t*)realloc(v->a, v->cap * sizeof(uint64_t));
  }
  v->a[v->n++] = x;
}

static int u64_cmp(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static void v_sort_unique(vec64* v) {
  if (v->n == 0) return;
  qsort(v->a, v->n, sizeof(uint64_t), u64_cmp);
  uint64_t k = 1;
  for (uint64_t i = 1; i < v->n; ++i)
    if (v->a[i] != v->a[k - 1]) v->a[k++] = v->a[i];
  v->n = k;
}

/* ------------------------------------------------------------------------- */
/* Problem view: one subfunction per edge, value w*[x_u != x_v]              */
/* (maxcut.hpp:67-79); var -> subfunctions in ascending edge id              */
/* (graybox.hpp:59-72); VIG adjacency sorted unique (graybox.hpp:305-323).   */
/* ------------------------------------------------------------------------- */
typedef struct {
  uint64_t nv, q;
  const uint32_t* eu;
  const uint32_t* ev;
  const double* ew;
  vec64* subs_of;  /* nv lists of edge ids */
  vec64* vig;      /* nv lists of neighbours */
  int exact;
} orc_problem;

static void problem_build(orc_problem* P, uint64_t nv, uint64_t q, const uint32_t* eu,
                          const uint32_t* ev, const double* ew) {
  P->nv = nv;
  P->q = q;
  P->eu = eu;
  P->ev = ev;
  P->ew = ew;
  P->subs_of = (vec64*)calloc(nv, sizeof(vec64));
  P->vig = (vec64*)calloc(nv, sizeof(vec64));
  for (uint64_t i = 0; i < q; ++i) {
    v_push(&P->subs_of[eu[i]], i);
    v_push(&P->subs_of[ev[i]], i);
    v_push(&P->vig[eu[i]], ev[i]);
    v_push(&P->vig[ev[i]], eu[i]);
  }
  for (uint64_t v = 0; v < nv; ++v) v_sort_unique(&P->vig[v]);
  P->exact = integer_weights(ew, q);
}

static void problem_free(orc_problem* P) {
  for (uint64_t v = 0; v < P->nv; ++v) {
    free(P->subs_of[v].a);
    free(P->vig[v].a);
  }
  free(P->subs_of);
  free(P->vig);
}

/* FitnessComparator (graybox.hpp:22-35). */
static double cmp_scale(double a, double b) {
  double m = 1.0;
  if (fabs(a) > m) m = fabs(a);
  if (fabs(b) > m) m = fabs(b);
  return 1e-9 * m;
}
static int cmp_better(int exact, double a, double b) {
  return exact ? a > b : a - b > cmp_scale(a, b);
}
static int cmp_equal(int exact, double a, double b) {
  return exact ? a == b : fabs(a - b) <= cmp_scale(a, b);
}

/* ------------------------------------------------------------------------- */
/* LMIG (scheduling.hpp:35-68) and Welsh-Powell (scheduling.hpp:85-114).     */
/* Returns the number of colours; colour[i] per set.                         */
/* ------------------------------------------------------------------------- */
static uint64_t g_deg_for_sort_n;
static const uint64_t* g_deg_for_sort;
static int wp_cmp(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  const uint64_t dx = g_deg_for_sort[x], dy = g_deg_for_sort[y];
  if (dx != dy) return dx > dy ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static vec64* build_lmig(const orc_problem* P, uint64_t m, const uint64_t* set_off,
                         const uint32_t* set_vars) {
  vec64* var_sets = (vec64*)calloc(P->nv, sizeof(vec64));
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t k = set_off[i]; k < set_off[i + 1]; ++k) v_push(&var_sets[set_vars[k]], i);
  vec64* adj = (vec64*)calloc(m, sizeof(vec64));
  uint64_t* stamp = (uint64_t*)calloc(m, sizeof(uint64_t));
  uint64_t epoch = 0;
  for (uint64_t i = 0; i < m; ++i) {
    ++epoch;
    stamp[i] = epoch;
    for (uint64_t k = set_off[i]; k < set_off[i + 1]; ++k) {
      const uint64_t u = set_vars[k];
      for (uint64_t t = 0; t < var_sets[u].n; ++t) {
        const uint64_t j = var_sets[u].a[t];
        if (stamp[j] != epoch) { stamp[j] = epoch; v_push(&adj[i], j); }
      }
      for (uint64_t a = 0; a < P->vig[u].n; ++a) {
        const uint64_t x = P->vig[u].a[a];
        for (uint64_t t = 0; t < var_sets[x].n; ++t) {
          const uint64_t j = var_sets[x].a[t];
          if (stamp[j] != epoch) { stamp[j] = epoch; v_push(&adj[i], j); }
        }
      }
    }
    v_sort_unique(&adj[i]);
  }
  for (uint64_t v = 0; v < P->nv; ++v) free(var_sets[v].a);
  free(var_sets);
  free(stamp);
  return adj;
}

static uint64_t welsh_powell(const vec64* adj, uint64_t m, int32_t* colour) {
  uint64_t* deg = (uint64_t*)malloc(m * sizeof(uint64_t));
  uint64_t* order = (uint64_t*)malloc(m * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) { deg[i] = adj[i].n; order[i] = i; }
  g_deg_for_sort = deg;
  g_deg_for_sort_n = m;
  qsort(order, m, sizeof(uint64_t), wp_cmp); /* total order: stable not needed */
  for (uint64_t i = 0; i < m; ++i) colour[i] = -1;
  uint64_t* used = (uint64_t*)calloc(m + 1, sizeof(uint64_t));
  uint64_t epoch = 0, k = 0;
  for (uint64_t t = 0; t < m; ++t) {
    const uint64_t v = order[t];
    ++epoch;
    for (uint64_t a = 0; a < adj[v].n; ++a) {
      const int32_t c = colour[adj[v].a[a]];
      if (c >= 0) used[c] = epoch;
    }
    uint64_t c = 0;
    while (used[c] == epoch) ++c;
    colour[v] = (int32_t)c;
    if (c + 1 > k) k = c + 1;
  }
  free(deg);
  free(order);
  free(used);
  return k;
}

/* Public: colour the sets of a FOS over a Max-Cut graph.  Also reports the
 * LMIG edge count (scheduling.hpp:37-41) for KAT checks. */
ORC_API int64_t orc_color_sets(uint64_t nv, uint64_t q, const uint32_t* eu, const uint32_t* ev,
                               const double* ew, uint64_t m, const uint64_t* set_off,
                               const uint32_t* set_vars, int32_t* colour_out,
                               uint64_t* lmig_edges_out) {
  orc_problem P;
  problem_build(&P, nv, q, eu, ev, ew);
  vec64* adj = build_lmig(&P, m, set_off, set_vars);
  uint64_t twice = 0;
  for (uint64_t i = 0; i < m; ++i) twice += adj[i].n;
  if (lmig_edges_out) *lmig_edges_out = twice / 2;
  const uint64_t k = welsh_powell(adj, m, colour_out);
  for (uint64_t i = 0; i < m; ++i) free(adj[i].a);
  free(adj);
  problem_free(&P);
  return (int64_t)k;
}

/* ------------------------------------------------------------------------- */
/* Engine: ParallelEngine (engine_parallel.hpp:255-368).                     */
/* ------------------------------------------------------------------------- */

enum { ORC_STOP_NONE = 0, ORC_STOP_BUDGET = 1, ORC_STOP_CLOCK = 2, ORC_STOP_TARGET = 3,
       ORC_STOP_GENLIMIT = 4 };

typedef struct {
  uint64_t size;
  uint64_t* set_ids;   /* ascending (engine_parallel.hpp:40-41) */
  uint64_t* fp_off;    /* size+1 */
  uint64_t* fp;        /* dependent subfunctions, sorted unique per set (:44-57) */
} orc_plan;

typedef struct {
  double fitness;
  uint64_t evaluator_calls;
  int64_t generation;
} orc_trace_row;

typedef struct {
  orc_problem P;
  uint64_t m;
  uint64_t* set_off;
  uint32_t* set_vars;
  uint64_t k;
  orc_plan* plans;
  uint64_t n;
  orc_mt64 rng;
  int pop_id;
  /* population: genotypes, fitness and per-subfunction cache (graybox.hpp:113-117) */
  uint8_t* geno;   /* n * nv */
  double* fit;
  double* cache;   /* n * q */
  uint8_t* shadow; /* n * nv */
  uint8_t* elit;
  double elit_fit;
  int64_t generation;
  /* run control (runtime.hpp:60-123) */
  uint64_t calls;
  int has_budget, has_target, has_genlimit;
  double max_evals, target;
  int64_t max_gens;
  int stop, reason;
  int has_best;
  double best;
  /* trace of improvements (runtime.hpp:136-143) */
  orc_trace_row* trace;
  uint64_t trace_n, trace_cap;
  /* group counters (runtime.hpp:170-175) */
  uint64_t* ctr_steps;
  uint64_t* ctr_calls;
  /* batch dump of every group of the last generation, in execution order */
  uint64_t last_groups;
  uint64_t* last_group_ids;
  int32_t** last_donor;
  double** last_delta;
  uint8_t** last_present;
  uint8_t** last_accept;
  uint64_t* perm; /* n scratch for select_donor */
} orc_engine;

static void ctl_request_stop(orc_engine* E, int reason) {
  if (!E->stop) { E->stop = 1; E->reason = reason; }
}

/* RunControl::add_evaluator_calls (runtime.hpp:75-80); clock not modelled. */
static void ctl_add_calls(orc_engine* E, uint64_t c) {
  E->calls += c;
  if (E->has_budget && E->P.q && (double)E->calls / (double)E->P.q >= E->max_evals)
    ctl_request_stop(E, ORC_STOP_BUDGET);
}

/* RunContext::report_improvement (runtime.hpp:136-143) + note_best (:88-93). */
static void ctx_report_improvement(orc_engine* E, double fitness) {
  if (E->has_best && !cmp_better(E->P.exact, fitness, E->best)) return;
  E->has_best = 1;
  E->best = fitness;
  if (!E->stop && E->has_target &&
      (cmp_better(E->P.exact, fitness, E->target) || cmp_equal(E->P.exact, fitness, E->target)))
    ctl_request_stop(E, ORC_STOP_TARGET);
  if (E->trace_n == E->trace_cap) {
    E->trace_cap = E->trace_cap ? 2 * E->trace_cap : 64;
    E->trace = (orc_trace_row*)realloc(E->trace, E->trace_cap * sizeof(orc_trace_row));
  }
  E->trace[E->trace_n].fitness = fitness;
  E->trace[E->trace_n].evaluator_calls = E->calls;
  E->trace[E->trace_n].generation = E->generation;
  ++E->trace_n;
}

/* full_evaluate (graybox.hpp:131-148): left-to-right sum in edge order. */
static double full_evaluate(const orc_problem* P, const uint8_t* g, double* cache) {
  double sum = 0.0;
  for (uint64_t i = 0; i < P->q; ++i) {
    cache[i] = g[P->eu[i]] != g[P->ev[i]] ? P->ew[i] : 0.0;
    sum += cache[i];
  }
  return sum;
}

/* make_group_plan (engine_parallel.hpp:37-59). */
static void make_plan(orc_engine* E, orc_plan* pl, const uint64_t* members, uint64_t cnt) {
  pl->size = cnt;
  pl->set_ids = (uint64_t*)malloc((cnt ? cnt : 1) * sizeof(uint64_t));
  memcpy(pl->set_ids, members, cnt * sizeof(uint64_t));
  qsort(pl->set_ids, cnt, sizeof(uint64_t), u64_cmp);
  pl->fp_off = (uint64_t*)malloc((cnt + 1) * sizeof(uint64_t));
  vec64 all = {0}, deps = {0};
  pl->fp_off[0] = 0;
  for (uint64_t p = 0; p < cnt; ++p) {
    const uint64_t sid = pl->set_ids[p];
    deps.n = 0;
    for (uint64_t t = E->set_off[sid]; t < E->set_off[sid + 1]; ++t) {
      const vec64* s = &E->P.subs_of[E->set_vars[t]];
      for (uint64_t a = 0; a < s->n; ++a) v_push(&deps, s->a[a]);
    }
    v_sort_unique(&deps);
    for (uint64_t a = 0; a < deps.n; ++a) v_push(&all, deps.a[a]);
    pl->fp_off[p + 1] = all.n;
  }
  pl->fp = all.a ? all.a : (uint64_t*)malloc(sizeof(uint64_t));
  free(deps.a);
}

/* select_donor (engine_serial.hpp:30-46): lazy Fisher-Yates over the pool. */
static uint64_t select_donor(orc_engine* E, uint64_t s, uint64_t sid) {
  const uint64_t n = E->n, nv = E->P.nv;
  for (uint64_t i = 0; i < n; ++i) E->perm[i] = i;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t j = i + orc_uniform_index(&E->rng, n - i);
    const uint64_t t = E->perm[i];
    E->perm[i] = E->perm[j];
    E->perm[j] = t;
    const uint8_t* cand = E->geno + E->perm[i] * nv;
    const uint8_t* par = E->geno + s * nv;
    for (uint64_t a = E->set_off[sid]; a < E->set_off[sid + 1]; ++a) {
      const uint32_t v = E->set_vars[a];
      if (cand[v] != par[v]) return E->perm[i];
    }
  }
  return ORC_NPOS;
}

/* init_population (engine_parallel.hpp:331-346). */
static void init_population(orc_engine* E, const uint8_t* given) {
  const uint64_t n = E->n, nv = E->P.nv, q = E->P.q;
  for (uint64_t i = 0; i < n; ++i) {
    uint8_t* g = E->geno + i * nv;
    for (uint64_t v = 0; v < nv; ++v)
      g[v] = given ? given[i * nv + v] : (uint8_t)orc_uniform_index(&E->rng, 2);
    E->fit[i] = full_evaluate(&E->P, g, E->cache + i * q);
    ctl_add_calls(E, q);
    if (i == 0 || cmp_better(E->P.exact, E->fit[i], E->elit_fit)) {
      memcpy(E->elit, g, nv);
      E->elit_fit = E->fit[i];
      ctx_report_improvement(E, E->elit_fit);
    }
  }
  memcpy(E->shadow, E->geno, n * nv);
}

/* ParallelEngine ctor (engine_parallel.hpp:257-281).  colour == NULL colours
 * the FOS with Welsh-Powell like build_fixed_model (model.hpp:510-511). */
ORC_API orc_engine* orc_engine_create(uint64_t nv, uint64_t q, const uint32_t* eu,
                                      const uint32_t* ev, const double* ew, uint64_t m,
                                      const uint64_t* set_off, const uint32_t* set_vars,
                                      const int32_t* colour, uint64_t n, uint64_t seed,
                                      const uint8_t* initial_genotypes) {
  if (n == 0 || m == 0 || nv == 0) return NULL;
  orc_engine* E = (orc_engine*)calloc(1, sizeof(orc_engine));
  problem_build(&E->P, nv, q, eu, ev, ew);
  E->m = m;
  E->set_off = (uint64_t*)malloc((m + 1) * sizeof(uint64_t));
  memcpy(E->set_off, set_off, (m + 1) * sizeof(uint64_t));
  E->set_vars = (uint32_t*)malloc(set_off[m] * sizeof(uint32_t));
  memcpy(E->set_vars, set_vars, set_off[m] * sizeof(uint32_t));
  int32_t* col = (int32_t*)malloc(m * sizeof(int32_t));
  if (colour) {
    memcpy(col, colour, m * sizeof(int32_t));
    E->k = 0;
    for (uint64_t i = 0; i < m; ++i)
      if ((uint64_t)col[i] + 1 > E->k) E->k = (uint64_t)col[i] + 1;
  } else {
    vec64* adj = build_lmig(&E->P, m, set_off, set_vars);
    E->k = welsh_powell(adj, m, col);
    for (uint64_t i = 0; i < m; ++i) free(adj[i].a);
    free(adj);
  }
  /* ColorGroups: groups indexed by colour, members ascending (scheduling.hpp:418-422) */
  E->plans = (orc_plan*)calloc(E->k, sizeof(orc_plan));
  uint64_t* members = (uint64_t*)malloc(m * sizeof(uint64_t));
  for (uint64_t c = 0; c < E->k; ++c) {
    uint64_t cnt = 0;
    for (uint64_t i = 0; i < m; ++i)
      if ((uint64_t)col[i] == c) members[cnt++] = i;
    make_plan(E, &E->plans[c], members, cnt);
  }
  free(members);
  free(col);
  E->n = n;
  E->pop_id = 1;
  orc_stream_init(&E->rng, seed);
  E->geno = (uint8_t*)malloc(n * nv);
  E->shadow = (uint8_t*)malloc(n * nv);
  E->fit = (double*)malloc(n * sizeof(double));
  E->cache = (double*)malloc(n * (q ? q : 1) * sizeof(double));
  E->elit = (uint8_t*)malloc(nv);
  E->ctr_steps = (uint64_t*)calloc(E->k, sizeof(uint64_t));
  E->ctr_calls = (uint64_t*)calloc(E->k, sizeof(uint64_t));
  E->last_group_ids = (uint64_t*)calloc(E->k, sizeof(uint64_t));
  E->last_donor = (int32_t**)calloc(E->k, sizeof(void*));
  E->last_delta = (double**)calloc(E->k, sizeof(void*));
  E->last_present = (uint8_t**)calloc(E->k, sizeof(void*));
  E->last_accept = (uint8_t**)calloc(E->k, sizeof(void*));
  E->perm = (uint64_t*)malloc(n * sizeof(uint64_t));
  init_population(E, initial_genotypes);
  return E;
}

ORC_API void orc_engine_set_termination(orc_engine* E, int has_budget, double max_evals,
                                        int has_target, double target, int has_genlimit,
                                        int64_t max_gens) {
  E->has_budget = has_budget;
  E->max_evals = max_evals;
  E->has_target = has_target;
  E->target = target;
  E->has_genlimit = has_genlimit;
  E->max_gens = max_gens;
}

/* run_generation (engine_parallel.hpp:283-316) with the four batched phases
 * insert_donor_genes (:104-121), parallel_partial_evaluations (:130-187),
 * determine_improvements (:194-214) and apply_acceptance (:221-247). */
ORC_API int orc_engine_run_generation(orc_engine* E) {
  if (E->stop) return 1;
  if (E->has_genlimit && E->generation >= E->max_gens) {
    ctl_request_stop(E, ORC_STOP_GENLIMIT);
    return 1;
  }
  const uint64_t n = E->n, nv = E->P.nv, q = E->P.q;
  uint64_t* order = (uint64_t*)malloc(E->k * sizeof(uint64_t));
  orc_permutation(&E->rng, order, E->k);
  E->last_groups = 0;
  uint8_t* pie = (uint8_t*)malloc(n);
  for (uint64_t oi = 0; oi < E->k; ++oi) {
    const uint64_t gi = order[oi];
    const orc_plan* pl = &E->plans[gi];
    const uint64_t G = pl->size, pairs = n * G;
    const uint64_t slot = E->last_groups++;
    E->last_group_ids[slot] = gi;
    free(E->last_donor[slot]);
    free(E->last_delta[slot]);
    free(E->last_present[slot]);
    free(E->last_accept[slot]);
    int32_t* donor = E->last_donor[slot] = (int32_t*)malloc((pairs ? pairs : 1) * sizeof(int32_t));
    double* delta = E->last_delta[slot] = (double*)calloc(pairs ? pairs : 1, sizeof(double));
    uint8_t* present = E->last_present[slot] = (uint8_t*)calloc(pairs ? pairs : 1, 1);
    uint8_t* accept = E->last_accept[slot] = (uint8_t*)calloc(pairs ? pairs : 1, 1);
    for (uint64_t i = 0; i < pairs; ++i) donor[i] = -1;
    /* phase 1: sequential donor draws, set position major (:110-120) */
    uint64_t steps = 0;
    for (uint64_t p = 0; p < G; ++p) {
      const uint64_t sid = pl->set_ids[p];
      for (uint64_t s = 0; s < n; ++s) {
        const uint64_t d = select_donor(E, s, sid);
        if (d == ORC_NPOS) continue;
        donor[s * G + p] = (int32_t)d;
        for (uint64_t a = E->set_off[sid]; a < E->set_off[sid + 1]; ++a) {
          const uint32_t v = E->set_vars[a];
          E->shadow[s * nv + v] = E->geno[d * nv + v];
        }
        ++steps;
      }
    }
    /* phase 2: per pair, left-to-right sums of new (shadow) and old (cache)
     * values over the footprint; delta = sum_new - sum_old (:139-186). */
    uint64_t calls = 0;
    for (uint64_t s = 0; s < n; ++s) {
      const uint8_t* sh = E->shadow + s * nv;
      const double* cache = E->cache + s * q;
      for (uint64_t p = 0; p < G; ++p) {
        const uint64_t sp = s * G + p;
        present[sp] = donor[sp] >= 0;
        if (donor[sp] < 0) continue;
        calls += pl->fp_off[p + 1] - pl->fp_off[p];
        if (pl->fp_off[p + 1] == pl->fp_off[p]) continue; /* delta stays 0 */
        double sn = 0.0, so = 0.0;
        for (uint64_t e = pl->fp_off[p]; e < pl->fp_off[p + 1]; ++e) {
          const uint64_t sub = pl->fp[e];
          sn += sh[E->P.eu[sub]] != sh[E->P.ev[sub]] ? E->P.ew[sub] : 0.0;
        }
        for (uint64_t e = pl->fp_off[p]; e < pl->fp_off[p + 1]; ++e) so += cache[pl->fp[e]];
        delta[sp] = sn - so;
      }
    }
    ctl_add_calls(E, calls);
    /* phase 3: accept rule against group-start fitness/elitist (:194-214) */
    for (uint64_t s = 0; s < n; ++s) {
      pie[s] = memcmp(E->geno + s * nv, E->elit, nv) == 0;
      const double pf = E->fit[s];
      for (uint64_t p = 0; p < G; ++p) {
        const uint64_t sp = s * G + p;
        if (!present[sp]) continue;
        const double cand = pf + delta[sp];
        accept[sp] = cmp_better(E->P.exact, cand, pf) ||
                     (cmp_equal(E->P.exact, cand, pf) && !pie[s]);
      }
    }
    /* phase 4: commit or restore, positions ascending (:221-247) */
    for (uint64_t s = 0; s < n; ++s) {
      uint8_t* g = E->geno + s * nv;
      uint8_t* sh = E->shadow + s * nv;
      double* cache = E->cache + s * q;
      for (uint64_t p = 0; p < G; ++p) {
        const uint64_t sp = s * G + p;
        if (!present[sp]) continue;
        const uint64_t sid = pl->set_ids[p];
        if (accept[sp]) {
          for (uint64_t a = E->set_off[sid]; a < E->set_off[sid + 1]; ++a)
            g[E->set_vars[a]] = sh[E->set_vars[a]];
          E->fit[s] += delta[sp];
          for (uint64_t e = pl->fp_off[p]; e < pl->fp_off[p + 1]; ++e) {
            const uint64_t sub = pl->fp[e];
            cache[sub] = sh[E->P.eu[sub]] != sh[E->P.ev[sub]] ? E->P.ew[sub] : 0.0;
          }
        } else {
          for (uint64_t a = E->set_off[sid]; a < E->set_off[sid + 1]; ++a)
            sh[E->set_vars[a]] = g[E->set_vars[a]];
        }
      }
    }
    E->ctr_steps[gi] += steps;
    E->ctr_calls[gi] += calls;
    /* elitist chain scan (:305-310) */
    for (uint64_t s = 0; s < n; ++s) {
      if (cmp_better(E->P.exact, E->fit[s], E->elit_fit)) {
        memcpy(E->elit, E->geno + s * nv, nv);
        E->elit_fit = E->fit[s];
        ctx_report_improvement(E, E->elit_fit);
      }
    }
    if (E->stop) {
      free(order);
      free(pie);
      return 1;
    }
  }
  free(order);
  free(pie);
  ++E->generation;
  return 0;
}

/* offer_elitist (engine_parallel.hpp:320-322). */
ORC_API void orc_engine_offer_elitist(orc_engine* E, const uint8_t* g, double fitness) {
  if (cmp_better(E->P.exact, fitness, E->elit_fit)) {
    memcpy(E->elit, g, E->P.nv);
    E->elit_fit = fitness;
  }
}

ORC_API uint64_t orc_engine_num_groups(const orc_engine* E) { return E->k; }
ORC_API int64_t orc_engine_generation(const orc_engine* E) { return E->generation; }
ORC_API int orc_engine_stop_reason(const orc_engine* E) { return E->stop ? E->reason : 0; }
ORC_API uint64_t orc_engine_evaluator_calls(const orc_engine* E) { return E->calls; }
ORC_API int orc_engine_exact(const orc_engine* E) { return E->P.exact; }

ORC_API void orc_engine_population(const orc_engine* E, uint8_t* geno, double* fit) {
  if (geno) memcpy(geno, E->geno, E->n * E->P.nv);
  if (fit) memcpy(fit, E->fit, E->n * sizeof(double));
}

ORC_API double orc_engine_elitist(const orc_engine* E, uint8_t* geno) {
  if (geno) memcpy(geno, E->elit, E->P.nv);
  return E->elit_fit;
}

/* ColorGroups members of group c (ascending) and its footprint sizes. */
ORC_API uint64_t orc_engine_group(const orc_engine* E, uint64_t c, uint64_t* set_ids,
                                  uint64_t* fp_off) {
  const orc_plan* pl = &E->plans[c];
  if (set_ids) memcpy(set_ids, pl->set_ids, pl->size * sizeof(uint64_t));
  if (fp_off) memcpy(fp_off, pl->fp_off, (pl->size + 1) * sizeof(uint64_t));
  return pl->size;
}

ORC_API uint64_t orc_engine_group_fp(const orc_engine* E, uint64_t c, uint64_t* fp) {
  const orc_plan* pl = &E->plans[c];
  if (fp) memcpy(fp, pl->fp, pl->fp_off[pl->size] * sizeof(uint64_t));
  return pl->fp_off[pl->size];
}

ORC_API void orc_engine_counters(const orc_engine* E, uint64_t* steps, uint64_t* calls) {
  memcpy(steps, E->ctr_steps, E->k * sizeof(uint64_t));
  memcpy(calls, E->ctr_calls, E->k * sizeof(uint64_t));
}

/* Groups executed by the last run_generation call, in execution order. */
ORC_API uint64_t orc_engine_last_groups(const orc_engine* E, uint64_t* ids) {
  if (ids) memcpy(ids, E->last_group_ids, E->last_groups * sizeof(uint64_t));
  return E->last_groups;
}

ORC_API void orc_engine_last_batch(const orc_engine* E, uint64_t slot, int32_t* donor,
                                   double* delta, uint8_t* present, uint8_t* accept) {
  const uint64_t pairs = E->n * E->plans[E->last_group_ids[slot]].size;
  if (donor) memcpy(donor, E->last_donor[slot], pairs * sizeof(int32_t));
  if (delta) memcpy(delta, E->last_delta[slot], pairs * sizeof(double));
  if (present) memcpy(present, E->last_present[slot], pairs);
  if (accept) memcpy(accept, E->last_accept[slot], pairs);
}

ORC_API uint64_t orc_engine_trace(const orc_engine* E, double* fitness, uint64_t* calls,
                                  int64_t* generation) {
  for (uint64_t i = 0; i < E->trace_n; ++i) {
    if (fitness) fitness[i] = E->trace[i].fitness;
    if (calls) calls[i] = E->trace[i].evaluator_calls;
    if (generation) generation[i] = E->trace[i].generation;
  }
  return E->trace_n;
}

ORC_API void orc_engine_destroy(orc_engine* E) {
  if (!E) return;
  for (uint64_t c = 0; c < E->k; ++c) {
    free(E->plans[c].set_ids);
    free(E->plans[c].fp_off);
    free(E->plans[c].fp);
    free(E->last_donor[c]);
    free(E->last_delta[c]);
    free(E->last_present[c]);
    free(E->last_accept[c]);
  }
  free(E->plans);
  free(E->last_group_ids);
  free(E->last_donor);
  free(E->last_delta);
  free(E->last_present);
  free(E->last_accept);
  free(E->set_off);
  free(E->set_vars);
  free(E->geno);
  free(E->shadow);
  free(E->fit);
  free(E->cache);
  free(E->elit);
  free(E->ctr_steps);
  free(E->ctr_calls);
  free(E->perm);
  free(E->trace);
  problem_free(&E->P);
  free(E);
}
