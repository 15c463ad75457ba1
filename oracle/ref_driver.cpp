// ref_driver.cpp — drives the UNMODIFIED reference library (header-only C++20
// `gomix`, /root/reference/proj/include) so tests can pin the oracle
// restatement and the B200 engine against the reference itself, and so
// bench.py can time the reference CPU path on the GPU box's host cores.
//
// TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/, which
// is git-ignored).  Nothing under paper_2203_08680_b200/ links or calls it.
//
// Modes (all output is a flat binary "named array" stream, see write_arr):
//   run    : ParallelEngine (engine_parallel.hpp:255) for G generations; dumps
//            per-generation populations, fitness, elitist, evaluator calls,
//            group counters.  Also replays the same run through the public
//            phase functions (engine_parallel.hpp:104,130,194,221) and dumps
//            every group's donor / delta / present / accept arrays; the two
//            runs are asserted identical.
//   color  : FOS + LMIG + Welsh-Powell groups (scheduling.hpp:35,85).
//   bench  : wall time of ParallelEngine::run_generation with W workers.
//   ims    : run_parallel (run.hpp:106) with IMS and a target / budget.
//   fi     : the reference's forced_improvement (engine_serial.hpp:98-128) on
//            one solution of a given population (--pop: int64 header
//            [n, nv, o, e] then n*nv genotype bytes; o = the solution, e =
//            the elitist) with RngStream(--seed); dumps the set order it
//            draws, the result genotype / fitness, calls and the outcome.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "gomix/engine_parallel.hpp"
#include "gomix/engine_serial.hpp"
#include "gomix/graybox.hpp"
#include "gomix/linkage.hpp"
#include "gomix/maxcut.hpp"
#include "gomix/model.hpp"
#include "gomix/rng.hpp"
#include "gomix/run.hpp"
#include "gomix/runtime.hpp"
#include "gomix/scheduling.hpp"

using namespace gomix;

namespace {

struct Args {
  std::string mode = "run";
  std::size_t width = 10, height = 10;
  std::string weights = "int:1:10";
  std::uint64_t inst_seed = 1;
  std::string edges;  // edge-list file instead of a torus
  std::string fos = "univariate";
  std::size_t n = 32;
  std::uint64_t seed = 1;
  long gens = 5;
  std::size_t workers = 1;
  std::string out;
  double max_seconds = 0, target = 0, max_evals = 0;
  bool has_target = false, has_evals = false, use_ims = false, serial = false;
  bool light = false;  // run: no phase replica / batch arrays; per-generation populations as packed bits
  std::size_t ims_base = 16, ims_sub = 4;
  std::string pop;
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc > 1) a.mode = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument("missing value for " + k);
      return argv[++i];
    };
    if (k == "--torus") { a.width = std::stoull(next()); a.height = std::stoull(next()); }
    else if (k == "--weights") a.weights = next();
    else if (k == "--inst-seed") a.inst_seed = std::stoull(next());
    else if (k == "--edges") a.edges = next();
    else if (k == "--fos") a.fos = next();
    else if (k == "--n") a.n = std::stoull(next());
    else if (k == "--seed") a.seed = std::stoull(next());
    else if (k == "--gens") a.gens = std::stol(next());
    else if (k == "--workers") a.workers = std::stoull(next());
    else if (k == "--out") a.out = next();
    else if (k == "--max-seconds") a.max_seconds = std::stod(next());
    else if (k == "--target") { a.target = std::stod(next()); a.has_target = true; }
    else if (k == "--max-evals") { a.max_evals = std::stod(next()); a.has_evals = true; }
    else if (k == "--ims") a.use_ims = true;
    else if (k == "--light") a.light = true;
    else if (k == "--serial") a.serial = true;
    else if (k == "--ims-base") a.ims_base = std::stoull(next());
    else if (k == "--ims-sub") a.ims_sub = std::stoull(next());
    else if (k == "--pop") a.pop = next();
    else throw std::invalid_argument("unknown flag " + k);
  }
  return a;
}

MaxCutInstance make_instance(const Args& a) {
  if (!a.edges.empty()) {
    std::ifstream in(a.edges);
    if (!in) throw std::runtime_error("cannot open " + a.edges);
    return load_edge_list(in);
  }
  WeightSpec ws;
  if (a.weights == "unit") {
    ws.kind = WeightSpec::Kind::unit;
  } else if (a.weights.rfind("int:", 0) == 0) {
    ws.kind = WeightSpec::Kind::uniform_int;
    const std::string rest = a.weights.substr(4);
    const auto colon = rest.find(':');
    ws.lo = std::stoll(rest.substr(0, colon));
    ws.hi = std::stoll(rest.substr(colon + 1));
  } else {
    throw std::invalid_argument("weights: unit | int:LO:HI");
  }
  return generate_torus(a.width, a.height, ws, a.inst_seed);
}

Fos make_fos(const Args& a, const GrayBoxProblem& problem, const Vig& vig) {
  const std::size_t nv = problem.num_variables();
  Fos fos;
  fos.num_variables = nv;
  if (a.fos == "univariate") {
    for (std::size_t v = 0; v < nv; ++v) {
      fos.sets.push_back({v});
      fos.children.push_back({-1, -1});
    }
  } else if (a.fos == "neigh") {
    for (std::size_t v = 0; v < nv; ++v) {
      std::vector<std::size_t> s = vig.adjacency[v];
      s.push_back(v);
      std::sort(s.begin(), s.end());
      fos.sets.push_back(s);
      fos.children.push_back({-1, -1});
    }
  } else if (a.fos.rfind("bflt:", 0) == 0 || a.fos == "flt") {
    ModelConfig mc;
    if (a.fos != "flt") mc.bound = std::stoull(a.fos.substr(5));
    fos = build_fixed_model(problem, mc, false)->fos;
  } else if (a.fos.rfind("fosfile:", 0) == 0) {
    std::ifstream in(a.fos.substr(8));
    fos = read_fos(in, nv);
  } else {
    throw std::invalid_argument("fos: univariate | neigh | bflt:B | flt | fosfile:PATH");
  }
  return fos;
}

// ---- flat named-array output ------------------------------------------------
std::FILE* g_out = nullptr;

template <typename T>
void write_arr(const std::string& name, char code, const T* data, std::uint64_t count) {
  const std::uint32_t len = static_cast<std::uint32_t>(name.size());
  std::fwrite(&len, 4, 1, g_out);
  std::fwrite(name.data(), 1, len, g_out);
  std::fwrite(&code, 1, 1, g_out);
  std::fwrite(&count, 8, 1, g_out);
  if (count) std::fwrite(data, sizeof(T), count, g_out);
}
void write_u64(const std::string& name, const std::vector<std::uint64_t>& v) {
  write_arr(name, 'Q', v.data(), v.size());
}
void write_f64(const std::string& name, const std::vector<double>& v) {
  write_arr(name, 'd', v.data(), v.size());
}
void write_u8(const std::string& name, const std::vector<std::uint8_t>& v) {
  write_arr(name, 'B', v.data(), v.size());
}
void write_i32(const std::string& name, const std::vector<std::int32_t>& v) {
  write_arr(name, 'i', v.data(), v.size());
}

void dump_instance(const MaxCutInstance& inst) {
  std::vector<std::uint64_t> u, v;
  std::vector<double> w;
  for (const auto& e : inst.edges) { u.push_back(e.u); v.push_back(e.v); w.push_back(e.w); }
  write_u64("num_vertices", {inst.num_vertices});
  write_u64("edge_u", u);
  write_u64("edge_v", v);
  write_f64("edge_w", w);
}

void dump_model(const ModelArtifacts& m) {
  std::vector<std::uint64_t> off{0}, vars, goff{0}, gsets;
  for (const auto& s : m.fos.sets) {
    vars.insert(vars.end(), s.begin(), s.end());
    off.push_back(vars.size());
  }
  for (const auto& g : m.groups.groups) {
    gsets.insert(gsets.end(), g.begin(), g.end());
    goff.push_back(gsets.size());
  }
  write_u64("set_off", off);
  write_u64("set_vars", vars);
  write_u64("group_off", goff);
  write_u64("group_sets", gsets);
}

std::shared_ptr<ModelArtifacts> build_model(const Args& a, const GrayBoxProblem& problem) {
  auto arts = std::make_shared<ModelArtifacts>();
  arts->vig = build_vig(problem);
  arts->fos = make_fos(a, problem, arts->vig);
  arts->groups = welsh_powell(build_lmig(arts->fos, arts->vig));
  return arts;
}

void flatten_pop(const std::vector<EvaluatedSolution>& pop, std::vector<std::uint8_t>& g,
                 std::vector<double>& f) {
  for (const auto& s : pop) {
    g.insert(g.end(), s.genotype.begin(), s.genotype.end());
    f.push_back(s.fitness);
  }
}

// Replica of ParallelEngine::run_generation (engine_parallel.hpp:283-316) built
// from the library's public phase functions, so per-group batch arrays can be
// dumped.  Asserted equal to the real engine generation by generation.
struct PhaseReplica {
  const GrayBoxProblem& problem;
  std::shared_ptr<const ModelArtifacts> model;
  FitnessComparator cmp;
  RngStream rng;
  WorkerPool pool;
  std::vector<GroupPlan> plans;
  std::vector<EvaluatedSolution> pop;
  std::vector<Genotype> shadow;
  EvaluatedSolution elitist;
  GroupBatch batch;
  std::vector<std::size_t> order, perm;
  std::vector<std::vector<Allele>> scratch;

  PhaseReplica(const GrayBoxProblem& p, std::shared_ptr<const ModelArtifacts> m,
               std::size_t n, std::uint64_t seed, std::size_t workers)
      : problem(p), model(std::move(m)), cmp(p.comparator()), rng(seed), pool(workers) {
    for (const auto& members : model->groups.groups)
      plans.push_back(make_group_plan(problem, model->fos, members));
    Genotype g(problem.num_variables());
    for (std::size_t i = 0; i < n; ++i) {
      for (auto& x : g) x = static_cast<Allele>(rng.uniform_index(problem.alphabet_size()));
      pop.push_back(full_evaluate(problem, g));
      if (i == 0 || cmp.better(pop.back().fitness, elitist.fitness)) elitist = pop.back();
    }
    for (const auto& s : pop) shadow.push_back(s.genotype);
  }

  void generation(std::vector<std::uint64_t>& gorder, std::vector<std::int32_t>& donor,
                  std::vector<double>& delta, std::vector<std::uint8_t>& present,
                  std::vector<std::uint8_t>& accept) {
    rng.permutation(order, plans.size());
    for (const std::size_t gi : order) {
      gorder.push_back(gi);
      const GroupPlan& plan = plans[gi];
      insert_donor_genes(model->fos, plan, pop, shadow, rng, perm, batch);
      parallel_partial_evaluations(problem, plan, pop, shadow, pool, scratch, batch);
      determine_improvements(pop, elitist.genotype, cmp, pool, batch);
      apply_acceptance(model->fos, plan, pop, shadow, pool, batch);
      donor.insert(donor.end(), batch.donor.begin(), batch.donor.end());
      delta.insert(delta.end(), batch.delta.begin(), batch.delta.end());
      present.insert(present.end(), batch.present.begin(), batch.present.end());
      accept.insert(accept.end(), batch.accept.begin(), batch.accept.end());
      for (const auto& s : pop)
        if (cmp.better(s.fitness, elitist.fitness)) elitist = s;
    }
  }
};

struct TraceLog final : TraceSink {
  std::vector<double> fit, secs, evals;
  std::vector<std::uint64_t> gen;
  void improvement(const TraceRecord& r) override {
    fit.push_back(r.fitness);
    secs.push_back(r.seconds);
    evals.push_back(r.evaluations);
    gen.push_back(static_cast<std::uint64_t>(r.generation));
  }
};

// Packed populations (numpy.packbits order: solution-major, 8 alleles per
// byte, first allele in the high bit), for fixtures at sizes where the byte
// genotypes and GroupBatch arrays of every generation would not fit.
void pack_pop(const std::vector<EvaluatedSolution>& pop, std::vector<std::uint8_t>& out) {
  std::size_t bitpos = out.size() * 8;
  std::size_t total = 0;
  for (const auto& s : pop) total += s.genotype.size();
  out.resize(out.size() + (total + 7) / 8, 0);
  for (const auto& s : pop)
    for (const Allele x : s.genotype) {
      if (x) out[bitpos >> 3] |= static_cast<std::uint8_t>(0x80u >> (bitpos & 7));
      ++bitpos;
    }
}

int mode_run_light(const Args& a, ParallelEngine& engine, RunContext& ctx, TraceLog& log) {
  std::vector<std::uint8_t> g0;
  std::vector<double> f0;
  pack_pop(engine.population(), g0);
  for (const auto& s : engine.population()) f0.push_back(s.fitness);
  write_u8("init_packed", g0);
  write_f64("init_fitness", f0);
  write_f64("init_elitist", {engine.elitist().fitness});
  write_u64("init_calls", {ctx.control.evaluator_calls()});
  std::vector<std::uint8_t> G;
  std::vector<double> F, E;
  std::vector<std::uint64_t> C;
  for (long gen = 0; gen < a.gens; ++gen) {
    engine.run_generation();
    pack_pop(engine.population(), G);
    for (const auto& s : engine.population()) F.push_back(s.fitness);
    E.push_back(engine.elitist().fitness);
    C.push_back(ctx.control.evaluator_calls());
  }
  write_u8("packed", G);
  write_f64("fitness", F);
  write_f64("elitist", E);
  write_u64("calls", C);
  std::vector<std::uint64_t> steps, calls;
  for (const auto& c : engine.group_counters()) {
    steps.push_back(c.steps);
    calls.push_back(c.evaluator_calls);
  }
  write_u64("counter_steps", steps);
  write_u64("counter_calls", calls);
  write_f64("trace_fitness", log.fit);
  write_f64("trace_evals", log.evals);
  write_u64("trace_generation", log.gen);
  return 0;
}

int mode_run(const Args& a) {
  const MaxCutInstance inst = make_instance(a);
  const GrayBoxProblem problem = as_graybox(inst);
  auto arts = build_model(a, problem);
  dump_instance(inst);
  dump_model(*arts);

  TraceLog log;
  TerminationConfig term;
  RunContext ctx(term, problem.comparator(), problem.num_subfunctions(), &log);
  EngineConfig cfg;
  cfg.population_size = a.n;
  cfg.seed = a.seed;
  cfg.workers = a.workers;
  cfg.fixed_model = arts;
  ParallelEngine engine(problem, cfg, ctx);
  if (a.light) return mode_run_light(a, engine, ctx, log);
  PhaseReplica rep(problem, arts, a.n, a.seed, a.workers);

  std::vector<std::uint8_t> g0;
  std::vector<double> f0;
  flatten_pop(engine.population(), g0, f0);
  write_u8("init_genotypes", g0);
  write_f64("init_fitness", f0);
  write_f64("init_elitist", {engine.elitist().fitness});
  write_u64("init_calls", {ctx.control.evaluator_calls()});

  std::vector<std::uint8_t> G, P, A;
  std::vector<double> F, E, D;
  std::vector<std::uint64_t> C, order;
  std::vector<std::int32_t> donor;
  for (long gen = 0; gen < a.gens; ++gen) {
    engine.run_generation();
    rep.generation(order, donor, D, P, A);
    std::vector<std::uint8_t> g;
    std::vector<double> f, rf;
    std::vector<std::uint8_t> rg;
    flatten_pop(engine.population(), g, f);
    flatten_pop(rep.pop, rg, rf);
    if (g != rg || f != rf || engine.elitist().fitness != rep.elitist.fitness) {
      std::fprintf(stderr, "phase replica diverged from ParallelEngine at generation %ld\n", gen);
      return 3;
    }
    G.insert(G.end(), g.begin(), g.end());
    F.insert(F.end(), f.begin(), f.end());
    E.push_back(engine.elitist().fitness);
    C.push_back(ctx.control.evaluator_calls());
  }
  write_u8("genotypes", G);
  write_f64("fitness", F);
  write_f64("elitist", E);
  write_u64("calls", C);
  write_u64("group_order", order);
  write_i32("donor", donor);
  write_f64("delta", D);
  write_u8("present", P);
  write_u8("accept", A);
  std::vector<std::uint64_t> steps, calls;
  for (const auto& c : engine.group_counters()) {
    steps.push_back(c.steps);
    calls.push_back(c.evaluator_calls);
  }
  write_u64("counter_steps", steps);
  write_u64("counter_calls", calls);
  write_f64("trace_fitness", log.fit);
  write_f64("trace_evals", log.evals);
  write_u64("trace_generation", log.gen);
  return 0;
}

int mode_color(const Args& a) {
  const MaxCutInstance inst = make_instance(a);
  const GrayBoxProblem problem = as_graybox(inst);
  auto arts = build_model(a, problem);
  dump_instance(inst);
  dump_model(*arts);
  const Lmig lmig = build_lmig(arts->fos, arts->vig);
  write_u64("lmig_edges", {lmig.num_edges()});
  return 0;
}

// Times run_generation only (instance, model and init excluded), as
// BASELINE.md §3 prescribes.  Prints one JSON line.
int mode_bench(const Args& a) {
  const MaxCutInstance inst = make_instance(a);
  const GrayBoxProblem problem = as_graybox(inst);
  auto arts = build_model(a, problem);
  RunContext ctx({}, problem.comparator(), problem.num_subfunctions());
  EngineConfig cfg;
  cfg.population_size = a.n;
  cfg.seed = a.seed;
  cfg.workers = a.workers;
  cfg.fixed_model = arts;
  const auto t_init0 = std::chrono::steady_clock::now();
  ParallelEngine engine(problem, cfg, ctx);
  const double init_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_init0).count();
  std::printf("{\"groups\": %zu, \"init_seconds\": %.6f, \"gens\": [", arts->groups.num_groups(),
              init_s);
  std::uint64_t prev_steps = 0, prev_calls = ctx.control.evaluator_calls();
  double total = 0.0;
  for (long gen = 0; gen < a.gens; ++gen) {
    if (a.max_seconds > 0 && gen > 0 && total >= a.max_seconds) break;  // bounded sample
    const auto t0 = std::chrono::steady_clock::now();
    engine.run_generation();
    const double s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    total += s;
    std::uint64_t steps = 0;
    for (const auto& c : engine.group_counters()) steps += c.steps;
    const std::uint64_t calls = ctx.control.evaluator_calls();
    std::printf("%s{\"seconds\": %.6f, \"steps\": %llu, \"calls\": %llu, \"elitist\": %.17g}",
                gen ? ", " : "", s, static_cast<unsigned long long>(steps - prev_steps),
                static_cast<unsigned long long>(calls - prev_calls), engine.elitist().fitness);
    prev_steps = steps;
    prev_calls = calls;
    std::fflush(stdout);
  }
  std::printf("]}\n");
  return 0;
}

int mode_ims(const Args& a) {
  const MaxCutInstance inst = make_instance(a);
  const GrayBoxProblem problem = as_graybox(inst);
  auto arts = build_model(a, problem);
  RunSpec spec;
  spec.engine.population_size = a.n;
  spec.engine.seed = a.seed;
  spec.engine.workers = a.workers;
  spec.engine.fixed_model = arts;
  spec.use_ims = a.use_ims;
  spec.ims.base_population = a.ims_base;
  spec.ims.subgenerations = a.ims_sub;
  if (a.max_seconds > 0) spec.termination.max_seconds = a.max_seconds;
  if (a.has_target) spec.termination.target_fitness = a.target;
  if (a.has_evals) spec.termination.max_evaluations = a.max_evals;
  if (a.gens > 0 && !a.use_ims) spec.termination.max_generations = a.gens;
  TraceLog log;
  const auto t0 = std::chrono::steady_clock::now();
  const RunResult r = a.serial ? run_serial(problem, spec, &log) : run_parallel(problem, spec, &log);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"best\": %.17g, \"reason\": \"%s\", \"evaluations\": %.17g, \"generations\": %ld, "
              "\"populations\": %zu, \"seconds\": %.6f, \"trace\": [",
              r.best.fitness, to_string(r.reason), r.evaluations, r.generations, r.populations, s);
  for (std::size_t i = 0; i < log.fit.size(); ++i)
    std::printf("%s[%.6f, %.17g, %.17g]", i ? ", " : "", log.secs[i], log.evals[i], log.fit[i]);
  std::printf("]}\n");
  return 0;
}

}  // namespace

int mode_fi(const Args& a) {
  const MaxCutInstance inst = make_instance(a);
  const GrayBoxProblem problem = as_graybox(inst);
  auto arts = build_model(a, problem);
  std::ifstream in(a.pop, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + a.pop);
  std::int64_t hdr[4];
  in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
  const std::size_t n = (std::size_t)hdr[0], nv = (std::size_t)hdr[1];
  if (nv != problem.num_variables()) throw std::invalid_argument("fi: genotype length mismatch");
  std::vector<std::uint8_t> g(n * nv);
  in.read(reinterpret_cast<char*>(g.data()), (std::streamsize)g.size());
  auto row = [&](std::int64_t s) { return Genotype(g.begin() + s * (std::int64_t)nv, g.begin() + (s + 1) * (std::int64_t)nv); };
  EvaluatedSolution o = full_evaluate(problem, row(hdr[2]));
  const EvaluatedSolution elitist = full_evaluate(problem, row(hdr[3]));
  RngStream rng(a.seed);
  RngStream peek = rng;
  std::vector<std::size_t> order;
  peek.permutation(order, arts->fos.sets.size());
  EvalWorkspace ws;
  ws.bind(problem);
  const FiOutcome r = forced_improvement(problem, o, elitist, arts->fos, rng, problem.comparator(), ws);
  write_u64("set_order", std::vector<std::uint64_t>(order.begin(), order.end()));
  write_u8("genotype", std::vector<std::uint8_t>(o.genotype.begin(), o.genotype.end()));
  write_f64("fitness", {o.fitness});
  write_u64("evaluator_calls", {r.evaluator_calls});
  write_u64("strict_improvement", {r.strict_improvement ? 1u : 0u});
  write_u64("replaced_by_elitist", {r.replaced_by_elitist ? 1u : 0u});
  return 0;
}

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.mode == "run" || a.mode == "color" || a.mode == "fi") {
      if (a.out.empty()) throw std::invalid_argument("--out required");
      g_out = std::fopen(a.out.c_str(), "wb");
      if (!g_out) throw std::runtime_error("cannot write " + a.out);
      const int rc = a.mode == "run" ? mode_run(a) : (a.mode == "color" ? mode_color(a) : mode_fi(a));
      std::fclose(g_out);
      return rc;
    }
    if (a.mode == "bench") return mode_bench(a);
    if (a.mode == "ims") return mode_ims(a);
    throw std::invalid_argument("mode: run | color | bench | ims | fi");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_driver: %s\n", e.what());
    return 2;
  }
}
