// Drop-in test: the UNMODIFIED reference's run loop, IMS driver and RunContext
// drive gomix::GpuParallelEngine (include/gomix_b200/reference_adapter.hpp),
// and every observable is compared with the reference's ParallelEngine.
// Built by oracle/Makefile (needs the reference headers, so it is built in the
// build container and shipped as a binary); run by tests/test_cpp_adapter.py.
#include <cstdio>
#include <cstdlib>
#include <optional>
#include <string>
#include <vector>

#include "gomix/engine_parallel.hpp"
#include "gomix/maxcut.hpp"
#include "gomix/model.hpp"
#include "gomix/run.hpp"
#include "gomix/scheduling.hpp"
#include "gomix_b200/reference_adapter.hpp"

using namespace gomix;

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

struct Log final : TraceSink {
  std::vector<TraceRecord> rows;
  void improvement(const TraceRecord& r) override { rows.push_back(r); }
};

bool same_trace(const Log& a, const Log& b) {
  if (a.rows.size() != b.rows.size()) return false;
  for (std::size_t i = 0; i < a.rows.size(); ++i) {
    const auto &x = a.rows[i], &y = b.rows[i];
    if (x.fitness != y.fitness || x.generation != y.generation || x.population != y.population ||
        x.evaluations != y.evaluations)
      return false;
  }
  return true;
}

std::shared_ptr<ModelArtifacts> univariate_model(const GrayBoxProblem& problem) {
  auto m = std::make_shared<ModelArtifacts>();
  m->vig = build_vig(problem);
  m->fos.num_variables = problem.num_variables();
  for (std::size_t v = 0; v < problem.num_variables(); ++v) {
    m->fos.sets.push_back({v});
    m->fos.children.push_back({-1, -1});
  }
  m->groups = welsh_powell(build_lmig(m->fos, m->vig));
  return m;
}

void engine_lockstep(const char* name, const MaxCutInstance& inst, std::shared_ptr<ModelArtifacts> model,
                     std::size_t n, std::uint64_t seed, int gens, std::optional<std::size_t> bound = {}) {
  const GrayBoxProblem problem = as_graybox(inst);
  Log la, lb;
  RunContext ca({}, problem.comparator(), problem.num_subfunctions(), &la);
  RunContext cb({}, problem.comparator(), problem.num_subfunctions(), &lb);
  EngineConfig cfg;
  cfg.population_size = n;
  cfg.seed = seed;
  cfg.workers = 2;
  cfg.fixed_model = model;
  cfg.model.bound = bound;
  ParallelEngine ref(problem, cfg, ca);
  GpuParallelEngine gpu(problem, cfg, cb);
  bool pop_ok = true, elit_ok = true, calls_ok = true;
  for (int g = 0; g < gens; ++g) {
    ref.run_generation();
    gpu.run_generation();
    const auto& pa = ref.population();
    const auto& pb = gpu.population();
    for (std::size_t s = 0; s < n; ++s)
      if (pa[s].genotype != pb[s].genotype || pa[s].fitness != pb[s].fitness) pop_ok = false;
    if (ref.elitist().fitness != gpu.elitist().fitness ||
        ref.elitist().genotype != gpu.elitist().genotype)
      elit_ok = false;
    if (ca.control.evaluator_calls() != cb.control.evaluator_calls()) calls_ok = false;
  }
  bool ctr_ok = ref.group_counters().size() == gpu.group_counters().size();
  for (std::size_t i = 0; ctr_ok && i < ref.group_counters().size(); ++i) {
    const auto &x = ref.group_counters()[i], &y = gpu.group_counters()[i];
    ctr_ok = x.sets == y.sets && x.steps == y.steps && x.evaluator_calls == y.evaluator_calls;
  }
  const std::string tag = std::string(name) + ": ";
  check(pop_ok, tag + "populations identical every generation");
  check(elit_ok, tag + "elitist identical every generation");
  check(calls_ok, tag + "RunControl evaluator calls identical");
  check(ctr_ok, tag + "group counters identical");
  check(gpu.generation() == ref.generation(), tag + "generation counter");
  for (std::size_t s = 0; s < n; ++s)
    if (!solution_consistent(problem, gpu.population()[s])) {
      pop_ok = false;
    }
  check(pop_ok, tag + "population() consistent with full evaluation");
  // traces: same records (times differ)
  bool tr_ok = la.rows.size() == lb.rows.size();
  for (std::size_t i = 0; tr_ok && i < la.rows.size(); ++i)
    tr_ok = la.rows[i].fitness == lb.rows[i].fitness && la.rows[i].generation == lb.rows[i].generation &&
            la.rows[i].evaluations == lb.rows[i].evaluations;
  check(tr_ok, tag + "improvement traces identical (" + std::to_string(la.rows.size()) + " rows)");
}

void run_with_ims(const char* name, const MaxCutInstance& inst, TerminationConfig term) {
  const GrayBoxProblem problem = as_graybox(inst);
  RunSpec spec;
  spec.engine.seed = 5;
  spec.engine.workers = 2;
  spec.engine.fixed_model = univariate_model(problem);
  spec.use_ims = true;
  spec.ims.base_population = 16;
  spec.ims.subgenerations = 4;
  spec.termination = term;
  Log la, lb;
  const RunResult a = detail::run_with<ParallelEngine>(problem, spec, &la, true);
  const RunResult b = detail::run_with<GpuParallelEngine>(problem, spec, &lb, true);
  const std::string tag = std::string(name) + ": ";
  check(a.best.fitness == b.best.fitness && a.best.genotype == b.best.genotype, tag + "IMS best solution");
  check(a.evaluations == b.evaluations, tag + "IMS evaluations " + std::to_string(a.evaluations));
  check(a.generations == b.generations, tag + "IMS generations of population 1");
  check(a.populations == b.populations, tag + "IMS population count " + std::to_string(a.populations));
  check(a.reason == b.reason, tag + std::string("stop reason ") + to_string(a.reason));
  check(same_trace(la, lb), tag + "IMS improvement traces identical (" + std::to_string(la.rows.size()) + " rows)");
}

}  // namespace

int main() {
  try {
    const MaxCutInstance c1 = generate_torus(10, 10, WeightSpec{WeightSpec::Kind::uniform_int, 1, 10}, 1);
    engine_lockstep("C1 torus 10x10, n=32", c1, univariate_model(as_graybox(c1)), 32, 1, 20);
    const MaxCutInstance pm = generate_torus(12, 9, WeightSpec{WeightSpec::Kind::uniform_int, -5, 5}, 4);
    engine_lockstep("+-5 torus 12x9, n=48", pm, univariate_model(as_graybox(pm)), 48, 9, 15);
    {  // groupless model: rebuilt from the config (bflt:10 UPGMA) like the
       // reference (engine_parallel.hpp:271-274), coloured on the GPU
      auto m = univariate_model(as_graybox(c1));
      m->groups.groups.clear();
      engine_lockstep("groupless model -> rebuilt bflt:10, GPU-coloured, n=40", c1, m, 40, 3, 10, 10);
    }
    TerminationConfig budget;
    budget.max_evaluations = 4000.0;
    run_with_ims("run_with<GpuParallelEngine> IMS, budget", generate_torus(12, 12, WeightSpec{WeightSpec::Kind::uniform_int, 1, 10}, 2), budget);
    TerminationConfig target;
    target.target_fitness = 1110.0;  // optimum of the bipartite C1 torus
    target.max_evaluations = 200000.0;
    run_with_ims("run_with<GpuParallelEngine> IMS, target", c1, target);
    // anything that is not a Max-Cut gray box is rejected like a bad config
    {
      GrayBoxProblem other(3, {{0, 1, 2}}, [](std::size_t, std::span<const Allele>) { return 1.0; });
      RunContext ctx({}, other.comparator(), other.num_subfunctions());
      EngineConfig cfg;
      cfg.population_size = 4;
      auto m = std::make_shared<ModelArtifacts>();
      m->vig = build_vig(other);
      m->fos.num_variables = 3;
      m->fos.sets = {{0}, {1}, {2}};
      m->fos.children = {{-1, -1}, {-1, -1}, {-1, -1}};
      cfg.fixed_model = m;
      bool threw = false;
      try {
        GpuParallelEngine e(other, cfg, ctx);
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      check(threw, "non-Max-Cut gray box -> std::invalid_argument");
    }
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
