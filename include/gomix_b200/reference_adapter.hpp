// reference_adapter.hpp — drop-in GPU engine for the reference library.
//
// A maintainer of the reference (`gomix`, proj/include/gomix/) adds this header
// and links libgomix_b200.so; then
//
//     gomix::detail::run_with<gomix::GpuParallelEngine>(problem, spec, sink, true);
//
// runs the reference's own run loop / IMS driver (run.hpp:41-97, ims.hpp:38-101)
// with every generation executed on the B200.  GpuParallelEngine has
// ParallelEngine's constructor (engine_parallel.hpp:257-258) and its
// GenerationRunner face (ims.hpp:14-22), plus population()/model()/
// group_counters() (engine_parallel.hpp:324-328).
//
// The problem must be a Max-Cut gray box (as_graybox, maxcut.hpp:67-79): every
// subfunction has two sorted inputs and value w*[x_u != x_v].  That is checked
// by probing the evaluator, so the opaque std::function interface
// (graybox.hpp:41-42) is recovered as an explicit graph; anything else throws
// std::invalid_argument.  Default mode replays the reference's RngStream, so
// results are bit-identical to ParallelEngine; set
// GpuParallelEngine::default_mode = GOMIX_MODE_PHILOX for device-side donors.
//
// The reference's RunContext stays the source of truth: every call hands the
// run-wide evaluator count and termination to the device, and the returned
// per-improvement call counts are replayed through RunControl /
// RunContext::report_improvement in the reference's order.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "gomix/engine_parallel.hpp"
#include "gomix/graybox.hpp"
#include "gomix/ims.hpp"
#include "gomix/model.hpp"
#include "gomix/runtime.hpp"
#include "gomix_gpu.h"

namespace gomix {

namespace gpu_detail {

inline void check(int status) {
  if (status == GOMIX_OK) return;
  const std::string msg = gomix_gpu_last_error();
  if (status == GOMIX_E_INVALID) throw std::invalid_argument(msg);
  if (status == GOMIX_E_STATE) throw std::logic_error(msg);
  throw std::runtime_error("gomix_gpu: " + msg);
}

// Max-Cut view of a gray-box problem: inputs {u, v}, f(0,0) = f(1,1) = 0,
// f(0,1) = f(1,0) = w.
struct MaxCutView {
  std::vector<uint32_t> u, v;
  std::vector<double> w;
};

inline MaxCutView maxcut_view(const GrayBoxProblem& problem) {
  if (problem.alphabet_size() != 2)
    throw std::invalid_argument("gpu engine: binary alphabet required");
  MaxCutView g;
  const std::size_t q = problem.num_subfunctions();
  g.u.reserve(q);
  g.v.reserve(q);
  g.w.reserve(q);
  const Allele a00[2] = {0, 0}, a01[2] = {0, 1}, a10[2] = {1, 0}, a11[2] = {1, 1};
  for (std::size_t i = 0; i < q; ++i) {
    const auto& in = problem.inputs(i);
    if (in.size() != 2) throw std::invalid_argument("gpu engine: problem is not a Max-Cut gray box");
    const double w = problem.evaluate_subfunction(i, std::span<const Allele>(a01, 2));
    if (problem.evaluate_subfunction(i, std::span<const Allele>(a10, 2)) != w ||
        problem.evaluate_subfunction(i, std::span<const Allele>(a00, 2)) != 0.0 ||
        problem.evaluate_subfunction(i, std::span<const Allele>(a11, 2)) != 0.0)
      throw std::invalid_argument("gpu engine: problem is not a Max-Cut gray box");
    g.u.push_back(static_cast<uint32_t>(in[0]));
    g.v.push_back(static_cast<uint32_t>(in[1]));
    g.w.push_back(w);
  }
  return g;
}

}  // namespace gpu_detail

class GpuParallelEngine final : public GenerationRunner {
 public:
  static inline uint32_t default_mode = GOMIX_MODE_REPLAY;
  static inline int32_t device = 0;

  GpuParallelEngine(const GrayBoxProblem& problem, EngineConfig cfg, RunContext& ctx,
                    int population_id = 1)
      : problem_(problem), cfg_(std::move(cfg)), ctx_(ctx), cmp_(problem.comparator()),
        pop_id_(population_id) {
    if (cfg_.population_size == 0)
      throw std::invalid_argument("engine: population must be non-empty");
    if (cfg_.model.kind != LinkageKind::fixed_tree)
      throw std::invalid_argument("batch engine: needs a model that is fixed for the whole run");
    // same adoption rule as ParallelEngine (engine_parallel.hpp:271-274): a
    // model with groups is adopted, otherwise the FOS is rebuilt from the
    // config; the colouring of a rebuilt model is computed on the GPU
    if (cfg_.fixed_model && !cfg_.fixed_model->groups.groups.empty())
      model_ = cfg_.fixed_model;
    else
      model_ = build_fixed_model(problem_, cfg_.model, false);
    const gpu_detail::MaxCutView g = gpu_detail::maxcut_view(problem_);
    std::vector<uint64_t> off{0};
    std::vector<uint32_t> vars;
    for (const auto& s : model_->fos.sets) {
      for (std::size_t x : s) vars.push_back(static_cast<uint32_t>(x));
      off.push_back(vars.size());
    }
    std::vector<int32_t> colour;
    if (!model_->groups.groups.empty()) {
      colour.assign(model_->fos.sets.size(), -1);
      for (std::size_t c = 0; c < model_->groups.groups.size(); ++c)
        for (std::size_t s : model_->groups.groups[c]) colour[s] = static_cast<int32_t>(c);
    }
    const gomix_maxcut inst{problem_.num_variables(), g.u.size(), g.u.data(), g.v.data(),
                            g.w.data()};
    const gomix_fos fos{model_->fos.sets.size(), off.data(), vars.data()};
    shared_ = shared_problem(inst, fos, colour.empty() ? nullptr : colour.data());
    gomix_problem_info info{};
    gpu_detail::check(gomix_gpu_problem_info(shared_.get(), &info));
    k_ = info.num_groups;
    gomix_engine_config ec{};
    ec.population_size = cfg_.population_size;
    ec.seed = cfg_.seed;
    ec.mode = default_mode;
    ec.population_id = population_id;
    ec.world_size = 1;
    gomix_gpu_engine* e = nullptr;
    gpu_detail::check(gomix_gpu_engine_create(shared_.get(), &ec, &e));
    engine_.reset(e);
    gomix_stop_criteria stop = criteria();
    gomix_run_stats stats{};
    gpu_detail::check(gomix_gpu_init_population(engine_.get(), nullptr, &stop, &stats));
    absorb(stats, 0);
    counters_.resize(k_);
    std::vector<uint64_t> sets(k_);
    gpu_detail::check(gomix_gpu_group_counters(engine_.get(), sets.data(), nullptr, nullptr));
    for (std::size_t i = 0; i < k_; ++i) counters_[i].sets = sets[i];
  }

  void run_generation() override {
    if (ctx_.control.stop_requested()) return;
    const auto& term = ctx_.control.config();
    if (term.max_generations && generation_ >= *term.max_generations) {
      ctx_.control.request_stop(StopReason::generation_limit);
      return;
    }
    gomix_stop_criteria stop = criteria();
    gomix_run_stats stats{};
    gpu_detail::check(gomix_gpu_run_generation(engine_.get(), &stop, &stats));
    absorb(stats, generation_);
    if (stats.stopped) return;
    ++generation_;
    ctx_.report_boundary(elitist_.fitness, generation_, pop_id_);
  }

  long generation() const override { return generation_; }

  const EvaluatedSolution& elitist() const override {
    if (elitist_stale_) {
      elitist_.genotype.resize(problem_.num_variables());
      double f = 0.0;
      gpu_detail::check(gomix_gpu_read_elitist(engine_.get(), elitist_.genotype.data(), &f));
      elitist_.fitness = f;
      elitist_stale_ = false;
    }
    return elitist_;
  }

  void offer_elitist(const EvaluatedSolution& candidate) override {
    if (!cmp_.better(candidate.fitness, elitist_.fitness)) return;
    int32_t adopted = 0;
    gpu_detail::check(gomix_gpu_offer_elitist(engine_.get(), candidate.genotype.data(),
                                              candidate.fitness, &adopted));
    if (adopted) {
      elitist_.genotype = candidate.genotype;
      elitist_.fitness = candidate.fitness;
      elitist_stale_ = false;
    }
  }

  // population() materialises genotypes and fitness; the per-subfunction
  // cache is recomputed on the host only for callers that inspect it.
  const std::vector<EvaluatedSolution>& population() const {
    const std::size_t n = cfg_.population_size, nv = problem_.num_variables();
    std::vector<uint8_t> g(n * nv);
    std::vector<double> f(n);
    gpu_detail::check(gomix_gpu_read_population(engine_.get(), g.data(), f.data()));
    population_.resize(n);
    for (std::size_t s = 0; s < n; ++s) {
      population_[s] = full_evaluate(problem_, Genotype(g.begin() + s * nv, g.begin() + (s + 1) * nv));
      population_[s].fitness = f[s];
    }
    return population_;
  }

  const ModelArtifacts& model() const { return *model_; }

  const std::vector<RunResult::GroupCounter>& group_counters() const {
    std::vector<uint64_t> steps(k_), calls(k_);
    gpu_detail::check(gomix_gpu_group_counters(engine_.get(), nullptr, steps.data(), calls.data()));
    for (std::size_t i = 0; i < k_; ++i) {
      counters_[i].steps = steps[i];
      counters_[i].evaluator_calls = calls[i];
    }
    return counters_;
  }

 private:
  struct ProblemDel {
    void operator()(gomix_gpu_problem* p) const { gomix_gpu_problem_destroy(p); }
  };
  struct EngineDel {
    void operator()(gomix_gpu_engine* e) const { gomix_gpu_engine_destroy(e); }
  };

  // One device model per (problem, model) pair, shared by every population of
  // a run like the reference's shared ModelArtifacts (run.hpp:110).  Keyed on
  // the model's identity (owner_before of its shared_ptr, so a freed model's
  // address being reused cannot alias), the problem and the device; guarded
  // by a mutex because run_with may be called from several threads.
  struct CacheKey {
    const void* problem;
    std::weak_ptr<const ModelArtifacts> model;
    int32_t device;
  };
  struct CacheLess {
    bool operator()(const CacheKey& a, const CacheKey& b) const {
      if (a.problem != b.problem) return std::less<const void*>()(a.problem, b.problem);
      if (a.device != b.device) return a.device < b.device;
      return a.model.owner_before(b.model);
    }
  };

  std::shared_ptr<gomix_gpu_problem> shared_problem(const gomix_maxcut& inst, const gomix_fos& fos,
                                                    const int32_t* colour) {
    static std::mutex mu;
    static std::map<CacheKey, std::weak_ptr<gomix_gpu_problem>, CacheLess> cache;
    std::lock_guard<std::mutex> lock(mu);
    for (auto it = cache.begin(); it != cache.end();)  // drop entries whose model or device problem died
      it = (it->first.model.expired() || it->second.expired()) ? cache.erase(it) : std::next(it);
    const CacheKey key{&problem_, model_, device};
    if (auto it = cache.find(key); it != cache.end())
      if (auto p = it->second.lock()) return p;
    gomix_gpu_problem* raw = nullptr;
    gpu_detail::check(gomix_gpu_problem_create(&inst, &fos, colour, device, &raw));
    std::shared_ptr<gomix_gpu_problem> p(raw, ProblemDel{});
    cache[key] = p;
    return p;
  }

  gomix_stop_criteria criteria() const {
    const auto& t = ctx_.control.config();
    gomix_stop_criteria s{};
    s.has_max_evaluations = t.max_evaluations.has_value();
    s.max_evaluations = t.max_evaluations.value_or(0.0);
    s.evaluator_calls_before = ctx_.control.evaluator_calls();
    s.has_target = t.target_fitness.has_value();
    s.target_fitness = t.target_fitness.value_or(0.0);
    return s;
  }

  // Replays the device call into the reference's RunContext: evaluator calls
  // up to each improvement, the improvement, then the remainder.
  void absorb(const gomix_run_stats& stats, long generation) {
    std::vector<double> fit(stats.improvements);
    std::vector<uint64_t> at(stats.improvements);
    uint64_t got = 0;
    if (stats.improvements)
      gpu_detail::check(gomix_gpu_read_improvements(engine_.get(), fit.data(), at.data(),
                                                    stats.improvements, &got));
    uint64_t done = ctx_.control.evaluator_calls();
    const uint64_t end = done + stats.evaluator_calls;
    for (uint64_t i = 0; i < got; ++i) {
      if (at[i] > done) {
        ctx_.control.add_evaluator_calls(at[i] - done);
        done = at[i];
      }
      ctx_.report_improvement(fit[i], generation, pop_id_);
    }
    if (end > done) ctx_.control.add_evaluator_calls(end - done);
    // the elitist genotype changes only with a strictly better fitness
    // (engine_parallel.hpp:305-310, :320-322): the host copy is refreshed
    // lazily, and only after a generation that replaced it
    if (stats.improvements > 0 || stats.elitist_fitness != elitist_.fitness) elitist_stale_ = true;
    elitist_.fitness = stats.elitist_fitness;
  }

  const GrayBoxProblem& problem_;
  EngineConfig cfg_;
  RunContext& ctx_;
  FitnessComparator cmp_;
  int pop_id_;
  std::shared_ptr<const ModelArtifacts> model_;
  std::shared_ptr<gomix_gpu_problem> shared_;
  std::unique_ptr<gomix_gpu_engine, EngineDel> engine_;
  std::size_t k_ = 0;
  long generation_ = 0;
  mutable EvaluatedSolution elitist_;
  mutable bool elitist_stale_ = true;
  mutable std::vector<EvaluatedSolution> population_;
  mutable std::vector<RunResult::GroupCounter> counters_;
};

}  // namespace gomix
