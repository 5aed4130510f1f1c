// labsolve::run_replicas on the B200 (labs_run_replicas), plus the host-side
// SharedState and the paper's sizing helpers.
#include "labsolve/parallel.hpp"

#include <algorithm>
#include <stdexcept>

#include "device.hpp"

namespace labsolve {

bool SharedState::publish(const RunResult& result) {
  std::lock_guard<std::mutex> lock(mutex_);
  if (best_ && !(result.best_energy < best_->best_energy)) return false;
  best_ = result;
  return true;
}

std::optional<RunResult> SharedState::best() const {
  std::lock_guard<std::mutex> lock(mutex_);
  return best_;
}

RunResult run_replicas(const ParallelConfig& cfg, ReplicaReport* report) {
  if (cfg.n < 2) throw std::invalid_argument("run needs length >= 2");
  if (cfg.replicas < 1) throw std::invalid_argument("replicas must be >= 1");
  const MemeticParams& m = cfg.memetic;
  if (m.scan_workers < 1) throw std::invalid_argument("scan workers must be >= 1");
  labs_memetic_params p{};
  p.population_size = m.population_size;
  p.rng_kind = LABS_RNG_MT19937_64;
  p.p_comb = m.p_comb;
  p.p_mutate = m.p_mutate.value_or(-1.0);
  if (m.p_mutate && !(*m.p_mutate > 0.0))
    throw std::invalid_argument("mutation probability must be in (0, 1]");
  p.target_energy = m.target_energy;
  p.max_seconds = m.max_seconds.value_or(-1.0);
  p.max_iterations = m.max_iterations.value_or(-1);
  p.tabu = {m.tabu.min_tabu_factor, m.tabu.max_tabu_factor, LABS_TIE_REFERENCE, 0};
  const bool traces = report && report->collect_traces;
  const int64_t cap = traces ? (m.max_iterations ? *m.max_iterations + 1 : 1 << 16) : 0;
  std::vector<labs_memetic_record> recs(traces ? cap * cfg.replicas : 0);
  std::vector<int64_t> lens(traces ? cfg.replicas : 0);
  std::vector<labs_run_result> per(cfg.replicas);
  labs_run_result best{};
  detail::check(labs_run_replicas(detail::device(), cfg.n, cfg.replicas, cfg.base_seed, &p,
                                  &best, per.data(), traces ? recs.data() : nullptr, cap,
                                  traces ? lens.data() : nullptr));
  auto convert = [&](const labs_run_result& o) {
    RunResult r;
    r.best = Sequence(cfg.n);
    for (int w = 0; w < r.best.word_count(); ++w) r.best.set_word(w, o.best[w]);
    r.best_energy = o.best_energy;
    r.merit = merit_factor(cfg.n, o.best_energy);
    r.iterations = o.iterations;
    r.wall_seconds = o.wall_seconds;
    r.seed = o.seed;
    r.replica_id = o.replica_id;
    r.reached_target = o.reached_target != 0;
    return r;
  };
  if (report) {
    report->results.clear();
    for (const auto& o : per) report->results.push_back(convert(o));
    report->traces.assign(traces ? cfg.replicas : 0, MemeticTrace{});
    for (int r = 0; traces && r < cfg.replicas; ++r)
      for (int64_t i = 0; i < lens[r]; ++i) {
        const auto& rec = recs[static_cast<size_t>(r) * cap + i];
        report->traces[r].iters.push_back({rec.iteration, rec.stop_seen != 0, rec.child_energy});
      }
  }
  return convert(best);
}

int suggested_scan_workers(int n) {
  if (n < 1) throw std::invalid_argument("length must be positive");
  return 32 * (n / 32 + 1);
}

long long suggested_replicas(long long units, long long max_per_unit,
                             long long max_workers_per_unit, long long workers_per_replica) {
  if (units < 1 || max_per_unit < 1 || max_workers_per_unit < 1 || workers_per_replica < 1)
    throw std::invalid_argument("replica sizing arguments must be positive");
  const long long fit = max_workers_per_unit / workers_per_replica;
  if (fit < 1) throw std::invalid_argument("a replica's workers exceed one unit's budget");
  return units * std::min(max_per_unit, fit);
}

std::size_t shared_footprint(int n, int population) {
  if (n < 2) throw std::invalid_argument("length must be >= 2");
  if (population < 1) throw std::invalid_argument("population must be >= 1");
  const std::size_t len = static_cast<std::size_t>(n);
  const std::size_t pop_bytes = (static_cast<std::size_t>(population) * len + 7) / 8;
  const std::size_t table_bytes = (len * (len - 1) / 2 + 7) / 8;
  return pop_bytes + table_bytes + 2 * (len - 1) + 2 * len;
}

}  // namespace labsolve
