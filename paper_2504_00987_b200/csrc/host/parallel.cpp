// labsolve::run_replicas on the B200 (labs_run_replicas, or
// labs_run_replicas_multi over the GPUs in LABS_DEVICES), plus the host-side
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
  const labs_memetic_params p = detail::device_params(cfg.n, cfg.memetic);
  const bool traces = report && report->collect_traces;
  // Bounded runs keep every record; unbounded ones get 4096 per replica and
  // throw (never truncate) if a replica produced more.
  const int64_t cap = traces ? detail::trace_capacity(cfg.memetic, 4096) : 0;
  std::vector<labs_memetic_record> recs(traces ? cap * cfg.replicas : 0);
  std::vector<int64_t> lens(traces ? cfg.replicas : 0);
  std::vector<labs_run_result> per(cfg.replicas);
  labs_run_result best{};
  // One GPU, or every GPU in LABS_DEVICES (contiguous replica blocks, seeds
  // base_seed + r either way; labs_run_replicas_multi).
  const std::vector<labs_ctx*>& ctxs = detail::devices();
  if (ctxs.size() > 1)
    detail::check(labs_run_replicas_multi(ctxs.data(), static_cast<int>(ctxs.size()), cfg.n,
                                          cfg.replicas, cfg.base_seed, &p, &best, per.data(),
                                          traces ? recs.data() : nullptr, cap,
                                          traces ? lens.data() : nullptr));
  else
    detail::check(labs_run_replicas(ctxs.front(), cfg.n, cfg.replicas, cfg.base_seed, &p, &best,
                                    per.data(), traces ? recs.data() : nullptr, cap,
                                    traces ? lens.data() : nullptr));
  for (int r = 0; traces && r < cfg.replicas; ++r) detail::check_trace_len(lens[r], cap);
  if (!cfg.run_threaded) {
    // The reference's sequential loop publishes in replica order
    // (parallel.cpp:49-50), so a tie goes to the lowest replica index; the
    // device's first-publisher rule is the threaded run's.
    int win = 0;
    for (int r = 1; r < cfg.replicas; ++r)
      if (per[r].best_energy < per[win].best_energy) win = r;
    best = per[win];
  }
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
