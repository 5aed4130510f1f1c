// labsolve memetic layer. select_parents / combine / mutate are the host
// forms of the operators the device replica applies (labs_memetic.cuh);
// memetic_tabu itself runs on the B200 (labs_memetic).
#include "labsolve/memetic.hpp"

#include <atomic>
#include <chrono>
#include <stdexcept>
#include <thread>

#include "device.hpp"

namespace labsolve {
namespace {

int tournament(const std::vector<long long>& e, Rng& rng) {
  const long long k = static_cast<long long>(e.size());
  const int a = static_cast<int>(rng.uniform_int(0, k - 1));
  const int b = static_cast<int>(rng.uniform_int(0, k - 1));
  if (e[a] != e[b]) return e[a] < e[b] ? a : b;
  return rng.uniform_int(0, 1) == 0 ? a : b;
}

}  // namespace

std::pair<int, int> select_parents(const std::vector<long long>& energies, Rng& rng) {
  if (energies.size() < 2) throw std::invalid_argument("tournament needs population >= 2");
  const int first = tournament(energies, rng);
  return {first, tournament(energies, rng)};
}

Sequence combine(const Sequence& p1, const Sequence& p2, Rng& rng) {
  if (p1.size() != p2.size()) throw std::invalid_argument("combine needs equal lengths");
  Sequence child(p1.size());
  for (int w = 0; w < child.word_count(); ++w) {
    const std::uint64_t take_first = rng.bits64();
    child.set_word(w, (p1.word(w) & take_first) | (p2.word(w) & ~take_first));
  }
  return child;
}

Sequence mutate(const Sequence& child, double p_mutate, Rng& rng) {
  if (!(p_mutate > 0.0) || p_mutate > 1.0)
    throw std::invalid_argument("mutation probability must be in (0, 1]");
  Sequence out = child;
  for (int i = 0; i < out.size(); ++i)
    if (rng.uniform01() < p_mutate) out.flip(i);
  return out;
}

RunResult memetic_tabu(int n, const MemeticParams& params, std::uint64_t seed,
                       const std::atomic<bool>* stop, MemeticTrace* trace, int replica_id) {
  const labs_memetic_params p = detail::device_params(n, params);

  // The device polls an int32 flag between epochs; mirror the caller's
  // atomic<bool> into it while the run is in flight.
  volatile int32_t flag = 0;
  std::atomic<bool> done{false};
  std::thread watcher;
  if (stop) {
    if (stop->load(std::memory_order_acquire)) flag = 1;
    watcher = std::thread([&] {
      while (!done.load(std::memory_order_acquire)) {
        if (stop->load(std::memory_order_acquire)) flag = 1;
        std::this_thread::sleep_for(std::chrono::microseconds(200));
      }
    });
  }
  labs_run_result out{};
  const int64_t cap = trace ? detail::trace_capacity(params, 1 << 20) : 0;
  std::vector<labs_memetic_record> recs(trace ? cap : 0);
  int64_t len = 0;
  const int rc = labs_memetic(detail::device(), n, &p, seed, stop ? &flag : nullptr, replica_id,
                              &out, trace ? recs.data() : nullptr, cap, trace ? &len : nullptr);
  done.store(true, std::memory_order_release);
  if (watcher.joinable()) watcher.join();
  detail::check(rc);
  if (trace) detail::check_trace_len(len, cap);
  RunResult r;
  r.best = Sequence(n);
  for (int w = 0; w < r.best.word_count(); ++w) r.best.set_word(w, out.best[w]);
  r.best_energy = out.best_energy;
  r.merit = merit_factor(n, out.best_energy);
  r.iterations = out.iterations;
  r.wall_seconds = out.wall_seconds;
  r.seed = seed;
  r.replica_id = replica_id;
  r.reached_target = out.reached_target != 0;
  if (trace)
    for (int64_t i = 0; i < len; ++i)
      trace->iters.push_back({recs[i].iteration, recs[i].stop_seen != 0, recs[i].child_energy});
  return r;
}

}  // namespace labsolve
