// labsolve exhaustive ground truth on the B200 (oracle.hpp).
#include "labsolve/oracle.hpp"

#include <cmath>
#include <fstream>
#include <set>
#include <sstream>
#include <stdexcept>

#include "device.hpp"
#include "labsolve/skew.hpp"

namespace labsolve {

BruteForceResult brute_force_optimum_device(int n) {
  if (n < 2 || n > 64) throw std::invalid_argument("device exhaustive search needs 2 <= n <= 64");
  const int64_t cap = 1 << 16;  // the reference's witness cap (oracle.cpp:19)
  std::vector<uint64_t> raw(cap);
  int64_t e = 0, count = 0;
  detail::check(labs_exhaustive_optimum(detail::device(), n, &e, raw.data(), cap, &count));
  if (count > cap) throw std::runtime_error("optimal witness set exceeded the tracking cap");
  std::set<Sequence> uniq;
  for (int64_t i = 0; i < count; ++i) {
    Sequence s(n);
    s.set_word(0, raw[i]);
    uniq.insert(canonical(s));
  }
  BruteForceResult r;
  r.optimal_energy = e;
  r.witnesses.assign(uniq.begin(), uniq.end());
  return r;
}

BruteForceResult brute_force_optimum(int n, int workers) {
  if (n < 2 || n > 30) throw std::invalid_argument("exhaustive search is limited to 2 <= n <= 30");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  return brute_force_optimum_device(n);
}

long long enumerate_local_optima_device(int n) {
  int64_t c = 0;
  detail::check(labs_local_optima(detail::device(), n, &c));
  return c;
}

long long enumerate_local_optima(int n, int workers) {
  if (n < 2 || n > 24)
    throw std::invalid_argument("local-optima census is limited to 2 <= n <= 24");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  return enumerate_local_optima_device(n);
}

std::vector<TableEntry> read_table_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open table file: " + path);
  std::vector<TableEntry> out;
  std::string line;
  int no = 0;
  while (std::getline(in, line)) {
    ++no;
    const std::size_t p = line.find_first_not_of(" \t\r");
    if (p == std::string::npos || line[p] == '#') continue;
    std::istringstream f(line);
    TableEntry e;
    if (!(f >> e.n >> e.hex >> e.energy >> e.merit >> e.deviation))
      throw std::runtime_error(path + ":" + std::to_string(no) +
                               ": expected 'n hex energy merit deviation'");
    out.push_back(e);
  }
  return out;
}

// verify_published (oracle.cpp:174-199): energy, merit within 0.005, skew
// deviation under the budget; a row that fails to decode records the error
// and the run continues.
VerifyReport verify_published(const std::vector<TableEntry>& entries,
                              std::uint64_t deviation_budget) {
  VerifyReport rep;
  rep.all_pass = true;
  for (const TableEntry& want : entries) {
    VerifyEntry v;
    v.expected = want;
    try {
      const Sequence s = decode_hex(want.hex, want.n);
      v.energy = energy(s);
      v.merit = merit_factor(want.n, v.energy);
      const DeviationResult d = deviation(s, deviation_budget);
      v.deviation = d.value;
      v.budget_exceeded = d.budget_exceeded;
      v.energy_ok = v.energy == want.energy;
      v.merit_ok = std::fabs(v.merit - want.merit) <= 0.005;
      v.deviation_ok = !d.budget_exceeded && d.value == want.deviation;
    } catch (const std::exception& e) {
      v.error = e.what();
    }
    rep.all_pass = rep.all_pass && v.pass();
    rep.entries.push_back(v);
  }
  return rep;
}

}  // namespace labsolve
