// CPU tests of the fit.hpp drop-in (no device needed): the reference's own
// expectations (proj/tests/test_fit.cpp) plus Student-t quantile values.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "labsolve/fit.hpp"

using namespace labsolve;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                       \
  do {                                                                                    \
    ++g_checks;                                                                           \
    if (!(cond)) {                                                                        \
      ++g_fail;                                                                           \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond);       \
    }                                                                                     \
  } while (0)
#define NEAR(a, b, tol) CHECK(std::fabs((a) - (b)) <= (tol) * (1.0 + std::fabs(b)))
#define THROWS(expr, type)                                                                \
  do {                                                                                    \
    ++g_checks;                                                                           \
    bool ok_ = false;                                                                     \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const type&) {                                                               \
      ok_ = true;                                                                         \
    }                                                                                     \
    if (!ok_) {                                                                           \
      ++g_fail;                                                                           \
      std::fprintf(stderr, "%s:%d: %s did not throw\n", __FILE__, __LINE__, #expr);       \
    }                                                                                     \
  } while (0)

int main(int argc, char** argv) {
  NEAR(quantile({3.0, 1.0, 2.0}, 0.5), 2.0, 1e-12);
  NEAR(quantile({1.0, 2.0, 3.0, 4.0}, 0.5), 2.5, 1e-12);
  NEAR(quantile({1.0, 2.0, 3.0, 4.0}, 0.25), 1.75, 1e-12);
  NEAR(quantile({5.0}, 0.9), 5.0, 1e-12);
  NEAR(quantile({1.0, 9.0}, 1.0), 9.0, 1e-12);
  THROWS(quantile({}, 0.5), std::invalid_argument);
  THROWS(quantile({1.0}, 1.5), std::invalid_argument);

  std::vector<TtsSample> s{{10, 5, 1.0, true, 0, 1}, {10, 5, 3.0, true, 0, 1},
                           {10, 5, 99.0, false, 0, 1}, {11, 5, 7.0, true, 0, 1},
                           {12, 5, 50.0, false, 0, 1}};
  auto med = median_runtime_by_n(s);
  CHECK(med.size() == 2);
  NEAR(med.at(10), 2.0, 1e-12);
  NEAR(med.at(11), 7.0, 1e-12);

  std::vector<TtsSample> ex;
  for (int n = 20; n <= 40; ++n)
    for (int r = 0; r < 3; ++r) ex.push_back({n, 0, 2.0e-7 * std::pow(1.3, n), true, 0, 1});
  ex.push_back({41, 0, 1e9, true, 0, 1});  // outside the window
  FitResult f = fit_exponential(ex, 20, 40);
  CHECK(f.points_used == 21);
  NEAR(f.a, 2.0e-7, 1e-9);
  NEAR(f.b, 1.3, 1e-12);
  CHECK(f.b_ci.second - f.b_ci.first < 1e-9);
  THROWS(fit_exponential(ex, 20, 21), std::invalid_argument);
  THROWS(fit_exponential(ex, 30, 20), std::invalid_argument);

  // Student-t 97.5% quantiles (standard table values)
  NEAR(student_t_quantile(1, 0.975), 12.706204736174707, 1e-9);
  NEAR(student_t_quantile(2, 0.975), 4.302652729749464, 1e-9);
  NEAR(student_t_quantile(10, 0.975), 2.228138851986274, 1e-9);
  NEAR(student_t_quantile(30, 0.975), 2.042272456301238, 1e-9);
  NEAR(student_t_quantile(19, 0.025), -2.093024054408263, 1e-9);

  const std::string path = argc > 1 ? argv[1] : "/tmp/labs_fit_roundtrip.jsonl";
  write_samples(path, s);
  auto back = read_samples(path);
  CHECK(back.size() == s.size());
  for (std::size_t i = 0; i < s.size() && i < back.size(); ++i) {
    CHECK(back[i].n == s[i].n && back[i].target_energy == s[i].target_energy);
    CHECK(back[i].runtime_seconds == s[i].runtime_seconds);
    CHECK(back[i].reached_target == s[i].reached_target && back[i].replicas == s[i].replicas);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
