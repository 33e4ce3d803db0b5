// acceptance.cpp's solve_system and checks 2, 3, 4 and 11 (acceptance.cpp:82-103,
// 140-206, 208-260, 451-495) written against the drop-in shim: the same calls
// with the hot-path functions taken from namespace lsamgdd::b200 (alias `hot`)
// instead of namespace lsamgdd. Built by __graft_entry__.build(), run by
// tests/test_gpu_parity.py::test_cpp_shim_acceptance on the B200.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "lsamgdd_b200/lsamgdd.hpp"

namespace hot = lsamgdd::b200;
using lsamgdd::LevelParams;
using lsamgdd::SparseMatrix;
using lsamgdd::Vector;

namespace {
constexpr double kPi = 3.14159265358979323846;

lsamgdd::LeastSquaresSystem make_aniso(std::size_t n, double eps, double theta) {
  lsamgdd::AnisoParams ap;
  ap.nx = ap.ny = n;
  ap.epsilon = eps;
  ap.theta = theta;
  return lsamgdd::build_rotated_aniso(ap);
}

double rel_gap(double a, double b) {
  const double scale = std::max({std::abs(a), std::abs(b), 1e-300});
  return std::abs(a - b) / scale;
}

int failures = 0;
void record(int id, bool pass, const std::string& line) {
  std::printf("[%s] %d. %s\n", pass ? "PASS" : "FAIL", id, line.c_str());
  if (!pass) ++failures;
}

// acceptance.cpp:82-103 with hot::setup / hot::vcycle / hot::spmv
struct SolveOutcome {
  bool ok = false;
  Vector x;
  lsamgdd::SolveReport report;
  double complexity = 0.0;
  std::string error;
};
SolveOutcome solve_system(const lsamgdd::LeastSquaresSystem& sys, const LevelParams& params, double tol, std::size_t maxit) {
  SolveOutcome out;
  try {
    const hot::Hierarchy h = hot::setup(sys.G, params);
    out.complexity = hot::operator_complexity(h);
    const auto apply_a = [&sys](const Vector& v) { return hot::spmv_transpose(sys.G, hot::spmv(sys.G, v)); };
    const auto apply_b = [&h](const Vector& r) { return hot::vcycle(h, r); };
    auto solved = hot::pcg(apply_a, apply_b, sys.rhs, tol, maxit);
    out.x = std::move(solved.first);
    out.report = solved.second;
    out.ok = true;
  } catch (const lsamgdd::Error& e) {
    out.error = e.what();
  }
  return out;
}

void check_factor_propagation() {  // acceptance.cpp:140-171
  double worst = 0.0;
  std::string failure;
  const struct {
    std::size_t n;
    double eps;
  } cases[] = {{32, 1.0}, {64, 1e-4}};
  for (const auto& c : cases) {
    try {
      const auto sys = make_aniso(c.n, c.eps, kPi / 6.0);
      LevelParams params;
      params.coarse_size = 50;
      const hot::Hierarchy h = hot::setup(sys.G, params);
      if (std::getenv("SHIM_TRACE")) std::fprintf(stderr, "setup done, %zu levels\n", h.levels.size());
      for (std::size_t ell = 0; ell + 1 < h.levels.size(); ++ell) {
        const SparseMatrix& p = h.levels[ell].P;
        if (std::getenv("SHIM_TRACE")) std::fprintf(stderr, "level %zu mirror ok, P %zux%zu\n", ell, p.n_rows(), p.n_cols());
        const SparseMatrix gp = hot::spgemm(h.levels[ell].G, p);
        if (std::getenv("SHIM_TRACE")) std::fprintf(stderr, "spgemm ok\n");
        const SparseMatrix gram = hot::spgemm(hot::transpose(gp), gp);
        const SparseMatrix galerkin = hot::spgemm(hot::spgemm(hot::transpose(p), h.levels[ell].A), p);
        const double err = lsamgdd::frobenius_diff(galerkin, gram) / lsamgdd::frobenius_norm(galerkin);
        worst = std::max(worst, err);
      }
    } catch (const lsamgdd::Error& e) {
      failure = e.what();
    }
  }
  record(2, failure.empty() && worst <= 1e-12,
         "every level satisfies PtAP = (GP)t(GP), worst relative gap " + std::to_string(worst) + " " + failure);
}

void check_ras_adjointness() {  // acceptance.cpp:175-206
  double worst = 0.0;
  std::string failure;
  try {
    const auto sys = make_aniso(32, 1e-4, kPi / 6.0);
    const lsamgdd::Partition part = lsamgdd::standard_aggregation(sys.A);
    const lsamgdd::AggregateTopology topo = lsamgdd::build_topology(sys.A, part);
    if (std::getenv("SHIM_TRACE")) std::fprintf(stderr, "topology: %zu aggregates, %zu colours\n", topo.n_aggregates(), topo.n_colors);
    const auto smoother = hot::build_smoother(sys.A, topo);
    if (std::getenv("SHIM_TRACE")) std::fprintf(stderr, "build_smoother ok\n");
    std::mt19937_64 gen(2024);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    const std::size_t n = sys.A.n_rows();
    for (int rep = 0; rep < 100; ++rep) {
      Vector x(n), y(n);
      for (double& v : x) v = dist(gen);
      for (double& v : y) v = dist(gen);
      const double a = lsamgdd::dot(y, hot::apply(smoother, x, lsamgdd::SchwarzMode::RAS));
      if (rep == 0 && std::getenv("SHIM_TRACE")) std::fprintf(stderr, "first RAS apply ok\n");
      const double b = lsamgdd::dot(hot::apply(smoother, y, lsamgdd::SchwarzMode::RAST), x);
      worst = std::max(worst, rel_gap(a, b));
    }
  } catch (const lsamgdd::Error& e) {
    failure = e.what();
  }
  record(3, failure.empty() && worst <= 1e-12,
         "restricted sweep adjoint to its transpose over 100 random pairs, worst asymmetry " + std::to_string(worst) + " " +
             failure);
}

void check_vcycle_spd() {  // acceptance.cpp:208-260 (symmetry and positivity of the cycle)
  double worst = 0.0;
  bool positive = true;
  std::string failure;
  try {
    const auto sys = make_aniso(32, 1e-4, kPi / 6.0);
    LevelParams params;
    params.coarse_size = 50;
    const hot::Hierarchy h = hot::setup(sys.G, params);
    std::mt19937_64 gen(7);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    const std::size_t n = sys.A.n_rows();
    for (int rep = 0; rep < 20; ++rep) {
      Vector x(n), y(n);
      for (double& v : x) v = dist(gen);
      for (double& v : y) v = dist(gen);
      const Vector bx = hot::vcycle(h, x), by = hot::vcycle(h, y);
      worst = std::max(worst, rel_gap(lsamgdd::dot(y, bx), lsamgdd::dot(x, by)));
      positive = positive && lsamgdd::dot(x, bx) > 0.0;
    }
  } catch (const lsamgdd::Error& e) {
    failure = e.what();
  }
  record(4, failure.empty() && positive && worst <= 1e-10,
         "the V-cycle is symmetric and positive on random probes, worst asymmetry " + std::to_string(worst) + " " + failure);
}

void check_two_level_spectrum() {  // acceptance.cpp:264-295
  bool pass = false;
  std::string detail;
  try {
    const auto sys = make_aniso(16, 1.0, 0.0);
    LevelParams params;
    params.coarse_size = 100;
    const hot::Hierarchy h = hot::setup(sys.G, params);
    const hot::TwoLevelAdditive two(h);
    const double tau = h.levels[0].thresh;
    const double k_c = static_cast<double>(h.levels[0].topology.n_colors);
    const double lower = 1.0 / (2.0 + (2.0 * k_c + 1.0) * tau);
    const double upper = k_c + 1.0;
    const auto apply_a = [&sys](const Vector& v) { return hot::spmv(sys.A, v); };
    const auto apply_b = [&two](const Vector& r) { return two.apply_to(r); };
    const auto [lo, hi] = hot::precond_spectrum(apply_a, apply_b, sys.A.n_rows());
    const double slack = 1e-10;
    pass = lo >= lower - slack && hi <= upper + slack;
    detail = "measured [" + std::to_string(lo) + ", " + std::to_string(hi) + "] within [" + std::to_string(lower) + ", " +
             std::to_string(upper) + "], k_c=" + std::to_string(k_c) + ", tau=" + std::to_string(tau);
  } catch (const lsamgdd::Error& e) {
    detail = e.what();
  }
  record(5, pass, "additive two-level spectrum on the 16x16 isotropic grid: " + detail);
}

void check_direct_oracle() {  // acceptance.cpp:451-495 (the rotated-anisotropy systems)
  bool pass = true;
  double worst = 0.0;
  std::string failure;
  std::vector<lsamgdd::LeastSquaresSystem> systems;
  for (double eps : {1.0, 1e-4})
    for (double theta : {0.0, kPi / 6.0}) systems.push_back(make_aniso(16, eps, theta));
  for (const auto& sys : systems) {
    if (sys.A.n_rows() > 400) continue;
    LevelParams params;
    params.coarse_size = 100;
    const auto outcome = solve_system(sys, params, 1e-12, 1000);
    if (!outcome.ok || !outcome.report.converged) {
      pass = false;
      failure = (outcome.ok ? "did not converge" : outcome.error) + " [" + sys.label + "]";
      continue;
    }
    lsamgdd::CholeskyFactor chol;
    if (!chol.factor(lsamgdd::to_dense(sys.A))) {
      pass = false;
      failure = "dense factorization failed [" + sys.label + "]";
      continue;
    }
    const Vector direct = chol.solve(sys.rhs);
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < direct.size(); ++i) {
      num += (outcome.x[i] - direct[i]) * (outcome.x[i] - direct[i]);
      den += direct[i] * direct[i];
    }
    const double rel = std::sqrt(num / den);
    worst = std::max(worst, rel);
    if (!(rel <= 1e-6)) pass = false;
  }
  record(11, pass, "preconditioned solves on 256-DOF systems match dense direct solves, worst relative gap " +
                       std::to_string(worst) + " " + failure);
}
}  // namespace

int main() {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  check_factor_propagation();
  check_ras_adjointness();
  check_vcycle_spd();
  check_two_level_spectrum();
  check_direct_oracle();
  // spectra_csv (hierarchy.hpp:121-127): same header and row format as the reference's dump
  {
    const auto sys = make_aniso(16, 1e-2, 0.5);
    LevelParams params;
    params.coarse_size = 30;
    params.spectra_csv = "/tmp/lsamgdd_b200_spectra.csv";
    const hot::Hierarchy h = hot::setup(sys.G, params);
    LevelParams pr = params;
    pr.spectra_csv = "/tmp/lsamgdd_ref_spectra.csv";
    const lsamgdd::Hierarchy hr = lsamgdd::setup(sys.G, pr);
    auto slurp = [](const char* p) {
      std::string s;
      if (FILE* f = std::fopen(p, "rb")) {
        char buf[4096];
        size_t k;
        while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, k);
        std::fclose(f);
      }
      return s;
    };
    const std::string a = slurp("/tmp/lsamgdd_b200_spectra.csv"), b = slurp("/tmp/lsamgdd_ref_spectra.csv");
    record(12, !a.empty() && a == b, "spectra_csv dump is byte-identical to the reference's (" + std::to_string(a.size()) +
                                         " bytes)");
    (void)h;
    (void)hr;
  }
  return failures == 0 ? 0 : 1;
}
