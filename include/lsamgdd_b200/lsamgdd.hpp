// lsamgdd_b200/lsamgdd.hpp — C++ drop-in shim over the C ABI.
//
// A caller of the reference header library (lsamgdd/lsamgdd.hpp, whose value
// types SparseMatrix, Vector, LevelParams, SolveReport and exception classes
// this header reuses) switches the hot path to the B200 by calling the
// functions of namespace lsamgdd::b200, which keep the reference's
// signatures:
//
//   setup(const SparseMatrix&, const LevelParams&)            hierarchy.hpp:106
//   vcycle(const Hierarchy&, const Vector&)                   hierarchy.hpp:229
//   vcycle(const Hierarchy&, std::size_t level, const Vector&)  hierarchy.hpp:205
//   apply(const Hierarchy&, level, const Vector&, SchwarzMode)  smoother.hpp:65
//   pcg(const Hierarchy&, const SparseMatrix& g, const Vector& b, tol, maxit)
//                                  krylov.hpp:42 with apply_a = Gᵀ(G·), apply_b = vcycle
//   operator_complexity(const Hierarchy&)                     hierarchy.hpp:257
//
// Errors come back as the reference's own exception classes (same name(),
// same what() text), so existing catch blocks keep working. The Hierarchy is
// a move-only RAII handle; levels' host mirrors are fetched on request.
#pragma once

#include <cstring>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "lsamgdd/lsamgdd.hpp"
#include "lsamgdd_b200.h"

namespace lsamgdd::b200 {

[[noreturn]] inline void rethrow(int status, const char* msg) {
  const std::string what = msg ? msg : "";
  switch (status) {
    case LSAMGDD_ERR_INDEX: throw IndexError(what);
    case LSAMGDD_ERR_DIM: throw DimError(what);
    case LSAMGDD_ERR_INPUT: throw InputError(what);
    case LSAMGDD_ERR_FORMAT: throw FormatError(what);
    case LSAMGDD_ERR_SPLITTING: throw SplittingError(what);
    case LSAMGDD_ERR_EIG: throw EigError(what);
    case LSAMGDD_ERR_SETUP: throw SetupError(what);
    case LSAMGDD_ERR_INDEFINITE: throw IndefiniteError(what);
    case LSAMGDD_ERR_SIZE: throw SizeError(what);
    default: throw Error(what);
  }
}

inline void check(int status, const char* err) {
  if (status != LSAMGDD_OK) rethrow(status, err);
}

// Host CSR in the C ABI's int64 form (SparseMatrix holds size_t).
struct CsrView {
  std::vector<int64_t> off, col;
  lsamgdd_csr csr{};
  explicit CsrView(const SparseMatrix& m)
      : off(m.row_offsets().begin(), m.row_offsets().end()), col(m.col_indices().begin(), m.col_indices().end()) {
    csr.n_rows = static_cast<int64_t>(m.n_rows());
    csr.n_cols = static_cast<int64_t>(m.n_cols());
    csr.nnz = static_cast<int64_t>(m.nnz());
    csr.row_offsets = off.data();
    csr.col_indices = col.data();
    csr.values = m.values().data();
    csr.memory = LSAMGDD_HOST;
  }
};

struct Extensions {  // the config hooks of lsamgdd_params (defaults = reference behaviour)
  std::vector<int64_t> level0_partition;
  int64_t level0_n_aggregates = 0;
  int level0_overlap = 1;
  double thresh_override = 0.0;
  std::size_t level0_max_modes = 0;
  int device = 0;
};

class Hierarchy {
 public:
  Hierarchy() = default;
  explicit Hierarchy(void* h) : h_(h, &lsamgdd_destroy) {}
  void* handle() const { return h_.get(); }
  std::size_t num_levels() const {
    int64_t n = 0;
    check(lsamgdd_num_levels(h_.get(), &n), nullptr);
    return static_cast<std::size_t>(n);
  }
  std::vector<LevelSummary> summary() const {
    std::vector<LevelSummary> out;
    for (std::size_t l = 0; l < num_levels(); ++l) {
      lsamgdd_level_summary s{};
      check(lsamgdd_get_level_summary(h_.get(), static_cast<int64_t>(l), &s), nullptr);
      LevelSummary r;
      r.level = s.level;
      r.dim = s.dim;
      r.nnz = s.nnz;
      r.n_aggregates = s.n_aggregates;
      r.k_c = s.k_c;
      r.n_mult = s.n_mult;
      r.thresh = s.thresh;
      r.modes_kept = s.modes_kept;
      out.push_back(r);
    }
    return out;
  }
  // Host mirror of levels[l].A / .G / .P (hierarchy.hpp:46-51).
  SparseMatrix level_matrix(std::size_t level, int what) const {
    int64_t sz[3];
    check(lsamgdd_level_export(h_.get(), static_cast<int64_t>(level), what, sz, nullptr, nullptr, nullptr), nullptr);
    std::vector<int64_t> off(sz[0] + 1), col(sz[2]);
    std::vector<double> val(sz[2]);
    check(lsamgdd_level_export(h_.get(), static_cast<int64_t>(level), what, sz, off.data(), col.data(), val.data()),
          nullptr);
    return SparseMatrix(sz[0], sz[1], std::vector<std::size_t>(off.begin(), off.end()),
                        std::vector<std::size_t>(col.begin(), col.end()), std::move(val));
  }

 private:
  std::shared_ptr<void> h_;
};

inline Hierarchy setup(const SparseMatrix& g0, const LevelParams& params, const Extensions& ext = {}) {
  lsamgdd_params p;
  lsamgdd_params_default(&p);
  p.max_levels = params.max_levels;
  p.coarse_size = params.coarse_size;
  p.aggregation_passes = params.aggregation_passes;
  p.kappa = params.kappa;
  p.must_keep = params.must_keep;
  if (params.coarsening_ratios.size() > 8) throw InputError("setup: at most 8 coarsening ratios");
  p.n_ratios = params.coarsening_ratios.size();
  for (std::size_t i = 0; i < params.coarsening_ratios.size(); ++i) p.coarsening_ratios[i] = params.coarsening_ratios[i];
  p.pre_sweeps = params.pre_sweeps;
  p.post_sweeps = params.post_sweeps;
  p.gevp_variant = params.gevp_variant == GevpVariant::WeightedLhs ? 1 : 0;
  p.keep_spectra = params.spectra_csv.empty() ? 0 : 1;
  if (!ext.level0_partition.empty()) {
    p.level0_partition = ext.level0_partition.data();
    p.level0_n_aggregates = ext.level0_n_aggregates;
  }
  p.level0_overlap = ext.level0_overlap;
  p.thresh_override = ext.thresh_override;
  p.level0_max_modes = ext.level0_max_modes;
  p.device = ext.device;
  CsrView g(g0);
  void* h = nullptr;
  char err[1024];
  check(lsamgdd_setup(&g.csr, &p, &h, err, sizeof err), err);
  return Hierarchy(h);
}

inline Vector vcycle(const Hierarchy& h, std::size_t level, const Vector& r) {
  Vector e(r.size());
  char err[1024];
  check(lsamgdd_vcycle(h.handle(), static_cast<int64_t>(level), r.data(), e.data(), LSAMGDD_HOST, err, sizeof err), err);
  return e;
}

inline Vector vcycle(const Hierarchy& h, const Vector& r) { return vcycle(h, 0, r); }

inline Vector apply(const Hierarchy& h, std::size_t level, const Vector& r, SchwarzMode mode) {
  Vector e(r.size());
  char err[1024];
  const int m = mode == SchwarzMode::RAS ? LSAMGDD_RAS : mode == SchwarzMode::RAST ? LSAMGDD_RAST : LSAMGDD_ASM;
  check(lsamgdd_schwarz_apply(h.handle(), static_cast<int64_t>(level), m, r.data(), e.data(), LSAMGDD_HOST, err,
                              sizeof err),
        err);
  return e;
}

inline std::pair<Vector, SolveReport> pcg(const Hierarchy& h, const SparseMatrix& g, const Vector& b, double tol = 1e-8,
                                          std::size_t maxit = 1000) {
  Vector x(b.size());
  std::vector<double> hist(maxit + 2);
  lsamgdd_report rep{};
  rep.residual_history = hist.data();
  rep.history_capacity = hist.size();
  CsrView gv(g);
  char err[1024];
  check(lsamgdd_pcg(h.handle(), &gv.csr, b.data(), tol, maxit, x.data(), LSAMGDD_HOST, &rep, err, sizeof err), err);
  SolveReport out;
  out.iterations = rep.iterations;
  out.converged = rep.converged != 0;
  out.avg_conv_factor = rep.avg_conv_factor;
  out.iters_to_tenth = rep.iters_to_tenth;
  out.operator_complexity = rep.operator_complexity;
  out.setup_seconds = rep.setup_seconds;
  out.solve_seconds = rep.solve_seconds;
  out.residual_history.assign(hist.begin(), hist.begin() + static_cast<std::ptrdiff_t>(rep.history_len));
  return {std::move(x), std::move(out)};
}

inline double operator_complexity(const Hierarchy& h) {
  double v = 0.0;
  check(lsamgdd_operator_complexity(h.handle(), &v), nullptr);
  return v;
}

}  // namespace lsamgdd::b200
