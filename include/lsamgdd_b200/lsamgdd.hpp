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
//   spmv / spmv_transpose / transpose / spgemm on caller matrices  sparse.hpp:110-204
//   build_smoother(A, topo) + apply(smoother, r, mode)        smoother.hpp:38-83
//   h.levels[l].{A, G, P, has_interpolation, topology, thresh}  hierarchy.hpp:46-53
//   LevelParams::spectra_csv is honoured (hierarchy.hpp:121-127, :163-165)
//   pcg(apply_a, apply_b, b, tol, maxit) with caller functors is the reference's
//   own host loop (krylov.hpp:42), re-exported unchanged.
//
// Errors come back as the reference's own exception classes (same name(),
// same what() text), so existing catch blocks keep working. The Hierarchy is
// a move-only RAII handle; levels' host mirrors are fetched on request.
#pragma once

#include <array>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
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

class Hierarchy;

// h.levels[l] — host mirrors of Level (hierarchy.hpp:46-53), fetched from the
// device on first use and cached. `smoother` stays empty (the factors live on
// the device; apply(h, level, r, mode) runs them).
class LevelsView {
 public:
  explicit LevelsView(const Hierarchy* h = nullptr) : h_(h) {}
  std::size_t size() const;
  const Level& operator[](std::size_t l) const;
  const Level& back() const { return (*this)[size() - 1]; }
  const Level& front() const { return (*this)[0]; }

 private:
  const Hierarchy* h_;
};

class Hierarchy {
 public:
  Hierarchy() : levels(this) {}
  explicit Hierarchy(void* h) : levels(this), h_(h, &lsamgdd_destroy), cache_(std::make_shared<Cache>()) {}
  Hierarchy(const Hierarchy& o) : levels(this), params(o.params), h_(o.h_), cache_(o.cache_) {}
  Hierarchy(Hierarchy&& o) noexcept : levels(this), params(std::move(o.params)), h_(std::move(o.h_)), cache_(std::move(o.cache_)) {}
  Hierarchy& operator=(Hierarchy o) {
    params = std::move(o.params);
    h_ = std::move(o.h_);
    cache_ = std::move(o.cache_);
    return *this;
  }
  LevelsView levels;   // h.levels[l].A / .G / .P / .topology / .thresh / .has_interpolation
  LevelParams params;  // hierarchy.hpp:62
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
  std::vector<int64_t> export_ints(std::size_t level, int what, int which, int64_t sz_out[3] = nullptr) const {
    int64_t sz[3];
    check(lsamgdd_level_export(h_.get(), static_cast<int64_t>(level), what, sz, nullptr, nullptr, nullptr), nullptr);
    // sizes: PARTITION/COLORS/MULTIPLICITY {count, aux, 0}; GAMMA/SPECTRA {n_agg, total, 0}
    std::vector<int64_t> a(which == 0 ? (what == LSAMGDD_EXPORT_GAMMA || what == LSAMGDD_EXPORT_SPECTRA ? sz[0] + 1 : sz[0])
                                      : sz[1]);
    check(lsamgdd_level_export(h_.get(), static_cast<int64_t>(level), what, sz, which == 0 ? a.data() : nullptr,
                               which == 1 ? a.data() : nullptr, nullptr),
          nullptr);
    if (sz_out) std::memcpy(sz_out, sz, sizeof sz);
    return a;
  }
  // per-aggregate eigenvalues of one level (keep_spectra / spectra_csv)
  void spectra(std::size_t level, std::vector<int64_t>& off, std::vector<double>& vals) const {
    int64_t sz[3];
    check(lsamgdd_level_export(h_.get(), static_cast<int64_t>(level), LSAMGDD_EXPORT_SPECTRA, sz, nullptr, nullptr, nullptr),
          nullptr);
    off.assign(sz[0] + 1, 0);
    vals.assign(sz[1], 0.0);
    check(lsamgdd_level_export(h_.get(), static_cast<int64_t>(level), LSAMGDD_EXPORT_SPECTRA, sz, off.data(), nullptr,
                               vals.data()),
          nullptr);
  }
  const Level& level_mirror(std::size_t l) const {
    std::lock_guard<std::mutex> lk(cache_->mu);
    if (cache_->levels.size() < num_levels()) cache_->levels.resize(num_levels());
    if (l >= cache_->levels.size()) throw IndexError("levels: index out of range");
    auto& slot = cache_->levels[l];
    if (!slot) {
      auto lv = std::make_unique<Level>();
      lv->A = level_matrix(l, LSAMGDD_EXPORT_A);
      lv->G = level_matrix(l, LSAMGDD_EXPORT_G);
      lv->has_interpolation = l + 1 < num_levels();
      if (lv->has_interpolation) {
        lv->P = level_matrix(l, LSAMGDD_EXPORT_P);
        int64_t sz[3];
        const std::vector<int64_t> asg = export_ints(l, LSAMGDD_EXPORT_PARTITION, 0, sz);
        AggregateTopology& t = lv->topology;
        t.n_nodes = asg.size();
        t.omega.assign(static_cast<std::size_t>(sz[1]), {});
        for (std::size_t v = 0; v < asg.size(); ++v) t.omega[static_cast<std::size_t>(asg[v])].push_back(v);
        const std::vector<int64_t> goff = export_ints(l, LSAMGDD_EXPORT_GAMMA, 0);
        const std::vector<int64_t> gnodes = export_ints(l, LSAMGDD_EXPORT_GAMMA, 1);
        t.gamma.assign(t.omega.size(), {});
        for (std::size_t i = 0; i < t.omega.size(); ++i)
          t.gamma[i].assign(gnodes.begin() + goff[i], gnodes.begin() + goff[i + 1]);
        const std::vector<int64_t> col = export_ints(l, LSAMGDD_EXPORT_COLORS, 0, sz);
        t.colors.assign(col.begin(), col.end());
        t.n_colors = static_cast<std::size_t>(sz[1]);
        lsamgdd_level_summary s{};
        check(lsamgdd_get_level_summary(h_.get(), static_cast<int64_t>(l), &s), nullptr);
        t.multiplicity_max = s.n_mult;
        lv->thresh = s.thresh;
      }
      slot = std::move(lv);
    }
    return *slot;
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
  struct Cache {
    std::mutex mu;
    std::vector<std::unique_ptr<Level>> levels;
  };
  std::shared_ptr<void> h_;
  std::shared_ptr<Cache> cache_;
};

inline std::size_t LevelsView::size() const { return h_->num_levels(); }
inline const Level& LevelsView::operator[](std::size_t l) const { return h_->level_mirror(l); }

namespace detail {
inline Hierarchy setup_csr(const lsamgdd_csr* g0, const LevelParams& params, const Extensions& ext) {
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
  void* h = nullptr;
  char err[1024];
  check(lsamgdd_setup(g0, &p, &h, err, sizeof err), err);
  Hierarchy out(h);
  out.params = params;
  if (!params.spectra_csv.empty()) {  // hierarchy.hpp:121-127, :163-165: level,aggregate,index,eigenvalue
    std::ofstream spectra(params.spectra_csv);
    if (!spectra) throw SetupError("setup: cannot open " + params.spectra_csv);
    spectra.precision(17);
    spectra << "level,aggregate,index,eigenvalue\n";
    for (std::size_t ell = 0; ell + 1 < out.num_levels(); ++ell) {
      std::vector<int64_t> off;
      std::vector<double> vals;
      out.spectra(ell, off, vals);
      for (std::size_t i = 0; i + 1 < off.size(); ++i)
        for (int64_t k = off[i]; k < off[i + 1]; ++k) spectra << ell << "," << i << "," << (k - off[i]) << "," << vals[k] << "\n";
    }
  }
  return out;
}
}  // namespace detail

inline Hierarchy setup(const SparseMatrix& g0, const LevelParams& params, const Extensions& ext = {}) {
  CsrView g(g0);
  return detail::setup_csr(&g.csr, params, ext);
}

// A factor written on the device by lsamgdd_generate_stencil_rows (the constant-coefficient grid
// constructions of BASELINE configs 2, 3, 5; problems.hpp:84-132 has the same row shape): owns the
// device arrays, converts to a host SparseMatrix on request.
class DeviceFactor {
 public:
  // offsets: [rows_per_node][max_entries][3] (dx, dy, dz); coefs: [rows_per_node][max_entries], 0.0 = no entry
  DeviceFactor(const std::array<int64_t, 3>& grid, int rows_per_node, int max_entries, const std::vector<int32_t>& offsets,
               const std::vector<double>& coefs, int device = 0) {
    if (offsets.size() != static_cast<std::size_t>(rows_per_node) * max_entries * 3 ||
        coefs.size() != static_cast<std::size_t>(rows_per_node) * max_entries)
      throw DimError("DeviceFactor: offsets must be [rows][entries][3] and coefs [rows][entries]");
    char err[1024];
    check(lsamgdd_generate_stencil_rows(grid.data(), rows_per_node, max_entries, offsets.data(), coefs.data(), device,
                                        &owner_, &csr_, err, sizeof err),
          err);
  }
  DeviceFactor(const DeviceFactor&) = delete;
  DeviceFactor& operator=(const DeviceFactor&) = delete;
  DeviceFactor(DeviceFactor&& o) noexcept : owner_(o.owner_), csr_(o.csr_) { o.owner_ = nullptr; }
  ~DeviceFactor() {
    if (owner_) lsamgdd_generated_destroy(owner_);
  }
  const lsamgdd_csr& csr() const { return csr_; }
  std::size_t n_rows() const { return static_cast<std::size_t>(csr_.n_rows); }
  std::size_t n_cols() const { return static_cast<std::size_t>(csr_.n_cols); }
  std::size_t nnz() const { return static_cast<std::size_t>(csr_.nnz); }
  SparseMatrix to_host() const {
    std::vector<int64_t> off(n_rows() + 1), col(nnz());
    std::vector<double> val(nnz());
    char err[1024];
    check(lsamgdd_generated_export(owner_, off.data(), col.data(), val.data(), err, sizeof err), err);
    return SparseMatrix(n_rows(), n_cols(), std::vector<std::size_t>(off.begin(), off.end()),
                        std::vector<std::size_t>(col.begin(), col.end()), std::move(val));
  }

 private:
  void* owner_ = nullptr;
  lsamgdd_csr csr_{};
};

inline Hierarchy setup(const DeviceFactor& g0, const LevelParams& params, const Extensions& ext = {}) {
  return detail::setup_csr(&g0.csr(), params, ext);
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

// pcg with the factor the hierarchy was built from (no second copy of G: g == NULL in the C ABI)
inline std::pair<Vector, SolveReport> pcg(const Hierarchy& h, const Vector& b, double tol = 1e-8, std::size_t maxit = 1000) {
  Vector x(b.size());
  std::vector<double> hist(maxit + 2);
  lsamgdd_report rep{};
  rep.residual_history = hist.data();
  rep.history_capacity = hist.size();
  char err[1024];
  check(lsamgdd_pcg(h.handle(), nullptr, b.data(), tol, maxit, x.data(), LSAMGDD_HOST, &rep, err, sizeof err), err);
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

// ---- the sparse kernels on caller matrices (sparse.hpp:110-204) ----
inline SparseMatrix from_device_matrix(void* m) {
  std::unique_ptr<void, int (*)(void*)> guard(m, &lsamgdd_matrix_destroy);
  int64_t sz[3];
  check(lsamgdd_matrix_export(m, sz, nullptr, nullptr, nullptr), nullptr);
  std::vector<int64_t> off(sz[0] + 1), col(sz[2]);
  std::vector<double> val(sz[2]);
  check(lsamgdd_matrix_export(m, sz, off.data(), col.data(), val.data()), nullptr);
  return SparseMatrix(sz[0], sz[1], std::vector<std::size_t>(off.begin(), off.end()),
                      std::vector<std::size_t>(col.begin(), col.end()), std::move(val));
}

inline Vector spmv(const SparseMatrix& a, const Vector& x) {
  if (x.size() != a.n_cols())
    throw DimError("spmv: vector length " + std::to_string(x.size()) + " does not match " + std::to_string(a.n_cols()) +
                   " columns");
  Vector y(a.n_rows());
  CsrView v(a);
  char err[1024];
  check(lsamgdd_spmv(&v.csr, 0, x.data(), y.data(), LSAMGDD_HOST, err, sizeof err), err);
  return y;
}

inline Vector spmv_transpose(const SparseMatrix& a, const Vector& x) {
  if (x.size() != a.n_rows())
    throw DimError("spmv_transpose: vector length " + std::to_string(x.size()) + " does not match " +
                   std::to_string(a.n_rows()) + " rows");
  Vector y(a.n_cols());
  CsrView v(a);
  char err[1024];
  check(lsamgdd_spmv(&v.csr, 1, x.data(), y.data(), LSAMGDD_HOST, err, sizeof err), err);
  return y;
}

inline SparseMatrix transpose(const SparseMatrix& a) {
  CsrView v(a);
  void* m = nullptr;
  char err[1024];
  check(lsamgdd_transpose(&v.csr, &m, err, sizeof err), err);
  return from_device_matrix(m);
}

// Symbolic mode only (the hot path's mode; Numeric — exact zeros dropped — stays with the reference).
inline SparseMatrix spgemm(const SparseMatrix& a, const SparseMatrix& b, SpgemmMode mode = SpgemmMode::Symbolic) {
  if (mode != SpgemmMode::Symbolic) return lsamgdd::spgemm(a, b, mode);
  CsrView va(a), vb(b);
  void* m = nullptr;
  char err[1024];
  check(lsamgdd_spgemm(&va.csr, &vb.csr, &m, err, sizeof err), err);
  return from_device_matrix(m);
}

// ---- build_smoother / apply on a caller operator (smoother.hpp:38-83) ----
class Smoother {
 public:
  explicit Smoother(void* h, std::size_t n) : h_(h, &lsamgdd_smoother_destroy), n_(n) {}
  void* handle() const { return h_.get(); }
  std::size_t n() const { return n_; }

 private:
  std::shared_ptr<void> h_;
  std::size_t n_;
};

inline Smoother build_smoother(const SparseMatrix& a, const AggregateTopology& topo, SchwarzMode = SchwarzMode::RAS) {
  std::vector<int64_t> ooff{0}, om, goff{0}, gm, col(topo.colors.begin(), topo.colors.end());
  for (std::size_t i = 0; i < topo.n_aggregates(); ++i) {
    om.insert(om.end(), topo.omega[i].begin(), topo.omega[i].end());
    ooff.push_back(static_cast<int64_t>(om.size()));
    gm.insert(gm.end(), topo.gamma[i].begin(), topo.gamma[i].end());
    goff.push_back(static_cast<int64_t>(gm.size()));
  }
  CsrView v(a);
  void* h = nullptr;
  char err[1024];
  check(lsamgdd_build_smoother(&v.csr, static_cast<int64_t>(topo.n_aggregates()), ooff.data(), om.data(), goff.data(),
                               gm.data(), col.data(), &h, err, sizeof err),
        err);
  return Smoother(h, a.n_rows());
}

inline Vector apply(const Smoother& s, const Vector& r, SchwarzMode mode) {
  if (r.size() != s.n())
    throw DimError("schwarz apply: vector length " + std::to_string(r.size()) + " does not match system size " +
                   std::to_string(s.n()));
  Vector e(r.size());
  char err[1024];
  const int m = mode == SchwarzMode::RAS ? LSAMGDD_RAS : mode == SchwarzMode::RAST ? LSAMGDD_RAST : LSAMGDD_ASM;
  check(lsamgdd_smoother_apply(s.handle(), m, r.data(), e.data(), LSAMGDD_HOST, err, sizeof err), err);
  return e;
}

// pcg with caller functors (krylov.hpp:42): the reference's host loop, unchanged
using lsamgdd::pcg;
// precond_spectrum (krylov.hpp:101-143): a dense host probe capped at 2000 unknowns, unchanged;
// the functors it is given may be built from the device operators above
using lsamgdd::precond_spectrum;

// TwoLevelAdditive (hierarchy.hpp:234-254), a spectrum-study operator, not part of the solve:
// the coarse correction runs through the device SpMVs on the level-0 P mirror; the ASM sweep —
// which needs the full Ω×Ω inverses the device smoother does not keep (it stores the ω columns
// RAS and RAS-T read) — runs through the reference's host smoother built from the level-0 mirrors.
class TwoLevelAdditive {
 public:
  explicit TwoLevelAdditive(const Hierarchy& h) : h_(h) {
    if (h.levels.size() < 2) throw InputError("TwoLevelAdditive: hierarchy has fewer than two levels");
    coarse_ = factor_spd_block(to_dense(h.levels[1].A), "first coarse-level matrix");
    smoother_ = lsamgdd::build_smoother(h.levels[0].A, h.levels[0].topology, SchwarzMode::ASM);
  }
  Vector apply_to(const Vector& r) const {
    const Level& fine = h_.levels[0];
    Vector coarse = b200::spmv_transpose(fine.P, r);
    coarse_.solve_inplace(coarse);
    Vector y = b200::spmv(fine.P, coarse);
    axpy(1.0, lsamgdd::apply(smoother_, r, SchwarzMode::ASM), y);
    return y;
  }

 private:
  const Hierarchy& h_;
  CholeskyFactor coarse_;
  SchwarzSmoother smoother_;
};

inline double operator_complexity(const Hierarchy& h) {
  double v = 0.0;
  check(lsamgdd_operator_complexity(h.handle(), &v), nullptr);
  return v;
}

}  // namespace lsamgdd::b200
