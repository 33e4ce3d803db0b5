// oracle/ref_harness.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product). Builds the UNMODIFIED reference headers from
// /root/reference/proj/include into oracle/_ref/libref_lsamgdd.so with the
// reference's CMake Release flags (-std=gnu++20 -O3 -DNDEBUG, no -march, so
// no FMA contraction: SURVEY.md §8(c)). It exposes the reference's own
// setup/vcycle/apply/pcg through a C ABI that mirrors include/lsamgdd_b200.h
// so tests and bench.py --impl reference can drive it with identical inputs.
//
// The only logic here that is not a direct call into the reference is the
// stage replica of setup() (hierarchy.hpp:106-200) with the BASELINE config
// hooks of SURVEY.md Appendix A.1: an injected level-0 partition, a second
// Γ layer at level 0, a direct threshold and a level-0 mode cap. With no
// hook active the replica makes exactly the reference's calls in the
// reference's order (pinned by tests/test_oracle_pins.py against setup()).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <exception>
#include <mutex>
#include <thread>
#include <random>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "lsamgdd/lsamgdd.hpp"
#include "../include/lsamgdd_b200.h"

using namespace lsamgdd;

namespace {

struct RefHandle {
  Hierarchy h;
  SparseMatrix g0;
  std::vector<std::vector<std::vector<double>>> spectra;  // [level][aggregate]
  std::vector<std::vector<std::size_t>> multiplicity;     // [level]
  std::vector<std::pair<std::string, double>> timings;
};

int status_of(const Error& e) {
  const std::string n = e.name();
  if (n == "IndexError") return LSAMGDD_ERR_INDEX;
  if (n == "DimError") return LSAMGDD_ERR_DIM;
  if (n == "InputError") return LSAMGDD_ERR_INPUT;
  if (n == "FormatError") return LSAMGDD_ERR_FORMAT;
  if (n == "SplittingError") return LSAMGDD_ERR_SPLITTING;
  if (n == "EigError") return LSAMGDD_ERR_EIG;
  if (n == "SetupError") return LSAMGDD_ERR_SETUP;
  if (n == "IndefiniteError") return LSAMGDD_ERR_INDEFINITE;
  if (n == "SizeError") return LSAMGDD_ERR_SIZE;
  return LSAMGDD_ERR_ERROR;
}

void put_err(char* err, size_t errlen, const std::string& msg) {
  if (!err || errlen == 0) return;
  std::strncpy(err, msg.c_str(), errlen - 1);
  err[errlen - 1] = '\0';
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return LSAMGDD_OK;
  } catch (const Error& e) {
    put_err(err, errlen, std::string(e.name()) + ": " + e.what());
    return status_of(e);
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return LSAMGDD_ERR_ERROR;
  }
}

SparseMatrix from_csr(const lsamgdd_csr* g) {
  std::vector<std::size_t> offs(g->n_rows + 1), cols(g->nnz);
  std::vector<double> vals(g->values, g->values + g->nnz);
  for (int64_t i = 0; i <= g->n_rows; ++i) offs[i] = static_cast<std::size_t>(g->row_offsets[i]);
  for (int64_t k = 0; k < g->nnz; ++k) cols[k] = static_cast<std::size_t>(g->col_indices[k]);
  return SparseMatrix(g->n_rows, g->n_cols, std::move(offs), std::move(cols), std::move(vals));
}

LevelParams to_params(const lsamgdd_params* p) {
  LevelParams lp;
  lp.max_levels = p->max_levels;
  lp.coarse_size = p->coarse_size;
  lp.aggregation_passes = p->aggregation_passes;
  lp.kappa = p->kappa;
  lp.must_keep = p->must_keep;
  lp.coarsening_ratios.assign(p->coarsening_ratios, p->coarsening_ratios + p->n_ratios);
  lp.pre_sweeps = p->pre_sweeps;
  lp.post_sweeps = p->post_sweeps;
  lp.gevp_variant = p->gevp_variant == 1 ? GevpVariant::WeightedLhs : GevpVariant::SchurReduced;
  return lp;
}

bool hooks_active(const lsamgdd_params* p) {
  return p->level0_partition != nullptr || p->level0_overlap >= 2 || p->thresh_override > 0.0 ||
         p->level0_max_modes > 0 || p->probe_levels > 0;
}

// Second Γ layer: every node within graph distance 2 of omega_i, outside it,
// sorted (the one-layer rule of aggregation.hpp:184-193 applied to ω ∪ Γ).
// The adjacency and greedy colouring are then recomputed on the new
// subdomains with the rule of aggregation.hpp:197-229.
void widen_overlap(const SparseMatrix& a, const Partition& p, AggregateTopology& topo) {
  const std::size_t n_agg = topo.n_aggregates();
  for (std::size_t i = 0; i < n_agg; ++i) {
    std::vector<std::size_t> g;
    auto scan = [&](std::size_t u) {
      for (std::size_t k = a.row_begin(u); k < a.row_end(u); ++k)
        if (p.assignment[a.col_index(k)] != i) g.push_back(a.col_index(k));
    };
    for (std::size_t u : topo.omega[i]) scan(u);
    for (std::size_t u : topo.gamma[i]) scan(u);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    topo.gamma[i] = std::move(g);
  }
  const std::size_t n = topo.n_nodes;
  std::vector<std::vector<std::size_t>> holders(n);
  for (std::size_t v = 0; v < n; ++v) holders[v].push_back(p.assignment[v]);
  for (std::size_t i = 0; i < n_agg; ++i)
    for (std::size_t gn : topo.gamma[i]) holders[gn].push_back(i);
  std::vector<std::vector<std::size_t>> adj(n_agg);
  for (std::size_t v = 0; v < n; ++v)
    for (std::size_t x = 0; x < holders[v].size(); ++x)
      for (std::size_t y = x + 1; y < holders[v].size(); ++y) {
        adj[holders[v][x]].push_back(holders[v][y]);
        adj[holders[v][y]].push_back(holders[v][x]);
      }
  for (auto& l : adj) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  std::vector<std::size_t> order(n_agg);
  for (std::size_t i = 0; i < n_agg; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](std::size_t x, std::size_t y) { return adj[x].size() > adj[y].size(); });
  const std::size_t none = static_cast<std::size_t>(-1);
  topo.colors.assign(n_agg, none);
  std::size_t max_color = 0;
  for (std::size_t i : order) {
    std::vector<bool> used(adj[i].size() + 1, false);
    for (std::size_t j : adj[i])
      if (topo.colors[j] != none && topo.colors[j] < used.size()) used[topo.colors[j]] = true;
    std::size_t c = 0;
    while (used[c]) ++c;
    topo.colors[i] = c;
    max_color = std::max(max_color, c);
  }
  topo.n_colors = max_color + 1;
}

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int ref_threads() {
  if (const char* e = std::getenv("LSAMGDD_REF_THREADS")) return std::max(1, std::atoi(e));
  return 1;
}

// Runs f(i) for i in [0, n) on LSAMGDD_REF_THREADS host threads (chunks of 64,
// first exception rethrown); one thread by default, like the reference.
template <class F>
void for_each_aggregate(std::size_t n, F&& f) {
  const int n_thr = ref_threads();
  if (n_thr <= 1 || n < 64) {
    for (std::size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<std::size_t> next{0};
  std::exception_ptr first_err;
  std::mutex err_mu;
  std::vector<std::thread> pool;
  for (int w = 0; w < n_thr; ++w)
    pool.emplace_back([&] {
      try {
        for (;;) {
          const std::size_t i0 = next.fetch_add(64);
          if (i0 >= n) break;
          for (std::size_t i = i0; i < std::min(n, i0 + 64); ++i) f(i);
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (!first_err) first_err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (first_err) std::rethrow_exception(first_err);
}

// build_smoother (smoother.hpp:38-58): the reference's own function on one
// thread; with LSAMGDD_REF_THREADS > 1 its per-aggregate body (subdomain,
// submatrix, factor_spd_block — the reference's functions, unchanged) runs
// on several host threads. The factors do not depend on the order.
SchwarzSmoother threaded_build_smoother(const SparseMatrix& a, const AggregateTopology& topo) {
  if (ref_threads() <= 1) return build_smoother(a, topo, SchwarzMode::RAS);
  if (a.n_rows() != a.n_cols()) throw DimError("build_smoother: matrix is not square");
  if (a.n_rows() != topo.n_nodes) throw DimError("build_smoother: topology does not cover the matrix");
  SchwarzSmoother s;
  s.mode = SchwarzMode::RAS;
  s.n = a.n_rows();
  const std::size_t n_agg = topo.n_aggregates();
  s.subdomains.resize(n_agg);
  s.omega_sizes.resize(n_agg);
  s.factors.resize(n_agg);
  for_each_aggregate(n_agg, [&](std::size_t i) {
    s.subdomains[i] = topo.subdomain(i);
    s.omega_sizes[i] = topo.omega[i].size();
    const DenseMatrix block = submatrix(a, s.subdomains[i], s.subdomains[i]);
    s.factors[i] = factor_spd_block(block, "subdomain block of aggregate " + std::to_string(i));
  });
  return s;
}

// Stage replica of setup() (hierarchy.hpp:106-200) with the config hooks.
void replica_setup(RefHandle& rh, const lsamgdd_params* cp) {
  const LevelParams params = to_params(cp);
  if (params.max_levels < 2) throw InputError("setup: max_levels must be at least 2");
  if (params.coarse_size < 1) throw InputError("setup: coarse_size must be positive");
  if (params.aggregation_passes < 1) throw InputError("setup: aggregation_passes must be positive");
  if (!(params.kappa > 1.0)) throw InputError("setup: kappa must exceed 1");
  if (!(params.must_keep > 1.0)) throw InputError("setup: must_keep must exceed 1");
  if (params.coarsening_ratios.empty()) throw InputError("setup: coarsening_ratios must not be empty");
  for (std::size_t c : params.coarsening_ratios)
    if (c < 2) throw InputError("setup: coarsening ratios must be at least 2");
  const SparseMatrix& g0 = rh.g0;
  if (g0.n_rows() == 0 || g0.n_cols() == 0) throw InputError("setup: factor is empty");

  Hierarchy& h = rh.h;
  h.params = params;
  auto t = std::chrono::steady_clock::now();
  Level level;
  level.G = g0;
  level.A = spgemm(transpose(g0), g0, SpgemmMode::Symbolic);
  h.levels.push_back(std::move(level));
  rh.timings.push_back({"galerkin_A0", secs_since(t)});

  const std::size_t probe = static_cast<std::size_t>(cp->probe_levels);
  while (h.levels.size() < params.max_levels && h.levels.back().A.n_rows() > params.coarse_size &&
         (probe == 0 || h.levels.size() <= probe)) {
    const std::size_t ell = h.levels.size() - 1;
    Level& cur = h.levels.back();
    t = std::chrono::steady_clock::now();
    Partition part;
    if (ell == 0 && cp->level0_partition) {
      part.n_aggregates = static_cast<std::size_t>(cp->level0_n_aggregates);
      part.assignment.resize(cur.A.n_rows());
      for (std::size_t v = 0; v < part.assignment.size(); ++v)
        part.assignment[v] = static_cast<std::size_t>(cp->level0_partition[v]);
    } else {
      part = multi_pass_aggregation(cur.A, params.aggregation_passes);
    }
    cur.topology = build_topology(cur.A, part);
    if (ell == 0 && cp->level0_overlap >= 2) widen_overlap(cur.A, part, cur.topology);
    rh.timings.push_back({"aggregation_topology", secs_since(t)});
    t = std::chrono::steady_clock::now();
    cur.smoother = threaded_build_smoother(cur.A, cur.topology);
    rh.timings.push_back({"build_smoother", secs_since(t)});
    t = std::chrono::steady_clock::now();
    const RowSets rs = compute_row_sets(cur.G, cur.topology);
    rh.multiplicity.push_back(rs.multiplicity);
    cur.thresh = cp->thresh_override > 0.0
                     ? cp->thresh_override
                     : eigen_threshold(params.kappa, cur.topology.n_colors, cur.topology.multiplicity_max);
    const std::size_t ratio =
        params.coarsening_ratios[std::min(ell, params.coarsening_ratios.size() - 1)];
    std::vector<DenseMatrix> panels(cur.topology.n_aggregates());
    rh.spectra.emplace_back();
    auto& spec = rh.spectra.back();
    if (cp->keep_spectra) spec.resize(cur.topology.n_aggregates());
    // The per-aggregate problems are independent (splitting.hpp:200-275 reads shared
    // data only); LSAMGDD_REF_THREADS > 1 runs the reference's own functions on
    // several host threads (the reference-arm timing). The default is the
    // reference's single thread.
    auto one = [&](std::size_t i) {
      const LocalBlocks blocks = assemble_local(i, cur.G, cur.topology, rs);
      std::size_t cap = cur.topology.omega[i].size();
      if (ell > 0) {
        cap = cur.topology.omega[i].size() / ratio;
        if (cap == 0) cap = 1;
      } else if (cp->level0_max_modes > 0) {
        cap = cp->level0_max_modes;
      }
      panels[i] = local_gevp(i, blocks, cur.thresh, cap, params.gevp_variant,
                             cp->keep_spectra ? &spec[i] : nullptr, params.must_keep);
    };
    for_each_aggregate(cur.topology.n_aggregates(), one);
    rh.timings.push_back({"local_gevp", secs_since(t)});
    t = std::chrono::steady_clock::now();
    cur.P = assemble_P(cur.topology, panels);
    cur.has_interpolation = true;
    Level next;
    next.G = spgemm(cur.G, cur.P, SpgemmMode::Symbolic);
    next.A = spgemm(transpose(next.G), next.G, SpgemmMode::Symbolic);
    rh.timings.push_back({"galerkin", secs_since(t)});
    if (next.A.n_rows() >= cur.A.n_rows())
      throw SetupError("setup: stagnant coarsening at level " + std::to_string(ell) + " (" +
                       std::to_string(cur.A.n_rows()) + " -> " + std::to_string(next.A.n_rows()) + ")");
    LevelSummary row;
    row.level = ell;
    row.dim = cur.A.n_rows();
    row.nnz = cur.A.nnz();
    row.n_aggregates = cur.topology.n_aggregates();
    row.k_c = cur.topology.n_colors;
    row.n_mult = cur.topology.multiplicity_max;
    row.thresh = cur.thresh;
    row.modes_kept = cur.P.n_cols();
    h.summary.push_back(row);
    h.levels.push_back(std::move(next));
  }
  t = std::chrono::steady_clock::now();
  const Level& coarse = h.levels.back();
  if (probe == 0) {  // probe_levels: stage-wise runs of the fine levels stop before the dense coarsest factor
    h.coarse_factor = factor_spd_block(to_dense(coarse.A), "coarsest-level matrix");
    rh.timings.push_back({"coarse_factor", secs_since(t)});
  }
  LevelSummary last;
  last.level = h.levels.size() - 1;
  last.dim = coarse.A.n_rows();
  last.nnz = coarse.A.nnz();
  h.summary.push_back(last);
}

void export_csr(const SparseMatrix& m, int64_t sizes[3], int64_t* idx0, int64_t* idx1, double* vals) {
  sizes[0] = m.n_rows();
  sizes[1] = m.n_cols();
  sizes[2] = m.nnz();
  if (idx0)
    for (std::size_t i = 0; i <= m.n_rows(); ++i) idx0[i] = m.row_offsets()[i];
  if (idx1)
    for (std::size_t k = 0; k < m.nnz(); ++k) idx1[k] = m.col_indices()[k];
  if (vals) std::memcpy(vals, m.values().data(), m.nnz() * sizeof(double));
}

}  // namespace

extern "C" {

// plain = 1 forces the reference's own setup() (no replica; hooks rejected).
int ref_setup(const lsamgdd_csr* g0, const lsamgdd_params* p, int32_t plain, void** out, char* err,
              size_t errlen) {
  *out = nullptr;
  auto rh = std::make_unique<RefHandle>();
  const int st = guarded(err, errlen, [&] {
    rh->g0 = from_csr(g0);
    if (plain) {
      if (hooks_active(p)) throw InputError("ref_setup: plain setup() takes no config hooks");
      const auto t = std::chrono::steady_clock::now();
      rh->h = setup(rh->g0, to_params(p));
      rh->timings.push_back({"setup", secs_since(t)});
    } else {
      replica_setup(*rh, p);
    }
  });
  if (st == LSAMGDD_OK) *out = rh.release();
  return st;
}

int ref_destroy(void* h) {
  delete static_cast<RefHandle*>(h);
  return LSAMGDD_OK;
}

int ref_num_levels(const void* h, int64_t* out) {
  *out = static_cast<int64_t>(static_cast<const RefHandle*>(h)->h.levels.size());
  return LSAMGDD_OK;
}

int ref_level_summary(const void* vh, int64_t level, lsamgdd_level_summary* out) {
  const Hierarchy& h = static_cast<const RefHandle*>(vh)->h;
  if (level < 0 || static_cast<std::size_t>(level) >= h.summary.size()) return LSAMGDD_ERR_INDEX;
  const LevelSummary& s = h.summary[level];
  out->level = s.level;
  out->dim = s.dim;
  out->nnz = s.nnz;
  out->n_aggregates = s.n_aggregates;
  out->k_c = s.k_c;
  out->n_mult = s.n_mult;
  out->thresh = s.thresh;
  out->modes_kept = s.modes_kept;
  return LSAMGDD_OK;
}

int ref_operator_complexity(const void* vh, double* out) {
  *out = operator_complexity(static_cast<const RefHandle*>(vh)->h);
  return LSAMGDD_OK;
}

int ref_level_export(const void* vh, int64_t level, int32_t what, int64_t sizes[3], int64_t* idx0,
                     int64_t* idx1, double* vals) {
  const RefHandle& rh = *static_cast<const RefHandle*>(vh);
  const Hierarchy& h = rh.h;
  if (level < 0 || static_cast<std::size_t>(level) >= h.levels.size()) return LSAMGDD_ERR_INDEX;
  const Level& L = h.levels[level];
  sizes[0] = sizes[1] = sizes[2] = 0;
  switch (what) {
    case LSAMGDD_EXPORT_A: export_csr(L.A, sizes, idx0, idx1, vals); return LSAMGDD_OK;
    case LSAMGDD_EXPORT_G: export_csr(L.G, sizes, idx0, idx1, vals); return LSAMGDD_OK;
    case LSAMGDD_EXPORT_P:
      if (!L.has_interpolation) return LSAMGDD_ERR_INDEX;
      export_csr(L.P, sizes, idx0, idx1, vals);
      return LSAMGDD_OK;
    default: break;
  }
  if (!L.has_interpolation) return LSAMGDD_ERR_INDEX;
  const AggregateTopology& t = L.topology;
  switch (what) {
    case LSAMGDD_EXPORT_PARTITION:
      sizes[0] = t.n_nodes;
      sizes[1] = t.n_aggregates();
      if (idx0)
        for (std::size_t i = 0; i < t.n_aggregates(); ++i)
          for (std::size_t v : t.omega[i]) idx0[v] = i;
      return LSAMGDD_OK;
    case LSAMGDD_EXPORT_GAMMA: {
      sizes[0] = t.n_aggregates();
      int64_t tot = 0;
      for (const auto& g : t.gamma) tot += g.size();
      sizes[1] = tot;
      int64_t o = 0;
      for (std::size_t i = 0; i < t.n_aggregates(); ++i) {
        if (idx0) idx0[i] = o;
        for (std::size_t v : t.gamma[i]) {
          if (idx1) idx1[o] = v;
          ++o;
        }
      }
      if (idx0) idx0[t.n_aggregates()] = o;
      return LSAMGDD_OK;
    }
    case LSAMGDD_EXPORT_COLORS:
      sizes[0] = t.n_aggregates();
      sizes[1] = t.n_colors;
      if (idx0)
        for (std::size_t i = 0; i < t.n_aggregates(); ++i) idx0[i] = t.colors[i];
      return LSAMGDD_OK;
    case LSAMGDD_EXPORT_SPECTRA: {
      if (static_cast<std::size_t>(level) >= rh.spectra.size()) return LSAMGDD_ERR_INDEX;
      const auto& sp = rh.spectra[level];
      sizes[0] = sp.size();
      int64_t tot = 0;
      for (const auto& s : sp) tot += s.size();
      sizes[1] = tot;
      int64_t o = 0;
      for (std::size_t i = 0; i < sp.size(); ++i) {
        if (idx0) idx0[i] = o;
        for (double v : sp[i]) {
          if (vals) vals[o] = v;
          ++o;
        }
      }
      if (idx0) idx0[sp.size()] = o;
      return LSAMGDD_OK;
    }
    case LSAMGDD_EXPORT_MULTIPLICITY: {
      if (static_cast<std::size_t>(level) >= rh.multiplicity.size()) return LSAMGDD_ERR_INDEX;
      const auto& m = rh.multiplicity[level];
      sizes[0] = m.size();
      sizes[1] = t.multiplicity_max;
      if (idx0)
        for (std::size_t j = 0; j < m.size(); ++j) idx0[j] = m[j];
      return LSAMGDD_OK;
    }
    default: return LSAMGDD_ERR_INPUT;
  }
}

int ref_vcycle(const void* vh, int64_t level, const double* r, double* e, char* err, size_t errlen) {
  const Hierarchy& h = static_cast<const RefHandle*>(vh)->h;
  return guarded(err, errlen, [&] {
    if (level < 0 || static_cast<std::size_t>(level) >= h.levels.size())
      throw IndexError("vcycle: level out of range");
    const std::size_t n = h.levels[level].A.n_rows();
    const Vector out = vcycle(h, level, Vector(r, r + n));
    std::memcpy(e, out.data(), n * sizeof(double));
  });
}

int ref_schwarz_apply(const void* vh, int64_t level, int32_t mode, const double* r, double* e,
                      char* err, size_t errlen) {
  const Hierarchy& h = static_cast<const RefHandle*>(vh)->h;
  return guarded(err, errlen, [&] {
    if (level < 0 || static_cast<std::size_t>(level) + 1 >= h.levels.size())
      throw IndexError("schwarz: level has no smoother");
    const SchwarzSmoother& s = h.levels[level].smoother;
    const SchwarzMode m = mode == 0 ? SchwarzMode::RAS : mode == 1 ? SchwarzMode::RAST : SchwarzMode::ASM;
    const Vector out = apply(s, Vector(r, r + s.n), m);
    std::memcpy(e, out.data(), s.n * sizeof(double));
  });
}

int ref_level_spmv(const void* vh, int64_t level, int32_t what, int32_t trans, const double* x,
                   double* y, char* err, size_t errlen) {
  const Hierarchy& h = static_cast<const RefHandle*>(vh)->h;
  return guarded(err, errlen, [&] {
    if (level < 0 || static_cast<std::size_t>(level) >= h.levels.size())
      throw IndexError("spmv: level out of range");
    const Level& L = h.levels[level];
    const SparseMatrix& m = what == 0 ? L.A : what == 1 ? L.G : L.P;
    const std::size_t nin = trans ? m.n_rows() : m.n_cols();
    const Vector out = trans ? spmv_transpose(m, Vector(x, x + nin)) : spmv(m, Vector(x, x + nin));
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  });
}

// pcg with the factored operator apply_a = Gᵀ(G·) (lsamgdd_cli.cpp:137-142).
int ref_pcg(const void* vh, const lsamgdd_csr* g, const double* b, double tol, uint64_t maxit,
            double* x, lsamgdd_report* rep, char* err, size_t errlen) {
  const RefHandle& rh = *static_cast<const RefHandle*>(vh);
  return guarded(err, errlen, [&] {
    SparseMatrix gown;
    if (g) gown = from_csr(g);
    const SparseMatrix& G = g ? gown : rh.g0;
    const auto apply_a = [&G](const Vector& v) { return spmv_transpose(G, spmv(G, v)); };
    const auto apply_b = [&rh](const Vector& r) { return vcycle(rh.h, r); };
    const std::size_t n = G.n_cols();
    const auto t = std::chrono::steady_clock::now();
    auto solved = pcg(apply_a, apply_b, Vector(b, b + n), tol, maxit);
    const double secs = secs_since(t);
    std::memcpy(x, solved.first.data(), n * sizeof(double));
    if (rep) {
      const SolveReport& s = solved.second;
      rep->iterations = s.iterations;
      rep->converged = s.converged ? 1 : 0;
      rep->avg_conv_factor = s.avg_conv_factor;
      rep->iters_to_tenth = s.iters_to_tenth;
      rep->operator_complexity = operator_complexity(rh.h);
      rep->solve_seconds = secs;
      rep->history_len = s.residual_history.size();
      if (rep->residual_history)
        for (std::size_t k = 0; k < s.residual_history.size() && k < rep->history_capacity; ++k)
          rep->residual_history[k] = s.residual_history[k];
    }
  });
}

int ref_setup_timings(const void* vh, const char** names, double* secs, int64_t n, int64_t* count) {
  const RefHandle& rh = *static_cast<const RefHandle*>(vh);
  *count = static_cast<int64_t>(rh.timings.size());
  for (int64_t i = 0; i < n && i < *count; ++i) {
    names[i] = rh.timings[i].first.c_str();
    secs[i] = rh.timings[i].second;
  }
  return LSAMGDD_OK;
}

// ---- unit-level entry points (pins of the oracle's building blocks) ----

// sym_eig (eigen.hpp:35): values ascending, vectors column k (row-major n×n).
int ref_sym_eig(int64_t n, const double* a, double* values, double* vectors, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    DenseMatrix m(n, n);
    std::memcpy(m.values().data(), a, n * n * sizeof(double));
    const EigenPairs e = sym_eig(m);
    std::memcpy(values, e.values.data(), n * sizeof(double));
    std::memcpy(vectors, e.vectors.values().data(), n * n * sizeof(double));
  });
}

// spsd_gevp (eigen.hpp:142): returns count in *k, vectors n×k row-major.
int ref_spsd_gevp(int64_t n, const double* l, const double* b, double tau, double* values,
                  double* vectors, int64_t* k, int64_t* discarded, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    DenseMatrix L(n, n), B(n, n);
    std::memcpy(L.values().data(), l, n * n * sizeof(double));
    std::memcpy(B.values().data(), b, n * n * sizeof(double));
    const EigenPairs e = spsd_gevp(L, B, tau);
    *k = static_cast<int64_t>(e.values.size());
    *discarded = static_cast<int64_t>(e.discarded);
    std::memcpy(values, e.values.data(), e.values.size() * sizeof(double));
    std::memcpy(vectors, e.vectors.values().data(), e.vectors.values().size() * sizeof(double));
  });
}

int ref_pseudo_inverse(int64_t n, const double* a, double tau, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    DenseMatrix m(n, n);
    std::memcpy(m.values().data(), a, n * n * sizeof(double));
    const DenseMatrix p = pseudo_inverse(m, tau);
    std::memcpy(out, p.values().data(), n * n * sizeof(double));
  });
}

// standard_aggregation (aggregation.hpp:71) on a square CSR.
int ref_standard_aggregation(const lsamgdd_csr* a, int64_t* assignment, int64_t* n_agg, char* err,
                             size_t errlen) {
  return guarded(err, errlen, [&] {
    const Partition p = standard_aggregation(from_csr(a));
    for (std::size_t v = 0; v < p.assignment.size(); ++v) assignment[v] = p.assignment[v];
    *n_agg = p.n_aggregates;
  });
}

int ref_eigen_threshold(double kappa, int64_t kc, int64_t n_mult, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { *out = eigen_threshold(kappa, kc, n_mult); });
}

// mmio.hpp round trips for the tests of paper_2601_04112_b200/mmio.py
int ref_mm_write(const lsamgdd_csr* m, const char* path, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { mm_write(path, from_csr(m)); });
}

int ref_mm_read(const char* path, int64_t sizes[3], int64_t* off, int64_t* col, double* val, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { export_csr(mm_read(path), sizes, off, col, val); });
}

int ref_mm_write_vector(const double* v, int64_t n, const char* path, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { mm_write_vector(path, Vector(v, v + n)); });
}

int ref_mm_read_vector(const char* path, int64_t* n, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const Vector v = mm_read_vector(path);
    *n = static_cast<int64_t>(v.size());
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

void ref_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(gen);
}

}  // extern "C"
