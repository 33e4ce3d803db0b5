// hierarchy.cuh — the multilevel hierarchy (Hierarchy/Level of
// hierarchy.hpp:46-64) owned by one C-ABI handle: device operators, host
// mirrors of the topology, and the setup / vcycle / pcg drivers.
#pragma once

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "setup_kernels.cuh"
#include "solve.cuh"
#include "sparse.cuh"

namespace lsb {

struct HostCsr {
  int64_t nr = 0, nc = 0;
  std::vector<int64_t> off, col;
  std::vector<double> val;
};

struct Level {
  DevCsr A, G, P;
  Sell A_sell;
  bool has_interp = false;
  double thresh = 0.0;
  // topology (host mirror + device copy)
  std::vector<int32_t> h_omega_off, h_omega, h_gamma_off, h_gamma;
  std::vector<int64_t> colors;
  int64_t n_colors = 0, n_mult = 0;
  DevTopo topo;
  DevSmoother sm;
  DevInterp ip;
  DBuf<int32_t> col_agg;  // coarse column -> aggregate
  DBuf<int32_t> mult;     // row multiplicities of G (export)
  SchwarzView schwarz_view() const;
  InterpView interp_view() const;
};

struct StageTime {
  std::string name;
  double ms;
};

struct Hierarchy {
  std::vector<Level> levels;
  DBuf<double> coarse_inv;
  int64_t n_coarse = 0;
  bool probe = false;  // built with probe_levels: no coarsest factorisation, no cycles
  lsamgdd_params params{};
  std::vector<uint64_t> ratios;
  std::vector<lsamgdd_level_summary> summary;
  DevCsr g0;           // the factor given to setup (pcg's default operator)
  Sell g0_sell, g0t_sell;
  std::vector<StageTime> timings;
  int device = 0;
  cudaStream_t stream = nullptr;  // setup stream
  cudaStream_t side_stream = nullptr;  // Schwarz-block factorisations (owns the smoothers' buffers)
  mutable std::mutex mu;          // guards lazily built export caches
  ~Hierarchy();
};

// build_smoother(a, topo) on a caller matrix and topology (smoother.hpp:38-58)
// without a hierarchy: the level-0-style Schwarz blocks of one operator.
struct StandaloneSmoother {
  Level L;
  DBuf<double> rast_tmp;
  int64_t n = 0;
  cudaStream_t s = nullptr;
  ~StandaloneSmoother();
};
StandaloneSmoother* make_smoother(const lsamgdd_csr* a, int64_t n_agg, const int64_t* omega_off, const int64_t* omega,
                                  const int64_t* gamma_off, const int64_t* gamma, const int64_t* colors);
// apply(smoother, r, mode) (smoother.hpp:65-83), mode 0 RAS / 1 RAS-T; device vectors, on sm.s
void smoother_apply(const StandaloneSmoother& sm, int mode, const double* r, double* e);

// parameter / input checks of setup (hierarchy.hpp:107-117), host only
void validate_setup(const lsamgdd_csr* g0, const lsamgdd_params* p);

// setup(g0, params) — hierarchy.hpp:106-200 plus the config hooks.
Hierarchy* setup(const lsamgdd_csr* g0, const lsamgdd_params* params);

// Per-call solve workspace (concurrent calls on one handle each own one).
struct SolveWs {
  cudaStream_t s = nullptr;
  std::vector<DBuf<double>> e, res, rhs;  // per level
  std::vector<DBuf<double>> rast_tmp;     // per level: Γ-contribution slots of the one-launch RAS-T
  Reducer red;
  cudaEvent_t ev[6] = {};  // level-0 RAS / RAS-T brackets, then the PCG operator Gᵀ(G p)
  bool timing = false;
  explicit SolveWs(const Hierarchy& h);
  ~SolveWs();
};

// e = vcycle(h, level, r) on device pointers (hierarchy.hpp:205-227).
void vcycle(const Hierarchy& h, SolveWs& ws, int64_t level, const double* r, double* e);

struct PcgResult {
  uint64_t iterations = 0;
  bool converged = false;
  std::vector<double> history;
  double solve_seconds = 0.0;
  int64_t launches = 0;
};
// pcg with apply_a = Gᵀ(G·), apply_b = vcycle (krylov.hpp:42-92). b, x device.
PcgResult pcg(const Hierarchy& h, SolveWs& ws, const Sell& g, const Sell& gt, const double* b, double* x,
              double tol, uint64_t maxit, lsamgdd_kernel_stats* stats);

double operator_complexity(const Hierarchy& h);

}  // namespace lsb
