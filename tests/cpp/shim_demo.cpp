// Compiles the C++ drop-in shim against the reference's own headers and links
// the B200 library: the acceptance.cpp-style caller (acceptance.cpp:82-103)
// with lsamgdd::b200 in place of the reference's setup/vcycle/pcg.
#include <cmath>
#include <cstdio>

#include "lsamgdd_b200/lsamgdd.hpp"

// build_rotated_aniso's factor (problems.hpp:84-132) as stencil rows for the on-device generator: two
// rows per node, entries (0,0), (+1,0), (0,+1) with the reference's own coefficient arithmetic.
static lsamgdd::b200::DeviceFactor device_rotated_aniso(const lsamgdd::AnisoParams& p) {
  const double c = std::cos(p.theta), s = std::sin(p.theta);
  const double se = std::sqrt(p.epsilon);
  const double bmat_t[4] = {se * c, se * s, -s, c};
  std::vector<int32_t> off;
  std::vector<double> coef;
  for (int r = 0; r < 2; ++r) {
    const double cx = bmat_t[2 * r] / p.hx();
    const double cy = bmat_t[2 * r + 1] / p.hy();
    const int32_t o[9] = {0, 0, 0, 1, 0, 0, 0, 1, 0};
    off.insert(off.end(), o, o + 9);
    coef.insert(coef.end(), {-cx - cy, cx, cy});
  }
  return lsamgdd::b200::DeviceFactor({static_cast<int64_t>(p.nx), static_cast<int64_t>(p.ny), 1}, 2, 3, off, coef);
}

static bool same_matrix(const lsamgdd::SparseMatrix& a, const lsamgdd::SparseMatrix& b) {
  return a.n_rows() == b.n_rows() && a.n_cols() == b.n_cols() && a.row_offsets() == b.row_offsets() &&
         a.col_indices() == b.col_indices() && a.values() == b.values();
}

int main() {
  lsamgdd::AnisoParams ap;
  ap.nx = ap.ny = 16;
  ap.epsilon = 1e-2;
  ap.theta = 0.5;
  const auto sys = lsamgdd::build_rotated_aniso(ap);
  lsamgdd::LevelParams params;
  params.coarse_size = 30;
  try {
    const auto h = lsamgdd::b200::setup(sys.G, params);
    auto [x, rep] = lsamgdd::b200::pcg(h, sys.G, sys.rhs, 1e-8, 1000);
    // cross-check against the reference path on the same inputs
    const lsamgdd::Hierarchy hr = lsamgdd::setup(sys.G, params);
    const auto apply_a = [&](const lsamgdd::Vector& v) { return lsamgdd::spmv_transpose(sys.G, lsamgdd::spmv(sys.G, v)); };
    const auto apply_b = [&](const lsamgdd::Vector& r) { return lsamgdd::vcycle(hr, r); };
    auto [xr, repr] = lsamgdd::pcg(apply_a, apply_b, sys.rhs, 1e-8, 1000);
    std::printf("device iterations %zu reference %zu opcx %.6f ref %.6f\n", rep.iterations, repr.iterations,
                lsamgdd::b200::operator_complexity(h), lsamgdd::operator_complexity(hr));
    if (rep.iterations != repr.iterations) return 1;
    // the factor generated on the device equals the reference generator's, bit for bit (also with
    // theta = 0, where the exact-zero coefficients are dropped), and solves the same way
    const lsamgdd::b200::DeviceFactor gd = device_rotated_aniso(ap);
    if (!same_matrix(gd.to_host(), sys.G)) {
      std::printf("device-generated factor differs from build_rotated_aniso\n");
      return 4;
    }
    lsamgdd::AnisoParams ap0 = ap;
    ap0.theta = 0.0;
    ap0.nx = 7;
    if (!same_matrix(device_rotated_aniso(ap0).to_host(), lsamgdd::build_rotated_aniso(ap0).G)) {
      std::printf("device-generated factor (theta = 0) differs from build_rotated_aniso\n");
      return 5;
    }
    const auto hd = lsamgdd::b200::setup(gd, params);
    auto [xd, repd] = lsamgdd::b200::pcg(hd, sys.rhs, 1e-8, 1000);
    std::printf("device-generated factor: iterations %zu, x identical %d\n", repd.iterations, int(xd == x));
    return (repd.iterations == rep.iterations && xd == x) ? 0 : 6;
  } catch (const lsamgdd::Error& e) {
    std::printf("%s: %s\n", e.name(), e.what());
    return 3;
  }
}
