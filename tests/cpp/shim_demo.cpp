// Compiles the C++ drop-in shim against the reference's own headers and links
// the B200 library: the acceptance.cpp-style caller (acceptance.cpp:82-103)
// with lsamgdd::b200 in place of the reference's setup/vcycle/pcg.
#include <cstdio>

#include "lsamgdd_b200/lsamgdd.hpp"

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
    return rep.iterations == repr.iterations ? 0 : 1;
  } catch (const lsamgdd::Error& e) {
    std::printf("%s: %s\n", e.name(), e.what());
    return 3;
  }
}
