// dense_dev.cuh — team-parallel dense kernels of dense.hpp / eigen.hpp.
//
// Every routine runs on a Team (a warp or a CTA, common.cuh) over matrices in
// a per-problem workspace (shared or global memory). Parallelism is only over
// independent outputs; every reduction keeps the reference's sequential
// order, and the library is compiled with --fmad=false, so results are
// bit-identical to the reference's no-FMA build:
//   * matmul / matmul_transa / weighted Gram: one output per thread, the sum
//     over k in ascending order with the reference's zero-skip rule;
//   * cyclic Jacobi: the rotation sequence is inherently sequential, each
//     rotation updates O(n) disjoint entries in parallel (eigen.hpp:85-93
//     touches rows/columns p and q only), two team barriers per rotation.
#pragma once

#include "common.cuh"

namespace lsb {

// Deterministic bump allocator over a workspace. All team threads perform
// the same take() sequence, so they agree on every pointer.
struct Arena {
  double* base;
  int64_t used;
  __device__ double* take(int64_t n) {
    double* p = base + used;
    used += (n + 1) & ~int64_t(1);
    return p;
  }
  __device__ int* take_int(int64_t n) { return reinterpret_cast<int*>(take((n + 1) / 2)); }
};

// workspace doubles needed by t_sym_eig (excluding its outputs)
__host__ __device__ inline int64_t sym_eig_scratch(int64_t n) {
  return 2 * ((n * n + 1) & ~int64_t(1)) + 3 * ((n + 1) & ~int64_t(1)) + 4;
}

template <class Team>
__device__ void t_copy(const Team& t, double* dst, const double* src, int64_t cnt) {
  for (int64_t i = t.rank(); i < cnt; i += t.size()) dst[i] = src[i];
  t.sync();
}

template <class Team>
__device__ void t_fill(const Team& t, double* dst, double v, int64_t cnt) {
  for (int64_t i = t.rank(); i < cnt; i += t.size()) dst[i] = v;
  t.sync();
}

// a <- (a + aᵀ)/2                                           dense.hpp:103-111
template <class Team>
__device__ void t_symmetrize(const Team& t, double* a, int n) {
  const int64_t pairs = int64_t(n) * n;
  for (int64_t e = t.rank(); e < pairs; e += t.size()) {
    const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    if (j <= i) continue;
    const double m = 0.5 * (a[int64_t(i) * n + j] + a[int64_t(j) * n + i]);
    a[int64_t(i) * n + j] = m;
    a[int64_t(j) * n + i] = m;
  }
  t.sync();
}

// c(ar×bc) = a(ar×ac)·b(ac×bc), skipping a(i,k) == 0        dense.hpp:47-59
template <class Team>
__device__ void t_matmul(const Team& t, const double* a, int ar, int ac, const double* b, int bc, double* c) {
  const int64_t cnt = int64_t(ar) * bc;
  for (int64_t e = t.rank(); e < cnt; e += t.size()) {
    const int i = static_cast<int>(e / bc), j = static_cast<int>(e % bc);
    double s = 0.0;
    for (int k = 0; k < ac; ++k) {
      const double aik = a[int64_t(i) * ac + k];
      if (aik == 0.0) continue;
      s += aik * b[int64_t(k) * bc + j];
    }
    c[e] = s;
  }
  t.sync();
}

// c(ac×bc) = a(ar×ac)ᵀ·b(ar×bc), skipping a(k,i) == 0       dense.hpp:62-74
template <class Team>
__device__ void t_matmul_transa(const Team& t, const double* a, int ar, int ac, const double* b, int bc, double* c) {
  const int64_t cnt = int64_t(ac) * bc;
  for (int64_t e = t.rank(); e < cnt; e += t.size()) {
    const int i = static_cast<int>(e / bc), j = static_cast<int>(e % bc);
    double s = 0.0;
    for (int k = 0; k < ar; ++k) {
      const double aki = a[int64_t(k) * ac + i];
      if (aki == 0.0) continue;
      s += aki * b[int64_t(k) * bc + j];
    }
    c[e] = s;
  }
  t.sync();
}

// Sequential reductions by rank 0, broadcast through *slot.
template <class Team>
__device__ double t_seq_dot(const Team& t, const double* x, const double* y, int n, double* slot) {
  if (t.rank() == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * y[i];
    *slot = s;
  }
  t.sync();
  const double v = *slot;
  t.sync();
  return v;
}

// Cyclic Jacobi eigendecomposition (eigen.hpp:35-118): values ascending,
// vecs(i,k) = vecs[i*n+k] is eigenvector k. Returns 0, or 1 (no convergence
// in 64 sweeps) / 2 (non-finite value) for EigError.
template <class Team>
__device__ int t_sym_eig(const Team& t, int n, const double* m, double* vals, double* vecs, Arena ar) {
  const int64_t nn = int64_t(n) * n;
  for (int64_t e = t.rank(); e < nn; e += t.size()) vecs[e] = (e / n == e % n) ? 1.0 : 0.0;
  if (n == 0) {
    t.sync();
    return 0;
  }
  double* a = ar.take(nn);
  double* v = ar.take(nn);
  double* d = ar.take(n);
  double* bb = ar.take(n);
  double* z = ar.take(n);
  double* slot = ar.take(4);
  for (int64_t e = t.rank(); e < nn; e += t.size()) {
    a[e] = m[e];
    v[e] = (e / n == e % n) ? 1.0 : 0.0;
  }
  t.sync();
  t_symmetrize(t, a, n);
  for (int i = t.rank(); i < n; i += t.size()) {
    d[i] = bb[i] = a[int64_t(i) * n + i];
    z[i] = 0.0;
  }
  t.sync();
  bool converged = false;
  for (int sweep = 0; sweep < 64; ++sweep) {
    if (t.rank() == 0) {
      double sm = 0.0;
      for (int p = 0; p + 1 < n; ++p)
        for (int q = p + 1; q < n; ++q) sm += fabs(a[int64_t(p) * n + q]);
      slot[0] = sm;
    }
    t.sync();
    const double sm = slot[0];
    if (sm == 0.0) {
      converged = true;
      break;
    }
    const double tresh = sweep < 3 ? 0.2 * sm / static_cast<double>(static_cast<uint64_t>(n) * n) : 0.0;
    for (int p = 0; p + 1 < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[int64_t(p) * n + q];
        const double dp = d[p], dq = d[q];
        const double g = 100.0 * fabs(apq);
        if (sweep > 3 && fabs(dp) + g == fabs(dp) && fabs(dq) + g == fabs(dq)) {
          t.sync();
          if (t.rank() == 0) a[int64_t(p) * n + q] = 0.0;
          t.sync();
        } else if (fabs(apq) > tresh) {
          double h = dq - dp;
          double tt;
          if (fabs(h) + g == fabs(h)) {
            tt = apq / h;
          } else {
            const double theta = 0.5 * h / apq;
            tt = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
            if (theta < 0.0) tt = -tt;
          }
          const double c = 1.0 / sqrt(1.0 + tt * tt);
          const double s = tt * c;
          const double tau = s / (1.0 + c);
          h = tt * apq;
          t.sync();  // everyone has read apq, d[p], d[q]
          if (t.rank() == 0) {
            z[p] -= h;
            z[q] += h;
            d[p] -= h;
            d[q] += h;
            a[int64_t(p) * n + q] = 0.0;
          }
          for (int j = t.rank(); j < n; j += t.size()) {
            double *x = nullptr, *y = nullptr;
            if (j < p) {
              x = &a[int64_t(j) * n + p];
              y = &a[int64_t(j) * n + q];
            } else if (j > p && j < q) {
              x = &a[int64_t(p) * n + j];
              y = &a[int64_t(j) * n + q];
            } else if (j > q) {
              x = &a[int64_t(p) * n + j];
              y = &a[int64_t(q) * n + j];
            }
            if (x) {
              const double gx = *x, hy = *y;
              *x = gx - s * (hy + gx * tau);
              *y = hy + s * (gx - hy * tau);
            }
            double* vx = &v[int64_t(j) * n + p];
            double* vy = &v[int64_t(j) * n + q];
            const double gx = *vx, hy = *vy;
            *vx = gx - s * (hy + gx * tau);
            *vy = hy + s * (gx - hy * tau);
          }
          t.sync();
        }
      }
    }
    for (int i = t.rank(); i < n; i += t.size()) {
      bb[i] += z[i];
      d[i] = bb[i];
      z[i] = 0.0;
    }
    t.sync();
  }
  if (!converged) return 1;
  for (int i = 0; i < n; ++i)
    if (!isfinite(d[i])) return 2;
  // stable ascending sort (std::stable_sort, eigen.hpp:107-116)
  for (int k = t.rank(); k < n; k += t.size()) {
    const double dk = d[k];
    int pos = 0;
    for (int i = 0; i < n; ++i)
      if (d[i] < dk || (d[i] == dk && i < k)) ++pos;
    vals[pos] = dk;
    for (int i = 0; i < n; ++i) vecs[int64_t(i) * n + pos] = v[int64_t(i) * n + k];
  }
  t.sync();
  return 0;
}

// Spectral pseudo-inverse with a relative cut (eigen.hpp:215-231).
template <class Team>
__device__ int t_pseudo_inverse(const Team& t, int n, const double* m, double tau_rel, double* out, Arena ar) {
  double* ev = ar.take(n);
  double* eV = ar.take(int64_t(n) * n);
  const int st = t_sym_eig(t, n, m, ev, eV, ar);
  if (st) return st;
  const double cut = n == 0 ? 0.0 : tau_rel * fmax(ev[n - 1], 0.0);
  const int64_t nn = int64_t(n) * n;
  for (int64_t e = t.rank(); e < nn; e += t.size()) {
    const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    double s = 0.0;
    for (int k = 0; k < n; ++k) {
      if (ev[k] <= cut) continue;
      const double inv = 1.0 / ev[k];
      const double vik = eV[int64_t(i) * n + k] * inv;
      if (vik == 0.0) continue;
      s += vik * eV[int64_t(j) * n + k];
    }
    out[e] = s;
  }
  t.sync();
  return 0;
}

// Generalized SPSD pencil l u = λ b u (eigen.hpp:142-209). ls and bs are
// symmetrized in place. Outputs: values[cnt] and vectors column-major
// (vector k at outv + k*n). Returns status; *cnt and *discarded via slots.
template <class Team>
__device__ int t_spsd_gevp(const Team& t, int n, double* ls, double* bs, double tau_rel, double* values,
                           double* outv, int* cnt_out, Arena ar) {
  *cnt_out = 0;
  if (n == 0) return 0;
  t_symmetrize(t, ls, n);
  t_symmetrize(t, bs, n);
  double* ebv = ar.take(n);
  double* ebV = ar.take(int64_t(n) * n);
  double* slot = ar.take(4);
  int st = t_sym_eig(t, n, bs, ebv, ebV, ar);
  if (st) return st;
  const double mu_max = fmax(ebv[n - 1], 0.0);
  const double cut = tau_rel * mu_max;
  int n_null = 0;
  while (n_null < n && ebv[n_null] <= cut) ++n_null;
  const int n_ret = n - n_null;
  if (t.rank() == 0) {  // frobenius_norm (dense.hpp:96-100)
    double s = 0.0;
    for (int64_t e = 0; e < int64_t(n) * n; ++e) s += ls[e] * ls[e];
    slot[0] = sqrt(s);
  }
  t.sync();
  const double l_scale = slot[0];
  int cnt = 0;
  if (n_null > 0) {
    Arena a2 = ar;
    double* vn = a2.take(int64_t(n) * n_null);
    double* lv = a2.take(int64_t(n) * n_null);
    double* tm = a2.take(int64_t(n_null) * n_null);
    double* etv = a2.take(n_null);
    double* etV = a2.take(int64_t(n_null) * n_null);
    for (int64_t e = t.rank(); e < int64_t(n) * n_null; e += t.size()) {
      const int i = static_cast<int>(e / n_null), k = static_cast<int>(e % n_null);
      vn[e] = ebV[int64_t(i) * n + k];
    }
    t.sync();
    t_matmul(t, ls, n, n, vn, n_null, lv);
    t_matmul_transa(t, vn, n, n_null, lv, n_null, tm);
    t_symmetrize(t, tm, n_null);
    st = t_sym_eig(t, n_null, tm, etv, etV, a2);
    if (st) return st;
    for (int k = n_null; k-- > 0;) {
      if (etv[k] > tau_rel * l_scale) {
        double* u = outv + int64_t(cnt) * n;
        for (int i = t.rank(); i < n; i += t.size()) {
          double s = 0.0;
          for (int j = 0; j < n_null; ++j) s += vn[int64_t(i) * n_null + j] * etV[int64_t(j) * n_null + k];
          u[i] = s;
        }
        if (t.rank() == 0) values[cnt] = __longlong_as_double(0x7ff0000000000000LL);
        ++cnt;
      }
    }
    t.sync();
  }
  if (n_ret > 0) {
    Arena a2 = ar;
    double* w = a2.take(int64_t(n) * n_ret);
    double* lw = a2.take(int64_t(n) * n_ret);
    double* cm = a2.take(int64_t(n_ret) * n_ret);
    double* ecv = a2.take(n_ret);
    double* ecV = a2.take(int64_t(n_ret) * n_ret);
    for (int64_t e = t.rank(); e < int64_t(n) * n_ret; e += t.size()) {
      const int i = static_cast<int>(e / n_ret), j = static_cast<int>(e % n_ret);
      const double scale = 1.0 / sqrt(ebv[n_null + j]);
      w[e] = ebV[int64_t(i) * n + n_null + j] * scale;
    }
    t.sync();
    t_matmul(t, ls, n, n, w, n_ret, lw);
    t_matmul_transa(t, w, n, n_ret, lw, n_ret, cm);
    t_symmetrize(t, cm, n_ret);
    st = t_sym_eig(t, n_ret, cm, ecv, ecV, a2);
    if (st) return st;
    for (int k = n_ret; k-- > 0;) {
      double* u = outv + int64_t(cnt) * n;
      for (int i = t.rank(); i < n; i += t.size()) {
        double s = 0.0;
        for (int j = 0; j < n_ret; ++j) s += w[int64_t(i) * n_ret + j] * ecV[int64_t(j) * n_ret + k];
        u[i] = s;
      }
      if (t.rank() == 0) values[cnt] = ecv[k];
      ++cnt;
    }
    t.sync();
  }
  *cnt_out = cnt;
  return 0;
}

// workspace doubles of t_spsd_gevp beyond its outputs
__host__ __device__ inline int64_t spsd_gevp_scratch(int64_t n) {
  auto r2 = [](int64_t x) { return (x + 1) & ~int64_t(1); };
  // ebv, ebV, slot + max(eig(bs) scratch, null-part, finite-part)
  const int64_t part = r2(n * n) * 3 + r2(n) + r2(n * n) + sym_eig_scratch(n);
  return r2(n) + r2(n * n) + 4 + (sym_eig_scratch(n) > part ? sym_eig_scratch(n) : part);
}

}  // namespace lsb
