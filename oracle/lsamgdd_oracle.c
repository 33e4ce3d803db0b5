/* oracle/lsamgdd_oracle.c — TEST INFRASTRUCTURE ONLY: the parity checker.
 *
 * A plain-C restatement of the reference's hot path, function by function,
 * in the reference's operation order (built with -ffp-contract=off, like the
 * reference's own no-FMA Release build). Each function cites the reference
 * file:line it follows (paths relative to /root/reference/proj/include/lsamgdd).
 * It is never linked into, or called by, the product library; it is pinned
 * against oracle/_ref (the compiled reference) and the reference's golden
 * vectors by tests/test_oracle_pins.py.
 *
 * Errors follow the reference's exception classes through longjmp to the
 * C-ABI boundary, which returns the matching lsamgdd_status.
 */
#define _POSIX_C_SOURCE 200809L
#include "lsamgdd_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* error plumbing (errors.hpp:11-69)                                          */

static _Thread_local jmp_buf* g_jmp;
static _Thread_local int g_code;
static _Thread_local char g_msg[512];

static void fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof g_msg, fmt, ap);
  va_end(ap);
  g_code = code;
  longjmp(*g_jmp, 1);
}

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz ? sz : 1);
  if (!p) fail(LSAMGDD_ERR_ERROR, "out of memory");
  return p;
}
static void* xmalloc(size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p) fail(LSAMGDD_ERR_ERROR, "out of memory");
  return p;
}

/* growable int64 vector */
typedef struct {
  int64_t* a;
  int64_t n, cap;
} Vi;
static void vi_push(Vi* v, int64_t x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 8;
    v->a = (int64_t*)realloc(v->a, (size_t)v->cap * sizeof(int64_t));
    if (!v->a) fail(LSAMGDD_ERR_ERROR, "out of memory");
  }
  v->a[v->n++] = x;
}
static int cmp_i64(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return a < b ? -1 : a > b;
}
static void vi_sort_unique(Vi* v) {
  if (v->n == 0) return;
  qsort(v->a, (size_t)v->n, sizeof(int64_t), cmp_i64);
  int64_t w = 1;
  for (int64_t i = 1; i < v->n; ++i)
    if (v->a[i] != v->a[w - 1]) v->a[w++] = v->a[i];
  v->n = w;
}

/* ------------------------------------------------------------------------ */
/* dense helpers (dense.hpp)                                                  */

static void symmetrize(double* a, int64_t n) { /* dense.hpp:103-111 */
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      const double m = 0.5 * (a[i * n + j] + a[j * n + i]);
      a[i * n + j] = m;
      a[j * n + i] = m;
    }
}

/* c = a·b, skipping zero a(i,k)                        dense.hpp:47-59 */
static double* matmul(const double* a, int64_t ar, int64_t ac, const double* b, int64_t bc) {
  double* c = (double*)xcalloc((size_t)(ar * bc), sizeof(double));
  for (int64_t i = 0; i < ar; ++i)
    for (int64_t k = 0; k < ac; ++k) {
      const double aik = a[i * ac + k];
      if (aik == 0.0) continue;
      for (int64_t j = 0; j < bc; ++j) c[i * bc + j] += aik * b[k * bc + j];
    }
  return c;
}

/* c = aᵀ·b, skipping zero a(k,i)                       dense.hpp:62-74 */
static double* matmul_transa(const double* a, int64_t ar, int64_t ac, const double* b, int64_t bc) {
  double* c = (double*)xcalloc((size_t)(ac * bc), sizeof(double));
  for (int64_t k = 0; k < ar; ++k)
    for (int64_t i = 0; i < ac; ++i) {
      const double aki = a[k * ac + i];
      if (aki == 0.0) continue;
      for (int64_t j = 0; j < bc; ++j) c[i * bc + j] += aki * b[k * bc + j];
    }
  return c;
}

static double frob(const double* a, int64_t cnt) { /* dense.hpp:96-100 */
  double s = 0.0;
  for (int64_t i = 0; i < cnt; ++i) s += a[i] * a[i];
  return sqrt(s);
}

static double vdot(const double* x, const double* y, int64_t n) { /* sparse.hpp:297-302 */
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}
static double vnorm(const double* x, int64_t n) { return sqrt(vdot(x, x, n)); }

/* Cholesky, full storage, lower factor            dense.hpp:119-158 */
typedef struct {
  int64_t n;
  double* l;
} Chol;

static int chol_factor(Chol* f, const double* a, int64_t n) {
  free(f->l);
  f->n = n;
  f->l = (double*)xmalloc((size_t)(n * n) * sizeof(double));
  memcpy(f->l, a, (size_t)(n * n) * sizeof(double));
  double* l = f->l;
  for (int64_t j = 0; j < n; ++j) {
    double d = l[j * n + j];
    for (int64_t k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
    if (!(d > 0.0)) return 0;
    const double ljj = sqrt(d);
    l[j * n + j] = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double s = l[i * n + j];
      for (int64_t k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
      l[i * n + j] = s / ljj;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) l[i * n + j] = 0.0;
  return 1;
}

static void chol_solve(const Chol* f, double* x) { /* dense.hpp:145-158 */
  const int64_t n = f->n;
  const double* l = f->l;
  for (int64_t i = 0; i < n; ++i) {
    double s = x[i];
    for (int64_t k = 0; k < i; ++k) s -= l[i * n + k] * x[k];
    x[i] = s / l[i * n + i];
  }
  for (int64_t ii = n; ii-- > 0;) {
    double s = x[ii];
    for (int64_t k = ii + 1; k < n; ++k) s -= l[k * n + ii] * x[k];
    x[ii] = s / l[ii * n + ii];
  }
}

/* factor with one 1e-12·max|diag| retry           dense.hpp:175-185 */
static void factor_spd_block(Chol* f, const double* a, int64_t n, const char* ctx, int64_t id) {
  if (chol_factor(f, a, n)) return;
  double maxd = 0.0;
  for (int64_t i = 0; i < n; ++i) maxd = fmax(maxd, fabs(a[i * n + i]));
  double* sh = (double*)xmalloc((size_t)(n * n) * sizeof(double));
  memcpy(sh, a, (size_t)(n * n) * sizeof(double));
  const double jitter = 1e-12 * maxd;
  for (int64_t i = 0; i < n; ++i) sh[i * n + i] += jitter;
  const int ok = chol_factor(f, sh, n);
  free(sh);
  if (ok) return;
  if (id >= 0)
    fail(LSAMGDD_ERR_SETUP, "dense symmetric factorization failed for %s %lld", ctx, (long long)id);
  fail(LSAMGDD_ERR_SETUP, "dense symmetric factorization failed for %s", ctx);
}

/* ------------------------------------------------------------------------ */
/* eigensolvers (eigen.hpp)                                                   */

/* cyclic Jacobi, ascending values; vecs column k = vector k   eigen.hpp:35-118 */
static void sym_eig(int64_t n, const double* m, double* vals, double* vecs) {
  for (int64_t i = 0; i < n * n; ++i) vecs[i] = 0.0;
  for (int64_t i = 0; i < n; ++i) vecs[i * n + i] = 1.0;
  if (n == 0) return;
  double* a = (double*)xmalloc((size_t)(n * n) * sizeof(double));
  memcpy(a, m, (size_t)(n * n) * sizeof(double));
  symmetrize(a, n);
  double* v = (double*)xmalloc((size_t)(n * n) * sizeof(double));
  memcpy(v, vecs, (size_t)(n * n) * sizeof(double));
  double* d = (double*)xmalloc((size_t)n * sizeof(double));
  double* b = (double*)xmalloc((size_t)n * sizeof(double));
  double* z = (double*)xcalloc((size_t)n, sizeof(double));
  for (int64_t i = 0; i < n; ++i) d[i] = b[i] = a[i * n + i];
#define A(i, j) a[(i) * n + (j)]
#define V(i, j) v[(i) * n + (j)]
  int converged = 0;
  for (int64_t sweep = 0; sweep < 64; ++sweep) {
    double sm = 0.0;
    for (int64_t p = 0; p + 1 < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) sm += fabs(A(p, q));
    if (sm == 0.0) {
      converged = 1;
      break;
    }
    const double tresh = sweep < 3 ? 0.2 * sm / (double)((uint64_t)n * (uint64_t)n) : 0.0;
    for (int64_t p = 0; p + 1 < n; ++p) {
      for (int64_t q = p + 1; q < n; ++q) {
        const double g = 100.0 * fabs(A(p, q));
        if (sweep > 3 && fabs(d[p]) + g == fabs(d[p]) && fabs(d[q]) + g == fabs(d[q])) {
          A(p, q) = 0.0;
        } else if (fabs(A(p, q)) > tresh) {
          double h = d[q] - d[p];
          double t;
          if (fabs(h) + g == fabs(h)) {
            t = A(p, q) / h;
          } else {
            const double theta = 0.5 * h / A(p, q);
            t = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
            if (theta < 0.0) t = -t;
          }
          const double c = 1.0 / sqrt(1.0 + t * t);
          const double s = t * c;
          const double tau = s / (1.0 + c);
          h = t * A(p, q);
          z[p] -= h;
          z[q] += h;
          d[p] -= h;
          d[q] += h;
          A(p, q) = 0.0;
#define ROT(X, Y)                        \
  do {                                   \
    const double gx_ = (X), hy_ = (Y);   \
    (X) = gx_ - s * (hy_ + gx_ * tau);   \
    (Y) = hy_ + s * (gx_ - hy_ * tau);   \
  } while (0)
          for (int64_t j = 0; j < p; ++j) ROT(A(j, p), A(j, q));
          for (int64_t j = p + 1; j < q; ++j) ROT(A(p, j), A(j, q));
          for (int64_t j = q + 1; j < n; ++j) ROT(A(p, j), A(q, j));
          for (int64_t j = 0; j < n; ++j) ROT(V(j, p), V(j, q));
#undef ROT
        }
      }
    }
    for (int64_t i = 0; i < n; ++i) {
      b[i] += z[i];
      d[i] = b[i];
      z[i] = 0.0;
    }
  }
  if (!converged) fail(LSAMGDD_ERR_EIG, "sym_eig: Jacobi iteration did not converge");
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(d[i])) fail(LSAMGDD_ERR_EIG, "sym_eig: non-finite eigenvalue");
  /* stable ascending order (std::stable_sort, eigen.hpp:107-116) */
  int64_t* order = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) {
    int64_t pos = 0;
    for (int64_t i = 0; i < n; ++i)
      if (d[i] < d[k] || (d[i] == d[k] && i < k)) ++pos;
    order[pos] = k;
  }
  for (int64_t k = 0; k < n; ++k) {
    vals[k] = d[order[k]];
    for (int64_t i = 0; i < n; ++i) vecs[i * n + k] = V(i, order[k]);
  }
#undef A
#undef V
  free(order);
  free(a);
  free(v);
  free(d);
  free(b);
  free(z);
}

/* spsd pencil; vectors n×k row-major; returns k        eigen.hpp:142-209 */
static int64_t spsd_gevp(int64_t n, const double* l, const double* bm, double tau_rel, double* values,
                         double* vectors, int64_t* discarded) {
  *discarded = 0;
  if (n == 0) return 0;
  double* ls = (double*)xmalloc((size_t)(n * n) * sizeof(double));
  double* bs = (double*)xmalloc((size_t)(n * n) * sizeof(double));
  memcpy(ls, l, (size_t)(n * n) * sizeof(double));
  memcpy(bs, bm, (size_t)(n * n) * sizeof(double));
  symmetrize(ls, n);
  symmetrize(bs, n);
  double* ebv = (double*)xmalloc((size_t)n * sizeof(double));
  double* ebV = (double*)xmalloc((size_t)(n * n) * sizeof(double));
  sym_eig(n, bs, ebv, ebV);
  const double mu_max = fmax(ebv[n - 1], 0.0);
  const double cut = tau_rel * mu_max;
  int64_t n_null = 0;
  while (n_null < n && ebv[n_null] <= cut) ++n_null;
  const int64_t n_ret = n - n_null;
  const double l_scale = frob(ls, n * n);
  /* collected vectors, column-wise in a scratch (n × n) */
  double* cols = (double*)xcalloc((size_t)(n * n), sizeof(double));
  int64_t cnt = 0;
  if (n_null > 0) {
    double* vn = (double*)xmalloc((size_t)(n * n_null) * sizeof(double));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = 0; k < n_null; ++k) vn[i * n_null + k] = ebV[i * n + k];
    double* lv = matmul(ls, n, n, vn, n_null);
    double* t = matmul_transa(vn, n, n_null, lv, n_null);
    symmetrize(t, n_null);
    double* etv = (double*)xmalloc((size_t)n_null * sizeof(double));
    double* etV = (double*)xmalloc((size_t)(n_null * n_null) * sizeof(double));
    sym_eig(n_null, t, etv, etV);
    for (int64_t k = n_null; k-- > 0;) {
      if (etv[k] > tau_rel * l_scale) {
        for (int64_t i = 0; i < n; ++i) {
          double u = 0.0;
          for (int64_t j = 0; j < n_null; ++j) u += vn[i * n_null + j] * etV[j * n_null + k];
          cols[cnt * n + i] = u;
        }
        values[cnt++] = INFINITY;
      } else {
        ++*discarded;
      }
    }
    free(vn);
    free(lv);
    free(t);
    free(etv);
    free(etV);
  }
  if (n_ret > 0) {
    double* w = (double*)xmalloc((size_t)(n * n_ret) * sizeof(double));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n_ret; ++j) w[i * n_ret + j] = ebV[i * n + n_null + j];
    for (int64_t j = 0; j < n_ret; ++j) {
      const double scale = 1.0 / sqrt(ebv[n_null + j]);
      for (int64_t i = 0; i < n; ++i) w[i * n_ret + j] *= scale;
    }
    double* lw = matmul(ls, n, n, w, n_ret);
    double* c = matmul_transa(w, n, n_ret, lw, n_ret);
    symmetrize(c, n_ret);
    double* ecv = (double*)xmalloc((size_t)n_ret * sizeof(double));
    double* ecV = (double*)xmalloc((size_t)(n_ret * n_ret) * sizeof(double));
    sym_eig(n_ret, c, ecv, ecV);
    for (int64_t k = n_ret; k-- > 0;) {
      for (int64_t i = 0; i < n; ++i) {
        double u = 0.0;
        for (int64_t j = 0; j < n_ret; ++j) u += w[i * n_ret + j] * ecV[j * n_ret + k];
        cols[cnt * n + i] = u;
      }
      values[cnt++] = ecv[k];
    }
    free(w);
    free(lw);
    free(c);
    free(ecv);
    free(ecV);
  }
  for (int64_t k = 0; k < cnt; ++k)
    for (int64_t i = 0; i < n; ++i) vectors[i * cnt + k] = cols[k * n + i];
  free(cols);
  free(ls);
  free(bs);
  free(ebv);
  free(ebV);
  return cnt;
}

/* spectral pseudo-inverse                                eigen.hpp:215-231 */
static void pseudo_inverse(int64_t n, const double* m, double tau_rel, double* out) {
  double* ev = (double*)xmalloc((size_t)(n ? n : 1) * sizeof(double));
  double* eV = (double*)xmalloc((size_t)(n * n ? n * n : 1) * sizeof(double));
  sym_eig(n, m, ev, eV);
  const double cut = n == 0 ? 0.0 : tau_rel * fmax(ev[n - 1], 0.0);
  for (int64_t i = 0; i < n * n; ++i) out[i] = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    if (ev[k] <= cut) continue;
    const double inv = 1.0 / ev[k];
    for (int64_t i = 0; i < n; ++i) {
      const double vik = eV[i * n + k] * inv;
      if (vik == 0.0) continue;
      for (int64_t j = 0; j < n; ++j) out[i * n + j] += vik * eV[j * n + k];
    }
  }
  free(ev);
  free(eV);
}

/* ------------------------------------------------------------------------ */
/* sparse core (sparse.hpp)                                                   */

typedef struct {
  int64_t nr, nc;
  int64_t* off; /* nr+1 */
  int64_t* col;
  double* val;
} Csr;

static int64_t csr_nnz(const Csr* m) { return m->off[m->nr]; }
static void csr_free(Csr* m) {
  free(m->off);
  free(m->col);
  free(m->val);
  memset(m, 0, sizeof *m);
}
static Csr csr_copy(const Csr* m) {
  Csr c = *m;
  const int64_t nnz = csr_nnz(m);
  c.off = (int64_t*)xmalloc((size_t)(m->nr + 1) * sizeof(int64_t));
  c.col = (int64_t*)xmalloc((size_t)nnz * sizeof(int64_t));
  c.val = (double*)xmalloc((size_t)nnz * sizeof(double));
  memcpy(c.off, m->off, (size_t)(m->nr + 1) * sizeof(int64_t));
  memcpy(c.col, m->col, (size_t)nnz * sizeof(int64_t));
  memcpy(c.val, m->val, (size_t)nnz * sizeof(double));
  return c;
}

typedef struct {
  int64_t r, c;
  double v;
} Trip;
static int cmp_trip(const void* x, const void* y) {
  const Trip* a = (const Trip*)x;
  const Trip* b = (const Trip*)y;
  if (a->r != b->r) return a->r < b->r ? -1 : 1;
  if (a->c != b->c) return a->c < b->c ? -1 : 1;
  return 0;
}

/* sum duplicates, drop exact zeros                      sparse.hpp:79-108 */
static Csr csr_from_triplets(int64_t nr, int64_t nc, Trip* t, int64_t nt) {
  for (int64_t k = 0; k < nt; ++k)
    if (t[k].r < 0 || t[k].r >= nr || t[k].c < 0 || t[k].c >= nc)
      fail(LSAMGDD_ERR_INDEX, "csr_from_triplets: entry (%lld, %lld) outside %lldx%lld", (long long)t[k].r,
           (long long)t[k].c, (long long)nr, (long long)nc);
  qsort(t, (size_t)nt, sizeof(Trip), cmp_trip);
  Csr m;
  m.nr = nr;
  m.nc = nc;
  m.off = (int64_t*)xcalloc((size_t)(nr + 1), sizeof(int64_t));
  m.col = (int64_t*)xmalloc((size_t)(nt ? nt : 1) * sizeof(int64_t));
  m.val = (double*)xmalloc((size_t)(nt ? nt : 1) * sizeof(double));
  int64_t k = 0, cnt = 0;
  for (int64_t i = 0; i < nr; ++i) {
    while (k < nt && t[k].r == i) {
      const int64_t c = t[k].c;
      double s = 0.0;
      while (k < nt && t[k].r == i && t[k].c == c) s += t[k++].v;
      if (s != 0.0) {
        m.col[cnt] = c;
        m.val[cnt] = s;
        ++cnt;
      }
    }
    m.off[i + 1] = cnt;
  }
  return m;
}

static void spmv(const Csr* m, const double* x, double* y) { /* sparse.hpp:110-122 */
  for (int64_t i = 0; i < m->nr; ++i) {
    double s = 0.0;
    for (int64_t k = m->off[i]; k < m->off[i + 1]; ++k) s += m->val[k] * x[m->col[k]];
    y[i] = s;
  }
}

static void spmv_transpose(const Csr* m, const double* x, double* y) { /* sparse.hpp:125-137 */
  for (int64_t j = 0; j < m->nc; ++j) y[j] = 0.0;
  for (int64_t i = 0; i < m->nr; ++i) {
    const double xi = x[i];
    if (xi == 0.0) continue;
    for (int64_t k = m->off[i]; k < m->off[i + 1]; ++k) y[m->col[k]] += m->val[k] * xi;
  }
}

static Csr csr_transpose(const Csr* m) { /* sparse.hpp:139-153 */
  const int64_t nnz = csr_nnz(m);
  Csr t;
  t.nr = m->nc;
  t.nc = m->nr;
  t.off = (int64_t*)xcalloc((size_t)(m->nc + 1), sizeof(int64_t));
  t.col = (int64_t*)xmalloc((size_t)(nnz ? nnz : 1) * sizeof(int64_t));
  t.val = (double*)xmalloc((size_t)(nnz ? nnz : 1) * sizeof(double));
  for (int64_t k = 0; k < nnz; ++k) ++t.off[m->col[k] + 1];
  for (int64_t j = 0; j < m->nc; ++j) t.off[j + 1] += t.off[j];
  int64_t* cur = (int64_t*)xmalloc((size_t)(m->nc ? m->nc : 1) * sizeof(int64_t));
  memcpy(cur, t.off, (size_t)m->nc * sizeof(int64_t));
  for (int64_t i = 0; i < m->nr; ++i)
    for (int64_t k = m->off[i]; k < m->off[i + 1]; ++k) {
      const int64_t p = cur[m->col[k]]++;
      t.col[p] = i;
      t.val[p] = m->val[k];
    }
  free(cur);
  return t;
}

/* Gustavson product, Symbolic mode (keeps exact zeros)  sparse.hpp:167-204 */
static Csr spgemm_symbolic(const Csr* a, const Csr* b) {
  if (a->nc != b->nr)
    fail(LSAMGDD_ERR_DIM, "spgemm: inner dimensions %lld and %lld do not match", (long long)a->nc, (long long)b->nr);
  const int64_t nr = a->nr, nc = b->nc;
  double* acc = (double*)xcalloc((size_t)nc, sizeof(double));
  char* seen = (char*)xcalloc((size_t)nc, 1);
  Vi touched = {0};
  Vi cols = {0};
  double* vals = NULL;
  int64_t vcap = 0;
  int64_t* off = (int64_t*)xcalloc((size_t)(nr + 1), sizeof(int64_t));
  for (int64_t i = 0; i < nr; ++i) {
    touched.n = 0;
    for (int64_t ka = a->off[i]; ka < a->off[i + 1]; ++ka) {
      const int64_t kk = a->col[ka];
      const double av = a->val[ka];
      for (int64_t kb = b->off[kk]; kb < b->off[kk + 1]; ++kb) {
        const int64_t j = b->col[kb];
        if (!seen[j]) {
          seen[j] = 1;
          vi_push(&touched, j);
        }
        acc[j] += av * b->val[kb];
      }
    }
    if (touched.n > 1) qsort(touched.a, (size_t)touched.n, sizeof(int64_t), cmp_i64);
    for (int64_t t = 0; t < touched.n; ++t) {
      const int64_t j = touched.a[t];
      vi_push(&cols, j);
      if (cols.n > vcap) {
        vcap = cols.cap;
        vals = (double*)realloc(vals, (size_t)vcap * sizeof(double));
        if (!vals) fail(LSAMGDD_ERR_ERROR, "out of memory");
      }
      vals[cols.n - 1] = acc[j];
      acc[j] = 0.0;
      seen[j] = 0;
    }
    off[i + 1] = cols.n;
  }
  free(acc);
  free(seen);
  free(touched.a);
  Csr c;
  c.nr = nr;
  c.nc = nc;
  c.off = off;
  c.col = cols.a ? cols.a : (int64_t*)xmalloc(sizeof(int64_t));
  c.val = vals ? vals : (double*)xmalloc(sizeof(double));
  return c;
}

/* dense gather m(rows, cols) in the given orders           sparse.hpp:210-236 */
static double* submatrix(const Csr* m, const int64_t* rows, int64_t nr, const int64_t* cols, int64_t nc,
                         int64_t* colmap /* scratch of m->nc, all -1 */) {
  for (int64_t p = 0; p < nc; ++p) {
    if (colmap[cols[p]] != -1) fail(LSAMGDD_ERR_INDEX, "submatrix: duplicate column index");
    colmap[cols[p]] = p;
  }
  double* out = (double*)xcalloc((size_t)(nr * nc), sizeof(double));
  for (int64_t p = 0; p < nr; ++p) {
    const int64_t r = rows[p];
    for (int64_t k = m->off[r]; k < m->off[r + 1]; ++k) {
      const int64_t q = colmap[m->col[k]];
      if (q != -1) out[p * nc + q] = m->val[k];
    }
  }
  for (int64_t p = 0; p < nc; ++p) colmap[cols[p]] = -1;
  return out;
}

/* ------------------------------------------------------------------------ */
/* aggregation and topology (aggregation.hpp)                                 */

typedef struct {
  int64_t n_nodes, n_agg;
  int64_t* omega_off; /* n_agg+1 */
  int64_t* omega;
  int64_t* gamma_off;
  int64_t* gamma;
  int64_t* colors;
  int64_t n_colors;
  int64_t multiplicity_max;
} Topo;

static void topo_free(Topo* t) {
  free(t->omega_off);
  free(t->omega);
  free(t->gamma_off);
  free(t->gamma);
  free(t->colors);
  memset(t, 0, sizeof *t);
}

/* three-pass greedy aggregation                       aggregation.hpp:71-117 */
static int64_t standard_aggregation(const Csr* a, int64_t* asg) {
  if (a->nr == 0) fail(LSAMGDD_ERR_INPUT, "standard_aggregation: matrix is empty");
  if (a->nr != a->nc) fail(LSAMGDD_ERR_DIM, "standard_aggregation: matrix is not square");
  const int64_t n = a->nr;
  for (int64_t i = 0; i < n; ++i) asg[i] = -1;
  int64_t next = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (asg[i] != -1) continue;
    int has_nb = 0, all_free = 1;
    for (int64_t k = a->off[i]; k < a->off[i + 1] && all_free; ++k) {
      const int64_t c = a->col[k];
      if (c == i) continue;
      has_nb = 1;
      if (asg[c] != -1) all_free = 0;
    }
    if (!has_nb || !all_free) continue;
    asg[i] = next;
    for (int64_t k = a->off[i]; k < a->off[i + 1]; ++k) asg[a->col[k]] = next;
    ++next;
  }
  /* pass 2 against the pass-1 snapshot */
  int64_t* att_node = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
  int64_t* att_agg = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
  int64_t n_att = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (asg[i] != -1) continue;
    double best = -1.0;
    int64_t best_agg = -1;
    for (int64_t k = a->off[i]; k < a->off[i + 1]; ++k) {
      const int64_t c = a->col[k];
      if (c == i || asg[c] == -1) continue;
      const double w = fabs(a->val[k]);
      if (w > best || (w == best && (uint64_t)asg[c] < (uint64_t)best_agg)) {
        best = w;
        best_agg = asg[c];
      }
    }
    if (best_agg != -1) {
      att_node[n_att] = i;
      att_agg[n_att++] = best_agg;
    }
  }
  for (int64_t t = 0; t < n_att; ++t) asg[att_node[t]] = att_agg[t];
  free(att_node);
  free(att_agg);
  for (int64_t i = 0; i < n; ++i)
    if (asg[i] == -1) asg[i] = next++;
  return next;
}

/* compose passes through Tᵀ A T                        aggregation.hpp:138-155 */
static int64_t multi_pass_aggregation(const Csr* a, int64_t passes, int64_t* composed) {
  if (passes < 1) fail(LSAMGDD_ERR_INPUT, "multi_pass_aggregation: need at least one pass");
  int64_t* part = (int64_t*)xmalloc((size_t)a->nr * sizeof(int64_t));
  int64_t n_agg = standard_aggregation(a, part);
  memcpy(composed, part, (size_t)a->nr * sizeof(int64_t));
  Csr coarse = csr_copy(a);
  for (int64_t pass = 1; pass < passes; ++pass) {
    if (n_agg <= 1) {
      fprintf(stderr, "lsamgdd: warning: aggregation stopped after %lld pass(es); the coarse graph collapsed to one node\n",
              (long long)pass);
      break;
    }
    Csr t;
    t.nr = coarse.nr;
    t.nc = n_agg;
    t.off = (int64_t*)xmalloc((size_t)(coarse.nr + 1) * sizeof(int64_t));
    t.col = (int64_t*)xmalloc((size_t)coarse.nr * sizeof(int64_t));
    t.val = (double*)xmalloc((size_t)coarse.nr * sizeof(double));
    for (int64_t i = 0; i <= coarse.nr; ++i) t.off[i] = i;
    for (int64_t i = 0; i < coarse.nr; ++i) {
      t.col[i] = part[i];
      t.val[i] = 1.0;
    }
    Csr tt = csr_transpose(&t);
    Csr ta = spgemm_symbolic(&tt, &coarse);
    Csr c2 = spgemm_symbolic(&ta, &t);
    csr_free(&tt);
    csr_free(&ta);
    csr_free(&t);
    csr_free(&coarse);
    coarse = c2;
    free(part);
    part = (int64_t*)xmalloc((size_t)coarse.nr * sizeof(int64_t));
    n_agg = standard_aggregation(&coarse, part);
    for (int64_t v = 0; v < a->nr; ++v) composed[v] = part[composed[v]];
  }
  csr_free(&coarse);
  free(part);
  return n_agg;
}

/* adjacency of intersecting subdomains + greedy colouring  aggregation.hpp:197-229 */
static void color_topology(Topo* t, const int64_t* asg) {
  const int64_t n = t->n_nodes, na = t->n_agg;
  Vi* holders = (Vi*)xcalloc((size_t)n, sizeof(Vi));
  for (int64_t v = 0; v < n; ++v) vi_push(&holders[v], asg[v]);
  for (int64_t i = 0; i < na; ++i)
    for (int64_t k = t->gamma_off[i]; k < t->gamma_off[i + 1]; ++k) vi_push(&holders[t->gamma[k]], i);
  Vi* adj = (Vi*)xcalloc((size_t)na, sizeof(Vi));
  for (int64_t v = 0; v < n; ++v) {
    for (int64_t x = 0; x < holders[v].n; ++x)
      for (int64_t y = x + 1; y < holders[v].n; ++y) {
        vi_push(&adj[holders[v].a[x]], holders[v].a[y]);
        vi_push(&adj[holders[v].a[y]], holders[v].a[x]);
      }
    free(holders[v].a);
  }
  free(holders);
  for (int64_t i = 0; i < na; ++i) vi_sort_unique(&adj[i]);
  /* stable sort by descending degree: bucket by degree, ascending id in a bucket */
  int64_t* order = (int64_t*)xmalloc((size_t)na * sizeof(int64_t));
  int64_t maxdeg = 0;
  for (int64_t i = 0; i < na; ++i) maxdeg = adj[i].n > maxdeg ? adj[i].n : maxdeg;
  int64_t* cnt = (int64_t*)xcalloc((size_t)(maxdeg + 2), sizeof(int64_t));
  for (int64_t i = 0; i < na; ++i) ++cnt[maxdeg - adj[i].n + 1];
  for (int64_t d = 0; d <= maxdeg; ++d) cnt[d + 1] += cnt[d];
  for (int64_t i = 0; i < na; ++i) order[cnt[maxdeg - adj[i].n]++] = i;
  free(cnt);
  free(t->colors);
  t->colors = (int64_t*)xmalloc((size_t)na * sizeof(int64_t));
  for (int64_t i = 0; i < na; ++i) t->colors[i] = -1;
  int64_t max_color = 0;
  char* used = NULL;
  int64_t used_cap = 0;
  for (int64_t oi = 0; oi < na; ++oi) {
    const int64_t i = order[oi];
    const int64_t sz = adj[i].n + 1;
    if (sz > used_cap) {
      used_cap = sz;
      used = (char*)realloc(used, (size_t)used_cap);
    }
    memset(used, 0, (size_t)sz);
    for (int64_t k = 0; k < adj[i].n; ++k) {
      const int64_t cj = t->colors[adj[i].a[k]];
      if (cj != -1 && cj < sz) used[cj] = 1;
    }
    int64_t c = 0;
    while (used[c]) ++c;
    t->colors[i] = c;
    if (c > max_color) max_color = c;
  }
  free(used);
  free(order);
  for (int64_t i = 0; i < na; ++i) free(adj[i].a);
  free(adj);
  t->n_colors = max_color + 1;
}

/* Γ sets (one layer, or two for the overlap-2 hook) + colouring  aggregation.hpp:165-231 */
static Topo build_topology(const Csr* a, const int64_t* asg, int64_t n_agg, int layers) {
  const int64_t n = a->nr;
  if (a->nr != a->nc) fail(LSAMGDD_ERR_DIM, "build_topology: matrix is not square");
  if (n_agg == 0) fail(LSAMGDD_ERR_INPUT, "build_topology: partition has no aggregates");
  for (int64_t v = 0; v < n; ++v)
    if (asg[v] < 0 || asg[v] >= n_agg) fail(LSAMGDD_ERR_INPUT, "build_topology: aggregate id out of range");
  Topo t;
  memset(&t, 0, sizeof t);
  t.n_nodes = n;
  t.n_agg = n_agg;
  t.omega_off = (int64_t*)xcalloc((size_t)(n_agg + 1), sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) ++t.omega_off[asg[v] + 1];
  for (int64_t i = 0; i < n_agg; ++i) {
    if (t.omega_off[i + 1] == 0) fail(LSAMGDD_ERR_INPUT, "build_topology: aggregate %lld is empty", (long long)i);
    t.omega_off[i + 1] += t.omega_off[i];
  }
  t.omega = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
  int64_t* cur = (int64_t*)xmalloc((size_t)n_agg * sizeof(int64_t));
  memcpy(cur, t.omega_off, (size_t)n_agg * sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) t.omega[cur[asg[v]]++] = v;
  free(cur);
  Vi* gam = (Vi*)xcalloc((size_t)n_agg, sizeof(Vi));
  for (int64_t i = 0; i < n_agg; ++i) {
    for (int64_t p = t.omega_off[i]; p < t.omega_off[i + 1]; ++p) {
      const int64_t u = t.omega[p];
      for (int64_t k = a->off[u]; k < a->off[u + 1]; ++k)
        if (asg[a->col[k]] != i) vi_push(&gam[i], a->col[k]);
    }
    vi_sort_unique(&gam[i]);
    if (layers >= 2) { /* second layer: neighbours of ω ∪ Γ outside ω (ref_harness.cpp widen_overlap) */
      Vi g2 = {0};
      for (int64_t p = t.omega_off[i]; p < t.omega_off[i + 1]; ++p) {
        const int64_t u = t.omega[p];
        for (int64_t k = a->off[u]; k < a->off[u + 1]; ++k)
          if (asg[a->col[k]] != i) vi_push(&g2, a->col[k]);
      }
      for (int64_t p = 0; p < gam[i].n; ++p) {
        const int64_t u = gam[i].a[p];
        for (int64_t k = a->off[u]; k < a->off[u + 1]; ++k)
          if (asg[a->col[k]] != i) vi_push(&g2, a->col[k]);
      }
      vi_sort_unique(&g2);
      free(gam[i].a);
      gam[i] = g2;
    }
  }
  t.gamma_off = (int64_t*)xcalloc((size_t)(n_agg + 1), sizeof(int64_t));
  for (int64_t i = 0; i < n_agg; ++i) t.gamma_off[i + 1] = t.gamma_off[i] + gam[i].n;
  t.gamma = (int64_t*)xmalloc((size_t)(t.gamma_off[n_agg] ? t.gamma_off[n_agg] : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n_agg; ++i) {
    if (gam[i].n) memcpy(t.gamma + t.gamma_off[i], gam[i].a, (size_t)gam[i].n * sizeof(int64_t));
    free(gam[i].a);
  }
  free(gam);
  color_topology(&t, asg);
  return t;
}

/* ------------------------------------------------------------------------ */
/* splitting (splitting.hpp)                                                  */

typedef struct {
  int64_t* nz_off; /* n_agg+1 */
  int64_t* nz;
  int64_t* mult; /* rows of G */
  int64_t n_mult;
} RowSets;

static void rowsets_free(RowSets* r) {
  free(r->nz_off);
  free(r->nz);
  free(r->mult);
  memset(r, 0, sizeof *r);
}

/* nz_i, M(j), n_mult                                   splitting.hpp:53-84 */
static RowSets compute_row_sets(const Csr* g, Topo* t) {
  if (g->nc != t->n_nodes) fail(LSAMGDD_ERR_DIM, "compute_row_sets: factor has %lld columns, topology covers %lld nodes",
                                (long long)g->nc, (long long)t->n_nodes);
  const int64_t na = t->n_agg;
  int64_t* owner = (int64_t*)xmalloc((size_t)t->n_nodes * sizeof(int64_t));
  for (int64_t i = 0; i < na; ++i)
    for (int64_t p = t->omega_off[i]; p < t->omega_off[i + 1]; ++p) owner[t->omega[p]] = i;
  RowSets rs;
  rs.mult = (int64_t*)xcalloc((size_t)g->nr, sizeof(int64_t));
  rs.n_mult = 0;
  Vi* nz = (Vi*)xcalloc((size_t)na, sizeof(Vi));
  Vi hit = {0};
  int64_t empty = 0;
  for (int64_t j = 0; j < g->nr; ++j) {
    hit.n = 0;
    for (int64_t k = g->off[j]; k < g->off[j + 1]; ++k) vi_push(&hit, owner[g->col[k]]);
    vi_sort_unique(&hit);
    if (hit.n == 0) {
      ++empty;
      continue;
    }
    for (int64_t h = 0; h < hit.n; ++h) vi_push(&nz[hit.a[h]], j);
    rs.mult[j] = hit.n;
    if (hit.n > rs.n_mult) rs.n_mult = hit.n;
  }
  free(hit.a);
  free(owner);
  if (empty > 0) fprintf(stderr, "lsamgdd: note: %lld empty factor row(s) belong to no row set\n", (long long)empty);
  rs.nz_off = (int64_t*)xcalloc((size_t)(na + 1), sizeof(int64_t));
  for (int64_t i = 0; i < na; ++i) rs.nz_off[i + 1] = rs.nz_off[i] + nz[i].n;
  rs.nz = (int64_t*)xmalloc((size_t)(rs.nz_off[na] ? rs.nz_off[na] : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < na; ++i) {
    if (nz[i].n) memcpy(rs.nz + rs.nz_off[i], nz[i].a, (size_t)nz[i].n * sizeof(int64_t));
    free(nz[i].a);
  }
  free(nz);
  t->multiplicity_max = rs.n_mult;
  return rs;
}

/* xᵀ·diag(w)·y, skipping zero w_r·x(r,i)               splitting.hpp:102-115 */
static double* weighted_gram(const double* x, int64_t rows, int64_t xc, const double* y, int64_t yc, const double* w) {
  double* out = (double*)xcalloc((size_t)(xc * yc), sizeof(double));
  for (int64_t r = 0; r < rows; ++r) {
    const double wr = w[r];
    for (int64_t i = 0; i < xc; ++i) {
      const double xi = wr * x[r * xc + i];
      if (xi == 0.0) continue;
      for (int64_t j = 0; j < yc; ++j) out[i * yc + j] += xi * y[r * yc + j];
    }
  }
  return out;
}

/* max{0.1, (κ - k_c)/(k_c·n_mult)}                      splitting.hpp:170-180 */
static double eigen_threshold(double kappa, int64_t kc, int64_t n_mult) {
  if (kc == 0 || n_mult == 0) fail(LSAMGDD_ERR_INPUT, "eigen_threshold: k_c and n_mult must be positive");
  if (kappa <= (double)kc) {
    fprintf(stderr, "lsamgdd: warning: target condition number %g does not exceed the color count %lld; using the floor threshold\n",
            kappa, (long long)kc);
    return 0.1;
  }
  const double t = (kappa - (double)kc) / ((double)kc * (double)n_mult);
  return t > 0.1 ? t : 0.1;
}

/* Schur-reduced pencil, keep rule, two-pass MGS, sign rule.  splitting.hpp:200-275
 * g_omega: rows×nw, g_gamma: rows×ng. Returns panel (nw×*kcols, row-major). */
static double* local_gevp(int64_t agg, const double* gw, const double* gg, const double* w, int64_t rows, int64_t nw,
                          int64_t ng, double thresh, int64_t max_modes, int variant, double must_keep,
                          int64_t* kcols, double** eig_out, int64_t* n_eig) {
  if (nw == 0) fail(LSAMGDD_ERR_INPUT, "local_gevp: aggregate %lld has no interior", (long long)agg);
  if (max_modes == 0) max_modes = 1;
  const double tau_rel = 1e-10;
  double* unit = (double*)xmalloc((size_t)(rows ? rows : 1) * sizeof(double));
  for (int64_t r = 0; r < rows; ++r) unit[r] = 1.0;
  double* lhs = weighted_gram(gw, rows, nw, gw, nw, variant == 1 ? w : unit);
  double* rhs = weighted_gram(gw, rows, nw, gw, nw, w);
  free(unit);
  if (ng > 0) {
    double* cross = weighted_gram(gw, rows, nw, gg, ng, w);    /* nw×ng */
    double* boundary = weighted_gram(gg, rows, ng, gg, ng, w); /* ng×ng */
    double* pinv = (double*)xmalloc((size_t)(ng * ng) * sizeof(double));
    pseudo_inverse(ng, boundary, tau_rel, pinv);
    double* crossT = (double*)xmalloc((size_t)(ng * nw) * sizeof(double));
    for (int64_t i = 0; i < nw; ++i)
      for (int64_t j = 0; j < ng; ++j) crossT[j * nw + i] = cross[i * ng + j];
    double* tmp = matmul(pinv, ng, ng, crossT, nw);      /* ng×nw */
    double* schur = matmul(cross, nw, ng, tmp, nw);      /* nw×nw */
    for (int64_t r = 0; r < nw; ++r)
      for (int64_t c = 0; c < nw; ++c) rhs[r * nw + c] -= schur[r * nw + c];
    free(cross);
    free(boundary);
    free(pinv);
    free(crossT);
    free(tmp);
    free(schur);
  }
  symmetrize(rhs, nw);
  double* vals = (double*)xmalloc((size_t)nw * sizeof(double));
  double* vecs = (double*)xmalloc((size_t)(nw * nw) * sizeof(double));
  int64_t disc = 0;
  const int64_t nv = spsd_gevp(nw, lhs, rhs, tau_rel, vals, vecs, &disc);
  free(lhs);
  free(rhs);
  if (eig_out) {
    *eig_out = (double*)xmalloc((size_t)(nv ? nv : 1) * sizeof(double));
    memcpy(*eig_out, vals, (size_t)nv * sizeof(double));
    *n_eig = nv;
  }
  for (int64_t k = 0; k < nv; ++k)
    if (isnan(vals[k])) fail(LSAMGDD_ERR_EIG, "local_gevp: aggregate %lld: NaN eigenvalue", (long long)agg);
  int64_t n_null = 0;
  while (n_null < nv && isinf(vals[n_null])) ++n_null;
  int64_t above = n_null;
  while (above < nv && vals[above] > thresh) ++above;
  int64_t severe = n_null;
  while (severe < above && vals[severe] >= must_keep) ++severe;
  int64_t fin = above - n_null < max_modes ? above - n_null : max_modes;
  if (severe - n_null > fin) fin = severe - n_null;
  int64_t keep = n_null + fin;
  if (keep == 0) keep = 1;
  if (keep > nv) keep = nv;
  double* panel = (double*)xcalloc((size_t)(nw * (keep ? keep : 1)), sizeof(double));
  double* v = (double*)xmalloc((size_t)nw * sizeof(double));
  int64_t cols = 0;
  for (int64_t k = 0; k < keep; ++k) {
    for (int64_t r = 0; r < nw; ++r) v[r] = vecs[r * nv + k];
    const double orig = vnorm(v, nw);
    for (int pass = 0; pass < 2; ++pass)
      for (int64_t c = 0; c < cols; ++c) {
        double proj = 0.0;
        for (int64_t r = 0; r < nw; ++r) proj += panel[r * keep + c] * v[r];
        for (int64_t r = 0; r < nw; ++r) v[r] -= proj * panel[r * keep + c];
      }
    const double nvv = vnorm(v, nw);
    if (!(nvv > 1e-12 * fmax(orig, 1e-300))) continue;
    int64_t arg = 0;
    for (int64_t r = 1; r < nw; ++r)
      if (fabs(v[r]) > fabs(v[arg])) arg = r;
    const double sign = v[arg] < 0.0 ? -1.0 : 1.0;
    for (int64_t r = 0; r < nw; ++r) panel[r * keep + cols] = sign * v[r] / nvv;
    ++cols;
  }
  free(v);
  free(vals);
  free(vecs);
  double* out;
  if (cols == 0) {
    out = (double*)xmalloc((size_t)nw * sizeof(double));
    const double unitv = 1.0 / sqrt((double)nw);
    for (int64_t r = 0; r < nw; ++r) out[r] = unitv;
    *kcols = 1;
  } else {
    out = (double*)xmalloc((size_t)(nw * cols) * sizeof(double));
    for (int64_t r = 0; r < nw; ++r)
      for (int64_t c = 0; c < cols; ++c) out[r * cols + c] = panel[r * keep + c];
    *kcols = cols;
  }
  free(panel);
  return out;
}

/* ------------------------------------------------------------------------ */
/* Schwarz smoother (smoother.hpp)                                            */

typedef struct {
  int64_t n, n_agg;
  int64_t* sub_off;
  int64_t* sub; /* ω ‖ Γ per aggregate */
  int64_t* omega_sizes;
  Chol* factors;
} Smoother;

static void smoother_free(Smoother* s) {
  for (int64_t i = 0; i < s->n_agg; ++i) free(s->factors[i].l);
  free(s->factors);
  free(s->sub_off);
  free(s->sub);
  free(s->omega_sizes);
  memset(s, 0, sizeof *s);
}

static Smoother build_smoother(const Csr* a, const Topo* t) { /* smoother.hpp:38-58 */
  if (a->nr != a->nc) fail(LSAMGDD_ERR_DIM, "build_smoother: matrix is not square");
  if (a->nr != t->n_nodes)
    fail(LSAMGDD_ERR_DIM, "build_smoother: topology covers %lld nodes, matrix has %lld", (long long)t->n_nodes,
         (long long)a->nr);
  Smoother s;
  s.n = a->nr;
  s.n_agg = t->n_agg;
  s.sub_off = (int64_t*)xcalloc((size_t)(t->n_agg + 1), sizeof(int64_t));
  for (int64_t i = 0; i < t->n_agg; ++i)
    s.sub_off[i + 1] = s.sub_off[i] + (t->omega_off[i + 1] - t->omega_off[i]) + (t->gamma_off[i + 1] - t->gamma_off[i]);
  s.sub = (int64_t*)xmalloc((size_t)s.sub_off[t->n_agg] * sizeof(int64_t));
  s.omega_sizes = (int64_t*)xmalloc((size_t)t->n_agg * sizeof(int64_t));
  s.factors = (Chol*)xcalloc((size_t)t->n_agg, sizeof(Chol));
  int64_t* colmap = (int64_t*)xmalloc((size_t)a->nc * sizeof(int64_t));
  for (int64_t c = 0; c < a->nc; ++c) colmap[c] = -1;
  for (int64_t i = 0; i < t->n_agg; ++i) {
    int64_t o = s.sub_off[i];
    for (int64_t p = t->omega_off[i]; p < t->omega_off[i + 1]; ++p) s.sub[o++] = t->omega[p];
    for (int64_t p = t->gamma_off[i]; p < t->gamma_off[i + 1]; ++p) s.sub[o++] = t->gamma[p];
    s.omega_sizes[i] = t->omega_off[i + 1] - t->omega_off[i];
    const int64_t m = s.sub_off[i + 1] - s.sub_off[i];
    double* block = submatrix(a, s.sub + s.sub_off[i], m, s.sub + s.sub_off[i], m, colmap);
    factor_spd_block(&s.factors[i], block, m, "subdomain block of aggregate", i);
    free(block);
  }
  free(colmap);
  return s;
}

/* RAS / RAS-T / ASM, ascending aggregate order         smoother.hpp:65-83 */
static void smoother_apply(const Smoother* s, const double* r, int mode, double* y) {
  for (int64_t j = 0; j < s->n; ++j) y[j] = 0.0;
  int64_t maxm = 0;
  for (int64_t i = 0; i < s->n_agg; ++i)
    if (s->sub_off[i + 1] - s->sub_off[i] > maxm) maxm = s->sub_off[i + 1] - s->sub_off[i];
  double* local = (double*)xmalloc((size_t)(maxm ? maxm : 1) * sizeof(double));
  for (int64_t i = 0; i < s->n_agg; ++i) {
    const int64_t* sub = s->sub + s->sub_off[i];
    const int64_t m = s->sub_off[i + 1] - s->sub_off[i];
    const int64_t interior = s->omega_sizes[i];
    for (int64_t k = 0; k < m; ++k) local[k] = r[sub[k]];
    if (mode == LSAMGDD_RAST)
      for (int64_t k = interior; k < m; ++k) local[k] = 0.0;
    chol_solve(&s->factors[i], local);
    const int64_t scatter = mode == LSAMGDD_RAS ? interior : m;
    for (int64_t k = 0; k < scatter; ++k) y[sub[k]] += local[k];
  }
  free(local);
}

/* ------------------------------------------------------------------------ */
/* hierarchy (hierarchy.hpp)                                                  */

typedef struct {
  Csr A, G, P;
  int has_interp;
  Topo topo;
  Smoother sm;
  double thresh;
  int64_t* mult;
  int64_t mult_n;
  int64_t spec_n;
  int64_t* spec_off;
  double* spec;
} Level;

typedef struct {
  Level* lv;
  int64_t n_levels;
  Chol coarse;
  lsamgdd_params params;
  lsamgdd_level_summary* summary;
  int64_t n_summary;
  Csr g0;
  double timings[64];
  const char* timing_names[64];
  int64_t n_timings;
} Hier;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
static void add_timing(Hier* h, const char* name, double t0) {
  if (h->n_timings < 64) {
    h->timing_names[h->n_timings] = name;
    h->timings[h->n_timings++] = now_s() - t0;
  }
}

static void hier_free(Hier* h) {
  for (int64_t l = 0; l < h->n_levels; ++l) {
    Level* L = &h->lv[l];
    csr_free(&L->A);
    csr_free(&L->G);
    if (L->has_interp) {
      csr_free(&L->P);
      topo_free(&L->topo);
      smoother_free(&L->sm);
    }
    free(L->mult);
    free(L->spec_off);
    free(L->spec);
  }
  free(h->lv);
  free(h->coarse.l);
  free(h->summary);
  csr_free(&h->g0);
  free(h);
}

/* block-diagonal P from panels, exact zeros dropped      hierarchy.hpp:72-95 */
static Csr assemble_P(const Topo* t, double** panels, const int64_t* kcols) {
  int64_t n_coarse = 0, nt = 0;
  for (int64_t i = 0; i < t->n_agg; ++i) {
    if (kcols[i] == 0) fail(LSAMGDD_ERR_SETUP, "assemble_P: aggregate %lld has an empty panel", (long long)i);
    n_coarse += kcols[i];
    nt += (t->omega_off[i + 1] - t->omega_off[i]) * kcols[i];
  }
  Trip* tr = (Trip*)xmalloc((size_t)(nt ? nt : 1) * sizeof(Trip));
  int64_t o = 0, offset = 0;
  for (int64_t i = 0; i < t->n_agg; ++i) {
    const int64_t nw = t->omega_off[i + 1] - t->omega_off[i];
    for (int64_t r = 0; r < nw; ++r)
      for (int64_t c = 0; c < kcols[i]; ++c) {
        tr[o].r = t->omega[t->omega_off[i] + r];
        tr[o].c = offset + c;
        tr[o].v = panels[i][r * kcols[i] + c];
        ++o;
      }
    offset += kcols[i];
  }
  Csr p = csr_from_triplets(t->n_nodes, n_coarse, tr, nt);
  free(tr);
  return p;
}

static void setup_impl(Hier* h, const lsamgdd_params* cp) { /* hierarchy.hpp:106-200 + hooks */
  if (cp->max_levels < 2) fail(LSAMGDD_ERR_INPUT, "setup: max_levels must be at least 2");
  if (cp->coarse_size < 1) fail(LSAMGDD_ERR_INPUT, "setup: coarse_size must be positive");
  if (cp->aggregation_passes < 1) fail(LSAMGDD_ERR_INPUT, "setup: aggregation_passes must be positive");
  if (!(cp->kappa > 1.0)) fail(LSAMGDD_ERR_INPUT, "setup: kappa must exceed 1");
  if (!(cp->must_keep > 1.0)) fail(LSAMGDD_ERR_INPUT, "setup: must_keep must exceed 1");
  if (cp->n_ratios == 0) fail(LSAMGDD_ERR_INPUT, "setup: coarsening_ratios must not be empty");
  for (uint64_t k = 0; k < cp->n_ratios; ++k)
    if (cp->coarsening_ratios[k] < 2) fail(LSAMGDD_ERR_INPUT, "setup: coarsening ratios must be at least 2");
  if (h->g0.nr == 0 || h->g0.nc == 0) fail(LSAMGDD_ERR_INPUT, "setup: factor is empty");
  h->params = *cp;
  h->lv = (Level*)xcalloc((size_t)cp->max_levels, sizeof(Level));
  h->summary = (lsamgdd_level_summary*)xcalloc((size_t)cp->max_levels + 1, sizeof(lsamgdd_level_summary));
  double t0 = now_s();
  h->lv[0].G = csr_copy(&h->g0);
  {
    Csr gt = csr_transpose(&h->g0);
    h->lv[0].A = spgemm_symbolic(&gt, &h->g0);
    csr_free(&gt);
  }
  h->n_levels = 1;
  add_timing(h, "galerkin_A0", t0);
  while ((uint64_t)h->n_levels < cp->max_levels && (uint64_t)h->lv[h->n_levels - 1].A.nr > cp->coarse_size) {
    const int64_t ell = h->n_levels - 1;
    Level* cur = &h->lv[ell];
    const int64_t n = cur->A.nr;
    t0 = now_s();
    int64_t* asg = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
    int64_t n_agg;
    if (ell == 0 && cp->level0_partition) {
      memcpy(asg, cp->level0_partition, (size_t)n * sizeof(int64_t));
      n_agg = cp->level0_n_aggregates;
    } else {
      n_agg = multi_pass_aggregation(&cur->A, (int64_t)cp->aggregation_passes, asg);
    }
    cur->topo = build_topology(&cur->A, asg, n_agg, (ell == 0 && cp->level0_overlap >= 2) ? 2 : 1);
    free(asg);
    add_timing(h, "aggregation_topology", t0);
    t0 = now_s();
    cur->sm = build_smoother(&cur->A, &cur->topo);
    add_timing(h, "build_smoother", t0);
    t0 = now_s();
    RowSets rs = compute_row_sets(&cur->G, &cur->topo);
    cur->mult = rs.mult;
    cur->mult_n = cur->G.nr;
    rs.mult = NULL;
    cur->thresh = cp->thresh_override > 0.0 ? cp->thresh_override
                                            : eigen_threshold(cp->kappa, cur->topo.n_colors, cur->topo.multiplicity_max);
    const uint64_t ridx = (uint64_t)ell < cp->n_ratios - 1 ? (uint64_t)ell : cp->n_ratios - 1;
    const int64_t ratio = (int64_t)cp->coarsening_ratios[ridx];
    const int64_t na = cur->topo.n_agg;
    double** panels = (double**)xcalloc((size_t)na, sizeof(double*));
    int64_t* kcols = (int64_t*)xcalloc((size_t)na, sizeof(int64_t));
    double** eigs = cp->keep_spectra ? (double**)xcalloc((size_t)na, sizeof(double*)) : NULL;
    int64_t* neig = (int64_t*)xcalloc((size_t)na, sizeof(int64_t));
    int64_t* colmap = (int64_t*)xmalloc((size_t)cur->G.nc * sizeof(int64_t));
    for (int64_t c = 0; c < cur->G.nc; ++c) colmap[c] = -1;
    double* wts = NULL;
    int64_t wcap = 0;
    for (int64_t i = 0; i < na; ++i) {
      /* assemble_local                                  splitting.hpp:87-97 */
      const int64_t rows = rs.nz_off[i + 1] - rs.nz_off[i];
      const int64_t* nzr = rs.nz + rs.nz_off[i];
      const int64_t nw = cur->topo.omega_off[i + 1] - cur->topo.omega_off[i];
      const int64_t ng = cur->topo.gamma_off[i + 1] - cur->topo.gamma_off[i];
      double* gw = submatrix(&cur->G, nzr, rows, cur->topo.omega + cur->topo.omega_off[i], nw, colmap);
      double* gg = submatrix(&cur->G, nzr, rows, cur->topo.gamma + cur->topo.gamma_off[i], ng, colmap);
      if (rows > wcap) {
        wcap = rows;
        wts = (double*)realloc(wts, (size_t)wcap * sizeof(double));
      }
      for (int64_t r = 0; r < rows; ++r) wts[r] = 1.0 / (double)cur->mult[nzr[r]];
      int64_t cap = nw;
      if (ell > 0) {
        cap = nw / ratio;
        if (cap == 0) cap = 1;
      } else if (cp->level0_max_modes > 0) {
        cap = (int64_t)cp->level0_max_modes;
      }
      panels[i] = local_gevp(i, gw, gg, wts, rows, nw, ng, cur->thresh, cap, cp->gevp_variant, cp->must_keep, &kcols[i],
                             eigs ? &eigs[i] : NULL, &neig[i]);
      free(gw);
      free(gg);
    }
    free(wts);
    free(colmap);
    rowsets_free(&rs);
    if (eigs) {
      cur->spec_n = na;
      cur->spec_off = (int64_t*)xcalloc((size_t)(na + 1), sizeof(int64_t));
      for (int64_t i = 0; i < na; ++i) cur->spec_off[i + 1] = cur->spec_off[i] + neig[i];
      cur->spec = (double*)xmalloc((size_t)(cur->spec_off[na] ? cur->spec_off[na] : 1) * sizeof(double));
      for (int64_t i = 0; i < na; ++i) {
        memcpy(cur->spec + cur->spec_off[i], eigs[i], (size_t)neig[i] * sizeof(double));
        free(eigs[i]);
      }
      free(eigs);
    }
    free(neig);
    add_timing(h, "local_gevp", t0);
    t0 = now_s();
    cur->P = assemble_P(&cur->topo, panels, kcols);
    cur->has_interp = 1;
    for (int64_t i = 0; i < na; ++i) free(panels[i]);
    free(panels);
    free(kcols);
    Level* nx = &h->lv[ell + 1];
    nx->G = spgemm_symbolic(&cur->G, &cur->P);
    {
      Csr gt = csr_transpose(&nx->G);
      nx->A = spgemm_symbolic(&gt, &nx->G);
      csr_free(&gt);
    }
    h->n_levels++;
    add_timing(h, "galerkin", t0);
    if (nx->A.nr >= cur->A.nr)
      fail(LSAMGDD_ERR_SETUP, "setup: stagnant coarsening at level %lld (%lld -> %lld)", (long long)ell,
           (long long)cur->A.nr, (long long)nx->A.nr);
    lsamgdd_level_summary* row = &h->summary[h->n_summary++];
    row->level = (uint64_t)ell;
    row->dim = (uint64_t)cur->A.nr;
    row->nnz = (uint64_t)csr_nnz(&cur->A);
    row->n_aggregates = (uint64_t)na;
    row->k_c = (uint64_t)cur->topo.n_colors;
    row->n_mult = (uint64_t)cur->topo.multiplicity_max;
    row->thresh = cur->thresh;
    row->modes_kept = (uint64_t)cur->P.nc;
  }
  t0 = now_s();
  const Level* co = &h->lv[h->n_levels - 1];
  const int64_t nc = co->A.nr;
  double* dense = (double*)xcalloc((size_t)(nc * nc), sizeof(double));
  for (int64_t i = 0; i < nc; ++i)
    for (int64_t k = co->A.off[i]; k < co->A.off[i + 1]; ++k) dense[i * nc + co->A.col[k]] = co->A.val[k];
  factor_spd_block(&h->coarse, dense, nc, "coarsest-level matrix", -1);
  free(dense);
  add_timing(h, "coarse_factor", t0);
  lsamgdd_level_summary* last = &h->summary[h->n_summary++];
  last->level = (uint64_t)(h->n_levels - 1);
  last->dim = (uint64_t)nc;
  last->nnz = (uint64_t)csr_nnz(&co->A);
}

/* one V(pre,post) cycle                                   hierarchy.hpp:205-227 */
static void vcycle_impl(const Hier* h, int64_t level, const double* r, double* e) {
  if (level < 0 || level >= h->n_levels) fail(LSAMGDD_ERR_INDEX, "vcycle: level out of range");
  const Level* cur = &h->lv[level];
  const int64_t n = cur->A.nr;
  if (level + 1 == h->n_levels) {
    memcpy(e, r, (size_t)n * sizeof(double));
    chol_solve(&h->coarse, e);
    return;
  }
  double* res = (double*)xmalloc((size_t)n * sizeof(double));
  double* tmp = (double*)xmalloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) e[i] = 0.0;
  for (uint64_t sw = 0; sw < h->params.pre_sweeps; ++sw) {
    memcpy(res, r, (size_t)n * sizeof(double));
    spmv(&cur->A, e, tmp);
    for (int64_t i = 0; i < n; ++i) res[i] += -1.0 * tmp[i];
    smoother_apply(&cur->sm, res, LSAMGDD_RAS, tmp);
    for (int64_t i = 0; i < n; ++i) e[i] += 1.0 * tmp[i];
  }
  memcpy(res, r, (size_t)n * sizeof(double));
  spmv(&cur->A, e, tmp);
  for (int64_t i = 0; i < n; ++i) res[i] += -1.0 * tmp[i];
  const int64_t ncoarse = cur->P.nc;
  double* rc = (double*)xmalloc((size_t)ncoarse * sizeof(double));
  double* ec = (double*)xmalloc((size_t)ncoarse * sizeof(double));
  spmv_transpose(&cur->P, res, rc);
  vcycle_impl(h, level + 1, rc, ec);
  spmv(&cur->P, ec, tmp);
  for (int64_t i = 0; i < n; ++i) e[i] += 1.0 * tmp[i];
  free(rc);
  free(ec);
  for (uint64_t sw = 0; sw < h->params.post_sweeps; ++sw) {
    memcpy(res, r, (size_t)n * sizeof(double));
    spmv(&cur->A, e, tmp);
    for (int64_t i = 0; i < n; ++i) res[i] += -1.0 * tmp[i];
    smoother_apply(&cur->sm, res, LSAMGDD_RAST, tmp);
    for (int64_t i = 0; i < n; ++i) e[i] += 1.0 * tmp[i];
  }
  free(res);
  free(tmp);
}

/* ------------------------------------------------------------------------ */
/* C ABI (mirrors ref_harness.cpp)                                            */

#define GUARD_BEGIN                 \
  jmp_buf jb_;                      \
  jmp_buf* saved_ = g_jmp;          \
  g_jmp = &jb_;                     \
  if (setjmp(jb_)) {                \
    g_jmp = saved_;                 \
    if (err && errlen) {            \
      strncpy(err, g_msg, errlen - 1); \
      err[errlen - 1] = '\0';       \
    }                               \
    return g_code;                  \
  }
#define GUARD_END   \
  g_jmp = saved_;   \
  return LSAMGDD_OK;

static Csr csr_from_abi(const lsamgdd_csr* g) {
  Csr m;
  m.nr = g->n_rows;
  m.nc = g->n_cols;
  m.off = (int64_t*)xmalloc((size_t)(g->n_rows + 1) * sizeof(int64_t));
  m.col = (int64_t*)xmalloc((size_t)(g->nnz ? g->nnz : 1) * sizeof(int64_t));
  m.val = (double*)xmalloc((size_t)(g->nnz ? g->nnz : 1) * sizeof(double));
  memcpy(m.off, g->row_offsets, (size_t)(g->n_rows + 1) * sizeof(int64_t));
  memcpy(m.col, g->col_indices, (size_t)g->nnz * sizeof(int64_t));
  memcpy(m.val, g->values, (size_t)g->nnz * sizeof(double));
  return m;
}

int oracle_setup(const lsamgdd_csr* g0, const lsamgdd_params* p, int32_t plain, void** out, char* err, size_t errlen) {
  (void)plain; /* the restatement has one setup path; hooks default to off */
  *out = NULL;
  Hier* h = (Hier*)calloc(1, sizeof(Hier));
  GUARD_BEGIN
  h->g0 = csr_from_abi(g0);
  setup_impl(h, p);
  *out = h;
  GUARD_END
}

int oracle_destroy(void* h) {
  if (h) hier_free((Hier*)h);
  return LSAMGDD_OK;
}

int oracle_num_levels(const void* h, int64_t* out) {
  *out = ((const Hier*)h)->n_levels;
  return LSAMGDD_OK;
}

int oracle_level_summary(const void* vh, int64_t level, lsamgdd_level_summary* out) {
  const Hier* h = (const Hier*)vh;
  if (level < 0 || level >= h->n_summary) return LSAMGDD_ERR_INDEX;
  *out = h->summary[level];
  return LSAMGDD_OK;
}

int oracle_operator_complexity(const void* vh, double* out) { /* hierarchy.hpp:257-261 */
  const Hier* h = (const Hier*)vh;
  double total = 0.0;
  for (int64_t l = 0; l < h->n_levels; ++l) total += (double)csr_nnz(&h->lv[l].A);
  *out = total / (double)csr_nnz(&h->lv[0].A);
  return LSAMGDD_OK;
}

static void export_csr(const Csr* m, int64_t sizes[3], int64_t* i0, int64_t* i1, double* v) {
  sizes[0] = m->nr;
  sizes[1] = m->nc;
  sizes[2] = csr_nnz(m);
  if (i0) memcpy(i0, m->off, (size_t)(m->nr + 1) * sizeof(int64_t));
  if (i1) memcpy(i1, m->col, (size_t)sizes[2] * sizeof(int64_t));
  if (v) memcpy(v, m->val, (size_t)sizes[2] * sizeof(double));
}

int oracle_level_export(const void* vh, int64_t level, int32_t what, int64_t sizes[3], int64_t* i0, int64_t* i1,
                        double* vals) {
  const Hier* h = (const Hier*)vh;
  if (level < 0 || level >= h->n_levels) return LSAMGDD_ERR_INDEX;
  const Level* L = &h->lv[level];
  sizes[0] = sizes[1] = sizes[2] = 0;
  if (what == LSAMGDD_EXPORT_A) {
    export_csr(&L->A, sizes, i0, i1, vals);
    return LSAMGDD_OK;
  }
  if (what == LSAMGDD_EXPORT_G) {
    export_csr(&L->G, sizes, i0, i1, vals);
    return LSAMGDD_OK;
  }
  if (!L->has_interp) return LSAMGDD_ERR_INDEX;
  const Topo* t = &L->topo;
  switch (what) {
    case LSAMGDD_EXPORT_P:
      export_csr(&L->P, sizes, i0, i1, vals);
      return LSAMGDD_OK;
    case LSAMGDD_EXPORT_PARTITION:
      sizes[0] = t->n_nodes;
      sizes[1] = t->n_agg;
      if (i0)
        for (int64_t i = 0; i < t->n_agg; ++i)
          for (int64_t p = t->omega_off[i]; p < t->omega_off[i + 1]; ++p) i0[t->omega[p]] = i;
      return LSAMGDD_OK;
    case LSAMGDD_EXPORT_GAMMA:
      sizes[0] = t->n_agg;
      sizes[1] = t->gamma_off[t->n_agg];
      if (i0) memcpy(i0, t->gamma_off, (size_t)(t->n_agg + 1) * sizeof(int64_t));
      if (i1) memcpy(i1, t->gamma, (size_t)sizes[1] * sizeof(int64_t));
      return LSAMGDD_OK;
    case LSAMGDD_EXPORT_COLORS:
      sizes[0] = t->n_agg;
      sizes[1] = t->n_colors;
      if (i0) memcpy(i0, t->colors, (size_t)t->n_agg * sizeof(int64_t));
      return LSAMGDD_OK;
    case LSAMGDD_EXPORT_SPECTRA:
      if (!L->spec_off) return LSAMGDD_ERR_INDEX;
      sizes[0] = L->spec_n;
      sizes[1] = L->spec_off[L->spec_n];
      if (i0) memcpy(i0, L->spec_off, (size_t)(L->spec_n + 1) * sizeof(int64_t));
      if (vals) memcpy(vals, L->spec, (size_t)sizes[1] * sizeof(double));
      return LSAMGDD_OK;
    case LSAMGDD_EXPORT_MULTIPLICITY:
      sizes[0] = L->mult_n;
      sizes[1] = t->multiplicity_max;
      if (i0) memcpy(i0, L->mult, (size_t)L->mult_n * sizeof(int64_t));
      return LSAMGDD_OK;
    default:
      return LSAMGDD_ERR_INPUT;
  }
}

int oracle_vcycle(const void* vh, int64_t level, const double* r, double* e, char* err, size_t errlen) {
  const Hier* h = (const Hier*)vh;
  GUARD_BEGIN
  vcycle_impl(h, level, r, e);
  GUARD_END
}

int oracle_schwarz_apply(const void* vh, int64_t level, int32_t mode, const double* r, double* e, char* err,
                         size_t errlen) {
  const Hier* h = (const Hier*)vh;
  GUARD_BEGIN
  if (level < 0 || level + 1 >= h->n_levels) fail(LSAMGDD_ERR_INDEX, "schwarz: level has no smoother");
  smoother_apply(&h->lv[level].sm, r, mode, e);
  GUARD_END
}

int oracle_level_spmv(const void* vh, int64_t level, int32_t what, int32_t trans, const double* x, double* y,
                      char* err, size_t errlen) {
  const Hier* h = (const Hier*)vh;
  GUARD_BEGIN
  if (level < 0 || level >= h->n_levels) fail(LSAMGDD_ERR_INDEX, "spmv: level out of range");
  const Level* L = &h->lv[level];
  const Csr* m = what == 0 ? &L->A : what == 1 ? &L->G : &L->P;
  if (trans)
    spmv_transpose(m, x, y);
  else
    spmv(m, x, y);
  GUARD_END
}

/* pcg with apply_a = Gᵀ(G·), apply_b = vcycle            krylov.hpp:42-92 */
int oracle_pcg(const void* vh, const lsamgdd_csr* gabi, const double* b, double tol, uint64_t maxit, double* x,
               lsamgdd_report* rep, char* err, size_t errlen) {
  const Hier* h = (const Hier*)vh;
  Csr gown;
  memset(&gown, 0, sizeof gown);
  GUARD_BEGIN
  if (gabi) gown = csr_from_abi(gabi);
  const Csr* G = gabi ? &gown : &h->g0;
  const int64_t n = G->nc, m = G->nr;
  const double t0 = now_s();
  double* r = (double*)xmalloc((size_t)n * sizeof(double));
  double* z = (double*)xmalloc((size_t)n * sizeof(double));
  double* p = (double*)xmalloc((size_t)n * sizeof(double));
  double* ap = (double*)xmalloc((size_t)n * sizeof(double));
  double* gp = (double*)xmalloc((size_t)(m ? m : 1) * sizeof(double));
  double* hist = (double*)xmalloc((size_t)(maxit + 2) * sizeof(double));
  int64_t nh = 0;
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  memcpy(r, b, (size_t)n * sizeof(double));
  const double r0 = vnorm(r, n);
  hist[nh++] = r0;
  int converged = 0;
  uint64_t k = 0;
  if (r0 == 0.0) {
    converged = 1;
  } else {
    vcycle_impl(h, 0, r, z);
    double rz = vdot(r, z, n);
    if (!(rz > 0.0)) fail(LSAMGDD_ERR_INDEFINITE, "pcg: preconditioned product <r, Br> is not positive");
    memcpy(p, z, (size_t)n * sizeof(double));
    while (k < maxit) {
      spmv(G, p, gp);
      spmv_transpose(G, gp, ap);
      const double pap = vdot(p, ap, n);
      if (!(pap > 0.0)) fail(LSAMGDD_ERR_INDEFINITE, "pcg: curvature <p, Ap> is not positive");
      const double alpha = rz / pap;
      for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
      for (int64_t i = 0; i < n; ++i) r[i] += -alpha * ap[i];
      ++k;
      const double rn = vnorm(r, n);
      hist[nh++] = rn;
      if (rn <= tol * r0) {
        converged = 1;
        break;
      }
      vcycle_impl(h, 0, r, z);
      const double rz_next = vdot(r, z, n);
      if (!(rz_next > 0.0)) fail(LSAMGDD_ERR_INDEFINITE, "pcg: preconditioned product <r, Br> is not positive");
      const double beta = rz_next / rz;
      rz = rz_next;
      for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
  }
  if (rep) {
    rep->iterations = r0 == 0.0 ? 0 : k;
    rep->converged = converged;
    double avg = 1.0, itt = 0.0;
    if (r0 != 0.0) {
      const double ratio = hist[nh - 1] / r0;
      avg = k > 0 ? pow(ratio, 1.0 / (double)k) : 1.0;
      if (avg > 0.0 && avg < 1.0)
        itt = log(0.1) / log(avg);
      else if (avg == 0.0)
        itt = 0.0;
      else
        itt = INFINITY;
    }
    rep->avg_conv_factor = r0 == 0.0 ? 0.0 : avg;
    rep->iters_to_tenth = itt;
    oracle_operator_complexity(h, &rep->operator_complexity);
    rep->solve_seconds = now_s() - t0;
    rep->history_len = (uint64_t)nh;
    if (rep->residual_history)
      for (int64_t i = 0; i < nh && (uint64_t)i < rep->history_capacity; ++i) rep->residual_history[i] = hist[i];
  }
  free(r);
  free(z);
  free(p);
  free(ap);
  free(gp);
  free(hist);
  csr_free(&gown);
  GUARD_END
}

int oracle_setup_timings(const void* vh, const char** names, double* secs, int64_t n, int64_t* count) {
  const Hier* h = (const Hier*)vh;
  *count = h->n_timings;
  for (int64_t i = 0; i < n && i < h->n_timings; ++i) {
    names[i] = h->timing_names[i];
    secs[i] = h->timings[i];
  }
  return LSAMGDD_OK;
}

int oracle_sym_eig(int64_t n, const double* a, double* values, double* vectors, char* err, size_t errlen) {
  GUARD_BEGIN
  sym_eig(n, a, values, vectors);
  GUARD_END
}

int oracle_spsd_gevp(int64_t n, const double* l, const double* b, double tau, double* values, double* vectors,
                     int64_t* k, int64_t* discarded, char* err, size_t errlen) {
  GUARD_BEGIN
  *k = spsd_gevp(n, l, b, tau, values, vectors, discarded);
  GUARD_END
}

int oracle_pseudo_inverse(int64_t n, const double* a, double tau, double* out, char* err, size_t errlen) {
  GUARD_BEGIN
  pseudo_inverse(n, a, tau, out);
  GUARD_END
}

int oracle_standard_aggregation(const lsamgdd_csr* a, int64_t* assignment, int64_t* n_agg, char* err, size_t errlen) {
  GUARD_BEGIN
  Csr m = csr_from_abi(a);
  *n_agg = standard_aggregation(&m, assignment);
  csr_free(&m);
  GUARD_END
}

/* mt19937_64 + uniform_real_distribution (libstdc++), lsamgdd_cli.cpp:103-107 */
void oracle_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
  uint64_t mt[312];
  int idx = 312;
  mt[0] = seed;
  for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  for (int64_t k = 0; k < n; ++k) {
    if (idx >= 312) {
      for (int i = 0; i < 312; ++i) {
        const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        mt[i] = mt[(i + 156) % 312] ^ xa;
      }
      idx = 0;
    }
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    double c = (double)y / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    out[k] = c * (hi - lo) + lo;
  }
}

int oracle_eigen_threshold(double kappa, int64_t kc, int64_t n_mult, double* out, char* err, size_t errlen) {
  GUARD_BEGIN
  *out = eigen_threshold(kappa, kc, n_mult);
  GUARD_END
}
