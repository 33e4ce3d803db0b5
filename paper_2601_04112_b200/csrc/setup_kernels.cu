// setup_kernels.cu — batched per-aggregate setup stages (splitting.hpp,
// smoother.hpp, hierarchy.hpp:72-95/193) on sm_100a.
//
// Each aggregate is one independent problem solved by a Team (a warp for
// small problems, a CTA otherwise) over a private workspace in shared memory
// when it fits, global memory otherwise. All FP64 arithmetic follows the
// reference's operation order (see dense_dev.cuh), so panels, spectra and
// factors are bit-identical to the reference's no-FMA build.
#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>
#include <tuple>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "dense_dev.cuh"
#include "setup_kernels.cuh"

// Diagnostics (per-phase cycle counters, the tiled-Gram cross-check) exist only in builds made
// with `make DIAG=1` (-DLSB_DIAG); the product library reads no environment variable.
#ifdef LSB_DIAG
#define LSB_DIAG_ENV(name) (getenv(name) != nullptr)
#else
#define LSB_DIAG_ENV(name) false
#endif

namespace lsb {

namespace {

constexpr int kThreads = 256;

int grid_for(int64_t n, int threads = kThreads) {
  const int64_t cap = int64_t(sm_count()) * 16;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap)));
}

int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (uint64_t(1) << b) <= v) ++b;
  return b;
}

__host__ __device__ inline int64_t r2(int64_t x) { return (x + 1) & ~int64_t(1); }

// position of node c in Ω_i = ω_i ‖ Γ_i (both ascending), or -1
__device__ inline int lookup_sub(int c, const int32_t* om, int nw, const int32_t* ga, int ng) {
  int lo = 0, hi = nw - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int v = om[mid];
    if (v == c) return mid;
    if (v < c)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  lo = 0;
  hi = ng - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int v = ga[mid];
    if (v == c) return nw + mid;
    if (v < c)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  return -1;
}

// ---- row sets ---------------------------------------------------------------

__global__ void k_owner_keys(const int64_t* goff, const int32_t* gcol, int64_t m, const int32_t* node_agg,
                             uint64_t* keys) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x)
    for (int64_t k = goff[r]; k < goff[r + 1]; ++k)
      keys[k] = static_cast<uint64_t>(node_agg[gcol[k]]) * static_cast<uint64_t>(m) + static_cast<uint64_t>(r);
}

__global__ void k_rowset_fill(const uint64_t* keys, int64_t n, uint64_t m, int64_t* agg_cnt, int32_t* mult,
                              int32_t* nz, int64_t* nz_pos_flag) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x)
    nz_pos_flag[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

__global__ void k_rowset_scatter(const uint64_t* keys, const int64_t* flag, const int64_t* pos, int64_t n, uint64_t m,
                                 int64_t* agg_cnt, int32_t* mult, int32_t* nz) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    if (!flag[p]) continue;
    const uint64_t key = keys[p];
    const int64_t agg = static_cast<int64_t>(key / m);
    const int64_t row = static_cast<int64_t>(key % m);
    nz[pos[p]] = static_cast<int32_t>(row);
    atomicAdd(reinterpret_cast<unsigned long long*>(&agg_cnt[agg + 1]), 1ull);
    atomicAdd(&mult[row], 1);
  }
}

__global__ void k_row_stats(const int64_t* goff, const int32_t* mult, int64_t m, unsigned long long* out3) {
  // out3[0] = max mult, out3[1] = empty rows, out3[2] = max row nnz
  unsigned long long mx = 0, empty = 0, mr = 0;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long mu = static_cast<unsigned long long>(mult[r]);
    mx = mu > mx ? mu : mx;
    empty += mu == 0 ? 1 : 0;
    const unsigned long long len = static_cast<unsigned long long>(goff[r + 1] - goff[r]);
    mr = len > mr ? len : mr;
  }
  atomicMax(&out3[0], mx);
  atomicAdd(&out3[1], empty);
  atomicMax(&out3[2], mr);
}

// ---- team problem dispatch ----------------------------------------------------

struct TeamSlot {
  int prob;
  double* ws;
};

// ---- local GEVP (splitting.hpp:200-275) -----------------------------------------

struct GevpArgs {
  const int64_t* goff;
  const int32_t* gcol;
  const double* gval;
  const int32_t* mult;
  const int32_t* omega_off;
  const int32_t* omega;
  const int32_t* gamma_off;
  const int32_t* gamma;
  const int64_t* nz_off;
  const int32_t* nz;
  const int32_t* list;
  int n_list;
  int list_base;
  int maxrow;
  GevpParams p;
  double* panel_tmp;
  const int64_t* panel_off;  // per list entry (capacity nω²)
  double* spec;
  const int64_t* spec_off;   // per aggregate (capacity nω)
  int32_t* kcols;            // per aggregate
  int32_t* nspec;            // per aggregate
  int32_t* status;           // per aggregate
  double* gws;
  int64_t ws_stride;
  const double* pre;         // Grams precomputed by tiled_grams (grams.cu), or null
  const int64_t* pre_off;    // per aggregate: offset into pre, -1 when not precomputed
};

__host__ __device__ inline int64_t gevp_ws(int64_t nw, int64_t ng, int64_t maxrow) {
  int64_t a = r2(nw * ng) + r2(ng * ng) + r2((maxrow + 1) / 2) + r2(maxrow);
  if (ng > 0) a += r2(ng * ng) + r2(ng * nw) + r2(nw * nw) + r2(ng) + r2(ng * ng) + sym_eig_scratch(ng);
  const int64_t b = r2(nw) + r2(nw * nw) + r2(nw * nw) + r2(nw) + spsd_gevp_scratch(nw);
  return r2(8) + 2 * r2(nw * nw) + (a > b ? a : b);
}

// diagnostic hook (LSB_GRAM_CHECK): recompute tiled Grams per team and count mismatches
__device__ int g_gram_check = 0;
__device__ unsigned long long g_gram_bad[8];
// optional per-aggregate phase cycle counters (diagnostic hook, LSB_GEVP_PROF)
__device__ long long* g_gevp_prof = nullptr;

template <class Team>
__device__ void gevp_problem(const Team& t, const GevpArgs& g, int idx, double* ws, double* fast = nullptr,
                             int64_t fast_cap = 0, WaveCtl* wctl = nullptr, double* wws = nullptr, int wave_min = 0) {
  const int agg = g.list[idx];
  long long* const gprof = g_gevp_prof;
  long long ck = gprof ? clock64() : 0;
  auto mark = [&](int k) {
    if (gprof && t.rank() == 0) {
      const long long now = clock64();
      gprof[int64_t(agg) * 6 + k] = now - ck;
      ck = now;
    }
  };
  const int32_t* om = g.omega + g.omega_off[agg];
  const int nw = g.omega_off[agg + 1] - g.omega_off[agg];
  const int32_t* ga = g.gamma + g.gamma_off[agg];
  const int ng = g.gamma_off[agg + 1] - g.gamma_off[agg];
  constexpr double tau_rel = 1e-10;
  Arena ar{ws, 0, fast, fast_cap};
  ar.wctl = wctl;
  ar.wws = wws;
  ar.wave_min = wave_min;
  double* slot = ar.take(8);
  double* L = ar.take(int64_t(nw) * nw);
  double* W = ar.take(int64_t(nw) * nw);
  const Arena base = ar;

  // ---- phase A: Grams straight from G's sparse rows (weighted_gram,
  // splitting.hpp:102-115: rows ascending, zero w·x skipped).
  Arena pa = base;
  double* C = pa.take(int64_t(nw) * ng);
  double* B = pa.take(int64_t(ng) * ng);
  int* rpos = pa.take_int(g.maxrow);
  double* rval = pa.take(g.maxrow);
  const int64_t pre_chk = g.pre_off ? g.pre_off[agg] : -1;
  const int64_t pre_at = g_gram_check ? -1 : pre_chk;
  if (pre_at >= 0) {
    const double* src = g.pre + pre_at;
    t_copy(t, L, src, int64_t(nw) * nw);
    t_copy(t, W, src + int64_t(nw) * nw, int64_t(nw) * nw);
    t_copy(t, C, src + 2 * int64_t(nw) * nw, int64_t(nw) * ng);
    t_copy(t, B, src + 2 * int64_t(nw) * nw + int64_t(nw) * ng, int64_t(ng) * ng);
  } else {
    t_fill(t, L, 0.0, 2 * r2(int64_t(nw) * nw));
    t_fill(t, C, 0.0, r2(int64_t(nw) * ng) + r2(int64_t(ng) * ng));
  }
  const bool weighted_lhs = g.p.variant == 1;
  for (int64_t ri = pre_at >= 0 ? 0 : g.nz_off[agg]; ri < (pre_at >= 0 ? 0 : g.nz_off[agg + 1]); ++ri) {
    const int r = g.nz[ri];
    const double w = 1.0 / static_cast<double>(g.mult[r]);
    const int64_t k0 = g.goff[r];
    const int len = static_cast<int>(g.goff[r + 1] - k0);
    for (int e = t.rank(); e < len; e += t.size()) {
      rpos[e] = lookup_sub(g.gcol[k0 + e], om, nw, ga, ng);
      rval[e] = g.gval[k0 + e];
    }
    t.sync();
    const int pairs = len * len;
    for (int pe = t.rank(); pe < pairs; pe += t.size()) {
      const int e1 = pe / len, e2 = pe % len;
      const int a = rpos[e1], b = rpos[e2];
      if (a < 0 || b < 0) continue;
      const double va = rval[e1], vb = rval[e2];
      const double xw = w * va;
      if (a < nw) {
        if (b < nw) {
          L[int64_t(a) * nw + b] += (weighted_lhs ? xw : va) * vb;
          W[int64_t(a) * nw + b] += xw * vb;
        } else {
          C[int64_t(a) * ng + (b - nw)] += xw * vb;
        }
      } else if (b >= nw) {
        B[int64_t(a - nw) * ng + (b - nw)] += xw * vb;
      }
    }
    t.sync();
  }
  if (g_gram_check && pre_chk >= 0) {  // diagnostic: compare the tiled Grams with this sweep
    const double* src = g.pre + pre_chk;
    const double* mats[4] = {L, W, C, B};
    const int64_t sz[4] = {int64_t(nw) * nw, int64_t(nw) * nw, int64_t(nw) * ng, int64_t(ng) * ng};
    int64_t at = 0;
    for (int q = 0; q < 4; ++q) {
      for (int64_t e = t.rank(); e < sz[q]; e += t.size()) {
        const double a = mats[q][e], b = src[at + e];
        if (__double_as_longlong(a) != __double_as_longlong(b)) {
          const unsigned long long k = atomicAdd(&g_gram_bad[0], 1ull);
          if (k == 0) {
            g_gram_bad[1] = agg;
            g_gram_bad[2] = q;
            g_gram_bad[3] = e;
            g_gram_bad[4] = __double_as_longlong(a);
            g_gram_bad[5] = __double_as_longlong(b);
          }
        }
      }
      at += sz[q];
    }
    t.sync();
  }
  mark(0);
  if (ng > 0) {
    double* Pm = pa.take(int64_t(ng) * ng);
    double* T = pa.take(int64_t(ng) * nw);
    double* S = pa.take(int64_t(nw) * nw);
    const int st = t_pseudo_inverse(t, ng, B, tau_rel, Pm, pa);
    if (st) {
      if (t.rank() == 0) g.status[agg] = st;
      return;
    }
    mark(1);
    // T = pinv·crossᵀ, S = cross·T (dense.hpp:47-59 with the transposed copy)
    if (nw <= 2 * ng) {  // crossᵀ materialised in the eigensolver's scratch: coalesced reads
      double* Ct = pa.take(int64_t(ng) * nw);
      for (int64_t e = t.rank(); e < int64_t(ng) * nw; e += t.size()) {
        const int k = static_cast<int>(e / nw), j = static_cast<int>(e % nw);
        Ct[e] = C[int64_t(j) * ng + k];
      }
      t.sync();
      t_matmul(t, Pm, ng, ng, Ct, nw, T);
    } else {
      for (int64_t e = t.rank(); e < int64_t(ng) * nw; e += t.size()) {
        const int i = static_cast<int>(e / nw), j = static_cast<int>(e % nw);
        double s = 0.0;
        for (int k = 0; k < ng; ++k) {
          const double aik = Pm[int64_t(i) * ng + k];
          if (aik == 0.0) continue;
          s += aik * C[int64_t(j) * ng + k];
        }
        T[e] = s;
      }
      t.sync();
    }
    t_matmul(t, C, nw, ng, T, nw, S);
    for (int64_t e = t.rank(); e < int64_t(nw) * nw; e += t.size()) W[e] -= S[e];
    t.sync();
  }
  t_symmetrize(t, W, nw);
  mark(2);

  // ---- phase B: pencil, keep rule, MGS, sign rule
  Arena pb = base;
  double* values = pb.take(nw);
  double* outv = pb.take(int64_t(nw) * nw);
  double* panel = pb.take(int64_t(nw) * nw);  // column-major nw × keep
  double* v = pb.take(nw);
  int cnt = 0;
  int st = t_spsd_gevp(t, nw, L, W, tau_rel, values, outv, &cnt, pb);
  if (st) {
    if (t.rank() == 0) g.status[agg] = st;
    return;
  }
  mark(3);
  for (int k = t.rank(); k < cnt; k += t.size()) g.spec[g.spec_off[agg] + k] = values[k];
  if (t.rank() == 0) g.nspec[agg] = cnt;
  for (int k = 0; k < cnt; ++k)
    if (isnan(values[k])) {
      if (t.rank() == 0) g.status[agg] = 3;
      return;
    }
  int64_t max_modes = nw;
  if (g.p.level > 0) {
    max_modes = nw / g.p.ratio;
    if (max_modes == 0) max_modes = 1;
  } else if (g.p.level0_max_modes > 0) {
    max_modes = g.p.level0_max_modes;
  }
  if (max_modes == 0) max_modes = 1;
  int n_null = 0;
  while (n_null < cnt && isinf(values[n_null])) ++n_null;
  int above = n_null;
  while (above < cnt && values[above] > g.p.thresh) ++above;
  int severe = n_null;
  while (severe < above && values[severe] >= g.p.must_keep) ++severe;
  int64_t fin = min(int64_t(above - n_null), max_modes);
  if (severe - n_null > fin) fin = severe - n_null;
  int64_t keep = n_null + fin;
  if (keep == 0) keep = 1;
  if (keep > cnt) keep = cnt;
  int cols = 0;
  double* const dsm = (fast && fast_cap >= nw + 1) ? fast : nullptr;  // shared scratch of the ordered dots
  for (int k = 0; k < keep; ++k) {
    for (int r = t.rank(); r < nw; r += t.size()) v[r] = outv[int64_t(k) * nw + r];
    t.sync();
    const double orig = sqrt(t_seq_dot(t, v, v, nw, slot, dsm));
    for (int pass = 0; pass < 2; ++pass)
      for (int c = 0; c < cols; ++c) {
        const double* pc = panel + int64_t(c) * nw;
        const double proj = t_seq_dot(t, pc, v, nw, slot, dsm);
        for (int r = t.rank(); r < nw; r += t.size()) v[r] -= proj * pc[r];
        t.sync();
      }
    const double nv = sqrt(t_seq_dot(t, v, v, nw, slot, dsm));
    if (!(nv > 1e-12 * fmax(orig, 1e-300))) continue;
    if (t.rank() == 0) {
      int arg = 0;
      for (int r = 1; r < nw; ++r)
        if (fabs(v[r]) > fabs(v[arg])) arg = r;
      slot[1] = v[arg] < 0.0 ? -1.0 : 1.0;
    }
    t.sync();
    const double sign = slot[1];
    for (int r = t.rank(); r < nw; r += t.size()) panel[int64_t(cols) * nw + r] = sign * v[r] / nv;
    t.sync();
    ++cols;
  }
  double* out = g.panel_tmp + g.panel_off[g.list_base + idx];
  if (cols == 0) {
    const double unit = 1.0 / sqrt(static_cast<double>(nw));
    for (int r = t.rank(); r < nw; r += t.size()) out[r] = unit;
    if (t.rank() == 0) g.kcols[agg] = 1;
  } else {
    for (int64_t e = t.rank(); e < int64_t(nw) * cols; e += t.size()) {
      const int r = static_cast<int>(e / cols), c = static_cast<int>(e % cols);
      out[e] = panel[int64_t(c) * nw + r];
    }
    if (t.rank() == 0) g.kcols[agg] = cols;
  }
  t.sync();
  mark(4);
}

extern __shared__ __align__(128) double dyn_smem[];

template <int WPB>
__global__ void __launch_bounds__(WPB * 32) k_gevp_warp(GevpArgs g) {
  WarpTeam t;
  const int warp = threadIdx.x >> 5;
  double* ws = dyn_smem + int64_t(warp) * g.ws_stride;
  for (int idx = blockIdx.x * WPB + warp; idx < g.n_list; idx += gridDim.x * WPB) gevp_problem(t, g, idx, ws);
}

// Mid-size subdomains (workspace beyond the shared-memory warp class, eigenproblems up to
// kWarpGlobMax): one warp per problem with its workspace in global memory (L1/L2-resident), many
// problems per SM — the per-problem latency of the warp team matches the one-CTA-per-problem
// kernels at these sizes (measured), the occupancy is 16 problems per SM instead of one.
template <int WPB>
__global__ void __launch_bounds__(WPB * 32) k_gevp_warp_g(GevpArgs g) {
  WarpTeam t;
  const int warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * WPB + warp;
  double* ws = g.gws + int64_t(slot) * g.ws_stride;
  for (int idx = slot; idx < g.n_list; idx += gridDim.x * WPB) gevp_problem(t, g, idx, ws);
}

// shared doubles for the pipelined Jacobi: 207 KiB dynamic + the kernels'
// static shared arrays (15 KiB) stay within the 227 KiB per CTA
constexpr int64_t kFastCap = 26500;
constexpr int kWaveCluster = 4;  // CTAs per cluster of the wavefront Jacobi: 1 leader + 3 replay CTAs
constexpr int64_t kWaveClassMin = 100;  // subdomains with max(nω, nΓ) >= this run in clusters
constexpr int64_t kWaveSmallMax = 256;  // ... of 2 CTAs up to this size, of 4 CTAs above
constexpr int64_t kWarpGlobMax = 99;    // below the cluster class: warp teams with global workspaces
constexpr int kWaveMinN = 1;            // ... where every eigensolve takes the wavefront path

template <bool SMEM>
__global__ void __launch_bounds__(512) k_gevp_block(GevpArgs g) {
  BlockTeam t;
  double* ws = SMEM ? dyn_smem : g.gws + int64_t(blockIdx.x) * g.ws_stride;
  for (int idx = blockIdx.x; idx < g.n_list; idx += gridDim.x) {
    if (SMEM)
      gevp_problem(t, g, idx, ws);
    else
      gevp_problem(t, g, idx, ws, dyn_smem, kFastCap);
  }
}

// Large subdomains: one cluster per problem slot. CTA 0 runs the problem; its
// eigensolves with n >= wave_min take the wavefront Jacobi (jacobi_wave.cuh),
// for which CTAs 1..C-1 replay the rotation log on V and the finished rows.
constexpr int64_t kWaveSmemCap = 28752;  // doubles: wave_smem_doubles(608)
__global__ void __launch_bounds__(512, 1) k_gevp_wave(GevpArgs g, WaveCtl* ctls, double* wws, int64_t wws_stride,
                                                    int wave_min) {
  const cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int slot = blockIdx.x / C, nslots = gridDim.x / C;
  WaveCtl* ctl = ctls + slot;
  if (cl.block_rank() != 0) {
    wave_helper_main(ctl, dyn_smem);
    return;
  }
  ClusterLeadTeam t;
  double* ws = g.gws + int64_t(slot) * g.ws_stride;
  // the list is sorted largest first; a cluster takes the next problem when it finishes one
  __shared__ int s_idx;
  (void)nslots;
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(&ctls[0].next, 1);
    __syncthreads();
    const int idx = s_idx;
    __syncthreads();
    if (idx >= g.n_list) break;
#ifdef LSB_DIAG
    if (threadIdx.x == 0 && ctl->n_done == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ctl->t_start));
#endif
    gevp_problem(t, g, idx, ws, dyn_smem, kWaveSmemCap, ctl, wws + int64_t(slot) * wws_stride, wave_min);
#ifdef LSB_DIAG
    if (threadIdx.x == 0) {
      ctl->n_done += 1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ctl->t_end));
    }
#endif
  }
  wave_quit(ctl);
}

// ---- smoother blocks (smoother.hpp:38-58, dense.hpp:119-185) ---------------------

struct SmArgs {
  const int64_t* aoff;
  const int32_t* acol;
  const double* aval;
  const int32_t* omega_off;
  const int32_t* omega;
  const int32_t* gamma_off;
  const int32_t* gamma;
  const int32_t* list;
  int n_list;
  int list_base;
  const int64_t* sm_off;
  double* sm_data;
  int32_t* status;
  double* gws;
  int64_t ws_stride;
};

constexpr int kSmBigSub = 96;  // CTA teams factor subdomains of at least this size warp-parallel

__host__ __device__ inline int64_t sm_ws(int64_t nw, int64_t ng) {
  const int64_t m = nw + ng;
  return r2(8) + 2 * r2(m * m) + r2(nw * m);
}

// Right-looking Cholesky of the full block (dense.hpp:135-153). Returns
// false on a non-positive pivot.
template <class Team>
__device__ bool t_cholesky(const Team& t, double* l, int m, double* slot) {
  for (int j = 0; j < m; ++j) {
    if (t.rank() == 0) {
      double d = l[int64_t(j) * m + j];
      for (int k = 0; k < j; ++k) d -= l[int64_t(j) * m + k] * l[int64_t(j) * m + k];
      slot[0] = d;
    }
    t.sync();
    const double d = slot[0];
    if (!(d > 0.0)) {
      t.sync();
      return false;
    }
    const double ljj = sqrt(d);
    for (int i = j + 1 + t.rank(); i < m; i += t.size()) {
      double s = l[int64_t(i) * m + j];
      for (int k = 0; k < j; ++k) s -= l[int64_t(i) * m + k] * l[int64_t(j) * m + k];
      l[int64_t(i) * m + j] = s / ljj;
    }
    if (t.rank() == 0) l[int64_t(j) * m + j] = ljj;
    t.sync();
  }
  return true;
}

// factor_spd_block with its single jitter retry
template <class Team>
__device__ bool t_factor_spd(const Team& t, double* blk, const double* orig, int m, double* slot) {
  if (t_cholesky(t, blk, m, slot)) return true;
  if (t.rank() == 0) {
    double maxd = 0.0;
    for (int i = 0; i < m; ++i) maxd = fmax(maxd, fabs(orig[int64_t(i) * m + i]));
    slot[1] = 1e-12 * maxd;
  }
  t.sync();
  const double jitter = slot[1];
  for (int64_t e = t.rank(); e < int64_t(m) * m; e += t.size())
    blk[e] = orig[e] + ((e / m == e % m) ? jitter : 0.0);
  t.sync();
  return t_cholesky(t, blk, m, slot);
}

// column j of (L Lᵀ)⁻¹ by forward then backward substitution (dense.hpp:145-158)
__device__ inline void chol_solve_unit(const double* l, int m, int j, double* x) {
  for (int i = 0; i < m; ++i) x[i] = (i == j) ? 1.0 : 0.0;
  for (int i = 0; i < m; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= l[int64_t(i) * m + k] * x[k];
    x[i] = s / l[int64_t(i) * m + i];
  }
  for (int ii = m; ii-- > 0;) {
    double s = x[ii];
    for (int k = ii + 1; k < m; ++k) s -= l[int64_t(k) * m + ii] * x[k];
    x[ii] = s / l[int64_t(ii) * m + ii];
  }
}

// Large blocks (CTA team): the same factorization and inverse columns with a
// warp per dot product (coalesced rows, fixed xor-tree order). The Schwarz
// blocks only feed the smoother (solve tolerance), so the
// reordered sums are deterministic but not the reference's bits.
__device__ inline double warp_dot(const double* a, const double* b, int n, int lane) {
  double s0 = 0.0, s1 = 0.0;
  int k = lane;
  for (; k + 32 < n; k += 64) {
    s0 += a[k] * b[k];
    s1 += a[k + 32] * b[k + 32];
  }
  if (k < n) s0 += a[k] * b[k];
  double s = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__device__ bool cta_cholesky_rows(const BlockTeam& t, double* l, int m, double* slot) {
  const int warp = t.rank() >> 5, lane = t.rank() & 31, nwarps = t.size() >> 5;
  for (int j = 0; j < m; ++j) {
    const double* rj = l + int64_t(j) * m;
    if (warp == 0) {
      const double dd = warp_dot(rj, rj, j, lane);
      if (lane == 0) slot[0] = rj[j] - dd;
    }
    t.sync();
    const double d = slot[0];
    if (!(d > 0.0)) {
      t.sync();
      return false;
    }
    const double ljj = sqrt(d);
    for (int i = j + 1 + warp; i < m; i += nwarps) {
      double* ri = l + int64_t(i) * m;
      const double sdot = warp_dot(ri, rj, j, lane);
      if (lane == 0) ri[j] = (ri[j] - sdot) / ljj;
    }
    if (t.rank() == 0) l[int64_t(j) * m + j] = ljj;
    t.sync();
  }
  return true;
}

__device__ bool cta_factor_spd(const BlockTeam& t, double* blk, const double* orig, int m, double* slot) {
  if (cta_cholesky_rows(t, blk, m, slot)) return true;
  if (t.rank() == 0) {
    double maxd = 0.0;
    for (int i = 0; i < m; ++i) maxd = fmax(maxd, fabs(orig[int64_t(i) * m + i]));
    slot[1] = 1e-12 * maxd;
  }
  t.sync();
  const double jitter = slot[1];
  for (int64_t e = t.rank(); e < int64_t(m) * m; e += t.size())
    blk[e] = orig[e] + ((e / m == e % m) ? jitter : 0.0);
  t.sync();
  return cta_cholesky_rows(t, blk, m, slot);
}

// columns j < nw of (L Lᵀ)⁻¹, a warp per column: forward over rows of L,
// backward over rows of Lt = Lᵀ (both contiguous)
__device__ void cta_inverse_columns(const BlockTeam& t, const double* l, double* lt, int m, int nw, double* X) {
  const int warp = t.rank() >> 5, lane = t.rank() & 31, nwarps = t.size() >> 5;
  for (int64_t e = t.rank(); e < int64_t(m) * m; e += t.size()) {
    const int i = static_cast<int>(e / m), k = static_cast<int>(e % m);
    lt[int64_t(k) * m + i] = l[e];
  }
  t.sync();
  for (int j = warp; j < nw; j += nwarps) {
    double* x = X + int64_t(j) * m;
    for (int i = lane; i < j; i += 32) x[i] = 0.0;
    __syncwarp();
    for (int i = j; i < m; ++i) {
      const double* ri = l + int64_t(i) * m;
      const double sdot = warp_dot(ri + j, x + j, i - j, lane);
      if (lane == 0) x[i] = ((i == j ? 1.0 : 0.0) - sdot) / ri[i];
      __syncwarp();
    }
    for (int ii = m - 1; ii >= 0; --ii) {
      const double* ci = lt + int64_t(ii) * m;
      const double sdot = warp_dot(ci + ii + 1, x + ii + 1, m - ii - 1, lane);
      if (lane == 0) x[ii] = (x[ii] - sdot) / ci[ii];
      __syncwarp();
    }
  }
  t.sync();
}

template <class Team>
__device__ void smoother_problem(const Team& t, const SmArgs& g, int idx, double* ws) {
  const int agg = g.list[idx];
  const int32_t* om = g.omega + g.omega_off[agg];
  const int nw = g.omega_off[agg + 1] - g.omega_off[agg];
  const int32_t* ga = g.gamma + g.gamma_off[agg];
  const int ng = g.gamma_off[agg + 1] - g.gamma_off[agg];
  const int m = nw + ng;
  Arena ar{ws, 0};
  double* slot = ar.take(8);
  double* blk = ar.take(int64_t(m) * m);
  double* orig = ar.take(int64_t(m) * m);
  double* X = ar.take(int64_t(nw) * m);
  t_fill(t, orig, 0.0, int64_t(m) * m);
  for (int i = t.rank(); i < m; i += t.size()) {  // submatrix(A, Ω, Ω)
    const int node = i < nw ? om[i] : ga[i - nw];
    for (int64_t k = g.aoff[node]; k < g.aoff[node + 1]; ++k) {
      const int q = lookup_sub(g.acol[k], om, nw, ga, ng);
      if (q >= 0) orig[int64_t(i) * m + q] = g.aval[k];
    }
  }
  t.sync();
  t_copy(t, blk, orig, int64_t(m) * m);
  bool big = false;
  if constexpr (std::is_same<Team, BlockTeam>::value) big = m >= kSmBigSub && t.size() >= 256;
  if (big) {
    if constexpr (std::is_same<Team, BlockTeam>::value) {
      if (!cta_factor_spd(t, blk, orig, m, slot)) {
        if (t.rank() == 0) g.status[agg] = 1;
        return;
      }
      cta_inverse_columns(t, blk, orig, m, nw, X);  // orig is free now: it holds Lᵀ
    }
  } else {
    if (!t_factor_spd(t, blk, orig, m, slot)) {
      if (t.rank() == 0) g.status[agg] = 1;
      return;
    }
    for (int j = t.rank(); j < nw; j += t.size()) chol_solve_unit(blk, m, j, X + int64_t(j) * m);
    t.sync();
  }
  double* out = g.sm_data + g.sm_off[agg];
  const int64_t packed = int64_t(nw) * (nw + 1) / 2;
  for (int64_t e = t.rank(); e < packed; e += t.size()) {
    // e -> (i, j), i <= j, row-major packed upper
    int i = 0;
    int64_t rem = e;
    while (rem >= nw - i) {
      rem -= nw - i;
      ++i;
    }
    const int j = i + static_cast<int>(rem);
    out[e] = X[int64_t(j) * m + i];
  }
  for (int64_t e = t.rank(); e < int64_t(nw) * ng; e += t.size()) {
    const int i = static_cast<int>(e / ng), gg = static_cast<int>(e % ng);
    out[packed + e] = X[int64_t(i) * m + nw + gg];
  }
  t.sync();
}

template <int WPB>
__global__ void __launch_bounds__(WPB * 32) k_sm_warp(SmArgs g) {
  WarpTeam t;
  const int warp = threadIdx.x >> 5;
  double* ws = dyn_smem + int64_t(warp) * g.ws_stride;
  for (int idx = blockIdx.x * WPB + warp; idx < g.n_list; idx += gridDim.x * WPB) smoother_problem(t, g, idx, ws);
}

template <bool SMEM>
__global__ void k_sm_block(SmArgs g) {
  BlockTeam t;
  double* ws = SMEM ? dyn_smem : g.gws + int64_t(blockIdx.x) * g.ws_stride;
  for (int idx = blockIdx.x; idx < g.n_list; idx += gridDim.x) smoother_problem(t, g, idx, ws);
}

// ---- lane-interleaved Schwarz layout ------------------------------------------------

__global__ void k_lane_pack(const int32_t* g_agg, const int32_t* g_nw, const int32_t* g_ng, const int64_t* g_ids_off,
                            const int64_t* g_blk_off, int64_t n_groups, const int32_t* omega_off, const int32_t* omega,
                            const int32_t* gamma_off, const int32_t* gamma, const int64_t* sm_off, const double* sm_data,
                            int32_t* lane_ids, double* lane_blk) {
  const int lane = threadIdx.x & 31;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); g < n_groups;
       g += int64_t(gridDim.x) * (blockDim.x >> 5)) {
    const int a = g_agg[g * 32 + lane];
    const int nw = g_nw[g], ng = g_ng[g];
    const int m = nw + ng;
    const int64_t nblk = int64_t(nw) * (nw + 1) / 2 + int64_t(nw) * ng;
    int32_t* ids = lane_ids + g_ids_off[g];
    double* blk = lane_blk + g_blk_off[g];
    for (int e = 0; e < m; ++e) {
      int id = -1;
      if (a >= 0) id = e < nw ? omega[omega_off[a] + e] : gamma[gamma_off[a] + e - nw];
      ids[e * 32 + lane] = id;
    }
    for (int64_t k = 0; k < nblk; ++k) blk[k * 32 + lane] = a >= 0 ? sm_data[sm_off[a] + k] : 0.0;
  }
}

void build_lane_layout(const DevTopo& topo, const std::vector<int32_t>& hoo, const std::vector<int32_t>& hgo,
                       const std::vector<int64_t>& colors, int64_t n_colors, DevSmoother& sm, cudaStream_t s,
                       const std::vector<int32_t>* h_gamma) {
  const int64_t na = topo.n_agg;
  // groups: (colour, nω, nΓ) keys in colour order, aggregates ascending inside a key
  std::vector<int64_t> order(na);
  std::iota(order.begin(), order.end(), 0);
  auto key = [&](int64_t a) {
    return std::make_tuple(colors[a], hoo[a + 1] - hoo[a], hgo[a + 1] - hgo[a]);
  };
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return key(x) < key(y); });
  std::vector<int32_t> g_agg, g_nw, g_ng, g_cnt;
  std::vector<int64_t> g_ids_off{0}, g_blk_off{0};
  sm.color_goff.assign(n_colors + 1, 0);
  size_t i = 0;
  while (i < order.size()) {
    const auto k = key(order[i]);
    size_t j = i;
    while (j < order.size() && j - i < 32 && key(order[j]) == k) ++j;
    const int nw = std::get<1>(k), ng = std::get<2>(k);
    for (size_t t = i; t < i + 32; ++t) g_agg.push_back(t < j ? static_cast<int32_t>(order[t]) : -1);
    g_nw.push_back(nw);
    g_ng.push_back(ng);
    g_cnt.push_back(static_cast<int32_t>(j - i));
    g_ids_off.push_back(g_ids_off.back() + int64_t(nw + ng) * 32);
    g_blk_off.push_back(g_blk_off.back() + (int64_t(nw) * (nw + 1) / 2 + int64_t(nw) * ng) * 32);
    ++sm.color_goff[std::get<0>(k) + 1];
    i = j;
  }
  for (int64_t c = 0; c < n_colors; ++c) sm.color_goff[c + 1] += sm.color_goff[c];
  sm.n_groups = static_cast<int64_t>(g_nw.size());
  {
    std::vector<int32_t> ri, ti;
    sm.lane_rast_color_off.assign(n_colors + 1, 0);
    for (int64_t g = 0; g < sm.n_groups; ++g)
      for (int r = 0; r < g_nw[g]; ++r) ri.push_back(static_cast<int32_t>((g << 8) | r));
    for (int64_t c = 0; c < n_colors; ++c) {
      for (int64_t g = sm.color_goff[c]; g < sm.color_goff[c + 1]; ++g)
        for (int r = 0; r < g_nw[g] + g_ng[g]; ++r) ti.push_back(static_cast<int32_t>((g << 8) | r));
      sm.lane_rast_color_off[c + 1] = static_cast<int64_t>(ti.size());
    }
    sm.lane_ras_items.upload(ri, s);
    sm.lane_rast_items.upload(ti, s);
  }
  {  // inputs of the persistent TMA-pipelined sweep
    std::vector<int32_t> gc(sm.n_groups), cg(n_colors + 1, 0);
    int64_t blk_b = 0, ids_b = 0;
    for (int64_t c = 0; c < n_colors; ++c) {
      cg[c] = static_cast<int32_t>(sm.color_goff[c + 1] - sm.color_goff[c]);
      for (int64_t g = sm.color_goff[c]; g < sm.color_goff[c + 1]; ++g) gc[g] = static_cast<int32_t>(c);
    }
    for (int64_t g = 0; g < sm.n_groups; ++g) {
      blk_b = std::max<int64_t>(blk_b, (g_blk_off[g + 1] - g_blk_off[g]) * 8);
      ids_b = std::max<int64_t>(ids_b, (g_ids_off[g + 1] - g_ids_off[g]) * 4);
    }
    sm.g_color.upload(gc, s);
    sm.color_groups.upload(cg, s);
    sm.n_colors = n_colors;
    sm.stage_blk_bytes = blk_b;
    sm.stage_ids_bytes = ids_b;
    sm.n_slots = 0;
    if (h_gamma) {
      // per-node slots of the Γ contributions: node-major, holders in ascending aggregate order
      const int64_t n = topo.n_nodes;
      std::vector<int32_t> noff(n + 1, 0);
      for (int32_t v : *h_gamma) ++noff[v + 1];
      for (int64_t v = 0; v < n; ++v) noff[v + 1] += noff[v];
      std::vector<int32_t> cur(noff.begin(), noff.end() - 1);
      std::vector<int32_t> slot_of(h_gamma->size());  // per Γ entry, in (aggregate ascending, position) order
      for (int64_t a = 0; a < na; ++a)
        for (int32_t p = hgo[a]; p < hgo[a + 1]; ++p) slot_of[p] = cur[(*h_gamma)[p]]++;
      std::vector<int64_t> soff(sm.n_groups + 1, 0);
      int64_t slot_b = 0;
      for (int64_t g = 0; g < sm.n_groups; ++g) {
        soff[g + 1] = soff[g] + int64_t(g_ng[g]) * 32;
        slot_b = std::max<int64_t>(slot_b, int64_t(g_ng[g]) * 32 * 4);
      }
      std::vector<int32_t> ls(std::max<int64_t>(soff.back(), 1), -1);
      for (int64_t g = 0; g < sm.n_groups; ++g)
        for (int l = 0; l < 32; ++l) {
          const int32_t a = g_agg[g * 32 + l];
          if (a < 0) continue;
          for (int j = 0; j < g_ng[g]; ++j) ls[soff[g] + int64_t(j) * 32 + l] = slot_of[hgo[a] + j];
        }
      sm.g_slot_off.upload(soff, s);
      sm.lane_slots.upload(ls, s);
      sm.node_slot_off.upload(noff, s);
      sm.n_slots = static_cast<int64_t>(h_gamma->size());
      sm.stage_slot_bytes = slot_b;
    }
  }
  DBuf<int32_t> d_agg;
  d_agg.upload(g_agg, s);
  sm.g_nw.upload(g_nw, s);
  sm.g_ng.upload(g_ng, s);
  sm.g_cnt.upload(g_cnt, s);
  sm.g_ids_off.upload(g_ids_off, s);
  sm.g_blk_off.upload(g_blk_off, s);
  sm.lane_ids.alloc(std::max<int64_t>(g_ids_off.back(), 1), s);
  sm.lane_blk.alloc(std::max<int64_t>(g_blk_off.back(), 1), s);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(sm.n_groups, 8), sm_count() * 8)));
  k_lane_pack<<<grid, 256, 0, s>>>(d_agg.get(), sm.g_nw.get(), sm.g_ng.get(), sm.g_ids_off.get(), sm.g_blk_off.get(),
                                   sm.n_groups, topo.omega_off.get(), topo.omega.get(), topo.gamma_off.get(),
                                   topo.gamma.get(), sm.off.get(), sm.data.get(), sm.lane_ids.get(), sm.lane_blk.get());
  LSB_LAUNCH();
}

// ---- row layout of large Schwarz blocks -------------------------------------------

__global__ void k_expand_rows(const int32_t* omega_off, const int32_t* gamma_off, const int64_t* sm_off,
                              const double* sm_data, const int64_t* row_off, double* row_data, int64_t n_agg) {
  for (int64_t a = blockIdx.x; a < n_agg; a += gridDim.x) {
    const int nw = omega_off[a + 1] - omega_off[a], ng = gamma_off[a + 1] - gamma_off[a];
    const int m = nw + ng;
    const double* pk = sm_data + sm_off[a];
    const double* pg = pk + int64_t(nw) * (nw + 1) / 2;
    double* F = row_data + row_off[a];
    double* Gt = F + int64_t(nw) * m;
    for (int64_t e = threadIdx.x; e < int64_t(nw) * m; e += blockDim.x) {
      const int i = static_cast<int>(e / m), j = static_cast<int>(e % m);
      double v;
      if (j < nw) {
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        v = pk[int64_t(lo) * nw - (int64_t(lo) * (lo - 1)) / 2 + (hi - lo)];
      } else {
        v = pg[int64_t(i) * ng + (j - nw)];
      }
      F[e] = v;
    }
    for (int64_t e = threadIdx.x; e < int64_t(ng) * nw; e += blockDim.x) {
      const int g = static_cast<int>(e / nw), i = static_cast<int>(e % nw);
      Gt[e] = pg[int64_t(i) * ng + g];
    }
  }
}

void build_row_layout(const DevTopo& topo, const std::vector<int32_t>& hoo, const std::vector<int32_t>& hgo,
                      const std::vector<int32_t>& byc, DevSmoother& sm, cudaStream_t s) {
  const int64_t na = topo.n_agg;
  std::vector<int64_t> roff(na + 1, 0);
  std::vector<int32_t> ra, rr, ta, tr;
  // short rows (nΩ <= 128): a RAS item is a chunk of kRowsCh ω rows sharing
  // one gather of the Ω ids and r values (k_schwarz_rows_ch)
  sm.ras_ch = sm.max_sub <= 128 ? kRowsCh : 1;
  for (int64_t i = 0; i < na; ++i) {
    const int64_t nw = hoo[i + 1] - hoo[i], ng = hgo[i + 1] - hgo[i];
    roff[i + 1] = roff[i] + nw * (nw + ng) + ng * nw;
    for (int64_t r = 0; r < nw; r += sm.ras_ch) {
      ra.push_back(static_cast<int32_t>(i));
      rr.push_back(static_cast<int32_t>(r));
    }
  }
  sm.rast_color_off.assign(sm.color_off.size(), 0);
  // 64 < nω <= 128: a RAS-T item is a chunk of kRowsCh Ω rows sharing one
  // gather of the ω ids and r values (k_schwarz_rows_tch); shorter ω sets
  // take the sub-warp rows of k_schwarz_rows_t instead
  sm.rast_ch = sm.max_omega > 64 && sm.max_omega <= 128 ? kRowsCh : 1;
  for (size_t c = 0; c + 1 < sm.color_off.size(); ++c) {
    for (int64_t k = sm.color_off[c]; k < sm.color_off[c + 1]; ++k) {
      const int32_t a = byc[k];
      const int64_t m = (hoo[a + 1] - hoo[a]) + (hgo[a + 1] - hgo[a]);
      for (int64_t r = 0; r < m; r += sm.rast_ch) {
        ta.push_back(a);
        tr.push_back(static_cast<int32_t>(r));
      }
    }
    sm.rast_color_off[c + 1] = static_cast<int64_t>(ta.size());
  }
  sm.row_off.upload(roff, s);
  sm.row_data.alloc(std::max<int64_t>(roff[na], 1), s);
  sm.ras_agg.upload(ra, s);
  sm.ras_row.upload(rr, s);
  sm.rast_agg.upload(ta, s);
  sm.rast_row.upload(tr, s);
  k_expand_rows<<<static_cast<int>(std::min<int64_t>(std::max<int64_t>(na, 1), sm_count() * 8)), 256, 0, s>>>(
      topo.omega_off.get(), topo.gamma_off.get(), sm.off.get(), sm.data.get(), sm.row_off.get(), sm.row_data.get(),
      na);
  LSB_LAUNCH();
}

// ---- coarse factor -------------------------------------------------------------

__global__ void k_coarse_dense(const int64_t* off, const int32_t* col, const double* val, int64_t n, double* d) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    for (int64_t k = off[i]; k < off[i + 1]; ++k) d[i * n + col[k]] = val[k];
}

__global__ void k_coarse_factor(double* blk, const double* orig, int m, double* X, double* inv, int32_t* status,
                                double* slot) {
  BlockTeam t;
  if (!t_factor_spd(t, blk, orig, m, slot)) {
    if (t.rank() == 0) *status = 1;
    return;
  }
  for (int j = t.rank(); j < m; j += t.size()) chol_solve_unit(blk, m, j, X + int64_t(j) * m);
  t.sync();
  for (int64_t e = t.rank(); e < int64_t(m) * m; e += t.size()) {
    const int i = static_cast<int>(e / m), j = static_cast<int>(e % m);
    inv[e] = X[int64_t(j) * m + i];
  }
}

// ---- P assembly ------------------------------------------------------------------

__global__ void k_p_count(const int32_t* node_agg, const int32_t* node_pos, const int32_t* kc, const int64_t* poff,
                          const double* panels, int64_t n, int64_t* cnt) {
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
    const int a = node_agg[v], r = node_pos[v], k = kc[a];
    const double* row = panels + poff[a] + int64_t(r) * k;
    int64_t c = 0;
    for (int j = 0; j < k; ++j) c += row[j] != 0.0 ? 1 : 0;
    cnt[v + 1] = c;
  }
}

__global__ void k_p_fill(const int32_t* node_agg, const int32_t* node_pos, const int32_t* kc, const int64_t* poff,
                         const double* panels, const int32_t* coff, const int64_t* off, int64_t n, int32_t* pcol,
                         double* pval) {
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
    const int a = node_agg[v], r = node_pos[v], k = kc[a];
    const double* row = panels + poff[a] + int64_t(r) * k;
    int64_t o = off[v];
    for (int j = 0; j < k; ++j)
      if (row[j] != 0.0) {
        pcol[o] = coff[a] + j;
        pval[o] = row[j];
        ++o;
      }
  }
}

__global__ void k_compact_panels(const int32_t* list, int n_list, const int32_t* omega_off, const int32_t* kc,
                                 const int64_t* src_off, const double* src, const int64_t* dst_off, double* dst) {
  for (int idx = blockIdx.x; idx < n_list; idx += gridDim.x) {
    const int a = list[idx];
    const int64_t cnt = int64_t(omega_off[a + 1] - omega_off[a]) * kc[a];
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) dst[dst_off[a] + e] = src[src_off[idx] + e];
  }
}

// workspace class of a problem: 0 warp+smem, 1 CTA+smem, 2 CTA+global
inline int ws_class(int64_t w) { return w <= 3072 ? 0 : (w <= 26000 ? 1 : 2); }

// Launch a batched per-aggregate stage in three workspace classes.
template <class Args, class WarpK, class BlockSmemK, class BlockGlobK>
void launch_classes(Args args, const std::vector<int32_t>& aggs, const std::vector<int64_t>& ws_need,
                    WarpK warpk, BlockSmemK bsk, BlockGlobK bgk, std::vector<int32_t>& list_order, cudaStream_t s,
                    std::vector<std::pair<int, int>>* ranges = nullptr) {
  // classes: 0 warp+smem (ws <= 3072 doubles), 1 CTA+smem (<= 26000), 2 CTA+global
  std::vector<int32_t> cls[3];
  for (int32_t a : aggs) cls[ws_class(ws_need[a])].push_back(a);
  list_order.clear();
  for (int c = 0; c < 3; ++c) list_order.insert(list_order.end(), cls[c].begin(), cls[c].end());
  DBuf<int32_t> dlist;
  dlist.upload(list_order, s);
  int64_t base = 0;
  for (int c = 0; c < 3; ++c) {
    const int cnt = static_cast<int>(cls[c].size());
    if (cnt == 0) continue;
    int64_t wmax = 0;
    for (int32_t a : cls[c]) wmax = std::max(wmax, ws_need[a]);
    wmax = r2(wmax);
    Args g = args;
    g.list = dlist.get() + base;
    g.list_base = static_cast<int>(base);
    g.n_list = cnt;
    g.ws_stride = wmax;
    if (c == 0) {
      constexpr int WPB = 4;
      const size_t smem = size_t(WPB) * wmax * 8;
      LSB_CUDA(cudaFuncSetAttribute(warpk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      const int grid = static_cast<int>(std::min<int64_t>(ceil_div(cnt, WPB), int64_t(sm_count()) * 8));
      warpk<<<grid, WPB * 32, smem, s>>>(g);
      LSB_LAUNCH();
    } else if (c == 1) {
      const size_t smem = size_t(wmax) * 8;
      LSB_CUDA(cudaFuncSetAttribute(bsk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      const int grid = static_cast<int>(std::min<int64_t>(cnt, int64_t(sm_count()) * 4));
      bsk<<<grid, 128, smem, s>>>(g);
      LSB_LAUNCH();
    } else {
      // global workspace slots; bound the footprint to ~2 GiB
      const int64_t slots = std::max<int64_t>(1, std::min<int64_t>({int64_t(cnt), int64_t(sm_count()) * 2,
                                                                    (int64_t(1) << 28) / std::max<int64_t>(wmax, 1)}));
      DBuf<double> gws(slots * wmax, s);
      g.gws = gws.get();
      const size_t fsm = size_t(kFastCap) * 8;
      LSB_CUDA(cudaFuncSetAttribute(bgk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fsm)));
      bgk<<<static_cast<int>(slots), 512, fsm, s>>>(g);
      LSB_LAUNCH();
    }
    if (ranges) ranges->push_back({static_cast<int>(base), cnt});
    base += cnt;
  }
}

__global__ void k_dense_eig_warp(int n, const double* a, double* vals, double* vecs, double* ws, int32_t* status) {
  WarpTeam t;
  if (threadIdx.x >= 32) return;
  Arena ar{ws, 0};
  const int st = t_sym_eig(t, n, a, vals, vecs, ar);
  if (t.rank() == 0) *status = st;
}

__global__ void __launch_bounds__(512) k_dense_eig_block(int n, const double* a, double* vals, double* vecs, double* ws, int32_t* status,
                                  int use_fast, int sched) {
  BlockTeam t;
  Arena ar{ws, 0, use_fast ? dyn_smem : nullptr, use_fast ? kFastCap : 0};
  ar.sched = sched;
  const int st = t_sym_eig(t, n, a, vals, vecs, ar);
  if (t.rank() == 0) *status = st;
}

// one cluster: CTA 0 runs the wavefront Jacobi, the other CTAs replay its rotation log
__global__ void __launch_bounds__(512, 1) k_dense_eig_wave(int n, const double* a, double* vals, double* vecs, double* ws,
                                                        WaveCtl* ctl, int32_t* status) {
  if (cooperative_groups::this_cluster().block_rank() != 0) {
    wave_helper_main(ctl, dyn_smem);
    return;
  }
  const int st = wave_sym_eig_leader(n, a, vals, vecs, ctl, ws, dyn_smem);
  if (threadIdx.x == 0) *status = st;
  wave_quit(ctl);
}

}  // namespace

// Test hook: one eigensolve on a chosen device path. 0: warp team, 1: CTA
// team, 2: CTA producer/consumer pipeline, 3: CTA pipeline with one barrier
// per rotation, 4: cluster wavefront (jacobi_wave.cuh).
int dense_sym_eig(int64_t n, const double* h_a, double* h_vals, double* h_vecs, int path, cudaStream_t s) {
  if (path == 4 && (n < 2 || n > kWaveMaxN)) raise(LSAMGDD_ERR_INPUT, "dense_sym_eig: wavefront path needs 2 <= n <= 608");
  DBuf<double> a(n * n, s), vals(std::max<int64_t>(n, 1), s), vecs(std::max<int64_t>(n * n, 1), s),
      ws((path == 4 ? wave_ws_doubles(n) : sym_eig_scratch(n)) + 64, s);
  DBuf<int32_t> st(1, s);
  st.zero(s);
  a.upload(h_a, n * n, s);
  if (path == 0) {
    k_dense_eig_warp<<<1, 32, 0, s>>>(static_cast<int>(n), a.get(), vals.get(), vecs.get(), ws.get(), st.get());
  } else if (path == 4) {
    DBuf<WaveCtl> ctl(1, s);
    ctl.zero(s);
    DBuf<long long> prof(16, s);
    prof.zero(s);
    const bool want_prof = LSB_DIAG_ENV("LSB_WAVE_PROF");  // diagnostic: phase cycle counters of this test hook
    if (want_prof) {
      long long* pp = prof.get();
      LSB_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(ctl.get()) + offsetof(WaveCtl, prof), &pp, sizeof(pp),
                               cudaMemcpyHostToDevice, s));
    }
    const size_t smem = size_t(wave_smem_doubles(n)) * 8;
    LSB_CUDA(cudaFuncSetAttribute(k_dense_eig_wave, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kWaveCluster);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kWaveCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    LSB_CUDA(cudaLaunchKernelEx(&cfg, k_dense_eig_wave, static_cast<int>(n), static_cast<const double*>(a.get()),
                                vals.get(), vecs.get(), ws.get(), ctl.get(), st.get()));
    LSB_LAUNCH();
    const int status = read_scalar(st.get(), s);
    if (want_prof) {
      const auto hp = prof.download(s);
      fprintf(stderr, "wave prof n=%lld (Mcycles): warps: wait %.1f first %.1f pivots %.1f second %.1f finalise %.1f | "
              "diag-load %.1f diag-writeback %.1f steps %lld | leader: init %.1f sum %.1f wavefront %.1f helper-wait %.1f copyback %.1f | sweeps %lld rotations %lld\n", (long long)n,
              hp[0] / 1e6, hp[1] / 1e6, hp[2] / 1e6, hp[3] / 1e6, hp[4] / 1e6, hp[12] / 1e6, hp[13] / 1e6, hp[14], hp[10] / 1e6, hp[5] / 1e6, hp[11] / 1e6, hp[6] / 1e6,
              hp[7] / 1e6, hp[8], hp[9]);
    }
    const auto hv = vals.download(s);
    const auto hV = vecs.download(s);
    std::copy(hv.begin(), hv.begin() + n, h_vals);
    std::copy(hV.begin(), hV.begin() + n * n, h_vecs);
    return status;
  } else {
    const size_t fsm = path >= 2 ? size_t(kFastCap) * 8 : 0;
    LSB_CUDA(cudaFuncSetAttribute(k_dense_eig_block, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kFastCap * 8)));
    k_dense_eig_block<<<1, 512, fsm, s>>>(static_cast<int>(n), a.get(), vals.get(), vecs.get(), ws.get(), st.get(),
                                          path >= 2 ? 1 : 0, path == 3 ? 1 : 0);
  }
  LSB_LAUNCH();
  const int status = read_scalar(st.get(), s);
  const auto hv = vals.download(s);
  const auto hV = vecs.download(s);
  std::copy(hv.begin(), hv.begin() + n, h_vals);
  std::copy(hV.begin(), hV.begin() + n * n, h_vecs);
  return status;
}

void row_sets(const DevCsr& g, const DevTopo& topo, DevRowSets& rs, cudaStream_t s) {
  const int64_t m = g.nr, nnz = g.nnz;
  rs.mult.alloc(m, s);
  rs.mult.zero(s);
  rs.nz_off.alloc(topo.n_agg + 1, s);
  DBuf<int64_t> cnt(topo.n_agg + 1, s);
  cnt.zero(s);
  int64_t uniq = 0;
  if (nnz > 0) {
    DBuf<uint64_t> k1(nnz, s), k2(nnz, s);
    k_owner_keys<<<grid_for(m), kThreads, 0, s>>>(g.off.get(), g.col.get(), m, topo.node_agg.get(), k1.get());
    LSB_LAUNCH();
    size_t tmp = 0;
    const int eb = bits_for(static_cast<uint64_t>(topo.n_agg) * static_cast<uint64_t>(m));
    LSB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k1.get(), k2.get(), nnz, 0, eb, s));
    {
      DBuf<unsigned char> tb(tmp, s);
      LSB_CUDA(cub::DeviceRadixSort::SortKeys(tb.get(), tmp, k1.get(), k2.get(), nnz, 0, eb, s));
    }
    k1.release();
    DBuf<int64_t> flag(nnz, s), pos(nnz, s);
    k_rowset_fill<<<grid_for(nnz), kThreads, 0, s>>>(k2.get(), nnz, m, nullptr, nullptr, nullptr, flag.get());
    LSB_LAUNCH();
    tmp = 0;
    LSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag.get(), pos.get(), nnz, s));
    {
      DBuf<unsigned char> tb(tmp, s);
      LSB_CUDA(cub::DeviceScan::ExclusiveSum(tb.get(), tmp, flag.get(), pos.get(), nnz, s));
    }
    uniq = read_scalar(pos.get() + nnz - 1, s) + read_scalar(flag.get() + nnz - 1, s);
    rs.nz.alloc(uniq, s);
    k_rowset_scatter<<<grid_for(nnz), kThreads, 0, s>>>(k2.get(), flag.get(), pos.get(), nnz, static_cast<uint64_t>(m),
                                                         cnt.get(), rs.mult.get(), rs.nz.get());
    LSB_LAUNCH();
  }
  size_t tmp = 0;
  LSB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt.get(), rs.nz_off.get(), topo.n_agg + 1, s));
  {
    DBuf<unsigned char> tb(tmp, s);
    LSB_CUDA(cub::DeviceScan::InclusiveSum(tb.get(), tmp, cnt.get(), rs.nz_off.get(), topo.n_agg + 1, s));
  }
  DBuf<unsigned long long> st(3, s);
  st.zero(s);
  if (m) k_row_stats<<<grid_for(m), kThreads, 0, s>>>(g.off.get(), rs.mult.get(), m, st.get());
  LSB_LAUNCH();
  const auto h = st.download(s);
  rs.n_mult = static_cast<int64_t>(h[0]);
  rs.empty_rows = static_cast<int64_t>(h[1]);
  rs.max_row_nnz = static_cast<int64_t>(h[2]);
}

namespace {
void build_row_layout(const DevTopo& topo, const std::vector<int32_t>& hoo, const std::vector<int32_t>& hgo,
                      const std::vector<int32_t>& byc, DevSmoother& sm, cudaStream_t s);
}

void build_smoother(const DevCsr& a, const DevTopo& topo, const std::vector<int32_t>& hoo,
                    const std::vector<int32_t>& hgo, const std::vector<int64_t>& colors, int64_t n_colors,
                    DevSmoother& sm, cudaStream_t s, const std::vector<int32_t>* h_gamma) {
  const int64_t na = topo.n_agg;
  sm.n_agg = na;
  std::vector<int64_t> off(na + 1, 0), need(na);
  std::vector<int32_t> aggs(na);
  sm.max_omega = sm.max_sub = 0;
  double b_ras = 0, b_rast = 0;
  for (int64_t i = 0; i < na; ++i) {
    const int64_t nw = hoo[i + 1] - hoo[i], ng = hgo[i + 1] - hgo[i];
    off[i + 1] = off[i] + r2(nw * (nw + 1) / 2 + nw * ng);
    need[i] = sm_ws(nw, ng);
    aggs[i] = static_cast<int32_t>(i);
    sm.max_omega = std::max(sm.max_omega, nw);
    sm.max_sub = std::max(sm.max_sub, nw + ng);
    const double blk = 8.0 * (nw * (nw + 1) / 2 + nw * ng);
    b_ras += blk + 4.0 * (nw + ng);   // block (ω columns of the inverse) + Ω index list
    b_rast += blk + 4.0 * (nw + ng);
  }
  // every vector entry counts once per sweep, however many
  // subdomains gather it — RAS reads r and writes e (16 n), RAS-T reads r and
  // read-modify-writes e (24 n)
  sm.bytes_ras = b_ras + 16.0 * static_cast<double>(topo.n_nodes);
  sm.bytes_rast = b_rast + 24.0 * static_cast<double>(topo.n_nodes);
  sm.off.upload(off, s);
  sm.data.alloc(off[na], s);
  DBuf<int32_t> status(na, s);
  status.zero(s);
  SmArgs g{};
  g.aoff = a.off.get();
  g.acol = a.col.get();
  g.aval = a.val.get();
  g.omega_off = topo.omega_off.get();
  g.omega = topo.omega.get();
  g.gamma_off = topo.gamma_off.get();
  g.gamma = topo.gamma.get();
  g.sm_off = sm.off.get();
  g.sm_data = sm.data.get();
  g.status = status.get();
  std::vector<int32_t> order;
  launch_classes(g, aggs, need, k_sm_warp<4>, k_sm_block<true>, k_sm_block<false>, order, s);
  const auto hs = status.download(s);
  for (int64_t i = 0; i < na; ++i)
    if (hs[i]) raise(LSAMGDD_ERR_SETUP, "dense symmetric factorization failed for subdomain block of aggregate " +
                                            std::to_string(i));
  if (sm.max_sub <= kLaneMaxSub && sm.max_omega <= kLaneMaxOmega)
    build_lane_layout(topo, hoo, hgo, colors, n_colors, sm, s, h_gamma);
  // colour-sorted aggregate order for the race-free RAS-T scatter
  std::vector<int32_t> byc(na);
  sm.color_off.assign(n_colors + 1, 0);
  for (int64_t i = 0; i < na; ++i) ++sm.color_off[colors[i] + 1];
  for (int64_t c = 0; c < n_colors; ++c) sm.color_off[c + 1] += sm.color_off[c];
  std::vector<int64_t> cur(sm.color_off.begin(), sm.color_off.end() - 1);
  for (int64_t i = 0; i < na; ++i) byc[cur[colors[i]]++] = static_cast<int32_t>(i);
  sm.order.upload(byc, s);
  const int64_t max_blk = sm.max_omega * (sm.max_omega + 1) / 2 + sm.max_omega * (sm.max_sub - sm.max_omega);
  sm.rows = sm.n_groups == 0 && (max_blk > kRowsMinBlk || sm.max_sub > 512);
  if (sm.rows) build_row_layout(topo, hoo, hgo, byc, sm, s);
  // the sweeps read only the lane or row layout built from the packed blocks
  if (sm.rows || sm.n_groups > 0) sm.data.release();
}

void local_gevp_all(const DevCsr& gm, const DevTopo& topo, const std::vector<int32_t>& hoo,
                    const std::vector<int32_t>& hgo, const DevRowSets& rs, const std::vector<int64_t>& h_nz_off,
                    const GevpParams& gp, DevInterp& ip, DevCsr& p, bool keep_spectra, cudaStream_t s) {
  (void)h_nz_off;
  const bool tprof = LSB_DIAG_ENV("LSB_STAGE_PROF");  // diagnostics: synchronised wall-clock marks
  const auto tp0 = std::chrono::steady_clock::now();
  auto tmark = [&](const char* what) {
    if (!tprof) return;
    cudaStreamSynchronize(s);
    fprintf(stderr, "  local_gevp level %d: %-28s %8.1f ms\n", gp.level, what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count());
  };
  const int64_t na = topo.n_agg;
  const int64_t maxrow = std::max<int64_t>(rs.max_row_nnz, 1);
  std::vector<int64_t> need(na), spec_off(na + 1, 0);
  for (int64_t i = 0; i < na; ++i) {
    const int64_t nw = hoo[i + 1] - hoo[i], ng = hgo[i + 1] - hgo[i];
    need[i] = gevp_ws(nw, ng, maxrow);
    spec_off[i + 1] = spec_off[i] + nw;
  }
  DBuf<int64_t> d_spec_off;
  d_spec_off.upload(spec_off, s);
  DBuf<double> spec(spec_off[na], s);
  DBuf<int32_t> kcols(na, s), nspec(na, s), status(na, s);
  status.zero(s);
  nspec.zero(s);
  {
    const int chk = LSB_DIAG_ENV("LSB_GRAM_CHECK") ? 1 : 0;
    unsigned long long z[8] = {0};
    LSB_CUDA(cudaMemcpyToSymbolAsync(g_gram_check, &chk, sizeof(chk), 0, cudaMemcpyHostToDevice, s));
    LSB_CUDA(cudaMemcpyToSymbolAsync(g_gram_bad, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
  }
  const bool prof_on = LSB_DIAG_ENV("LSB_GEVP_PROF");
  DBuf<long long> eprof(prof_on ? 8 : 1, s);
  if (prof_on) {
    eprof.zero(s);
    long long* ep = eprof.get();
    LSB_CUDA(cudaMemcpyToSymbol(g_eig_prof, &ep, sizeof(ep)));
  }
  DBuf<long long> gprof(prof_on ? na * 6 : 1, s);
  if (prof_on) {
    gprof.zero(s);
    long long* gp_ptr = gprof.get();
    LSB_CUDA(cudaMemcpyToSymbol(g_gevp_prof, &gp_ptr, sizeof(gp_ptr)));
  }
  // Grams of large subdomains: multi-CTA tiles (grams.cu) instead of one team
  DBuf<double> pre;
  DBuf<int64_t> pre_off;
  {
    std::vector<int32_t> big;
    std::vector<int64_t> hpo(na, -1);
    int64_t tot = 0;
    for (int64_t i = 0; i < na; ++i) {
      const int64_t nw = hoo[i + 1] - hoo[i], ng = hgo[i + 1] - hgo[i];
      if (nw + ng >= kTileMinSub && nw + ng <= kTileMaxSub) {
        big.push_back(static_cast<int32_t>(i));
        hpo[i] = tot;
        tot += pre_gram_doubles(nw, ng);
      }
    }
    if (!big.empty()) {
      const auto h_nzo = rs.nz_off.download(s);
      pre.alloc(tot, s);
      pre_off.upload(hpo, s);
      tiled_grams(gm, topo, hoo, hgo, rs, h_nzo, big, gp.variant == 1 ? 1 : 0, pre.get(), pre_off.get(), s);
    }
  }
  tmark("tiled grams done");
  // chunk aggregates (id order) so the nω² panel scratch stays bounded
  const int64_t budget = int64_t(1) << 27;  // doubles (1 GiB)
  std::vector<int32_t> h_k(na, 0);
  ip.panel_off.alloc(na + 1, s);
  std::vector<int64_t> final_off(na + 1, 0);
  struct Chunk {
    std::vector<int32_t> order;
    std::vector<int64_t> tmp_off;
  };
  DBuf<double> final_panels;
  std::vector<std::pair<int64_t, int64_t>> chunks;
  {
    int64_t a0 = 0;
    while (a0 < na) {
      int64_t tot = 0, a1 = a0;
      while (a1 < na) {
        const int64_t nw = hoo[a1 + 1] - hoo[a1];
        if (a1 > a0 && tot + nw * nw > budget) break;
        tot += nw * nw;
        ++a1;
      }
      chunks.push_back({a0, a1});
      a0 = a1;
    }
  }
  struct Fork {
    cudaStream_t s = nullptr;
    cudaEvent_t e = nullptr;
    ~Fork() {
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
      if (e) cudaEventDestroy(e);
    }
  } fork;
  constexpr int kSideSms = 4;  // SMs a cluster launch leaves to the side stream's small problems
  // first pass: run all chunks, keep each chunk's panels on the device
  std::vector<DBuf<double>> chunk_panels(chunks.size());
  std::vector<DBuf<int64_t>> chunk_off(chunks.size());
  std::vector<DBuf<int32_t>> chunk_list(chunks.size());
  for (size_t ci = 0; ci < chunks.size(); ++ci) {
    const int64_t a0 = chunks[ci].first, a1 = chunks[ci].second;
    // subdomains whose eigenproblems are large enough for the cluster wavefront Jacobi
    auto wave_class = [&](int64_t a) {
      const int64_t nw = hoo[a + 1] - hoo[a], ng = hgo[a + 1] - hgo[a], mx = std::max(nw, ng);
      return mx >= kWaveClassMin && mx <= kWaveMaxN;
    };
    // mid-size subdomains: warp teams with global workspaces
    auto mid_class = [&](int64_t a) {
      const int64_t nw = hoo[a + 1] - hoo[a], ng = hgo[a + 1] - hgo[a], mx = std::max(nw, ng);
      return ws_class(need[a]) >= 1 && mx <= kWarpGlobMax && !wave_class(a);
    };
    std::vector<int32_t> aggs, big, mid;
    for (int64_t a = a0; a < a1; ++a)
      (wave_class(a) ? big : mid_class(a) ? mid : aggs).push_back(static_cast<int32_t>(a));
    // classes decide the list order; panel scratch offsets follow that order
    std::vector<int32_t> order;
    {
      std::vector<int32_t> cls[3];
      for (int32_t a : aggs) cls[ws_class(need[a])].push_back(a);
      for (int c = 0; c < 3; ++c) order.insert(order.end(), cls[c].begin(), cls[c].end());
      std::stable_sort(mid.begin(), mid.end(), [&](int32_t x, int32_t y) { return need[x] > need[y]; });
      order.insert(order.end(), mid.begin(), mid.end());
      // largest first: the longest problems start first (the > 256 class launches before the <= 256 class)
      std::stable_sort(big.begin(), big.end(), [&](int32_t x, int32_t y) { return need[x] > need[y]; });
      auto big_mx = [&](int32_t a) { return std::max(hoo[a + 1] - hoo[a], hgo[a + 1] - hgo[a]); };
      for (int32_t a : big)
        if (big_mx(a) > kWaveSmallMax) order.push_back(a);
      for (int32_t a : big)
        if (big_mx(a) <= kWaveSmallMax) order.push_back(a);
    }
    std::vector<int64_t> toff(order.size() + 1, 0);
    for (size_t k = 0; k < order.size(); ++k) {
      const int64_t nw = hoo[order[k] + 1] - hoo[order[k]];
      toff[k + 1] = toff[k] + r2(nw * nw);
    }
    chunk_panels[ci].alloc(toff.back(), s);
    chunk_off[ci].upload(toff, s);
    GevpArgs g{};
    g.goff = gm.off.get();
    g.gcol = gm.col.get();
    g.gval = gm.val.get();
    g.mult = rs.mult.get();
    g.omega_off = topo.omega_off.get();
    g.omega = topo.omega.get();
    g.gamma_off = topo.gamma_off.get();
    g.gamma = topo.gamma.get();
    g.nz_off = rs.nz_off.get();
    g.nz = rs.nz.get();
    g.maxrow = static_cast<int>(maxrow);
    g.p = gp;
    g.panel_tmp = chunk_panels[ci].get();
    g.panel_off = chunk_off[ci].get();
    g.spec = spec.get();
    g.spec_off = d_spec_off.get();
    g.kcols = kcols.get();
    g.nspec = nspec.get();
    g.status = status.get();
    g.pre = pre.get();
    g.pre_off = pre.get() ? pre_off.get() : nullptr;
    std::vector<int32_t> lo;
    // A few small subdomains beside a cluster class: they run on a side stream (launched first, on
    // SMs the cluster launch leaves free) instead of holding the cluster kernels back.
    const bool side = !big.empty() && (!aggs.empty() || !mid.empty());
    cudaStream_t fs = s;
    if (side) {
      if (!fork.s) LSB_CUDA(cudaStreamCreateWithFlags(&fork.s, cudaStreamNonBlocking));
      if (!fork.e) LSB_CUDA(cudaEventCreateWithFlags(&fork.e, cudaEventDisableTiming));
      LSB_CUDA(cudaEventRecord(fork.e, s));  // the chunk's buffers and uploads are ordered on s
      LSB_CUDA(cudaStreamWaitEvent(fork.s, fork.e, 0));
      fs = fork.s;
    }
    if (!aggs.empty()) launch_classes(g, aggs, need, k_gevp_warp<4>, k_gevp_block<true>, k_gevp_block<false>, lo, fs);
    DBuf<int32_t> mid_list;
    DBuf<double> mid_ws;
    if (!mid.empty()) {
      constexpr int WPB = 4;
      const int base = static_cast<int>(lo.size());
      const int cnt = static_cast<int>(mid.size());
      int64_t wmax = 0;
      for (int32_t a : mid) wmax = std::max(wmax, need[a]);
      wmax = r2(wmax);
      // 16 warps (problems) per SM; bound the footprint to ~2 GiB
      const int64_t slots = std::max<int64_t>(WPB, std::min<int64_t>({int64_t(ceil_div(cnt, WPB)) * WPB, int64_t(sm_count()) * 16,
                                                                      ((int64_t(1) << 28) / std::max<int64_t>(wmax, 1)) / WPB * WPB}));
      mid_list.upload(mid, fs);
      mid_ws.alloc(slots * wmax, fs);
      GevpArgs gm2 = g;
      gm2.list = mid_list.get();
      gm2.list_base = base;
      gm2.n_list = cnt;
      gm2.ws_stride = wmax;
      gm2.gws = mid_ws.get();
      k_gevp_warp_g<WPB><<<static_cast<int>(slots / WPB), WPB * 32, 0, fs>>>(gm2);
      LSB_LAUNCH();
      lo.insert(lo.end(), mid.begin(), mid.end());
    }
    // cluster classes: subdomains up to 256 run on 2-CTA clusters (16 replay warps cover
    // their 2·NB row groups), larger ones on 4-CTA clusters
    std::vector<DBuf<int32_t>> big_lists;
    std::vector<DBuf<double>> big_ws;
    std::vector<DBuf<WaveCtl>> big_ctl;
    for (int pass = 0; pass < 2 && !big.empty(); ++pass) {
      const int C = pass == 0 ? 4 : 2;
      std::vector<int32_t> part;
      for (int32_t a : big) {
        const int64_t mx = std::max(hoo[a + 1] - hoo[a], hgo[a + 1] - hgo[a]);
        if ((mx > kWaveSmallMax) == (pass == 0)) part.push_back(a);
      }
      if (part.empty()) continue;
      const int base = static_cast<int>(lo.size());
      const int cnt = static_cast<int>(part.size());
      int64_t wmax = 0, nmax = 0;
      for (int32_t a : part) {
        wmax = std::max(wmax, need[a]);
        nmax = std::max<int64_t>(nmax, std::max(hoo[a + 1] - hoo[a], hgo[a + 1] - hgo[a]));
      }
      wmax = r2(wmax);
      const int64_t wws = r2(wave_ws_doubles(nmax));
      // one cluster per slot; bound the footprint to ~2 GiB
      int64_t slots = std::max<int64_t>(1, std::min<int64_t>({int64_t(cnt), int64_t(sm_count()) / C,
                                                                    (int64_t(1) << 28) / std::max<int64_t>(wmax + wws, 1)}));
      if (side) slots = std::max<int64_t>(1, std::min<int64_t>(slots, (int64_t(sm_count()) - kSideSms) / C));
      big_lists.emplace_back();
      big_lists.back().upload(part, s);
      big_ws.emplace_back(slots * wmax, s);
      double* gws = big_ws.back().get();
      big_ws.emplace_back(slots * wws, s);
      double* wbuf = big_ws.back().get();
      big_ctl.emplace_back(slots, s);
      big_ctl.back().zero(s);
      GevpArgs gb = g;
      gb.list = big_lists.back().get();
      gb.list_base = base;
      gb.n_list = cnt;
      gb.ws_stride = wmax;
      gb.gws = gws;
      const size_t smem = size_t(kWaveSmemCap) * 8;
      LSB_CUDA(cudaFuncSetAttribute(k_gevp_wave, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(slots * C));
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      LSB_CUDA(cudaLaunchKernelEx(&cfg, k_gevp_wave, gb, big_ctl.back().get(), wbuf, wws, static_cast<int>(kWaveMinN)));
      LSB_LAUNCH();
      lo.insert(lo.end(), part.begin(), part.end());
      if (LSB_DIAG_ENV("LSB_WAVE_SLOTS")) {  // diagnostics: per-cluster activity window
        const auto hc = big_ctl.back().download(s);
        long long t0 = LLONG_MAX, t1 = 0;
        for (const auto& c : hc)
          if (c.n_done) {
            t0 = std::min(t0, c.t_start);
            t1 = std::max(t1, c.t_end);
          }
        fprintf(stderr, "wave class C=%d level %d: %lld problems, %lld slots, span %.1f ms; per slot (count start end ms):", C,
                gp.level, (long long)cnt, (long long)slots, (t1 - t0) / 1e6);
        for (const auto& c : hc)
          fprintf(stderr, " %d:%.0f-%.0f", c.n_done, c.n_done ? (c.t_start - t0) / 1e6 : -1.0, c.n_done ? (c.t_end - t0) / 1e6 : -1.0);
        fprintf(stderr, "\n");
      }
    }
    if (side) {  // join before the chunk's buffers are released
      LSB_CUDA(cudaEventRecord(fork.e, fork.s));
      LSB_CUDA(cudaStreamWaitEvent(s, fork.e, 0));
    }
    chunk_list[ci].upload(lo, s);
  }
  if (prof_on) {
    const auto hp = gprof.download(s);
    long long mx[6] = {0}, sm[6] = {0};
    for (int64_t i = 0; i < na; ++i)
      for (int k = 0; k < 5; ++k) {
        mx[k] = std::max(mx[k], hp[i * 6 + k]);
        sm[k] += hp[i * 6 + k];
      }
    fprintf(stderr, "gevp prof level %d (%lld aggs) Mcycles max/sum: grams %.1f/%.1f pinv %.1f/%.1f schur %.1f/%.1f "
            "spsd_gevp %.1f/%.1f mgs %.1f/%.1f\n", gp.level, (long long)na, mx[0] / 1e6, sm[0] / 1e6, mx[1] / 1e6,
            sm[1] / 1e6, mx[2] / 1e6, sm[2] / 1e6, mx[3] / 1e6, sm[3] / 1e6, mx[4] / 1e6, sm[4] / 1e6);
    long long* np = nullptr;
    LSB_CUDA(cudaMemcpyToSymbol(g_gevp_prof, &np, sizeof(np)));
    const auto he = eprof.download(s);
    fprintf(stderr, "   large-n Jacobi steps %lld, rotations %lld; wavefront eigensolves %lld, %.1f Mcycles in total\n",
            he[6], he[7], he[5], he[4] / 1e6);
    LSB_CUDA(cudaMemcpyToSymbol(g_eig_prof, &np, sizeof(np)));
  }
  if (LSB_DIAG_ENV("LSB_GRAM_CHECK") && pre.get()) {
    unsigned long long hb[8];
    LSB_CUDA(cudaMemcpyFromSymbolAsync(hb, g_gram_bad, sizeof(hb), 0, cudaMemcpyDeviceToHost, s));
    LSB_CUDA(cudaStreamSynchronize(s));
    double va, vb;
    memcpy(&va, &hb[4], 8);
    memcpy(&vb, &hb[5], 8);
    fprintf(stderr, "gram check level %d: %llu mismatches; first agg %llu mat %llu idx %llu team %.17g tiled %.17g\n",
            gp.level, hb[0], hb[1], hb[2], hb[3], va, vb);
  }
  tmark("eigenproblem kernels done");
  const auto hs = status.download(s);
  for (int64_t i = 0; i < na; ++i) {
    if (hs[i] == 1) raise(LSAMGDD_ERR_EIG, "sym_eig: Jacobi iteration did not converge");
    if (hs[i] == 2) raise(LSAMGDD_ERR_EIG, "sym_eig: non-finite eigenvalue");
    if (hs[i] == 3) raise(LSAMGDD_ERR_EIG, "local_gevp: aggregate " + std::to_string(i) + ": NaN eigenvalue");
  }
  h_k = kcols.download(s);
  ip.h_k = h_k;
  std::vector<int32_t> coff(na + 1, 0);
  for (int64_t i = 0; i < na; ++i) {
    const int64_t nw = hoo[i + 1] - hoo[i];
    final_off[i + 1] = final_off[i] + nw * h_k[i];
    coff[i + 1] = coff[i] + h_k[i];
  }
  ip.n_coarse = coff[na];
  ip.coarse_off.upload(coff, s);
  ip.panel_off.upload(final_off, s);
  ip.panels.alloc(std::max<int64_t>(final_off[na], 1), s);
  for (size_t ci = 0; ci < chunks.size(); ++ci) {
    const int n_list = static_cast<int>(chunks[ci].second - chunks[ci].first);
    k_compact_panels<<<std::min(n_list, sm_count() * 8), 128, 0, s>>>(
        chunk_list[ci].get(), n_list, topo.omega_off.get(), kcols.get(), chunk_off[ci].get(), chunk_panels[ci].get(),
        ip.panel_off.get(), ip.panels.get());
    LSB_LAUNCH();
  }
  chunk_panels.clear();
  // spectra to the host mirror when requested
  ip.spectra.clear();
  if (keep_spectra) {
    const auto hsp = spec.download(s);
    const auto hn = nspec.download(s);
    ip.spectra.resize(na);
    for (int64_t i = 0; i < na; ++i) ip.spectra[i].assign(hsp.begin() + spec_off[i], hsp.begin() + spec_off[i] + hn[i]);
  }
  // assemble_P: CSR with exact zeros dropped
  const int64_t n = topo.n_nodes;
  p.nr = n;
  p.nc = ip.n_coarse;
  DBuf<int64_t> cnt(n + 1, s);
  cnt.zero(s);
  k_p_count<<<grid_for(n), kThreads, 0, s>>>(topo.node_agg.get(), topo.node_pos.get(), kcols.get(), ip.panel_off.get(),
                                             ip.panels.get(), n, cnt.get());
  LSB_LAUNCH();
  p.off.alloc(n + 1, s);
  size_t tmp = 0;
  LSB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt.get(), p.off.get(), n + 1, s));
  {
    DBuf<unsigned char> tb(tmp, s);
    LSB_CUDA(cub::DeviceScan::InclusiveSum(tb.get(), tmp, cnt.get(), p.off.get(), n + 1, s));
  }
  p.nnz = read_scalar(p.off.get() + n, s);
  p.col.alloc(p.nnz, s);
  p.val.alloc(p.nnz, s);
  k_p_fill<<<grid_for(n), kThreads, 0, s>>>(topo.node_agg.get(), topo.node_pos.get(), kcols.get(), ip.panel_off.get(),
                                            ip.panels.get(), ip.coarse_off.get(), p.off.get(), n, p.col.get(),
                                            p.val.get());
  LSB_LAUNCH();
  tmark("panels and P assembled");
}

void coarse_factor(const DevCsr& a, DBuf<double>& inv, cudaStream_t s) {
  const int64_t m = a.nr;
  DBuf<double> orig(m * m, s), blk(m * m, s), X(m * m, s), slot(8, s);
  DBuf<int32_t> status(1, s);
  status.zero(s);
  orig.zero(s);
  k_coarse_dense<<<grid_for(m), kThreads, 0, s>>>(a.off.get(), a.col.get(), a.val.get(), m, orig.get());
  LSB_LAUNCH();
  LSB_CUDA(cudaMemcpyAsync(blk.get(), orig.get(), m * m * 8, cudaMemcpyDeviceToDevice, s));
  inv.alloc(m * m, s);
  k_coarse_factor<<<1, 1024, 0, s>>>(blk.get(), orig.get(), static_cast<int>(m), X.get(), inv.get(), status.get(),
                                     slot.get());
  LSB_LAUNCH();
  if (read_scalar(status.get(), s)) raise(LSAMGDD_ERR_SETUP, "dense symmetric factorization failed for coarsest-level matrix");
}

}  // namespace lsb
