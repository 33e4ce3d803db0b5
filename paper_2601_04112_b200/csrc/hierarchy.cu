// hierarchy.cu — host orchestration of setup (hierarchy.hpp:106-200), the
// V-cycle (:205-229) and PCG (krylov.hpp:42-92).
//
// Host C++ keeps exactly the sequential, order-dependent pieces the
// reference runs: the greedy aggregation (aggregation.hpp:71-155), the Γ sets
// and the greedy colouring (:165-231), and the setup control flow with its
// error order. Every FP64 stage runs on the device (setup_kernels.cu,
// sparse.cu, solve.cu).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <iostream>
#include <memory>
#include <numeric>
#include <thread>

#include "galerkin.cuh"
#include "hierarchy.cuh"

namespace lsb {

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

constexpr int64_t kNone = -1;

// ---- greedy aggregation (aggregation.hpp:71-117) ------------------------------------
int64_t standard_aggregation(const HostCsr& a, std::vector<int64_t>& asg) {
  if (a.nr == 0) raise(LSAMGDD_ERR_INPUT, "standard_aggregation: matrix is empty");
  if (a.nr != a.nc) raise(LSAMGDD_ERR_DIM, "standard_aggregation: matrix is not square");
  const int64_t n = a.nr;
  asg.assign(n, kNone);
  int64_t next = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (asg[i] != kNone) continue;
    bool has_nb = false, all_free = true;
    for (int64_t k = a.off[i]; k < a.off[i + 1] && all_free; ++k) {
      const int64_t c = a.col[k];
      if (c == i) continue;
      has_nb = true;
      if (asg[c] != kNone) all_free = false;
    }
    if (!has_nb || !all_free) continue;
    asg[i] = next;
    for (int64_t k = a.off[i]; k < a.off[i + 1]; ++k) asg[a.col[k]] = next;
    ++next;
  }
  std::vector<std::pair<int64_t, int64_t>> attached;
  for (int64_t i = 0; i < n; ++i) {
    if (asg[i] != kNone) continue;
    double best = -1.0;
    uint64_t best_agg = ~uint64_t(0);
    for (int64_t k = a.off[i]; k < a.off[i + 1]; ++k) {
      const int64_t c = a.col[k];
      if (c == i || asg[c] == kNone) continue;
      const double w = std::abs(a.val[k]);
      if (w > best || (w == best && static_cast<uint64_t>(asg[c]) < best_agg)) {
        best = w;
        best_agg = static_cast<uint64_t>(asg[c]);
      }
    }
    if (best_agg != ~uint64_t(0)) attached.emplace_back(i, static_cast<int64_t>(best_agg));
  }
  for (const auto& [node, agg] : attached) asg[node] = agg;
  for (int64_t i = 0; i < n; ++i)
    if (asg[i] == kNone) asg[i] = next++;
  return next;
}

HostCsr download(const DevCsr& d, cudaStream_t s) {
  HostCsr h;
  h.nr = d.nr;
  h.nc = d.nc;
  csr_download(d, h.off, h.col, h.val, s);
  return h;
}

void upload(DevCsr& d, const HostCsr& h, cudaStream_t s) {
  lsamgdd_csr c{h.nr, h.nc, static_cast<int64_t>(h.col.size()), h.off.data(), h.col.data(), h.val.data(),
                LSAMGDD_HOST, 0};
  csr_upload(d, &c, s);
}

// multi_pass_aggregation (aggregation.hpp:138-155): the coarse graphs Tᵀ A T
// use the device's ordered Symbolic product, bit-identical to the reference.
int64_t multi_pass_aggregation(const HostCsr& a, const DevCsr& dA, uint64_t passes, std::vector<int64_t>& composed,
                               cudaStream_t s) {
  if (passes < 1) raise(LSAMGDD_ERR_INPUT, "multi_pass_aggregation: need at least one pass");
  std::vector<int64_t> part;
  int64_t n_agg = standard_aggregation(a, part);
  composed = part;
  HostCsr coarse_h;
  DevCsr coarse_d;
  bool first = true;
  for (uint64_t pass = 1; pass < passes; ++pass) {
    if (n_agg <= 1) {
      std::cerr << "lsamgdd: warning: aggregation stopped after " << pass
                << " pass(es); the coarse graph collapsed to one node\n";
      break;
    }
    const int64_t nr = first ? a.nr : coarse_h.nr;
    HostCsr t;
    t.nr = nr;
    t.nc = n_agg;
    t.off.resize(nr + 1);
    t.col.resize(nr);
    t.val.assign(nr, 1.0);
    for (int64_t i = 0; i <= nr; ++i) t.off[i] = i;
    for (int64_t i = 0; i < nr; ++i) t.col[i] = part[i];
    DevCsr td, ttd, tad, cd;
    upload(td, t, s);
    csr_transpose(td, ttd, s);
    csr_spgemm_symbolic(ttd, first ? dA : coarse_d, tad, s);
    csr_spgemm_symbolic(tad, td, cd, s);
    coarse_d = std::move(cd);
    coarse_h = download(coarse_d, s);
    first = false;
    n_agg = standard_aggregation(coarse_h, part);
    for (auto& v : composed) v = part[v];
  }
  return n_agg;
}

// host threads for the per-aggregate loops of the topology (independent aggregates)
static int host_threads(int64_t n_items) {
  const unsigned hc = std::thread::hardware_concurrency();
  const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(hc ? hc : 1, 16));
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cap, n_items / 2048)));
}

// Γ sets, subdomain-intersection adjacency, greedy colouring
// (aggregation.hpp:165-231; second Γ layer for the overlap-2 hook).
void build_topology(const HostCsr& a, const std::vector<int64_t>& asg, int64_t n_agg, int layers, Level& L) {
  const int64_t n = a.nr;
  if (a.nr != a.nc) raise(LSAMGDD_ERR_DIM, "build_topology: matrix is not square");
  if (static_cast<int64_t>(asg.size()) != n)
    raise(LSAMGDD_ERR_INPUT, "build_topology: partition covers " + std::to_string(asg.size()) + " nodes, matrix has " +
                                 std::to_string(n));
  if (n_agg == 0) raise(LSAMGDD_ERR_INPUT, "build_topology: partition has no aggregates");
  for (int64_t v = 0; v < n; ++v)
    if (asg[v] < 0 || asg[v] >= n_agg) raise(LSAMGDD_ERR_INPUT, "build_topology: aggregate id out of range");
  auto& oo = L.h_omega_off;
  auto& om = L.h_omega;
  oo.assign(n_agg + 1, 0);
  for (int64_t v = 0; v < n; ++v) ++oo[asg[v] + 1];
  for (int64_t i = 0; i < n_agg; ++i) {
    if (oo[i + 1] == 0) raise(LSAMGDD_ERR_INPUT, "build_topology: aggregate " + std::to_string(i) + " is empty");
    oo[i + 1] += oo[i];
  }
  om.resize(n);
  {
    std::vector<int32_t> cur(oo.begin(), oo.end() - 1);
    for (int64_t v = 0; v < n; ++v) om[cur[asg[v]]++] = static_cast<int32_t>(v);
  }
  auto& go = L.h_gamma_off;
  auto& gm = L.h_gamma;
  go.assign(n_agg + 1, 0);
  gm.clear();
  // The Γ set of an aggregate depends on nothing but A and the partition: contiguous ranges of
  // aggregates are built by host threads into their own buffers and concatenated in order.
  auto gamma_range = [&](int64_t lo, int64_t hi, std::vector<int32_t>& out, std::vector<int32_t>& cnt) {
    std::vector<int32_t> buf, buf2;
    for (int64_t i = lo; i < hi; ++i) {
      buf.clear();
      for (int32_t p = oo[i]; p < oo[i + 1]; ++p) {
        const int64_t u = om[p];
        for (int64_t k = a.off[u]; k < a.off[u + 1]; ++k)
          if (asg[a.col[k]] != i) buf.push_back(static_cast<int32_t>(a.col[k]));
      }
      std::sort(buf.begin(), buf.end());
      buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
      if (layers >= 2) {
        buf2 = buf;
        for (int32_t u : buf)
          for (int64_t k = a.off[u]; k < a.off[u + 1]; ++k)
            if (asg[a.col[k]] != i) buf2.push_back(static_cast<int32_t>(a.col[k]));
        std::sort(buf2.begin(), buf2.end());
        buf2.erase(std::unique(buf2.begin(), buf2.end()), buf2.end());
        buf.swap(buf2);
      }
      out.insert(out.end(), buf.begin(), buf.end());
      cnt[i - lo] = static_cast<int32_t>(buf.size());
    }
  };
  const int nt = host_threads(n_agg);
  {
    std::vector<std::vector<int32_t>> parts(nt), cnts(nt);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
      const int64_t lo = n_agg * t / nt, hi = n_agg * (t + 1) / nt;
      cnts[t].assign(hi - lo, 0);
      if (t + 1 < nt)
        th.emplace_back(gamma_range, lo, hi, std::ref(parts[t]), std::ref(cnts[t]));
      else
        gamma_range(lo, hi, parts[t], cnts[t]);
    }
    for (auto& x : th) x.join();
    size_t total = 0;
    for (auto& x : parts) total += x.size();
    gm.reserve(total);
    int64_t i = 0;
    for (int t = 0; t < nt; ++t) {
      gm.insert(gm.end(), parts[t].begin(), parts[t].end());
      for (int32_t c : cnts[t]) {
        go[i + 1] = go[i] + c;
        ++i;
      }
    }
  }
  // holders: owner first, then Γ-holders in ascending aggregate order
  std::vector<int64_t> hoff(n + 1, 0);
  for (int64_t v = 0; v < n; ++v) hoff[v + 1] = 1;
  for (int32_t gnode : gm) ++hoff[gnode + 1];
  for (int64_t v = 0; v < n; ++v) hoff[v + 1] += hoff[v];
  std::vector<int32_t> hold(hoff[n]);
  {
    std::vector<int64_t> cur(hoff.begin(), hoff.end() - 1);
    for (int64_t v = 0; v < n; ++v) hold[cur[v]++] = static_cast<int32_t>(asg[v]);
    for (int64_t i = 0; i < n_agg; ++i)
      for (int32_t p = go[i]; p < go[i + 1]; ++p) hold[cur[gm[p]]++] = static_cast<int32_t>(i);
  }
  std::vector<int64_t> aoff(n_agg + 1, 0);
  for (int64_t v = 0; v < n; ++v) {
    const int64_t c = hoff[v + 1] - hoff[v];
    for (int64_t x = hoff[v]; x < hoff[v + 1]; ++x) aoff[hold[x] + 1] += c - 1;
  }
  for (int64_t i = 0; i < n_agg; ++i) aoff[i + 1] += aoff[i];
  std::vector<int32_t> adj(aoff[n_agg]);
  {
    std::vector<int64_t> cur(aoff.begin(), aoff.end() - 1);
    for (int64_t v = 0; v < n; ++v)
      for (int64_t x = hoff[v]; x < hoff[v + 1]; ++x)
        for (int64_t y = x + 1; y < hoff[v + 1]; ++y) {
          adj[cur[hold[x]]++] = hold[y];
          adj[cur[hold[y]]++] = hold[x];
        }
  }
  std::vector<int64_t> deg(n_agg);
  {
    auto sort_range = [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        auto b = adj.begin() + aoff[i], e = adj.begin() + aoff[i + 1];
        std::sort(b, e);
        deg[i] = std::unique(b, e) - b;
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t + 1 < nt; ++t) th.emplace_back(sort_range, n_agg * t / nt, n_agg * (t + 1) / nt);
    sort_range(n_agg * (nt - 1) / nt, n_agg);
    for (auto& x : th) x.join();
  }
  std::vector<int64_t> order(n_agg);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return deg[x] > deg[y]; });
  L.colors.assign(n_agg, kNone);
  int64_t max_color = 0;
  std::vector<char> used;
  for (int64_t i : order) {
    used.assign(deg[i] + 1, 0);
    for (int64_t k = aoff[i]; k < aoff[i] + deg[i]; ++k) {
      const int64_t cj = L.colors[adj[k]];
      if (cj != kNone && cj < static_cast<int64_t>(used.size())) used[cj] = 1;
    }
    int64_t c = 0;
    while (used[c]) ++c;
    L.colors[i] = c;
    max_color = std::max(max_color, c);
  }
  L.n_colors = max_color + 1;
}

void upload_topology(Level& L, const std::vector<int64_t>& asg, cudaStream_t s) {
  DevTopo& t = L.topo;
  t.n_nodes = static_cast<int64_t>(asg.size());
  t.n_agg = static_cast<int64_t>(L.h_omega_off.size()) - 1;
  t.omega_off.upload(L.h_omega_off, s);
  t.omega.upload(L.h_omega, s);
  t.gamma_off.upload(L.h_gamma_off, s);
  t.gamma.upload(L.h_gamma, s);
  std::vector<int32_t> na(t.n_nodes), np(t.n_nodes);
  for (int64_t i = 0; i < t.n_agg; ++i)
    for (int32_t p = L.h_omega_off[i]; p < L.h_omega_off[i + 1]; ++p) {
      na[L.h_omega[p]] = static_cast<int32_t>(i);
      np[L.h_omega[p]] = p - L.h_omega_off[i];
    }
  t.node_agg.upload(na, s);
  t.node_pos.upload(np, s);
}

double eigen_threshold(double kappa, int64_t kc, int64_t n_mult) {  // splitting.hpp:170-180
  if (kc == 0 || n_mult == 0) raise(LSAMGDD_ERR_INPUT, "eigen_threshold: k_c and n_mult must be positive");
  if (kappa <= static_cast<double>(kc)) {
    std::cerr << "lsamgdd: warning: target condition number " << kappa << " does not exceed the color count " << kc
              << "; using the floor threshold\n";
    return 0.1;
  }
  const double t = (kappa - static_cast<double>(kc)) / (static_cast<double>(kc) * static_cast<double>(n_mult));
  return std::max(0.1, t);
}

}  // namespace

void validate_setup(const lsamgdd_csr* g0, const lsamgdd_params* p) {  // hierarchy.hpp:107-117
  if (p->max_levels < 2) raise(LSAMGDD_ERR_INPUT, "setup: max_levels must be at least 2");
  if (p->coarse_size < 1) raise(LSAMGDD_ERR_INPUT, "setup: coarse_size must be positive");
  if (p->aggregation_passes < 1) raise(LSAMGDD_ERR_INPUT, "setup: aggregation_passes must be positive");
  if (!(p->kappa > 1.0)) raise(LSAMGDD_ERR_INPUT, "setup: kappa must exceed 1");
  if (!(p->must_keep > 1.0)) raise(LSAMGDD_ERR_INPUT, "setup: must_keep must exceed 1");
  if (p->n_ratios == 0) raise(LSAMGDD_ERR_INPUT, "setup: coarsening_ratios must not be empty");
  if (p->n_ratios > 8) raise(LSAMGDD_ERR_INPUT, "setup: at most 8 coarsening ratios");
  for (uint64_t k = 0; k < p->n_ratios; ++k)
    if (p->coarsening_ratios[k] < 2) raise(LSAMGDD_ERR_INPUT, "setup: coarsening ratios must be at least 2");
  if (g0->n_rows == 0 || g0->n_cols == 0) raise(LSAMGDD_ERR_INPUT, "setup: factor is empty");
  if (g0->n_rows >= (int64_t(1) << 31) || g0->n_cols >= (int64_t(1) << 31))
    raise(LSAMGDD_ERR_SIZE, "setup: dimensions must stay below 2^31");
  if (p->level0_partition && p->level0_n_aggregates <= 0)
    raise(LSAMGDD_ERR_INPUT, "build_topology: partition has no aggregates");
}

namespace {

__global__ void k_col_agg(const int32_t* coff, int64_t n_agg, int32_t* col_agg) {
  for (int64_t a = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; a < n_agg; a += int64_t(gridDim.x) * blockDim.x)
    for (int32_t c = coff[a]; c < coff[a + 1]; ++c) col_agg[c] = static_cast<int32_t>(a);
}

}  // namespace

SchwarzView Level::schwarz_view() const {
  SchwarzView v;
  v.n_agg = topo.n_agg;
  v.omega_off = topo.omega_off.get();
  v.omega = topo.omega.get();
  v.gamma_off = topo.gamma_off.get();
  v.gamma = topo.gamma.get();
  v.sm_off = sm.off.get();
  v.sm_data = sm.data.get();
  v.order = sm.order.get();
  v.max_omega = sm.max_omega;
  v.max_sub = sm.max_sub;
  v.n_groups = sm.n_groups;
  v.g_nw = sm.g_nw.get();
  v.g_ng = sm.g_ng.get();
  v.g_cnt = sm.g_cnt.get();
  v.g_ids_off = sm.g_ids_off.get();
  v.g_blk_off = sm.g_blk_off.get();
  v.lane_ids = sm.lane_ids.get();
  v.lane_blk = sm.lane_blk.get();
  v.color_goff = &sm.color_goff;
  v.lane_ras_items = sm.lane_ras_items.get();
  v.n_lane_ras_items = static_cast<int64_t>(sm.lane_ras_items.size());
  v.lane_rast_items = sm.lane_rast_items.get();
  v.lane_rast_color_off = &sm.lane_rast_color_off;
  v.g_color = sm.g_color.get();
  v.color_groups = sm.color_groups.get();
  v.rast_tmp = nullptr;  // the caller's workspace supplies the RAS-T slot buffer
  v.g_slot_off = sm.g_slot_off.get();
  v.lane_slots = sm.lane_slots.get();
  v.node_slot_off = sm.node_slot_off.get();
  v.n_slots = sm.n_slots;
  v.stage_slot_bytes = sm.stage_slot_bytes;
  v.n_nodes = topo.n_nodes;
  v.n_colors = static_cast<int>(sm.n_colors);
  v.stage_blk_bytes = sm.stage_blk_bytes;
  v.stage_ids_bytes = sm.stage_ids_bytes;
  v.rows = sm.rows;
  v.row_off = sm.row_off.get();
  v.row_data = sm.row_data.get();
  v.ras_agg = sm.ras_agg.get();
  v.ras_row = sm.ras_row.get();
  v.n_ras_items = static_cast<int64_t>(sm.ras_agg.size());
  v.ras_ch = sm.ras_ch;
  v.rast_ch = sm.rast_ch;
  v.rast_agg = sm.rast_agg.get();
  v.rast_row = sm.rast_row.get();
  v.rast_color_off = &sm.rast_color_off;
  return v;
}

InterpView Level::interp_view() const {
  InterpView v;
  v.n_fine = topo.n_nodes;
  v.n_coarse = ip.n_coarse;
  v.n_agg = topo.n_agg;
  v.node_agg = topo.node_agg.get();
  v.node_pos = topo.node_pos.get();
  v.omega_off = topo.omega_off.get();
  v.omega = topo.omega.get();
  v.coarse_off = ip.coarse_off.get();
  v.panel_off = ip.panel_off.get();
  v.panels = ip.panels.get();
  v.col_agg = col_agg.get();
  return v;
}

Hierarchy::~Hierarchy() {
  if (stream) {
    cudaStreamSynchronize(stream);
    levels.clear();
    coarse_inv.release();
    g0_sell = Sell();
    g0t_sell = Sell();
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
  if (side_stream) {
    cudaStreamSynchronize(side_stream);
    cudaStreamDestroy(side_stream);
  }
}

Hierarchy* setup(const lsamgdd_csr* g0, const lsamgdd_params* p) {
  validate_setup(g0, p);
  auto h = std::make_unique<Hierarchy>();
  h->params = *p;
  h->params.level0_partition = nullptr;
  h->ratios.assign(p->coarsening_ratios, p->coarsening_ratios + p->n_ratios);
  h->device = p->device;
  LSB_CUDA(cudaSetDevice(p->device));
  LSB_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  cudaStream_t s = h->stream;
  LSB_CUDA(cudaStreamCreateWithFlags(&h->side_stream, cudaStreamNonBlocking));
  cudaStream_t s2 = h->side_stream;
  auto stage = [&](const char* name, Clock::time_point t0) {
    LSB_CUDA(cudaStreamSynchronize(s));
    h->timings.push_back({name, ms_since(t0)});
  };
  auto t0 = Clock::now();
  h->levels.emplace_back();
  {
    Level& L0 = h->levels[0];
    csr_upload(L0.G, g0, s);
    DevCsr gt;
    csr_transpose(L0.G, gt, s);
    csr_spgemm_symbolic(gt, L0.G, L0.A, s);
    sell_from_csr(L0.G, h->g0_sell, s);
    sell_from_csr(gt, h->g0t_sell, s);
  }
  stage("upload_galerkin_A0", t0);
  const uint64_t probe = p->probe_levels;
  const int64_t lvl0 = static_cast<int64_t>(p->level_offset);  // global index of this hierarchy's first level
  while (h->levels.size() + lvl0 < p->max_levels && static_cast<uint64_t>(h->levels.back().A.nr) > p->coarse_size &&
         (probe == 0 || h->levels.size() <= probe)) {
    const int64_t ell = static_cast<int64_t>(h->levels.size()) - 1 + lvl0;
    Level& cur = h->levels.back();
    t0 = Clock::now();
    HostCsr a_host = download(cur.A, s);
    std::vector<int64_t> asg;
    int64_t n_agg;
    if (ell == 0 && p->level0_partition) {
      asg.assign(p->level0_partition, p->level0_partition + cur.A.nr);
      n_agg = p->level0_n_aggregates;
    } else {
      n_agg = multi_pass_aggregation(a_host, cur.A, p->aggregation_passes, asg, s);
    }
    build_topology(a_host, asg, n_agg, (ell == 0 && p->level0_overlap >= 2) ? 2 : 1, cur);
    upload_topology(cur, asg, s);
    stage("aggregation_topology", t0);
    // The Schwarz blocks depend on A_l and the topology only: they are factorised on a second
    // stream by a side thread while this one runs the local eigenproblems (which leave most SMs
    // idle on the coarse levels). Joined before the Galerkin products.
    t0 = Clock::now();
    std::exception_ptr sm_err;
    std::thread sm_thread([&, dev = p->device] {
      try {
        LSB_CUDA(cudaSetDevice(dev));
        build_smoother(cur.A, cur.topo, cur.h_omega_off, cur.h_gamma_off, cur.colors, cur.n_colors, cur.sm, s2,
                       &cur.h_gamma);
        sell_from_csr(cur.A, cur.A_sell, s2);
        LSB_CUDA(cudaStreamSynchronize(s2));
      } catch (...) {
        sm_err = std::current_exception();
      }
    });
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{sm_thread};
    DevRowSets rs;
    row_sets(cur.G, cur.topo, rs, s);
    if (rs.empty_rows > 0)
      std::cerr << "lsamgdd: note: " << rs.empty_rows << " empty factor row(s) belong to no row set\n";
    cur.n_mult = rs.n_mult;
    cur.thresh = p->thresh_override > 0.0 ? p->thresh_override : eigen_threshold(p->kappa, cur.n_colors, rs.n_mult);
    GevpParams gp;
    gp.thresh = cur.thresh;
    gp.must_keep = p->must_keep;
    gp.variant = p->gevp_variant;
    gp.level = static_cast<int>(ell);
    gp.ratio = static_cast<int64_t>(h->ratios[std::min<size_t>(ell, h->ratios.size() - 1)]);
    gp.level0_max_modes = static_cast<int64_t>(p->level0_max_modes);
    local_gevp_all(cur.G, cur.topo, cur.h_omega_off, cur.h_gamma_off, rs, {}, gp, cur.ip, cur.P, p->keep_spectra != 0,
                   s);
    cur.mult.alloc(rs.mult.size(), s);
    LSB_CUDA(cudaMemcpyAsync(cur.mult.get(), rs.mult.get(), rs.mult.bytes(), cudaMemcpyDeviceToDevice, s));
    cur.has_interp = true;
    cur.col_agg.alloc(std::max<int64_t>(cur.ip.n_coarse, 1), s);
    k_col_agg<<<std::max(1, static_cast<int>(std::min<int64_t>(ceil_div(n_agg, 256), 1024))), 256, 0, s>>>(
        cur.ip.coarse_off.get(), n_agg, cur.col_agg.get());
    LSB_LAUNCH();
    stage("local_gevp", t0);
    t0 = Clock::now();
    sm_thread.join();
    if (sm_err) std::rethrow_exception(sm_err);
    stage("build_smoother", t0);  // what is left of it after the eigenproblems
    t0 = Clock::now();
    Level next;
    galerkin_gp(cur.G, cur.topo, cur.ip, next.G, s);
    galerkin_gtg(next.G, rs, n_agg, cur.ip, cur.col_agg.get(), next.A, s);
    stage("galerkin", t0);
    if (next.A.nr >= cur.A.nr)
      raise(LSAMGDD_ERR_SETUP, "setup: stagnant coarsening at level " + std::to_string(ell) + " (" +
                                   std::to_string(cur.A.nr) + " -> " + std::to_string(next.A.nr) + ")");
    lsamgdd_level_summary row{};
    row.level = static_cast<uint64_t>(ell);
    row.dim = static_cast<uint64_t>(cur.A.nr);
    row.nnz = static_cast<uint64_t>(cur.A.nnz);
    row.n_aggregates = static_cast<uint64_t>(n_agg);
    row.k_c = static_cast<uint64_t>(cur.n_colors);
    row.n_mult = static_cast<uint64_t>(cur.n_mult);
    row.thresh = cur.thresh;
    row.modes_kept = static_cast<uint64_t>(cur.ip.n_coarse);
    h->summary.push_back(row);
    h->levels.push_back(std::move(next));
  }
  t0 = Clock::now();
  {
    const Level& co = h->levels.back();
    h->n_coarse = co.A.nr;
    h->probe = probe > 0;
    if (!h->probe) coarse_factor(co.A, h->coarse_inv, s);
  }
  stage("coarse_factor", t0);
  lsamgdd_level_summary last{};
  last.level = h->levels.size() - 1;
  last.dim = static_cast<uint64_t>(h->levels.back().A.nr);
  last.nnz = static_cast<uint64_t>(h->levels.back().A.nnz);
  h->summary.push_back(last);
  LSB_CUDA(cudaStreamSynchronize(s));
  return h.release();
}

StandaloneSmoother::~StandaloneSmoother() {
  if (s) {
    cudaStreamSynchronize(s);
    rast_tmp.release();
    L = Level();
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
}

StandaloneSmoother* make_smoother(const lsamgdd_csr* a, int64_t n_agg, const int64_t* omega_off, const int64_t* omega,
                                  const int64_t* gamma_off, const int64_t* gamma, const int64_t* colors) {
  if (a->n_rows != a->n_cols) raise(LSAMGDD_ERR_DIM, "build_smoother: matrix is not square");
  if (n_agg <= 0 || !omega_off || !omega || !gamma_off || !colors)
    raise(LSAMGDD_ERR_INPUT, "build_smoother: topology arrays are required");
  const int64_t n = a->n_rows;
  if (omega_off[n_agg] != n)
    raise(LSAMGDD_ERR_DIM, "build_smoother: topology covers " + std::to_string(omega_off[n_agg]) + " nodes, matrix has " +
                               std::to_string(n));
  auto sm = std::make_unique<StandaloneSmoother>();
  sm->n = n;
  LSB_CUDA(cudaStreamCreateWithFlags(&sm->s, cudaStreamNonBlocking));
  Level& L = sm->L;
  L.h_omega_off.assign(omega_off, omega_off + n_agg + 1);
  L.h_omega.assign(omega, omega + n);
  L.h_gamma_off.assign(gamma_off, gamma_off + n_agg + 1);
  L.h_gamma.assign(gamma, gamma + gamma_off[n_agg]);
  L.colors.assign(colors, colors + n_agg);
  L.n_colors = 0;
  for (int64_t c : L.colors) {
    if (c < 0) raise(LSAMGDD_ERR_INPUT, "build_smoother: negative colour");
    L.n_colors = std::max(L.n_colors, c + 1);
  }
  std::vector<int64_t> asg(n, -1);
  for (int64_t i = 0; i < n_agg; ++i)
    for (int64_t p = omega_off[i]; p < omega_off[i + 1]; ++p) {
      if (omega[p] < 0 || omega[p] >= n || asg[omega[p]] != -1)
        raise(LSAMGDD_ERR_INPUT, "build_smoother: the interiors must partition the nodes");
      asg[omega[p]] = i;
    }
  for (int64_t k = 0; k < gamma_off[n_agg]; ++k)
    if (gamma[k] < 0 || gamma[k] >= n) raise(LSAMGDD_ERR_INDEX, "build_smoother: boundary node out of range");
  csr_upload(L.A, a, sm->s);
  upload_topology(L, asg, sm->s);
  build_smoother(L.A, L.topo, L.h_omega_off, L.h_gamma_off, L.colors, L.n_colors, L.sm, sm->s, &L.h_gamma);
  if (L.sm.n_slots > 0) sm->rast_tmp.alloc(L.sm.n_slots, sm->s);
  LSB_CUDA(cudaStreamSynchronize(sm->s));
  return sm.release();
}

void smoother_apply(const StandaloneSmoother& sm, int mode, const double* r, double* e) {
  SchwarzView sv = sm.L.schwarz_view();
  sv.rast_tmp = sm.rast_tmp.get();
  if (mode == 0) {
    schwarz_ras(sv, r, e, false, sm.s);
  } else {
    LSB_CUDA(cudaMemsetAsync(e, 0, sm.n * 8, sm.s));
    schwarz_rast(sv, sm.L.sm.color_off, r, e, sm.s);
  }
}

double operator_complexity(const Hierarchy& h) {  // hierarchy.hpp:257-261
  double total = 0.0;
  for (const Level& L : h.levels) total += static_cast<double>(L.A.nnz);
  return total / static_cast<double>(h.levels.front().A.nnz);
}

SolveWs::SolveWs(const Hierarchy& h) {
  LSB_CUDA(cudaSetDevice(h.device));
  LSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t nl = h.levels.size();
  e.resize(nl);
  res.resize(nl);
  rhs.resize(nl);
  rast_tmp.resize(nl);
  for (size_t l = 0; l < nl; ++l) {
    const int64_t n = std::max<int64_t>(h.levels[l].A.nr, 1);
    e[l].alloc(n, s);
    res[l].alloc(n, s);
    rhs[l].alloc(n, s);
    if (h.levels[l].sm.n_slots > 0) rast_tmp[l].alloc(h.levels[l].sm.n_slots, s);
  }
  red.init(s);
  for (auto& e : ev) LSB_CUDA(cudaEventCreate(&e));
}

SolveWs::~SolveWs() {
  if (s) {
    cudaStreamSynchronize(s);
    e.clear();
    res.clear();
    rhs.clear();
    rast_tmp.clear();
    red.partial.release();
    red.ticket.release();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
}

// res = r - A_l e: SELL thread-per-row on short rows, warp per row on long ones
static void level_residual(const Level& L, const double* e, double* res, const double* r, cudaStream_t s) {
  if (L.A.nr > 0 && L.A.nnz >= 48 * L.A.nr)
    csr_spmv_warp(L.A, e, res, r, s);
  else
    sell_spmv(L.A_sell, e, res, r, s);
}

void vcycle(const Hierarchy& h, SolveWs& ws, int64_t level, const double* r, double* e) {
  if (level < 0 || level >= static_cast<int64_t>(h.levels.size())) raise(LSAMGDD_ERR_INDEX, "vcycle: level out of range");
  if (h.probe) raise(LSAMGDD_ERR_INPUT, "vcycle: the hierarchy was built with probe_levels (no coarsest factorisation)");
  const Level& L = h.levels[level];
  cudaStream_t s = ws.s;
  const int64_t n = L.A.nr;
  if (level + 1 == static_cast<int64_t>(h.levels.size())) {
    dense_matvec(h.coarse_inv.get(), h.n_coarse, r, e, s);
    return;
  }
  SchwarzView sv = L.schwarz_view();
  sv.rast_tmp = ws.rast_tmp[level].get();  // this call's own slot buffer: concurrent solves share the handle
  double* res = ws.res[level].get();
  if (h.params.pre_sweeps == 0) LSB_CUDA(cudaMemsetAsync(e, 0, n * 8, s));
  for (uint64_t sw = 0; sw < h.params.pre_sweeps; ++sw) {
    if (sw == 0) {
      if (ws.timing && level == 0) LSB_CUDA(cudaEventRecordWithFlags(ws.ev[0], s, cudaEventRecordExternal));
      schwarz_ras(sv, r, e, false, s);  // e = 0 + RAS(r - A·0)
      if (ws.timing && level == 0) LSB_CUDA(cudaEventRecordWithFlags(ws.ev[1], s, cudaEventRecordExternal));
    } else {
      level_residual(L, e, res, r, s);
      schwarz_ras(sv, res, e, true, s);
    }
  }
  level_residual(L, e, res, r, s);
  double* rc = ws.rhs[level + 1].get();
  double* ec = ws.e[level + 1].get();
  const InterpView iv = L.interp_view();
  restrict_pt(iv, res, rc, s);
  vcycle(h, ws, level + 1, rc, ec);
  prolong_add(iv, ec, e, s);
  for (uint64_t sw = 0; sw < h.params.post_sweeps; ++sw) {
    level_residual(L, e, res, r, s);
    const bool tm = ws.timing && level == 0 && sw == 0;
    if (tm) LSB_CUDA(cudaEventRecordWithFlags(ws.ev[2], s, cudaEventRecordExternal));
    schwarz_rast(sv, L.sm.color_off, res, e, s);
    if (tm) LSB_CUDA(cudaEventRecordWithFlags(ws.ev[3], s, cudaEventRecordExternal));
  }
}

PcgResult pcg(const Hierarchy& h, SolveWs& ws, const Sell& g, const Sell& gt, const double* b, double* x, double tol,
              uint64_t maxit, lsamgdd_kernel_stats* stats) {
  PcgResult out;
  cudaStream_t s = ws.s;
  const int64_t n = gt.nr, m = g.nr;
  if (n != h.levels[0].A.nr) raise(LSAMGDD_ERR_DIM, "pcg: factor columns do not match the hierarchy");
  const int64_t launches0 = launch_counter();
  DBuf<double> r(n, s), z(n, s), p(n, s), ap(n, s), gp(std::max<int64_t>(m, 1), s);
  DBuf<PcgScalars> sc(1, s);
  sc.zero(s);
  PcgScalars* hsc = nullptr;
  LSB_CUDA(cudaMallocHost(&hsc, sizeof(PcgScalars)));
  struct HostFree {
    PcgScalars* p;
    ~HostFree() { cudaFreeHost(p); }
  } hf{hsc};
  auto readback = [&]() {
    LSB_CUDA(cudaMemcpyAsync(hsc, sc.get(), sizeof(PcgScalars), cudaMemcpyDeviceToHost, s));
    LSB_CUDA(cudaStreamSynchronize(s));
  };
  const auto t0 = Clock::now();
  LSB_CUDA(cudaMemsetAsync(x, 0, n * 8, s));
  LSB_CUDA(cudaMemcpyAsync(r.get(), b, n * 8, cudaMemcpyDeviceToDevice, s));
  dot(ws.red, r.get(), r.get(), n, &sc.get()->r0_2, s);
  readback();
  const double r0 = std::sqrt(hsc->r0_2);
  out.history.push_back(r0);
  if (r0 == 0.0) {
    out.converged = true;
    out.solve_seconds = ms_since(t0) / 1e3;
    return out;
  }
  vcycle(h, ws, 0, r.get(), z.get());
  pcg_rz(ws.red, r.get(), z.get(), n, sc.get(), true, s);
  pcg_update_p(p.get(), z.get(), n, sc.get(), true, s);
  // loop body, captured once as a CUDA graph:
  //   [vcycle(r)->z, rz_next, beta, p = z + beta p]
  //   gp = G p, ap = Gᵀ gp, <p,ap>, alpha, x += αp, r -= α·ap, ‖r‖²
  auto tail = [&]() {
    if (ws.timing) LSB_CUDA(cudaEventRecordWithFlags(ws.ev[4], s, cudaEventRecordExternal));
    sell_spmv(g, p.get(), gp.get(), nullptr, s);
    pcg_ap_dot(gt, gp.get(), p.get(), ap.get(), ws.red, sc.get(), s);
    if (ws.timing) LSB_CUDA(cudaEventRecordWithFlags(ws.ev[5], s, cudaEventRecordExternal));
    pcg_update_xr(ws.red, x, r.get(), p.get(), ap.get(), n, sc.get(), s);
  };
  const int64_t c0 = launch_counter();
  cudaGraph_t graph;
  ws.timing = true;  // level-0 Schwarz sweeps bracketed by events inside the graph
  LSB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  vcycle(h, ws, 0, r.get(), z.get());
  pcg_rz(ws.red, r.get(), z.get(), n, sc.get(), false, s);
  pcg_update_p(p.get(), z.get(), n, sc.get(), false, s);
  tail();
  LSB_CUDA(cudaStreamEndCapture(s, &graph));
  ws.timing = false;
  const int64_t per_iter = launch_counter() - c0;
  cudaGraphExec_t gexec = nullptr;
  LSB_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
  LSB_CUDA(cudaGraphDestroy(graph));
  struct GraphFree {
    cudaGraphExec_t g;
    ~GraphFree() {
      if (g) cudaGraphExecDestroy(g);
    }
  } gf{gexec};
  readback();
  if (!(hsc->rz > 0.0)) raise(LSAMGDD_ERR_INDEFINITE, "pcg: preconditioned product <r, Br> is not positive");
  tail();  // first iteration's operator application
  readback();
  uint64_t k = 0;
  int64_t graph_launches = 0;
  double sw_ms = 0.0, op_ms = 0.0;
  while (k < maxit) {
    if (!(hsc->pap > 0.0)) raise(LSAMGDD_ERR_INDEFINITE, "pcg: curvature <p, Ap> is not positive");
    ++k;
    const double rn = std::sqrt(hsc->rn2);
    out.history.push_back(rn);
    if (rn <= tol * r0) {
      out.converged = true;
      break;
    }
    if (k == maxit) {
      // krylov.hpp:75-77: the reference still applies the preconditioner after its last
      // iteration and throws IndefiniteError on a non-positive <r, Br>
      vcycle(h, ws, 0, r.get(), z.get());
      pcg_rz(ws.red, r.get(), z.get(), n, sc.get(), false, s);
      readback();
      if (!(hsc->rz_next > 0.0)) raise(LSAMGDD_ERR_INDEFINITE, "pcg: preconditioned product <r, Br> is not positive");
      break;
    }
    LSB_CUDA(cudaGraphLaunch(gexec, s));
    ++graph_launches;
    readback();
    float a = 0, b2 = 0;
    LSB_CUDA(cudaEventElapsedTime(&a, ws.ev[0], ws.ev[1]));
    LSB_CUDA(cudaEventElapsedTime(&b2, ws.ev[2], ws.ev[3]));
    sw_ms += a + b2;
    float c2 = 0;
    LSB_CUDA(cudaEventElapsedTime(&c2, ws.ev[4], ws.ev[5]));
    op_ms += c2;
    if (!(hsc->rz_next > 0.0)) raise(LSAMGDD_ERR_INDEFINITE, "pcg: preconditioned product <r, Br> is not positive");
  }
  out.iterations = k;
  out.solve_seconds = ms_since(t0) / 1e3;
  out.launches = (launch_counter() - launches0) + graph_launches * per_iter - per_iter;
  launch_counter() += graph_launches * per_iter - per_iter;  // graph replays launch the captured kernels
  if (stats) {
    *stats = lsamgdd_kernel_stats{};
    stats->schwarz_ms = sw_ms;
    stats->schwarz_bytes = static_cast<double>(graph_launches) * (h.levels.size() > 1 ? h.levels[0].sm.bytes_ras + h.levels[0].sm.bytes_rast : 0.0);
    // launches per RAS + RAS-T pair: 3 on the TMA path (RAS, RAS-T, slot gather), else 1 + the colour launches
    const int64_t per_pair = h.levels.size() > 1
                                 ? (h.levels[0].sm.n_slots > 0 ? 3 : static_cast<int64_t>(h.levels[0].sm.color_off.size()))
                                 : 0;
    stats->schwarz_launches = graph_launches * per_pair;
    // PCG operator y = Gᵀ(G p) (SpMV with G, then with the stored Gᵀ fused with ⟨p, y⟩):
    // algorithmic bytes B(spmv_G) + B(spmvT_G) of SURVEY.md §8(d)
    const double nnz = static_cast<double>(g.nnz), mm = static_cast<double>(g.nr), nn = static_cast<double>(n);
    stats->spmv_ms = op_ms;
    stats->spmv_bytes = static_cast<double>(graph_launches) *
                        ((12 * nnz + 4 * (mm + 1) + 8 * nn + 8 * mm) + (12 * nnz + 4 * (nn + 1) + 8 * mm + 8 * nn));
    stats->spmv_launches = graph_launches * 2;
    stats->total_launches = out.launches;
  }
  return out;
}

}  // namespace lsb
