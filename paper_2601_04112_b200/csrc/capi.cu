// capi.cu — the C ABI of include/lsamgdd_b200.h (the drop-in boundary for the
// reference's header API).
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <new>
#include <random>

#include "generate.cuh"
#include "hierarchy.cuh"

using namespace lsb;

namespace {

void put_err(char* err, size_t errlen, const char* msg) {
  if (!err || errlen == 0) return;
  std::strncpy(err, msg, errlen - 1);
  err[errlen - 1] = '\0';
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    return LSAMGDD_OK;
  } catch (const lsb::Error& e) {
    put_err(err, errlen, e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    put_err(err, errlen, "host allocation failed");
    return LSAMGDD_ERR_OOM;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return LSAMGDD_ERR_ERROR;
  }
}

bool device_ok() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return false;
  }
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, 0);
  return major == 10;
}

void require_device() {
  if (!device_ok())
    raise(LSAMGDD_ERR_CUDA, "no usable sm_100 (B200) device: this library has no CPU fallback");
}

const Hierarchy& H(const void* h) {
  if (!h) raise(LSAMGDD_ERR_INPUT, "null hierarchy handle");
  return *static_cast<const Hierarchy*>(h);
}

// ---- ordering against the caller's device work ---------------------------------
// The library works on its own non-blocking streams. Device-memory inputs may
// still be in flight on a caller stream, so before the first read the call
// either waits on that stream (lsamgdd_set_caller_stream, per host thread) or,
// when none was given, synchronises the device.
thread_local cudaStream_t t_caller_stream = nullptr;
thread_local bool t_has_caller_stream = false;

void wait_for_caller(cudaStream_t lib_stream) {
  if (!t_has_caller_stream) {
    LSB_CUDA(cudaDeviceSynchronize());
    return;
  }
  cudaEvent_t ev;
  LSB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  LSB_CUDA(cudaEventRecord(ev, t_caller_stream));
  LSB_CUDA(cudaStreamWaitEvent(lib_stream, ev, 0));
  LSB_CUDA(cudaEventDestroy(ev));
}

// Runs f(d_in, d_out) on device vectors, staging host arrays when needed.
template <class F>
void with_vectors(cudaStream_t ws_s, const double* in, int64_t nin, double* out, int64_t nout, int32_t memory, F&& f) {
  if (memory == LSAMGDD_DEVICE) {
    wait_for_caller(ws_s);
    f(in, out);
    LSB_CUDA(cudaStreamSynchronize(ws_s));  // results are complete when the call returns
    return;
  }
  DBuf<double> din(std::max<int64_t>(nin, 1), ws_s), dout(std::max<int64_t>(nout, 1), ws_s);
  if (nin) LSB_CUDA(cudaMemcpyAsync(din.get(), in, nin * 8, cudaMemcpyHostToDevice, ws_s));
  f(din.get(), dout.get());
  if (nout) LSB_CUDA(cudaMemcpyAsync(out, dout.get(), nout * 8, cudaMemcpyDeviceToHost, ws_s));
  LSB_CUDA(cudaStreamSynchronize(ws_s));
}

void fill_report(lsamgdd_report* rep, const Hierarchy& h, const PcgResult& pr) {
  if (!rep) return;
  rep->iterations = pr.iterations;
  rep->converged = pr.converged ? 1 : 0;
  const double r0 = pr.history.front();
  double avg = 0.0, itt = 0.0;
  if (r0 != 0.0) {  // krylov.hpp:82-90
    const double ratio = pr.history.back() / r0;
    const uint64_t k = pr.iterations;
    avg = k > 0 ? std::pow(ratio, 1.0 / static_cast<double>(k)) : 1.0;
    if (avg > 0.0 && avg < 1.0)
      itt = std::log(0.1) / std::log(avg);
    else if (avg == 0.0)
      itt = 0.0;
    else
      itt = std::numeric_limits<double>::infinity();
  }
  rep->avg_conv_factor = avg;
  rep->iters_to_tenth = itt;
  rep->operator_complexity = operator_complexity(h);
  double setup_ms = 0;
  for (const auto& t : h.timings) setup_ms += t.ms;
  rep->setup_seconds = setup_ms / 1e3;
  rep->solve_seconds = pr.solve_seconds;
  rep->history_len = pr.history.size();
  if (rep->residual_history)
    for (uint64_t i = 0; i < pr.history.size() && i < rep->history_capacity; ++i) rep->residual_history[i] = pr.history[i];
}

const Level& level_of(const Hierarchy& h, int64_t level) {
  if (level < 0 || level >= static_cast<int64_t>(h.levels.size())) raise(LSAMGDD_ERR_INDEX, "level out of range");
  return h.levels[level];
}

int run_pcg(const void* handle, const lsamgdd_csr* g, const double* b, double tol, uint64_t maxit, double* x,
            int32_t memory, lsamgdd_report* report, lsamgdd_kernel_stats* stats, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    require_device();
    const Hierarchy& h = H(handle);
    SolveWs ws(h);
    Sell own_g, own_gt;
    const Sell* gs = &h.g0_sell;
    const Sell* gts = &h.g0t_sell;
    if (g) {
      DevCsr dg, dgt;
      if (g->memory == LSAMGDD_DEVICE) wait_for_caller(ws.s);
      csr_upload(dg, g, ws.s);
      csr_transpose(dg, dgt, ws.s);
      sell_from_csr(dg, own_g, ws.s);
      sell_from_csr(dgt, own_gt, ws.s);
      gs = &own_g;
      gts = &own_gt;
    }
    const int64_t n = gts->nr;
    PcgResult pr;
    with_vectors(ws.s, b, n, x, n, memory, [&](const double* db, double* dx) {
      pr = pcg(h, ws, *gs, *gts, db, dx, tol, maxit, stats);
    });
    fill_report(report, h, pr);
  });
}

}  // namespace

extern "C" {

void lsamgdd_params_default(lsamgdd_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->max_levels = 25;
  p->coarse_size = 400;
  p->aggregation_passes = 1;
  p->kappa = 50.0;
  p->must_keep = 5.0;
  p->n_ratios = 2;
  p->coarsening_ratios[0] = 2;
  p->coarsening_ratios[1] = 3;
  p->pre_sweeps = 1;
  p->post_sweeps = 1;
  p->level0_overlap = 1;
}

int32_t lsamgdd_abi_version(void) { return LSAMGDD_B200_ABI_VERSION; }

int32_t lsamgdd_device_available(void) { return device_ok() ? 1 : 0; }

int lsamgdd_setup(const lsamgdd_csr* g0, const lsamgdd_params* params, void** out, char* err, size_t errlen) {
  *out = nullptr;
  return guarded(err, errlen, [&] {
    lsamgdd_params p;
    if (params)
      p = *params;
    else
      lsamgdd_params_default(&p);
    lsb::validate_setup(g0, &p);  // host-side InputError contract first (hierarchy.hpp:107-117)
    require_device();
    if (g0->memory == LSAMGDD_DEVICE) {  // setup reads the factor on its own stream
      LSB_CUDA(cudaSetDevice(p.device));
      if (t_has_caller_stream)
        LSB_CUDA(cudaStreamSynchronize(t_caller_stream));
      else
        LSB_CUDA(cudaDeviceSynchronize());
    }
    *out = lsb::setup(g0, &p);
  });
}

int lsamgdd_set_caller_stream(void* stream, int32_t enable) {
  t_caller_stream = static_cast<cudaStream_t>(stream);
  t_has_caller_stream = enable != 0;
  return LSAMGDD_OK;
}

int lsamgdd_destroy(void* handle) {
  delete static_cast<Hierarchy*>(handle);
  return LSAMGDD_OK;
}

int lsamgdd_num_levels(const void* handle, int64_t* out) {
  return guarded(nullptr, 0, [&] { *out = static_cast<int64_t>(H(handle).levels.size()); });
}

int lsamgdd_get_level_summary(const void* handle, int64_t level, lsamgdd_level_summary* out) {
  return guarded(nullptr, 0, [&] {
    const Hierarchy& h = H(handle);
    if (level < 0 || level >= static_cast<int64_t>(h.summary.size())) raise(LSAMGDD_ERR_INDEX, "summary level out of range");
    *out = h.summary[level];
  });
}

int lsamgdd_operator_complexity(const void* handle, double* out) {
  return guarded(nullptr, 0, [&] { *out = operator_complexity(H(handle)); });
}

int lsamgdd_vcycle(const void* handle, int64_t level, const double* r, double* e, int32_t memory, char* err,
                   size_t errlen) {
  return guarded(err, errlen, [&] {
    require_device();
    const Hierarchy& h = H(handle);
    const Level& L = level_of(h, level);
    SolveWs ws(h);
    const int64_t n = L.A.nr;
    with_vectors(ws.s, r, n, e, n, memory, [&](const double* dr, double* de) { vcycle(h, ws, level, dr, de); });
  });
}

int lsamgdd_schwarz_apply(const void* handle, int64_t level, int32_t mode, const double* r, double* e, int32_t memory,
                          char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    require_device();
    const Hierarchy& h = H(handle);
    const Level& L = level_of(h, level);
    if (!L.has_interp) raise(LSAMGDD_ERR_INDEX, "schwarz: level has no smoother");
    if (mode != LSAMGDD_RAS && mode != LSAMGDD_RAST)
      raise(LSAMGDD_ERR_INPUT, "schwarz: only RAS and RAS-T are built on the device (ASM is out of scope)");
    SolveWs ws(h);
    const int64_t n = L.A.nr;
    with_vectors(ws.s, r, n, e, n, memory, [&](const double* dr, double* de) {
      SchwarzView sv = L.schwarz_view();
      sv.rast_tmp = ws.rast_tmp[level].get();
      if (mode == LSAMGDD_RAS) {
        schwarz_ras(sv, dr, de, false, ws.s);
      } else {
        LSB_CUDA(cudaMemsetAsync(de, 0, n * 8, ws.s));
        schwarz_rast(sv, L.sm.color_off, dr, de, ws.s);
      }
    });
  });
}

int lsamgdd_pcg(const void* handle, const lsamgdd_csr* g, const double* b, double tol, uint64_t maxit, double* x,
                int32_t memory, lsamgdd_report* report, char* err, size_t errlen) {
  return run_pcg(handle, g, b, tol, maxit, x, memory, report, nullptr, err, errlen);
}

int lsamgdd_profile_pcg(const void* handle, const double* b, double tol, uint64_t maxit, double* x, int32_t memory,
                        lsamgdd_report* report, lsamgdd_kernel_stats* stats, char* err, size_t errlen) {
  return run_pcg(handle, nullptr, b, tol, maxit, x, memory, report, stats, err, errlen);
}

int lsamgdd_level_spmv(const void* handle, int64_t level, int32_t what, int32_t transpose, const double* x, double* y,
                       int32_t memory, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    require_device();
    const Hierarchy& h = H(handle);
    const Level& L = level_of(h, level);
    SolveWs ws(h);
    if (what == 2) {
      if (!L.has_interp) raise(LSAMGDD_ERR_INDEX, "spmv: level has no interpolation");
      const InterpView iv = L.interp_view();
      const int64_t nin = transpose ? iv.n_fine : iv.n_coarse;
      const int64_t nout = transpose ? iv.n_coarse : iv.n_fine;
      with_vectors(ws.s, x, nin, y, nout, memory, [&](const double* dx, double* dy) {
        if (transpose) {
          restrict_pt(iv, dx, dy, ws.s, /*exact=*/true);
        } else {
          LSB_CUDA(cudaMemsetAsync(dy, 0, nout * 8, ws.s));
          prolong_add(iv, dx, dy, ws.s, /*exact=*/true);
        }
      });
      return;
    }
    if (what != 0 && what != 1) raise(LSAMGDD_ERR_INPUT, "spmv: what must be 0 (A), 1 (G) or 2 (P)");
    const DevCsr& m = what == 0 ? L.A : L.G;
    Sell own;
    const Sell* sp = nullptr;
    if (!transpose) {
      if (what == 0 && L.has_interp) sp = &L.A_sell;
      if (what == 1 && level == 0) sp = &h.g0_sell;
      if (!sp) {
        sell_from_csr(m, own, ws.s);
        sp = &own;
      }
    } else {
      if (what == 1 && level == 0) {
        sp = &h.g0t_sell;
      } else {
        DevCsr t;
        csr_transpose(m, t, ws.s);
        sell_from_csr(t, own, ws.s);
        sp = &own;
      }
    }
    const int64_t nin = sp->nc, nout = sp->nr;
    with_vectors(ws.s, x, nin, y, nout, memory, [&](const double* dx, double* dy) { sell_spmv(*sp, dx, dy, nullptr, ws.s); });
  });
}

// ---- standalone sparse kernels on caller matrices (sparse.hpp:110-204) ----------

namespace {
struct OwnStream {
  cudaStream_t s = nullptr;
  OwnStream() { LSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~OwnStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};
struct MatrixHandle {
  DevCsr m;
  Sell sell, sell_t;  // SpMV forms, built on first use
  bool has_sell = false, has_sell_t = false;
  std::mutex mu;
  cudaStream_t s = nullptr;
  ~MatrixHandle() {
    if (s) {
      cudaStreamSynchronize(s);
      sell = Sell();
      sell_t = Sell();
      m = DevCsr();
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};
void check_csr(const lsamgdd_csr* a, const char* who) {
  if (!a || a->n_rows < 0 || a->n_cols < 0 || a->nnz < 0 || (a->nnz > 0 && (!a->col_indices || !a->values)) ||
      !a->row_offsets)
    raise(LSAMGDD_ERR_INPUT, std::string(who) + ": malformed CSR argument");
}
}  // namespace

int lsamgdd_spmv(const lsamgdd_csr* a, int32_t transpose, const double* x, double* y, int32_t memory, char* err,
                 size_t errlen) {
  return guarded(err, errlen, [&] {
    check_csr(a, "spmv");
    require_device();
    OwnStream st;
    if (a->memory == LSAMGDD_DEVICE) wait_for_caller(st.s);
    DevCsr d;
    csr_upload(d, a, st.s);
    Sell sell;
    if (transpose) {
      DevCsr t;
      csr_transpose(d, t, st.s);
      sell_from_csr(t, sell, st.s);
    } else {
      sell_from_csr(d, sell, st.s);
    }
    with_vectors(st.s, x, sell.nc, y, sell.nr, memory,
                 [&](const double* dx, double* dy) { sell_spmv(sell, dx, dy, nullptr, st.s); });
  });
}

int lsamgdd_spgemm(const lsamgdd_csr* a, const lsamgdd_csr* b, void** out_matrix, char* err, size_t errlen) {
  if (out_matrix) *out_matrix = nullptr;
  return guarded(err, errlen, [&] {
    check_csr(a, "spgemm");
    check_csr(b, "spgemm");
    if (!out_matrix) raise(LSAMGDD_ERR_INPUT, "spgemm: null output");
    if (a->n_cols != b->n_rows)  // sparse.hpp:169-171
      raise(LSAMGDD_ERR_DIM, "spgemm: inner dimensions " + std::to_string(a->n_cols) + " and " +
                                 std::to_string(b->n_rows) + " differ");
    require_device();
    auto h = std::make_unique<MatrixHandle>();
    LSB_CUDA(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    if (a->memory == LSAMGDD_DEVICE || b->memory == LSAMGDD_DEVICE) wait_for_caller(h->s);
    DevCsr da, db;
    csr_upload(da, a, h->s);
    csr_upload(db, b, h->s);
    csr_spgemm_symbolic(da, db, h->m, h->s);
    LSB_CUDA(cudaStreamSynchronize(h->s));
    *out_matrix = h.release();
  });
}

int lsamgdd_transpose(const lsamgdd_csr* a, void** out_matrix, char* err, size_t errlen) {
  if (out_matrix) *out_matrix = nullptr;
  return guarded(err, errlen, [&] {
    check_csr(a, "transpose");
    if (!out_matrix) raise(LSAMGDD_ERR_INPUT, "transpose: null output");
    require_device();
    auto h = std::make_unique<MatrixHandle>();
    LSB_CUDA(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    if (a->memory == LSAMGDD_DEVICE) wait_for_caller(h->s);
    DevCsr da;
    csr_upload(da, a, h->s);
    csr_transpose(da, h->m, h->s);
    LSB_CUDA(cudaStreamSynchronize(h->s));
    *out_matrix = h.release();
  });
}

int lsamgdd_build_smoother(const lsamgdd_csr* a, int64_t n_aggregates, const int64_t* omega_offsets,
                           const int64_t* omega, const int64_t* gamma_offsets, const int64_t* gamma,
                           const int64_t* colors, void** out_smoother, char* err, size_t errlen) {
  if (out_smoother) *out_smoother = nullptr;
  return guarded(err, errlen, [&] {
    check_csr(a, "build_smoother");
    if (!out_smoother) raise(LSAMGDD_ERR_INPUT, "build_smoother: null output");
    require_device();
    if (a->memory == LSAMGDD_DEVICE) LSB_CUDA(cudaDeviceSynchronize());
    *out_smoother = make_smoother(a, n_aggregates, omega_offsets, omega, gamma_offsets, gamma, colors);
  });
}

int lsamgdd_smoother_apply(const void* smoother, int32_t mode, const double* r, double* e, int32_t memory, char* err,
                           size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!smoother) raise(LSAMGDD_ERR_INPUT, "null smoother handle");
    if (mode != LSAMGDD_RAS && mode != LSAMGDD_RAST)
      raise(LSAMGDD_ERR_INPUT, "schwarz apply: this path implements RAS and RAST (ASM is a study mode)");
    require_device();
    const StandaloneSmoother& sm = *static_cast<const StandaloneSmoother*>(smoother);
    with_vectors(sm.s, r, sm.n, e, sm.n, memory, [&](const double* dr, double* de) { smoother_apply(sm, mode, dr, de); });
  });
}

int lsamgdd_smoother_destroy(void* smoother) {
  delete static_cast<StandaloneSmoother*>(smoother);
  return LSAMGDD_OK;
}

int lsamgdd_matrix_create(const lsamgdd_csr* a, void** out_matrix, char* err, size_t errlen) {
  if (out_matrix) *out_matrix = nullptr;
  return guarded(err, errlen, [&] {
    check_csr(a, "matrix_create");
    if (!out_matrix) raise(LSAMGDD_ERR_INPUT, "matrix_create: null output");
    require_device();
    auto h = std::make_unique<MatrixHandle>();
    LSB_CUDA(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    if (a->memory == LSAMGDD_DEVICE) wait_for_caller(h->s);
    csr_upload(h->m, a, h->s);
    LSB_CUDA(cudaStreamSynchronize(h->s));
    *out_matrix = h.release();
  });
}

int lsamgdd_matrix_spmv(void* matrix, int32_t transpose, const double* x, double* y, int32_t memory, char* err,
                        size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!matrix) raise(LSAMGDD_ERR_INPUT, "null matrix handle");
    require_device();
    MatrixHandle& h = *static_cast<MatrixHandle*>(matrix);
    std::lock_guard<std::mutex> lock(h.mu);  // one stream per handle
    if (!transpose && !h.has_sell) {
      sell_from_csr(h.m, h.sell, h.s);
      h.has_sell = true;
    }
    if (transpose && !h.has_sell_t) {
      DevCsr t;
      csr_transpose(h.m, t, h.s);
      sell_from_csr(t, h.sell_t, h.s);
      h.has_sell_t = true;
    }
    const Sell& sp = transpose ? h.sell_t : h.sell;
    with_vectors(h.s, x, sp.nc, y, sp.nr, memory, [&](const double* dx, double* dy) { sell_spmv(sp, dx, dy, nullptr, h.s); });
  });
}

int lsamgdd_matrix_export(const void* matrix, int64_t sizes[3], int64_t* offsets, int64_t* cols, double* vals) {
  return guarded(nullptr, 0, [&] {
    if (!matrix) raise(LSAMGDD_ERR_INPUT, "null matrix handle");
    const MatrixHandle& h = *static_cast<const MatrixHandle*>(matrix);
    sizes[0] = h.m.nr;
    sizes[1] = h.m.nc;
    sizes[2] = h.m.nnz;
    if (!offsets && !cols && !vals) return;
    std::vector<int64_t> off, col;
    std::vector<double> val;
    csr_download(h.m, off, col, val, h.s);
    if (offsets) std::copy(off.begin(), off.end(), offsets);
    if (cols) std::copy(col.begin(), col.end(), cols);
    if (vals) std::copy(val.begin(), val.end(), vals);
  });
}

int lsamgdd_matrix_destroy(void* matrix) {
  delete static_cast<MatrixHandle*>(matrix);
  return LSAMGDD_OK;
}

int lsamgdd_level_export(const void* handle, int64_t level, int32_t what, int64_t sizes[3], int64_t* idx0, int64_t* idx1,
                         double* vals) {
  return guarded(nullptr, 0, [&] {
    const Hierarchy& h = H(handle);
    const Level& L = level_of(h, level);
    std::lock_guard<std::mutex> lock(h.mu);
    sizes[0] = sizes[1] = sizes[2] = 0;
    cudaStream_t s = h.stream;
    if (what == LSAMGDD_EXPORT_A || what == LSAMGDD_EXPORT_G || what == LSAMGDD_EXPORT_P) {
      if (what == LSAMGDD_EXPORT_P && !L.has_interp) raise(LSAMGDD_ERR_INDEX, "export: level has no interpolation");
      const DevCsr& m = what == LSAMGDD_EXPORT_A ? L.A : what == LSAMGDD_EXPORT_G ? L.G : L.P;
      sizes[0] = m.nr;
      sizes[1] = m.nc;
      sizes[2] = m.nnz;
      if (idx0 || idx1 || vals) {
        std::vector<int64_t> off, col;
        std::vector<double> val;
        csr_download(m, off, col, val, s);
        if (idx0) std::memcpy(idx0, off.data(), off.size() * 8);
        if (idx1) std::memcpy(idx1, col.data(), col.size() * 8);
        if (vals) std::memcpy(vals, val.data(), val.size() * 8);
      }
      return;
    }
    if (!L.has_interp) raise(LSAMGDD_ERR_INDEX, "export: level has no topology");
    const int64_t na = static_cast<int64_t>(L.h_omega_off.size()) - 1;
    switch (what) {
      case LSAMGDD_EXPORT_PARTITION:
        sizes[0] = static_cast<int64_t>(L.h_omega.size());
        sizes[1] = na;
        if (idx0)
          for (int64_t i = 0; i < na; ++i)
            for (int32_t p = L.h_omega_off[i]; p < L.h_omega_off[i + 1]; ++p) idx0[L.h_omega[p]] = i;
        return;
      case LSAMGDD_EXPORT_GAMMA:
        sizes[0] = na;
        sizes[1] = static_cast<int64_t>(L.h_gamma.size());
        if (idx0)
          for (int64_t i = 0; i <= na; ++i) idx0[i] = L.h_gamma_off[i];
        if (idx1)
          for (size_t k = 0; k < L.h_gamma.size(); ++k) idx1[k] = L.h_gamma[k];
        return;
      case LSAMGDD_EXPORT_COLORS:
        sizes[0] = na;
        sizes[1] = L.n_colors;
        if (idx0)
          for (int64_t i = 0; i < na; ++i) idx0[i] = L.colors[i];
        return;
      case LSAMGDD_EXPORT_SPECTRA: {
        if (L.ip.spectra.empty()) raise(LSAMGDD_ERR_INDEX, "export: spectra were not kept (params.keep_spectra)");
        sizes[0] = na;
        int64_t tot = 0;
        for (const auto& v : L.ip.spectra) tot += static_cast<int64_t>(v.size());
        sizes[1] = tot;
        int64_t o = 0;
        for (int64_t i = 0; i < na; ++i) {
          if (idx0) idx0[i] = o;
          for (double v : L.ip.spectra[i]) {
            if (vals) vals[o] = v;
            ++o;
          }
        }
        if (idx0) idx0[na] = o;
        return;
      }
      case LSAMGDD_EXPORT_MULTIPLICITY: {
        sizes[0] = L.G.nr;
        sizes[1] = L.n_mult;
        if (idx0) {
          const auto m = L.mult.download(s);
          for (size_t j = 0; j < m.size(); ++j) idx0[j] = m[j];
        }
        return;
      }
      default:
        raise(LSAMGDD_ERR_INPUT, "export: unknown item");
    }
  });
}

int lsamgdd_setup_timings(const void* handle, const char** names, double* ms, int64_t n, int64_t* count) {
  return guarded(nullptr, 0, [&] {
    const Hierarchy& h = H(handle);
    *count = static_cast<int64_t>(h.timings.size());
    for (int64_t i = 0; i < n && i < *count; ++i) {
      names[i] = h.timings[i].name.c_str();
      ms[i] = h.timings[i].ms;
    }
  });
}

int lsamgdd_dense_sym_eig(int64_t n, const double* a, double* values, double* vectors, int32_t path, char* err,
                          size_t errlen) {
  return guarded(err, errlen, [&] {
    require_device();
    cudaStream_t s;
    LSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int st = dense_sym_eig(n, a, values, vectors, path, s);
    cudaStreamDestroy(s);
    if (st == 1) raise(LSAMGDD_ERR_EIG, "sym_eig: Jacobi iteration did not converge");
    if (st == 2) raise(LSAMGDD_ERR_EIG, "sym_eig: non-finite eigenvalue");
  });
}

int64_t lsamgdd_launch_count(void) { return launch_counter(); }

int lsamgdd_trim_memory(int32_t device) {
  return guarded(nullptr, 0, [&] {
    LSB_CUDA(cudaSetDevice(device));
    trim_device_pool(device);
  });
}

int lsamgdd_generate_stencil_rows(const int64_t grid[3], int32_t rows_per_node, int32_t max_entries, const int32_t* offsets,
                                  const double* coefs, int32_t device, void** out_owner, lsamgdd_csr* out_csr, char* err,
                                  size_t errlen) {
  if (out_owner) *out_owner = nullptr;
  return guarded(err, errlen, [&] {
    if (!out_owner || !out_csr) raise(LSAMGDD_ERR_INPUT, "generate_stencil_rows: null output argument");
    require_device();
    GeneratedCsr* g = generate_stencil_rows(grid, rows_per_node, max_entries, offsets, coefs, device);
    generated_view(g, out_csr);
    *out_owner = g;
  });
}

int lsamgdd_generated_export(const void* owner, int64_t* offsets, int64_t* cols, double* values, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (!owner) raise(LSAMGDD_ERR_INPUT, "null generated-matrix handle");
    generated_export(static_cast<const GeneratedCsr*>(owner), offsets, cols, values);
  });
}

int lsamgdd_generated_destroy(void* owner) {
  generated_destroy(static_cast<GeneratedCsr*>(owner));
  return LSAMGDD_OK;
}

void lsamgdd_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(gen);
}

}  // extern "C"
