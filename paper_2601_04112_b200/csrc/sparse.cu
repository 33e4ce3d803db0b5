// sparse.cu — ordered sparse kernels (sparse.hpp on the GPU).
//
// Bit-exactness: every FP64 sum here runs in the reference's order with
// separate multiply and add (the library is built with --fmad=false), so
// products and sums round exactly as in the reference's no-FMA Release build.
#include <cub/cub.cuh>

#include <mutex>

#include <algorithm>

#include "sparse.cuh"

namespace lsb {

namespace {

constexpr int kThreads = 256;

template <class T>
void cub_scan_exclusive(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  LSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  DBuf<unsigned char> t(tmp, s);
  LSB_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, n, s));
}

template <class T>
void cub_scan_inclusive(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  LSB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, n, s));
  DBuf<unsigned char> t(tmp, s);
  LSB_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, in, out, n, s));
}

int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (uint64_t(1) << b) <= v) ++b;
  return b;
}

__global__ void k_i64_to_i32(const int64_t* in, int32_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(in[i]);
}

__global__ void k_i32_to_i64(const int32_t* in, int64_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

// row id of every stored entry
__global__ void k_row_ids(const int64_t* off, int64_t nr, int32_t* rows) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nr; i += int64_t(gridDim.x) * blockDim.x)
    for (int64_t k = off[i]; k < off[i + 1]; ++k) rows[k] = static_cast<int32_t>(i);
}

__global__ void k_iota(int64_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) v[i] = i;
}

__global__ void k_count_cols(const int32_t* col, int64_t nnz, int64_t* cnt) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[col[k] + 1]), 1ull);
}

__global__ void k_transpose_gather(const int64_t* perm, const int32_t* rows, const double* val, int64_t nnz,
                                   int32_t* tcol, double* tval) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < nnz; p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = perm[p];
    tcol[p] = rows[k];
    tval[p] = val[k];
  }
}

int grid_for(int64_t n, int threads = kThreads) {
  const int64_t cap = int64_t(sm_count()) * 16;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap)));
}

// ---- ESC SpGEMM -------------------------------------------------------------

// candidates contributed by entry ka of a: nnz of b's row a.col[ka]
__global__ void k_entry_counts(const int32_t* acol, int64_t annz, const int64_t* boff, int64_t* cnt) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < annz; k += int64_t(gridDim.x) * blockDim.x) {
    const int32_t c = acol[k];
    cnt[k] = boff[c + 1] - boff[c];
  }
}

// expand rows [r0, r1): key = (row - r0)·nc + col, value = a·b, in (row, ka, kb) order
__global__ void k_expand(const int64_t* aoff, const int32_t* acol, const double* aval, const int64_t* boff,
                         const int32_t* bcol, const double* bval, const int64_t* epos, int64_t r0, int64_t r1,
                         int64_t base, uint64_t nc, uint64_t* keys, double* vals) {
  const int64_t k0 = aoff[r0], k1 = aoff[r1];
  for (int64_t ka = k0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ka < k1; ka += int64_t(gridDim.x) * blockDim.x) {
    // row of entry ka: binary search in aoff[r0..r1]
    int64_t lo = r0, hi = r1 - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (aoff[mid] <= ka)
        lo = mid;
      else
        hi = mid - 1;
    }
    const uint64_t lrow = static_cast<uint64_t>(lo - r0);
    const double av = aval[ka];
    const int32_t kk = acol[ka];
    int64_t pos = epos[ka] - base;
    for (int64_t kb = boff[kk]; kb < boff[kk + 1]; ++kb, ++pos) {
      keys[pos] = lrow * nc + static_cast<uint64_t>(bcol[kb]);
      vals[pos] = av * bval[kb];
    }
  }
}

__global__ void k_heads(const uint64_t* keys, int64_t n, int32_t* head) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x)
    head[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

// run u spans [start_u, start_{u+1}); sum in order (sparse.hpp:189 acc[j] += ...)
__global__ void k_run_sums(const uint64_t* keys, const double* vals, const int32_t* head, const int32_t* uidx,
                           int64_t n, uint64_t nc, int64_t r0, int64_t out_base, int32_t* ocol, double* oval,
                           int64_t* row_cnt) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    if (!head[p]) continue;
    const uint64_t key = keys[p];
    double acc = 0.0;
    int64_t q = p;
    do {
      acc += vals[q];
      ++q;
    } while (q < n && keys[q] == key);
    const int64_t u = out_base + uidx[p];
    ocol[u] = static_cast<int32_t>(key % nc);
    oval[u] = acc;
    atomicAdd(reinterpret_cast<unsigned long long*>(&row_cnt[r0 + static_cast<int64_t>(key / nc) + 1]), 1ull);
  }
}

// ---- SELL ------------------------------------------------------------------

__global__ void k_row_len(const int64_t* off, int64_t nr, int32_t* len) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nr; i += int64_t(gridDim.x) * blockDim.x)
    len[i] = static_cast<int32_t>(off[i + 1] - off[i]);
}

__global__ void k_slice_width(const int32_t* len, int64_t nr, int64_t ns, int64_t* w) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < ns; s += int64_t(gridDim.x) * blockDim.x) {
    int32_t m = 0;
    for (int64_t i = s * 32; i < min(nr, s * 32 + 32); ++i) m = max(m, len[i]);
    w[s] = int64_t(m) * 32;
  }
}

__global__ void k_sell_fill(const int64_t* off, const int32_t* col, const double* val, int64_t nr,
                            const int64_t* soff, int32_t* scol, double* sval) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nr; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = i >> 5;
    const int lane = static_cast<int>(i & 31);
    const int64_t base = soff[s];
    const int64_t w = (soff[s + 1] - base) >> 5;
    const int64_t len = off[i + 1] - off[i];
    for (int64_t k = 0; k < w; ++k) {
      const int64_t dst = base + k * 32 + lane;
      if (k < len) {
        scol[dst] = col[off[i] + k];
        sval[dst] = val[off[i] + k];
      } else {
        scol[dst] = -1;
        sval[dst] = 0.0;
      }
    }
  }
}

// the row slots past the last row of a partial final slice
__global__ void k_sell_pad_tail(int64_t nr, const int64_t* soff, int64_t ns, int32_t* scol, double* sval) {
  const int64_t s = ns - 1;
  const int64_t base = soff[s];
  const int64_t w = (soff[s + 1] - base) >> 5;
  for (int64_t i = nr + threadIdx.x; i < (s + 1) * 32; i += blockDim.x) {
    const int lane = static_cast<int>(i & 31);
    for (int64_t k = 0; k < w; ++k) {
      scol[base + k * 32 + lane] = -1;
      sval[base + k * 32 + lane] = 0.0;
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_sell_spmv(const int64_t* __restrict__ soff, const int32_t* __restrict__ len,
                                                   const int32_t* __restrict__ col, const double* __restrict__ val,
                                                   int64_t nr, const double* __restrict__ x, double* __restrict__ y,
                                                   const double* __restrict__ r) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nr; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t base = soff[i >> 5] + (i & 31);
    const int n = len[i];
    double s = 0.0;
    for (int k = 0; k < n; ++k) {
      const int64_t e = base + int64_t(k) * 32;
      s += __ldcs(&val[e]) * __ldg(&x[__ldcs(&col[e])]);
    }
    if (MODE == 0)
      y[i] = s;
    else
      y[i] = r[i] - s;  // r + (-1.0)·(A e)   hierarchy.hpp:213-214
  }
}

// CSR, one warp per row (long rows of the coarse levels): lanes stride the
// row with two accumulators, fixed xor-tree reduction (deterministic).
template <int MODE>
__global__ void __launch_bounds__(256) k_csr_spmv_warp(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                                                       const double* __restrict__ val, int64_t nr,
                                                       const double* __restrict__ x, double* __restrict__ y,
                                                       const double* __restrict__ r) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < nr; i += warps) {
    const int64_t b = off[i], e = off[i + 1];
    double s0 = 0.0, s1 = 0.0;
    int64_t k = b + lane;
    for (; k + 32 < e; k += 64) {
      s0 += __ldcs(&val[k]) * __ldg(&x[__ldcs(&col[k])]);
      s1 += __ldcs(&val[k + 32]) * __ldg(&x[__ldcs(&col[k + 32])]);
    }
    if (k < e) s0 += __ldcs(&val[k]) * __ldg(&x[__ldcs(&col[k])]);
    double sum = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) y[i] = MODE == 0 ? sum : r[i] - sum;
  }
}

}  // namespace

void csr_spmv_warp(const DevCsr& a, const double* x, double* y, const double* r, cudaStream_t s) {
  if (a.nr == 0) return;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(a.nr, 8), int64_t(sm_count()) * 16)));
  if (r)
    k_csr_spmv_warp<1><<<grid, 256, 0, s>>>(a.off.get(), a.col.get(), a.val.get(), a.nr, x, y, r);
  else
    k_csr_spmv_warp<0><<<grid, 256, 0, s>>>(a.off.get(), a.col.get(), a.val.get(), a.nr, x, y, r);
  LSB_LAUNCH();
}

int sm_count() {
  static std::atomic<int> cache[64];  // per device ordinal, 0 = not queried yet
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

namespace {
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};
}  // namespace

cudaMemPool_t device_pool() {
  int dev = 0;
  LSB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) raise(LSAMGDD_ERR_CUDA, "device ordinal out of range");
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    LSB_CUDA(cudaMemPoolCreate(&pool, &props));
    uint64_t keep = UINT64_MAX;
    LSB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    g_pools[dev] = pool;
  }
  return g_pools[dev];
}

void trim_device_pool(int device) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (device >= 0 && device < 64 && g_pools[device]) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(g_pools[device], 0);
  }
}

bool first_on_device(std::atomic<uint64_t>& flags) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const uint64_t bit = uint64_t(1) << dev;
  return (flags.fetch_or(bit, std::memory_order_acq_rel) & bit) == 0;
}

void csr_upload(DevCsr& d, const lsamgdd_csr* h, cudaStream_t s) {
  d.nr = h->n_rows;
  d.nc = h->n_cols;
  d.nnz = h->nnz;
  if (h->memory == LSAMGDD_DEVICE) {
    d.off.alloc(d.nr + 1, s);
    LSB_CUDA(cudaMemcpyAsync(d.off.get(), h->row_offsets, (d.nr + 1) * 8, cudaMemcpyDeviceToDevice, s));
    d.col.alloc(d.nnz, s);
    if (d.nnz) k_i64_to_i32<<<grid_for(d.nnz), kThreads, 0, s>>>(h->col_indices, d.col.get(), d.nnz);
    LSB_LAUNCH();
    d.val.alloc(d.nnz, s);
    LSB_CUDA(cudaMemcpyAsync(d.val.get(), h->values, d.nnz * 8, cudaMemcpyDeviceToDevice, s));
    return;
  }
  d.off.upload(h->row_offsets, d.nr + 1, s);
  DBuf<int64_t> c64;
  c64.upload(h->col_indices, d.nnz, s);
  d.col.alloc(d.nnz, s);
  if (d.nnz) k_i64_to_i32<<<grid_for(d.nnz), kThreads, 0, s>>>(c64.get(), d.col.get(), d.nnz);
  LSB_LAUNCH();
  d.val.upload(h->values, d.nnz, s);
}

void csr_download(const DevCsr& d, std::vector<int64_t>& off, std::vector<int64_t>& col, std::vector<double>& val,
                  cudaStream_t s) {
  off = d.off.download(s);
  DBuf<int64_t> c64(d.nnz, s);
  if (d.nnz) k_i32_to_i64<<<grid_for(d.nnz), kThreads, 0, s>>>(d.col.get(), c64.get(), d.nnz);
  LSB_LAUNCH();
  col = c64.download(s);
  val = d.val.download(s);
}

void csr_transpose(const DevCsr& a, DevCsr& t, cudaStream_t s) {
  t.nr = a.nc;
  t.nc = a.nr;
  t.nnz = a.nnz;
  t.off.alloc(a.nc + 1, s);
  t.off.zero(s);
  t.col.alloc(a.nnz, s);
  t.val.alloc(a.nnz, s);
  if (a.nnz == 0) return;
  DBuf<int64_t> cnt(a.nc + 1, s);
  cnt.zero(s);
  k_count_cols<<<grid_for(a.nnz), kThreads, 0, s>>>(a.col.get(), a.nnz, cnt.get());
  LSB_LAUNCH();
  cub_scan_inclusive(cnt.get(), t.off.get(), a.nc + 1, s);
  DBuf<int32_t> rows(a.nnz, s);
  k_row_ids<<<grid_for(a.nr), kThreads, 0, s>>>(a.off.get(), a.nr, rows.get());
  LSB_LAUNCH();
  DBuf<int64_t> idx(a.nnz, s), perm(a.nnz, s);
  DBuf<int32_t> kout(a.nnz, s);
  k_iota<<<grid_for(a.nnz), kThreads, 0, s>>>(idx.get(), a.nnz);
  LSB_LAUNCH();
  size_t tmp = 0;
  const int eb = bits_for(static_cast<uint64_t>(a.nc));
  LSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, a.col.get(), kout.get(), idx.get(), perm.get(), a.nnz, 0, eb, s));
  DBuf<unsigned char> tb(tmp, s);
  LSB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), tmp, a.col.get(), kout.get(), idx.get(), perm.get(), a.nnz, 0, eb, s));
  k_transpose_gather<<<grid_for(a.nnz), kThreads, 0, s>>>(perm.get(), rows.get(), a.val.get(), a.nnz, t.col.get(),
                                                           t.val.get());
  LSB_LAUNCH();
}

void csr_spgemm_symbolic(const DevCsr& a, const DevCsr& b, DevCsr& c, cudaStream_t s, int64_t budget) {
  if (a.nc != b.nr)
    raise(LSAMGDD_ERR_DIM, "spgemm: inner dimensions " + std::to_string(a.nc) + " and " + std::to_string(b.nr) +
                               " do not match");
  c.nr = a.nr;
  c.nc = b.nc;
  DBuf<int64_t> row_cnt(a.nr + 1, s);
  row_cnt.zero(s);
  // candidate position of every a-entry
  DBuf<int64_t> epos(a.nnz + 1, s);
  {
    DBuf<int64_t> ecnt(a.nnz + 1, s);
    ecnt.zero(s);
    if (a.nnz) k_entry_counts<<<grid_for(a.nnz), kThreads, 0, s>>>(a.col.get(), a.nnz, b.off.get(), ecnt.get());
    LSB_LAUNCH();
    cub_scan_exclusive(ecnt.get(), epos.get(), a.nnz + 1, s);
  }
  std::vector<int64_t> hoff = a.off.download(s);
  std::vector<int64_t> hepos = epos.download(s);
  // candidates at each row start
  auto cand_at_row = [&](int64_t r) { return hepos[hoff[r]]; };
  struct Part {
    DBuf<int32_t> col;
    DBuf<double> val;
    int64_t n;
  };
  std::vector<Part> parts;
  int64_t total = 0;
  int64_t r0 = 0;
  const uint64_t nc = static_cast<uint64_t>(std::max<int64_t>(b.nc, 1));
  while (r0 < a.nr) {
    // grow the chunk while it fits the budget (at least one row)
    int64_t lo = r0 + 1, hi = a.nr;
    const int64_t c0 = cand_at_row(r0);
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (cand_at_row(mid) - c0 <= budget)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int64_t r1 = lo;
    const int64_t n = cand_at_row(r1) - c0;
    if (n > 0) {
      DBuf<uint64_t> k1(n, s), k2(n, s);
      DBuf<double> v1(n, s), v2(n, s);
      const int64_t aent = hoff[r1] - hoff[r0];
      k_expand<<<grid_for(aent), kThreads, 0, s>>>(a.off.get(), a.col.get(), a.val.get(), b.off.get(), b.col.get(),
                                                   b.val.get(), epos.get(), r0, r1, c0, nc, k1.get(), v1.get());
      LSB_LAUNCH();
      size_t tmp = 0;
      const int eb = bits_for(static_cast<uint64_t>(r1 - r0) * nc);
      LSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k1.get(), k2.get(), v1.get(), v2.get(), n, 0, eb, s));
      {
        DBuf<unsigned char> tb(tmp, s);
        LSB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), tmp, k1.get(), k2.get(), v1.get(), v2.get(), n, 0, eb, s));
      }
      k1.release();
      v1.release();
      DBuf<int32_t> head(n, s), uidx(n, s);
      k_heads<<<grid_for(n), kThreads, 0, s>>>(k2.get(), n, head.get());
      LSB_LAUNCH();
      cub_scan_exclusive(head.get(), uidx.get(), n, s);
      int32_t last_u = 0, last_h = 0;
      LSB_CUDA(cudaMemcpyAsync(&last_u, uidx.get() + n - 1, 4, cudaMemcpyDeviceToHost, s));
      LSB_CUDA(cudaMemcpyAsync(&last_h, head.get() + n - 1, 4, cudaMemcpyDeviceToHost, s));
      LSB_CUDA(cudaStreamSynchronize(s));
      const int64_t uniq = int64_t(last_u) + last_h;
      Part p;
      p.n = uniq;
      p.col.alloc(uniq, s);
      p.val.alloc(uniq, s);
      k_run_sums<<<grid_for(n), kThreads, 0, s>>>(k2.get(), v2.get(), head.get(), uidx.get(), n, nc, r0, 0,
                                                  p.col.get(), p.val.get(), row_cnt.get());
      LSB_LAUNCH();
      total += uniq;
      parts.push_back(std::move(p));
    }
    r0 = r1;
  }
  c.nnz = total;
  c.off.alloc(a.nr + 1, s);
  cub_scan_inclusive(row_cnt.get(), c.off.get(), a.nr + 1, s);
  if (parts.size() == 1) {
    c.col = std::move(parts[0].col);
    c.val = std::move(parts[0].val);
    return;
  }
  c.col.alloc(total, s);
  c.val.alloc(total, s);
  int64_t o = 0;
  for (auto& p : parts) {
    if (p.n) {
      LSB_CUDA(cudaMemcpyAsync(c.col.get() + o, p.col.get(), p.n * 4, cudaMemcpyDeviceToDevice, s));
      LSB_CUDA(cudaMemcpyAsync(c.val.get() + o, p.val.get(), p.n * 8, cudaMemcpyDeviceToDevice, s));
    }
    o += p.n;
  }
}

void sell_from_csr(const DevCsr& a, Sell& out, cudaStream_t s) {
  out.nr = a.nr;
  out.nc = a.nc;
  out.nnz = a.nnz;
  out.n_slices = ceil_div(a.nr, 32);
  out.row_len.alloc(a.nr, s);
  out.slice_off.alloc(out.n_slices + 1, s);
  if (a.nr == 0) {
    out.slice_off.zero(s);
    out.stored = 0;
    return;
  }
  k_row_len<<<grid_for(a.nr), kThreads, 0, s>>>(a.off.get(), a.nr, out.row_len.get());
  LSB_LAUNCH();
  DBuf<int64_t> w(out.n_slices + 1, s);
  w.zero(s);
  k_slice_width<<<grid_for(out.n_slices), kThreads, 0, s>>>(out.row_len.get(), a.nr, out.n_slices, w.get());
  LSB_LAUNCH();
  cub_scan_exclusive(w.get(), out.slice_off.get(), out.n_slices + 1, s);
  out.stored = read_scalar(out.slice_off.get() + out.n_slices, s);
  out.col.alloc(out.stored, s);
  out.val.alloc(out.stored, s);
  k_sell_fill<<<grid_for(a.nr), kThreads, 0, s>>>(a.off.get(), a.col.get(), a.val.get(), a.nr, out.slice_off.get(),
                                                  out.col.get(), out.val.get());
  LSB_LAUNCH();
  if (a.nr % 32) k_sell_pad_tail<<<1, 32, 0, s>>>(a.nr, out.slice_off.get(), out.n_slices, out.col.get(), out.val.get());
  LSB_LAUNCH();
}

void sell_spmv(const Sell& a, const double* x, double* y, const double* r, cudaStream_t s) {
  if (a.nr == 0) return;
  const int grid = grid_for(a.nr, 256);
  if (r)
    k_sell_spmv<1><<<grid, 256, 0, s>>>(a.slice_off.get(), a.row_len.get(), a.col.get(), a.val.get(), a.nr, x, y, r);
  else
    k_sell_spmv<0><<<grid, 256, 0, s>>>(a.slice_off.get(), a.row_len.get(), a.col.get(), a.val.get(), a.nr, x, y, r);
  LSB_LAUNCH();
}

}  // namespace lsb
