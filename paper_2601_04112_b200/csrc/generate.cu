// generate.cu — on-device generators of the constant-coefficient BASELINE
// factors: the least-squares factor G is written straight
// into HBM as CSR, so a caller that only needs the solve never ships the
// 243 MB (config 2) … 3.9 GB (config 3 at 4096²) factor over PCIe.
//
// A factor is described the way SURVEY.md Appendix A.1 builds configs 2, 3
// and 5: every grid node owns `rows_per_node` rows; a row is a short list of
// (offset, coefficient) pairs; a neighbour outside the grid is dropped
// (homogeneous Dirichlet closure, as in problems.hpp:84-104); an exact-zero
// coefficient is dropped (sparse.hpp:75-100 keeps no explicit zeros); the
// columns of a row ascend. Row r = rows_per_node·node + k, node = (z·ny + y)·nx + x.
#include <algorithm>
#include <cmath>
#include <memory>
#include <cub/cub.cuh>
#include <vector>

#include "common.cuh"
#include "sparse.cuh"

namespace lsb {

namespace {

constexpr int kGenMaxEntries = 8;
constexpr int kGenMaxRows = 8;

struct GenStencil {
  int rows, entries;
  int dx[kGenMaxRows][kGenMaxEntries], dy[kGenMaxRows][kGenMaxEntries], dz[kGenMaxRows][kGenMaxEntries];
  double coef[kGenMaxRows][kGenMaxEntries];  // 0.0: no entry
};

__device__ __forceinline__ bool gen_inside(int64_t x, int64_t y, int64_t z, int dx, int dy, int dz, int64_t nx, int64_t ny,
                                           int64_t nz) {
  const int64_t X = x + dx, Y = y + dy, Z = z + dz;
  return X >= 0 && X < nx && Y >= 0 && Y < ny && Z >= 0 && Z < nz;
}

// off[r + 1] = entries of row r; off[0] = 0
__global__ void __launch_bounds__(256) k_gen_count(GenStencil st, int64_t nx, int64_t ny, int64_t nz, int64_t* off) {
  const int64_t m = nx * ny * nz * st.rows;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t node = r / st.rows;
    const int k = static_cast<int>(r - node * st.rows);
    const int64_t x = node % nx, y = (node / nx) % ny, z = node / (nx * ny);
    int cnt = 0;
#pragma unroll
    for (int e = 0; e < kGenMaxEntries; ++e)
      if (e < st.entries && st.coef[k][e] != 0.0 && gen_inside(x, y, z, st.dx[k][e], st.dy[k][e], st.dz[k][e], nx, ny, nz))
        ++cnt;
    off[r + 1] = cnt;
    if (r == 0) off[0] = 0;
  }
}

__global__ void __launch_bounds__(256) k_gen_fill(GenStencil st, int64_t nx, int64_t ny, int64_t nz,
                                                  const int64_t* __restrict__ off, int64_t* __restrict__ col,
                                                  double* __restrict__ val) {
  const int64_t m = nx * ny * nz * st.rows;
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t node = r / st.rows;
    const int k = static_cast<int>(r - node * st.rows);
    const int64_t x = node % nx, y = (node / nx) % ny, z = node / (nx * ny);
    int64_t p = off[r];
#pragma unroll
    for (int e = 0; e < kGenMaxEntries; ++e)
      if (e < st.entries && st.coef[k][e] != 0.0 && gen_inside(x, y, z, st.dx[k][e], st.dy[k][e], st.dz[k][e], nx, ny, nz)) {
        col[p] = node + (int64_t(st.dz[k][e]) * ny + st.dy[k][e]) * nx + st.dx[k][e];
        val[p] = st.coef[k][e];
        ++p;
      }
  }
}

}  // namespace

struct GeneratedCsr {
  int device = 0;
  cudaStream_t s = nullptr;
  int64_t nr = 0, nc = 0, nnz = 0;
  DBuf<int64_t> off, col;
  DBuf<double> val;
  ~GeneratedCsr() {
    if (s) {
      cudaSetDevice(device);
      cudaStreamSynchronize(s);
      off = DBuf<int64_t>();
      col = DBuf<int64_t>();
      val = DBuf<double>();
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

GeneratedCsr* generate_stencil_rows(const int64_t grid[3], int32_t rows_per_node, int32_t max_entries, const int32_t* offsets,
                                    const double* coefs, int32_t device) {
  if (!grid || !offsets || !coefs) raise(LSAMGDD_ERR_INPUT, "generate_stencil_rows: null argument");
  const int64_t nx = grid[0], ny = grid[1], nz = grid[2];
  if (nx < 1 || ny < 1 || nz < 1) raise(LSAMGDD_ERR_INPUT, "generate_stencil_rows: grid extents must be positive");
  if (rows_per_node < 1 || rows_per_node > kGenMaxRows || max_entries < 1 || max_entries > kGenMaxEntries)
    raise(LSAMGDD_ERR_INPUT, "generate_stencil_rows: at most 8 rows per node and 8 entries per row");
  const int64_t n = nx * ny * nz;
  if (n >= (int64_t(1) << 31) / rows_per_node) raise(LSAMGDD_ERR_SIZE, "generate_stencil_rows: dimensions must stay below 2^31");
  GenStencil st = {};
  st.rows = rows_per_node;
  st.entries = max_entries;
  for (int k = 0; k < rows_per_node; ++k) {
    // ascending linear offset = ascending column for every node that keeps the entry
    struct Ent {
      int64_t lin;
      int dx, dy, dz;
      double c;
    };
    std::vector<Ent> ents;
    for (int e = 0; e < max_entries; ++e) {
      const int32_t* o = offsets + (int64_t(k) * max_entries + e) * 3;
      const double c = coefs[int64_t(k) * max_entries + e];
      if (!std::isfinite(c)) raise(LSAMGDD_ERR_INPUT, "generate_stencil_rows: coefficients must be finite");
      if (c == 0.0) continue;
      if (std::abs(o[0]) >= nx || std::abs(o[1]) >= ny || std::abs(o[2]) >= nz) continue;  // no node has this neighbour
      ents.push_back({(int64_t(o[2]) * ny + o[1]) * nx + o[0], o[0], o[1], o[2], c});
    }
    std::stable_sort(ents.begin(), ents.end(), [](const Ent& a, const Ent& b) { return a.lin < b.lin; });
    // equal linear values: a repeated offset, or two offsets that alias across a grid edge
    for (size_t e = 1; e < ents.size(); ++e)
      if (ents[e].lin == ents[e - 1].lin) raise(LSAMGDD_ERR_INPUT, "generate_stencil_rows: duplicate or aliasing offsets in a row");
    for (size_t e = 0; e < ents.size(); ++e) {
      st.dx[k][e] = ents[e].dx;
      st.dy[k][e] = ents[e].dy;
      st.dz[k][e] = ents[e].dz;
      st.coef[k][e] = ents[e].c;
    }
  }
  auto g = std::make_unique<GeneratedCsr>();
  g->device = device;
  LSB_CUDA(cudaSetDevice(device));
  LSB_CUDA(cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking));
  cudaStream_t s = g->s;
  const int64_t m = n * rows_per_node;
  g->nr = m;
  g->nc = n;
  g->off.alloc(m + 1, s);
  const int grid_dim = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), int64_t(sm_count()) * 16)));
  k_gen_count<<<grid_dim, 256, 0, s>>>(st, nx, ny, nz, g->off.get());
  LSB_LAUNCH();
  size_t tmp = 0;
  LSB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, g->off.get() + 1, g->off.get() + 1, m, s));
  DBuf<unsigned char> t(tmp, s);
  LSB_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, g->off.get() + 1, g->off.get() + 1, m, s));
  int64_t nnz = 0;
  LSB_CUDA(cudaMemcpyAsync(&nnz, g->off.get() + m, 8, cudaMemcpyDeviceToHost, s));
  LSB_CUDA(cudaStreamSynchronize(s));
  g->nnz = nnz;
  g->col.alloc(nnz, s);
  g->val.alloc(nnz, s);
  if (nnz) k_gen_fill<<<grid_dim, 256, 0, s>>>(st, nx, ny, nz, g->off.get(), g->col.get(), g->val.get());
  LSB_LAUNCH();
  LSB_CUDA(cudaStreamSynchronize(s));  // the arrays are handed to the caller's streams
  return g.release();
}

void generated_view(const GeneratedCsr* g, lsamgdd_csr* out) {
  out->n_rows = g->nr;
  out->n_cols = g->nc;
  out->nnz = g->nnz;
  out->row_offsets = g->off.get();
  out->col_indices = g->col.get();
  out->values = g->val.get();
  out->memory = LSAMGDD_DEVICE;
  out->reserved = 0;
}

void generated_export(const GeneratedCsr* g, int64_t* off, int64_t* col, double* val) {
  LSB_CUDA(cudaSetDevice(g->device));
  LSB_CUDA(cudaStreamSynchronize(g->s));
  if (off) LSB_CUDA(cudaMemcpyAsync(off, g->off.get(), (g->nr + 1) * 8, cudaMemcpyDeviceToHost, g->s));
  if (col && g->nnz) LSB_CUDA(cudaMemcpyAsync(col, g->col.get(), g->nnz * 8, cudaMemcpyDeviceToHost, g->s));
  if (val && g->nnz) LSB_CUDA(cudaMemcpyAsync(val, g->val.get(), g->nnz * 8, cudaMemcpyDeviceToHost, g->s));
  LSB_CUDA(cudaStreamSynchronize(g->s));
}

void generated_destroy(GeneratedCsr* g) { delete g; }

}  // namespace lsb
