// sparse.cuh — device CSR / SELL-32 storage and the ordered sparse kernels
// (transpose, symbolic Gustavson product, SpMV) of sparse.hpp on the GPU.
#pragma once

#include "common.cuh"

namespace lsb {

// CSR on the device: int64 row offsets (G keeps all m rows on every level
// and can exceed 2^31 stored entries), int32 columns, FP64 values.
struct DevCsr {
  int64_t nr = 0, nc = 0, nnz = 0;
  DBuf<int64_t> off;
  DBuf<int32_t> col;
  DBuf<double> val;
};

// SELL-32: slices of 32 consecutive rows stored column-major inside the
// slice and padded to the slice's longest row, so one thread per row reads
// its entries in CSR order (bit-exact sequential row sums) while a warp's
// loads are fully coalesced. Padding columns are -1.
struct Sell {
  int64_t nr = 0, nc = 0, nnz = 0, stored = 0;
  int64_t n_slices = 0;
  DBuf<int64_t> slice_off;  // n_slices + 1, in elements
  DBuf<int32_t> row_len;    // nr
  DBuf<int32_t> col;
  DBuf<double> val;
  int64_t bytes() const { return stored * 12 + n_slices * 8 + nr * 4; }
};

void csr_upload(DevCsr& d, const lsamgdd_csr* h, cudaStream_t s);
void csr_download(const DevCsr& d, std::vector<int64_t>& off, std::vector<int64_t>& col,
                  std::vector<double>& val, cudaStream_t s);
// Stable transpose: rows of the result list the source rows in ascending
// order, exactly like the counting sort of sparse.hpp:139-153.
void csr_transpose(const DevCsr& a, DevCsr& t, cudaStream_t s);
// Symbolic-mode product a·b (sparse.hpp:167-204): the structural pattern
// with exact zeros kept, each entry accumulated over k in the reference's
// order (expand in (row, k_a, k_b) order, stable radix sort by (row, col),
// ordered run sums). Chunked over rows to bound scratch memory.
void csr_spgemm_symbolic(const DevCsr& a, const DevCsr& b, DevCsr& c, cudaStream_t s,
                         int64_t budget = int64_t(1) << 27);
void sell_from_csr(const DevCsr& a, Sell& out, cudaStream_t s);

// y = A x (mode 0), y = r - A x (mode 1, the fused V-cycle residual of
// hierarchy.hpp:213-214). Thread per row, sequential in CSR order.
void sell_spmv(const Sell& a, const double* x, double* y, const double* r, cudaStream_t s);
// y = A x (r == null) or y = r - A x with one warp per row (long rows)
void csr_spmv_warp(const DevCsr& a, const double* x, double* y, const double* r, cudaStream_t s);

}  // namespace lsb
