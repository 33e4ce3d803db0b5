// galerkin.cu — the Galerkin recursion G_{l+1} = G_l·P_l, A_{l+1} = G_{l+1}ᵀG_{l+1}
// (hierarchy.hpp:171-172) exploiting P's block-diagonal panel structure.
//
// Both products keep the reference's Symbolic pattern (sparse.hpp:167-204:
// exact-zero sums stay, entries exist iff some stored-by-stored product
// does) and accumulate every entry over the inner index in the reference's
// ascending order, so the result is bit-identical to spgemm(..., Symbolic):
//  * G·P: one warp per row of G; the row's entries are grouped by the
//    aggregate of their column (ascending aggregates = ascending coarse
//    columns), one lane per coarse column sums g_k·P(k,c) over the group's
//    entries in column order.
//  * GᵀG: the coarse columns of G_{l+1} come in aggregate blocks, so A is
//    assembled from dense k_a×k_b tiles, one CTA per aggregate pair (a ≤ b)
//    sharing rows of G; every thread owns tile entries and walks the shared
//    rows in ascending order (the Gustavson order of the reference). Tiles
//    (b, a) are the transposes (products commute, the row order is the same,
//    so A is exactly symmetric as in the reference).
#include <cub/cub.cuh>

#include <algorithm>

#include "galerkin.cuh"

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

template <class T>
void scan_inclusive(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  LSB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out, n, s));
  DBuf<unsigned char> t(tmp, s);
  LSB_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, in, out, n, s));
}

template <class T>
void scan_exclusive(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  LSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, s));
  DBuf<unsigned char> t(tmp, s);
  LSB_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, n, s));
}

// ---- G·P ----------------------------------------------------------------------------

constexpr int kGpWarps = 8;
constexpr int kGpCap = 256;  // row entries cached per warp in shared memory

struct GpArgs {
  const int64_t* goff;
  const int32_t* gcol;
  const double* gval;
  int64_t m;
  const int32_t* node_agg;
  const int32_t* node_pos;
  const int32_t* coff;
  const int64_t* poff;
  const double* panels;
  int64_t* cnt;        // pass 0: per row count at [r+1]
  const int64_t* off;  // pass 1: output offsets
  int32_t* ocol;
  double* oval;
};

template <int PASS>
__global__ void __launch_bounds__(kGpWarps * 32) k_gp(GpArgs g) {
  __shared__ double sval[kGpWarps][kGpCap];
  __shared__ int32_t sagg[kGpWarps][kGpCap];
  __shared__ int32_t spos[kGpWarps][kGpCap];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwarps = int64_t(gridDim.x) * kGpWarps;
  for (int64_t r = int64_t(blockIdx.x) * kGpWarps + warp; r < g.m; r += nwarps) {
    const int64_t k0 = g.goff[r];
    const int len = static_cast<int>(g.goff[r + 1] - k0);
    const bool cached = len <= kGpCap;
    if (cached)
      for (int e = lane; e < len; e += 32) {
        const int k = g.gcol[k0 + e];
        sval[warp][e] = g.gval[k0 + e];
        sagg[warp][e] = g.node_agg[k];
        spos[warp][e] = g.node_pos[k];
      }
    __syncwarp();
    auto agg_of = [&](int e) { return cached ? sagg[warp][e] : g.node_agg[g.gcol[k0 + e]]; };
    int64_t written = 0;
    int cur = -1;
    while (true) {
      int mn = 0x7fffffff;  // smallest aggregate above cur
      for (int e = lane; e < len; e += 32) {
        const int a = agg_of(e);
        if (a > cur && a < mn) mn = a;
      }
      for (int o = 16; o; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if (mn == 0x7fffffff) break;
      const int a = mn;
      cur = a;
      const int ka = g.coff[a + 1] - g.coff[a];
      const double* pan = g.panels + g.poff[a];
      for (int c0 = 0; c0 < ka; c0 += 32) {
        const int c = c0 + lane;
        double s = 0.0;
        bool present = false;
        if (c < ka) {
          for (int e = 0; e < len; ++e) {
            if (agg_of(e) != a) continue;
            const int pos = cached ? spos[warp][e] : g.node_pos[g.gcol[k0 + e]];
            const double v = cached ? sval[warp][e] : g.gval[k0 + e];
            const double p = pan[int64_t(pos) * ka + c];
            if (p != 0.0) {  // stored entries of P only (csr_from_triplets drops zeros)
              s += v * p;
              present = true;
            }
          }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, present);
        if (PASS == 1 && present) {
          const int64_t o = g.off[r] + written + __popc(mask & ((1u << lane) - 1u));
          g.ocol[o] = g.coff[a] + c;
          g.oval[o] = s;
        }
        written += __popc(mask);
      }
    }
    if (PASS == 0 && lane == 0) g.cnt[r + 1] = written;
    __syncwarp();
  }
}

// ---- GᵀG tiles -----------------------------------------------------------------------

// (agg, row) pairs of the row sets re-sorted by row: every G row's hit
// aggregates in ascending order
// one thread per (aggregate, row) pair; the aggregate by binary search in
// nz_off (deep levels have few aggregates with millions of rows each)
__global__ void k_rs_pairs(const int64_t* nz_off, const int32_t* nz, int64_t n_agg, uint32_t* key_row,
                           int32_t* val_agg) {
  const int64_t total = nz_off[n_agg];
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < total; p += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = n_agg - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (nz_off[mid] <= p)
        lo = mid;
      else
        hi = mid - 1;
    }
    key_row[p] = static_cast<uint32_t>(nz[p]);
    val_agg[p] = static_cast<int32_t>(lo);
  }
}

__global__ void k_mult_to_cnt(const int32_t* mult, int64_t m, int64_t* c) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x)
    c[r + 1] = mult[r];
}

__global__ void k_row_pair_count(const int64_t* roff, int64_t m, int64_t* cnt) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
    const int64_t h = roff[r + 1] - roff[r];
    cnt[r] = h * (h + 1) / 2;
  }
}

__global__ void k_row_pairs(const int64_t* roff, const int32_t* raggs, int64_t m, const int64_t* ppos, uint64_t n_agg,
                            uint64_t* key, int32_t* row) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
    int64_t o = ppos[r];
    for (int64_t x = roff[r]; x < roff[r + 1]; ++x)
      for (int64_t y = x; y < roff[r + 1]; ++y) {
        key[o] = static_cast<uint64_t>(raggs[x]) * n_agg + static_cast<uint64_t>(raggs[y]);
        row[o] = static_cast<int32_t>(r);
        ++o;
      }
  }
}

__global__ void k_run_heads(const uint64_t* key, int64_t n, int32_t* head) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x)
    head[p] = (p == 0 || key[p] != key[p - 1]) ? 1 : 0;
}

__global__ void k_tiles(const uint64_t* key, const int32_t* head, const int32_t* hpos, int64_t n, uint64_t n_agg,
                        int32_t* ta, int32_t* tb, int64_t* tstart) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    if (!head[p]) continue;
    const int64_t t = hpos[p];
    ta[t] = static_cast<int32_t>(key[p] / n_agg);
    tb[t] = static_cast<int32_t>(key[p] % n_agg);
    tstart[t] = p;
  }
}

constexpr int kSub = 32;          // output sub-tile edge

struct TileArgs {
  const int64_t* goff;  // G_{l+1}
  const int32_t* gcol;
  const double* gval;
  const int32_t* coff;
  const int32_t* ta;
  const int32_t* tb;
  const int64_t* tstart;  // n_tiles + 1 into rows
  const int32_t* rows;
  const int64_t* tval_off;  // tile value offsets (k_a × k_b)
  double* tval;
  uint8_t* tmask;
  const int32_t* wi_tile;  // work items: (tile, i0, j0) sub-tiles
  const int32_t* wi_i0;
  const int32_t* wi_j0;
  int64_t n_items;
};

// One CTA per (tile, sub-tile): stages ROWS shared rows of the a- and
// b-segments (dense, with a presence flag = stored entry), then every thread
// advances its outputs over those rows in ascending order. Two shapes: 256
// threads × 32 rows where the items fill the SMs several times over, 512
// threads × 64 rows (two outputs per thread, four rows in flight per warp) on
// the coarse levels, where a handful of items walk millions of rows each.
template <int THREADS, int ROWS>
__global__ void __launch_bounds__(THREADS) k_gtg_tile(TileArgs g) {
  // Segments are staged dense (absent entries = +0: adding the ±0 products
  // leaves every sum unchanged, it starts at +0 and never becomes -0) with a
  // presence mask per row; an output exists in the Symbolic pattern iff some
  // row holds both of its entries.
  static_assert(kSub == 32, "presence masks are 32-bit");
  __shared__ double sa[ROWS][kSub];
  __shared__ double sb[ROWS][kSub];
  __shared__ unsigned ma[ROWS], mb[ROWS];
  constexpr int kPer = kSub * kSub / THREADS;
  constexpr int kIStep = THREADS / kSub;  // output rows of a thread: i0 + kIStep*q, column j
  constexpr int kWarps = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = threadIdx.x / kSub, tj = threadIdx.x % kSub;
  for (int64_t w = blockIdx.x; w < g.n_items; w += gridDim.x) {
    const int t = g.wi_tile[w];
    const int i0 = g.wi_i0[w], j0 = g.wi_j0[w];
    const int a = g.ta[t], b = g.tb[t];
    const int ca = g.coff[a] + i0, ka = g.coff[a + 1] - g.coff[a];
    const int cb = g.coff[b] + j0, kb = g.coff[b + 1] - g.coff[b];
    const int bi = min(kSub, ka - i0), bj = min(kSub, kb - j0);
    const int64_t r0 = g.tstart[t], r1 = g.tstart[t + 1];
    double acc[kPer];
    unsigned touched = 0u;
#pragma unroll
    for (int q = 0; q < kPer; ++q) acc[q] = 0.0;
    for (int64_t rb = r0; rb < r1; rb += ROWS) {
      const int nr = static_cast<int>(r1 - rb < ROWS ? r1 - rb : ROWS);
      // a warp owns its rows: clear, scatter the segment entries, publish the masks
      int64_t lo[(ROWS + kWarps - 1) / kWarps], hi[(ROWS + kWarps - 1) / kWarps];
#pragma unroll
      for (int u = 0; u < (ROWS + kWarps - 1) / kWarps; ++u) {
        const int rr = warp + u * kWarps;
        lo[u] = hi[u] = 0;
        if (rr < nr) {
          const int64_t r = __ldg(g.rows + rb + rr);
          lo[u] = __ldg(g.goff + r);
          hi[u] = __ldg(g.goff + r + 1);
          sa[rr][lane] = 0.0;
          sb[rr][lane] = 0.0;
        }
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < (ROWS + kWarps - 1) / kWarps; ++u) {
        const int rr = warp + u * kWarps;
        if (rr >= nr) continue;
        unsigned bits_a = 0u, bits_b = 0u;
#pragma unroll 2
        for (int64_t k = lo[u] + lane; k < hi[u]; k += 32) {  // one coalesced pass over the row
          const int col = __ldg(g.gcol + k);
          const double v = __ldg(g.gval + k);
          const unsigned ea = static_cast<unsigned>(col - ca), eb = static_cast<unsigned>(col - cb);
          if (ea < static_cast<unsigned>(bi)) {
            sa[rr][ea] = v;
            bits_a |= 1u << ea;
          }
          if (eb < static_cast<unsigned>(bj)) {
            sb[rr][eb] = v;
            bits_b |= 1u << eb;
          }
        }
        bits_a = __reduce_or_sync(0xffffffffu, bits_a);
        bits_b = __reduce_or_sync(0xffffffffu, bits_b);
        if (lane == 0) {
          ma[rr] = bits_a;
          mb[rr] = bits_b;
        }
      }
      __syncthreads();
#pragma unroll 4
      for (int rr = 0; rr < nr; ++rr) {
        const double yb = sb[rr][tj];
        touched |= ((mb[rr] >> tj) & 1u) ? ma[rr] : 0u;  // a-entries met by a stored b-entry of column tj
#pragma unroll
        for (int q = 0; q < kPer; ++q) acc[q] += sa[rr][ti + kIStep * q] * yb;
      }
      __syncthreads();
    }
    double* tv = g.tval + g.tval_off[t];
    uint8_t* tm = g.tmask + g.tval_off[t];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = ti + kIStep * q, j = tj;
      if (i >= bi || j >= bj) continue;
      const int64_t e = int64_t(i0 + i) * kb + (j0 + j);
      tv[e] = acc[q];
      tm[e] = ((touched >> i) & 1u) ? 1 : 0;
    }
  }
}

// per aggregate: its tiles ordered by partner aggregate (both orientations)
struct RowArgs {
  const int32_t* coff;
  const int32_t* col_agg;
  const int64_t* nb_off;  // per aggregate
  const int32_t* nb_tile;
  const int32_t* nb_partner;
  const uint8_t* nb_trans;
  const int32_t* ta;
  const int32_t* tb;
  const int64_t* tval_off;
  const double* tval;
  const uint8_t* tmask;
  int64_t n;
  int64_t* cnt;
  const int64_t* off;
  int32_t* ocol;
  double* oval;
};

template <int PASS>
__global__ void k_gtg_rows(RowArgs g) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < g.n; i += int64_t(gridDim.x) * blockDim.x) {
    const int a = g.col_agg[i];
    const int li = static_cast<int>(i - g.coff[a]);
    int64_t o = PASS == 1 ? g.off[i] : 0;
    int64_t c = 0;
    for (int64_t q = g.nb_off[a]; q < g.nb_off[a + 1]; ++q) {
      const int t = g.nb_tile[q];
      const int p = g.nb_partner[q];
      const int cp = g.coff[p], kp = g.coff[p + 1] - cp;
      const int kb = g.coff[g.tb[t] + 1] - g.coff[g.tb[t]];
      const double* tv = g.tval + g.tval_off[t];
      const uint8_t* tm = g.tmask + g.tval_off[t];
      const bool tr = g.nb_trans[q];
      for (int j = 0; j < kp; ++j) {
        const int64_t e = tr ? int64_t(j) * kb + li : int64_t(li) * kb + j;
        if (!tm[e]) continue;
        if (PASS == 1) {
          g.ocol[o] = cp + j;
          g.oval[o] = tv[e];
          ++o;
        }
        ++c;
      }
    }
    if (PASS == 0) g.cnt[i + 1] = c;
  }
}

}  // namespace

void galerkin_gp(const DevCsr& g, const DevTopo& topo, const DevInterp& ip, DevCsr& out, cudaStream_t s) {
  out.nr = g.nr;
  out.nc = ip.n_coarse;
  DBuf<int64_t> cnt(g.nr + 1, s);
  cnt.zero(s);
  GpArgs a{};
  a.goff = g.off.get();
  a.gcol = g.col.get();
  a.gval = g.val.get();
  a.m = g.nr;
  a.node_agg = topo.node_agg.get();
  a.node_pos = topo.node_pos.get();
  a.coff = ip.coarse_off.get();
  a.poff = ip.panel_off.get();
  a.panels = ip.panels.get();
  a.cnt = cnt.get();
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(g.nr, kGpWarps), sm_count() * 8)));
  if (g.nr) k_gp<0><<<grid, kGpWarps * 32, 0, s>>>(a);
  LSB_LAUNCH();
  out.off.alloc(g.nr + 1, s);
  scan_inclusive(cnt.get(), out.off.get(), g.nr + 1, s);
  out.nnz = read_scalar(out.off.get() + g.nr, s);
  out.col.alloc(out.nnz, s);
  out.val.alloc(out.nnz, s);
  a.off = out.off.get();
  a.ocol = out.col.get();
  a.oval = out.val.get();
  if (g.nr) k_gp<1><<<grid, kGpWarps * 32, 0, s>>>(a);
  LSB_LAUNCH();
}

void galerkin_gtg(const DevCsr& gn, const DevRowSets& rs, int64_t n_agg, const DevInterp& ip, const int32_t* col_agg,
                  DevCsr& out, cudaStream_t s) {
  const int64_t m = gn.nr, n = ip.n_coarse;
  out.nr = n;
  out.nc = n;
  // 1) hit aggregates of every G row, ascending (row sets re-sorted by row)
  const int64_t npairs = static_cast<int64_t>(rs.nz.size());
  DBuf<int64_t> roff(m + 1, s);
  DBuf<int32_t> raggs(std::max<int64_t>(npairs, 1), s);
  {
    DBuf<uint32_t> k1(std::max<int64_t>(npairs, 1), s), k2(std::max<int64_t>(npairs, 1), s);
    DBuf<int32_t> v1(std::max<int64_t>(npairs, 1), s);
    k_rs_pairs<<<grid_for(npairs), kThreads, 0, s>>>(rs.nz_off.get(), rs.nz.get(), n_agg, k1.get(), v1.get());
    LSB_LAUNCH();
    size_t tmp = 0;
    const int eb = bits_for(static_cast<uint64_t>(m));
    LSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k1.get(), k2.get(), v1.get(), raggs.get(), npairs, 0, eb, s));
    DBuf<unsigned char> tb(tmp, s);
    LSB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), tmp, k1.get(), k2.get(), v1.get(), raggs.get(), npairs, 0, eb, s));
    // row offsets from the multiplicities (mult[r] hits per row)
    DBuf<int64_t> c64(m + 1, s);
    c64.zero(s);
    k_mult_to_cnt<<<grid_for(m), kThreads, 0, s>>>(rs.mult.get(), m, c64.get());
    LSB_LAUNCH();
    scan_inclusive(c64.get(), roff.get(), m + 1, s);
  }
  // 2) (a ≤ b, row) pairs in row order, stable-sorted by tile key
  DBuf<int64_t> pcnt(m + 1, s), ppos(m + 1, s);
  pcnt.zero(s);
  k_row_pair_count<<<grid_for(m), kThreads, 0, s>>>(roff.get(), m, pcnt.get());
  LSB_LAUNCH();
  scan_exclusive(pcnt.get(), ppos.get(), m + 1, s);
  const int64_t np = read_scalar(ppos.get() + m, s);
  DBuf<uint64_t> key1(std::max<int64_t>(np, 1), s), key2(std::max<int64_t>(np, 1), s);
  DBuf<int32_t> row1(std::max<int64_t>(np, 1), s), rows(std::max<int64_t>(np, 1), s);
  k_row_pairs<<<grid_for(m), kThreads, 0, s>>>(roff.get(), raggs.get(), m, ppos.get(), static_cast<uint64_t>(n_agg),
                                               key1.get(), row1.get());
  LSB_LAUNCH();
  {
    size_t tmp = 0;
    const int eb = bits_for(static_cast<uint64_t>(n_agg) * static_cast<uint64_t>(n_agg));
    LSB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key1.get(), key2.get(), row1.get(), rows.get(), np, 0, eb, s));
    DBuf<unsigned char> tb(tmp, s);
    LSB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), tmp, key1.get(), key2.get(), row1.get(), rows.get(), np, 0, eb, s));
  }
  key1.release();
  row1.release();
  DBuf<int32_t> head(std::max<int64_t>(np, 1), s), hpos(std::max<int64_t>(np, 1), s);
  k_run_heads<<<grid_for(np), kThreads, 0, s>>>(key2.get(), np, head.get());
  LSB_LAUNCH();
  scan_exclusive(head.get(), hpos.get(), np, s);
  const int64_t n_tiles = np ? int64_t(read_scalar(hpos.get() + np - 1, s)) + read_scalar(head.get() + np - 1, s) : 0;
  DBuf<int32_t> ta(std::max<int64_t>(n_tiles, 1), s), tbv(std::max<int64_t>(n_tiles, 1), s);
  DBuf<int64_t> tstart(n_tiles + 1, s);
  k_tiles<<<grid_for(np), kThreads, 0, s>>>(key2.get(), head.get(), hpos.get(), np, static_cast<uint64_t>(n_agg), ta.get(),
                                            tbv.get(), tstart.get());
  LSB_LAUNCH();
  LSB_CUDA(cudaMemcpyAsync(tstart.get() + n_tiles, &np, 8, cudaMemcpyHostToDevice, s));
  key2.release();
  head.release();
  hpos.release();
  // 3) tile sizes and sub-tile work items on the host (k per aggregate is known there)
  const std::vector<int32_t> h_ta = ta.download(s), h_tb = tbv.download(s);
  const std::vector<int32_t>& hk = ip.h_k;
  std::vector<int64_t> tval_off(n_tiles + 1, 0);
  std::vector<int32_t> wt, wi, wj;
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int64_t ka = hk[h_ta[t]], kb = hk[h_tb[t]];
    tval_off[t + 1] = tval_off[t] + ka * kb;
    for (int64_t i0 = 0; i0 < ka; i0 += kSub)
      for (int64_t j0 = 0; j0 < kb; j0 += kSub) {
        wt.push_back(static_cast<int32_t>(t));
        wi.push_back(static_cast<int32_t>(i0));
        wj.push_back(static_cast<int32_t>(j0));
      }
  }
  DBuf<int64_t> d_tval_off;
  d_tval_off.upload(tval_off, s);
  DBuf<double> tval(std::max<int64_t>(tval_off[n_tiles], 1), s);
  DBuf<uint8_t> tmask(std::max<int64_t>(tval_off[n_tiles], 1), s);
  DBuf<int32_t> d_wt, d_wi, d_wj;
  d_wt.upload(wt, s);
  d_wi.upload(wi, s);
  d_wj.upload(wj, s);
  TileArgs targ{gn.off.get(), gn.col.get(), gn.val.get(), ip.coarse_off.get(), ta.get(), tbv.get(), tstart.get(),
                rows.get(), d_tval_off.get(), tval.get(), tmask.get(), d_wt.get(), d_wi.get(), d_wj.get(),
                static_cast<int64_t>(wt.size())};
  if (!wt.empty()) {
    const int64_t items = static_cast<int64_t>(wt.size());
    if (items <= 2 * int64_t(sm_count()))
      k_gtg_tile<512, 64><<<static_cast<int>(std::min<int64_t>(items, sm_count())), 512, 0, s>>>(targ);
    else
      k_gtg_tile<256, 32><<<static_cast<int>(std::min<int64_t>(items, sm_count() * 8)), 256, 0, s>>>(targ);
    LSB_LAUNCH();
  }
  // 4) per aggregate tile lists sorted by partner, then rows of A
  std::vector<std::vector<std::tuple<int32_t, int32_t, uint8_t>>> nb(n_agg);
  for (int64_t t = 0; t < n_tiles; ++t) {
    nb[h_ta[t]].emplace_back(h_tb[t], static_cast<int32_t>(t), 0);
    if (h_ta[t] != h_tb[t]) nb[h_tb[t]].emplace_back(h_ta[t], static_cast<int32_t>(t), 1);
  }
  std::vector<int64_t> nb_off(n_agg + 1, 0);
  std::vector<int32_t> nb_tile, nb_partner;
  std::vector<uint8_t> nb_trans;
  for (int64_t a = 0; a < n_agg; ++a) {
    std::sort(nb[a].begin(), nb[a].end());
    for (auto& [p, t, tr] : nb[a]) {
      nb_partner.push_back(p);
      nb_tile.push_back(t);
      nb_trans.push_back(tr);
    }
    nb_off[a + 1] = static_cast<int64_t>(nb_tile.size());
  }
  DBuf<int64_t> d_nb_off;
  DBuf<int32_t> d_nb_tile, d_nb_partner;
  DBuf<uint8_t> d_nb_trans;
  d_nb_off.upload(nb_off, s);
  d_nb_tile.upload(nb_tile, s);
  d_nb_partner.upload(nb_partner, s);
  d_nb_trans.upload(nb_trans, s);
  DBuf<int64_t> cnt(n + 1, s);
  cnt.zero(s);
  RowArgs ra{ip.coarse_off.get(), col_agg, d_nb_off.get(), d_nb_tile.get(), d_nb_partner.get(), d_nb_trans.get(),
             ta.get(), tbv.get(), d_tval_off.get(), tval.get(), tmask.get(), n, cnt.get(), nullptr, nullptr, nullptr};
  k_gtg_rows<0><<<grid_for(n), kThreads, 0, s>>>(ra);
  LSB_LAUNCH();
  out.off.alloc(n + 1, s);
  scan_inclusive(cnt.get(), out.off.get(), n + 1, s);
  out.nnz = read_scalar(out.off.get() + n, s);
  out.col.alloc(out.nnz, s);
  out.val.alloc(out.nnz, s);
  ra.off = out.off.get();
  ra.ocol = out.col.get();
  ra.oval = out.val.get();
  k_gtg_rows<1><<<grid_for(n), kThreads, 0, s>>>(ra);
  LSB_LAUNCH();
  LSB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace lsb
