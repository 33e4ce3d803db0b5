// grams.cu — the local weighted Grams of large aggregates as a multi-CTA
// tiled product (splitting.hpp:102-115, 210-221).
//
// For aggregate i with subdomain Ω_i = ω_i ‖ Γ_i and row set nz_i the
// reference forms, over rows r ∈ nz_i in ascending order,
//   M(a,b) = Σ_r (w_r·g_ra)·g_rb          (W = M[ω,ω], C = M[ω,Γ], B = M[Γ,Γ])
//   L(a,b) = Σ_r (1·g_ra)·g_rb  (a,b ∈ ω) (SchurReduced; WeightedLhs: L = W)
// with w_r = 1/multiplicity(r). On deep levels nz_i holds millions of rows
// of G_l with ~100 stored entries each, which one CTA cannot sweep in time.
// Here every aggregate's Ω is cut into chunks of 64 local positions and one
// CTA owns one 64×64 output tile (X, Y): it walks the rows that touch both
// chunks in ascending order, densifies their X and Y segments in shared
// memory and accumulates each output in that order. Rows that do not touch
// both chunks contribute only exact ±0 products to the reference's sums
// (which start at +0 and never become -0), so skipping them — like the
// zero entries densified here — leaves every output bit-identical.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "setup_kernels.cuh"

namespace lsb {

namespace {

constexpr int kCW = 64;       // chunk width (local positions)
constexpr int kTileThreads = 256;
constexpr int kRowBatch = 32;  // candidate rows staged per round

// map[gi * n + node] = local position of node in Ω of group aggregate gi
__global__ void k_fill_posmap(const int32_t* group, int n_group, const int32_t* omega_off, const int32_t* omega,
                              const int32_t* gamma_off, const int32_t* gamma, int64_t n_nodes, int32_t* map) {
  const int gi = blockIdx.y;
  if (gi >= n_group) return;
  const int agg = group[gi];
  const int nw = omega_off[agg + 1] - omega_off[agg];
  const int ng = gamma_off[agg + 1] - gamma_off[agg];
  int32_t* m = map + int64_t(gi) * n_nodes;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nw + ng; e += gridDim.x * blockDim.x)
    m[e < nw ? omega[omega_off[agg] + e] : gamma[gamma_off[agg] + e - nw]] = e;
}

// one warp per row of the group: the mask of Ω chunks the row touches
__global__ void k_row_masks(const int64_t* goff, const int32_t* gcol, const int32_t* nz, const int64_t* row_src,
                            const int64_t* row_off, int n_group, const int32_t* map, int64_t n_nodes,
                            unsigned long long* mask) {
  const int64_t total = row_off[n_group];
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t k = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); k < total; k += warps) {
    int lo = 0, hi = n_group - 1;  // group aggregate of row slot k
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (row_off[mid] <= k)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int32_t* m = map + int64_t(lo) * n_nodes;
    const int r = nz[row_src[lo] + (k - row_off[lo])];
    unsigned long long bits = 0;
    for (int64_t e = goff[r] + lane; e < goff[r + 1]; e += 32) {
      const int p = m[gcol[e]];
      if (p >= 0) bits |= 1ull << (p / kCW);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
    if (lane == 0) mask[k] = bits;
  }
}

// CTA per (group aggregate, chunk): ordered list of the aggregate's row slots
// touching the chunk.
__global__ void __launch_bounds__(256) k_chunk_rows(const int64_t* row_off, const int32_t* nchunk,
                                                    const int64_t* list_off, const int32_t* pair_agg,
                                                    const int32_t* pair_chunk, const unsigned long long* mask,
                                                    int32_t* list, int32_t* list_cnt) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int base_s;
  const int pr = blockIdx.x;
  const int gi = pair_agg[pr], x = pair_chunk[pr];
  const int64_t r0 = row_off[gi], r1 = row_off[gi + 1];
  int32_t* out = list + list_off[pr];
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  for (int64_t k0 = r0; k0 < r1; k0 += 256) {
    const int64_t k = k0 + threadIdx.x;
    const int flag = (k < r1 && ((mask[k] >> x) & 1ull)) ? 1 : 0;
    int pos, tot;
    Scan(tmp).ExclusiveSum(flag, pos, tot);
    const int base = base_s;
    if (flag) out[base + pos] = static_cast<int32_t>(k - r0);
    __syncthreads();
    if (threadIdx.x == 0) base_s = base + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) list_cnt[pr] = base_s;
  (void)nchunk;
}

struct TileArgs {
  const int64_t* goff;
  const int32_t* gcol;
  const double* gval;
  const int32_t* mult;
  const int32_t* nz;
  const int64_t* row_src;   // per group aggregate: offset of its rows in nz
  const int64_t* row_off;   // per group aggregate: offset of its row slots
  const unsigned long long* mask;
  const int32_t* map;
  int64_t n_nodes;
  const int32_t* group;
  const int32_t* omega_off;
  const int32_t* gamma_off;
  const int32_t* nchunk;     // per group aggregate
  const int64_t* tile_off;   // per group aggregate (prefix of nchunk²), n_group + 1
  const int64_t* pair_off;   // per group aggregate: first (agg, chunk) pair index
  const int64_t* list_off;   // per pair
  const int32_t* list;
  const int32_t* list_cnt;   // per pair
  int n_group;
  int weighted_lhs;
  double* out;               // pre-gram storage
  const int64_t* out_off;    // per aggregate id
};

__global__ void __launch_bounds__(kTileThreads) k_gram_tile(TileArgs g) {
  __shared__ double segx[kRowBatch][kCW];
  __shared__ double segy[kRowBatch][kCW];
  __shared__ double wt[kRowBatch];
  __shared__ int sel[kRowBatch];
  __shared__ int nsel;
  const int64_t tile = blockIdx.x;
  int lo = 0, hi = g.n_group - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g.tile_off[mid] <= tile)
      lo = mid;
    else
      hi = mid - 1;
  }
  const int gi = lo;
  const int agg = g.group[gi];
  const int nw = g.omega_off[agg + 1] - g.omega_off[agg];
  const int ng = g.gamma_off[agg + 1] - g.gamma_off[agg];
  const int nc = g.nchunk[gi];
  const int t_in = static_cast<int>(tile - g.tile_off[gi]);
  const int X = t_in / nc, Y = t_in % nc;
  const int x0 = X * kCW, y0 = Y * kCW;
  if (x0 >= nw && y0 + kCW <= nw) return;  // the Γ×ω block is never read
  const bool need_l = x0 < nw && y0 < nw && !g.weighted_lhs;
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  double accm[4][4], accl[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) accm[u][v] = accl[u][v] = 0.0;
  const int64_t pr = g.pair_off[gi] + X;
  const int32_t* lst = g.list + g.list_off[pr];
  const int cnt = g.list_cnt[pr];
  const int64_t rbase = g.row_off[gi];
  const int32_t* nzr = g.nz + g.row_src[gi];
  const int32_t* m = g.map + int64_t(gi) * g.n_nodes;
  const int warp = tid >> 5, lane = tid & 31;
  for (int c0 = 0; c0 < cnt; c0 += kRowBatch) {
    if (warp == 0) {
      const int c = c0 + lane;
      int slot = -1;
      bool hit = false;
      if (c < cnt) {
        slot = lst[c];
        hit = ((g.mask[rbase + slot] >> Y) & 1ull) != 0;
      }
      const unsigned b = __ballot_sync(0xffffffffu, hit);
      if (hit) sel[__popc(b & ((1u << lane) - 1u))] = slot;
      if (lane == 0) nsel = __popc(b);
    }
    for (int e = tid; e < kRowBatch * kCW; e += kTileThreads) {
      (&segx[0][0])[e] = 0.0;
      (&segy[0][0])[e] = 0.0;
    }
    __syncthreads();
    const int ns = nsel;
    for (int j = warp; j < ns; j += kTileThreads / 32) {
      const int r = nzr[sel[j]];
      if (lane == 0) wt[j] = 1.0 / static_cast<double>(g.mult[r]);
      for (int64_t e = g.goff[r] + lane; e < g.goff[r + 1]; e += 32) {
        const int p = m[g.gcol[e]];
        const double v = g.gval[e];
        if (p >= x0 && p < x0 + kCW) segx[j][p - x0] = v;
        if (p >= y0 && p < y0 + kCW) segy[j][p - y0] = v;
      }
    }
    __syncthreads();
    for (int j = 0; j < ns; ++j) {
      const double w = wt[j];
      double xa[4], yb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xa[u] = segx[j][ty * 4 + u];
#pragma unroll
      for (int v = 0; v < 4; ++v) yb[v] = segy[j][tx * 4 + v];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double wx = w * xa[u];
#pragma unroll
        for (int v = 0; v < 4; ++v) accm[u][v] += wx * yb[v];
      }
      if (need_l) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) accl[u][v] += xa[u] * yb[v];
      }
    }
    __syncthreads();
  }
  double* base = g.out + g.out_off[agg];
  double* L = base;
  double* W = L + int64_t(nw) * nw;
  double* C = W + int64_t(nw) * nw;
  double* B = C + int64_t(nw) * ng;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int a = x0 + ty * 4 + u;
    if (a >= nw + ng) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int b = y0 + tx * 4 + v;
      if (b >= nw + ng) continue;
      if (a < nw) {
        if (b < nw) {
          W[int64_t(a) * nw + b] = accm[u][v];
          L[int64_t(a) * nw + b] = g.weighted_lhs ? accm[u][v] : accl[u][v];
        } else {
          C[int64_t(a) * ng + (b - nw)] = accm[u][v];
        }
      } else if (b >= nw) {
        B[int64_t(a - nw) * ng + (b - nw)] = accm[u][v];
      }
    }
  }
}

}  // namespace

int64_t pre_gram_doubles(int64_t nw, int64_t ng) { return 2 * nw * nw + nw * ng + ng * ng; }

void tiled_grams(const DevCsr& gm, const DevTopo& topo, const std::vector<int32_t>& hoo,
                 const std::vector<int32_t>& hgo, const DevRowSets& rs, const std::vector<int64_t>& h_nz_off,
                 const std::vector<int32_t>& aggs, int weighted_lhs, double* out, const int64_t* d_out_off,
                 cudaStream_t s) {
  const int64_t n_nodes = topo.n_nodes;
  const int64_t map_budget = int64_t(1) << 26;    // int32 entries of position maps per group
  const int64_t list_budget = int64_t(1) << 28;   // int32 entries of chunk row lists per group
  size_t a0 = 0;
  while (a0 < aggs.size()) {
    // group: bounded map and list footprint
    std::vector<int32_t> grp;
    int64_t lists = 0;
    size_t a1 = a0;
    while (a1 < aggs.size()) {
      const int32_t a = aggs[a1];
      const int64_t nsub = (hoo[a + 1] - hoo[a]) + (hgo[a + 1] - hgo[a]);
      const int64_t nc = ceil_div(nsub, kCW);
      const int64_t rows = h_nz_off[a + 1] - h_nz_off[a];
      if (!grp.empty() && (int64_t(grp.size() + 1) * n_nodes > map_budget || lists + nc * rows > list_budget)) break;
      grp.push_back(a);
      lists += nc * rows;
      ++a1;
    }
    const int n_group = static_cast<int>(grp.size());
    std::vector<int64_t> row_src(n_group), row_off(n_group + 1, 0), tile_off(n_group + 1, 0), pair_off(n_group + 1, 0);
    std::vector<int32_t> nchunk(n_group), pair_agg, pair_chunk;
    std::vector<int64_t> list_off;
    int64_t lo = 0;
    for (int gi = 0; gi < n_group; ++gi) {
      const int32_t a = grp[gi];
      const int64_t nsub = (hoo[a + 1] - hoo[a]) + (hgo[a + 1] - hgo[a]);
      const int nc = static_cast<int>(ceil_div(nsub, kCW));
      nchunk[gi] = nc;
      row_src[gi] = h_nz_off[a];
      const int64_t rows = h_nz_off[a + 1] - h_nz_off[a];
      row_off[gi + 1] = row_off[gi] + rows;
      tile_off[gi + 1] = tile_off[gi] + int64_t(nc) * nc;
      pair_off[gi + 1] = pair_off[gi] + nc;
      for (int x = 0; x < nc; ++x) {
        pair_agg.push_back(gi);
        pair_chunk.push_back(x);
        list_off.push_back(lo);
        lo += rows;
      }
    }
    DBuf<int32_t> d_grp, d_nchunk, d_pair_agg, d_pair_chunk, map(int64_t(n_group) * n_nodes, s);
    DBuf<int64_t> d_row_src, d_row_off, d_tile_off, d_pair_off, d_list_off;
    d_grp.upload(grp, s);
    d_nchunk.upload(nchunk, s);
    d_pair_agg.upload(pair_agg, s);
    d_pair_chunk.upload(pair_chunk, s);
    d_row_src.upload(row_src, s);
    d_row_off.upload(row_off, s);
    d_tile_off.upload(tile_off, s);
    d_pair_off.upload(pair_off, s);
    d_list_off.upload(list_off, s);
    LSB_CUDA(cudaMemsetAsync(map.get(), 0xff, map.bytes(), s));
    {
      dim3 grid(4, n_group);
      k_fill_posmap<<<grid, 256, 0, s>>>(d_grp.get(), n_group, topo.omega_off.get(), topo.omega.get(),
                                         topo.gamma_off.get(), topo.gamma.get(), n_nodes, map.get());
      LSB_LAUNCH();
    }
    const int64_t total_rows = row_off[n_group];
    DBuf<unsigned long long> mask(std::max<int64_t>(total_rows, 1), s);
    {
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total_rows, 8), sm_count() * 16)));
      k_row_masks<<<grid, 256, 0, s>>>(gm.off.get(), gm.col.get(), rs.nz.get(), d_row_src.get(), d_row_off.get(),
                                       n_group, map.get(), n_nodes, mask.get());
      LSB_LAUNCH();
    }
    const int n_pairs = static_cast<int>(pair_agg.size());
    DBuf<int32_t> list(std::max<int64_t>(lo, 1), s), list_cnt(n_pairs, s);
    k_chunk_rows<<<n_pairs, 256, 0, s>>>(d_row_off.get(), d_nchunk.get(), d_list_off.get(), d_pair_agg.get(),
                                         d_pair_chunk.get(), mask.get(), list.get(), list_cnt.get());
    LSB_LAUNCH();
    TileArgs ta{};
    ta.goff = gm.off.get();
    ta.gcol = gm.col.get();
    ta.gval = gm.val.get();
    ta.mult = rs.mult.get();
    ta.nz = rs.nz.get();
    ta.row_src = d_row_src.get();
    ta.row_off = d_row_off.get();
    ta.mask = mask.get();
    ta.map = map.get();
    ta.n_nodes = n_nodes;
    ta.group = d_grp.get();
    ta.omega_off = topo.omega_off.get();
    ta.gamma_off = topo.gamma_off.get();
    ta.nchunk = d_nchunk.get();
    ta.tile_off = d_tile_off.get();
    ta.pair_off = d_pair_off.get();
    ta.list_off = d_list_off.get();
    ta.list = list.get();
    ta.list_cnt = list_cnt.get();
    ta.n_group = n_group;
    ta.weighted_lhs = weighted_lhs;
    ta.out = out;
    ta.out_off = d_out_off;
    k_gram_tile<<<static_cast<unsigned>(tile_off[n_group]), kTileThreads, 0, s>>>(ta);
    LSB_LAUNCH();
    a0 = a1;
  }
}

}  // namespace lsb
