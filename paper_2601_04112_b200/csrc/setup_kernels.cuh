// setup_kernels.cuh — batched per-aggregate setup stages on the device.
#pragma once

#include "common.cuh"
#include "sparse.cuh"

namespace lsb {

// Per-level aggregate topology on the device (AggregateTopology,
// aggregation.hpp:33-54): ω and Γ lists, both ascending, as in the reference.
struct DevTopo {
  int64_t n_nodes = 0, n_agg = 0;
  DBuf<int32_t> omega_off, omega, gamma_off, gamma;
  DBuf<int32_t> node_agg, node_pos;  // owner aggregate and position in its ω
};

// RowSets (splitting.hpp:26-30) on the device.
struct DevRowSets {
  DBuf<int32_t> mult;   // per G row
  DBuf<int64_t> nz_off; // n_agg + 1
  DBuf<int32_t> nz;     // G rows, ascending within an aggregate
  int64_t n_mult = 0;
  int64_t empty_rows = 0;
  int64_t max_row_nnz = 0;
};

// compute_row_sets (splitting.hpp:53-84)
void row_sets(const DevCsr& g, const DevTopo& topo, DevRowSets& rs, cudaStream_t s);

// Schwarz storage of one level: per aggregate, the ω columns of the explicit
// inverse of A(Ω,Ω) (the only part RAS and RAS-T read): the ω×ω block as a
// packed upper triangle, then the ω×Γ block row-major.
struct DevSmoother {
  int64_t n_agg = 0;
  DBuf<int64_t> off;      // n_agg + 1 (doubles)
  DBuf<double> data;
  DBuf<int32_t> order;    // aggregates sorted by colour
  std::vector<int64_t> color_off;  // host, n_colors + 1
  int64_t max_omega = 0, max_sub = 0;
  double bytes_ras = 0, bytes_rast = 0;  // algorithmic bytes per sweep
  // Lane-interleaved layout for small subdomains (nΩ <= kLaneMaxSub): groups
  // of up to 32 aggregates with one (colour, nω, nΓ) shape; element e of lane
  // l lives at [e][l], so every warp load is one 256-byte transaction.
  int64_t n_groups = 0;
  DBuf<int32_t> g_nw, g_ng, g_cnt;   // per group
  DBuf<int64_t> g_ids_off, g_blk_off;  // per group, in int32 / double units
  DBuf<int32_t> lane_ids;             // [nΩ][32] per group
  DBuf<double> lane_blk;              // [nblk][32] per group
  std::vector<int64_t> color_goff;    // host, n_colors + 1 (groups are colour-sorted)
  // warp-per-output-row work items over the groups: (group << 8) | row
  DBuf<int32_t> lane_ras_items, lane_rast_items;
  std::vector<int64_t> lane_rast_color_off;  // host, n_colors + 1
  // persistent TMA-pipelined sweep over the groups (k_schwarz_tma): per-group colour, groups
  // per colour (the RAS-T completion counters live in each call's workspace); stage capacity
  // in bytes of the largest group (0: path not available)
  DBuf<int32_t> g_color, color_groups;
  int64_t n_colors = 0;
  int64_t stage_blk_bytes = 0, stage_ids_bytes = 0;
  // one-launch RAS-T: the Γ contributions of a subdomain go to per-node slots (node-major,
  // holders in ascending aggregate order) and a second kernel adds each node's slots into e
  DBuf<int64_t> g_slot_off;            // per group (int32 units)
  DBuf<int32_t> lane_slots;            // [nΓ][32] per group: slot of the lane's Γ node j, -1 for padding
  DBuf<int32_t> node_slot_off;         // n_nodes + 1
  int64_t n_slots = 0, stage_slot_bytes = 0;
  // Row layout for large subdomains (warp per output row, many warps per
  // aggregate): per aggregate the full ω×Ω rows of the inverse (F, nω×nΩ)
  // then its Γ columns transposed (Gt, nΓ×nω), so that RAS (rows of F) and
  // RAS-T (ω rows of F, rows of Gt) read contiguous rows.
  bool rows = false;
  DBuf<int64_t> row_off;              // n_agg + 1 (doubles)
  DBuf<double> row_data;
  DBuf<int32_t> ras_agg, ras_row;     // RAS work items: (aggregate, first ω row of a chunk of ras_ch rows)
  int ras_ch = 1;
  int rast_ch = 1;                    // Ω rows per RAS-T item
  DBuf<int32_t> rast_agg, rast_row;   // RAS-T work items, colour-sorted: (aggregate, Ω row)
  std::vector<int64_t> rast_color_off;  // host, n_colors + 1
};

constexpr int kLaneMaxSub = 48;
constexpr int kRowsCh = 4;  // ω rows per RAS item in the row layout when nΩ <= 128
constexpr int64_t kRowsMinBlk = 0;  // larger blocks use the row layout (warp per output row)
constexpr int kLaneMaxOmega = 24;

// build_smoother (smoother.hpp:38-58): extract A(Ω,Ω), Cholesky with the
// jitter retry of factor_spd_block (dense.hpp:175-185), explicit ω columns of
// the inverse. Throws SetupError for the first failing aggregate.
// h_gamma (optional): the host copy of the Γ lists, needed for the one-launch RAS-T slots
void build_smoother(const DevCsr& a, const DevTopo& topo, const std::vector<int32_t>& h_omega_off,
                    const std::vector<int32_t>& h_gamma_off, const std::vector<int64_t>& colors, int64_t n_colors,
                    DevSmoother& sm, cudaStream_t s, const std::vector<int32_t>* h_gamma = nullptr);

struct GevpParams {
  double thresh;
  double must_keep;
  int variant;
  int level;
  int64_t ratio;
  int64_t level0_max_modes;
};

// Interpolation of one level: dense panels (nω_i × k_i, row-major) plus P
// in CSR with exact zeros dropped (assemble_P, hierarchy.hpp:72-95).
struct DevInterp {
  int64_t n_coarse = 0;
  std::vector<int32_t> h_k;  // k_i
  DBuf<int32_t> coarse_off;  // n_agg + 1
  DBuf<int64_t> panel_off;   // n_agg + 1
  DBuf<double> panels;
  std::vector<std::vector<double>> spectra;  // per aggregate (host)
};

// local_gevp for every aggregate (splitting.hpp:200-275) + assemble_P.
void local_gevp_all(const DevCsr& g, const DevTopo& topo, const std::vector<int32_t>& h_omega_off,
                    const std::vector<int32_t>& h_gamma_off, const DevRowSets& rs, const std::vector<int64_t>& h_nz_off,
                    const GevpParams& gp, DevInterp& ip, DevCsr& p, bool keep_spectra, cudaStream_t s);

// Local Grams of large subdomains as multi-CTA tiles (grams.cu): for each
// listed aggregate, L (nω²), W (nω²), C (nω×nΓ), B (nΓ²) row-major at
// out + out_off[agg], bit-identical to the per-aggregate sweep.
constexpr int64_t kTileMinSub = 96;
constexpr int64_t kTileMaxSub = 4096;
int64_t pre_gram_doubles(int64_t nw, int64_t ng);
void tiled_grams(const DevCsr& gm, const DevTopo& topo, const std::vector<int32_t>& hoo,
                 const std::vector<int32_t>& hgo, const DevRowSets& rs, const std::vector<int64_t>& h_nz_off,
                 const std::vector<int32_t>& aggs, int weighted_lhs, double* out, const int64_t* d_out_off,
                 cudaStream_t s);

// One dense eigensolve through a chosen device path (0 warp team, 1 CTA
// team, 2 CTA pipelined); returns 0 or the EigError code. Test hook.
int dense_sym_eig(int64_t n, const double* a, double* vals, double* vecs, int path, cudaStream_t s);

// Dense Cholesky of the coarsest matrix with the jitter retry, returning the
// full explicit inverse (row-major) for the coarse solve (hierarchy.hpp:193).
void coarse_factor(const DevCsr& a, DBuf<double>& inv, cudaStream_t s);

}  // namespace lsb
