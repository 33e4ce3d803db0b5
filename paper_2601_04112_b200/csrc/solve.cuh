// solve.cuh — V-cycle and PCG kernels (hierarchy.hpp:205-229, krylov.hpp:42-92).
#pragma once

#include "common.cuh"
#include "setup_kernels.cuh"
#include "sparse.cuh"

namespace lsb {

struct SchwarzView {
  int64_t n_agg;
  const int32_t* omega_off;
  const int32_t* omega;
  const int32_t* gamma_off;
  const int32_t* gamma;
  const int64_t* sm_off;
  const double* sm_data;
  const int32_t* order;  // colour-sorted aggregate ids
  int64_t max_omega, max_sub;
  // lane-interleaved groups (small subdomains), see DevSmoother
  int64_t n_groups;
  const int32_t* g_nw;
  const int32_t* g_ng;
  const int32_t* g_cnt;
  const int64_t* g_ids_off;
  const int64_t* g_blk_off;
  const int32_t* lane_ids;
  const double* lane_blk;
  const std::vector<int64_t>* color_goff;
  const int32_t* lane_ras_items;
  int64_t n_lane_ras_items;
  const int32_t* lane_rast_items;
  const std::vector<int64_t>* lane_rast_color_off;
  // persistent TMA-pipelined sweep (k_schwarz_tma)
  const int32_t* g_color;
  const int32_t* color_groups;
  int n_colors;
  int64_t stage_blk_bytes, stage_ids_bytes;
  // one-launch RAS-T: per-node slots of the Γ contributions
  double* rast_tmp;
  const int64_t* g_slot_off;
  const int32_t* lane_slots;
  const int32_t* node_slot_off;
  int64_t n_slots, stage_slot_bytes, n_nodes;
  // row layout (large subdomains), see DevSmoother
  bool rows;
  const int64_t* row_off;
  const double* row_data;
  const int32_t* ras_agg;
  const int32_t* ras_row;
  int64_t n_ras_items;
  int ras_ch;   // ω rows per RAS item (DevSmoother::ras_ch)
  int rast_ch;  // Ω rows per RAS-T item (DevSmoother::rast_ch)
  const int32_t* rast_agg;
  const int32_t* rast_row;
  const std::vector<int64_t>* rast_color_off;
};

// RAS (smoother.hpp:65-83, mode RAS): e[ω_i] = (A_i⁻¹ r[Ω_i])|ω  (accumulate
// adds into e instead of overwriting). ω sets are disjoint: no atomics.
void schwarz_ras(const SchwarzView& v, const double* r, double* e, bool accumulate, cudaStream_t s);
// RAS-T: e[Ω_i] += A_i⁻¹ [r[ω_i]; 0], launched colour by colour (subdomains of
// one colour are disjoint, aggregation.hpp:197-229), so plain read-modify-
// writes are race-free and the sum order is deterministic.
void schwarz_rast(const SchwarzView& v, const std::vector<int64_t>& color_off, const double* r, double* e,
                  cudaStream_t s);

struct InterpView {
  int64_t n_fine, n_coarse, n_agg;
  const int32_t* node_agg;
  const int32_t* node_pos;
  const int32_t* omega_off;
  const int32_t* omega;
  const int32_t* coarse_off;
  const int64_t* panel_off;
  const double* panels;
  const int32_t* col_agg;  // aggregate of every coarse column
};

// rc = Pᵀ res (spmv_transpose, sparse.hpp:125-137): owner-computes per coarse
// column, fine rows in ascending order — bit-identical to the scatter.
// rc = Pᵀ res. `exact`: always the thread-per-column kernel (fine rows
// ascending, the reference's spmv_transpose order, sparse.hpp:125-137); the
// V-cycle lets large aggregates use a warp-per-column tree sum instead.
void restrict_pt(const InterpView& v, const double* res, double* rc, cudaStream_t s, bool exact = false);
// e += P ec (spmv + axpy, hierarchy.hpp:220): per fine row, panel order
// (`exact`, the level_spmv export); the V-cycle uses a warp per fine row
// (tree sum) when the panels are wide.
void prolong_add(const InterpView& v, const double* ec, double* e, cudaStream_t s, bool exact = false);
// e = M r with the explicit coarsest inverse
void dense_matvec(const double* m, int64_t n, const double* r, double* e, cudaStream_t s);

// Deterministic dot product: fixed grid, fixed-order tree, last-block final
// sum. Writes the result to *out (device).
struct Reducer {
  int nblocks = 0;
  DBuf<double> partial;
  DBuf<unsigned int> ticket;
  void init(cudaStream_t s);
};

struct PcgScalars {
  double rz, pap, alpha, beta, rn2, rz_next, r0_2, pad;
};

void dot(const Reducer& red, const double* x, const double* y, int64_t n, double* out, cudaStream_t s);

// PCG building blocks (krylov.hpp:61-80), scalars kept on the device.
void pcg_ap_dot(const Sell& gt, const double* gp, const double* p, double* ap, const Reducer& red, PcgScalars* sc,
                cudaStream_t s);
void pcg_update_xr(const Reducer& red, double* x, double* r, const double* p, const double* ap, int64_t n,
                   PcgScalars* sc, cudaStream_t s);
void pcg_rz(const Reducer& red, const double* r, const double* z, int64_t n, PcgScalars* sc, bool first,
            cudaStream_t s);
void pcg_update_p(double* p, const double* z, int64_t n, const PcgScalars* sc, bool first, cudaStream_t s);

}  // namespace lsb
