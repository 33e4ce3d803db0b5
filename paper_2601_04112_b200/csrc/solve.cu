// solve.cu — the V-cycle and PCG hot loop on sm_100a.
//
// The level-0 Schwarz sweep is the dominant HBM stream of the solve
// (75-80% of the reference's solve time). Each warp
// stages one aggregate's inverse block (the ω columns only: packed ω×ω upper
// triangle + ω×Γ, the part RAS/RAS-T read) and its residual patch in shared
// memory with coalesced loads, then one lane per output row forms its dot
// product. Grids are persistent, sized in multiples of the SM count.
#include <algorithm>
#include <atomic>

#include "solve.cuh"

namespace lsb {

namespace {

extern __shared__ double smem_solve[];

__device__ __forceinline__ int64_t pidx(int i, int j, int nw) {  // i <= j, row-major packed upper
  return int64_t(i) * nw - (int64_t(i) * (i - 1)) / 2 + (j - i);
}

// MODE 0: RAS overwrite, 1: RAS accumulate, 2: RAS-T accumulate
template <int MODE, class Team>
__device__ __forceinline__ void schwarz_one(const Team& t, const SchwarzView& v, int a, const double* __restrict__ r,
                                            double* __restrict__ e, double* sb, double* sr) {
  const int32_t* om = v.omega + v.omega_off[a];
  const int nw = v.omega_off[a + 1] - v.omega_off[a];
  const int32_t* ga = v.gamma + v.gamma_off[a];
  const int ng = v.gamma_off[a + 1] - v.gamma_off[a];
  const int m = nw + ng;
  const int64_t p0 = int64_t(nw) * (nw + 1) / 2;
  const int64_t nblk = p0 + int64_t(nw) * ng;
  const double* blk = v.sm_data + v.sm_off[a];
  if (MODE < 2) {
    for (int i = t.rank(); i < m; i += t.size()) sr[i] = __ldg(&r[i < nw ? om[i] : ga[i - nw]]);
  } else {
    for (int i = t.rank(); i < nw; i += t.size()) sr[i] = __ldg(&r[om[i]]);
  }
  const double* B = blk;
  if (sb) {
    for (int64_t q = t.rank(); q < nblk; q += t.size()) sb[q] = __ldcs(&blk[q]);
    B = sb;
  }
  t.sync();
  if (MODE < 2) {
    for (int i = t.rank(); i < nw; i += t.size()) {
      double s = 0.0;
      for (int j = 0; j < nw; ++j) s += B[i <= j ? pidx(i, j, nw) : pidx(j, i, nw)] * sr[j];
      const double* rowg = B + p0 + int64_t(i) * ng;
      for (int g = 0; g < ng; ++g) s += rowg[g] * sr[nw + g];
      if (MODE == 0)
        e[om[i]] = s;
      else
        e[om[i]] += s;
    }
  } else {
    for (int j = t.rank(); j < m; j += t.size()) {
      double s = 0.0;
      if (j < nw) {
        for (int i = 0; i < nw; ++i) s += B[i <= j ? pidx(i, j, nw) : pidx(j, i, nw)] * sr[i];
        e[om[j]] += s;
      } else {
        const int g = j - nw;
        for (int i = 0; i < nw; ++i) s += B[p0 + int64_t(i) * ng + g] * sr[i];
        e[ga[g]] += s;
      }
    }
  }
  t.sync();
}

template <int MODE, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_schwarz_warp(SchwarzView v, const int32_t* list, int64_t count,
                                                           const double* r, double* e, int stage, int rstage) {
  WarpTeam t;
  const int warp = threadIdx.x >> 5;
  double* sb = smem_solve + int64_t(warp) * (stage + rstage);
  double* sr = sb + stage;
  for (int64_t idx = int64_t(blockIdx.x) * WPB + warp; idx < count; idx += int64_t(gridDim.x) * WPB) {
    const int a = list ? list[idx] : static_cast<int>(idx);
    schwarz_one<MODE>(t, v, a, r, e, sb, sr);
  }
}

template <int MODE>
__global__ void k_schwarz_block(SchwarzView v, const int32_t* list, int64_t count, const double* r, double* e,
                                int stage, int rstage) {
  BlockTeam t;
  double* sb = stage > 0 ? smem_solve : nullptr;
  double* sr = smem_solve + stage;
  for (int64_t idx = blockIdx.x; idx < count; idx += gridDim.x) {
    const int a = list ? list[idx] : static_cast<int>(idx);
    schwarz_one<MODE>(t, v, a, r, e, sb, sr);
  }
}

template <int MODE>
void schwarz_launch(const SchwarzView& v, const int32_t* list, int64_t count, const double* r, double* e,
                    cudaStream_t s) {
  if (count == 0) return;
  const int64_t max_blk = v.max_omega * (v.max_omega + 1) / 2 + v.max_omega * (v.max_sub - v.max_omega);
  const int rstage = static_cast<int>((v.max_sub + 1) & ~int64_t(1));
  if (max_blk <= 2048 && v.max_sub <= 512) {
    constexpr int WPB = 8;
    const int stage = static_cast<int>((max_blk + 1) & ~int64_t(1));
    const size_t smem = size_t(WPB) * (stage + rstage) * 8;
    static std::atomic<uint64_t> attr_set{0};  // per device (the attribute is per device)
    if (first_on_device(attr_set))
      LSB_CUDA(cudaFuncSetAttribute(k_schwarz_warp<MODE, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(8, (200 * 1024) / std::max<size_t>(smem, 1)));
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, WPB), sm_count() * per_sm)));
    k_schwarz_warp<MODE, WPB><<<grid, WPB * 32, smem, s>>>(v, list, count, r, e, stage, rstage);
  } else {
    const int stage = max_blk <= 24000 ? static_cast<int>((max_blk + 1) & ~int64_t(1)) : 0;
    const size_t smem = size_t(stage + rstage) * 8;
    static std::atomic<uint64_t> attr_set_b{0};
    if (first_on_device(attr_set_b))
      LSB_CUDA(cudaFuncSetAttribute(k_schwarz_block<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    const int grid = static_cast<int>(std::min<int64_t>(count, int64_t(sm_count()) * 4));
    k_schwarz_block<MODE><<<grid, 256, smem, s>>>(v, list, count, r, e, stage, rstage);
  }
  LSB_LAUNCH();
}

// Lane-per-aggregate sweep over groups of 32 same-shape aggregates stored
// lane-interleaved ([element][lane]): every block load is a 256-byte warp
// transaction and each lane streams its own block with no cross-lane
// dependency, so a warp keeps hundreds of independent loads in flight. Per
// lane the residual patch and the outputs live in a private shared-memory
// column. MODE 0: RAS overwrite, 1: RAS accumulate, 2: RAS-T accumulate.
template <int MODE>
__global__ void __launch_bounds__(256) k_schwarz_lane(SchwarzView v, int64_t g_begin, int64_t g_end,
                                                      const double* __restrict__ r, double* __restrict__ e, int big,
                                                      int small) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* wbuf = smem_solve + int64_t(warp) * (big + small) * 32;
  // RAS reads r[Ω] (big) and forms y[ω] (small); RAS-T the other way round
  double* R = MODE < 2 ? wbuf : wbuf + int64_t(big) * 32;
  double* Y = MODE < 2 ? wbuf + int64_t(big) * 32 : wbuf;
  const int64_t wstride = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t g = g_begin + int64_t(blockIdx.x) * (blockDim.x >> 5) + warp; g < g_end; g += wstride) {
    const int nw = v.g_nw[g], ng = v.g_ng[g];
    const int m = nw + ng;
    const int32_t* ids = v.lane_ids + v.g_ids_off[g];
    const double* __restrict__ blk = v.lane_blk + v.g_blk_off[g] + lane;
    const int nin = MODE < 2 ? m : nw;
    const int nout = MODE < 2 ? nw : m;
#pragma unroll 8
    for (int q = 0; q < nin; ++q) {
      const int id = ids[q * 32 + lane];
      R[q * 32 + lane] = id >= 0 ? __ldg(&r[id]) : 0.0;
    }
    for (int q = 0; q < nout; ++q) Y[q * 32 + lane] = 0.0;
    int64_t k = 0;
    for (int i = 0; i < nw; ++i) {  // packed ω×ω upper triangle
      const double ri = R[i * 32 + lane];
      double yi = Y[i * 32 + lane];
#pragma unroll 4
      for (int j = i; j < nw; ++j) {
        const double val = __ldcs(&blk[(k + (j - i)) * 32]);
        yi += val * R[j * 32 + lane];
        if (j != i) Y[j * 32 + lane] += val * ri;
      }
      Y[i * 32 + lane] = yi;
      k += nw - i;
    }
    if (MODE < 2) {
      for (int i = 0; i < nw; ++i) {  // ω×Γ rows
        double yi = Y[i * 32 + lane];
        const double* bi = blk + (k + int64_t(i) * ng) * 32;
#pragma unroll 8
        for (int gg = 0; gg < ng; ++gg) yi += __ldcs(&bi[int64_t(gg) * 32]) * R[(nw + gg) * 32 + lane];
        Y[i * 32 + lane] = yi;
      }
      for (int i = 0; i < nw; ++i) {
        const int id = ids[i * 32 + lane];
        if (id < 0) continue;
        if (MODE == 0)
          e[id] = Y[i * 32 + lane];
        else
          e[id] += Y[i * 32 + lane];
      }
    } else {
      for (int i = 0; i < nw; ++i) {  // ω×Γ feeds the Γ outputs
        const double ri = R[i * 32 + lane];
        const double* bi = blk + (k + int64_t(i) * ng) * 32;
#pragma unroll 8
        for (int gg = 0; gg < ng; ++gg) Y[(nw + gg) * 32 + lane] += __ldcs(&bi[int64_t(gg) * 32]) * ri;
      }
      for (int q = 0; q < m; ++q) {
        const int id = ids[q * 32 + lane];
        if (id >= 0) e[id] += Y[q * 32 + lane];
      }
    }
  }
}

template <int MODE>
void schwarz_lane_launch(const SchwarzView& v, int64_t g_begin, int64_t g_end, const double* r, double* e,
                         cudaStream_t s) {
  if (g_end <= g_begin) return;
  const int big = static_cast<int>(v.max_sub), small = static_cast<int>(v.max_omega);
  constexpr int WPB = 8;
  const size_t smem = size_t(WPB) * (big + small) * 32 * 8;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr))
    LSB_CUDA(cudaFuncSetAttribute(k_schwarz_lane<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  const int64_t per_sm = std::max<int64_t>(1, (220 * 1024) / std::max<size_t>(smem, 1));
  const int grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(g_end - g_begin, WPB), int64_t(sm_count()) * std::min<int64_t>(per_sm, 8))));
  k_schwarz_lane<MODE><<<grid, WPB * 32, smem, s>>>(v, g_begin, g_end, r, e, big, small);
  LSB_LAUNCH();
}

// Lane-interleaved groups, one warp per (group, output row): lane l computes
// row `row` of aggregate l of the group, so every block load is one 256-byte
// warp transaction and each lane has nΩ (RAS) or nω (RAS-T) independent
// loads in flight. The ω×ω triangle is read by both of its rows (L1 keeps
// the second read on chip: the rows of a group are consecutive items).
// Fully unrolled row of a group with the dominant interior shape (NW, NG):
// every block and residual load of the lane is issued before the first use.
template <int MODE, int NW, int NG>
__device__ __forceinline__ double lrow_fixed(const int32_t* __restrict__ ids, const double* __restrict__ blk, int row,
                                             const double* __restrict__ r) {
  constexpr int P0 = NW * (NW + 1) / 2;
  double s0 = 0.0, s1 = 0.0;
  if (MODE < 2) {
    double rv[NW + NG], bv[NW + NG];
#pragma unroll
    for (int j = 0; j < NW + NG; ++j) {
      const int id = ids[j * 32];
      rv[j] = id >= 0 ? __ldg(&r[id]) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const int lo = row < j ? row : j, hi = row < j ? j : row;
      const int k = lo * NW - (lo * (lo - 1)) / 2 + (hi - lo);
      bv[j] = __ldg(&blk[k * 32]);
    }
#pragma unroll
    for (int q = 0; q < NG; ++q) bv[NW + q] = __ldcs(&blk[(P0 + row * NG + q) * 32]);
#pragma unroll
    for (int j = 0; j < NW + NG; ++j) {
      if (j & 1)
        s1 += bv[j] * rv[j];
      else
        s0 += bv[j] * rv[j];
    }
  } else {
    double rv[NW], bv[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const int id = ids[i * 32];
      rv[i] = id >= 0 ? __ldg(&r[id]) : 0.0;
    }
    if (row < NW) {
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int lo = row < i ? row : i, hi = row < i ? i : row;
        const int k = lo * NW - (lo * (lo - 1)) / 2 + (hi - lo);
        bv[i] = __ldg(&blk[k * 32]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < NW; ++i) bv[i] = __ldcs(&blk[(P0 + i * NG + (row - NW)) * 32]);
    }
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      if (i & 1)
        s1 += bv[i] * rv[i];
      else
        s0 += bv[i] * rv[i];
    }
  }
  return s0 + s1;
}

// Launch with programmatic stream serialization (PDL): the kernel's
// griddepcontrol.wait orders it after its predecessor, while its launch and
// CTA rasterisation overlap the predecessor's drain.
static bool pdl_enabled() {
#ifdef LSB_DIAG  // make DIAG=1: LSB_NO_PDL=1 launches the sweeps without programmatic dependent launch
  static const bool on = getenv("LSB_NO_PDL") == nullptr;
  return on;
#else
  return true;
#endif
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  LSB_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

template <int MODE>
__global__ void __launch_bounds__(256) k_schwarz_lrow(SchwarzView v, const int32_t* __restrict__ items, int64_t i0,
                                                      int64_t i1, const double* __restrict__ r,
                                                      double* __restrict__ e) {
  // Programmatic dependent launch (schwarz_lrow_launch): wait for the
  // previous kernel's results, then let the next launch start filling the
  // SMs this grid drains (it waits in turn for this grid to complete).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t it = i0 + blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); it < i1; it += warps) {
    const int code = items[it];
    const int g = code >> 8, row = code & 255;
    const int nw = v.g_nw[g], ng = v.g_ng[g];
    const int32_t* ids = v.lane_ids + v.g_ids_off[g] + lane;
    const double* __restrict__ blk = v.lane_blk + v.g_blk_off[g] + lane;
    const int64_t p0 = int64_t(nw) * (nw + 1) / 2;
    const int out = ids[row * 32];
    if (nw == 9 && ng == 16) {  // 3x3 aggregates with overlap 1 (config 2 interior)
      const double sum = lrow_fixed<MODE, 9, 16>(ids, blk, row, r);
      if (out >= 0) {
        if (MODE == 0)
          e[out] = sum;
        else
          e[out] += sum;
      }
      continue;
    }
    double s0 = 0.0, s1 = 0.0;
    if (MODE < 2) {
#pragma unroll 4
      for (int j = 0; j < nw; ++j) {
        const int lo = row < j ? row : j, hi = row < j ? j : row;
        const int64_t k = int64_t(lo) * nw - (int64_t(lo) * (lo - 1)) / 2 + (hi - lo);
        const int id = ids[j * 32];
        const double rv = id >= 0 ? __ldg(&r[id]) : 0.0;
        if (j & 1)
          s1 += __ldg(&blk[k * 32]) * rv;
        else
          s0 += __ldg(&blk[k * 32]) * rv;
      }
      const double* bg = blk + (p0 + int64_t(row) * ng) * 32;
#pragma unroll 8
      for (int q = 0; q < ng; ++q) {
        const int id = ids[(nw + q) * 32];
        const double rv = id >= 0 ? __ldg(&r[id]) : 0.0;
        if (q & 1)
          s1 += __ldcs(&bg[int64_t(q) * 32]) * rv;
        else
          s0 += __ldcs(&bg[int64_t(q) * 32]) * rv;
      }
    } else if (row < nw) {
#pragma unroll 4
      for (int i = 0; i < nw; ++i) {
        const int lo = row < i ? row : i, hi = row < i ? i : row;
        const int64_t k = int64_t(lo) * nw - (int64_t(lo) * (lo - 1)) / 2 + (hi - lo);
        const int id = ids[i * 32];
        const double rv = id >= 0 ? __ldg(&r[id]) : 0.0;
        if (i & 1)
          s1 += __ldg(&blk[k * 32]) * rv;
        else
          s0 += __ldg(&blk[k * 32]) * rv;
      }
    } else {
      const double* bg = blk + (p0 + (row - nw)) * 32;
#pragma unroll 4
      for (int i = 0; i < nw; ++i) {
        const int id = ids[i * 32];
        const double rv = id >= 0 ? __ldg(&r[id]) : 0.0;
        if (i & 1)
          s1 += __ldcs(&bg[int64_t(i) * ng * 32]) * rv;
        else
          s0 += __ldcs(&bg[int64_t(i) * ng * 32]) * rv;
      }
    }
    if (out >= 0) {
      const double sum = s0 + s1;
      if (MODE == 0)
        e[out] = sum;
      else
        e[out] += sum;
    }
  }
}

template <int MODE>
void schwarz_lrow_launch(const SchwarzView& v, const int32_t* items, int64_t i0, int64_t i1, const double* r, double* e,
                         cudaStream_t s) {
  if (i1 <= i0) return;
  // one full wave of resident CTAs (grid-stride over the items): a partial
  // last wave left most SMs idle during the drain (ncu: 3.2 waves for MODE 2)
  const int resident = [] {  // per call: launches are captured once per solve, and the value is per device
    int b = 0;
    LSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_schwarz_lrow<MODE>, 256, 0));
    return std::max(b, 1);
  }();
  const int grid = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(ceil_div(i1 - i0, 8), int64_t(sm_count()) * resident)));
  launch_pdl(k_schwarz_lrow<MODE>, grid, 256, s, v, items, i0, i1, r, e);
  LSB_LAUNCH();
}

// ---- persistent TMA-pipelined sweep over the lane-interleaved groups --------------------
//
// One CTA per SM walks the groups g = blockIdx.x, blockIdx.x + gridDim.x, …
// (the groups are colour-sorted). A producer thread streams each group's
// contiguous block ([nblk][32] doubles, ~48 KB for 3×3 aggregates with
// overlap 1) and index list ([nΩ][32] int32) into a ring of shared-memory
// stages with two 1-D bulk copies (cp.async.bulk, completion on an mbarrier);
// nine consumer warps gather the group's r values once into shared memory,
// compute one output row per warp and lane (lane = aggregate of the group)
// from the staged block and release the stage. HBM sees only long bulk reads;
// the LSU handles just the r gather and the e scatter.
// RAS-T (MODE 2): the ω rows add into e directly (interiors are disjoint), the Γ
// rows store their contributions into per-node slots that k_rast_slots sums in
// ascending holder order afterwards — one launch, no ordering between groups,
// deterministic sums. The stage ring is shared by the consumer teams; the
// producer tags each stage with its group's sequence number so that a team's
// mbarrier parity wait cannot alias a phase another team has yet to consume.
constexpr int kTmaConsumers = 9;  // consumer warps per team
constexpr int kTmaTeams = 3;      // consumer teams; team t takes this CTA's groups k ≡ t (mod 3)
constexpr int kTmaThreads = (kTmaTeams * kTmaConsumers + 1) * 32;  // + one producer warp
constexpr int kTmaHead = 256;     // barriers and per-stage metadata; then r staging [teams][rs_rows][32], then the stages

// One output row of a group of compile-time shape (NW, NG) from the staged block (blk, rs already
// offset by the lane): every shared load is issued before the sums; same summation order as the
// generic loop (even terms into s0, odd into s1).
template <int MODE, int NW, int NG>
__device__ __forceinline__ double tma_row_fixed(const double* blk, const double* rs, int row) {
  constexpr int P0 = NW * (NW + 1) / 2;
  double s0 = 0.0, s1 = 0.0;
  if (MODE < 2 || row < NW) {
    double bv[NW], rv[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const int lo = row < j ? row : j, hi = row < j ? j : row;
      bv[j] = blk[(lo * NW - (lo * (lo - 1)) / 2 + (hi - lo)) * 32];
      rv[j] = rs[j * 32];
    }
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      if (j & 1)
        s1 += bv[j] * rv[j];
      else
        s0 += bv[j] * rv[j];
    }
    if (MODE < 2) {
      const double* bg = blk + (P0 + row * NG) * 32;
      double gv[NG], gr[NG];
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        gv[q] = bg[q * 32];
        gr[q] = rs[(NW + q) * 32];
      }
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        if (q & 1)
          s1 += gv[q] * gr[q];
        else
          s0 += gv[q] * gr[q];
      }
    }
  } else {
    const double* bg = blk + (P0 + (row - NW)) * 32;
    double bv[NW], rv[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      bv[i] = bg[i * NG * 32];
      rv[i] = rs[i * 32];
    }
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      if (i & 1)
        s1 += bv[i] * rv[i];
      else
        s0 += bv[i] * rv[i];
    }
  }
  return s0 + s1;
}

__device__ __forceinline__ uint32_t s_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void s_mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void s_mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(s_u32(bar)), "r"(parity)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void s_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ void s_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s_u32(dst)),
               "l"(src), "r"(bytes), "r"(s_u32(bar))
               : "memory");
}

// MODE 2 (RAS-T): the ω rows add into e directly (the interiors are disjoint); the Γ rows store
// their contributions into per-node slots (tmp, L2-resident), which k_rast_slots adds into e.
template <int MODE>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k_schwarz_tma(SchwarzView v, const double* __restrict__ r, double* __restrict__ e, double* __restrict__ tmp,
                  int n_stage, int stage_bytes, int blk_cap, int ids_cap, int rs_rows) {
  extern __shared__ __align__(128) unsigned char tma_smem[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint64_t* full = reinterpret_cast<uint64_t*>(tma_smem);  // [8]
  uint64_t* empty = full + 8;                                // [8]
  int4* meta = reinterpret_cast<int4*>(tma_smem + 128);      // [8] {nω, nΓ, -, -}
  double* rs_all = reinterpret_cast<double*>(tma_smem + kTmaHead);
  unsigned char* stages = tma_smem + kTmaHead + ((kTmaTeams * rs_rows * 32 * 8 + 127) & ~127);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int k = 0; k < n_stage; ++k) {
      s_mbar_init(&full[k], 1);
      s_mbar_init(&empty[k], kTmaConsumers);
      meta[k] = make_int4(0, 0, -1, 0);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ng_total = v.n_groups;
  if (warp == kTmaTeams * kTmaConsumers) {  // producer
    if (lane == 0) {
      int k = 0;
      for (int64_t g = blockIdx.x; g < ng_total; g += gridDim.x, ++k) {
        const int st = k % n_stage;
        const int64_t b0 = v.g_blk_off[g], i0 = v.g_ids_off[g];
        const uint32_t bb = static_cast<uint32_t>((v.g_blk_off[g + 1] - b0) * 8);
        const uint32_t ib = static_cast<uint32_t>((v.g_ids_off[g + 1] - i0) * 4);
        const int64_t s0 = MODE == 2 ? v.g_slot_off[g] : 0;
        const uint32_t sb = MODE == 2 ? static_cast<uint32_t>((v.g_slot_off[g + 1] - s0) * 4) : 0u;
        const int4 mt = make_int4(v.g_nw[g], v.g_ng[g], k, 0);  // .z: the sequence number the consumers check
        if (k >= n_stage) s_mbar_wait(&empty[st], ((k / n_stage) - 1) & 1);
        meta[st] = mt;
        unsigned char* dst = stages + int64_t(st) * stage_bytes;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[st])), "r"(bb + ib + sb)
                     : "memory");
        s_bulk_load(dst, v.lane_blk + b0, bb, &full[st]);
        s_bulk_load(dst + blk_cap, v.lane_ids + i0, ib, &full[st]);
        if (MODE == 2 && sb) s_bulk_load(dst + blk_cap + ids_cap, v.lane_slots + s0, sb, &full[st]);
      }
    }
  } else {  // consumer teams
    const int team = warp / kTmaConsumers, cw = warp % kTmaConsumers;
    double* rs = rs_all + team * (rs_rows * 32);
    auto cbar = [team]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "n"(kTmaConsumers * 32) : "memory"); };
    int k = team;
    for (int64_t g = blockIdx.x + int64_t(team) * gridDim.x; g < ng_total; g += int64_t(kTmaTeams) * gridDim.x, k += kTmaTeams) {
      const int st = k % n_stage;
      // A stage's phases are consumed by the three teams in turn, so a team does not observe every
      // phase of its `full` barrier, and a parity wait alone cannot tell "phase k/n_stage complete"
      // from "two phases behind" (a fill that completes late while this team has already finished
      // its previous group: the parities coincide and the team would read a stage still being
      // filled for an earlier group). The producer tags the stage with the group's sequence number
      // before it arms the barrier; the parity wait starts only once the tag is this team's group.
      {
        const volatile int* seq = reinterpret_cast<const volatile int*>(&meta[st]) + 2;
        while (*seq != k) __nanosleep(20);
      }
      s_mbar_wait(&full[st], (k / n_stage) & 1);
      const int4 mt = meta[st];
      const int nw = mt.x, ngm = mt.y, m = nw + ngm;
      const unsigned char* base = stages + int64_t(st) * stage_bytes;
      const double* blk = reinterpret_cast<const double*>(base) + lane;
      const int32_t* ids = reinterpret_cast<const int32_t*>(base + blk_cap) + lane;
      const int32_t* slots = reinterpret_cast<const int32_t*>(base + blk_cap + ids_cap) + lane;
      const int nr = MODE < 2 ? m : nw;
      const int p0 = nw * (nw + 1) / 2;
      const int nout = MODE < 2 ? nw : m;
      // this warp's rows: cw, cw + 9, …
      constexpr int kMaxRows = (kLaneMaxSub + kTmaConsumers - 1) / kTmaConsumers;
      // Every global load of the group (the warp's share of the r gather and the old e of its ω rows)
      // is issued before the first one is used: one trip to L2/HBM per group instead of one per row.
      int gid[kMaxRows], outs[kMaxRows];
      double gval[kMaxRows], eold[kMaxRows];
#pragma unroll
      for (int q = 0; q < kMaxRows; ++q) {
        const int row = cw + q * kTmaConsumers;
        gid[q] = row < nr ? ids[row * 32] : -1;
        // ω rows: the node; Γ rows of RAS-T: the slot of the contribution
        outs[q] = row < nout ? ((MODE == 2 && row >= nw) ? slots[(row - nw) * 32] : ids[row * 32]) : -1;
      }
#pragma unroll
      for (int q = 0; q < kMaxRows; ++q) gval[q] = gid[q] >= 0 ? __ldcg(&r[gid[q]]) : 0.0;
#pragma unroll
      for (int q = 0; q < kMaxRows; ++q) {
        const int row = cw + q * kTmaConsumers;
        eold[q] = (MODE != 0 && row < nw && outs[q] >= 0) ? e[outs[q]] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kMaxRows; ++q) {
        const int row = cw + q * kTmaConsumers;
        if (row < nr) rs[row * 32 + lane] = gval[q];
      }
      cbar();
#pragma unroll
      for (int q = 0; q < kMaxRows; ++q) {
        const int row = cw + q * kTmaConsumers;
        if (row >= nout) break;
        double s0 = 0.0, s1 = 0.0;
        if (nw == 9 && ngm == 16) {  // 3×3 aggregates with overlap 1 (config 2 interior)
          s0 = tma_row_fixed<MODE, 9, 16>(blk, rs + lane, row);
        } else if (MODE < 2 || row < nw) {  // the ω×ω triangle, then (RAS) the row of the ω×Γ block
#pragma unroll 3
          for (int j = 0; j < nw; ++j) {
            const int lo = row < j ? row : j, hi = row < j ? j : row;
            const int kk = lo * nw - (lo * (lo - 1)) / 2 + (hi - lo);
            const double pr = blk[kk * 32] * rs[j * 32 + lane];
            if (j & 1)
              s1 += pr;
            else
              s0 += pr;
          }
          if (MODE < 2) {
            const double* bg = blk + (p0 + row * ngm) * 32;
#pragma unroll 4
            for (int qq = 0; qq < ngm; ++qq) {
              const double pr = bg[qq * 32] * rs[(nw + qq) * 32 + lane];
              if (qq & 1)
                s1 += pr;
              else
                s0 += pr;
            }
          }
        } else {  // RAS-T, Γ row: column (row - nω) of the ω×Γ block
          const double* bg = blk + (p0 + (row - nw)) * 32;
#pragma unroll 3
          for (int i = 0; i < nw; ++i) {
            const double pr = bg[i * ngm * 32] * rs[i * 32 + lane];
            if (i & 1)
              s1 += pr;
            else
              s0 += pr;
          }
        }
        if (outs[q] >= 0) {
          const double sum = s0 + s1;
          if (MODE == 2 && row >= nw)
            tmp[outs[q]] = sum;
          else if (MODE == 0)
            e[outs[q]] = sum;
          else
            e[outs[q]] = eold[q] + sum;
        }
      }
      cbar();  // every row of the group is out; rs and the stage may be reused
      if (lane == 0) s_mbar_arrive(&empty[st]);
    }
  }
}

// e[v] += Σ slots of node v, in slot order (ascending holder aggregate): second step of the one-launch RAS-T
__global__ void __launch_bounds__(256) k_rast_slots(const int32_t* __restrict__ off, const double* __restrict__ tmp,
                                                    int64_t n, double* __restrict__ e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n; v += int64_t(gridDim.x) * blockDim.x) {
    const int a = off[v], b = off[v + 1];
    if (b > a) {
      double s = 0.0;
      for (int k = a; k < b; ++k) s += tmp[k];
      e[v] += s;
    }
  }
}

// true when the launch ran (lane layout present and at least two stages fit)
template <int MODE>
bool schwarz_tma_launch(const SchwarzView& v, const double* r, double* e, cudaStream_t s) {
  if (v.n_groups == 0 || v.stage_blk_bytes == 0) return false;
#ifdef LSB_DIAG  // make DIAG=1: LSB_NO_TMA=1 falls back to the lane-layout sweeps (k_schwarz_lrow)
  static const bool no_tma = getenv("LSB_NO_TMA") != nullptr;
  if (no_tma) return false;
#endif
  if (MODE == 2 && (!v.rast_tmp || v.n_slots == 0)) return false;
  const int blk_cap = static_cast<int>((v.stage_blk_bytes + 127) & ~int64_t(127));
  const int ids_cap = static_cast<int>((v.stage_ids_bytes + 127) & ~int64_t(127));
  const int stage_bytes = blk_cap + ids_cap + (MODE == 2 ? static_cast<int>((v.stage_slot_bytes + 127) & ~int64_t(127)) : 0);
  const int rs_rows = static_cast<int>(v.max_sub);
  const int fixed = kTmaHead + ((kTmaTeams * rs_rows * 32 * 8 + 127) & ~127);
  constexpr int kMaxSmem = 226 * 1024;  // 227 KB per CTA minus the kernel's static 1 KB
  const int budget = kMaxSmem - fixed;
  const int n_stage = std::min(8, budget / stage_bytes);
  if (n_stage < 2 || rs_rows > kLaneMaxSub) return false;
  const size_t smem = size_t(fixed) + size_t(n_stage) * stage_bytes;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr))
    LSB_CUDA(cudaFuncSetAttribute(k_schwarz_tma<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
  const int grid = static_cast<int>(std::min<int64_t>(v.n_groups, sm_count()));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTmaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  LSB_CUDA(cudaLaunchKernelEx(&cfg, k_schwarz_tma<MODE>, v, r, e, v.rast_tmp, n_stage, stage_bytes, blk_cap, ids_cap, rs_rows));
  LSB_LAUNCH();
  if (MODE == 2) {
    const int g2 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(v.n_nodes, 256), int64_t(sm_count()) * 8)));
    launch_pdl(k_rast_slots, g2, 256, s, v.node_slot_off, static_cast<const double*>(v.rast_tmp), v.n_nodes, e);
    LSB_LAUNCH();
  }
  return true;
}

// Row layout (large subdomains): one warp per output row, lanes over a
// contiguous row of the explicit inverse, fixed xor-tree reduction (the
// result is deterministic). RAS (MODE 0/1): row i of F · r[Ω] -> e[ω_i];
// RAS-T (MODE 2): row j of [F_ωω; Gt] · r[ω] -> e[Ω_j] += (one colour per
// launch: disjoint Ω, no atomics).
template <int MODE>
__global__ void __launch_bounds__(256) k_schwarz_rows(SchwarzView v, const int32_t* __restrict__ item_agg,
                                                      const int32_t* __restrict__ item_row, int64_t i0, int64_t i1,
                                                      const double* __restrict__ r, double* __restrict__ e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL, see k_schwarz_lrow
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t it = i0 + blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); it < i1; it += warps) {
    const int a = item_agg[it], row = item_row[it];
    const int32_t* om = v.omega + v.omega_off[a];
    const int nw = v.omega_off[a + 1] - v.omega_off[a];
    const int32_t* ga = v.gamma + v.gamma_off[a];
    const int ng = v.gamma_off[a + 1] - v.gamma_off[a];
    const int m = nw + ng;
    const double* F = v.row_data + v.row_off[a];
    double s0 = 0.0, s1 = 0.0;
    if (MODE < 2) {
      const double* fr = F + int64_t(row) * m;
      int j = lane;
      for (; j + 32 < m; j += 64) {
        const int c0 = j < nw ? om[j] : ga[j - nw];
        const int c1 = j + 32 < nw ? om[j + 32] : ga[j + 32 - nw];
        s0 += __ldcs(&fr[j]) * __ldg(&r[c0]);
        s1 += __ldcs(&fr[j + 32]) * __ldg(&r[c1]);
      }
      if (j < m) s0 += __ldcs(&fr[j]) * __ldg(&r[j < nw ? om[j] : ga[j - nw]]);
    } else {
      const double* fr = row < nw ? F + int64_t(row) * m : F + int64_t(nw) * m + int64_t(row - nw) * nw;
      int i = lane;
      for (; i + 32 < nw; i += 64) {
        s0 += __ldcs(&fr[i]) * __ldg(&r[om[i]]);
        s1 += __ldcs(&fr[i + 32]) * __ldg(&r[om[i + 32]]);
      }
      if (i < nw) s0 += __ldcs(&fr[i]) * __ldg(&r[om[i]]);
    }
    double sum = s0 + s1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      if (MODE == 0) {
        e[om[row]] = sum;
      } else if (MODE == 1) {
        e[om[row]] += sum;
      } else {
        const int c = row < nw ? om[row] : ga[row - nw];
        e[c] += sum;
      }
    }
  }
}

// RAS-T rows with L lanes per output row (L < 32 when the level's ω sets are
// short): 32/L items per warp, so the per-item chain of dependent loads
// (item -> offsets -> row and ω ids -> r) overlaps across items instead of
// idling 32 - nω lanes. Sum order: strided lane partial sums, xor tree.
template <int L>
__global__ void __launch_bounds__(256) k_schwarz_rows_t(SchwarzView v, const int32_t* __restrict__ item_agg,
                                                        const int32_t* __restrict__ item_row, int64_t i0, int64_t i1,
                                                        const double* __restrict__ r, double* __restrict__ e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL, see k_schwarz_lrow
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int PER_WARP = 32 / L;
  const int lane = threadIdx.x & 31, sub = lane % L;
  const int64_t teams = int64_t(gridDim.x) * (blockDim.x >> 5) * PER_WARP;
  const int64_t team0 = (blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5)) * PER_WARP + lane / L;
  // every lane of a warp runs the same number of iterations (shuffles need the full warp)
  for (int64_t base = team0 - lane / L; base < i1 - i0; base += teams) {
    const int64_t it = i0 + base + lane / L;
    double sum = 0.0;
    int c = -1;
    if (it < i1) {
      const int a = item_agg[it], row = item_row[it];
      const int32_t* om = v.omega + v.omega_off[a];
      const int nw = v.omega_off[a + 1] - v.omega_off[a];
      const int32_t* ga = v.gamma + v.gamma_off[a];
      const int ng = v.gamma_off[a + 1] - v.gamma_off[a];
      const double* F = v.row_data + v.row_off[a];
      const double* fr = row < nw ? F + int64_t(row) * (nw + ng) : F + int64_t(nw) * (nw + ng) + int64_t(row - nw) * nw;
      double s0 = 0.0, s1 = 0.0;
      int i = sub;
      for (; i + L < nw; i += 2 * L) {
        s0 += __ldcs(&fr[i]) * __ldg(&r[om[i]]);
        s1 += __ldcs(&fr[i + L]) * __ldg(&r[om[i + L]]);
      }
      if (i < nw) s0 += __ldcs(&fr[i]) * __ldg(&r[om[i]]);
      sum = s0 + s1;
      if (sub == 0) c = row < nw ? om[row] : ga[row - nw];
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (c >= 0) e[c] += sum;
  }
}

// RAS on short rows (nΩ <= 128): one warp per chunk of kRowsCh consecutive
// ω rows of one aggregate; the lane's Ω ids and r values (j = lane + 32t) are
// gathered once per chunk, then each row is the same even/odd-split lane sum
// and xor tree as k_schwarz_rows, so the results are bit-identical to it.
template <int MODE>
__global__ void __launch_bounds__(256) k_schwarz_rows_ch(SchwarzView v, const int32_t* __restrict__ item_agg,
                                                         const int32_t* __restrict__ item_row, int64_t i0, int64_t i1,
                                                         const double* __restrict__ r, double* __restrict__ e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL, see k_schwarz_lrow
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t it = i0 + blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); it < i1; it += warps) {
    const int a = item_agg[it], row0 = item_row[it];
    const int32_t* om = v.omega + v.omega_off[a];
    const int nw = v.omega_off[a + 1] - v.omega_off[a];
    const int32_t* ga = v.gamma + v.gamma_off[a];
    const int ng = v.gamma_off[a + 1] - v.gamma_off[a];
    const int m = nw + ng;
    const double* F = v.row_data + v.row_off[a];
    double rv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int j = lane + 32 * t;
      rv[t] = j < m ? __ldg(&r[j < nw ? om[j] : ga[j - nw]]) : 0.0;
    }
    const int rend = row0 + kRowsCh < nw ? row0 + kRowsCh : nw;
    for (int row = row0; row < rend; ++row) {
      const double* fr = F + int64_t(row) * m;
      double f[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) f[t] = lane + 32 * t < m ? __ldcs(&fr[lane + 32 * t]) : 0.0;
      // k_schwarz_rows' order: s0 over t = 0, 2 and s1 over t = 1, 3, each
      // term only where its column exists
      double s0 = 0.0, s1 = 0.0;
      if (lane < m) s0 += f[0] * rv[0];
      if (lane + 32 < m) s1 += f[1] * rv[1];
      if (lane + 64 < m) s0 += f[2] * rv[2];
      if (lane + 96 < m) s1 += f[3] * rv[3];
      double sum = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) {
        if (MODE == 0)
          e[om[row]] = sum;
        else
          e[om[row]] += sum;
      }
    }
  }
}

// RAS-T counterpart of k_schwarz_rows_ch (nω <= 128): chunks of kRowsCh Ω
// rows share one gather of the ω ids and r values; per row the sum order of
// k_schwarz_rows<2> (bit-identical).
__global__ void __launch_bounds__(256) k_schwarz_rows_tch(SchwarzView v, const int32_t* __restrict__ item_agg,
                                                          const int32_t* __restrict__ item_row, int64_t i0,
                                                          int64_t i1, const double* __restrict__ r,
                                                          double* __restrict__ e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL, see k_schwarz_lrow
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t it = i0 + blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); it < i1; it += warps) {
    const int a = item_agg[it], row0 = item_row[it];
    const int32_t* om = v.omega + v.omega_off[a];
    const int nw = v.omega_off[a + 1] - v.omega_off[a];
    const int32_t* ga = v.gamma + v.gamma_off[a];
    const int ng = v.gamma_off[a + 1] - v.gamma_off[a];
    const int m = nw + ng;
    const double* F = v.row_data + v.row_off[a];
    double rv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = lane + 32 * t;
      rv[t] = i < nw ? __ldg(&r[om[i]]) : 0.0;
    }
    const int rend = row0 + kRowsCh < m ? row0 + kRowsCh : m;
    for (int row = row0; row < rend; ++row) {
      const double* fr = row < nw ? F + int64_t(row) * m : F + int64_t(nw) * m + int64_t(row - nw) * nw;
      double f[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) f[t] = lane + 32 * t < nw ? __ldcs(&fr[lane + 32 * t]) : 0.0;
      double s0 = 0.0, s1 = 0.0;
      if (lane < nw) s0 += f[0] * rv[0];
      if (lane + 32 < nw) s1 += f[1] * rv[1];
      if (lane + 64 < nw) s0 += f[2] * rv[2];
      if (lane + 96 < nw) s1 += f[3] * rv[3];
      double sum = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) e[row < nw ? om[row] : ga[row - nw]] += sum;
    }
  }
}

template <int MODE>
void schwarz_rows_launch(const SchwarzView& v, const int32_t* ia, const int32_t* ir, int64_t i0, int64_t i1,
                         const double* r, double* e, cudaStream_t s) {
  if (i1 <= i0) return;
  // grids of one full wave of resident CTAs (see schwarz_lrow_launch)
  auto resident = [](auto kern) {
    int b = 0;
    LSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 0));
    return std::max(b, 1);
  };
  const int res_rows = resident(k_schwarz_rows<MODE>);
  const int grid = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(ceil_div(i1 - i0, 8), int64_t(sm_count()) * res_rows)));
  if (MODE < 2 && v.ras_ch > 1) {
    const int res_ch = resident(k_schwarz_rows_ch<MODE>);
    const int g3 = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(ceil_div(i1 - i0, 8), int64_t(sm_count()) * res_ch)));
    launch_pdl(k_schwarz_rows_ch<MODE>, g3, 256, s, v, ia, ir, i0, i1, r, e);
  } else if (MODE == 2 && v.rast_ch > 1) {
    const int res_tch = resident(k_schwarz_rows_tch);
    const int g3 = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(ceil_div(i1 - i0, 8), int64_t(sm_count()) * res_tch)));
    launch_pdl(k_schwarz_rows_tch, g3, 256, s, v, ia, ir, i0, i1, r, e);
  } else if (MODE == 2 && v.max_omega <= 64) {
    // lanes per row: 4 / 8 / 16 for nω up to 8 / 16 / 64 (≤ 4 entries per lane)
    const int lanes = v.max_omega <= 8 ? 4 : v.max_omega <= 16 ? 8 : 16;
    const int per_warp = 32 / lanes;
    const int res_t = std::min({resident(k_schwarz_rows_t<4>), resident(k_schwarz_rows_t<8>),
                                       resident(k_schwarz_rows_t<16>)});
    const int g2 = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(ceil_div(i1 - i0, 8 * per_warp), int64_t(sm_count()) * res_t)));
    if (lanes == 4)
      launch_pdl(k_schwarz_rows_t<4>, g2, 256, s, v, ia, ir, i0, i1, r, e);
    else if (lanes == 8)
      launch_pdl(k_schwarz_rows_t<8>, g2, 256, s, v, ia, ir, i0, i1, r, e);
    else
      launch_pdl(k_schwarz_rows_t<16>, g2, 256, s, v, ia, ir, i0, i1, r, e);
  } else {
    launch_pdl(k_schwarz_rows<MODE>, grid, 256, s, v, ia, ir, i0, i1, r, e);
  }
  LSB_LAUNCH();
}

__global__ void k_restrict(InterpView v, const double* __restrict__ res, double* __restrict__ rc) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < v.n_coarse; c += int64_t(gridDim.x) * blockDim.x) {
    const int a = v.col_agg[c];
    const int j = static_cast<int>(c - v.coarse_off[a]);
    const int k = v.coarse_off[a + 1] - v.coarse_off[a];
    const double* pan = v.panels + v.panel_off[a];
    const int32_t* om = v.omega + v.omega_off[a];
    const int nw = v.omega_off[a + 1] - v.omega_off[a];
    double s = 0.0;
    for (int rr = 0; rr < nw; ++rr) {
      const double x = res[om[rr]];
      if (x == 0.0) continue;
      s += pan[int64_t(rr) * k + j] * x;
    }
    rc[c] = s;
  }
}

// Pᵀ res with one warp per coarse column (large aggregates): lanes over the
// aggregate's fine rows, fixed xor-tree reduction.
__global__ void __launch_bounds__(256) k_restrict_warp(InterpView v, const double* __restrict__ res,
                                                       double* __restrict__ rc) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); c < v.n_coarse; c += warps) {
    const int a = v.col_agg[c];
    const int j = static_cast<int>(c - v.coarse_off[a]);
    const int k = v.coarse_off[a + 1] - v.coarse_off[a];
    const double* pan = v.panels + v.panel_off[a];
    const int32_t* om = v.omega + v.omega_off[a];
    const int nw = v.omega_off[a + 1] - v.omega_off[a];
    double s = 0.0;
    for (int rr = lane; rr < nw; rr += 32) s += pan[int64_t(rr) * k + j] * res[om[rr]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rc[c] = s;
  }
}

__global__ void k_prolong(InterpView v, const double* __restrict__ ec, double* __restrict__ e) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < v.n_fine; i += int64_t(gridDim.x) * blockDim.x) {
    const int a = v.node_agg[i];
    const int rr = v.node_pos[i];
    const int k = v.coarse_off[a + 1] - v.coarse_off[a];
    const double* row = v.panels + v.panel_off[a] + int64_t(rr) * k;
    const double* x = ec + v.coarse_off[a];
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += row[j] * x[j];
    e[i] += s;
  }
}

// Wide panels (coarse levels, tens to hundreds of modes per aggregate): warp
// per fine row, lanes over the row's contiguous panel entries, xor-tree sum.
__global__ void k_prolong_warp(InterpView v, const double* __restrict__ ec, double* __restrict__ e) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < v.n_fine; i += warps) {
    const int a = v.node_agg[i];
    const int rr = v.node_pos[i];
    const int k = v.coarse_off[a + 1] - v.coarse_off[a];
    const double* row = v.panels + v.panel_off[a] + int64_t(rr) * k;
    const double* x = ec + v.coarse_off[a];
    double s = 0.0;
    for (int j = lane; j < k; j += 32) s += __ldcs(&row[j]) * __ldg(&x[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) e[i] += s;
  }
}

__global__ void k_dense_mv(const double* __restrict__ m, int64_t n, const double* __restrict__ r, double* __restrict__ e) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    double s = 0.0;
    for (int64_t j = lane; j < n; j += 32) s += m[i * n + j] * r[j];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) e[i] = s;
  }
}

int grid_for(int64_t n, int threads = 256) {
  const int64_t cap = int64_t(sm_count()) * 16;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap)));
}

// ---- deterministic reductions ----------------------------------------------------

constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = lane < (blockDim.x >> 5) ? sh[lane] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;  // valid in thread 0
}

// Returns true in thread 0 of the last block to finish, with the total.
__device__ bool finish_reduction(double block_total, double* partial, unsigned int* ticket, double* total) {
  __shared__ bool last;
  __shared__ double sh[32];
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = block_total;
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double v = 0.0;
  for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += blockDim.x) v += __ldcg(&partial[b]);
  const double s = block_sum(v, sh);
  if (threadIdx.x == 0) {
    *total = s;
    *ticket = 0;
  }
  return threadIdx.x == 0;
}

__device__ __forceinline__ void chunk_of(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t chunk = ((n + gridDim.x - 1) / gridDim.x + 31) & ~int64_t(31);
  lo = min(n, int64_t(blockIdx.x) * chunk);
  hi = min(n, lo + chunk);
}

__global__ void __launch_bounds__(kRedThreads) k_dot(const double* x, const double* y, int64_t n, double* partial,
                                                     unsigned int* ticket, double* out) {
  __shared__ double sh[32];
  int64_t lo, hi;
  chunk_of(n, lo, hi);
  double v = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) v += x[i] * y[i];
  const double bt = block_sum(v, sh);
  double tot;
  if (finish_reduction(bt, partial, ticket, &tot)) *out = tot;
}

// ap = Gᵀ gp (SELL, thread per row) fused with <p, ap>; alpha = rz / pap
__global__ void __launch_bounds__(kRedThreads) k_ap_dot(const int64_t* __restrict__ soff, const int32_t* __restrict__ len,
                                                        const int32_t* __restrict__ col, const double* __restrict__ val,
                                                        int64_t nr, const double* __restrict__ gp,
                                                        const double* __restrict__ p, double* __restrict__ ap,
                                                        double* partial, unsigned int* ticket, PcgScalars* sc) {
  __shared__ double sh[32];
  int64_t lo, hi;
  chunk_of(nr, lo, hi);
  double v = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const int64_t base = soff[i >> 5] + (i & 31);
    const int n = len[i];
    double s = 0.0;
    // sequential row sum (bit-exact order); the loads of 4 entries are issued ahead
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
      const int64_t e = base + int64_t(k) * 32;
      s += __ldcs(&val[e]) * __ldg(&gp[__ldcs(&col[e])]);
    }
    ap[i] = s;
    v += p[i] * s;
  }
  const double bt = block_sum(v, sh);
  double tot;
  if (finish_reduction(bt, partial, ticket, &tot)) {
    sc->pap = tot;
    sc->alpha = sc->rz / tot;
  }
}

__global__ void __launch_bounds__(kRedThreads) k_update_xr(double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p, const double* __restrict__ ap,
                                                           int64_t n, double* partial, unsigned int* ticket,
                                                           PcgScalars* sc) {
  __shared__ double sh[32];
  const double alpha = sc->alpha;
  int64_t lo, hi;
  chunk_of(n, lo, hi);
  double v = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] + (-alpha) * ap[i];
    r[i] = ri;
    v += ri * ri;
  }
  const double bt = block_sum(v, sh);
  double tot;
  if (finish_reduction(bt, partial, ticket, &tot)) sc->rn2 = tot;
}

__global__ void __launch_bounds__(kRedThreads) k_rz(const double* r, const double* z, int64_t n, double* partial,
                                                    unsigned int* ticket, PcgScalars* sc, int first) {
  __shared__ double sh[32];
  int64_t lo, hi;
  chunk_of(n, lo, hi);
  double v = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) v += r[i] * z[i];
  const double bt = block_sum(v, sh);
  double tot;
  if (finish_reduction(bt, partial, ticket, &tot)) {
    sc->rz_next = tot;
    if (!first) sc->beta = tot / sc->rz;
    sc->rz = tot;
  }
}

__global__ void k_update_p(double* __restrict__ p, const double* __restrict__ z, int64_t n, const PcgScalars* sc,
                           int first) {
  const double beta = sc->beta;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = first ? z[i] : z[i] + beta * p[i];
}

}  // namespace

void schwarz_ras(const SchwarzView& v, const double* r, double* e, bool accumulate, cudaStream_t s) {
  if (v.rows) {
    if (accumulate)
      schwarz_rows_launch<1>(v, v.ras_agg, v.ras_row, 0, v.n_ras_items, r, e, s);
    else
      schwarz_rows_launch<0>(v, v.ras_agg, v.ras_row, 0, v.n_ras_items, r, e, s);
    return;
  }
  if (v.n_groups > 0) {
    if (accumulate) {
      if (schwarz_tma_launch<1>(v, r, e, s)) return;
      schwarz_lrow_launch<1>(v, v.lane_ras_items, 0, v.n_lane_ras_items, r, e, s);
    } else {
      if (schwarz_tma_launch<0>(v, r, e, s)) return;
      schwarz_lrow_launch<0>(v, v.lane_ras_items, 0, v.n_lane_ras_items, r, e, s);
    }
    return;
  }
  if (accumulate)
    schwarz_launch<1>(v, nullptr, v.n_agg, r, e, s);
  else
    schwarz_launch<0>(v, nullptr, v.n_agg, r, e, s);
}

void schwarz_rast(const SchwarzView& v, const std::vector<int64_t>& color_off, const double* r, double* e,
                  cudaStream_t s) {
  if (v.rows) {
    const auto& co = *v.rast_color_off;
    for (size_t c = 0; c + 1 < co.size(); ++c) schwarz_rows_launch<2>(v, v.rast_agg, v.rast_row, co[c], co[c + 1], r, e, s);
    return;
  }
  if (v.n_groups > 0) {
    if (schwarz_tma_launch<2>(v, r, e, s)) return;
    const auto& co = *v.lane_rast_color_off;
    for (size_t c = 0; c + 1 < co.size(); ++c) schwarz_lrow_launch<2>(v, v.lane_rast_items, co[c], co[c + 1], r, e, s);
    return;
  }
  for (size_t c = 0; c + 1 < color_off.size(); ++c)
    schwarz_launch<2>(v, v.order + color_off[c], color_off[c + 1] - color_off[c], r, e, s);
}

void restrict_pt(const InterpView& v, const double* res, double* rc, cudaStream_t s, bool exact) {
  if (v.n_coarse == 0) return;
  if (!exact && v.n_coarse > 0 && v.n_fine >= 32 * v.n_agg) {  // large aggregates (mean nω >= 32): warp per coarse column
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(v.n_coarse, 8), int64_t(sm_count()) * 16)));
    k_restrict_warp<<<grid, 256, 0, s>>>(v, res, rc);
  } else {
    k_restrict<<<grid_for(v.n_coarse), 256, 0, s>>>(v, res, rc);
  }
  LSB_LAUNCH();
}

void prolong_add(const InterpView& v, const double* ec, double* e, cudaStream_t s, bool exact) {
  if (v.n_fine == 0) return;
  if (!exact && v.n_coarse >= 16 * v.n_agg) {  // ≥ 16 modes per aggregate on average
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(v.n_fine, 8), int64_t(sm_count()) * 8)));
    k_prolong_warp<<<grid, 256, 0, s>>>(v, ec, e);
  } else {
    k_prolong<<<grid_for(v.n_fine), 256, 0, s>>>(v, ec, e);
  }
  LSB_LAUNCH();
}

void dense_matvec(const double* m, int64_t n, const double* r, double* e, cudaStream_t s) {
  if (n == 0) return;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(n, 8), int64_t(sm_count()) * 8));
  k_dense_mv<<<grid, 256, 0, s>>>(m, n, r, e);
  LSB_LAUNCH();
}

void Reducer::init(cudaStream_t s) {
  nblocks = sm_count() * 8;  // 8 CTAs of 256 threads per SM: full occupancy for the gather-bound Gᵀ rows
  partial.alloc(nblocks, s);
  ticket.alloc(1, s);
  ticket.zero(s);
}

void dot(const Reducer& red, const double* x, const double* y, int64_t n, double* out, cudaStream_t s) {
  k_dot<<<red.nblocks, kRedThreads, 0, s>>>(x, y, n, red.partial.get(), red.ticket.get(), out);
  LSB_LAUNCH();
}

void pcg_ap_dot(const Sell& gt, const double* gp, const double* p, double* ap, const Reducer& red, PcgScalars* sc,
                cudaStream_t s) {
  k_ap_dot<<<red.nblocks, kRedThreads, 0, s>>>(gt.slice_off.get(), gt.row_len.get(), gt.col.get(), gt.val.get(), gt.nr,
                                               gp, p, ap, red.partial.get(), red.ticket.get(), sc);
  LSB_LAUNCH();
}

void pcg_update_xr(const Reducer& red, double* x, double* r, const double* p, const double* ap, int64_t n,
                   PcgScalars* sc, cudaStream_t s) {
  k_update_xr<<<red.nblocks, kRedThreads, 0, s>>>(x, r, p, ap, n, red.partial.get(), red.ticket.get(), sc);
  LSB_LAUNCH();
}

void pcg_rz(const Reducer& red, const double* r, const double* z, int64_t n, PcgScalars* sc, bool first,
            cudaStream_t s) {
  k_rz<<<red.nblocks, kRedThreads, 0, s>>>(r, z, n, red.partial.get(), red.ticket.get(), sc, first ? 1 : 0);
  LSB_LAUNCH();
}

void pcg_update_p(double* p, const double* z, int64_t n, const PcgScalars* sc, bool first, cudaStream_t s) {
  k_update_p<<<grid_for(n), 256, 0, s>>>(p, z, n, sc, first ? 1 : 0);
  LSB_LAUNCH();
}

}  // namespace lsb
