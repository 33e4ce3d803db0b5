// dense_dev.cuh — team-parallel dense kernels of dense.hpp / eigen.hpp.
//
// Every routine runs on a Team (a warp or a CTA, common.cuh) over matrices in
// a per-problem workspace (shared or global memory). Parallelism is only over
// independent outputs; every reduction keeps the reference's sequential
// order, and the library is compiled with --fmad=false, so results are
// bit-identical to the reference's no-FMA build:
//   * matmul / matmul_transa / weighted Gram: one output per thread, the sum
//     over k in ascending order with the reference's zero-skip rule;
//   * cyclic Jacobi: the rotation sequence is inherently sequential, each
//     rotation updates O(n) disjoint entries in parallel (eigen.hpp:85-93
//     touches rows/columns p and q only), two team barriers per rotation.
#pragma once

#include <cuda/atomic>
#include <type_traits>

#include "common.cuh"
#include "jacobi_wave.cuh"

namespace lsb {

// Deterministic bump allocator over a workspace. All team threads perform
// the same take() sequence, so they agree on every pointer.
struct Arena {
  double* base;
  int64_t used;
  double* fast = nullptr;   // optional shared-memory scratch (CTA teams, global workspace)
  int64_t fast_cap = 0;     // doubles
  WaveCtl* wctl = nullptr;  // cluster launches: command block and workspace of the wavefront Jacobi
  double* wws = nullptr;
  int wave_min = 0;         // smallest n that takes the wavefront path
  int sched = 0;            // schedule of the single-CTA large-n path (test hook)
  __device__ double* take(int64_t n) {
    double* p = base + used;
    used += (n + 1) & ~int64_t(1);
    return p;
  }
  __device__ int* take_int(int64_t n) { return reinterpret_cast<int*>(take((n + 1) / 2)); }
};

// workspace doubles needed by t_sym_eig (excluding its outputs); includes the
// rotation log of the pipelined CTA path
__host__ __device__ inline int64_t sym_eig_scratch(int64_t n) {
  const int64_t ld = (n + 1) & ~int64_t(1);
  return 2 * (n * ld + 2) + 3 * ((n + 1) & ~int64_t(1)) + 4 + ((n * (n - 1) + 1) & ~int64_t(1)) + 2;
}

// ---- pipelined CTA Jacobi for large n (global workspace) -----------------------------
//
// Same rotation sequence and arithmetic as eigen.hpp:35-118. The matrix is
// kept as a full symmetric array in global memory (both triangles updated).
// While row p is swept, index p's vector a(p,·) lives in shared memory; the
// partner rows q are prefetched with cp.async into a ring of R shared buffers
// (prefetch depth R-2, so a slot is only refilled after every thread has
// passed the barrier that retires it), patched with the entries rotated after
// their prefetch, and written back (row and mirrored column) right after their
// rotation. Every rotation pairs (a(p,j), a(q,j)) for j ∉ {p,q}, and thread
// j mod T owns pair j for the whole sweep, so the single-writer updates of a
// rotation (a(p,q) = 0, d[q] += h, z[q] += h) are deferred to the next step
// and each rotation costs one CTA barrier with a shared-memory critical path.
// Eigenvector rotations are logged (s, tau) and applied per sweep, one row of
// V per thread, off the critical path.

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kPipeThreads = 512;   // the pipelined path runs on exactly this CTA size

// shared doubles of the pipelined path with R ring slots
__host__ __device__ inline int64_t pipelined_smem_doubles(int64_t n, int R) {
  const int64_t ld = (n + 1) & ~int64_t(1);
  return (2 + 2 * R) * ld + 3 * ld + 16 + 3 * 2 * R * R;
}

__device__ long long* g_eig_prof = nullptr;  // optional per-phase cycle counters (test hook)

// Returns 0/1/2 like t_sym_eig. A: global scratch n×ld (ld = n rounded to
// even, 16-byte rows), Vt: global n×ld (Vᵀ, row k = eigenvector column k),
// sm: shared scratch of pipelined_smem_doubles(n, R). Requires blockDim.x == 512.
//
// Ring protocol (R slots, depth D = R-2): at step q every thread issues its
// cp.async pieces of rows q+D of A and Vᵀ into slot (q+D) mod R (whose
// previous rows, q-2, were consumed before the barrier of step q-1), commits,
// waits for row q (wait_group D) and meets the barrier. A row r of A in flight
// can miss entries (r, q') rotated at steps q' in [r-D-1, r-1] (step r-D-1 may
// still be writing while r's copy is issued); each such entry is recorded in
// row r's patch list (indexed r mod 2R, reset at step r-R) and applied by the
// entry's owner when row r is rotated. Rows of Vᵀ need no patches: within row
// p's sweep, Vᵀ row q changes only at step q.
template <int R>
__device__ int cta_sym_eig_pipelined(int n, const double* m, double* vals, double* vecs, double* A, double* Vt,
                                     double* sm) {
  constexpr int D = R - 2, NL = 2 * R, T = kPipeThreads;
  const int tid = threadIdx.x;
  const int64_t ld = (n + 1) & ~int64_t(1);
  double* pv = sm;                       // a(p,·)
  double* vp = pv + ld;                  // Vᵀ row p
  double* ring = vp + ld;                // R slots × (A row, Vᵀ row)
  double* d = ring + int64_t(2 * R) * ld;
  double* bb = d + ld;
  double* z = bb + ld;
  double* slot = z + ld;
  double* pend_val = slot + 16;                                 // [NL][R]
  int* pend_pos = reinterpret_cast<int*>(pend_val + NL * R);  // [NL][R]
  __shared__ int pend_n[NL];
  long long t_sm = 0, t_wait = 0, t_par = 0, t_rot = 0, tc = 0;
  auto tick = [&](long long& acc) {
    const long long now = clock64();
    acc += now - tc;
    tc = now;
  };
  for (int64_t e = tid; e < int64_t(n) * n; e += T) {  // full symmetric copy (eigen.hpp:44)
    const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    double val = m[e];
    if (i != j) {
      const int lo = i < j ? i : j, hi = i < j ? j : i;
      val = 0.5 * (m[int64_t(lo) * n + hi] + m[int64_t(hi) * n + lo]);
    }
    A[int64_t(i) * ld + j] = val;
    Vt[int64_t(i) * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  for (int i = tid; i < n; i += T) {
    d[i] = bb[i] = m[int64_t(i) * n + i];
    z[i] = 0.0;
  }
  __syncthreads();
  const int chunks = static_cast<int>(ld / 2);  // 16-byte pieces per row
  auto prefetch = [&](int row) {
    if (row < n) {
      double* dst = ring + int64_t(2 * (row % R)) * ld;
      const double* srca = A + int64_t(row) * ld;
      const double* srcv = Vt + int64_t(row) * ld;
      for (int c = tid; c < chunks; c += T) {
        cp_async16(dst + 2 * c, srca + 2 * c);
        cp_async16(dst + ld + 2 * c, srcv + 2 * c);
      }
    }
    cp_async_commit();
  };
  bool converged = false;
  for (int sweep = 0; sweep < 64; ++sweep) {
    // Σ_{p<q} |a(p,q)| in the reference's order: rows staged in shared memory,
    // summed sequentially by thread 0
    double smv = 0.0;
    tc = clock64();
    for (int p = 0; p + 1 < n; ++p) {
      for (int q = p + 1 + tid; q < n; q += T) ring[q] = A[int64_t(p) * ld + q];
      __syncthreads();
      if (tid == 0)
        for (int q = p + 1; q < n; ++q) smv += fabs(ring[q]);
      __syncthreads();
    }
    if (tid == 0) slot[0] = smv;
    __syncthreads();
    tick(t_sm);
    smv = slot[0];
    if (smv == 0.0) {
      converged = true;
      break;
    }
    const double tresh = sweep < 3 ? 0.2 * smv / static_cast<double>(static_cast<uint64_t>(n) * n) : 0.0;
    for (int p = 0; p + 1 < n; ++p) {
      for (int j = tid; j < n; j += T) {
        pv[j] = A[int64_t(p) * ld + j];
        vp[j] = Vt[int64_t(p) * ld + j];
      }
      if (tid < NL) pend_n[tid] = 0;
      __syncthreads();
      for (int k = 1; k <= D; ++k) prefetch(p + k);
      double dp = d[p];
      double zp = z[p];
      int prev_q = -1, prev_zero = 0;
      double prev_h = 0.0;
      for (int q = p + 1; q < n; ++q) {
        tick(t_rot);
        prefetch(q + D);
        cp_async_wait<D>();
        __syncthreads();
        tick(t_wait);
        // single-owner writes deferred from step q-1 (their readers passed the barrier)
        if (prev_q >= 0) {
          if (prev_zero && (prev_q & (T - 1)) == tid) pv[prev_q] = 0.0;
          if (tid == 0 && prev_h != 0.0) {
            z[prev_q] += prev_h;
            d[prev_q] += prev_h;
          }
        }
        if (tid == 0) pend_n[(q + R) % NL] = 0;
        const double* qv = ring + int64_t(2 * (q % R)) * ld;
        const double* qvv = qv + ld;
        const double apq = pv[q];
        const double dq = d[q];
        const double g = 100.0 * fabs(apq);
        double h = 0.0;
        int zero = 0;
        if (sweep > 3 && fabs(dp) + g == fabs(dp) && fabs(dq) + g == fabs(dq)) {
          zero = 1;
        } else if (fabs(apq) > tresh) {
          double hh = dq - dp;
          double tt;
          if (fabs(hh) + g == fabs(hh)) {
            tt = apq / hh;
          } else {
            const double theta = 0.5 * hh / apq;
            tt = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
            if (theta < 0.0) tt = -tt;
          }
          const double c = 1.0 / sqrt(1.0 + tt * tt);
          const double s = tt * c;
          const double tau = s / (1.0 + c);
          h = tt * apq;
          zp -= h;
          dp -= h;
          zero = 1;
          tick(t_par);
          const int li = q % NL;
          const int np = pend_n[li];
          for (int j = tid; j < n; j += T) {
            // eigenvectors: rotate(v(j,p), v(j,q)) (eigen.hpp:93)
            const double vx = vp[j], vy = qvv[j];
            vp[j] = vx - s * (vy + vx * tau);
            Vt[int64_t(q) * ld + j] = vy + s * (vx - vy * tau);
            if (j == p || j == q) continue;
            double hy = qv[j];
            for (int e = 0; e < np; ++e)
              if (pend_pos[li * R + e] == j) hy = pend_val[li * R + e];
            const double gx = pv[j];
            const double nx = gx - s * (hy + gx * tau);
            const double ny = hy + s * (gx - hy * tau);
            pv[j] = nx;
            A[int64_t(q) * ld + j] = ny;  // row q and its mirrored column
            A[int64_t(j) * ld + q] = ny;
            if (j > q && j < q + R) {  // row j may hold a stale (j, q) entry
              const int lj = j % NL;
              const int e = pend_n[lj]++;
              pend_pos[lj * R + e] = q;
              pend_val[lj * R + e] = ny;
            }
          }
        }
        prev_q = q;
        prev_h = h;
        prev_zero = zero;
      }
      tick(t_rot);
      cp_async_wait<0>();
      __syncthreads();
      if (prev_zero && (prev_q & (T - 1)) == tid) pv[prev_q] = 0.0;
      if (tid == 0) {
        if (prev_h != 0.0) {
          z[prev_q] += prev_h;
          d[prev_q] += prev_h;
        }
        d[p] = dp;
        z[p] = zp;
      }
      __syncthreads();
      for (int j = tid; j < n; j += T) {  // index p's final vectors back to A (row and column) and Vᵀ
        Vt[int64_t(p) * ld + j] = vp[j];
        if (j == p) continue;
        A[int64_t(p) * ld + j] = pv[j];
        A[int64_t(j) * ld + p] = pv[j];
      }
      __syncthreads();
    }
    for (int i = tid; i < n; i += T) {
      bb[i] += z[i];
      d[i] = bb[i];
      z[i] = 0.0;
    }
    __syncthreads();
  }
  if (tid == 0 && g_eig_prof) {
    g_eig_prof[0] += t_sm;
    g_eig_prof[1] += t_wait;
    g_eig_prof[2] += t_par;
    g_eig_prof[3] += t_rot;
  }
  if (!converged) return 1;
  for (int i = 0; i < n; ++i)
    if (!isfinite(d[i])) return 2;
  for (int k = tid; k < n; k += T) {
    const double dk = d[k];
    int pos = 0;
    for (int i = 0; i < n; ++i)
      if (d[i] < dk || (d[i] == dk && i < k)) ++pos;
    vals[pos] = dk;
    for (int i = 0; i < n; ++i) vecs[int64_t(i) * n + pos] = Vt[int64_t(k) * ld + i];
  }
  __syncthreads();
  return 0;
}

// ---- producer/consumer variant --------------------------------------------------------
//
// Same arithmetic and sequence as cta_sym_eig_pipelined. Warp 0 (producer)
// runs only the sequential chain: for rotation (p,q) it applies rotation
// (p,q-1) to pair j = q, computes (s, tau, h) of rotation (p,q), updates d/z
// and publishes. Warps 1..15 (consumers) apply each published rotation to all
// other pairs (j ∉ {p, q, q+1}) and to Vᵀ one or two rotations behind, keep
// the cp.async ring of partner rows full, and meet at a named barrier. To keep
// the consumers off the L1/LSU limit:
//   * a(p,j) and v(j,p) live in the owner thread's registers for the whole row
//     (thread j mod 480 owns pair j); the producer receives a(p,q+1) through a
//     shared hand-off slot and returns the pivot's final value in the queue;
//   * patches of in-flight rows are direct-mapped by rotation distance;
//   * mirrored-column stores of rotations (2k, 2k+1) go out as one 16-byte
//     store during rotation 2k+1 (still inside the patch window).
constexpr int kMaxOwn = 5;  // pairs per consumer thread: n <= 384 * kMaxOwn

template <int R, int NCW = 12>
__device__ int cta_sym_eig_pc(int n, const double* m, double* vals, double* vecs, double* A, double* Vt, double* sm) {
  // Warp 0 (SMSP 0) produces; warps 4, 8, 12 idle so SMSP 0 issues only the
  // producer's dependent chain; the other 12 warps consume.
  // NCW = 12: warps 4, 8, 12 idle; NCW = 15: every warp but the producer consumes
  constexpr int D = R - 2, NL = 2 * R, PS = R + 1, T = kPipeThreads, NC = NCW * 32, QN = 64;
  const int tid = threadIdx.x;
  const int wid = tid >> 5;
  const bool producer = wid == 0;
  const bool idle = NCW == 12 && (wid & 3) == 0 && wid != 0;
  const int ctid = (NCW == 12 ? wid - 1 - (wid >> 2) : wid - 1) * 32 + (tid & 31);  // consumer index 0..383
  const int64_t ld = (n + 1) & ~int64_t(1);
  double* pvs = sm;                      // a(p,·) at row start / hand-offs
  double* vp = pvs + ld;                 // Vᵀ row p at row start
  double* ring = vp + ld;
  double* d = ring + int64_t(2 * R) * ld;
  double* bb = d + ld;
  double* z = bb + ld;
  double* slot = z + ld;
  double* patch = slot + 16;             // [NL][R+1] by rotation distance 1..R
  __shared__ unsigned pmask[NL];
  __shared__ double q_s[QN], q_tau[QN], q_piv[QN], q_ny[QN];
  __shared__ int q_rot[QN];
  __shared__ int q_first;  // first rotating step of the current row
  for (int64_t e = tid; e < int64_t(n) * n; e += T) {  // full symmetric copy (eigen.hpp:44)
    const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    double val = m[e];
    if (i != j) {
      const int lo = i < j ? i : j, hi = i < j ? j : i;
      val = 0.5 * (m[int64_t(lo) * n + hi] + m[int64_t(hi) * n + lo]);
    }
    A[int64_t(i) * ld + j] = val;
    Vt[int64_t(i) * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  for (int i = tid; i < n; i += T) {
    d[i] = bb[i] = m[int64_t(i) * n + i];
    z[i] = 0.0;
  }
  __syncthreads();
  const int chunks = static_cast<int>(ld / 2);
  auto prefetch = [&](int row) {  // consumers only
    if (row < n) {
      double* dst = ring + int64_t(2 * (row % R)) * ld;
      const double* srca = A + int64_t(row) * ld;
      const double* srcv = Vt + int64_t(row) * ld;
      for (int c = ctid; c < chunks; c += NC) {
        cp_async16(dst + 2 * c, srca + 2 * c);
        cp_async16(dst + ld + 2 * c, srcv + 2 * c);
      }
    }
    cp_async_commit();
  };
  // Round q of the rotation barrier: the consumers have finished rotation q-1
  // and landed row q; the producer has published rotation q.
  auto rbar = []() { asm volatile("bar.sync 1, %0;" ::"n"(NC + 32) : "memory"); };
  long long base = 0;
  bool converged = false;
  long long* const prof = g_eig_prof;  // optional cycle counters (test hook)
  long long c_w = 0, c_c = 0, c_b = 0, c_p = 0, c_r = 0, c_e = 0, c_n = 0, c_rot = 0, c_skip = 0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double smv = 0.0;
    for (int p = 0; p + 1 < n; ++p) {
      for (int q = p + 1 + tid; q < n; q += T) ring[q] = A[int64_t(p) * ld + q];
      __syncthreads();
      if (tid == 0)
        for (int q = p + 1; q < n; ++q) smv += fabs(ring[q]);
      __syncthreads();
    }
    if (tid == 0) slot[0] = smv;
    __syncthreads();
    smv = slot[0];
    if (smv == 0.0) {
      converged = true;
      break;
    }
    const double tresh = sweep < 3 ? 0.2 * smv / static_cast<double>(static_cast<uint64_t>(n) * n) : 0.0;
    for (int p = 0; p + 1 < n; ++p) {
      for (int j = tid; j < n; j += T) {
        pvs[j] = A[int64_t(p) * ld + j];
        vp[j] = Vt[int64_t(p) * ld + j];
      }
      if (tid < NL) pmask[tid] = 0u;
      if (tid == 0) q_first = n;
      __syncthreads();
      // Steps before the row's first rotation see the row as loaded: find that
      // step with the reference's predicates (eigen.hpp:62-65) in parallel,
      // apply the "zeroed" pairs before it, and start the pipeline there.
      {
        const double dp0 = d[p];
        for (int q = p + 1 + tid; q < n; q += T) {
          const double a = pvs[q], g = 100.0 * fabs(a), dq = d[q];
          const bool zero = sweep > 3 && fabs(dp0) + g == fabs(dp0) && fabs(dq) + g == fabs(dq);
          if (!zero && fabs(a) > tresh) atomicMin(&q_first, q);
        }
        __syncthreads();
        const int q1 = q_first;
        for (int q = p + 1 + tid; q < q1; q += T) {
          const double a = pvs[q], g = 100.0 * fabs(a), dq = d[q];
          if (sweep > 3 && fabs(dp0) + g == fabs(dp0) && fabs(dq) + g == fabs(dq)) pvs[q] = 0.0;
        }
        __syncthreads();
      }
      const int q_start = q_first;
      if (producer) {
        // all 32 lanes walk the rounds (bar.sync is warp-aligned); lane 0 computes
        double dp = d[p], zp = z[p];
        double ps = 0.0, ptau = 0.0, ph = 0.0;
        int prot = 0;
        double ny_prev = 0.0;
        for (int q = q_start; q < n; ++q) {
          const long long t = base + (q - p - 1);
          const long long k1 = prof ? clock64() : 0;
          if (tid == 0) {
            double apq = pvs[q];  // a(p,q) after the consumers' rotations <= q-2 (hand-off)
            if (q > q_start) {
              if (prot) {  // rotation q-1 on pair q; the owner of q-1 stores a(q-1,q) at rotation q
                const int pq = q - 1;
                const double hy = ring[int64_t(2 * (pq % R)) * ld + q];
                const double gx = apq;
                ny_prev = hy + ps * (gx - hy * ptau);
                apq = gx - ps * (hy + gx * ptau);
                z[pq] += ph;
                d[pq] += ph;
              }
            }
            const double dq = d[q];
            const double g = 100.0 * fabs(apq);
            double s = 0.0, tau = 0.0, h = 0.0;
            int rot = 0, zero = 0;
            if (sweep > 3 && fabs(dp) + g == fabs(dp) && fabs(dq) + g == fabs(dq)) {
              zero = 1;
            } else if (fabs(apq) > tresh) {
              double hh = dq - dp;
              double tt;
              if (fabs(hh) + g == fabs(hh)) {
                tt = apq / hh;
              } else {
                const double theta = 0.5 * hh / apq;
                tt = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
                if (theta < 0.0) tt = -tt;
              }
              const double c = 1.0 / sqrt(1.0 + tt * tt);
              s = tt * c;
              tau = s / (1.0 + c);
              h = tt * apq;
              zp -= h;
              dp -= h;
              zero = 1;
              rot = 1;
            }
            const int qi = static_cast<int>(t % QN);
            q_s[qi] = s;
            q_tau[qi] = tau;
            q_rot[qi] = rot;
            q_piv[qi] = zero ? 0.0 : apq;  // a(p,q) after rotation q (pair q resumes at q+1)
            q_ny[qi] = ny_prev;            // a(q,q-1) after rotation q-1 (valid when rotation q-1 rotated)
            ps = s;
            ptau = tau;
            ph = h;
            prot = rot;
          }
          __syncwarp();
          const long long k2 = prof ? clock64() : 0;
          rbar();  // round q: publish rotation q; rotation q-1 done, row q landed
          if (prof) {
            c_c += k2 - k1;
            c_w += clock64() - k2;
            ++c_n;
            c_rot += prot;
          }
        }
        if (tid == 0) {
          if (prot) {  // the row's last rotation: its diagonal updates
            z[n - 1] += ph;
            d[n - 1] += ph;
          }
          d[p] = dp;
          z[p] = zp;
        }
      } else if (!idle) {
        // owner registers: pair j = ctid + k*NC
        double pr[kMaxOwn], vr[kMaxOwn], pend[kMaxOwn];
#pragma unroll
        for (int k = 0; k < kMaxOwn; ++k) {
          const int j = ctid + k * NC;
          pr[k] = j < n ? pvs[j] : 0.0;
          vr[k] = j < n ? vp[j] : 0.0;
          pend[k] = 0.0;
        }
        int pend_q = -1;  // rotation whose mirror stores are held back
        for (int k = 0; k < D; ++k) prefetch(q_start + k);
        for (int q = q_start; q < n; ++q) {
          const long long t = base + (q - p - 1);
          const long long k0 = prof ? clock64() : 0;
          prefetch(q + D);
          cp_async_wait<D>();
          const long long k1 = prof ? clock64() : 0;
          rbar();  // round q
          const long long k2 = prof ? clock64() : 0;
          if (ctid == 0) pmask[(q + R + 1) % NL] = 0u;  // before any rotation can patch row q+R+1
          const int qi = static_cast<int>(t % QN);
          const int qp = static_cast<int>((t + QN - 1) % QN);  // rotation q-1 (when q-1 > p)
          const bool rot = q_rot[qi] != 0;
          const double s = q_s[qi], tau = q_tau[qi];
          const double* qv = ring + int64_t(2 * (q % R)) * ld;
          const double* qvv = qv + ld;
          double* const arow = A + int64_t(q) * ld;
          double* const vrow = Vt + int64_t(q) * ld;
          const bool pair_odd = (q & 1) != 0;
          const bool held_q = pend_q == q - 1;
#pragma unroll
          for (int k = 0; k < kMaxOwn; ++k) {
            const int j = ctid + k * NC;
            if (j >= n) break;
            double* const mir = A + int64_t(j) * ld;  // row j: mirrored column entries
            if (static_cast<unsigned>(j - q + R) > static_cast<unsigned>(2 * R) && j != p) {
              // fast path: not excluded, no patch to read or write, no hand-off
              if (rot) {
                const double vx = vr[k], vy = qvv[j];
                vr[k] = vx - s * (vy + vx * tau);
                vrow[j] = vy + s * (vx - vy * tau);
                const double hy = qv[j], gx = pr[k];
                const double ny = hy + s * (gx - hy * tau);
                pr[k] = gx - s * (hy + gx * tau);
                arow[j] = ny;
                if (held_q) {  // rotations (q-1, q): one 16-byte store, q-1 even, ld even
                  double2 v2;
                  v2.x = pend[k];
                  v2.y = ny;
                  *reinterpret_cast<double2*>(mir + q - 1) = v2;
                } else if (pair_odd) {
                  mir[q] = ny;
                } else {
                  pend[k] = ny;  // held until rotation q+1
                }
              } else if (held_q) {
                mir[q - 1] = pend[k];
              }
              continue;
            }
            if (j == q - 1 && j >= q_start) pr[k] = q_piv[qp];  // the pivot of rotation q-1 resumes
            const bool held = held_q && j != p && j != q - 1 && j != q;
            if (rot) {
              const double vx = vr[k], vy = qvv[j];
              vr[k] = vx - s * (vy + vx * tau);
              vrow[j] = vy + s * (vx - vy * tau);
            }
            const bool prev_rot = j == q - 1 && j >= q_start && q_rot[qp] != 0;  // a(q,q-1) from the producer
            if (!rot || j == p || j == q || j == q + 1) {
              if (held) mir[q - 1] = pend[k];
              if (prev_rot) {
                arow[j] = q_ny[qi];
                mir[q] = q_ny[qi];
              }
            } else {
              const int lr = q % NL;
              double hy = qv[j];
              const int dist = q - j;
              if (prev_rot) {
                hy = q_ny[qi];
              } else if (dist >= 2 && dist <= R && ((pmask[lr] >> dist) & 1u)) {
                hy = patch[lr * PS + dist];
              }
              const double gx = pr[k];
              const double ny = hy + s * (gx - hy * tau);
              pr[k] = gx - s * (hy + gx * tau);
              arow[j] = ny;
              if (held) {
                double2 v2;
                v2.x = pend[k];
                v2.y = ny;
                *reinterpret_cast<double2*>(mir + q - 1) = v2;
              } else if (pair_odd) {
                mir[q] = ny;
              } else {
                pend[k] = ny;
              }
              // rows up to q+R may have been fetched before this rotation's mirror
              // store (held one rotation) becomes visible
              if (j > q + 1 && j <= q + R) {
                const int lj = j % NL;
                patch[lj * PS + (j - q)] = ny;
                atomicOr(&pmask[lj], 1u << (j - q));
              }
            }
            if (j == q + 2) pvs[j] = pr[k];  // hand-off: the producer applies rotation q+1
          }
          if (rot && !pair_odd)
            pend_q = q;
          else
            pend_q = -1;
          if (prof) {
            const long long k3 = clock64();
            c_b += k1 - k0;
            c_p += k2 - k1;
            c_r += k3 - k2;
            if (!rot) c_skip += k3 - k0;  // whole step time of non-rotating steps
          }
        }
        cp_async_wait<0>();
        // flush a mirror still held from the row's last even rotation
        if (pend_q >= 0) {
#pragma unroll
          for (int k = 0; k < kMaxOwn; ++k) {
            const int j = ctid + k * NC;
            if (j < n && j != p && j != pend_q && j != pend_q + 1) A[int64_t(j) * ld + pend_q] = pend[k];
          }
        }
        const double piv_last = q_piv[(base + (n - 1 - p - 1)) % QN];  // the last pivot's final value
#pragma unroll
        for (int k = 0; k < kMaxOwn; ++k) {
          const int j = ctid + k * NC;
          if (j < n) {
            pvs[j] = (j == n - 1 && j > p && q_start < n) ? piv_last : pr[k];
            vp[j] = vr[k];
          }
        }
      }
      base += n - p - 1;
      const long long k4 = prof ? clock64() : 0;
      __syncthreads();
      for (int j = tid; j < n; j += T) {
        Vt[int64_t(p) * ld + j] = vp[j];
        if (j == p) continue;
        A[int64_t(p) * ld + j] = pvs[j];
        A[int64_t(j) * ld + p] = pvs[j];
      }
      __syncthreads();
      if (prof) c_e += clock64() - k4;
    }
    for (int i = tid; i < n; i += T) {
      bb[i] += z[i];
      d[i] = bb[i];
      z[i] = 0.0;
    }
    __syncthreads();
  }
  if (prof) {
    if (tid == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[0]), c_w);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[1]), c_c);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[5]), c_e);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[6]), c_n);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[7]), c_rot);
    }
    if (tid == 32) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[0]), c_skip);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[2]), c_b);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[3]), c_p);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[4]), c_r);
    }
  }
  if (!converged) return 1;
  for (int i = 0; i < n; ++i)
    if (!isfinite(d[i])) return 2;
  for (int k = tid; k < n; k += T) {
    const double dk = d[k];
    int pos = 0;
    for (int i = 0; i < n; ++i)
      if (d[i] < dk || (d[i] == dk && i < k)) ++pos;
    vals[pos] = dk;
    for (int i = 0; i < n; ++i) vecs[int64_t(i) * n + pos] = Vt[int64_t(k) * ld + i];
  }
  __syncthreads();
  return 0;
}

// sched 0: producer/consumer with 15 consumer warps (default); 1: one barrier
// per rotation (the only schedule for n > 384*kMaxOwn; also a test path)
__device__ __noinline__ int cta_sym_eig_pipelined_any(int n, const double* m, double* vals, double* vecs, double* A,
                                                double* Vt, double* sm, int R, int sched) {
  if (sched == 0 && n <= 384 * kMaxOwn) {
    if (R >= 8) return cta_sym_eig_pc<8, 15>(n, m, vals, vecs, A, Vt, sm);
    if (R >= 6) return cta_sym_eig_pc<6, 15>(n, m, vals, vecs, A, Vt, sm);
    return cta_sym_eig_pc<4, 15>(n, m, vals, vecs, A, Vt, sm);
  }
  if (R >= 8) return cta_sym_eig_pipelined<8>(n, m, vals, vecs, A, Vt, sm);
  if (R >= 6) return cta_sym_eig_pipelined<6>(n, m, vals, vecs, A, Vt, sm);
  return cta_sym_eig_pipelined<4>(n, m, vals, vecs, A, Vt, sm);
}

template <class Team>
__device__ void t_copy(const Team& t, double* dst, const double* src, int64_t cnt) {
  for (int64_t i = t.rank(); i < cnt; i += t.size()) dst[i] = src[i];
  t.sync();
}

template <class Team>
__device__ void t_fill(const Team& t, double* dst, double v, int64_t cnt) {
  for (int64_t i = t.rank(); i < cnt; i += t.size()) dst[i] = v;
  t.sync();
}

// a <- (a + aᵀ)/2                                           dense.hpp:103-111
template <class Team>
__device__ void t_symmetrize(const Team& t, double* a, int n) {
  const int64_t pairs = int64_t(n) * n;
  for (int64_t e = t.rank(); e < pairs; e += t.size()) {
    const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    if (j <= i) continue;
    const double m = 0.5 * (a[int64_t(i) * n + j] + a[int64_t(j) * n + i]);
    a[int64_t(i) * n + j] = m;
    a[int64_t(j) * n + i] = m;
  }
  t.sync();
}

// Core of the dense products: c(i,j) = Σ_k a(i,k)·b(k,j) with k ascending, a(i,k) = a[i·sa_i + k·sa_k],
// optionally skipping a(i,k) == 0 (select, not a branch, so the loads pipeline). A thread owns four
// consecutive rows i of one column j: the b(k,j) load is shared and coalesced across the team, the
// a loads are uniform across the lanes of a row block. Every sum keeps the reference's order.
template <bool SKIP, class Team, class Store>
__device__ __forceinline__ void t_mm_core(const Team& t, const double* a, int64_t sa_i, int64_t sa_k, int ar, int ac,
                                          const double* b, int bc, Store store) {
  const int rb = (ar + 3) >> 2;
  const int64_t cnt = int64_t(rb) * bc;
  for (int64_t e = t.rank(); e < cnt; e += t.size()) {
    const int i0 = static_cast<int>(e / bc) << 2, j = static_cast<int>(e % bc);
    const double* p0 = a + int64_t(i0) * sa_i;
    const double* p1 = a + int64_t(min(i0 + 1, ar - 1)) * sa_i;
    const double* p2 = a + int64_t(min(i0 + 2, ar - 1)) * sa_i;
    const double* p3 = a + int64_t(min(i0 + 3, ar - 1)) * sa_i;
    const double* pb = b + j;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 2
    for (int k = 0; k < ac; ++k) {
      const double bk = pb[int64_t(k) * bc];
      const int64_t o = int64_t(k) * sa_k;
      const double x0 = p0[o], x1 = p1[o], x2 = p2[o], x3 = p3[o];
      if (SKIP) {
        s0 = x0 != 0.0 ? s0 + x0 * bk : s0;
        s1 = x1 != 0.0 ? s1 + x1 * bk : s1;
        s2 = x2 != 0.0 ? s2 + x2 * bk : s2;
        s3 = x3 != 0.0 ? s3 + x3 * bk : s3;
      } else {
        s0 += x0 * bk;
        s1 += x1 * bk;
        s2 += x2 * bk;
        s3 += x3 * bk;
      }
    }
    store(i0, j, s0);
    if (i0 + 1 < ar) store(i0 + 1, j, s1);
    if (i0 + 2 < ar) store(i0 + 2, j, s2);
    if (i0 + 3 < ar) store(i0 + 3, j, s3);
  }
  t.sync();
}

// c(ar×bc) = a(ar×ac)·b(ac×bc), skipping a(i,k) == 0        dense.hpp:47-59
template <class Team>
__device__ void t_matmul(const Team& t, const double* a, int ar, int ac, const double* b, int bc, double* c) {
  t_mm_core<true>(t, a, ac, 1, ar, ac, b, bc, [&](int i, int j, double v) { c[int64_t(i) * bc + j] = v; });
}

// c(ac×bc) = a(ar×ac)ᵀ·b(ar×bc), skipping a(k,i) == 0       dense.hpp:62-74
template <class Team>
__device__ void t_matmul_transa(const Team& t, const double* a, int ar, int ac, const double* b, int bc, double* c) {
  t_mm_core<true>(t, a, 1, ac, ac, ar, b, bc, [&](int i, int j, double v) { c[int64_t(i) * bc + j] = v; });
}

// Sequential reductions by rank 0, broadcast through *slot. With a shared-memory scratch `sm`
// (n + 1 doubles) the team forms the products in parallel and rank 0 only runs the ordered sum.
template <class Team>
__device__ double t_seq_dot(const Team& t, const double* x, const double* y, int n, double* slot, double* sm = nullptr) {
  if (sm) {
    for (int i = t.rank(); i < n; i += t.size()) sm[i] = x[i] * y[i];
    t.sync();
    if (t.rank() == 0) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += sm[i];
      sm[n] = s;
    }
    t.sync();
    const double v = sm[n];
    t.sync();
    return v;
  }
  if (t.rank() == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i] * y[i];
    *slot = s;
  }
  t.sync();
  const double v = *slot;
  t.sync();
  return v;
}

// Cyclic Jacobi eigendecomposition (eigen.hpp:35-118): values ascending,
// vecs(i,k) = vecs[i*n+k] is eigenvector k. Returns 0, or 1 (no convergence
// in 64 sweeps) / 2 (non-finite value) for EigError.
template <class Team>
__device__ int t_sym_eig(const Team& t, int n, const double* m, double* vals, double* vecs, Arena ar) {
  const int64_t nn = int64_t(n) * n;
  for (int64_t e = t.rank(); e < nn; e += t.size()) vecs[e] = (e / n == e % n) ? 1.0 : 0.0;
  if (n == 0) {
    t.sync();
    return 0;
  }
  if constexpr (!std::is_same<Team, WarpTeam>::value) {
    if (ar.wctl && n >= ar.wave_min && n <= kWaveMaxN && wave_smem_doubles(n) <= ar.fast_cap)
    {
#ifdef LSB_DIAG
      const long long c0 = clock64();
      const int st = wave_sym_eig_leader(n, m, vals, vecs, ar.wctl, ar.wws, ar.fast);
      if (t.rank() == 0 && g_eig_prof) {  // diagnostics: cycles and calls of the wavefront eigensolves
        atomicAdd(reinterpret_cast<unsigned long long*>(g_eig_prof) + 4, static_cast<unsigned long long>(clock64() - c0));
        atomicAdd(reinterpret_cast<unsigned long long*>(g_eig_prof) + 5, 1ull);
      }
      return st;
#else
      return wave_sym_eig_leader(n, m, vals, vecs, ar.wctl, ar.wws, ar.fast);
#endif
    }
    if (std::is_same<Team, BlockTeam>::value && ar.fast && n >= 48 && blockDim.x == kPipeThreads) {
      int R = 8;
      while (R > 4 && pipelined_smem_doubles(n, R) > ar.fast_cap) R -= 2;
      if (pipelined_smem_doubles(n, R) <= ar.fast_cap) {
        const int64_t ld = (n + 1) & ~int64_t(1);
        double* A = ar.take(int64_t(n) * ld);
        double* Vt = ar.take(int64_t(n) * ld);
        return cta_sym_eig_pipelined_any(n, m, vals, vecs, A, Vt, ar.fast, R, ar.sched);
      }
    }
  }
  double* a = ar.take(nn);
  double* v = ar.take(nn);
  double* d = ar.take(n);
  double* bb = ar.take(n);
  double* z = ar.take(n);
  double* slot = ar.take(4);
  for (int64_t e = t.rank(); e < nn; e += t.size()) {
    a[e] = m[e];
    v[e] = (e / n == e % n) ? 1.0 : 0.0;
  }
  t.sync();
  t_symmetrize(t, a, n);
  for (int i = t.rank(); i < n; i += t.size()) {
    d[i] = bb[i] = a[int64_t(i) * n + i];
    z[i] = 0.0;
  }
  t.sync();
  bool converged = false;
  for (int sweep = 0; sweep < 64; ++sweep) {
    if (t.rank() == 0) {
      double sm = 0.0;
      for (int p = 0; p + 1 < n; ++p)
        for (int q = p + 1; q < n; ++q) sm += fabs(a[int64_t(p) * n + q]);
      slot[0] = sm;
    }
    t.sync();
    const double sm = slot[0];
    if (sm == 0.0) {
      converged = true;
      break;
    }
    const double tresh = sweep < 3 ? 0.2 * sm / static_cast<double>(static_cast<uint64_t>(n) * n) : 0.0;
    for (int p = 0; p + 1 < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[int64_t(p) * n + q];
        const double dp = d[p], dq = d[q];
        const double g = 100.0 * fabs(apq);
        if (sweep > 3 && fabs(dp) + g == fabs(dp) && fabs(dq) + g == fabs(dq)) {
          t.sync();
          if (t.rank() == 0) a[int64_t(p) * n + q] = 0.0;
          t.sync();
        } else if (fabs(apq) > tresh) {
          double h = dq - dp;
          double tt;
          if (fabs(h) + g == fabs(h)) {
            tt = apq / h;
          } else {
            const double theta = 0.5 * h / apq;
            tt = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
            if (theta < 0.0) tt = -tt;
          }
          const double c = 1.0 / sqrt(1.0 + tt * tt);
          const double s = tt * c;
          const double tau = s / (1.0 + c);
          h = tt * apq;
          t.sync();  // everyone has read apq, d[p], d[q]
          if (t.rank() == 0) {
            z[p] -= h;
            z[q] += h;
            d[p] -= h;
            d[q] += h;
            a[int64_t(p) * n + q] = 0.0;
          }
          for (int j = t.rank(); j < n; j += t.size()) {
            double *x = nullptr, *y = nullptr;
            if (j < p) {
              x = &a[int64_t(j) * n + p];
              y = &a[int64_t(j) * n + q];
            } else if (j > p && j < q) {
              x = &a[int64_t(p) * n + j];
              y = &a[int64_t(j) * n + q];
            } else if (j > q) {
              x = &a[int64_t(p) * n + j];
              y = &a[int64_t(q) * n + j];
            }
            if (x) {
              const double gx = *x, hy = *y;
              *x = gx - s * (hy + gx * tau);
              *y = hy + s * (gx - hy * tau);
            }
            double* vx = &v[int64_t(j) * n + p];
            double* vy = &v[int64_t(j) * n + q];
            const double gx = *vx, hy = *vy;
            *vx = gx - s * (hy + gx * tau);
            *vy = hy + s * (gx - hy * tau);
          }
          t.sync();
        }
      }
    }
    for (int i = t.rank(); i < n; i += t.size()) {
      bb[i] += z[i];
      d[i] = bb[i];
      z[i] = 0.0;
    }
    t.sync();
  }
  if (!converged) return 1;
  for (int i = 0; i < n; ++i)
    if (!isfinite(d[i])) return 2;
  // stable ascending sort (std::stable_sort, eigen.hpp:107-116)
  for (int k = t.rank(); k < n; k += t.size()) {
    const double dk = d[k];
    int pos = 0;
    for (int i = 0; i < n; ++i)
      if (d[i] < dk || (d[i] == dk && i < k)) ++pos;
    vals[pos] = dk;
    for (int i = 0; i < n; ++i) vecs[int64_t(i) * n + pos] = v[int64_t(i) * n + k];
  }
  t.sync();
  return 0;
}

// Spectral pseudo-inverse with a relative cut (eigen.hpp:215-231).
template <class Team>
__device__ int t_pseudo_inverse(const Team& t, int n, const double* m, double tau_rel, double* out, Arena ar) {
  double* ev = ar.take(n);
  double* eV = ar.take(int64_t(n) * n);
  const int st = t_sym_eig(t, n, m, ev, eV, ar);
  if (st) return st;
  const double cut = n == 0 ? 0.0 : tau_rel * fmax(ev[n - 1], 0.0);
  const int64_t nn = int64_t(n) * n;
  // out(i,j) = Σ_k (V(i,k)·(1/λ_k))·V(j,k) over λ_k > cut, skipping zero V(i,k)/λ_k. The reciprocals
  // are taken once, V is scaled in place and read against a transposed copy (coalesced); a cut λ
  // scales its column to ±0, which the product skips like the reference's `continue`.
  double* vt = ar.take(nn);  // the eigensolver's scratch is free again
  t.sync();
  for (int k = t.rank(); k < n; k += t.size()) ev[k] = ev[k] <= cut ? 0.0 : 1.0 / ev[k];
  for (int64_t e = t.rank(); e < nn; e += t.size()) {
    const int k = static_cast<int>(e / n), j = static_cast<int>(e % n);
    vt[e] = eV[int64_t(j) * n + k];
  }
  t.sync();
  for (int64_t e = t.rank(); e < nn; e += t.size()) eV[e] *= ev[e % n];
  t.sync();
  t_matmul(t, eV, n, n, vt, n, out);
  return 0;
}

// Generalized SPSD pencil l u = λ b u (eigen.hpp:142-209). ls and bs are
// symmetrized in place. Outputs: values[cnt] and vectors column-major
// (vector k at outv + k*n). Returns status; *cnt and *discarded via slots.
template <class Team>
__device__ int t_spsd_gevp(const Team& t, int n, double* ls, double* bs, double tau_rel, double* values,
                           double* outv, int* cnt_out, Arena ar) {
  *cnt_out = 0;
  if (n == 0) return 0;
  t_symmetrize(t, ls, n);
  t_symmetrize(t, bs, n);
  double* ebv = ar.take(n);
  double* ebV = ar.take(int64_t(n) * n);
  double* slot = ar.take(4);
  int st = t_sym_eig(t, n, bs, ebv, ebV, ar);
  if (st) return st;
  const double mu_max = fmax(ebv[n - 1], 0.0);
  const double cut = tau_rel * mu_max;
  int n_null = 0;
  while (n_null < n && ebv[n_null] <= cut) ++n_null;
  const int n_ret = n - n_null;
  if (ar.fast && ar.fast_cap >= 64) {  // frobenius_norm (dense.hpp:96-100): squares by the team, ordered sum by rank 0
    const int64_t nn = int64_t(n) * n, cap = ar.fast_cap;
    double s = 0.0;
    for (int64_t e0 = 0; e0 < nn; e0 += cap) {
      const int64_t len = nn - e0 < cap ? nn - e0 : cap;
      for (int64_t e = t.rank(); e < len; e += t.size()) ar.fast[e] = ls[e0 + e] * ls[e0 + e];
      t.sync();
      if (t.rank() == 0)
        for (int64_t e = 0; e < len; ++e) s += ar.fast[e];
      t.sync();
    }
    if (t.rank() == 0) slot[0] = sqrt(s);
  } else if (t.rank() == 0) {
    double s = 0.0;
    for (int64_t e = 0; e < int64_t(n) * n; ++e) s += ls[e] * ls[e];
    slot[0] = sqrt(s);
  }
  t.sync();
  const double l_scale = slot[0];
  int cnt = 0;
  if (n_null > 0) {
    Arena a2 = ar;
    double* vn = a2.take(int64_t(n) * n_null);
    double* lv = a2.take(int64_t(n) * n_null);
    double* tm = a2.take(int64_t(n_null) * n_null);
    double* etv = a2.take(n_null);
    double* etV = a2.take(int64_t(n_null) * n_null);
    for (int64_t e = t.rank(); e < int64_t(n) * n_null; e += t.size()) {
      const int i = static_cast<int>(e / n_null), k = static_cast<int>(e % n_null);
      vn[e] = ebV[int64_t(i) * n + k];
    }
    t.sync();
    t_matmul(t, ls, n, n, vn, n_null, lv);
    t_matmul_transa(t, vn, n, n_null, lv, n_null, tm);
    t_symmetrize(t, tm, n_null);
    st = t_sym_eig(t, n_null, tm, etv, etV, a2);
    if (st) return st;
    for (int k = n_null; k-- > 0;) {
      if (etv[k] > tau_rel * l_scale) {
        double* u = outv + int64_t(cnt) * n;
        for (int i = t.rank(); i < n; i += t.size()) {
          double s = 0.0;
          for (int j = 0; j < n_null; ++j) s += vn[int64_t(i) * n_null + j] * etV[int64_t(j) * n_null + k];
          u[i] = s;
        }
        if (t.rank() == 0) values[cnt] = __longlong_as_double(0x7ff0000000000000LL);
        ++cnt;
      }
    }
    t.sync();
  }
  if (n_ret > 0) {
    Arena a2 = ar;
    double* w = a2.take(int64_t(n) * n_ret);
    double* lw = a2.take(int64_t(n) * n_ret);
    double* cm = a2.take(int64_t(n_ret) * n_ret);
    double* ecv = a2.take(n_ret);
    double* ecV = a2.take(int64_t(n_ret) * n_ret);
    for (int64_t e = t.rank(); e < int64_t(n) * n_ret; e += t.size()) {
      const int i = static_cast<int>(e / n_ret), j = static_cast<int>(e % n_ret);
      const double scale = 1.0 / sqrt(ebv[n_null + j]);
      w[e] = ebV[int64_t(i) * n + n_null + j] * scale;
    }
    t.sync();
    t_matmul(t, ls, n, n, w, n_ret, lw);
    t_matmul_transa(t, w, n, n_ret, lw, n_ret, cm);
    t_symmetrize(t, cm, n_ret);
    st = t_sym_eig(t, n_ret, cm, ecv, ecV, a2);
    if (st) return st;
    // u_k = w·ecV(·,k), k descending: one product, vector k stored as output column cnt + (n_ret-1-k)
    t_mm_core<false>(t, w, n_ret, 1, n, n_ret, ecV, n_ret, [&](int i, int k, double v) {
      outv[int64_t(cnt + (n_ret - 1 - k)) * n + i] = v;
    });
    for (int k = t.rank(); k < n_ret; k += t.size()) values[cnt + (n_ret - 1 - k)] = ecv[k];
    cnt += n_ret;
    t.sync();
  }
  *cnt_out = cnt;
  return 0;
}

// workspace doubles of t_spsd_gevp beyond its outputs
__host__ __device__ inline int64_t spsd_gevp_scratch(int64_t n) {
  auto r2 = [](int64_t x) { return (x + 1) & ~int64_t(1); };
  // ebv, ebV, slot + max(eig(bs) scratch, null-part, finite-part)
  const int64_t part = r2(n * n) * 3 + r2(n) + r2(n * n) + sym_eig_scratch(n);
  return r2(n) + r2(n * n) + 4 + (sym_eig_scratch(n) > part ? sym_eig_scratch(n) : part);
}

}  // namespace lsb
