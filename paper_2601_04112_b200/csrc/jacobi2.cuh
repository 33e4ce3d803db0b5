// jacobi2.cuh — cyclic Jacobi (eigen.hpp:35-118) with the row-p sweep held in
// the registers of four bulk warps. EXPERIMENTAL (LSB_EIG_SPLIT=2 on the
// dense_sym_eig test hook / g_eig_split = 2): bit-exact, but measured slower
// than the producer/consumer path of dense_dev.cuh (n=550: ~4200 vs ~1750
// cycles per rotation), so it is not the default. The split roles below are
// the current state of the experiment.
//
// Same rotation sequence and IEEE operations as the reference (the library
// is built with --fmad=false), so values and vectors are bit-identical.
//
// Row sweep p applies rotations (p,t), t = p+1..n-1. Rotation t pairs every
// element j ∉ {p,t} of row p, x_j = a(p,j) (for j < p: a(j,p)), with
// y_j = the current entry (min(j,t), max(j,t)):
//     x_j <- x_j - s(y_j + x_j τ),   y_j <- y_j + s(x_j - y_j τ).
// y_j is "row t, position j" of the matrix as the sweep left it: the start-
// of-sweep value for j > t or j < p, and for p < j < t the value rotation j
// wrote (first update of entry (j,t)).
//
// Roles (512 threads):
//   * producer (warp 0, SMSP 0 alone): holds row p in registers (element
//     j = 32k + lane in slot k), computes the rotation parameters (uniform,
//     branch-free, software-pipelined one rotation ahead of the bulk update),
//     applies every rotation to all of row p, writes the rotated y_j of
//     rotation t to an out buffer, and patches the rows t+1..t+W of the ring
//     at position t;
//   * consumers (12 warps on SMSPs 1-3): stream rows of A and Vᵀ into a ring
//     (cp.async), write each out buffer back (row t, and the mirrored column
//     t), patch ring rows at positions the producer does not cover, apply the
//     rotations to Vᵀ (row p in registers);
//   * warps 4, 8, 12 idle.
// Producer and consumers meet through counters in shared memory, not a
// barrier per rotation: the producer waits only when the consumers lag by
// more than W rotations, or a ring row it must patch has not landed.
//
// Included by dense_dev.cuh inside namespace lsb (uses its cp.async helpers).
#pragma once

namespace jac2 {
constexpr int W = 4;    // positions t-W..t-1 of a ring row are patched by the producer
constexpr int DL = 2;   // consumer steps a ring fetch may stay in flight
constexpr int NCT = 352;  // consumer threads (warps 1-3, 8-15)
constexpr int NBW = 4;    // bulk warps (4-7, one per SMSP)
constexpr int NBW_LOG = 2;
constexpr int KC = 3;   // Vᵀ row-p elements per consumer thread (n <= 1152)
}  // namespace jac2

__host__ __device__ inline int64_t jac2_ld(int64_t n) { return (n + 3) & ~int64_t(3); }

// shared doubles used by cta_sym_eig_jac2 with RA ring slots and NO out buffers
__host__ __device__ inline int64_t jac2_smem_doubles(int64_t n, int RA, int NO) {
  return (2 * RA + NO + 3) * jac2_ld(n) + 2 * NO + 64 + 8;
}

// flag handoff in shared memory with release/acquire at CTA scope (not the
// sequentially consistent MEMBAR of __threadfence_block, which also drains
// the thread's outstanding global stores)
__device__ int g_jac2_dbg = 0;

#ifdef LSB_JAC2_ACQREL
__device__ __forceinline__ int ld_vol(const volatile int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];"
               : "=r"(v)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(const_cast<int*>(p))))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(volatile int* p, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(const_cast<int*>(p)))),
               "r"(v)
               : "memory");
}
#else
// Shared-memory flags: the shared-memory pipeline executes one warp's
// accesses in issue order, so a volatile flag store issued after the data
// stores (compiler barrier on both sides) is observed after them; a fence
// here (MEMBAR.*.CTA) costs ~1000 cycles per rotation.
__device__ __forceinline__ int ld_vol(const volatile int* p) {
  const int v = *p;
  asm volatile("" ::: "memory");
  return v;
}
__device__ __forceinline__ void st_rel(volatile int* p, int v) {
  asm volatile("" ::: "memory");
  *p = v;
}
#endif

// branch-free rotation parameters of eigen.hpp:64-80 (selects only)
__device__ __forceinline__ void jac2_params(double apq, double dp, double dq, double tresh, bool late, double& s,
                                            double& tau, double& h, bool& rot, bool& zero) {
  const double g = 100.0 * fabs(apq);
  zero = late && (fabs(dp) + g == fabs(dp)) && (fabs(dq) + g == fabs(dq));
  rot = !zero && (fabs(apq) > tresh);
  const double hh = dq - dp;
  const double t1 = apq / hh;
  const double theta = 0.5 * hh / apq;
  double t2 = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
  t2 = theta < 0.0 ? -t2 : t2;
  const double tt = (fabs(hh) + g == fabs(hh)) ? t1 : t2;
  const double c = 1.0 / sqrt(1.0 + tt * tt);
  const double sv = tt * c;
  const double tv = sv / (1.0 + c);
  const double hv = tt * apq;
  s = rot ? sv : 0.0;
  tau = rot ? tv : 0.0;
  h = rot ? hv : 0.0;
}

// Returns 0, or 1 (no convergence in 64 sweeps) / 2 (non-finite value).
// A, Vt: global n×ld (ld = jac2_ld(n)); sm: shared, jac2_smem_doubles(n,RA,NO).
// Requires blockDim.x == 512, n <= 32*KMAX (KMAX a multiple of NBW), n <= NCT*KC.
template <int KMAX>
__device__ int cta_sym_eig_jac2(int n, const double* m, double* vals, double* vecs, double* A, double* Vt, double* sm,
                                int RA, int NO) {
  using namespace jac2;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  constexpr int KB = KMAX / NBW;  // row-p slots per bulk warp
  // consumers: warps 1-3 and 8-15 -> 0..351
  const int ctid = (wid < 4 ? wid - 1 : wid - 5) * 32 + lane;
  const int64_t ld = jac2_ld(n);
  double* ringA = sm;
  double* ringV = ringA + int64_t(RA) * ld;
  double* outb = ringV + int64_t(RA) * ld;
  double* d = outb + int64_t(NO) * ld;
  double* bb = d + ld;
  double* z = bb + ld;
  double* q_s = z + ld;
  double* q_tau = q_s + NO;
  double* slot = q_tau + NO;                          // 8 doubles
  // [1] consumer step done, [2] rows landed, [3] params published,
  // [5+b] bulk warp b step done, [9+b] bulk warp b early element published
  volatile int* fl = reinterpret_cast<volatile int*>(slot + 8);
  int* q_rot = reinterpret_cast<int*>(slot + 16);     // NO ints (NO <= 32): bit 0 rotate, bit 1 zero
  int* fetch_hi = q_rot + 32;                         // 8 ints: highest row fetched at step % 8
  int* flushed_at = fetch_hi + 8;                     // 8 ints: last flushed rotation at that fetch
  double* eq = slot + 64;                             // 8 doubles: early-published elements

  for (int64_t e = tid; e < int64_t(n) * n; e += blockDim.x) {  // symmetric copy (eigen.hpp:44)
    const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    double val = m[e];
    if (i != j) {
      const int lo = i < j ? i : j, hi = i < j ? j : i;
      val = 0.5 * (m[int64_t(lo) * n + hi] + m[int64_t(hi) * n + lo]);
    }
    A[int64_t(i) * ld + j] = val;
    Vt[int64_t(i) * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  for (int i = tid; i < n; i += blockDim.x) {
    d[i] = bb[i] = m[int64_t(i) * n + i];
    z[i] = 0.0;
  }
  __syncthreads();
  const int chunks = static_cast<int>(ld / 2);
  auto rslot = [&](int row) { return row % RA; };
  // consumers: issue the cp.async pieces of rows [r0, r1] of A and Vᵀ
  auto fetch_rows = [&](int r0, int r1) {
    for (int r = r0; r <= r1; ++r) {
      double* da = ringA + int64_t(rslot(r)) * ld;
      double* dv = ringV + int64_t(rslot(r)) * ld;
      const double* sa = A + int64_t(r) * ld;
      const double* sv = Vt + int64_t(r) * ld;
      for (int c = ctid; c < chunks; c += NCT) {
        cp_async16(da + 2 * c, sa + 2 * c);
        cp_async16(dv + 2 * c, sv + 2 * c);
      }
    }
  };
  auto cbar = []() { asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory"); };
  bool converged = false;
  const bool dbg = g_jac2_dbg != 0;     // timing experiment: consumers idle, 2 sweeps
  const bool nowait = g_jac2_dbg == 2;  // ... and no waiting at all (values meaningless)
  long long* const prof = g_eig_prof;  // optional cycle counters (test hook)
  long long p_wait = 0, p_tot = 0, p_rot = 0, c_wait = 0, c_cpw = 0, c_bar = 0, c_tot = 0, b_wait = 0, b_tot = 0;
  for (int sweep = 0; sweep < (dbg ? 2 : 64); ++sweep) {
    // off-diagonal sum in the reference's order (eigen.hpp:52-54)
    double smv = 0.0;
    for (int p = 0; p + 1 < n; ++p) {
      for (int q = p + 1 + tid; q < n; q += blockDim.x) ringA[q] = A[int64_t(p) * ld + q];
      __syncthreads();
      if (tid == 0)
        for (int q = p + 1; q < n; ++q) smv += fabs(ringA[q]);
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
    const bool late = sweep > 3;
    for (int p = 0; p + 1 < n; ++p) {
      // ---- row start: rows p+1..p+RA land, counters reset
      const int first_hi = min(p + RA, n - 1);
      const bool consumer = wid != 0 && (wid < 4 || wid >= 4 + NBW);
      if (consumer) {
        fetch_rows(p + 1, first_hi);
        cp_async_commit();
        cp_async_wait<0>();
      }
      if (tid == 0) {
        fl[0] = p;
        fl[1] = p;
        fl[2] = first_hi;
        fl[3] = p;
        fl[4] = p;
        for (int k = 5; k < 5 + 2 * NBW; ++k) fl[k] = p;
        for (int k = 0; k < 8; ++k) fetch_hi[k] = first_hi;
      }
      __syncthreads();
      if (wid == 0 && lane == 0) {
        // ---- params thread (lane 0 of warp 0): the sequential chain only
        double dp = d[p], zp = z[p];
        double s_p = 0.0, tau_p = 0.0;  // rotation t-1
        bool rot_p = false;
        const long long pr0 = prof ? clock64() : 0;
        for (int t = p + 1; t < n; ++t) {
          double P;
          if (t == p + 1) {
            P = A[int64_t(p) * ld + t];
          } else {
            // e_t after rotation t-2: initial value for t = p+2, else the bulk warp's early publish
            double pin;
            if (t == p + 2) {
              pin = A[int64_t(p) * ld + t];
            } else {
              const long long w0 = prof ? clock64() : 0;
              const int owner = (t >> 5) & (NBW - 1);  // bulk warp holding element t
              if (!nowait)
                while (ld_vol(fl + 9 + owner) < t - 2) {
                }
              if (prof) p_wait += clock64() - w0;
              pin = eq[t & 7];
            }
            const double y = ringA[int64_t(rslot(t - 1)) * ld + t];  // a(t-1, t), start of sweep
            P = rot_p ? pin - s_p * (y + pin * tau_p) : pin;
          }
          // eigen.hpp:64-80 (uniform branches)
          const double dq = d[t];
          const double g = 100.0 * fabs(P);
          double sv = 0.0, tv = 0.0, hv = 0.0;
          bool rot = false, zero = false;
          if (late && fabs(dp) + g == fabs(dp) && fabs(dq) + g == fabs(dq)) {
            zero = true;
          } else if (fabs(P) > tresh) {
            const double hh = dq - dp;
            double tt;
            if (fabs(hh) + g == fabs(hh)) {
              tt = P / hh;
            } else {
              const double theta = 0.5 * hh / P;
              tt = 1.0 / (fabs(theta) + sqrt(1.0 + theta * theta));
              if (theta < 0.0) tt = -tt;
            }
            const double c = 1.0 / sqrt(1.0 + tt * tt);
            sv = tt * c;
            tv = sv / (1.0 + c);
            hv = tt * P;
            rot = true;
            dp -= hv;
            zp -= hv;
          }
          if (lane == 0) {
            if (rot) {
              d[t] += hv;
              z[t] += hv;
            }
            q_s[t % NO] = sv;
            q_tau[t % NO] = tv;
            q_rot[t % NO] = (rot ? 1 : 0) | (zero ? 2 : 0);
            st_rel(fl + 3, t);
          }
          s_p = sv;
          tau_p = tv;
          rot_p = rot;
        }
        if (lane == 0) {
          d[p] = dp;
          z[p] = zp;
        }
        if (prof) {
          p_tot += clock64() - pr0;
          p_rot += n - p - 1;
        }
      } else if (wid >= 4 && wid < 4 + NBW) {
        // ---- bulk warps (one per SMSP): rotation t on their part of row p.
        // Warp b owns elements j = 32*(NBW*k + b) + lane, k < KB.
        const int b = wid - 4;
        double x[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          const int j = 32 * (NBW * k + b) + lane;
          x[k] = (j < n && j != p) ? A[int64_t(p) * ld + j] : 0.0;
        }
        const long long b0 = prof ? clock64() : 0;
        int st = rslot(p + 1);  // ring slot of row t
        for (int t = p + 1; t < n; ++t) {
          const long long w0 = prof ? clock64() : 0;
          if (lane == 0 && !nowait) {
            const int need_c = max(t - W - 1, t - NO + DL + 9);
            const int need_l = min(t + W, n - 1);
            // ring row t's positions t-W..t-1 are patched by the bulk warp owning element t
            const int own = (t >> 5) & (NBW - 1);
            while (ld_vol(fl + 3) < t || ld_vol(fl + 1) < need_c || ld_vol(fl + 2) < need_l ||
                   ld_vol(fl + 5 + own) < t - 1)
              __nanosleep(16);
          }
          __syncwarp();
          if (prof) b_wait += clock64() - w0;
          const int qi = t % NO;
          const double s_c = q_s[qi], tau_c = q_tau[qi];
          const int fr = q_rot[qi];
          const bool rot_c = (fr & 1) != 0, zero_c = (fr & 2) != 0;
          const double* rt = ringA + int64_t(st) * ld;
          // early publish: element t+2 after rotation t (the params warp's next-but-one pivot)
          const int j2 = t + 2;
          if (j2 < n && ((j2 >> 5) & (NBW - 1)) == b) {
            const int k2 = j2 >> 5 >> NBW_LOG;
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < KB; ++k) v = k == k2 ? x[k] : v;
            if (lane == (j2 & 31)) {
              const double y = rt[j2];
              eq[j2 & 7] = rot_c ? v - s_c * (y + v * tau_c) : v;
              st_rel(fl + 9 + b, t);
            }
          }
          double* ob = outb + int64_t(qi) * ld;
          double yv[KB];
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            const int j = 32 * (NBW * k + b) + lane;
            yv[k] = rt[j < n ? j : n - 1];
          }
#pragma unroll
          for (int k = 0; k < KB; ++k) {
            const int j = 32 * (NBW * k + b) + lane;
            const double y = yv[k];
            const double xv = x[k];
            const double xn = xv - s_c * (y + xv * tau_c);
            const double yn = y + s_c * (xv - y * tau_c);
            const double out = rot_c ? yn : y;
            x[k] = (j == t) ? ((rot_c || zero_c) ? 0.0 : xv) : ((rot_c && j != p) ? xn : xv);
            if (j < n) ob[j] = out;
            const int dj = j - t;
            if (dj > 0 && dj <= W && j < n) {
              const int sj = st + dj >= RA ? st + dj - RA : st + dj;
              ringA[int64_t(sj) * ld + t] = out;
            }
          }
          __syncwarp();  // orders the other lanes' out-buffer stores before lane 0's flag
          if (lane == 0) st_rel(fl + 5 + b, t);
          st = st + 1 == RA ? 0 : st + 1;
        }
        if (prof) b_tot += clock64() - b0;
        // row p is final for this sweep: write this warp's part and its mirror column
#pragma unroll
        for (int k = 0; k < KB; ++k) {
          const int j = 32 * (NBW * k + b) + lane;
          if (j < n && j != p) {
            A[int64_t(p) * ld + j] = x[k];
            A[int64_t(j) * ld + p] = x[k];
          }
        }
      } else if (consumer) {
        double vr[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const int j = ctid + k * NCT;
          vr[k] = j < n ? Vt[int64_t(p) * ld + j] : 0.0;
        }
        int next_fetch = first_hi + 1;
        int last_flushed = p;  // mirrors of rotations <= last_flushed are in global memory
        const long long cs0 = prof ? clock64() : 0;
        for (int c = p + 1; c < n; ++c) {
          const long long w0 = prof ? clock64() : 0;
          if (lane == 0)
            while (ld_vol(fl + 5) < c || ld_vol(fl + 6) < c || ld_vol(fl + 7) < c || ld_vol(fl + 8) < c)
              __nanosleep(32);
          __syncwarp();
          if (prof) c_wait += clock64() - w0;
          if (dbg) {
            if (ctid == 0) {
              st_rel(fl + 2, n - 1);
              st_rel(fl + 1, c);
            }
            continue;
          }
          const int qi = c % NO;
          const bool rot = q_rot[qi] != 0;
          const double s = q_s[qi], tau = q_tau[qi];
          const double* ob = outb + int64_t(qi) * ld;
          const double* vq = ringV + int64_t(rslot(c)) * ld;
          double* vrow = Vt + int64_t(c) * ld;
          double* arow = A + int64_t(c) * ld;
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const int j = ctid + k * NCT;
            if (j < n) {
              if (rot) {
                const double vx = vr[k], vy = vq[j];
                vr[k] = vx - s * (vy + vx * tau);
                vrow[j] = vy + s * (vx - vy * tau);
              }
              if (j != p && j < c) arow[j] = ob[j];  // entry (j,c) final for this sweep
            }
          }
          // mirrored columns, flushed in aligned batches of 8 rotations: row j
          // gets out_t[j] at positions t of the batch as 16-byte pairs, four
          // consecutive threads per row (one 64-byte segment)
          if (((c + 1) & 7) == 0 || c == n - 1) {
            const int c0 = max(p + 1, c & ~7);
            for (int e = ctid; e < 4 * n; e += NCT) {
              const int j = e >> 2, q = e & 3;
              if (j == p) continue;
              const int t0 = (c & ~7) + 2 * q, t1 = t0 + 1;
              double* dst = A + int64_t(j) * ld + t0;
              const bool in0 = t0 >= c0 && t0 <= c, in1 = t1 >= c0 && t1 <= c;
              if (in0 && in1) {
                double2 v2;
                v2.x = outb[int64_t(t0 % NO) * ld + j];
                v2.y = outb[int64_t(t1 % NO) * ld + j];
                *reinterpret_cast<double2*>(dst) = v2;
              } else if (in0) {
                dst[0] = outb[int64_t(t0 % NO) * ld + j];
              } else if (in1) {
                dst[1] = outb[int64_t(t1 % NO) * ld + j];
              }
            }
            last_flushed = c;
          }
          cbar();
          // patch landed ring rows beyond the producer's window at position c
          const int landed = c - 1 - DL > p ? fetch_hi[(c - 1 - DL) & 7] : first_hi;  // landed before this step
          for (int r = c + W + 1 + ctid; r <= landed; r += NCT) ringA[int64_t(rslot(r)) * ld + c] = ob[r];
          // refill the ring: rows up to c+RA (their slots were released by the producer)
          const int hi = min(c + RA, n - 1);
          if (next_fetch <= hi) {
            fetch_rows(next_fetch, hi);
            next_fetch = hi + 1;
          }
          cp_async_commit();
          if (ctid == 0) {
            fetch_hi[c & 7] = next_fetch - 1;
            flushed_at[c & 7] = last_flushed;
          }
          const long long w1 = prof ? clock64() : 0;
          cp_async_wait<DL>();
          const long long w2 = prof ? clock64() : 0;
          cbar();
          if (prof) {
            c_cpw += w2 - w1;
            c_bar += clock64() - w2;
          }
          // rows fetched at step c-DL have landed: catch up the positions whose
          // mirrors were not yet in global memory when they were fetched
          const int f = c - DL;
          if (f > p) {
            const int lo_r = fetch_hi[(f - 1) & 7] + 1, hi_r = fetch_hi[f & 7];
            const int nr = hi_r - lo_r + 1;
            const int t_lo = flushed_at[f & 7] + 1;
            const int np = c - t_lo + 1;
            for (int e = ctid; e < nr * np; e += NCT) {
              const int r = lo_r + e / np, t = t_lo + e % np;
              ringA[int64_t(rslot(r)) * ld + t] = outb[int64_t(t % NO) * ld + r];
            }
          }
          cbar();
          if (ctid == 0) {
            st_rel(fl + 2, f > p ? fetch_hi[f & 7] : first_hi);
            st_rel(fl + 1, c);
          }
        }
        cp_async_wait<0>();
        if (prof) c_tot += clock64() - cs0;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const int j = ctid + k * NCT;
          if (j < n) Vt[int64_t(p) * ld + j] = vr[k];
        }
      }
      __syncthreads();
    }
    for (int i = tid; i < n; i += blockDim.x) {
      bb[i] += z[i];
      d[i] = bb[i];
      z[i] = 0.0;
    }
    __syncthreads();
  }
  if (prof) {
    if (tid == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[0]), p_wait);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[1]), p_tot);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[6]), p_rot);

    }
    if (tid == 128) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[2]), b_wait);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[3]), b_tot);
    }
    if (tid == 32) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[4]), c_wait);
      atomicAdd(reinterpret_cast<unsigned long long*>(&prof[5]), c_tot);
    }
  }
  if (!converged) return 1;
  for (int i = 0; i < n; ++i)
    if (!isfinite(d[i])) return 2;
  for (int k = tid; k < n; k += blockDim.x) {
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

__device__ __noinline__ int cta_sym_eig_jac2_any(int n, const double* m, double* vals, double* vecs, double* A,
                                                 double* Vt, double* sm, int RA, int NO) {
  if (n <= 256) return cta_sym_eig_jac2<8>(n, m, vals, vecs, A, Vt, sm, RA, NO);
  if (n <= 512) return cta_sym_eig_jac2<16>(n, m, vals, vecs, A, Vt, sm, RA, NO);
  return cta_sym_eig_jac2<24>(n, m, vals, vecs, A, Vt, sm, RA, NO);
}
