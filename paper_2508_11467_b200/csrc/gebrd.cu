// One-stage bidiagonalization (GEBRD) on the GPU.
//
// Reference: pkg/src/dcsvd/bidiag.py:113-204 (merged rank-2b LABRD panel +
// single trailing GEMM), arxiv 2508.11467 Alg. 1.
//
// Design: one persistent cooperative kernel per panel, in
// two variants chosen per panel:
//  * labrd2_kernel (small panels, latency-bound): two phases / two grid
//    barriers per column, the panel corrections folded into the GEMVs and the
//    P/Q block rows/columns cached in shared memory (see the kernel comment);
//  * labrd4_kernel (large panels, HBM-bound): each column step is five phases
//    separated by four grid barriers, 1-D work split into per-CTA slices:
//   P1/P5  column update  c = a[k:,k] - P[k:,:2k] Q[k,:2k]   (1-D over rows)
//   P2     LARFG(col) + partial A^T v (2-D blocks) + partial P^T v
//   P3     y = tau (A^T v - Q (P^T v)), row update, row norm   (1-D over cols)
//   P4     LARFG(row) + partial A u (2-D blocks) + partial Q^T u
//   P5     x = pi (A u - P (Q^T u)), fused with the next column update.
// The two big GEMVs read the panel-start trailing matrix (untouched until the
// trailing update), so the A u pass walks each CTA's block in the opposite
// column order of the A^T v pass: the tail of one pass is still in L2 when
// the next one starts ("snake").  All reductions use fixed trees / fixed
// partial order (bit-reproducible).  The trailing update A -= P Q^T is one
// DMMA GEMM (gemm.cu).  The final <= nb columns use a single-CTA GEBD2.
#include <algorithm>
#include <mutex>
#include <cooperative_groups.h>

#include "ctx.cuh"
#include "gemm.cuh"
#include "launch.cuh"

namespace dc {

struct LabrdArgs {
  double* A;
  long long lda;
  int m, n, nb;
  double* P;
  double* Q;
  long long ldp, ldq;
  double *d, *e, *tauq, *taup;
  double *cvec, *rvec, *normc, *normr, *py, *px, *pw, *ps;
  long long ldpy, ldpx;  // leading dims of py (>= n) and px (>= m)
  unsigned* bar;
  int Gr, Gc, RB, CB, CBp;   // 2-D grid Gr x Gc of RB x CB blocks (CBp = CB padded)
  int R1, C1;                // 1-D slices (labrd4_kernel)
  unsigned long long* tlog;  // optional phase timestamps (CTA 0, thread 0)
  int cache_pq;              // labrd4_kernel: P/Q 1-D slices cached in shared memory
  double l2keep;             // labrd4_kernel: bytes of each GEMV pass's tail kept in L2 (evict_last), 0 = plain loads
};

// L2 eviction-priority loads for the GEMV passes: the tail of each pass (read
// first by the next, snake-ordered pass) is loaded evict_last, the rest
// evict_first, so the streamed head cannot push the reusable tail out of L2.
__device__ __forceinline__ unsigned long long l2_policy(bool keep) {
  unsigned long long p;
  if (keep) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_l2hint(const double* ptr, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(ptr), "l"(pol));
  return v;
}

unsigned long long* g_labrd_tlog = nullptr;  // debug: set by dcsvd_debug_labrd_tlog
bool g_labrd_last_two_phase = false;          // debug: variant of the last launch

__device__ __forceinline__ void tmark(const LabrdArgs& a, int idx) {
  if (a.tlog && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.tlog[idx] = t;
  }
}
// debug: per-CTA timestamp (slot base + CTA) for one column step (skew analysis, tools/labrd_skew.py)
__device__ __forceinline__ void tmark_cta(const LabrdArgs& a, int k, int base) {
  if (a.tlog && k == 5 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.tlog[base + blockIdx.x] = t;
  }
}

constexpr int kLabrdThreads = 512;
constexpr int kLabrdWarps = kLabrdThreads / 32;

// Sum of `cnt` partials in fixed order by a fixed block tree.
__device__ __forceinline__ double sum_partials(const double* p, int cnt, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) v += p[i];
  return block_sum(v, sh);
}

// Fixed-order sum of `cnt` strided partials, loads issued 16 at a time.
__device__ __forceinline__ double sum_strided(const double* p, int cnt, long long stride) {
  double s = 0.0;
  for (int q0 = 0; q0 < cnt; q0 += 16) {
    double t[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) t[q] = (q0 + q < cnt) ? p[(long long)(q0 + q) * stride] : 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (q0 + q < cnt) s += t[q];
  }
  return s;
}

// Fixed-order sum of cnt strided partials, up to 32 loads in flight.
__device__ __forceinline__ double sum_strided32(const double* p, int cnt, long long stride) {
  double t[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) t[q] = q < cnt ? p[(long long)q * stride] : 0.0;
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) s += t[q];
  for (int q = 32; q < cnt; ++q) s += p[(long long)q * stride];
  return s;
}

// Fixed-order sum of cnt <= 160 partials, computed redundantly by every warp:
// the same value in every thread without a block barrier.
__device__ __forceinline__ double warp_allsum(const double* p, int cnt) {
  const int lane = threadIdx.x & 31;
  double t[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) t[i] = lane + 32 * i < cnt ? p[lane + 32 * i] : 0.0;
  return warp_sum(((t[0] + t[1]) + (t[2] + t[3])) + t[4]);
}

// Split form of warp_allsum: issue the loads, reduce later (same order).
__device__ __forceinline__ void allsum_load(const double* p, int cnt, double (&t)[5]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 5; ++i) t[i] = lane + 32 * i < cnt ? p[lane + 32 * i] : 0.0;
}
__device__ __forceinline__ double allsum_finish(const double (&t)[5]) {
  return warp_sum(((t[0] + t[1]) + (t[2] + t[3])) + t[4]);
}

// sum_{t < cnt} x[t * stride] * c[t] with four independent partial chains
// (fixed combination order -> deterministic).
__device__ __forceinline__ double dot4(const double* x, long long stride, const double* c, int cnt) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int t = 0;
  for (; t + 4 <= cnt; t += 4) {
    s0 += x[(t + 0) * stride] * c[t + 0];
    s1 += x[(t + 1) * stride] * c[t + 1];
    s2 += x[(t + 2) * stride] * c[t + 2];
    s3 += x[(t + 3) * stride] * c[t + 3];
  }
  for (; t < cnt; ++t) s0 += x[t * stride] * c[t];
  return (s0 + s1) + (s2 + s3);
}

__device__ __forceinline__ void larfg_scalars(double alpha, double nrm2, double& tau, double& beta) {
  const double xn = sqrt(nrm2);
  if (xn == 0.0) {
    tau = 0.0;
    beta = alpha;
  } else {
    beta = -copysign(hypot(alpha, xn), alpha);
    tau = (beta - alpha) / beta;
  }
}

// Four-phase variant (large panels): five phases per column separated by four
// grid barriers with the 1-D work split across CTAs in R1-row / C1-column
// slices (see the file header).  Per-CTA caches of the panel rows of P (1-D row slice) and of Q (1-D column
// slice): every entry of those slices is produced by this CTA (row/column
// ownership is the same in every phase), so the per-row / per-column
// corrections never touch global P/Q for them.
template <int RPL, bool HINT>
__global__ void __launch_bounds__(kLabrdThreads, 1) labrd4_kernel(LabrdArgs a) {
  extern __shared__ double dsm[];
  __shared__ double sh_red[32];
  __shared__ double sh_coef[64];
  __shared__ double sh_row[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x;
  const int G = gridDim.x;
  const int gr = g % a.Gr, gc = g / a.Gr;
  const int m = a.m, n = a.n, nb = a.nb;
  double* __restrict__ A = a.A;
  const long long lda = a.lda, ldp = a.ldp, ldq = a.ldq;
  double* __restrict__ P = a.P;
  double* __restrict__ Q = a.Q;
  unsigned epoch = 0;
  // 2-D block of this CTA
  const int br0 = gr * a.RB, br1 = min(m, br0 + a.RB);
  const int bc0 = gc * a.CB, bc1 = min(n, bc0 + a.CB);
  // 1-D slices
  const int R1 = a.R1, C1 = a.C1;
  const int r1lo = g * R1, r1hi = min(m, r1lo + R1);
  const int c1lo = g * C1, c1hi = min(n, c1lo + C1);
  double* sh_u = dsm;                                      // CB
  double* sh_acc = sh_u + ((a.CB + 1) & ~1);               // kLabrdWarps * RB
  const int myr = r1lo + tid;  // this thread's row in the 1-D slice
  const int myj = c1lo + tid;  // this thread's column in the 1-D slice
  const bool own_r = tid < R1 && myr < r1hi;
  const bool own_c = tid < C1 && myj < c1hi;
  // P/Q slice caches in shared memory when they fit (a.cache_pq), else the
  // same accesses go to global P/Q (writes below then hit the same address twice).
  double* prow;
  double* qrow;
  long long pst, qst;
  if (a.cache_pq) {
    double* Pc = sh_acc + (size_t)kLabrdWarps * a.RB;        // R1 x 2nb (ld R1)
    double* Qc = Pc + (size_t)R1 * 2 * nb;                   // C1 x 2nb (ld C1)
    for (int i = tid; i < (R1 + C1) * 2 * nb; i += blockDim.x) Pc[i] = 0.0;
    prow = Pc + tid;
    qrow = Qc + tid;
    pst = R1;
    qst = C1;
  } else {
    prow = P + myr;
    qrow = Q + myj;
    pst = ldp;
    qst = ldq;
  }

  // ---- phase 1 for k = 0: c = a[:,0]
  {
    double part = 0.0;
    if (own_r) {
      const double c = A[myr];
      a.cvec[myr] = c;
      if (myr > 0) part = c * c;
    }
    part = block_sum(part, sh_red);
    if (tid == 0) a.normc[g] = part;
  }
  tmark(a, 0);
  grid_barrier(a.bar, G, epoch);

  for (int k = 0; k < nb; ++k) {
    const int c0 = 2 * k, c1 = 2 * k + 1;
    const int tb = 1 + 10 * k;
    tmark(a, tb + 0);
    // ================= phase 2: LARFG(col), A^T v, P^T v
    double tau, beta;
    double v[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {  // issue the block-row loads before the reduction
      const int r = br0 + lane + 32 * i;
      v[i] = (r < br1 && r > k) ? a.cvec[r] : 0.0;
    }
    const double cmine = (own_r && myr > k) ? a.cvec[myr] : 0.0;
    const double alpha = a.cvec[k];
    larfg_scalars(alpha, sum_partials(a.normc, G, sh_red), tau, beta);
    tmark(a, tb + 1);
    const double den = alpha - beta;
    if (own_r && myr >= k) {
      if (myr == k) {
        a.d[k] = beta;
        a.tauq[k] = tau;
        A[k + (long long)k * lda] = beta;
        P[k + (long long)c0 * ldp] = 1.0;
        prow[c0 * pst] = 1.0;
      } else {
        const double c = cmine;
        const double ess = tau != 0.0 ? c / den : c;
        A[myr + (long long)k * lda] = ess;
        P[myr + (long long)c0 * ldp] = ess;
        prow[c0 * pst] = ess;
      }
    }
    if (tau != 0.0) {
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = br0 + lane + 32 * i;
        v[i] = (r == k) ? 1.0 : (r > k ? v[i] / den : 0.0);
      }
      const int jstart = max(bc0, k + 1);
      // columns >= jkeep (this block's tail of the pass) are kept in L2 for the A u pass
      const double pass_bytes = 8.0 * (double)(a.m - k) * (double)(a.n - k - 1);
      const double fkeep = a.l2keep > 0.0 ? fmin(1.0, a.l2keep / fmax(pass_bytes, 1.0)) : 1.0;
      const int jkeep = bc1 - (int)ceil(fkeep * (double)max(0, bc1 - jstart));
      const unsigned long long pol_keep = HINT ? l2_policy(true) : 0ull, pol_drop = HINT ? l2_policy(false) : 0ull;
      for (int j = jstart + warp; j < bc1; j += 2 * kLabrdWarps) {
        const int j2 = j + kLabrdWarps;
        const bool has2 = j2 < bc1;
        const double* col0 = A + (long long)j * lda;
        const double* col1 = A + (long long)(has2 ? j2 : j) * lda;
        double x0[RPL], x1[RPL];
        if (HINT) {
          const unsigned long long p0 = j >= jkeep ? pol_keep : pol_drop;
          const unsigned long long p1 = (has2 ? j2 : j) >= jkeep ? pol_keep : pol_drop;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = br0 + lane + 32 * i;
            const bool ok = r < br1;
            x0[i] = ok ? ld_l2hint(col0 + r, p0) : 0.0;
            x1[i] = ok ? ld_l2hint(col1 + r, p1) : 0.0;
          }
        } else {
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = br0 + lane + 32 * i;
            const bool ok = r < br1;
            x0[i] = ok ? col0[r] : 0.0;
            x1[i] = ok ? col1[r] : 0.0;
          }
        }
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          s0 += x0[i] * v[i];
          s1 += x1[i] * v[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s0 += __shfl_xor_sync(0xffffffffu, s0, o);
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        }
        if (lane == 0) {
          a.py[(long long)gr * a.ldpy + j] = s0;
          if (has2) a.py[(long long)gr * a.ldpy + j2] = s1;
        }
      }
      // P^T v over this block's rows for t = gc, gc+Gc, ... < 2k
      for (int t = gc + a.Gc * warp; t < c0; t += a.Gc * kLabrdWarps) {
        const double* pc = P + (long long)t * ldp;
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const int r = br0 + lane + 32 * i;
          if (r < br1) s += pc[r] * v[i];
        }
        s = warp_sum(s);
        if (lane == 0) a.pw[gr * 64 + t] = s;
      }
    }
    tmark_cta(a, k, 400);
    tmark(a, tb + 2);
    grid_barrier(a.bar, G, epoch);
    tmark(a, tb + 3);
    tmark_cta(a, k, 600);

    // ================= phase 3: y, row update, row norm partial
    double pys = 0.0, akj = 0.0;
    if (own_c && myj > k) {  // independent loads first: one L2 round trip
      akj = A[k + (long long)myj * lda];
      if (tau != 0.0) pys = sum_strided(a.py + myj, a.Gr, a.ldpy);
    }
    if (tid < c0) {
      double s = 0.0;
      if (tau != 0.0) s = sum_strided(a.pw + tid, a.Gr, 64);
      sh_coef[tid] = s;
    } else if (tid >= 64 && tid < 64 + c0) {
      sh_row[tid - 64] = P[k + (long long)(tid - 64) * ldp];  // P[k, t], t < 2k
    }
    __syncthreads();
    {
      double part = 0.0;
      if (own_c && myj > k) {
        double y = 0.0;
        if (tau != 0.0) {
          const double s = pys;
          const double corr = dot4(qrow, qst, sh_coef, c0);
          y = tau * (s - corr);
          Q[myj + (long long)c0 * ldq] = y;
          qrow[c0 * qst] = y;
        }
        double upd = dot4(qrow, qst, sh_row, c0);
        upd += y;  // Q[j,2k] * P[k,2k] with P[k,2k] = 1
        const double r = akj - upd;
        A[k + (long long)myj * lda] = r;
        a.rvec[myj] = r;
        if (myj > k + 1) part = r * r;
      }
      part = block_sum(part, sh_red);
      if (tid == 0) a.normr[g] = part;
    }
    tmark(a, tb + 4);
    grid_barrier(a.bar, G, epoch);
    tmark(a, tb + 5);

    // ================= phase 4: LARFG(row), A u, Q^T u
    double pi, betar;
    const int jlo4 = max(bc0, k + 1);
    double rvb[4];  // block-column entries of row k (CB <= 4 * blockDim)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = jlo4 + tid + q * kLabrdThreads;
      rvb[q] = (j < bc1 && j > k + 1) ? a.rvec[j] : 0.0;
    }
    const double rmine = (own_c && myj > k + 1) ? a.rvec[myj] : 0.0;
    const double alr = a.rvec[k + 1];
    larfg_scalars(alr, sum_partials(a.normr, G, sh_red), pi, betar);
    const double denr = alr - betar;
    tmark(a, tb + 6);
    if (own_c && myj > k) {
      if (myj == k + 1) {
        a.e[k] = betar;
        a.taup[k] = pi;
        A[k + (long long)(k + 1) * lda] = betar;
        Q[(k + 1) + (long long)c1 * ldq] = 1.0;
        qrow[c1 * qst] = 1.0;
      } else {
        const double rv = rmine;
        const double ess = pi != 0.0 ? rv / denr : rv;
        A[k + (long long)myj * lda] = ess;
        Q[myj + (long long)c1 * ldq] = ess;
        qrow[c1 * qst] = ess;
      }
    }
    if (pi != 0.0) {
      const int jlo = jlo4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = jlo + tid + q * kLabrdThreads;
        if (j < bc1) sh_u[j - bc0] = (j == k + 1) ? 1.0 : rvb[q] / denr;
      }
      __syncthreads();
      double acc[RPL];
#pragma unroll
      for (int i = 0; i < RPL; ++i) acc[i] = 0.0;
      // descending column order (snake against the A^T v pass), 2 columns per step
      const int nj = bc1 - jlo;
      // this pass ends on the lowest columns: keep those (jj < nkeep) for the next column's A^T v pass
      const double pass_bytes = 8.0 * (double)(a.m - k - 1) * (double)(a.n - k - 1);
      const double fkeep = a.l2keep > 0.0 ? fmin(1.0, a.l2keep / fmax(pass_bytes, 1.0)) : 1.0;
      const int nkeep = (int)ceil(fkeep * (double)max(0, nj));
      const unsigned long long pol_keep = HINT ? l2_policy(true) : 0ull, pol_drop = HINT ? l2_policy(false) : 0ull;
      for (int jj = nj - 1 - warp; jj >= 0; jj -= 2 * kLabrdWarps) {
        const int j = jlo + jj;
        const int jj2 = jj - kLabrdWarps;
        const bool has2 = jj2 >= 0;
        const int j2 = has2 ? jlo + jj2 : j;
        const double u0 = sh_u[j - bc0];
        const double u1 = has2 ? sh_u[j2 - bc0] : 0.0;
        const double* col0 = A + (long long)j * lda;
        const double* col1 = A + (long long)j2 * lda;
        double x0[RPL], x1[RPL];
        if (HINT) {
          const unsigned long long p0 = jj < nkeep ? pol_keep : pol_drop;
          const unsigned long long p1 = (has2 ? jj2 : jj) < nkeep ? pol_keep : pol_drop;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = br0 + lane + 32 * i;
            const bool ok = r < br1;
            x0[i] = ok ? ld_l2hint(col0 + r, p0) : 0.0;
            x1[i] = ok ? ld_l2hint(col1 + r, p1) : 0.0;
          }
        } else {
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = br0 + lane + 32 * i;
            const bool ok = r < br1;
            x0[i] = ok ? col0[r] : 0.0;
            x1[i] = ok ? col1[r] : 0.0;
          }
        }
#pragma unroll
        for (int i = 0; i < RPL; ++i) acc[i] += x0[i] * u0 + x1[i] * u1;
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) sh_acc[warp * a.RB + lane + 32 * i] = acc[i];
      __syncthreads();
      for (int rr = tid; rr < a.RB; rr += blockDim.x) {
        const int r = br0 + rr;
        if (r < br1 && r > k) {
          double s = 0.0;
#pragma unroll
          for (int w = 0; w < kLabrdWarps; ++w) s += sh_acc[w * a.RB + rr];
          a.px[(long long)gc * a.ldpx + r] = s;
        }
      }
      // Q^T u over this block's columns for t = gr, gr+Gr, ... < 2k+1
      for (int t = gr + a.Gr * warp; t < c1; t += a.Gr * kLabrdWarps) {
        const double* qc = Q + (long long)t * ldq;
        double s = 0.0;
        for (int j = jlo + lane; j < bc1; j += 32) s += qc[j] * sh_u[j - bc0];
        s = warp_sum(s);
        if (lane == 0) a.ps[gc * 64 + t] = s;
      }
    }
    tmark_cta(a, k, 800);
    tmark(a, tb + 7);
    grid_barrier(a.bar, G, epoch);
    tmark(a, tb + 8);
    tmark_cta(a, k, 1000);

    // ================= phase 5: x, next column update
    const bool next = k + 1 < nb;
    double pxs = 0.0, ark = 0.0;
    if (own_r && myr > k) {
      if (next) ark = A[myr + (long long)(k + 1) * lda];
      if (pi != 0.0) pxs = sum_strided(a.px + myr, a.Gc, a.ldpx);
    }
    if (tid < c1) {
      double s = 0.0;
      if (pi != 0.0) s = sum_strided(a.ps + tid, a.Gc, 64);
      sh_coef[tid] = s;
    } else if (tid >= 64 && tid < 64 + c1) {
      sh_row[tid - 64] = Q[(k + 1) + (long long)(tid - 64) * ldq];  // Q[k+1, t], t < 2k+1
    }
    __syncthreads();
    {
      double part = 0.0;
      if (own_r && myr > k) {
        double x = 0.0;
        if (pi != 0.0) {
          const double s = pxs;
          const double corr = dot4(prow, pst, sh_coef, c1);
          x = pi * (s - corr);
          P[myr + (long long)c1 * ldp] = x;
          prow[c1 * pst] = x;
        }
        if (next) {
          // a[k+1:, k+1] -= P[k+1:, :2k+2] Q[k+1, :2k+2]   (Q[k+1,2k+1] = 1)
          double upd = dot4(prow, pst, sh_row, c1);
          upd += x;
          const double c = ark - upd;
          A[myr + (long long)(k + 1) * lda] = c;
          a.cvec[myr] = c;
          if (myr > k + 1) part = c * c;
        }
      }
      if (next) {
        part = block_sum(part, sh_red);
        if (tid == 0) a.normc[g] = part;
      }
    }
    tmark(a, tb + 9);
    if (next) grid_barrier(a.bar, G, epoch);
  }
}


// Two phases and two grid barriers per column.  With
// v = [1; c/den] and u = [1; r/den_r] (LARFG, bidiag.py:136-158), the panel
// corrections can be folded into the GEMVs on the implicitly updated matrix
// A - P Q^T:
//   y_j = tau (rt_j + S_j / den),  S_j = sum_{i>k} (A - P Q^T)[i,j] c_i
//   x_i = pi  (ct_i + T_i / den_r), T_i = sum_{j>k} (A - P Q^T)[i,j] r_j
// where ct = a[:,k] - P[:, :2k-1] Q[k, :2k-1]^T (column update before x) and
// rt = a[k,:] - Q[:, :2k] P[k, :2k]^T (row update before y).  So:
//   A_k  LARFG(row k-1) from the reduced row norm -> u; x_{k-1} = pi (ct + T/den_r)
//        and c = ct - x for the block rows (O(1) per row); norm partial of c;
//        then the local P^T c, the Q-correction of the block's partial A^T c,
//        E = Q[:, :2k-1] P[k, :2k-1]^T for the next phase, and the partial GEMV.
//   B_k  LARFG(col k) from the reduced norm -> v; y and r = rt - y for the
//        block columns (O(1) per column); norm partial of r; then the local
//        Q^T r, the P-correction of the partial A r, D = P[:, :2k] Q[k+1, :2k]^T
//        for the next phase, and the partial GEMV.
// Every CTA computes the 1-D quantities of its own block rows/columns
// (identically across the other grid dimension) and keeps its P rows / Q
// columns in shared memory; owners (gc == 0 for rows, gr == 0 for columns)
// write them back.  Values produced in a phase are read by other CTAs only
// after the next barrier.  Used when the P/Q block caches fit (small panels).
// Butterfly reduce-scatter of four per-lane partials v[q] (q = 0..3): returns
// in every lane the warp total of v[q] for q = 2 ((lane >> 4) & 1) + ((lane >> 3) & 1)
// (valid in all lanes; lanes with (lane & 7) == 0 are the natural writers).
// 3 + 3 shuffles instead of 4 x 5; fixed order, deterministic.
__device__ __forceinline__ double warp_reduce4_scatter(double (&v)[4], int lane) {
#pragma unroll
  for (int h = 2, off = 16; h >= 1; h >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int c = 0; c < h; ++c) {
      const double send = up ? v[c] : v[c + h];
      const double keep = up ? v[c + h] : v[c];
      v[c] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
  return v[0];
}

template <int RPL>
__global__ void __launch_bounds__(kLabrdThreads, 1) labrd2_kernel(LabrdArgs a) {
  extern __shared__ double dsm[];
  __shared__ double sh_red[32];
  __shared__ double sh_pl[64];   // local P^T c / Q^T r (entries past the live range stay 0)
  __shared__ double sh_row[64];  // P[k, :] (phase A) / Q[k+1, :] (phase B)
  constexpr int RB = 32 * RPL;
  constexpr int LP = RB + 1;     // padded leading dimension of the P cache
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x, G = gridDim.x;
  const int gr = g % a.Gr, gc = g / a.Gr;
  const int nb = a.nb;
  double* __restrict__ A = a.A;
  const long long lda = a.lda, ldp = a.ldp, ldq = a.ldq;
  double* __restrict__ P = a.P;
  double* __restrict__ Q = a.Q;
  unsigned epoch = 0;
  const int br0 = gr * RB, br1 = min(a.m, br0 + RB), nbr = br1 - br0;
  const int bc0 = gc * a.CB, bc1 = min(a.n, bc0 + a.CB), ncb = bc1 - bc0;
  const int CBp = a.CBp, LQ = CBp + 1;
  const bool rowowner = gc == 0, colowner = gr == 0;
  double* sh_c = dsm;                // RB   c (rows > k) = weights of A^T c
  double* sh_D = sh_c + RB;          // RB   P[:, :2k-2] Q[k, :2k-2]^T
  double* sh_cp = sh_D + RB;         // RB   P-correction of A r
  double* sh_r = sh_cp + RB;         // CBp  r (columns > k)
  double* sh_E = sh_r + CBp;         // CBp  Q[:, :2k-1] P[k, :2k-1]^T
  double* sh_cq = sh_E + CBp;        // CBp  Q-correction of A^T c
  double* sh_acc = sh_cq + CBp;      // kLabrdWarps x RB
  const int NC = (2 * nb + 3) & ~3;         // cached P/Q columns, padded to 4
  double* Pc = sh_acc + kLabrdWarps * RB;  // LP x NC: P rows of the block
  double* Qc = Pc + LP * NC;               // LQ x NC: Q rows of the block columns
  {
    const int nvec = 3 * RB + 3 * CBp;
    const int tot = nvec + (LP + LQ) * NC;
    for (int i = tid; i < tot; i += blockDim.x) (i < nvec ? dsm[i] : Pc[i - nvec]) = 0.0;
    if (tid < 64) {
      sh_pl[tid] = 0.0;
      sh_row[tid] = 0.0;
    }
  }
  __syncthreads();

  for (int k = 0; k <= nb; ++k) {
    const bool colstep = k < nb;
    const int tb = 1 + 8 * k;
    tmark(a, tb + 0);
    // ======================= phase A_k (critical part: one L2 round trip of loads)
    const int tx = 2 * k - 1;  // column of x_{k-1} (P) and u_{k-1} (Q)
    const int rr = tid;
    const int r = br0 + rr;
    const bool rv = rr < nbr && r >= k;
    double ark = 0.0, pxs = 0.0;
    if (rv) ark = A[r + (long long)k * lda];
    if (rv && k > 0) pxs = sum_strided32(a.px + r, a.Gc, a.ldpx);
    double prow = 0.0;
    if (colstep && tid < 2 * k - 1) prow = P[k + (long long)tid * ldp];  // P[k, t], t < 2k-1
    const double yk = k > 0 ? Q[k + (long long)(2 * k - 2) * ldq] : 0.0;  // y_{k-1}[k]
    double pi = 0.0, denr = 1.0, betar = 0.0;
    tmark(a, 600 + 8 * k + 0);
    if (k > 0) {
      const double alr = a.rvec[k];
      larfg_scalars(alr, warp_allsum(a.normr, a.Gc), pi, betar);
      denr = alr - betar;
      // u_{k-1} for the block columns j >= k; owners write Q[:, 2k-1] and row k-1 of A
      for (int jj = tid; jj < ncb; jj += blockDim.x) {
        const int j = bc0 + jj;
        double u = 0.0;
        if (j >= k) {
          const double rj = sh_r[jj];
          u = j == k ? 1.0 : (pi != 0.0 ? rj / denr : rj);
          if (colowner) {
            Q[j + (long long)tx * ldq] = u;
            A[(k - 1) + (long long)j * lda] = j == k ? betar : u;
          }
        }
        Qc[jj + tx * LQ] = u;
      }
      if (colowner && tid == 0 && bc0 <= k && k < bc1) {
        a.e[k - 1] = betar;
        a.taup[k - 1] = pi;
      }
    }
    tmark(a, 600 + 8 * k + 1);
    // x_{k-1} and c_k for the block rows
    double part = 0.0;
    if (rr < RB) {
      double x = 0.0, c = 0.0;
      if (rv) {
        const double ct = ark - sh_D[rr] - (k > 0 ? Pc[rr + (2 * k - 2) * LP] * yk : 0.0);
        if (k > 0 && pi != 0.0) x = pi * (ct + pxs / denr);
        c = ct - x;
        if (k > 0 && rowowner) P[r + (long long)tx * ldp] = x;
        if (colstep) {
          if (r == k && rowowner) a.cvec[k] = c;
          if (r > k) part = c * c;
        }
      }
      if (k > 0) Pc[rr + tx * LP] = x;
      sh_c[rr] = (rv && r > k) ? c : 0.0;
    }
    if (colstep && tid < 2 * k - 1) sh_row[tid] = prow;
    tmark(a, 600 + 8 * k + 2);
    if (!colstep) break;
    part = block_sum(part, sh_red);  // also publishes sh_c / Pc / Qc / sh_row
    if (rowowner && tid == 0) a.normc[gr] = part;
    tmark(a, tb + 1);
    // local P^T c over the block rows, t < 2k: warp w handles t = w + 16 q
    // (q < 4, 2k <= 62) together, one reduce-scatter for the four sums
    {
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = warp + kLabrdWarps * q;
        double s = 0.0;
        if (t < 2 * k) {
#pragma unroll
          for (int i = 0; i < RPL; ++i) s += Pc[lane + 32 * i + t * LP] * sh_c[lane + 32 * i];
        }
        v[q] = s;
      }
      const double tot = warp_reduce4_scatter(v, lane);
      const int t = warp + kLabrdWarps * (2 * ((lane >> 4) & 1) + ((lane >> 3) & 1));
      if ((lane & 7) == 0 && t < 2 * k) sh_pl[t] = tot;
    }
    __syncthreads();
    // Q-correction of the partial A^T c and E = Q[:, :2k-1] P[k, :2k-1]^T for
    // the block columns j > k (thread per column, four independent chains;
    // sh_row[2k-1] and everything past the live ranges are 0)
    for (int jj = max(k + 1 - bc0, 0) + tid; jj < ncb; jj += blockDim.x) {
      const double* qj = Qc + jj;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0, e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll 2
      for (int t = 0; t < 2 * k; t += 4) {
        const double q0 = qj[t * LQ], q1 = qj[(t + 1) * LQ], q2 = qj[(t + 2) * LQ], q3 = qj[(t + 3) * LQ];
        c0 += q0 * sh_pl[t];
        c1 += q1 * sh_pl[t + 1];
        c2 += q2 * sh_pl[t + 2];
        c3 += q3 * sh_pl[t + 3];
        e0 += q0 * sh_row[t];
        e1 += q1 * sh_row[t + 1];
        e2 += q2 * sh_row[t + 2];
        e3 += q3 * sh_row[t + 3];
      }
      sh_cq[jj] = (c0 + c1) + (c2 + c3);
      sh_E[jj] = (e0 + e1) + (e2 + e3);
    }
    __syncthreads();
    tmark(a, tb + 2);
    {
      double w[RPL];
#pragma unroll
      for (int i = 0; i < RPL; ++i) w[i] = sh_c[lane + 32 * i];
      // A^T c over the block (rows > k, columns > k): NC columns per warp step
      // (loads of all NC columns in flight), the NC lane partials reduced by a
      // butterfly reduce-scatter (NC - 1 + 5 - log2 NC shuffles instead of 5 NC)
      constexpr int NC = RPL >= 16 ? 2 : (RPL >= 8 ? 4 : 8);
      const int jstart = max(bc0, k + 1);
      for (int jb = jstart + warp; jb < bc1; jb += NC * kLabrdWarps) {
        double v[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int j = jb + c * kLabrdWarps;
          const double* col = A + (long long)(j < bc1 ? j : jb) * lda;
          double x[RPL];
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int rw = br0 + lane + 32 * i;
            x[i] = (rw < br1 && j < bc1) ? col[rw] : 0.0;
          }
          double sc = 0.0;
#pragma unroll
          for (int i = 0; i < RPL; ++i) sc += x[i] * w[i];
          v[c] = sc;
        }
        // reduce-scatter: after the halving steps lane l holds column
        // cl = bits (l>>4, l>>3, l>>2) (top log2 NC of them) summed over the
        // lanes that share those bits; then full xor reductions
#pragma unroll
        for (int h = NC / 2, off = 16; h >= 1; h >>= 1, off >>= 1) {
          const bool up = (lane & off) != 0;
#pragma unroll
          for (int c = 0; c < h; ++c) {
            const double send = up ? v[c] : v[c + h];
            const double keep = up ? v[c + h] : v[c];
            v[c] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        constexpr int LOGNC = NC == 2 ? 1 : (NC == 4 ? 2 : 3);
#pragma unroll
        for (int off = 16 >> LOGNC; off > 0; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
        int cl = 0;
#pragma unroll
        for (int b = 0; b < LOGNC; ++b) cl |= ((lane >> (4 - b)) & 1) << (LOGNC - 1 - b);
        const int j = jb + cl * kLabrdWarps;
        if ((lane & ((16 >> LOGNC) * 2 - 1)) == 0 && j < bc1)
          a.py[(long long)gr * a.ldpy + j] = v[0] - sh_cq[j - bc0];
      }
    }
    tmark(a, tb + 3);
    grid_barrier(a.bar, G, epoch);
    tmark(a, tb + 4);

    // ======================= phase B_k (critical part)
    const int ty = 2 * k;  // column of v_k (P) and y_k (Q)
    double akj[4], pys[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = tid + q * kLabrdThreads;
      const int j = bc0 + jj;
      akj[q] = (jj < ncb && j > k) ? A[k + (long long)j * lda] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = tid + q * kLabrdThreads;
      const int j = bc0 + jj;
      pys[q] = (jj < ncb && j > k) ? sum_strided32(a.py + j, a.Gr, a.ldpy) : 0.0;
    }
    double qrow = 0.0;
    if (tid < 2 * k) qrow = Q[(k + 1) + (long long)tid * ldq];  // Q[k+1, t], t < 2k
    const double xk = k > 0 ? P[k + (long long)(2 * k - 1) * ldp] : 0.0;  // x_{k-1}[k]
    const double alpha = a.cvec[k];
    double tau, beta;
    tmark(a, 600 + 8 * k + 4);
    larfg_scalars(alpha, warp_allsum(a.normc, a.Gr), tau, beta);
    tmark(a, 600 + 8 * k + 5);
    const double den = alpha - beta;
    // v_k for the block rows r >= k; owners write P[:, 2k] and column k of A
    if (rr < RB) {
      double v = 0.0;
      if (rv) {
        const double cr = sh_c[rr];
        v = r == k ? 1.0 : (tau != 0.0 ? cr / den : cr);
        if (rowowner) {
          P[r + (long long)ty * ldp] = v;
          A[r + (long long)k * lda] = r == k ? beta : v;
        }
      }
      Pc[rr + ty * LP] = v;
    }
    if (rowowner && tid == 0 && br0 <= k && k < br1) {
      a.d[k] = beta;
      a.tauq[k] = tau;
    }
    // y_k and r for the block columns j > k
    part = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = tid + q * kLabrdThreads;
      if (jj >= ncb) break;
      const int j = bc0 + jj;
      double y = 0.0, rj = 0.0;
      if (j > k) {
        const double rt = akj[q] - sh_E[jj] - (k > 0 ? Qc[jj + (ty - 1) * LQ] * xk : 0.0);
        if (tau != 0.0) y = tau * (rt + pys[q] / den);
        rj = rt - y;  // P[k, 2k] = 1
        if (colowner) {
          Q[j + (long long)ty * ldq] = y;
          if (j == k + 1) a.rvec[k + 1] = rj;
        }
        if (j > k + 1) part += rj * rj;
      }
      sh_r[jj] = rj;
      Qc[jj + ty * LQ] = y;
    }
    if (tid < 2 * k) sh_row[tid] = qrow;
    tmark(a, 600 + 8 * k + 6);
    part = block_sum(part, sh_red);  // also publishes sh_r / Pc / Qc / sh_row
    if (colowner && tid == 0) a.normr[gc] = part;
    tmark(a, tb + 5);
    const int jlo = max(bc0, k + 2);
    // local Q^T r over the block columns (> k+1), t < 2k+1 (<= 63): warp w
    // handles t = w + 16 q (q < 4) in one pass over the columns
    {
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      for (int jj = jlo - bc0 + lane; jj < ncb; jj += 32) {
        const double rj = sh_r[jj];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int t = warp + kLabrdWarps * q;
          if (t < ty + 1) v[q] += Qc[jj + t * LQ] * rj;
        }
      }
      const double tot = warp_reduce4_scatter(v, lane);
      const int t = warp + kLabrdWarps * (2 * ((lane >> 4) & 1) + ((lane >> 3) & 1));
      if ((lane & 7) == 0 && t < ty + 1) sh_pl[t] = tot;
    }
    __syncthreads();
    // P-correction of the partial A r and D = P[:, :2k] Q[k+1, :2k]^T for the
    // block rows r > k (thread per row, four independent chains; sh_row[2k..]
    // and sh_pl[2k+1..] are 0)
    for (int q = max(k + 1 - br0, 0) + tid; q < nbr; q += blockDim.x) {
      const double* pq = Pc + q;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll 2
      for (int t = 0; t <= ty; t += 4) {
        const double p0 = pq[t * LP], p1 = pq[(t + 1) * LP], p2 = pq[(t + 2) * LP], p3 = pq[(t + 3) * LP];
        c0 += p0 * sh_pl[t];
        c1 += p1 * sh_pl[t + 1];
        c2 += p2 * sh_pl[t + 2];
        c3 += p3 * sh_pl[t + 3];
        d0 += p0 * sh_row[t];
        d1 += p1 * sh_row[t + 1];
        d2 += p2 * sh_row[t + 2];
        d3 += p3 * sh_row[t + 3];
      }
      sh_cp[q] = (c0 + c1) + (c2 + c3);
      sh_D[q] = (d0 + d1) + (d2 + d3);
    }
    tmark(a, tb + 6);
    {
      // A r over the block (rows > k, columns > k+1), descending column order
      // (snake against the A^T c pass), NCB columns per warp step
      constexpr int NCB = RPL >= 8 ? 2 : (RPL >= 4 ? 4 : 8);
      double acc[RPL];
#pragma unroll
      for (int i = 0; i < RPL; ++i) acc[i] = 0.0;
      const int nj = bc1 - jlo;
      for (int jj = nj - 1 - warp; jj >= 0; jj -= NCB * kLabrdWarps) {
        double x[NCB][RPL], u[NCB];
#pragma unroll
        for (int c = 0; c < NCB; ++c) {
          const int jc = jj - c * kLabrdWarps;
          const int j = jlo + (jc >= 0 ? jc : jj);
          u[c] = jc >= 0 ? sh_r[j - bc0] : 0.0;
          const double* col = A + (long long)j * lda;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int rw = br0 + lane + 32 * i;
            x[c][i] = (rw < br1 && jc >= 0) ? col[rw] : 0.0;
          }
        }
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
          for (int i = 0; i < RPL; ++i) acc[i] += x[c][i] * u[c];
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) sh_acc[warp * RB + lane + 32 * i] = acc[i];
      __syncthreads();
      if (rr < nbr && r > k) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kLabrdWarps; ++w) s += sh_acc[w * RB + rr];
        a.px[(long long)gc * a.ldpx + r] = s - sh_cp[rr];
      }
    }
    tmark(a, tb + 7);
    grid_barrier(a.bar, G, epoch);
  }
}

// ---------------------------------------------------------------------------
// Unblocked GEBD2 on a small trailing matrix (bidiag.py:75-110), one CTA.
constexpr int kGebd2Threads = 1024;

__global__ void __launch_bounds__(kGebd2Threads) gebd2_kernel(double* A, long long lda, int m, int n,
                                                              double* d, double* e, double* tauq,
                                                              double* taup, double* wbuf) {
  __shared__ double sh_red[32];
  __shared__ double sh_s[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < n; ++k) {
    // column reflector
    double part = 0.0;
    for (int r = k + 1 + tid; r < m; r += blockDim.x) {
      const double x = A[r + (long long)k * lda];
      part += x * x;
    }
    const double nrm2 = block_sum(part, sh_red);
    const double alpha = A[k + (long long)k * lda];
    double tau, beta;
    larfg_scalars(alpha, nrm2, tau, beta);
    const double den = alpha - beta;
    __syncthreads();
    if (tid == 0) {
      tauq[k] = tau;
      d[k] = beta;
      A[k + (long long)k * lda] = beta;
    }
    if (tau != 0.0)
      for (int r = k + 1 + tid; r < m; r += blockDim.x) A[r + (long long)k * lda] /= den;
    __syncthreads();
    if (tau != 0.0 && k + 1 < n) {
      // w_j = sum_{r>=k} v_r a[r,j]  (v_k = 1)
      for (int j = k + 1 + warp; j < n; j += nw) {
        const double* col = A + (long long)j * lda;
        double s = 0.0;
        for (int r = k + lane; r < m; r += 32) s += (r == k ? 1.0 : A[r + (long long)k * lda]) * col[r];
        s = warp_sum(s);
        if (lane == 0) wbuf[j] = s;
      }
      __syncthreads();
      for (int j = k + 1; j < n; ++j) {
        const double wj = wbuf[j];
        for (int r = k + tid; r < m; r += blockDim.x) {
          const double vr = r == k ? 1.0 : A[r + (long long)k * lda];
          A[r + (long long)j * lda] -= tau * (vr * wj);
        }
      }
      __syncthreads();
    }
    if (k < n - 1) {
      // row reflector on a[k, k+1:]
      part = 0.0;
      for (int j = k + 2 + tid; j < n; j += blockDim.x) {
        const double x = A[k + (long long)j * lda];
        part += x * x;
      }
      const double nr2 = block_sum(part, sh_red);
      const double al = A[k + (long long)(k + 1) * lda];
      double pi, br;
      larfg_scalars(al, nr2, pi, br);
      const double dr = al - br;
      __syncthreads();
      if (tid == 0) {
        taup[k] = pi;
        e[k] = br;
        A[k + (long long)(k + 1) * lda] = br;
      }
      if (pi != 0.0)
        for (int j = k + 2 + tid; j < n; j += blockDim.x) A[k + (long long)j * lda] /= dr;
      __syncthreads();
      if (pi != 0.0) {
        // w_r = sum_{j>=k+1} a[r,j] u_j for r >= k+1 (u_{k+1} = 1)
        for (int r = k + 1 + tid; r < m; r += blockDim.x) {
          double s = A[r + (long long)(k + 1) * lda];
          for (int j = k + 2; j < n; ++j) s += A[r + (long long)j * lda] * A[k + (long long)j * lda];
          wbuf[r] = s;
        }
        __syncthreads();
        for (int j = k + 1; j < n; ++j) {
          const double uj = j == k + 1 ? 1.0 : A[k + (long long)j * lda];
          for (int r = k + 1 + tid; r < m; r += blockDim.x) A[r + (long long)j * lda] -= pi * (wbuf[r] * uj);
        }
        __syncthreads();
      }
    }
    (void)sh_s;
  }
  if (tid == 0) taup[n - 1] = 0.0;
}

// ---------------------------------------------------------------------------
// GEBD2 on one thread-block cluster (gebrd_unblocked, bidiag.py:75-110) for
// the trailing block once it fits in the cluster's distributed shared memory
// (<= ~600 x 600 on 16 SMs).  Each CTA keeps a row slab of the block (all
// columns) in shared memory; per column the only cross-CTA traffic is DSMEM
// reads behind four cluster barriers: the column norm partials, the w = A^T v
// partials (reduce-scatter, then gather) and the row reflector published by
// the owner of row k.  Replaces the latency-bound panel path at small sizes
// (two grid barriers plus L2 round trips per column).
constexpr int kG2cThreads = 512;
constexpr int kG2cSmemMax = 224 * 1024;
int g_gebd2_cluster = 1;  // debug: 0 = never use the cluster kernel, 8 = force 8-CTA clusters

struct Gebd2cArgs {
  double* A;
  long long lda;
  int m, n;
  double *d, *e, *tauq, *taup;
  int R, LD;  // rows per CTA, slab leading dimension
  double* ug;  // n: the row reflector u, broadcast through L2 (one source, 16 readers)
  unsigned long long* tlog;
};

__global__ void __launch_bounds__(kG2cThreads, 1) gebd2_cluster_kernel(Gebd2cArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int m = a.m, n = a.n, R = a.R, LD = a.LD;
  const int r0 = rank * R, nr = max(0, min(m, r0 + R) - r0);
  const int S = (n + CS - 1) / CS;  // w slice per CTA
  int rs = 0;
  while ((1 << rs) < R) ++rs;
  const int RP = 1 << rs;  // row lanes of the update loops (R <= 448 < kG2cThreads)
  extern __shared__ __align__(16) double sm[];
  double* slab = sm;                      // LD x n: rows r0 .. r0 + nr
  double* wpart = slab + (size_t)LD * n;  // this CTA's partial w
  double* wred = wpart + n;               // reduced w, this CTA's slice
  double* vec = wred + n;                 // local copy of w, then of u
  double* xr = vec + n;                   // x for own rows
  __shared__ double sh_red[32];
  __shared__ double sh_pn, sh_al, sh_s[2];
  for (int idx = tid; idx < nr * n; idx += blockDim.x) {
    const int rr = idx % nr, j = idx / nr;
    slab[rr + (size_t)j * LD] = a.A[(r0 + rr) + (long long)j * a.lda];
  }
  __syncthreads();
  auto mk = [&](int k, int slot) {  // debug: clock64 marks of CTA 0, column 5
    if (a.tlog && k == 5 && rank == 0 && tid == 0) a.tlog[slot] = clock64();
  };
  for (int k = 0; k < n; ++k) {
    const int ok = k / R;  // CTA owning row k
    mk(k, 0);
    // column reflector: partial ||a[k+1:, k]||^2 of own rows
    double part = 0.0;
    for (int rr = max(0, k + 1 - r0) + tid; rr < nr; rr += blockDim.x) {
      const double x = slab[rr + (size_t)k * LD];
      part += x * x;
    }
    part = block_sum(part, sh_red);
    mk(k, 1);
    if (tid == 0) {
      sh_pn = part;
      if (rank == ok) sh_al = slab[(k - r0) + (size_t)k * LD];
    }
    cl.sync();  // #1
    mk(k, 2);
    if (warp == 0) {  // the CS norm partials and alpha in one DSMEM round trip
      double v = lane < CS ? *cl.map_shared_rank(&sh_pn, lane) : 0.0;
      const double al = lane == 31 ? *cl.map_shared_rank(&sh_al, ok) : 0.0;
      v = warp_sum(lane == 31 ? 0.0 : v);
      if (lane == 0) sh_s[0] = v;
      if (lane == 31) sh_s[1] = al;
    }
    __syncthreads();
    const double alpha = sh_s[1];
    double tau, beta;
    larfg_scalars(alpha, sh_s[0], tau, beta);
    const double den = alpha - beta;
    if (rank == 0 && tid == 0) {
      a.tauq[k] = tau;
      a.d[k] = beta;
    }
    for (int rr = max(0, k - r0) + tid; rr < nr; rr += blockDim.x) {
      if (r0 + rr == k) slab[rr + (size_t)k * LD] = beta;
      else if (tau != 0.0) slab[rr + (size_t)k * LD] /= den;
    }
    __syncthreads();
    mk(k, 3);
    const bool left = tau != 0.0 && k + 1 < n;
    if (left) {  // partial w_j = sum_{own r >= k} v_r a[r, j]
      const int lo = max(0, k - r0);
      const double* vk = slab + (size_t)k * LD;
      for (int j = k + 1 + tid; j < n; j += blockDim.x) {
        const double* col = slab + (size_t)j * LD;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // four chains, fixed combination order
        int rr = lo;
        if (rr < nr && r0 + rr == k) s0 = col[rr++];  // v_k = 1
        for (; rr + 3 < nr; rr += 4) {
          s0 = fma(vk[rr], col[rr], s0);
          s1 = fma(vk[rr + 1], col[rr + 1], s1);
          s2 = fma(vk[rr + 2], col[rr + 2], s2);
          s3 = fma(vk[rr + 3], col[rr + 3], s3);
        }
        for (; rr < nr; ++rr) s0 = fma(vk[rr], col[rr], s0);
        wpart[j] = (s0 + s1) + (s2 + s3);
      }
    }
    mk(k, 4);
    cl.sync();  // #2
    mk(k, 5);
    if (left) {  // reduce this CTA's slice of w over the cluster (fixed order)
      for (int j = max(k + 1, rank * S) + tid; j < min(n, (rank + 1) * S); j += blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < CS; ++c) s += cl.map_shared_rank(wpart, c)[j];
        wred[j] = s;
      }
    }
    mk(k, 6);
    cl.sync();  // #3
    mk(k, 7);
    if (left) {
      for (int j = k + 1 + tid; j < n; j += blockDim.x) vec[j] = cl.map_shared_rank(wred, j / S)[j];
      __syncthreads();
      // thread (row lane, column group): RP = 2^rs >= R row lanes, no divisions
      const int rr = max(0, k - r0) + (tid & (RP - 1));
      if (rr < nr) {
        const double vr = r0 + rr == k ? 1.0 : slab[rr + (size_t)k * LD];
        for (int j = k + 1 + (tid >> rs); j < n; j += (kG2cThreads >> rs))
          slab[rr + (size_t)j * LD] -= tau * (vr * vec[j]);
      }
    }
    __syncthreads();
    mk(k, 8);
    if (k + 1 >= n) break;
    // row reflector on a[k, k+1:] (owner of row k), published through L2 (a.ug)
    if (rank == ok) {
      const int rk = k - r0;
      part = 0.0;
      for (int j = k + 2 + tid; j < n; j += blockDim.x) {
        const double x = slab[rk + (size_t)j * LD];
        part += x * x;
      }
      part = block_sum(part, sh_red);
      const double al = slab[rk + (size_t)(k + 1) * LD];
      double pi, br;
      larfg_scalars(al, part, pi, br);
      const double dr = al - br;
      __syncthreads();  // every thread has read alpha before it is overwritten by beta (racecheck WAR)
      if (tid == 0) {
        a.taup[k] = pi;
        a.e[k] = br;
        a.ug[k] = pi;  // pi travels with u
        slab[rk + (size_t)(k + 1) * LD] = br;
      }
      for (int j = k + 2 + tid; j < n; j += blockDim.x) {
        double* p = slab + rk + (size_t)j * LD;
        if (pi != 0.0) *p /= dr;
        a.ug[j] = *p;
      }
      if (tid == 0) a.ug[k + 1] = 1.0;
    }
    mk(k, 9);
    cl.sync();  // #4
    mk(k, 10);
    for (int j = k + tid; j < n; j += blockDim.x) vec[j] = __ldcg(a.ug + j);  // pi, then u
    __syncthreads();
    const double pi = vec[k];
    if (pi != 0.0) {
      // x_r = sum_{j>k} a[r, j] u_j for own rows r > k (warp per row), then a -= pi x u^T
      const int lo = max(0, k + 1 - r0);
      for (int rr = lo + warp; rr < nr; rr += nw) {
        double s = 0.0;
        for (int j = k + 1 + lane; j < n; j += 32) s += slab[rr + (size_t)j * LD] * vec[j];
        s = warp_sum(s);
        if (lane == 0) xr[rr] = s;
      }
      __syncthreads();
      const int rr = lo + (tid & (RP - 1));
      if (rr < nr) {
        const double xv = xr[rr];
        for (int j = k + 1 + (tid >> rs); j < n; j += (kG2cThreads >> rs))
          slab[rr + (size_t)j * LD] -= pi * (xv * vec[j]);
      }
    }
    __syncthreads();
    mk(k, 11);
  }
  if (rank == 0 && tid == 0) a.taup[n - 1] = 0.0;
  for (int idx = tid; idx < nr * n; idx += blockDim.x) {
    const int rr = idx % nr, j = idx / nr;
    a.A[(r0 + rr) + (long long)j * a.lda] = slab[rr + (size_t)j * LD];
  }
  cl.sync();  // no CTA exits while its shared memory may still be read
}

static size_t gebd2c_bytes(int m, int n, int cs, int* R, int* LD) {
  const int r = (m + cs - 1) / cs, ld = r | 1;  // odd stride: conflict-free column walks
  if (R) *R = r;
  if (LD) *LD = ld;
  return sizeof(double) * ((size_t)ld * n + 4 * (size_t)n + ld);
}

// cluster size for gebd2_cluster_kernel: 16 when the GPU can co-schedule it, else 8
static int gebd2c_cluster_size() {
  if (g_gebd2_cluster == 8) return 8;  // debug: force the portable cluster size
  // per-device probe, cached; thread-safe (batched SVDs call this from several host threads)
  static std::mutex mu;
  static int per_dev[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (per_dev[dev]) return per_dev[dev];
  per_dev[dev] = [] {
    func_attr(gebd2_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kG2cSmemMax);
    func_attr(gebd2_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(kG2cThreads); cfg.dynamicSmemBytes = kG2cSmemMax;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nclusters = 0;
    const bool ok16 = cudaOccupancyMaxActiveClusters(&nclusters, gebd2_cluster_kernel, &cfg) == cudaSuccess &&
                      nclusters >= 1;
    cudaGetLastError();
    return ok16 ? 16 : 8;
  }();
  return per_dev[dev];
}

// Measured per-column crossover with the two-phase LABRD panels (tools/gebd2_cluster_ab.py):
// the cluster kernel's work per CTA grows with n^2/16 while the panel path is
// latency-flat at ~11.5 us per column, so it takes over at n <= 512.
int g_g2c_max_cols = 512;  // debug / tuning: largest trailing block handed to the cluster GEBD2

static bool gebd2c_fits(int m, int n) {
  if (!g_gebd2_cluster || n < 64 || n > g_g2c_max_cols) return false;
  return gebd2c_bytes(m, n, gebd2c_cluster_size(), nullptr, nullptr) <= (size_t)kG2cSmemMax;
}

static int gebd2c_launch(cudaStream_t st, double* A, long long lda, int m, int n, double* d, double* e,
                         double* tauq, double* taup, double* ug) {
  const int cs = gebd2c_cluster_size();
  Gebd2cArgs ga;
  ga.A = A; ga.lda = lda; ga.m = m; ga.n = n; ga.d = d; ga.e = e; ga.tauq = tauq; ga.taup = taup;
  ga.ug = ug;
  ga.tlog = g_labrd_tlog;
  g_labrd_tlog = nullptr;
  const size_t smem = gebd2c_bytes(m, n, cs, &ga.R, &ga.LD);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cs); cfg.blockDim = dim3(kG2cThreads); cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cfg.attrs = at; cfg.numAttrs = 1;
  DC_CUDA_TRY(cudaLaunchKernelEx(&cfg, gebd2_cluster_kernel, ga));
  note_launch();
  return 0;
}

// ---------------------------------------------------------------------------
constexpr int kLabrdSmemMax = 225 * 1024;  // 227 KB opt-in minus static shared memory

template <typename K>
static int launch_coop(K kern, cudaStream_t st, LabrdArgs& la, int grid, size_t smem) {
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kLabrdSmemMax));
  void* args[] = {&la};
  DC_CUDA_TRY(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(kLabrdThreads), args, smem, st));
  note_launch();
  return 0;
}

static int launch_labrd(cudaStream_t st, LabrdArgs& la, int grid, size_t smem, bool two_phase, int rpl) {
  if (two_phase) {
    switch (rpl) {
      case 2: return launch_coop(labrd2_kernel<2>, st, la, grid, smem);
      case 4: return launch_coop(labrd2_kernel<4>, st, la, grid, smem);
      case 8: return launch_coop(labrd2_kernel<8>, st, la, grid, smem);
      default: return launch_coop(labrd2_kernel<16>, st, la, grid, smem);
    }
  }
  switch (rpl) {
    case 2: return la.l2keep > 0.0 ? launch_coop(labrd4_kernel<2, true>, st, la, grid, smem)
                                   : launch_coop(labrd4_kernel<2, false>, st, la, grid, smem);
    case 4: return la.l2keep > 0.0 ? launch_coop(labrd4_kernel<4, true>, st, la, grid, smem)
                                   : launch_coop(labrd4_kernel<4, false>, st, la, grid, smem);
    case 8: return la.l2keep > 0.0 ? launch_coop(labrd4_kernel<8, true>, st, la, grid, smem)
                                   : launch_coop(labrd4_kernel<8, false>, st, la, grid, smem);
    default: return la.l2keep > 0.0 ? launch_coop(labrd4_kernel<16, true>, st, la, grid, smem)
                                    : launch_coop(labrd4_kernel<16, false>, st, la, grid, smem);
  }
}

struct LabrdWork {
  double *cvec, *rvec, *normc, *normr, *py, *px, *pw, *ps;
  long long mp, np;
};

static size_t labrd_work_bytes(long long mp, long long np, int G) {
  return pool_bytes(mp, 8) + pool_bytes(np, 8) + 2 * pool_bytes(G, 8) + pool_bytes((size_t)G * np, 8) +
         pool_bytes((size_t)G * mp, 8) + 2 * pool_bytes((size_t)G * 64, 8);
}

static LabrdWork labrd_work_take(dcsvd_ctx* h, int pool, long long mp, long long np, int G) {
  LabrdWork w;
  w.cvec = pool_take<double>(h, pool, mp);
  w.rvec = pool_take<double>(h, pool, np);
  w.normc = pool_take<double>(h, pool, G);
  w.normr = pool_take<double>(h, pool, G);
  w.py = pool_take<double>(h, pool, (size_t)G * np);
  w.px = pool_take<double>(h, pool, (size_t)G * mp);
  w.pw = pool_take<double>(h, pool, (size_t)G * 64);
  w.ps = pool_take<double>(h, pool, (size_t)G * 64);
  w.mp = mp;
  w.np = np;
  return w;
}

// Does the two-phase kernel's P/Q block cache fit for an mv x nv view with panel width nb?
static bool labrd2_fits(int mv, int nv, int nb, int G) {
  for (int cand : {2, 4, 8, 16}) {
    const int RB = 32 * cand;
    const int Gr = (mv + RB - 1) / RB;
    int Gc = std::max(1, G / std::max(Gr, 1));
    const int CB = (nv + Gc - 1) / Gc;
    if (Gr > G || CB > 4 * kLabrdThreads) continue;
    const size_t CBp = (CB + 1) & ~1, NC = (2 * nb + 3) & ~3;
    const size_t bytes = sizeof(double) * (3 * RB + 3 * CBp + (size_t)kLabrdWarps * RB + (RB + CBp + 2) * NC);
    if (bytes <= (size_t)kLabrdSmemMax) return true;
  }
  return false;
}

// Panel width for the view: half-width panels where that lets the two-phase
// kernel (2 grid barriers per column) replace the four-phase one (4 barriers).
int g_labrd_halfwidth = 1;  // debug: 0 = always the requested width
long long g_labrd_halfwidth_max = 1LL << 62;  // debug: largest view (elements) given half-width panels
static int labrd_panel_width(int mv, int nv, int nb, int G) {
  if (!g_labrd_halfwidth || nb < 32 || labrd2_fits(mv, nv, nb, G)) return nb;
  if ((long long)mv * nv > g_labrd_halfwidth_max) return nb;
  if (labrd2_fits(mv, nv, nb / 2, G)) return nb / 2;
  if (g_labrd_halfwidth >= 2 && labrd2_fits(mv, nv, nb / 4, G)) return nb / 4;  // debug: quarter width
  return nb;
}

// One LABRD panel on the mv x nv view Av (bidiag.py:113-165): P (mv x 2nb,
// ldp) and Q (nv x 2nb, ldq) are zeroed here and filled; only the panel
// rows/columns of Av change.
int g_labrd_gmax = 0;  // debug: cap on the LABRD grid (0 = all SMs)
int g_labrd_skip_zero = 1;  // debug: 0 = zero P / Q before every GEBRD panel as well
int g_labrd4_rpl = 0;  // debug: rows per lane of the four-phase kernel (0 = square-block heuristic)
int g_labrd2_rpl = 0;  // debug: rows per lane of the two-phase kernel (0 = the fitting one with most CTAs)
// bytes of each large-panel GEMV pass kept in L2 with evict_last, the rest evict_first
// (tools/labrd_l2keep_ab.py at 8192^2: GEBRD 539 -> 532 ms for 16-24 MB; 64+ MB is slower)
double g_labrd_l2keep = 20.0 * (1 << 20);
double g_labrd_l2keep_min = 160.0 * (1 << 20);  // panels whose matrix is smaller use plain loads (n' < ~4600)

static int labrd_launch(dcsvd_ctx* h, cudaStream_t st, int mv, int nv, double* Av, long long lda, int nb, double* d,
                        double* e, double* tauq, double* taup, double* P, long long ldp, double* Q, long long ldq,
                        const LabrdWork& w, bool zero_pq = true) {
  const int G = g_labrd_gmax > 0 ? std::min(h->sms, g_labrd_gmax) : h->sms;
  // The kernels and the trailing GEMM only read P / Q entries written earlier in
  // the same panel (rows >= the column's pivot); the zero fill is for callers
  // that read whole P / Q (labrd_panel returns them as the reference does).
  if (zero_pq || !g_labrd_skip_zero) {
    DC_CUDA_TRY(cudaMemset2DAsync(P, sizeof(double) * ldp, 0, sizeof(double) * mv, 2 * nb, st));
    DC_CUDA_TRY(cudaMemset2DAsync(Q, sizeof(double) * ldq, 0, sizeof(double) * nv, 2 * nb, st));
  }
  DC_CUDA_TRY(cudaMemsetAsync(h->d_bar, 0, sizeof(unsigned), st));
  LabrdArgs la;
  la.A = Av; la.lda = lda; la.m = mv; la.n = nv; la.nb = nb;
  la.P = P; la.Q = Q; la.ldp = ldp; la.ldq = ldq;
  la.d = d; la.e = e; la.tauq = tauq; la.taup = taup;
  la.cvec = w.cvec; la.rvec = w.rvec; la.normc = w.normc; la.normr = w.normr;
  la.py = w.py; la.px = w.px; la.pw = w.pw; la.ps = w.ps; la.ldpy = w.np; la.ldpx = w.mp;
  la.bar = h->d_bar;
  la.tlog = g_labrd_tlog;
  g_labrd_tlog = nullptr;  // log one launch only
  // only where the panel's matrix is several times the L2: at 3072^2-4096^2 the
  // hinted loads are slower than plain ones (tools/labrd_l2keep_ab.py)
  la.l2keep = 8.0 * (double)mv * (double)nv > g_labrd_l2keep_min ? g_labrd_l2keep : 0.0;
  // 2-D geometry for rows-per-lane rpl: Gr x Gc <= G blocks of RB x CB
  auto geom = [&](int rpl, int& Gr, int& Gc, int& CB) {
    const int RB = 32 * rpl;
    Gr = (mv + RB - 1) / RB;
    Gc = std::max(1, G / std::max(Gr, 1));
    CB = (nv + Gc - 1) / Gc;
    Gc = (nv + CB - 1) / CB;
  };
  // Two-phase kernel when its P/Q block caches fit in shared memory (small
  // panels, latency-bound: two barriers per column); otherwise the four-phase
  // kernel with 1-D slices (large panels, HBM-bound).
  bool two_phase = false;
  int rpl = 16;
  size_t smem = 0;
  for (int cand : {2, 4, 8, 16}) {
    if (g_labrd2_rpl && cand != g_labrd2_rpl) continue;  // debug: force one geometry
    int Gr, Gc, CB;
    geom(cand, Gr, Gc, CB);
    if (Gr > G || CB > 4 * kLabrdThreads) continue;
    const size_t RB = 32 * cand, CBp = (CB + 1) & ~1, NC = (2 * nb + 3) & ~3;
    const size_t bytes = sizeof(double) * (3 * RB + 3 * CBp + (size_t)kLabrdWarps * RB + (RB + CBp + 2) * NC);
    // 4 rows per lane when it fits (measured best from 768^2 to 3072^2,
    // tools/labrd2_rpl_sweep.py), else the geometry with the most CTAs
    const bool better = !two_phase || (rpl != 4 && (cand == 4 || Gr * Gc > la.Gr * la.Gc));
    if (bytes <= (size_t)kLabrdSmemMax && better) {
      two_phase = true;
      rpl = cand;
      smem = bytes;
      la.Gr = Gr; la.Gc = Gc; la.RB = (int)RB; la.CB = CB; la.CBp = (int)CBp;
    }
  }
  if (!two_phase) {
    const double target_rows = mv / sqrt((double)G * mv / nv);
    rpl = 16;
    if (target_rows <= 32 * 2) rpl = 2;
    else if (target_rows <= 32 * 4) rpl = 4;
    else if (target_rows <= 32 * 8) rpl = 8;
    if (g_labrd4_rpl) rpl = g_labrd4_rpl;  // debug: force the four-phase geometry
    int Gr, Gc, CB;
    geom(rpl, Gr, Gc, CB);
    if (Gr > G) return set_error(h, DCSVD_EINVAL, "matrix too tall for the GPU LABRD panel (%d rows)", mv);
    la.Gr = Gr; la.Gc = Gc; la.RB = 32 * rpl; la.CB = CB; la.CBp = (CB + 1) & ~1;
    const int grid = Gr * Gc;
    la.R1 = (mv + grid - 1) / grid;
    la.C1 = (nv + grid - 1) / grid;
    if (la.R1 > kLabrdThreads || la.C1 > kLabrdThreads)
      return set_error(h, DCSVD_EINVAL, "matrix too large for one LABRD grid (%dx%d)", mv, nv);
    smem = sizeof(double) * (((CB + 1) & ~1) + (size_t)kLabrdWarps * la.RB + (size_t)(la.R1 + la.C1) * 2 * nb);
    la.cache_pq = 1;
    if (smem > 200 * 1024) {
      la.cache_pq = 0;
      smem = sizeof(double) * (((CB + 1) & ~1) + (size_t)kLabrdWarps * la.RB);
    }
    if (smem > 200 * 1024 || CB > 4 * kLabrdThreads)
      return set_error(h, DCSVD_EINVAL, "LABRD block too wide (%d columns)", CB);
  }
  const int grid = la.Gr * la.Gc;
  g_labrd_last_two_phase = two_phase;
  // algorithmic bytes of the two big GEMVs per column:
  // 8 * sum_k [(mv-k)(nv-k-1) + (mv-k-1)(nv-k-1)]
  double bytes = 0.0;
  for (int k = 0; k < nb; ++k) bytes += 8.0 * ((double)(mv - k) * (nv - k - 1) + (double)(mv - k - 1) * (nv - k - 1));
  const int sidx = stat_begin(h, 0, bytes, st);
  const int rc = launch_labrd(st, la, grid, smem, two_phase, rpl);
  stat_end(h, sidx, st);
  return rc;
}

int labrd_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda, int nb, double* d,
              double* e, double* tauq, double* taup, double* P, long long ldp, double* Q, long long ldq) {
  if (!(1 <= nb && nb < n && n <= m))
    return set_error(h, DCSVD_EINVAL, "panel width %d needs block < ncols <= nrows, view is %lldx%lld", nb, m, n);
  if (nb > 32) return set_error(h, DCSVD_EINVAL, "GPU LABRD supports block width <= 32, got %d", nb);
  int rc = pool_reserve(h, 0, labrd_work_bytes(m, n, h->sms), st);
  if (rc) return rc;
  LabrdWork w = labrd_work_take(h, 0, m, n, h->sms);
  rc = labrd_launch(h, st, (int)m, (int)n, A, lda, nb, d, e, tauq, taup, P, ldp, Q, ldq, w);
  if (rc) return rc;
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int gebrd_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda,
              double* d, double* e, double* tauq, double* taup, int nb) {
  if (n < 1 || m < n) return set_error(h, DCSVD_EINVAL, "bidiagonalization requires m >= n >= 1, got %lldx%lld", m, n);
  if (nb < 1) return set_error(h, DCSVD_EINVAL, "block width must be >= 1, got %d", nb);
  // Wider panels than the GPU panel kernel takes give the same reflectors (the
  // panel width only regroups the trailing updates): run them as 32-wide panels.
  if (nb > 32 && nb < n) nb = 32;
  const bool unblocked = nb >= n;
  if (unblocked) nb = (int)std::min<long long>(n, 32);  // no panel runs: the whole matrix goes through GEBD2
  const int G = h->sms;
  const long long mp = m, np = n;
  size_t need = pool_bytes(mp * 2 * nb, 8) + pool_bytes(np * 2 * nb, 8) + labrd_work_bytes(mp, np, G) +
                pool_bytes(mp + np, 8);
  int rc = pool_reserve(h, 0, need, st);
  if (rc) return rc;
  double* P = pool_take<double>(h, 0, mp * 2 * nb);
  double* Q = pool_take<double>(h, 0, np * 2 * nb);
  LabrdWork w = labrd_work_take(h, 0, mp, np, G);
  double* wbuf = pool_take<double>(h, 0, mp + np);
  long long off = 0;
  while (n - off > nb && !unblocked && !gebd2c_fits((int)(m - off), (int)(n - off))) {
    const int mv = (int)(m - off), nv = (int)(n - off);
    double* Av = A + off + off * lda;
    const int nbp = labrd_panel_width(mv, nv, nb, G);  // same reflectors for any width
    // whole-GPU handles skip the P / Q zero fill; batch sub-contexts keep it
    // (measured: C5 12.13 -> 12.50 ms/SVD without it, tools/c5_lib_ab.py)
    rc = labrd_launch(h, st, mv, nv, Av, lda, nbp, d + off, e + off, tauq + off, taup + off, P, mp, Q, np, w,
                      /*zero_pq=*/h->is_sub);
    if (rc) return rc;
    // trailing update A[nb:, nb:] -= P[nb:, :] Q[nb:, :]^T  (bidiag.py:195-197)
    GemmDesc gd;
    gd.m = mv - nbp; gd.n = nv - nbp; gd.k = 2 * nbp;
    gd.A = P + nbp; gd.lda = mp; gd.acol = nullptr;
    gd.B = Q + nbp; gd.ldb = np;
    gd.C = Av + nbp + (long long)nbp * lda; gd.ldc = lda; gd.ccol = nullptr;
    gd.alpha = -1.0; gd.beta = 1.0;
    rc = gemm_launch(st, false, true, gd);
    if (rc) return rc;
    off += nbp;
  }
  if (gebd2c_fits((int)(m - off), (int)(n - off))) {
    rc = gebd2c_launch(st, A + off + off * lda, lda, (int)(m - off), (int)(n - off), d + off, e + off, tauq + off,
                       taup + off, wbuf);
    if (rc) return rc;
  } else {
    gebd2_kernel<<<1, kGebd2Threads, 0, st>>>(A + off + off * lda, lda, (int)(m - off), (int)(n - off), d + off,
                                              e + off, tauq + off, taup + off, wbuf);
    note_launch();
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace dc
