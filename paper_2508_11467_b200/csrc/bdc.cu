// Bidiagonal divide and conquer (BDSDC) on the GPU.
//
// Reference: pkg/src/dcsvd/bdc.py (leaf QR iteration :201-359, split
// :366-379, build_z :382-412, deflate :423-508, secular solver :541-641,
// recompute_z :644-673, secular_vectors :676-694, structured merge
// :701-747, _merge :768-847, bdsdc :861-880); arxiv 2508.11467 Alg. 3/4
// (PAPER.md:731-802).
//
// Layout (LAPACK dlasd0 style): a node covering rows
// [r0, r0+n) owns the diagonal block [r0, r0+n)^2 of the global left basis W
// and [r0, r0+ncols)^2 of the right basis Q; its children own disjoint
// sub-blocks, the removed row r0+nl sits between them.  Off-diagonal blocks
// stay exactly zero and W[r0+nl, r0+nl] = 1, so the merge's pre-sort column
// sets l_pre / r_pre (bdc.py:796-813) are *physical* columns of W / Q reached
// through an index map -- nothing is assembled or permuted in memory.
//
// The tree is processed level-synchronously by height: one launch per kernel
// family covers every merge of a level (CTA / warp per merge / root / row),
// sizes that depend on deflation are read from device memory, and the host
// never waits inside the tree.  Per level:
//   bdc_prep      z-vector, coupling, stable 2-way merge of the children's
//                 values, deflation scan, class-ordered column lists
//   bdc_rotate    deflation Givens rotations applied to W/Q rows in parallel
//   bdc_secular   warp-per-root frozen-lane secular solver
//   bdc_loewner   warp-per-root Loewner z recomputation
//   bdc_vectors   warp-per-column singular vectors of the middle matrix
//                 (+ the edge-row companion, kept in both modes)
//   bdc_order     stable value order of [omega, deflated] (binary-search ranks)
//   merge GEMMs   grouped DMMA GEMM, 4 structured products per merge, A
//                 columns gathered and C columns scattered into sorted order
//   bdc_defl_copy deflated columns + unit row + null column into scratch
//   bdc_copyback  scratch -> W/Q node blocks.
#include <algorithm>
#include <vector>

#include <cstring>
#include "ctx.cuh"
#include "gemm.cuh"
#include "launch.cuh"

namespace dc {

enum : int { kUnit = 0, kFirst = 1, kSecond = 2, kMixed = 3 };

struct LeafDesc {
  int r0, n, bordered;
};
struct MergeDesc {
  int r0, n, nl, nr, bordered;
};
struct MergeMeta {
  int K, nd, nrot;
  int nFw, nMw, nSw, nFq, nMq, nSq;
  int sorted_ok;
  double tol, zz;
  double cc, ss;           // bordered coupling rotation
  double null_e0, null_e1; // null column edge entries
};

// Per-entry scratch (indexed r0 + i, length ncols_root + 1).
struct BdcBufs {
  double *dpre, *zpre;            // pre-sort
  int* perm;                      // working -> pre-sort
  double *dw, *zw;                // working order
  int *lcls, *rcls;               // working order classes
  double *ew0, *ew1;              // working edge rows
  int* kept;                      // kept working indices (K)
  int *kcl, *kcr;                 // classes of kept entries
  double *ke0, *ke1;              // edge entries of kept columns (after rotations)
  int* defl;                      // deflated working indices (nd)
  double* dval;                   // deflated values
  int* dkind;                     // 1 = paired with the zero pole (value 0.0)
  int *rot_p, *rot_j;             // rotations (working indices)
  double *rot_c, *rot_s;
  double *ds, *zs;                // secular system (K)
  double *omega, *mu;
  int* anc;
  double* zt;
  int *wpos, *qpos;               // kept k -> class-ordered position
  int *wphys, *qphys;             // class-ordered position -> physical column
  double *ekn0, *ekn1;            // new edge entries of kept columns
  double* uunit;                  // umat unit row (K)
  int *kdst, *ddst;               // sorted destination of kept / deflated
  int* physcol;                   // working idx -> physical column
  int* kdstphys;                  // r0 + kdst[k]
};

__device__ __forceinline__ int phys_of(int r0, int nl, int pre) {
  return r0 + (pre == 0 ? nl : (pre <= nl ? pre - 1 : pre));
}

// ===========================================================================
// Leaves: one warp per leaf (<= 32 rows), bdc.py:315-359.
constexpr int kLeafWarps = 2;
constexpr int kLdW = 32, kLdQ = 33;

struct LeafSmem {
  double W[32 * kLdW];
  double Q[33 * kLdQ];
  double d[33], e[33];
  int order[33];
};

__device__ __forceinline__ void leaf_rot(double* M, int ld, int rows, int p, int q, double c, double s, int lane) {
  for (int r = lane; r < rows; r += 32) {
    const double mp = M[r + p * ld], mq = M[r + q * ld];
    M[r + p * ld] = c * mp + s * mq;
    M[r + q * ld] = c * mq - s * mp;
  }
}

__device__ __forceinline__ bool leaf_small(double x, double a, double b, double bnorm) {
  return fabs(x) <= DC_EPS * (fabs(a) + fabs(b)) || fabs(x) <= DC_EPS * bnorm * 1e-3;
}

// The scalar recurrence (d, e) lives in registers, lane k holding d[k] and
// e[k]; reads are warp broadcasts (__shfl_sync) and writes are predicated on
// the owning lane, so every lane follows the identical (warp-uniform) control
// flow without shared-memory hazards.  Rotations act on the lane's own rows
// of W / Q in shared memory.
__global__ void __launch_bounds__(32 * kLeafWarps) bdc_leaf_kernel(const LeafDesc* __restrict__ leaves, int nleaves,
                                                                   const double* __restrict__ din,
                                                                   const double* __restrict__ ein, double* W,
                                                                   long long ldw, double* Q, long long ldq,
                                                                   double* dv, double* edge, int vectors,
                                                                   int* err) {
  __shared__ LeafSmem sm_all[kLeafWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int li = blockIdx.x * kLeafWarps + warp;
  if (li >= nleaves) return;
  LeafSmem& S = sm_all[warp];
  const LeafDesc L = leaves[li];
  const int n = L.n, nc = L.n + L.bordered, r0 = L.r0;
  double* Ws = S.W;
  double* Qs = S.Q;
  constexpr unsigned FULL = 0xffffffffu;
  for (int c = 0; c < n; ++c)
    for (int r = lane; r < n; r += 32) Ws[r + c * kLdW] = (r == c) ? 1.0 : 0.0;
  for (int c = 0; c < nc; ++c)
    for (int r = lane; r < nc; r += 32) Qs[r + c * kLdQ] = (r == c) ? 1.0 : 0.0;
  double dr = lane < n ? din[r0 + lane] : 0.0;
  double er = lane < n ? ein[r0 + lane] : 0.0;
  auto D = [&](int k) { return __shfl_sync(FULL, dr, k); };
  auto E = [&](int k) { return __shfl_sync(FULL, er, k); };
  auto setD = [&](int k, double v) { if (lane == k) dr = v; };
  auto setE = [&](int k, double v) { if (lane == k) er = v; };
  if (n > 0) {
    if (L.bordered) {
      // chase the trailing column in (bdc.py:337-347)
      double f = E(n - 1);
      for (int i = n - 1; i >= 0; --i) {
        double c, s, r;
        lartg(D(i), f, c, s, r);
        setD(i, r);
        if (i > 0) {
          const double em = E(i - 1);
          f = -s * em;
          setE(i - 1, c * em);
        }
        __syncwarp();
        leaf_rot(Qs, kLdQ, nc, i, n, c, s, lane);
        if (s == 0.0) break;
      }
    }
    if (lane == n - 1) er = 0.0;  // square part: e[0..n-1)
    // implicit-shift QR iteration (bdc.py:273-312)
    double bnorm = 0.0;
    for (int i = 0; i < n; ++i) bnorm = fmax(bnorm, fabs(D(i)));
    for (int i = 0; i + 1 < n; ++i) bnorm = fmax(bnorm, fabs(E(i)));
    if (bnorm != 0.0) {
      const long long budget = 60LL * n * (n > 4 ? n : 4);
      long long steps = 0;
      int hi = n - 1;
      while (hi > 0) {
        if (leaf_small(E(hi - 1), D(hi - 1), D(hi), bnorm)) {
          setE(hi - 1, 0.0);
          --hi;
          continue;
        }
        int lo = hi - 1;
        while (lo > 0 && !leaf_small(E(lo - 1), D(lo - 1), D(lo), bnorm)) --lo;
        if (lo > 0) setE(lo - 1, 0.0);
        int hit = -1;
        for (int k = lo; k <= hi; ++k)
          if (fabs(D(k)) <= DC_EPS * bnorm * 1e-3) { hit = k; break; }
        if (hit >= 0) {
          setD(hit, 0.0);
          if (hit < hi) {
            // chase zero row (bdc.py:247-257)
            double f = E(hit);
            setE(hit, 0.0);
            for (int j = hit + 1; j <= hi; ++j) {
              double c, s, r;
              lartg(D(j), f, c, s, r);
              setD(j, r);
              if (j < hi) {
                const double ej = E(j);
                f = -s * ej;
                setE(j, c * ej);
              }
              __syncwarp();
              leaf_rot(Ws, kLdW, n, j, hit, c, s, lane);
            }
          } else {
            // chase zero column (bdc.py:260-270)
            double f = E(hi - 1);
            setE(hi - 1, 0.0);
            for (int j = hi - 1; j >= lo; --j) {
              double c, s, r;
              lartg(D(j), f, c, s, r);
              setD(j, r);
              if (j > lo) {
                const double ej = E(j - 1);
                f = -s * ej;
                setE(j - 1, c * ej);
              }
              __syncwarp();
              leaf_rot(Qs, kLdQ, nc, j, hi, c, s, lane);
            }
          }
          continue;
        }
        // one bulge chase (bdc.py:218-244)
        double mu;
        {
          const double ep = (hi - 2 >= lo) ? E(hi - 2) : 0.0;
          const double dh1 = D(hi - 1), eh1 = E(hi - 1), dh = D(hi);
          const double t11 = dh1 * dh1 + ep * ep;
          const double t12 = dh1 * eh1;
          const double t22 = dh * dh + eh1 * eh1;
          const double delta = 0.5 * (t11 - t22);
          const double den = delta + copysign(hypot(delta, t12), delta != 0.0 ? delta : 1.0);
          mu = den == 0.0 ? t22 : t22 - t12 * t12 / den;
        }
        const double dlo = D(lo);
        double f = dlo * dlo - mu;
        double g = dlo * E(lo);
        for (int k = lo; k < hi; ++k) {
          double c, s, r;
          lartg(f, g, c, s, r);
          const double dk = D(k), ek = E(k), dk1 = D(k + 1);
          if (k > lo) setE(k - 1, r);
          f = c * dk + s * ek;
          const double ekn = c * ek - s * dk;
          g = s * dk1;
          const double dk1n = c * dk1;
          setE(k, ekn);
          __syncwarp();
          leaf_rot(Qs, kLdQ, nc, k, k + 1, c, s, lane);
          lartg(f, g, c, s, r);
          const double ekp1 = (k < hi - 1) ? E(k + 1) : 0.0;
          setD(k, r);
          f = c * ekn + s * dk1n;
          setD(k + 1, c * dk1n - s * ekn);
          if (k < hi - 1) {
            g = s * ekp1;
            setE(k + 1, c * ekp1);
          }
          __syncwarp();
          leaf_rot(Ws, kLdW, n, k, k + 1, c, s, lane);
        }
        setE(hi - 1, f);
        steps += hi - lo;
        if (steps > budget) {
          if (lane == 0) raise_dev(err, kDevNoConvergeQR);
          break;
        }
      }
    }
    // sign fix into W (bdc.py:349-353)
    for (int i = 0; i < n; ++i) {
      if (D(i) < 0.0) {
        for (int r = lane; r < n; r += 32) Ws[r + i * kLdW] = -Ws[r + i * kLdW];
      }
    }
    if (lane < n && dr < 0.0) dr = -dr;
    // stable ascending order: rank of each value
    {
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const double dj = D(j);
        rank += (dj < dr) || (dj == dr && j < lane);
      }
      if (lane < n) S.order[rank] = lane;
    }
    __syncwarp();
  }
  // outputs (sorted columns)
  for (int c = 0; c < n; ++c) {
    const int src = S.order[c];
    const double val = D(src);
    if (lane == 0) dv[r0 + c] = val;
    if (vectors) {
      for (int r = lane; r < n; r += 32) W[(r0 + r) + (long long)(r0 + c) * ldw] = Ws[r + src * kLdW];
      for (int r = lane; r < nc; r += 32) Q[(r0 + r) + (long long)(r0 + c) * ldq] = Qs[r + src * kLdQ];
    }
    if (lane == 0) {
      edge[2LL * (r0 + c) + 0] = Qs[0 + src * kLdQ];
      edge[2LL * (r0 + c) + 1] = Qs[(nc - 1) + src * kLdQ];
    }
  }
  if (L.bordered) {
    if (vectors)
      for (int r = lane; r < nc; r += 32) Q[(r0 + r) + (long long)(r0 + n) * ldq] = Qs[r + n * kLdQ];
    if (lane == 0) {
      edge[2LL * (r0 + n) + 0] = Qs[0 + n * kLdQ];
      edge[2LL * (r0 + n) + 1] = Qs[(nc - 1) + n * kLdQ];
    }
  }
}

// ===========================================================================
// Merge preparation: one CTA per merge.
constexpr int kPrepThreads = 512;
constexpr int kPrepChunk = 1024;

__device__ __forceinline__ int ub_count_le(const double* a, int n, double x) {
  // number of a[i] <= x, a ascending
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int lb_count_lt(const double* a, int n, double x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ double block_max(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = lane < nw ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kPrepThreads) bdc_prep_kernel(const MergeDesc* __restrict__ merges,
                                                                MergeMeta* __restrict__ meta,
                                                                const double* __restrict__ din,
                                                                const double* __restrict__ ein, const double* dv,
                                                                const double* edge, double* Q, long long ldq,
                                                                int vectors, double tol_mult, BdcBufs B, int* err) {
  __shared__ double sh_red[32];
  __shared__ int sh_has[kPrepThreads];
  __shared__ double sh_lastd[kPrepThreads];
  __shared__ int sh_cnt[kPrepThreads][6];
  __shared__ int sh_tot[8];
  const MergeDesc M = merges[blockIdx.x];
  MergeMeta& mt = meta[blockIdx.x];
  const int tid = threadIdx.x;
  const int r0 = M.r0, n = M.n, nl = M.nl, nr = M.nr, gam = M.bordered;
  const int ncols = n + gam;
  const double alpha = din[r0 + nl];
  const double beta = ein[r0 + nl];
  // child edge rows: left at columns [r0, r0+nl+1), right at [r0+nl+1, r0+ncols)
  const double* eL = edge + 2LL * r0;              // eL[2*c + row]
  const double* eR = edge + 2LL * (r0 + nl + 1);
  const double lam1 = eL[2 * nl + 1];
  const double f1n = eL[2 * nl + 0];
  double cc = 1.0, ss = 0.0, z0;
  double phi2 = 0.0, l2n = 0.0;
  if (gam) {
    phi2 = eR[2 * nr + 0];
    l2n = eR[2 * nr + 1];
    double r;
    lartg(alpha * lam1, beta * phi2, cc, ss, r);
    z0 = r;
  } else {
    z0 = alpha * lam1;
  }
  // pre-sort arrays (bdc.py:382-412, :777-795)
  double* dpre = B.dpre + r0;
  double* zpre = B.zpre + r0;
  for (int i = tid; i < n; i += blockDim.x) {
    double dd, zz, e0, e1;
    if (i == 0) {
      dd = 0.0;
      zz = z0;
      e0 = gam ? cc * f1n : f1n;
      e1 = gam ? ss * l2n : 0.0;
    } else if (i <= nl) {
      dd = dv[r0 + i - 1];
      zz = alpha * eL[2 * (i - 1) + 1];
      e0 = eL[2 * (i - 1) + 0];
      e1 = 0.0;
    } else {
      const int b = i - 1 - nl;
      dd = dv[r0 + nl + 1 + b];
      zz = beta * eR[2 * b + 0];
      e0 = 0.0;
      e1 = eR[2 * b + 1];
    }
    dpre[i] = dd;
    zpre[i] = zz;
    // stash pre-sort edge entries in the working edge arrays at the PRE index;
    // they are permuted below
    B.ke0[r0 + i] = e0;
    B.ke1[r0 + i] = e1;
  }
  if (tid == 0) {
    mt.cc = cc;
    mt.ss = ss;
    mt.null_e0 = -ss * f1n;
    mt.null_e1 = cc * l2n;
  }
  // bordered coupling rotation on the physical Q columns (r0+nl, r0+ncols-1)
  if (vectors && gam) {
    double* qa = Q + (long long)(r0 + nl) * ldq;
    double* qb = Q + (long long)(r0 + ncols - 1) * ldq;
    for (int r = r0 + tid; r < r0 + ncols; r += blockDim.x) {
      const double a = qa[r], b = qb[r];
      qa[r] = cc * a + ss * b;
      qb[r] = cc * b - ss * a;
    }
  }
  __syncthreads();
  // stable merge of [0] + D1 (ascending) and D2 (ascending)
  const double* D1 = dpre + 1;
  const double* D2 = dpre + 1 + nl;
  int* perm = B.perm + r0;
  for (int i = tid; i < n; i += blockDim.x) {
    int rank;
    if (i == 0) rank = 0;
    else if (i <= nl) rank = 1 + (i - 1) + lb_count_lt(D2, nr, D1[i - 1]);
    else rank = 1 + (i - 1 - nl) + ub_count_le(D1, nl, D2[i - 1 - nl]);
    perm[rank] = i;
  }
  __syncthreads();
  double lmax = 0.0;
  for (int j = tid; j < n; j += blockDim.x) {
    const int p = perm[j];
    const double dd = dpre[p], zz = zpre[p];
    B.dw[r0 + j] = dd;
    B.zw[r0 + j] = zz;
    B.ew0[r0 + j] = B.ke0[r0 + p];
    B.ew1[r0 + j] = B.ke1[r0 + p];
    B.lcls[r0 + j] = p == 0 ? kUnit : (p <= nl ? kFirst : kSecond);
    B.rcls[r0 + j] = p == 0 ? (gam ? kMixed : kFirst) : (p <= nl ? kFirst : kSecond);
    B.physcol[r0 + j] = phys_of(r0, nl, p);
    lmax = fmax(lmax, fmax(fabs(dd), fabs(zz)));
  }
  const double tol = tol_mult * DC_EPS * block_max(lmax, sh_red);
  // deflation (bdc.py:460-498) by groups.  In the sequential scan a non-tiny
  // entry j merges into the last kept entry p iff d_j - d_p <= tol, where d_p
  // is the previous survivor's d (it is copied into p on every merge) except
  // for p = 0, whose d stays 0.  So on the sorted survivors: the ones with
  // d <= tol join entry 0's group, any other starts a new group iff it lies
  // more than tol above the previous survivor.  Entries are classified in
  // parallel, and one thread walks each group in order (the Givens chain of
  // a group is sequential; groups are independent), writing outputs at
  // indices from block-wide prefix counts -- the same results, in the same
  // order, as the sequential scan.
  int* ecls = perm;  // reuse per entry: 0 tiny z (deflated), 1 leader (kept), 2 merged into its leader
  const int T = blockDim.x;
  const int CH = (n + T - 1) / T;
  const int c0 = min(n, tid * CH), c1 = min(n, c0 + CH);
  {
    int has = 0;
    double lastd = 0.0;
    for (int j = c0; j < c1; ++j)
      if (j == 0 || !(fabs(B.zw[r0 + j]) <= tol)) {
        has = 1;
        lastd = B.dw[r0 + j];
      }
    sh_has[tid] = has;
    sh_lastd[tid] = lastd;
  }
  __syncthreads();
  {
    double prevd = 0.0;  // d of the last survivor before c0 (entry 0 always survives)
    for (int u = tid - 1; u >= 0; --u)
      if (sh_has[u]) {
        prevd = sh_lastd[u];
        break;
      }
    int cnt_t = 0, cnt_l = 0, cnt_m = 0;
    for (int j = c0; j < c1; ++j) {
      int cls;
      if (j == 0) {
        cls = 1;
        prevd = 0.0;
      } else {
        const double dj = B.dw[r0 + j];
        if (fabs(B.zw[r0 + j]) <= tol) {
          cls = 0;
        } else {
          cls = (prevd <= tol ? dj > tol : dj - prevd > tol) ? 1 : 2;
          prevd = dj;
        }
      }
      ecls[j] = cls;
      cnt_t += cls == 0;
      cnt_l += cls == 1;
      cnt_m += cls == 2;
    }
    sh_cnt[tid][0] = cnt_t + cnt_m;  // deflated
    sh_cnt[tid][1] = cnt_l;          // kept
    sh_cnt[tid][2] = cnt_m;          // rotations
  }
  __syncthreads();
  if (tid < 3) {  // exclusive prefix over the chunks
    int run = 0;
    for (int t = 0; t < T; ++t) {
      const int v = sh_cnt[t][tid];
      sh_cnt[t][tid] = run;
      run += v;
    }
    sh_tot[tid] = run;
  }
  __syncthreads();
  {
    int dix = sh_cnt[tid][0], kix = sh_cnt[tid][1], rix = sh_cnt[tid][2];
    for (int j = c0; j < c1; ++j) {
      const int cls = ecls[j];
      if (cls == 0) {  // tiny z: deflated with its own value, edge entries unchanged
        B.defl[r0 + dix] = j;
        B.dval[r0 + dix] = B.dw[r0 + j];
        B.dkind[r0 + dix] = 0;
        ++dix;
        continue;
      }
      if (cls == 2) {  // written by its group's walker
        ++dix;
        ++rix;
        continue;
      }
      // leader: walk the group (up to the next leader) in scan order
      double pd = B.dw[r0 + j], pz = B.zw[r0 + j], pe0 = B.ew0[r0 + j], pe1 = B.ew1[r0 + j];
      int pcl = B.lcls[r0 + j], pcr = B.rcls[r0 + j];
      if (j == 0 && fabs(pz) <= tol) pz = copysign(fmax(tol, DC_TINY), pz != 0.0 ? pz : 1.0);  // z0 clamp
      int wd = dix, wr = rix;
      for (int jb = j + 1; jb < n; jb += 8) {
        int ec[8];
        double zq[8], dq[8], e0q[8], e1q[8];
        int lcq[8], rcq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // loads first: eight entries in flight
          const int jj = jb + q;
          ec[q] = jj < n ? ecls[jj] : 1;
          zq[q] = jj < n ? B.zw[r0 + jj] : 0.0;
          dq[q] = jj < n ? B.dw[r0 + jj] : 0.0;
          e0q[q] = jj < n ? B.ew0[r0 + jj] : 0.0;
          e1q[q] = jj < n ? B.ew1[r0 + jj] : 0.0;
          lcq[q] = jj < n ? B.lcls[r0 + jj] : 0;
          rcq[q] = jj < n ? B.rcls[r0 + jj] : 0;
        }
        bool stop = false;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (stop) break;
          const int jj = jb + q;
          if (ec[q] == 1) {  // next leader (or the end)
            stop = true;
            break;
          }
          if (ec[q] == 0) {  // tiny entry inside the group: counted, written by its owner
            ++wd;
            continue;
          }
          double c, sn, r;
          lartg(pz, zq[q], c, sn, r);
          pz = r;
          B.rot_p[r0 + wr] = j;
          B.rot_j[r0 + wr] = jj;
          B.rot_c[r0 + wr] = c;
          B.rot_s[r0 + wr] = sn;
          ++wr;
          const double a0 = pe0, b0 = e0q[q], a1 = pe1, b1 = e1q[q];
          pe0 = c * a0 + sn * b0;
          pe1 = c * a1 + sn * b1;
          B.ew0[r0 + jj] = c * b0 - sn * a0;
          B.ew1[r0 + jj] = c * b1 - sn * a1;
          pcr = (pcr == rcq[q]) ? pcr : kMixed;
          B.defl[r0 + wd] = jj;
          if (j == 0) {  // pairs with the zero pole: right side only, value 0
            B.dval[r0 + wd] = 0.0;
            B.dkind[r0 + wd] = 1;
          } else {
            pd = dq[q];
            pcl = (pcl == lcq[q]) ? pcl : kMixed;
            B.dval[r0 + wd] = dq[q];
            B.dkind[r0 + wd] = 0;
          }
          ++wd;
        }
        if (stop) break;
      }
      B.kept[r0 + kix] = j;
      B.ds[r0 + kix] = pd;
      B.zs[r0 + kix] = pz;
      B.kcl[r0 + kix] = pcl;
      B.kcr[r0 + kix] = pcr;
      B.ke0[r0 + kix] = pe0;
      B.ke1[r0 + kix] = pe1;
      ++kix;
    }
  }
  __syncthreads();
  const int K = sh_tot[1], nd = sh_tot[0], nrot = sh_tot[2];
  // class-ordered positions: W side [F, M, S] over kept k >= 1; Q side [F, M, S]
  {
    const int per = (K + blockDim.x - 1) / blockDim.x;
    const int k0 = tid * per, k1 = min(K, k0 + per);
    int cnt[6] = {0, 0, 0, 0, 0, 0};
    for (int k = k0; k < k1; ++k) {
      const int cl = B.kcl[r0 + k], cr = B.kcr[r0 + k];
      if (k >= 1) cnt[cl == kFirst ? 0 : (cl == kMixed ? 1 : 2)]++;
      cnt[3 + (cr == kFirst ? 0 : (cr == kMixed ? 1 : 2))]++;
    }
    for (int q = 0; q < 6; ++q) sh_cnt[tid][q] = cnt[q];
    __syncthreads();
    if (tid < 6) {
      int run = 0;
      for (int t = 0; t < (int)blockDim.x; ++t) {
        const int v = sh_cnt[t][tid];
        sh_cnt[t][tid] = run;
        run += v;
      }
      sh_tot[tid] = run;  // totals per class
    }
    __syncthreads();
    const int offw[3] = {0, sh_tot[0], sh_tot[0] + sh_tot[1]};
    const int offq[3] = {0, sh_tot[3], sh_tot[3] + sh_tot[4]};
    int run[6];
    for (int q = 0; q < 6; ++q) run[q] = sh_cnt[tid][q];
    for (int k = k0; k < k1; ++k) {
      const int cl = B.kcl[r0 + k], cr = B.kcr[r0 + k];
      const int pj = B.physcol[r0 + B.kept[r0 + k]];
      if (k >= 1) {
        const int c = cl == kFirst ? 0 : (cl == kMixed ? 1 : 2);
        const int pos = offw[c] + run[c]++;
        B.wpos[r0 + k] = pos;
        B.wphys[r0 + pos] = pj;
      } else {
        B.wpos[r0 + k] = -1;
      }
      const int c = cr == kFirst ? 0 : (cr == kMixed ? 1 : 2);
      const int pos = offq[c] + run[3 + c]++;
      B.qpos[r0 + k] = pos;
      B.qphys[r0 + pos] = pj;
    }
    __syncthreads();
  }
  // ||z||^2 of the system
  double zz = 0.0;
  for (int k = tid; k < K; k += blockDim.x) zz += B.zs[r0 + k] * B.zs[r0 + k];
  zz = block_sum(zz, sh_red);
  if (tid == 0) {
    mt.K = K;
    mt.nd = nd;
    mt.nrot = nrot;
    mt.nFw = sh_tot[0]; mt.nMw = sh_tot[1]; mt.nSw = sh_tot[2];
    mt.nFq = sh_tot[3]; mt.nMq = sh_tot[4]; mt.nSq = sh_tot[5];
    mt.tol = tol;
    mt.zz = zz;
  }
}

// ===========================================================================
// Deflation rotations on W/Q rows (vector mode).  grid (row chunks, merges).
__global__ void bdc_rotate_kernel(const MergeDesc* __restrict__ merges, const MergeMeta* __restrict__ meta,
                                  BdcBufs B, double* W, long long ldw, double* Q, long long ldq) {
  const MergeDesc M = merges[blockIdx.y];
  const int nrot = meta[blockIdx.y].nrot;
  if (nrot == 0) return;
  const int r0 = M.r0, n = M.n, ncols = M.n + M.bordered;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ncols) return;
  const int* pc = B.physcol + r0;
  double* qrow = Q + (r0 + i);
  double* wrow = W + (r0 + i);
  const bool dow = i < n;
  for (int t = 0; t < nrot; ++t) {
    const int p = B.rot_p[r0 + t], j = B.rot_j[r0 + t];
    const double c = B.rot_c[r0 + t], s = B.rot_s[r0 + t];
    const long long cp = pc[p], cj = pc[j];
    const double qp = qrow[cp * ldq], qj = qrow[cj * ldq];
    qrow[cp * ldq] = c * qp + s * qj;
    qrow[cj * ldq] = c * qj - s * qp;
    if (p != 0 && dow) {
      const double wp = wrow[cp * ldw], wj = wrow[cj * ldw];
      wrow[cp * ldw] = c * wp + s * wj;
      wrow[cj * ldw] = c * wj - s * wp;
    }
  }
}

// ===========================================================================
// Secular equation: one warp per root (bdc.py:541-641).
constexpr int kSecWarps = 8;

// One root of the secular equation per warp (all lanes participate; lane 0
// stores).  d ascending with d[0] = 0, z, zz = sum z^2.
__device__ void secular_root_warp(const double* __restrict__ d, const double* __restrict__ z, int K, double zz,
                                  int i, int lane, double* omega, int* anc_out, double* mu_out, int* err,
                                  int max_iter = 100) {
  if (K == 1) {
    if (lane == 0) {
      omega[0] = sqrt(zz);
      anc_out[0] = 0;
      mu_out[0] = zz;
    }
    return;
  }
  const bool top = (i == K - 1);
  const int lo_i = i, hi_i = top ? K - 1 : i + 1;
  const double dl = d[lo_i], dh = d[hi_i];
  const double width = top ? zz : (dh - dl) * (dh + dl);
  double fm = 0.0;
  for (int j = lane; j < K; j += 32) {
    const double dj = d[j], zj = z[j];
    fm += (zj * zj) / ((dj - dl) * (dj + dl) - 0.5 * width);
  }
  fm = 1.0 + warp_sum(fm);
  const bool lower = fm > 0.0;
  const int anc = (lower || top) ? lo_i : hi_i;
  const double da = d[anc];
  const double gl = (d[lo_i] - da) * (d[lo_i] + da);
  const double gh = top ? gl + zz : (d[hi_i] - da) * (d[hi_i] + da);
  double lo = lower ? 0.0 : (top ? 0.5 * width : -0.5 * width);
  double hi = lower ? 0.5 * width : (top ? width : 0.0);
  double mu = 0.5 * (lo + hi);
  const double ftol = 8.0 * K * DC_EPS;
  bool done = false;
  for (int it = 0; it < max_iter; ++it) {  // bdc.py:589, budget max_iterations (100)
    double psi = 0.0, phi = 0.0, sa = 0.0, dpsi = 0.0, dphi = 0.0;
    for (int j = lane; j < K; j += 32) {
      const double dj = d[j], zj = z[j];
      const double den = (dj - da) * (dj + da) - mu;
      const double t = (zj * zj) / den;
      const double t2 = t / den;
      if (j <= i) { psi += t; dpsi += t2; } else { phi += t; dphi += t2; }
      sa += fabs(t);
    }
    psi = warp_sum(psi);
    phi = warp_sum(phi);
    sa = 1.0 + warp_sum(sa);
    dpsi = warp_sum(dpsi);
    dphi = warp_sum(dphi);
    const double f = 1.0 + (psi + phi);
    const bool narrow = (hi - lo) <= 8.0 * DC_EPS * fmax(fabs(lo), fabs(hi));
    if (fabs(f) <= ftol * sa || narrow || !isfinite(f)) {
      done = true;
      break;
    }
    if (f < 0.0) lo = mu; else hi = mu;
    const double a_ = gl - mu, b_ = gh - mu;
    const double bigS = dpsi * a_ * a_;
    const double bigR = dphi * b_ * b_;
    const double s0 = 1.0 + (psi - dpsi * a_) + (phi - dphi * b_);
    const double qb = -(s0 * (a_ + b_) + bigS + bigR);
    const double qc = s0 * a_ * b_ + bigS * b_ + bigR * a_;
    const double sq = sqrt(fmax(qb * qb - 4.0 * s0 * qc, 0.0));
    const double qq = -0.5 * (qb + (qb >= 0.0 ? sq : -sq));
    const double e1 = qq / s0, e2 = qc / qq;
    const double c1 = mu + e1, c2 = mu + e2;
    const bool ok1 = isfinite(c1) && c1 > lo && c1 < hi;
    const bool ok2 = isfinite(c2) && c2 > lo && c2 < hi;
    const bool take1 = ok1 && (!ok2 || fabs(e1) <= fabs(e2));
    mu = take1 ? c1 : (ok2 ? c2 : 0.5 * (lo + hi));
  }
  if (lane == 0) {
    if (!done) raise_dev(err, kDevNoConvergeSecular);
    omega[i] = sqrt(fmax(da * da + mu, 0.0));
    anc_out[i] = anc;
    mu_out[i] = mu;
  }
}

__global__ void __launch_bounds__(32 * kSecWarps) bdc_secular_kernel(const MergeDesc* __restrict__ merges,
                                                                     const MergeMeta* __restrict__ meta, BdcBufs B,
                                                                     int* err) {
  const MergeDesc M = merges[blockIdx.y];
  const int K = meta[blockIdx.y].K;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSecWarps + (threadIdx.x >> 5);
  if (i >= K) return;
  const int r0 = M.r0;
  secular_root_warp(B.ds + r0, B.zs + r0, K, meta[blockIdx.y].zz, i, lane, B.omega + r0, B.anc + r0, B.mu + r0, err);
}

// Standalone secular solve (solve_all_roots, bdc.py:515-525); zz from device.
__global__ void __launch_bounds__(32 * kSecWarps) secular_standalone_kernel(const double* d, const double* z, int K,
                                                                            const double* zzp, double* omega,
                                                                            int* anc, double* mu, int* err,
                                                                            int max_iter) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSecWarps + (threadIdx.x >> 5);
  if (i >= K) return;
  secular_root_warp(d, z, K, *zzp, i, lane, omega, anc, mu, err, max_iter);
}

__global__ void sumsq_kernel(const double* z, int K, double* out) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) v += z[i] * z[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) *out = v;
}

// Loewner z recomputation: one warp per entry i (bdc.py:644-673).
__global__ void __launch_bounds__(32 * kSecWarps) bdc_loewner_kernel(const MergeDesc* __restrict__ merges,
                                                                     const MergeMeta* __restrict__ meta, BdcBufs B,
                                                                     int* err) {
  const MergeDesc M = merges[blockIdx.y];
  const int K = meta[blockIdx.y].K;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSecWarps + (threadIdx.x >> 5);
  if (i >= K) return;
  const int r0 = M.r0;
  const double* __restrict__ d = B.ds + r0;
  const double* __restrict__ mu = B.mu + r0;
  const int* __restrict__ anc = B.anc + r0;
  const double di = d[i];
  double prod = 1.0;
  for (int k = lane; k < K - 1; k += 32) {
    const double da = d[anc[k]];
    const double num = (da - di) * (da + di) + mu[k];
    const double dk = k < i ? d[k] : d[k + 1];
    const double den = (dk - di) * (dk + di);
    prod *= num / den;
  }
  prod = warp_prod(prod);
  if (lane == 0) {
    const double dl = d[anc[K - 1]];
    const double numl = (dl - di) * (dl + di) + mu[K - 1];
    const double rad = numl * prod;
    if (!(rad > 0.0)) raise_dev(err, kDevInterlacing);
    B.zt[r0 + i] = copysign(sqrt(rad), B.zs[r0 + i]);
  }
}

// Middle-matrix singular vectors + edge companion: one warp per column i
// (bdc.py:676-694, :830).  umat rows in W-class order (unit row apart),
// vmat rows in Q-class order; both stored in the node's diagonal block.
__global__ void __launch_bounds__(32 * kSecWarps) bdc_vectors_kernel(const MergeDesc* __restrict__ merges,
                                                                     const MergeMeta* __restrict__ meta, BdcBufs B,
                                                                     double* Us, double* Vs, long long lds,
                                                                     int vectors) {
  const MergeDesc M = merges[blockIdx.y];
  const int K = meta[blockIdx.y].K;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSecWarps + (threadIdx.x >> 5);
  if (i >= K) return;
  const int r0 = M.r0;
  const double* __restrict__ d = B.ds + r0;
  const double* __restrict__ zt = B.zt + r0;
  const double da = d[B.anc[r0 + i]], mu = B.mu[r0 + i];
  double sv = 0.0, su = 0.0;
  for (int j = lane; j < K; j += 32) {
    const double dj = d[j];
    const double v = zt[j] / ((dj - da) * (dj + da) - mu);
    const double u = j == 0 ? -1.0 : dj * v;
    sv += v * v;
    su += u * u;
  }
  const double nv = sqrt(warp_sum(sv));
  const double nu = sqrt(warp_sum(su));
  double e0 = 0.0, e1 = 0.0;
  double* Vcol = Vs + r0 + (long long)(r0 + i) * lds;
  double* Ucol = Us + r0 + (long long)(r0 + i) * lds;
  for (int j = lane; j < K; j += 32) {
    const double dj = d[j];
    const double vr = zt[j] / ((dj - da) * (dj + da) - mu);
    const double v = vr / nv;
    e0 += B.ke0[r0 + j] * v;
    e1 += B.ke1[r0 + j] * v;
    if (vectors) {
      Vcol[B.qpos[r0 + j]] = v;
      if (j >= 1) Ucol[B.wpos[r0 + j]] = (dj * vr) / nu;
    }
  }
  e0 = warp_sum(e0);
  e1 = warp_sum(e1);
  if (lane == 0) {
    B.ekn0[r0 + i] = e0;
    B.ekn1[r0 + i] = e1;
    B.uunit[r0 + i] = -1.0 / nu;
  }
}

// Stable ascending order of [omega (K), deflated values (nd)] (bdc.py:829-831)
// and write of the node's values / edge rows.  One CTA per merge.
__device__ __forceinline__ int count_before(const double* vals, const int* idx, int cnt, double x, int xi) {
  // #{t : vals[t] < x or (vals[t] == x and idx[t] < xi)}, vals ascending, idx ascending within ties
  int lo = 0, hi = cnt;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const double v = vals[mid];
    if (v < x || (v == x && idx[mid] < xi)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

constexpr int kOrderThreads = 512;

__global__ void __launch_bounds__(kOrderThreads) bdc_order_kernel(const MergeDesc* __restrict__ merges,
                                                                  MergeMeta* __restrict__ meta, BdcBufs B, double* dv,
                                                                  double* edge, double* scratch_v, int* scratch_i) {
  __shared__ int sh_flag;
  __shared__ int sh_cnt[kOrderThreads][2];
  __shared__ int sh_tot[2];
  const MergeDesc M = merges[blockIdx.x];
  MergeMeta& mt = meta[blockIdx.x];
  const int K = mt.K, nd = mt.nd;
  const int r0 = M.r0, n = M.n, tid = threadIdx.x;
  // runs: R0 = omega (concat idx 0..K-1); R1 = regular deflated; R2 = zero-pair
  // deflated (value 0.0).  Split deflated into R1/R2 preserving order.
  double* v1 = scratch_v + r0;        // R1 values (up to nd)
  int* i1 = scratch_i + r0;           // R1 concat idx
  const double* om = B.omega + r0;
  {
    const int per = (nd + blockDim.x - 1) / blockDim.x;
    const int t0 = tid * per, t1 = min(nd, t0 + per);
    int c1 = 0, c2 = 0;
    for (int t = t0; t < t1; ++t) (B.dkind[r0 + t] ? c2 : c1)++;
    sh_cnt[tid][0] = c1;
    sh_cnt[tid][1] = c2;
    __syncthreads();
    if (tid < 2) {
      int run = 0;
      for (int t = 0; t < (int)blockDim.x; ++t) {
        const int v = sh_cnt[t][tid];
        sh_cnt[t][tid] = run;
        run += v;
      }
      sh_tot[tid] = run;
    }
    if (tid == 0) sh_flag = 1;
    __syncthreads();
    int a1 = sh_cnt[tid][0], a2 = sh_cnt[tid][1];
    const int n1 = sh_tot[0];
    for (int t = t0; t < t1; ++t) {
      if (B.dkind[r0 + t]) {
        v1[n1 + a2] = 0.0;
        i1[n1 + a2] = K + t;
        ++a2;
      } else {
        v1[a1] = B.dval[r0 + t];
        i1[a1] = K + t;
        ++a1;
      }
    }
  }
  __syncthreads();
  const int n1 = sh_tot[0], n2 = sh_tot[1];
  // verify monotonicity of the runs (fall back to O(n^2) ranks otherwise)
  for (int t = tid; t + 1 < K; t += blockDim.x)
    if (om[t + 1] < om[t]) sh_flag = 0;
  for (int t = tid; t + 1 < n1; t += blockDim.x)
    if (v1[t + 1] < v1[t]) sh_flag = 0;
  __syncthreads();
  const bool fast = sh_flag != 0;
  // R0 indices are 0..K-1 implicitly
  for (int q = tid; q < K + nd; q += blockDim.x) {
    double x;
    int xi = q;
    if (q < K) x = om[q];
    else x = B.dkind[r0 + q - K] ? 0.0 : B.dval[r0 + q - K];
    int pos;
    if (fast) {
      // R0: count omega[t] < x or (== x and t < xi)
      int lo = 0, hi = K;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (om[mid] < x || (om[mid] == x && mid < xi)) lo = mid + 1; else hi = mid;
      }
      pos = lo + count_before(v1, i1, n1, x, xi) + count_before(v1 + n1, i1 + n1, n2, x, xi);
    } else {
      pos = 0;
      for (int t = 0; t < K + nd; ++t) {
        const double y = t < K ? om[t] : (B.dkind[r0 + t - K] ? 0.0 : B.dval[r0 + t - K]);
        pos += (y < x) || (y == x && t < xi);
      }
    }
    if (q < K) {
      B.kdst[r0 + q] = pos;
      B.kdstphys[r0 + q] = r0 + pos;
    } else {
      B.ddst[r0 + q - K] = pos;
    }
  }
  __syncthreads();
  // node values and edge rows (children's consumed in prep)
  for (int q = tid; q < K + nd; q += blockDim.x) {
    int pos;
    double x, e0, e1;
    if (q < K) {
      pos = B.kdst[r0 + q];
      x = om[q];
      e0 = B.ekn0[r0 + q];
      e1 = B.ekn1[r0 + q];
    } else {
      const int t = q - K;
      pos = B.ddst[r0 + t];
      x = B.dkind[r0 + t] ? 0.0 : B.dval[r0 + t];
      const int j = B.defl[r0 + t];
      e0 = B.ew0[r0 + j];
      e1 = B.ew1[r0 + j];
    }
    dv[r0 + pos] = x;
    edge[2LL * (r0 + pos) + 0] = e0;
    edge[2LL * (r0 + pos) + 1] = e1;
  }
  if (M.bordered && tid == 0) {
    edge[2LL * (r0 + n) + 0] = mt.null_e0;
    edge[2LL * (r0 + n) + 1] = mt.null_e1;
  }
}

// Grouped-GEMM descriptors for the structured merge products (bdc.py:701-747).
__global__ void bdc_gemm_desc_kernel(const MergeDesc* __restrict__ merges, const MergeMeta* __restrict__ meta,
                                     int nmerges, BdcBufs B, const double* W, const double* Q, long long ld,
                                     const double* Us, const double* Vs, double* S3, double* S4,
                                     GemmDesc* __restrict__ out, double* flops) {
  const int mi = blockIdx.x * blockDim.x + threadIdx.x;
  if (mi >= nmerges) return;
  const MergeDesc M = merges[mi];
  const MergeMeta mt = meta[mi];
  const int r0 = M.r0, nl = M.nl, ncols = M.n + M.bordered;
  GemmDesc g;
  g.alpha = 1.0;
  g.beta = 0.0;
  g.n = mt.K;
  g.ccol = B.kdstphys + r0;
  // W top: rows [0, nl), cols F u M
  g.m = nl; g.k = mt.nFw + mt.nMw;
  g.A = W + r0; g.lda = ld; g.acol = B.wphys + r0;
  g.B = Us + r0 + (long long)r0 * ld; g.ldb = ld;
  g.C = S3 + r0; g.ldc = ld;
  out[4 * mi + 0] = g;
  // W bottom: rows [nl+1, n), cols M u S
  g.m = M.nr; g.k = mt.nMw + mt.nSw;
  g.A = W + r0 + nl + 1; g.acol = B.wphys + r0 + mt.nFw;
  g.B = Us + (r0 + mt.nFw) + (long long)r0 * ld;
  g.C = S3 + r0 + nl + 1;
  out[4 * mi + 1] = g;
  // Q top: rows [0, nl+1)
  g.m = nl + 1; g.k = mt.nFq + mt.nMq;
  g.A = Q + r0; g.acol = B.qphys + r0;
  g.B = Vs + r0 + (long long)r0 * ld;
  g.C = S4 + r0;
  out[4 * mi + 2] = g;
  // Q bottom: rows [nl+1, ncols)
  g.m = ncols - nl - 1; g.k = mt.nMq + mt.nSq;
  g.A = Q + r0 + nl + 1; g.acol = B.qphys + r0 + mt.nFq;
  g.B = Vs + (r0 + mt.nFq) + (long long)r0 * ld;
  g.C = S4 + r0 + nl + 1;
  out[4 * mi + 3] = g;
  if (flops) {  // stats: 2 m n k of the four products (integers: exact in fp64)
    double f = 0.0;
    for (int q = 0; q < 4; ++q) f += 2.0 * out[4 * mi + q].m * (double)out[4 * mi + q].n * out[4 * mi + q].k;
    atomicAdd(flops, f);
    atomicAdd(flops + 1, 16.0 * mt.nd * (double)(M.n + ncols));  // deflated W/Q columns read + written
  }
}

// Deflated columns, unit row, null column into scratch.  One warp per output
// column; grid (column chunks, merges).
__global__ void bdc_defl_copy_kernel(const MergeDesc* __restrict__ merges, const MergeMeta* __restrict__ meta,
                                     BdcBufs B, const double* W, const double* Q, long long ld, double* S3,
                                     double* S4) {
  const MergeDesc M = merges[blockIdx.y];
  const MergeMeta& mt = meta[blockIdx.y];
  const int K = mt.K, nd = mt.nd;
  const int r0 = M.r0, n = M.n, nl = M.nl, ncols = n + M.bordered;
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q < nd) {
    const long long src = B.physcol[r0 + B.defl[r0 + q]];
    const long long dst = r0 + B.ddst[r0 + q];
    for (int r = lane; r < n; r += 32) S3[(r0 + r) + dst * ld] = W[(r0 + r) + src * ld];
    for (int r = lane; r < ncols; r += 32) S4[(r0 + r) + dst * ld] = Q[(r0 + r) + src * ld];
  } else if (q < nd + K) {
    const int k = q - nd;
    if (lane == 0) S3[(r0 + nl) + (long long)B.kdstphys[r0 + k] * ld] = B.uunit[r0 + k];
  } else if (q == nd + K && M.bordered) {
    const long long src = r0 + ncols - 1, dst = r0 + n;
    for (int r = lane; r < ncols; r += 32) S4[(r0 + r) + dst * ld] = Q[(r0 + r) + src * ld];
  }
}

// Node blocks scratch -> main.  grid (column chunks, merges), warp per column.
__global__ void bdc_copyback_kernel(const MergeDesc* __restrict__ merges, const double* S3, const double* S4,
                                    long long ld, double* W, double* Q) {
  const MergeDesc M = merges[blockIdx.y];
  const int r0 = M.r0, n = M.n, ncols = n + M.bordered;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const long long col = (long long)(r0 + c) * ld;
  if (c < n)
    for (int r = lane; r < n; r += 32) W[(r0 + r) + col] = S3[(r0 + r) + col];
  for (int r = lane; r < ncols; r += 32) Q[(r0 + r) + col] = S4[(r0 + r) + col];
}

__global__ void bdc_unit_kernel(const int* rows, int cnt, double* W, long long ld) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) W[rows[i] + (long long)rows[i] * ld] = 1.0;
}

// Final descending reversal (bdc.py:871-880) into the caller's outputs.
// Optionally writes U = [W_rev; 0] (m rows) and VT = Q_rev^T instead of W/Q.
__global__ void bdc_out_values_kernel(int n, int ncols, const double* dv, const double* edge, double* dvals,
                                      double* edge_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    dvals[i] = dv[n - 1 - i];
    if (edge_out) {
      edge_out[2 * i + 0] = edge[2LL * (n - 1 - i) + 0];
      edge_out[2 * i + 1] = edge[2LL * (n - 1 - i) + 1];
    }
  } else if (i < ncols && edge_out) {
    edge_out[2 * i + 0] = edge[2LL * i + 0];
    edge_out[2 * i + 1] = edge[2LL * i + 1];
  }
}

__global__ void bdc_out_w_kernel(int n, int mrows, const double* Wsrc, long long lds, double* Wout, long long ldo) {
  // Wout[:, i] = [Wsrc[:, n-1-i]; 0] (mrows >= n rows)
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n) return;
  const double* src = Wsrc + (long long)(n - 1 - c) * lds;
  double* dst = Wout + (long long)c * ldo;
  for (int r = lane; r < mrows; r += 32) dst[r] = r < n ? src[r] : 0.0;
}

__global__ void bdc_out_q_kernel(int n, int ncols, const double* Qsrc, long long lds, double* Qout, long long ldo) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= ncols) return;
  const int sc = c < n ? n - 1 - c : c;
  const double* src = Qsrc + (long long)sc * lds;
  double* dst = Qout + (long long)c * ldo;
  for (int r = lane; r < ncols; r += 32) dst[r] = src[r];
}

// VT[i, j] = Q_rev[j, i]  (square n, tiled transpose)
__global__ void bdc_out_qt_kernel(int n, const double* Qsrc, long long lds, double* VT, long long ldvt) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  // read Q_rev rows bx.., cols by..: Q_rev[r, c] = Qsrc[r, n-1-c]
  for (int k = ty; k < 32; k += 8) {
    const int r = bx + tx, c = by + k;
    tile[k][tx] = (r < n && c < n) ? Qsrc[r + (long long)(n - 1 - c) * lds] : 0.0;
  }
  __syncthreads();
  // VT[c, r] = Q_rev[r, c]; write rows c = by.., cols r = bx..
  for (int k = ty; k < 32; k += 8) {
    const int r = bx + k, c = by + tx;
    if (r < n && c < n) VT[c + (long long)r * ldvt] = tile[tx][k];
  }
}

// ===========================================================================
// Host driver.
struct TreeNode {
  int r0, n, nl, nr, bordered, height, leaf;
};

static int build_tree(std::vector<TreeNode>& out, int r0, int n, int bordered, int leaf) {
  TreeNode t;
  t.r0 = r0; t.n = n; t.bordered = bordered; t.nl = 0; t.nr = 0;
  if (n <= leaf) {
    t.leaf = 1;
    t.height = 0;
    out.push_back(t);
    return 0;
  }
  const int k = n / 2;
  t.nl = k - 1;
  t.nr = n - k;
  t.leaf = 0;
  const int hl = build_tree(out, r0, t.nl, 1, leaf);
  const int hr = build_tree(out, r0 + t.nl + 1, t.nr, bordered, leaf);
  t.height = 1 + std::max(hl, hr);
  out.push_back(t);
  return t.height;
}

int bdsdc_run(dcsvd_ctx* h, cudaStream_t st, long long n_, const double* d, const double* e, bool bordered,
              bool vectors, int leaf, double tol_mult, double* dvals, double* edge_out, double* Wout,
              long long ldwo, long long wrows, double* Qout, long long ldqo, double* VT, long long ldvt) {
  if (leaf < 1) return set_error(h, DCSVD_EINVAL, "leaf size must be >= 1, got %d", leaf);
  // Leaves above 32 (the warp-per-leaf QR kernel) split once more: the same
  // decomposition up to rounding.
  if (leaf > 32) leaf = 32;
  if (!(tol_mult > 0.0)) return set_error(h, DCSVD_EINVAL, "deflation multiple must be > 0");
  const int n = (int)n_;
  const int ncols = n + (bordered ? 1 : 0);
  if (n < 0) return set_error(h, DCSVD_EINVAL, "n must be >= 0");
  if (ncols == 0) return 0;  // 0 x 0 problem: empty outputs (bdc.py:754-765)
  std::vector<TreeNode> nodes;
  int H = 0;
  if (n > 0) H = build_tree(nodes, 0, n, bordered ? 1 : 0, leaf);
  else {
    TreeNode t{0, 0, 0, 0, bordered ? 1 : 0, 0, 1};
    nodes.push_back(t);
  }
  std::vector<LeafDesc> leaves;
  std::vector<std::vector<MergeDesc>> levels(H + 1);
  std::vector<int> unit_rows;
  int maxn_level_n = 0;
  for (auto& t : nodes) {
    if (t.leaf) leaves.push_back(LeafDesc{t.r0, t.n, t.bordered});
    else {
      levels[t.height].push_back(MergeDesc{t.r0, t.n, t.nl, t.nr, t.bordered});
      unit_rows.push_back(t.r0 + t.nl);
    }
  }
  (void)maxn_level_n;
  const long long ld = ncols > 0 ? ncols : 1;
  const size_t E = (size_t)ncols + 2;
  int nmerge_total = 0;
  for (auto& L : levels) nmerge_total += (int)L.size();
  // ---- device memory (pool 2)
  size_t need = 0;
  const size_t mat = (size_t)ld * ld;
  need += 2 * pool_bytes(E, 8) /*dv, edge(2E)*/ + pool_bytes(2 * E, 8);
  need += 40 * pool_bytes(E, 8);  // per-entry arrays (generous)
  need += pool_bytes(leaves.size() * sizeof(LeafDesc), 1) + pool_bytes(nmerge_total * sizeof(MergeDesc), 1) +
          pool_bytes(nmerge_total * sizeof(MergeMeta), 1) + pool_bytes(4 * nmerge_total * sizeof(GemmDesc), 1) +
          pool_bytes(unit_rows.size() + 1, 4);
  if (vectors) need += 6 * pool_bytes(mat, 8);
  int rc = pool_reserve(h, 2, need, st);
  if (rc) return rc;
  double* dv = pool_take<double>(h, 2, E);
  double* edge = pool_take<double>(h, 2, 2 * E);
  BdcBufs B;
  B.dpre = pool_take<double>(h, 2, E); B.zpre = pool_take<double>(h, 2, E);
  B.perm = pool_take<int>(h, 2, E);
  B.dw = pool_take<double>(h, 2, E); B.zw = pool_take<double>(h, 2, E);
  B.lcls = pool_take<int>(h, 2, E); B.rcls = pool_take<int>(h, 2, E);
  B.ew0 = pool_take<double>(h, 2, E); B.ew1 = pool_take<double>(h, 2, E);
  B.kept = pool_take<int>(h, 2, E); B.kcl = pool_take<int>(h, 2, E); B.kcr = pool_take<int>(h, 2, E);
  B.ke0 = pool_take<double>(h, 2, E); B.ke1 = pool_take<double>(h, 2, E);
  B.defl = pool_take<int>(h, 2, E); B.dval = pool_take<double>(h, 2, E); B.dkind = pool_take<int>(h, 2, E);
  B.rot_p = pool_take<int>(h, 2, E); B.rot_j = pool_take<int>(h, 2, E);
  B.rot_c = pool_take<double>(h, 2, E); B.rot_s = pool_take<double>(h, 2, E);
  B.ds = pool_take<double>(h, 2, E); B.zs = pool_take<double>(h, 2, E);
  B.omega = pool_take<double>(h, 2, E); B.mu = pool_take<double>(h, 2, E); B.anc = pool_take<int>(h, 2, E);
  B.zt = pool_take<double>(h, 2, E);
  B.wpos = pool_take<int>(h, 2, E); B.qpos = pool_take<int>(h, 2, E);
  B.wphys = pool_take<int>(h, 2, E); B.qphys = pool_take<int>(h, 2, E);
  B.ekn0 = pool_take<double>(h, 2, E); B.ekn1 = pool_take<double>(h, 2, E);
  B.uunit = pool_take<double>(h, 2, E);
  B.kdst = pool_take<int>(h, 2, E); B.ddst = pool_take<int>(h, 2, E);
  B.physcol = pool_take<int>(h, 2, E); B.kdstphys = pool_take<int>(h, 2, E);
  double* sv = pool_take<double>(h, 2, E);
  int* si = pool_take<int>(h, 2, E);
  LeafDesc* d_leaves = (LeafDesc*)pool_take<char>(h, 2, leaves.size() * sizeof(LeafDesc));
  MergeDesc* d_merges = (MergeDesc*)pool_take<char>(h, 2, std::max(1, nmerge_total) * sizeof(MergeDesc));
  MergeMeta* d_meta = (MergeMeta*)pool_take<char>(h, 2, std::max(1, nmerge_total) * sizeof(MergeMeta));
  GemmDesc* d_gd = (GemmDesc*)pool_take<char>(h, 2, std::max(1, 4 * nmerge_total) * sizeof(GemmDesc));
  int* d_units = pool_take<int>(h, 2, unit_rows.size() + 1);
  double *W = nullptr, *Q = nullptr, *Us = nullptr, *Vs = nullptr, *S3 = nullptr, *S4 = nullptr;
  if (vectors) {
    W = pool_take<double>(h, 2, mat); Q = pool_take<double>(h, 2, mat);
    Us = pool_take<double>(h, 2, mat); Vs = pool_take<double>(h, 2, mat);
    S3 = pool_take<double>(h, 2, mat); S4 = pool_take<double>(h, 2, mat);
    if (!S4) return set_error(h, DCSVD_ECUDA, "BDC workspace carve failed");
  }
  // ---- upload the tree (synchronous copies of small host arrays)
  std::vector<MergeDesc> flat;
  std::vector<int> level_off(H + 2, 0);
  for (int lv = 1; lv <= H; ++lv) {
    level_off[lv] = (int)flat.size();
    for (auto& m : levels[lv]) flat.push_back(m);
  }
  level_off[H + 1] = (int)flat.size();
  // Through the handle's pinned staging buffer: the copies stay asynchronous
  // (no stream drain, so the host builds the next call's tree while the GPU
  // still runs this one); only a previous upload from the same buffer is
  // waited for before it is overwritten.
  {
    const size_t b_leaves = leaves.size() * sizeof(LeafDesc), b_flat = flat.size() * sizeof(MergeDesc),
                 b_units = unit_rows.size() * sizeof(int);
    const size_t o_flat = (b_leaves + 255) & ~size_t(255), o_units = o_flat + ((b_flat + 255) & ~size_t(255));
    const size_t need = o_units + b_units + 256;
    if (h->stage_pending) DC_CUDA_TRY(cudaEventSynchronize(h->ev_stage));
    h->stage_pending = false;
    if (!h->ev_stage) DC_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_stage, cudaEventDisableTiming));
    if (h->h_stage_bytes < need) {
      if (h->h_stage) cudaFreeHost(h->h_stage);
      h->h_stage = nullptr;
      h->h_stage_bytes = 0;
      DC_CUDA_TRY(cudaMallocHost(&h->h_stage, need * 2));
      h->h_stage_bytes = need * 2;
    }
    memcpy(h->h_stage, leaves.data(), b_leaves);
    if (b_flat) memcpy(h->h_stage + o_flat, flat.data(), b_flat);
    if (b_units) memcpy(h->h_stage + o_units, unit_rows.data(), b_units);
    DC_CUDA_TRY(cudaMemcpyAsync(d_leaves, h->h_stage, b_leaves, cudaMemcpyHostToDevice, st));
    if (b_flat) DC_CUDA_TRY(cudaMemcpyAsync(d_merges, h->h_stage + o_flat, b_flat, cudaMemcpyHostToDevice, st));
    if (b_units) DC_CUDA_TRY(cudaMemcpyAsync(d_units, h->h_stage + o_units, b_units, cudaMemcpyHostToDevice, st));
    DC_CUDA_TRY(cudaEventRecord(h->ev_stage, st));
    h->stage_pending = true;
  }
  if (vectors) {
    DC_CUDA_TRY(cudaMemsetAsync(W, 0, mat * sizeof(double), st));
    DC_CUDA_TRY(cudaMemsetAsync(Q, 0, mat * sizeof(double), st));
    if (!unit_rows.empty()) {
      bdc_unit_kernel<<<((int)unit_rows.size() + 255) / 256, 256, 0, st>>>(d_units, (int)unit_rows.size(), W, ld);
      note_launch();
    }
  }
  // ---- leaves
  bdc_leaf_kernel<<<((int)leaves.size() + kLeafWarps - 1) / kLeafWarps, 32 * kLeafWarps, 0, st>>>(
      d_leaves, (int)leaves.size(), d, e, W, ld, Q, ld, dv, edge, vectors ? 1 : 0, h->d_err);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  // ---- merges, level by level
  for (int lv = 1; lv <= H; ++lv) {
    const int nm = level_off[lv + 1] - level_off[lv];
    if (nm == 0) continue;
    const MergeDesc* md = d_merges + level_off[lv];
    MergeMeta* mm = d_meta + level_off[lv];
    int maxn = 0;
    for (auto& m : levels[lv]) maxn = std::max(maxn, m.n + 1);
    bdc_prep_kernel<<<nm, kPrepThreads, 0, st>>>(md, mm, d, e, dv, edge, Q, ld, vectors ? 1 : 0, tol_mult, B,
                                                  h->d_err);
    note_launch();
    if (vectors) {
      bdc_rotate_kernel<<<dim3((maxn + 127) / 128, nm), 128, 0, st>>>(md, mm, B, W, ld, Q, ld);
      note_launch();
    }
    const dim3 gw((maxn + kSecWarps - 1) / kSecWarps, nm);
    bdc_secular_kernel<<<gw, 32 * kSecWarps, 0, st>>>(md, mm, B, h->d_err);
    bdc_loewner_kernel<<<gw, 32 * kSecWarps, 0, st>>>(md, mm, B, h->d_err);
    bdc_vectors_kernel<<<gw, 32 * kSecWarps, 0, st>>>(md, mm, B, Us, Vs, ld, vectors ? 1 : 0);
    bdc_order_kernel<<<nm, kOrderThreads, 0, st>>>(md, mm, B, dv, edge, sv, si);
    note_launch(4);
    DC_CUDA_TRY(cudaGetLastError());
    if (vectors) {
      GemmDesc* gd = d_gd + 4 * level_off[lv];
      bdc_gemm_desc_kernel<<<(nm + 127) / 128, 128, 0, st>>>(md, mm, nm, B, W, Q, ld, Us, Vs, S3, S4, gd,
                                                            h->stats_on ? h->d_flops : nullptr);
      note_launch();
      const int sidx = stat_begin(h, 2, 0.0, st);  // flops arrive through h->d_flops
      // TMA GEMM over the workspace stack W, Q, Us, Vs, S3, S4 when they are carved
      // back to back (ld^2 doubles a multiple of the 256-byte pool granule)
      rc = (Q == W + mat && S4 == W + 5 * mat) ? gemm_launch_device_stack(st, gd, 4 * nm, maxn, maxn, W, ld, 6) : -1;
      if (rc < 0) rc = gemm_launch_device(st, false, false, gd, 4 * nm, maxn, maxn);
      stat_end(h, sidx, st);
      if (rc) return rc;
      const int sc = stat_begin(h, 3, 0.0, st);  // bytes arrive through h->d_flops[1]
      bdc_defl_copy_kernel<<<dim3((maxn + 1 + 7) / 8, nm), 256, 0, st>>>(md, mm, B, W, Q, ld, S3, S4);
      stat_end(h, sc, st);
      note_launch();
      if (lv < H) {
        double cb = 0.0;
        for (const auto& mg : levels[lv]) cb += 16.0 * ((double)mg.n * mg.n + (double)(mg.n + mg.bordered) * (mg.n + mg.bordered));
        const int sb = stat_begin(h, 3, cb, st);
        bdc_copyback_kernel<<<dim3((maxn + 7) / 8, nm), 256, 0, st>>>(md, S3, S4, ld, W, Q);
        stat_end(h, sb, st);
        note_launch();
      }
      DC_CUDA_TRY(cudaGetLastError());
    }
  }
  // ---- outputs
  bdc_out_values_kernel<<<(ncols + 255) / 256, 256, 0, st>>>(n, ncols, dv, edge, dvals, edge_out);
  note_launch();
  if (vectors && ncols > 0) {
    const double* Wsrc = (H > 0) ? S3 : W;
    const double* Qsrc = (H > 0) ? S4 : Q;
    if (Wout && n > 0) {
      bdc_out_w_kernel<<<(n + 7) / 8, 256, 0, st>>>(n, (int)std::max<long long>(wrows, n), Wsrc, ld, Wout, ldwo);
      note_launch();
    }
    if (VT && n > 0) {
      bdc_out_qt_kernel<<<dim3((n + 31) / 32, (n + 31) / 32), 256, 0, st>>>(n, Qsrc, ld, VT, ldvt);
      note_launch();
    }
    if (Qout) {
      bdc_out_q_kernel<<<(ncols + 7) / 8, 256, 0, st>>>(n, ncols, Qsrc, ld, Qout, ldqo);
      note_launch();
    }
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// Standalone secular-equation pieces of the reference API (bdc.py:515-694),
// on one secular system of size K held in device memory.

__global__ void __launch_bounds__(32 * kSecWarps) loewner_standalone_kernel(const double* __restrict__ d,
                                                                            const double* __restrict__ z, int K,
                                                                            const int* __restrict__ anc,
                                                                            const double* __restrict__ mu, double* zt,
                                                                            int* err) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSecWarps + (threadIdx.x >> 5);
  if (i >= K) return;
  const double di = d[i];
  double prod = 1.0;
  for (int k = lane; k < K - 1; k += 32) {
    const double da = d[anc[k]];
    const double num = (da - di) * (da + di) + mu[k];
    const double dk = k < i ? d[k] : d[k + 1];
    prod *= num / ((dk - di) * (dk + di));
  }
  prod = warp_prod(prod);
  if (lane == 0) {
    const double dl = d[anc[K - 1]];
    const double rad = ((dl - di) * (dl + di) + mu[K - 1]) * prod;
    if (!(rad > 0.0)) raise_dev(err, kDevInterlacing);
    zt[i] = copysign(sqrt(rad), z[i]);
  }
}

__global__ void __launch_bounds__(32 * kSecWarps) secvec_standalone_kernel(const double* __restrict__ d, int K,
                                                                           const int* __restrict__ anc,
                                                                           const double* __restrict__ mu,
                                                                           const double* __restrict__ zt, double* U,
                                                                           long long ldu, double* V, long long ldv) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * kSecWarps + (threadIdx.x >> 5);
  if (i >= K) return;
  const double da = d[anc[i]], m = mu[i];
  double sv = 0.0, su = 0.0;
  for (int j = lane; j < K; j += 32) {
    const double dj = d[j];
    const double v = zt[j] / ((dj - da) * (dj + da) - m);
    const double u = j == 0 ? -1.0 : dj * v;
    sv += v * v;
    su += u * u;
  }
  const double nv = sqrt(warp_sum(sv)), nu = sqrt(warp_sum(su));
  for (int j = lane; j < K; j += 32) {
    const double dj = d[j];
    const double v = zt[j] / ((dj - da) * (dj + da) - m);
    V[j + (long long)i * ldv] = v / nv;
    U[j + (long long)i * ldu] = (j == 0 ? -1.0 : dj * v) / nu;
  }
}

int secular_run(dcsvd_ctx* h, cudaStream_t st, int K, const double* d, const double* z, double* omega, int* anc,
                double* mu, int max_iter) {
  if (K < 1) return set_error(h, DCSVD_EINVAL, "secular system must be nonempty");
  if (max_iter < 0) return set_error(h, DCSVD_EINVAL, "max_iterations must be >= 0, got %d", max_iter);
  int rc = pool_reserve(h, 0, pool_bytes(1, 8), st);
  if (rc) return rc;
  double* zz = pool_take<double>(h, 0, 1);
  sumsq_kernel<<<1, 256, 0, st>>>(z, K, zz);
  secular_standalone_kernel<<<(K + kSecWarps - 1) / kSecWarps, 32 * kSecWarps, 0, st>>>(d, z, K, zz, omega, anc, mu,
                                                                                        h->d_err, max_iter);
  note_launch(2);
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int loewner_run(dcsvd_ctx* h, cudaStream_t st, int K, const double* d, const double* z, const int* anc, const double* mu,
                double* zt) {
  loewner_standalone_kernel<<<(K + kSecWarps - 1) / kSecWarps, 32 * kSecWarps, 0, st>>>(d, z, K, anc, mu, zt, h->d_err);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int secvec_run(dcsvd_ctx* h, cudaStream_t st, int K, const double* d, const int* anc, const double* mu, const double* zt,
               double* U, long long ldu, double* V, long long ldv) {
  secvec_standalone_kernel<<<(K + kSecWarps - 1) / kSecWarps, 32 * kSecWarps, 0, st>>>(d, K, anc, mu, zt, U, ldu, V,
                                                                                       ldv);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace dc
