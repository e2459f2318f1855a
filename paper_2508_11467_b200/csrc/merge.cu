// Standalone merge stages of the bidiagonal divide and conquer, as single
// calls of the reference API (the fused tree in bdc.cu runs the same steps
// inside its level-synchronous kernels):
//   build_z        bdc.py:382-412   middle-row data of a merge
//   deflate        bdc.py:423-508   stable sort + deflation scan, applied to
//                                    the supplied column matrices in place
//   gather                           row/column gather used by merge_vectors
//                                    (bdc.py:701-747; the products are DMMA
//                                    GEMMs through dcsvd_dgemm)
#include "ctx.cuh"
#include "launch.cuh"

namespace dc {

// ---------------------------------------------------------------------------
// build_z: d = [0, D1, D2]; z = [z0, alpha * L1[:nl], beta * F2[:nr]];
// bordered: (c, s), z0 = givens(alpha * lambda1, beta * phi2), else z0 = alpha * lambda1.
__global__ void build_z_kernel(int nl, int nr, int bordered, double alpha, double beta, const double* __restrict__ ldv,
                               const double* __restrict__ ledge, long long lde_l, const double* __restrict__ rdv,
                               const double* __restrict__ redge, long long lde_r, double* __restrict__ d,
                               double* __restrict__ z, double* __restrict__ coupling) {
  const int n = nl + nr + 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i == 0) {
      d[0] = 0.0;
      const double lam1 = ledge[1 + (long long)nl * lde_l];  // last edge row of the left child, column nl
      if (bordered) {
        const double phi2 = redge[0 + (long long)nr * lde_r];  // first edge row of the right child, column nr
        double c, s, r;
        lartg(alpha * lam1, beta * phi2, c, s, r);
        z[0] = r;
        coupling[0] = c;
        coupling[1] = s;
      } else {
        z[0] = alpha * lam1;
        coupling[0] = 1.0;
        coupling[1] = 0.0;
      }
    } else if (i <= nl) {
      d[i] = ldv[i - 1];
      z[i] = alpha * ledge[1 + (long long)(i - 1) * lde_l];
    } else {
      const int j = i - 1 - nl;
      d[i] = rdv[j];
      z[i] = beta * redge[0 + (long long)j * lde_r];
    }
  }
}

// ---------------------------------------------------------------------------
// deflate, part 1 (one CTA): stable ascending order of d (rank = #smaller +
// #equal-and-earlier, the np.argsort(kind="stable") permutation), tolerance,
// z0 clamp and the sequential deflation scan against the last kept entry.
// Class arrays (int32, optional) are permuted and merged in place.
constexpr int kDeflThreads = 1024;

__device__ __forceinline__ int merge_class(int a, int b) { return a == b ? a : 3; }

__global__ void __launch_bounds__(kDeflThreads) deflate_scan_kernel(
    int n, const double* __restrict__ d_in, const double* __restrict__ z_in, double tol_multiple, long long* perm,
    double* d, double* z, long long* kept, long long* deflated, double* dvals, long long* rot_pq, double* rot_cs,
    long long* counts, int* lcls, int* rcls, int* cls_tmp, int* err) {
  __shared__ double sh_red[32];
  const int tid = threadIdx.x;
  for (int i = tid; i < n; i += blockDim.x) {
    const double di = d_in[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = d_in[j];
      rank += (dj < di) || (dj == di && j < i);
    }
    perm[rank] = i;
  }
  __syncthreads();
  double mx = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    const long long p = perm[i];
    d[i] = d_in[p];
    z[i] = z_in[p];
    mx = fmax(mx, fmax(fabs(d_in[p]), fabs(z_in[p])));
  }
  // class arrays follow the permutation
  for (int c = 0; c < 2; ++c) {
    int* cls = c == 0 ? lcls : rcls;
    if (!cls) continue;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) cls_tmp[i] = cls[perm[i]];
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) cls[i] = cls_tmp[i];
  }
  // block max (fixed tree)
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __syncthreads();
  if ((tid & 31) == 0) sh_red[tid >> 5] = mx;
  __syncthreads();
  if (tid != 0) return;
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sh_red[w]);
  mx = fmax(mx, sh_red[0]);
  if (d[0] != 0.0) {
    raise_dev(err, kDevBadDeflate);
    counts[0] = counts[1] = counts[2] = 0;
    return;
  }
  const double tol = tol_multiple * DC_EPS * fmax(mx, 0.0);
  if (fabs(z[0]) <= tol) z[0] = copysign(fmax(tol, DC_TINY), z[0] != 0.0 ? z[0] : 1.0);
  long long nk = 0, nd = 0, nr = 0;
  kept[nk++] = 0;
  for (int j = 1; j < n; ++j) {
    if (fabs(z[j]) <= tol) {
      z[j] = 0.0;
      deflated[nd] = j;
      dvals[nd++] = d[j];
      continue;
    }
    const long long p = kept[nk - 1];
    if (d[j] - d[p] <= tol) {
      double c, s, r;
      lartg(z[p], z[j], c, s, r);
      z[p] = r;
      z[j] = 0.0;
      rot_pq[2 * nr] = p;
      rot_pq[2 * nr + 1] = j;
      rot_cs[2 * nr] = c;
      rot_cs[2 * nr + 1] = s;
      ++nr;
      if (p == 0) {  // pairs with the zero entry: right side only, value 0
        if (rcls) rcls[p] = rcls[j] = merge_class(rcls[p], rcls[j]);
        deflated[nd] = j;
        dvals[nd++] = 0.0;
      } else {
        d[p] = d[j];
        if (lcls) lcls[p] = lcls[j] = merge_class(lcls[p], lcls[j]);
        if (rcls) rcls[p] = rcls[j] = merge_class(rcls[p], rcls[j]);
        deflated[nd] = j;
        dvals[nd++] = d[j];
      }
    } else {
      kept[nk++] = j;
    }
  }
  counts[0] = nk;
  counts[1] = nd;
  counts[2] = nr;
}

// dst[r, c] = src[ridx ? ridx[r] : r, cidx ? cidx[c] : c] (rows x cnt).
// deflate uses it to permute columns through a scratch copy.
__global__ void gather2d_kernel(int rows, int cnt, const double* __restrict__ src, long long lds,
                                const long long* __restrict__ ridx, const long long* __restrict__ cidx,
                                double* __restrict__ dst, long long ldd) {
  const long long tot = (long long)rows * cnt;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % rows), c = (int)(e / rows);
    const long long sr = ridx ? ridx[r] : r, sc = cidx ? cidx[c] : c;
    dst[r + c * ldd] = src[sr + sc * lds];
  }
}

__global__ void copy_cols_kernel(int rows, int cnt, const double* __restrict__ src, long long lds, double* __restrict__ dst,
                                 long long ldd) {
  const long long tot = (long long)rows * cnt;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % rows), c = (int)(e / rows);
    dst[r + c * ldd] = src[r + c * lds];
  }
}

// deflate, part 3: the recorded rotations [[c, s], [-s, c]] on column pairs
// (p, j), in scan order, one thread per row (rows are independent).
// `left_side`: rotations paired with entry 0 skip the left matrix.
__global__ void apply_rotations_kernel(int rows, double* M, long long ld, const long long* __restrict__ rot_pq,
                                       const double* __restrict__ rot_cs, const long long* __restrict__ counts,
                                       int left_side) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const long long nr = counts[2];
  for (long long t = 0; t < nr; ++t) {
    const long long p = rot_pq[2 * t], q = rot_pq[2 * t + 1];
    if (left_side && p == 0) continue;
    const double c = rot_cs[2 * t], s = rot_cs[2 * t + 1];
    double* mp = M + r + p * ld;
    double* mq = M + r + q * ld;
    const double a = *mp, b = *mq;
    *mp = c * a + s * b;
    *mq = -s * a + c * b;
  }
}

static int launch_grid(long long work) {
  const long long g = (work + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

int build_z_run(dcsvd_ctx* h, cudaStream_t st, int nl, int nr, int bordered, double alpha, double beta,
                const double* ldv, const double* ledge, long long lde_l, const double* rdv, const double* redge,
                long long lde_r, double* d, double* z, double* coupling) {
  if (nl < 0 || nr < 0) return set_error(h, DCSVD_EINVAL, "build_z: negative child size");
  const int n = nl + nr + 1;
  build_z_kernel<<<(n + 255) / 256, 256, 0, st>>>(nl, nr, bordered, alpha, beta, ldv, ledge, lde_l, rdv, redge, lde_r,
                                                  d, z, coupling);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int deflate_run(dcsvd_ctx* h, cudaStream_t st, int n, const double* d_in, const double* z_in, double tol_multiple,
                double* left, long long rows_l, long long ldl, double* right, long long rows_r, long long ldr,
                double* edge, long long lde, int* lcls, int* rcls, long long* perm, double* d, double* z,
                long long* kept, long long* deflated, double* dvals, long long* rot_pq, double* rot_cs,
                long long* counts) {
  if (n < 1) return set_error(h, DCSVD_EINVAL, "deflate expects at least the border entry");
  const long long maxrows = std::max(std::max(rows_l, rows_r), (long long)2);
  int rc = pool_reserve(h, 0, pool_bytes((size_t)maxrows * n, 8) + pool_bytes(n, 4), st);
  if (rc) return rc;
  double* tmp = pool_take<double>(h, 0, (size_t)maxrows * n);
  int* cls_tmp = pool_take<int>(h, 0, n);
  deflate_scan_kernel<<<1, kDeflThreads, 0, st>>>(n, d_in, z_in, tol_multiple, perm, d, z, kept, deflated, dvals,
                                                  rot_pq, rot_cs, counts, lcls, rcls, cls_tmp, h->d_err);
  note_launch();
  struct Side {
    double* M;
    long long rows, ld;
    int left;
  } sides[3] = {{left, rows_l, ldl, 1}, {right, rows_r, ldr, 0}, {edge, 2, lde, 0}};
  for (const Side& sd : sides) {
    if (!sd.M || sd.rows <= 0) continue;
    const long long work = sd.rows * n;
    gather2d_kernel<<<launch_grid(work), 256, 0, st>>>((int)sd.rows, n, sd.M, sd.ld, nullptr, perm, tmp, sd.rows);
    copy_cols_kernel<<<launch_grid(work), 256, 0, st>>>((int)sd.rows, n, tmp, sd.rows, sd.M, sd.ld);
    apply_rotations_kernel<<<(int)((sd.rows + 127) / 128), 128, 0, st>>>((int)sd.rows, sd.M, sd.ld, rot_pq, rot_cs,
                                                                         counts, sd.left);
    note_launch(3);
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int gather2d_run(dcsvd_ctx* h, cudaStream_t st, long long rows, long long cnt, const double* src, long long lds,
                 const long long* ridx, const long long* cidx, double* dst, long long ldd) {
  if (rows < 0 || cnt < 0) return set_error(h, DCSVD_EINVAL, "gather: negative size");
  if (rows == 0 || cnt == 0) return 0;
  gather2d_kernel<<<launch_grid(rows * cnt), 256, 0, st>>>((int)rows, (int)cnt, src, lds, ridx, cidx, dst, ldd);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace dc
