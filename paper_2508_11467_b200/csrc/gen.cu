// Test-matrix generation and accuracy metrics on the GPU (harness.py:69-187).
//
// The reference draws every random number from numpy's Philox-4x64-10 keyed
// by the seed, consumed as ONE word stream (harness.py:69-88): word w of the
// stream is lane w % 4 of the block with counter w / 4 + 1 (numpy increments
// the counter before the first block), uniform = ((w >> 11) + 0.5) * 2^-53,
// normals by Box-Muller on consecutive uniform pairs.  The Philox words and
// the uniforms here are bit-identical to the reference's; normals go through
// CUDA double-precision log/sqrt/cos/sin (within 1-2 ulp of glibc), so normals
// and the matrices built from them match the reference to rounding, not bitwise.
//
// generate_matrix (harness.py:131-146): 'random' = uniforms column-major;
// 'logrand'/'arith'/'geo' = U diag(sigma) V^T with U, V the Q factors of
// blocked QRs of standard-normal matrices (our GEQRF/ORGQR, R-diagonal signs
// absorbed, harness.py:117-128) and one DMMA GEMM.
#include <limits>

#include "ctx.cuh"
#include "gemm.cuh"
#include "launch.cuh"

namespace dc {

typedef unsigned long long u64;

__device__ __forceinline__ u64 philox_word(u64 k0, u64 k1, u64 w) {
  const u64 M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const u64 W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  const u64 b = (w >> 2) + 1;  // 128-bit counter; b + 1 never carries for < 2^64 words
  u64 c0 = b, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const u64 lo0 = M0 * c0, hi0 = __umul64hi(M0, c0);
    const u64 lo1 = M1 * c2, hi1 = __umul64hi(M1, c2);
    const u64 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  switch (w & 3) {
    case 0: return c0;
    case 1: return c1;
    case 2: return c2;
    default: return c3;
  }
}

__device__ __forceinline__ double word_uniform(u64 w) { return ((double)(w >> 11) + 0.5) * 1.1102230246251565e-16; }

// count outputs written column-major into a rows x * matrix with leading dim ld.
// normal == 0: out[e] = uniform(word off + e); normal == 1: Box-Muller pairs
// (words off + 2p, off + 2p + 1) -> (r cos, r sin) for outputs 2p, 2p + 1.
__global__ void philox_fill_kernel(u64 k0, u64 k1, u64 off, long long count, int normal, double* out, long long rows,
                                   long long ld) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (!normal) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count; e += stride)
      out[e % rows + (e / rows) * ld] = word_uniform(philox_word(k0, k1, off + e));
    return;
  }
  const long long pairs = (count + 1) / 2;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pairs; p += stride) {
    const double u1 = word_uniform(philox_word(k0, k1, off + 2 * p));
    const double u2 = word_uniform(philox_word(k0, k1, off + 2 * p + 1));
    const double r = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.141592653589793 * u2;
    const long long e0 = 2 * p, e1 = 2 * p + 1;
    out[e0 % rows + (e0 / rows) * ld] = r * cos(ang);
    if (e1 < count) out[e1 % rows + (e1 / rows) * ld] = r * sin(ang);
  }
}

// prescribed spectra (harness.py:91-105); kind 1 logrand (u = uniforms), 2 arith, 3 geo
__global__ void sigma_kernel(int kind, int n, double cond, const double* __restrict__ u, double* __restrict__ s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (kind == 1) {
    s[i] = exp(-log(cond) * u[i]);
  } else if (n == 1) {
    s[i] = 1.0;
  } else if (kind == 2) {
    s[i] = 1.0 - ((double)i / (n - 1)) * (1.0 - 1.0 / cond);
  } else {
    s[i] = pow(cond, -(double)i / (n - 1));
  }
}

// descending stable sort by rank (np.sort(...)[::-1]: ties keep reverse order,
// immaterial for equal values)
__global__ void sort_desc_kernel(int n, const double* __restrict__ in, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = in[i];
  int rank = 0;
  for (int j = 0; j < n; ++j) {
    const double w = in[j];
    rank += (w > v) || (w == v && j < i);
  }
  out[rank] = v;
}

// column signs: Q[:, j] *= -1 where R[j, j] < 0 (harness.py:125-127)
__global__ void sign_fix_kernel(long long rows, int cols, double* Q, long long ldq, const double* R, long long ldr) {
  const long long tot = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / rows, r = e % rows;
    if (R[j + j * ldr] < 0.0) Q[r + j * ldq] = -Q[r + j * ldq];
  }
}

__global__ void scale_cols_kernel(long long rows, int cols, double* U, long long ldu, const double* s) {
  const long long tot = rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / rows, r = e % rows;
    U[r + j * ldu] *= s[j];
  }
}

// ---------------------------------------------------------------------------
// Frobenius norms for the accuracy report, deterministic two-level sums.
// mode 0: sum (X - Y)^2; mode 1: sum (X - I)^2; mode 2: sum X^2 (Y unused).
constexpr int kNormBlocks = 296, kNormThreads = 256;

__global__ void __launch_bounds__(kNormThreads) sumsq_partial_kernel(long long rows, long long cols, const double* X,
                                                                     long long ldx, const double* Y, long long ldy,
                                                                     int mode, double* part) {
  __shared__ double sh[32];
  const long long tot = rows * cols;
  double s = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / rows, r = e % rows;
    double v = X[r + j * ldx];
    if (mode == 0) v -= Y[r + j * ldy];
    if (mode == 1 && r == j) v -= 1.0;
    s += v * v;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_final_kernel(const double* part, int cnt, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

static int grid_for(long long work) {
  const long long g = (work + 255) / 256;
  return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

int philox_run(dcsvd_ctx* h, cudaStream_t st, u64 k0, u64 k1, u64 off, long long count, int normal, double* out,
               long long rows, long long ld) {
  if (count < 0 || rows < 1 || ld < rows) return set_error(h, DCSVD_EINVAL, "philox: bad sizes");
  if (count == 0) return 0;
  philox_fill_kernel<<<grid_for(normal ? (count + 1) / 2 : count), 256, 0, st>>>(k0, k1, off, count, normal, out, rows,
                                                                                 ld);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// sigma (n) of kind 1..3 drawn at stream word `*off` (logrand consumes n words)
static int sigma_run(dcsvd_ctx* h, cudaStream_t st, int kind, int n, double cond, u64 k0, u64 k1, u64* off,
                     double* sigma, double* scratch) {
  if (kind == 1) {
    int rc = philox_run(h, st, k0, k1, *off, n, 0, scratch, n, n);
    if (rc) return rc;
    *off += n;
    sigma_kernel<<<(n + 255) / 256, 256, 0, st>>>(1, n, cond, scratch, scratch + n);
    sort_desc_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, scratch + n, sigma);
    note_launch(2);
  } else {
    sigma_kernel<<<(n + 255) / 256, 256, 0, st>>>(kind, n, cond, nullptr, sigma);
    note_launch();
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int prescribed_sigma_run(dcsvd_ctx* h, cudaStream_t st, int kind, int n, double cond, u64 k0, u64 k1, double* sigma) {
  if (kind < 1 || kind > 3) return set_error(h, DCSVD_EINVAL, "kind 'random' has no prescribed singular values");
  if (n < 1) return set_error(h, DCSVD_EINVAL, "need n >= 1");
  int rc = pool_reserve(h, 1, pool_bytes(2 * (size_t)n, 8), st);
  if (rc) return rc;
  double* scratch = pool_take<double>(h, 1, 2 * (size_t)n);
  u64 off = 0;
  return sigma_run(h, st, kind, n, cond, k0, k1, &off, sigma, scratch);
}

// Q factor (rows x cols) of the QR of a standard-normal matrix drawn at *off.
static int haar_run(dcsvd_ctx* h, cudaStream_t st, long long rows, int cols, u64 k0, u64 k1, u64* off, double* G,
                    double* tau, double* Q) {
  const long long cnt = rows * cols;
  int rc = philox_run(h, st, k0, k1, *off, cnt, 1, G, rows, rows);
  if (rc) return rc;
  *off += 2 * (u64)((cnt + 1) / 2);
  rc = geqrf_run(h, st, rows, cols, G, rows, tau, 32);  // harness.py:123 geqrf_blocked(g, block=32)
  if (rc) return rc;
  rc = orgqr_run(h, st, rows, cols, cols, G, rows, tau, Q, rows, 64);  // orgqr(fact, cols), block 64
  if (rc) return rc;
  sign_fix_kernel<<<grid_for(cnt), 256, 0, st>>>(rows, cols, Q, rows, G, rows);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int generate_run(dcsvd_ctx* h, cudaStream_t st, int kind, long long m, long long n, double cond, u64 k0, u64 k1,
                 double* A, long long lda) {
  if (m < 1 || n < 1 || lda < m) return set_error(h, DCSVD_EINVAL, "matrix must be nonempty, got %lldx%lld", m, n);
  if (kind < 0 || kind > 3) return set_error(h, DCSVD_EINVAL, "unknown matrix kind %d", kind);
  if (!(cond >= 1.0)) return set_error(h, DCSVD_EINVAL, "cond must be >= 1, got %g", cond);
  if (kind == 0) return philox_run(h, st, k0, k1, 0, m * n, 0, A, m, lda);
  const long long k = std::min(m, n);
  // pool 1: sigma scratch, G, tau, U, V
  const size_t need = pool_bytes(3 * (size_t)k, 8) + pool_bytes((size_t)std::max(m, n) * k, 8) +
                      pool_bytes((size_t)k, 8) + pool_bytes((size_t)m * k, 8) + pool_bytes((size_t)n * k, 8);
  int rc = pool_reserve(h, 1, need, st);
  if (rc) return rc;
  double* sig = pool_take<double>(h, 1, 3 * (size_t)k);
  double* G = pool_take<double>(h, 1, (size_t)std::max(m, n) * k);
  double* tau = pool_take<double>(h, 1, (size_t)k);
  double* U = pool_take<double>(h, 1, (size_t)m * k);
  double* V = pool_take<double>(h, 1, (size_t)n * k);
  u64 off = 0;
  rc = sigma_run(h, st, kind, (int)k, cond, k0, k1, &off, sig, sig + k);
  if (rc) return rc;
  rc = haar_run(h, st, m, (int)k, k0, k1, &off, G, tau, U);
  if (rc) return rc;
  rc = haar_run(h, st, n, (int)k, k0, k1, &off, G, tau, V);
  if (rc) return rc;
  scale_cols_kernel<<<grid_for(m * k), 256, 0, st>>>(m, (int)k, U, m, sig);
  note_launch();
  GemmDesc gd;  // A = (U sigma) V^T
  gd.m = (int)m; gd.n = (int)n; gd.k = (int)k;
  gd.A = U; gd.lda = m; gd.acol = nullptr;
  gd.B = V; gd.ldb = n;
  gd.C = A; gd.ldc = lda; gd.ccol = nullptr;
  gd.alpha = 1.0; gd.beta = 0.0;
  rc = gemm_launch(st, false, true, gd);
  if (rc) return rc;
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// AccuracyReport (harness.py:149-187): out = {e_sigma, e_svd, orth_u, orth_v};
// NaN marks "None" (no reference / no vectors).
int accuracy_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, const double* A, long long lda,
                 const double* S, const double* U, long long ldu, const double* VT, long long ldvt,
                 const double* ref, double* out_host) {
  const long long k = std::min(m, n);
  const bool vec = U && VT;
  const size_t need = pool_bytes(kNormBlocks, 8) + pool_bytes(8, 8) + (vec ? pool_bytes((size_t)m * n, 8) +
                      pool_bytes((size_t)m * k, 8) + pool_bytes((size_t)k * k, 8) : 0);
  int rc = pool_reserve(h, 1, need, st);
  if (rc) return rc;
  double* part = pool_take<double>(h, 1, kNormBlocks);
  double* res = pool_take<double>(h, 1, 8);
  auto sumsq = [&](long long rows, long long cols, const double* X, long long ldx, const double* Y, long long ldy,
                   int mode, int slot) {
    sumsq_partial_kernel<<<kNormBlocks, kNormThreads, 0, st>>>(rows, cols, X, ldx, Y, ldy, mode, part);
    sum_final_kernel<<<1, 256, 0, st>>>(part, kNormBlocks, res + slot);
    note_launch(2);
  };
  if (ref) sumsq(k, 1, S, k, ref, k, 0, 0);
  if (vec) {
    double* R = pool_take<double>(h, 1, (size_t)m * n);
    double* US = pool_take<double>(h, 1, (size_t)m * k);
    double* G = pool_take<double>(h, 1, (size_t)k * k);
    DC_CUDA_TRY(cudaMemcpy2DAsync(US, m * 8, U, ldu * 8, m * 8, k, cudaMemcpyDeviceToDevice, st));
    scale_cols_kernel<<<grid_for(m * k), 256, 0, st>>>(m, (int)k, US, m, S);
    note_launch();
    GemmDesc gd;  // R = (U sigma) Vt
    gd.m = (int)m; gd.n = (int)n; gd.k = (int)k;
    gd.A = US; gd.lda = m; gd.acol = nullptr;
    gd.B = VT; gd.ldb = ldvt;
    gd.C = R; gd.ldc = m; gd.ccol = nullptr;
    gd.alpha = 1.0; gd.beta = 0.0;
    rc = gemm_launch(st, false, false, gd);
    if (rc) return rc;
    sumsq(m, n, A, lda, R, m, 0, 1);
    sumsq(m, n, A, lda, nullptr, 0, 2, 2);
    gd.m = (int)k; gd.n = (int)k; gd.k = (int)m;  // G = U^T U
    gd.A = U; gd.lda = ldu; gd.B = U; gd.ldb = ldu; gd.C = G; gd.ldc = k;
    rc = gemm_launch(st, true, false, gd);
    if (rc) return rc;
    sumsq(k, k, G, k, nullptr, 0, 1, 3);
    gd.m = (int)k; gd.n = (int)k; gd.k = (int)n;  // G = Vt Vt^T
    gd.A = VT; gd.lda = ldvt; gd.B = VT; gd.ldb = ldvt;
    rc = gemm_launch(st, false, true, gd);
    if (rc) return rc;
    sumsq(k, k, G, k, nullptr, 0, 1, 4);
  }
  double hv[5] = {0, 0, 0, 0, 0};
  DC_CUDA_TRY(cudaMemcpyAsync(hv, res, sizeof(hv), cudaMemcpyDeviceToHost, st));
  DC_CUDA_TRY(cudaStreamSynchronize(st));
  const double nan = std::numeric_limits<double>::quiet_NaN();
  out_host[0] = ref ? sqrt(hv[0]) / (double)k : nan;
  if (vec) {
    const double na = sqrt(hv[2]);
    out_host[1] = na > 0.0 ? sqrt(hv[1]) / na : sqrt(hv[1]);
    out_host[2] = sqrt(hv[3]);
    out_host[3] = sqrt(hv[4]);
  } else {
    out_host[1] = out_host[2] = out_host[3] = nan;
  }
  return 0;
}

}  // namespace dc
