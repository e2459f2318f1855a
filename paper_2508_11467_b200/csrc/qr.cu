// Householder QR (GEQRF/ORGQR) and the bidiagonal back-transformations
// (ORMBR) with inverse-T compact-WY block reflectors.
//
// Reference: pkg/src/dcsvd/qrblock.py (geqrf_panel :51-71, _panel_y :74-87,
// build_tinv :90-100, apply_block_reflector_left/right :103-119, geqrf_blocked
// :122-144, orgqr :147-164) and pkg/src/dcsvd/backtransform.py:60-131;
// arxiv 2508.11467 modified CWY.
//
// Every block application is DMMA GEMM work: Z = Y^T C (split-K over the long
// dimension with a fixed-order partial reduction), G = Y^T Y in the same
// batched launch, one CTA turns G into T^-1 = triu(G,1) + diag(1/tau) and
// inverts it (so the reference's TRSM becomes one small GEMM X = T Z), then
// C -= Y X.  The unblocked QR panel is a cooperative kernel that keeps each
// CTA's row slab of the panel in shared memory for all its columns.
#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "gemm.cuh"
#include "launch.cuh"

namespace dc {

// ---------------------------------------------------------------------------
// Y / Y^T construction from packed reflector storage.
//  ymode 0 ('Q' / QR): Y (rows x w, ld rows) from src = packed + off + off*lda:
//     Y[r,t] = r == t ? 1 : r > t ? src[r + t*lda] : 0, zero column if tau[t] == 0
//  ymode 1 ('P'): Yt (w x rows, ld w) from src = packed + off + (off+1)*lda:
//     Yt[t,r] = r == t ? 1 : r > t ? src[t + r*lda] : 0, zero row if tau[t] == 0
__global__ void build_y_kernel(int ymode, const double* __restrict__ src, long long lda,
                               const double* __restrict__ tau, int rows, int w, double* __restrict__ Y) {
  const long long total = (long long)rows * w;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int r, t;
    if (ymode == 0) { r = (int)(idx % rows); t = (int)(idx / rows); }
    else { t = (int)(idx % w); r = (int)(idx / w); }
    double v = 0.0;
    if (tau[t] != 0.0) {
      if (r == t) v = 1.0;
      else if (r > t) v = ymode == 0 ? src[r + (long long)t * lda] : src[t + (long long)r * lda];
    }
    Y[idx] = v;
  }
}

// G = sum_s Gp[s]; Tinv = triu(G,1) + diag(1/tau) (1 when tau == 0)
// (qrblock.py:90-100), column-major into global scratch.
constexpr int kCwyMaxW = 128;

// (batched over blockIdx.y: block b reads Gp + b gstride, tau + b taustride, writes Tinv + b w^2)
__global__ void cwy_tinv_build_kernel(const double* __restrict__ Gp, int S, int w, const double* __restrict__ tau,
                                      double* __restrict__ Tinv, int* err, long long gstride = 0, int taustride = 0) {
  Gp += blockIdx.y * gstride;
  tau += blockIdx.y * taustride;
  Tinv += (long long)blockIdx.y * w * w;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= w * w) return;
  const int i = idx % w, l = idx / w;
  double v = 0.0;
  if (i < l) {
    for (int s = 0; s < S; ++s) v += Gp[(long long)s * w * w + idx];
  } else if (i == l) {
    v = tau[i] != 0.0 ? 1.0 / tau[i] : 1.0;
    if (v == 0.0) raise_dev(err, kDevSingularT);
  }
  Tinv[idx] = v;
}

// T = Tinv^-1, one warp per column c: right-looking back substitution with
// the column held in registers (lane owns rows lane + 32q) and Tinv staged
// in shared memory once per CTA.  Top = T or T^T.
constexpr int kTinvSolveWarps = 16;

__global__ void __launch_bounds__(32 * kTinvSolveWarps) cwy_tinv_solve_kernel(const double* __restrict__ Tinv, int w,
                                                                              int trans, double* __restrict__ Top) {
  extern __shared__ double ts[];  // w x w (ld w); diagonal replaced by its reciprocal
  Tinv += (long long)blockIdx.y * w * w;  // batched over blockIdx.y (one w x w block each)
  Top += (long long)blockIdx.y * w * w;
  {
    const int tot = w * w;
    if ((reinterpret_cast<uintptr_t>(Tinv) & 15) == 0) {  // 16-byte staging, 4 loads in flight
      const double2* src = reinterpret_cast<const double2*>(Tinv);
      double2* dst = reinterpret_cast<double2*>(ts);
      const int n2 = tot >> 1;
#pragma unroll 4
      for (int i = threadIdx.x; i < n2; i += blockDim.x) dst[i] = src[i];
      if ((tot & 1) && threadIdx.x == 0) ts[tot - 1] = Tinv[tot - 1];
    } else {
#pragma unroll 4
      for (int i = threadIdx.x; i < tot; i += blockDim.x) ts[i] = Tinv[i];
    }
    __syncthreads();
    if (threadIdx.x < w) ts[threadIdx.x * (w + 1)] = 1.0 / ts[threadIdx.x * (w + 1)];  // no division in the chain
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kTinvSolveWarps + (threadIdx.x >> 5);
  if (c >= w) return;
  double t[kCwyMaxW / 32];
#pragma unroll
  for (int q = 0; q < kCwyMaxW / 32; ++q) t[q] = (lane + 32 * q == c) ? 1.0 : 0.0;
  for (int i = c; i >= 0; --i) {
    const double* col = ts + i * w;  // Tinv[:, i]
    const int qi = i >> 5, li = i & 31;
    double ti = 0.0;
#pragma unroll
    for (int q = 0; q < kCwyMaxW / 32; ++q)
      if (q == qi) ti = t[q];
    ti = __shfl_sync(0xffffffffu, ti, li) * col[i];
#pragma unroll
    for (int q = 0; q < kCwyMaxW / 32; ++q) {
      const int l = lane + 32 * q;
      if (l < i) t[q] -= col[l] * ti;
      else if (l == i) t[q] = ti;
    }
  }
#pragma unroll
  for (int q = 0; q < kCwyMaxW / 32; ++q) {
    const int l = lane + 32 * q;
    if (l < w) {
      const double v = l <= c ? t[q] : 0.0;
      if (trans) Top[c + (long long)l * w] = v;  // Top = T^T: Top[c, l] = T[l, c]
      else Top[l + (long long)c * w] = v;
    }
  }
}

static int tinv_solve_launch(cudaStream_t st, const double* Tinv, int w, bool trans, double* Top, int nbatch = 1) {
  DC_CUDA_TRY((cudaError_t)func_attr(cwy_tinv_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kCwyMaxW * kCwyMaxW * 8));
  cwy_tinv_solve_kernel<<<dim3((w + kTinvSolveWarps - 1) / kTinvSolveWarps, nbatch), 32 * kTinvSolveWarps,
                          (size_t)w * w * 8, st>>>(Tinv, w, trans ? 1 : 0, Top);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

__global__ void splitk_reduce_kernel(double* __restrict__ Zp, long long count, int S) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double v = Zp[i];
    for (int s = 1; s < S; ++s) v += Zp[(long long)s * count + i];
    Zp[i] = v;
  }
}

// Split-K reduce for many partials and few outputs (the thin CWY products of
// the tall QR: 32 x 96 outputs, 74-127 slices): one warp per output, lanes
// over the slices in fixed order, then a fixed shuffle tree (deterministic).
__global__ void splitk_reduce_warp_kernel(double* __restrict__ Zp, long long count, int S) {
  const long long o = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (o >= count) return;
  double v = 0.0;
  for (int s = lane; s < S; s += 32) v += Zp[(long long)s * count + o];
  v = warp_sum(v);
  if (lane == 0) Zp[o] = v;
}

static int grid_for(long long n, int threads = 256) {
  long long g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

// Apply the block reflector with Y (ytrans == false: Y rows_y x w, ld rows_y;
// ytrans == true: Yt w x rows_y, ld w) to C.  side 'L': C (rows_y x ncols)
// <- (I - Y op(T) Y^T) C.  side 'R': C (nrows x rows_y) <- C (I - Y op(T) Y^T).
// op(T) = T or T^T (trans).  Scratch from pool 0 at `scratch` (caller sized
// via cwy_scratch_doubles).
// Split-K factor for Z = Y^T C (K = rows_y): enough 64x64 tiles x slices for
// ~3 CTAs per SM, slices of >= 128 rows, partials <= 16M doubles.
constexpr int kMaxKSplit = 128;  // split-K slices (in-kernel, GemmBatch::ksplit)

int g_cwy_split_mode = 1;  // debug: 0 = round-1 rule (>= 2 tiles of 64 x 128 per SM)
static int cwy_split(int sms, int w, long long c_other, long long rows_y) {
  if (g_cwy_split_mode == 0) {
    // count 64x128 tiles: enough of them (>= 2 per SM) selects the 2-CTA/SM DMMA config
    const long long zt = ((w + 63) / 64) * ((c_other + 127) / 128);
    int S = 1;
    while (S < kMaxKSplit && zt * S < 2LL * sms && rows_y / (S * 2) >= 256 &&
           (long long)(2 * S) * w * c_other <= (16LL << 20))
      S *= 2;
    return S;
  }
  // The inner products run on the TMA GEMM (128 x 64 tiles, one CTA per SM):
  // pick the split with the smallest wave-quantised time ceil(T S / sms) / S,
  // plus a ~2 us pipeline fill per CTA (a full-K CTA streams ~65 ns per row of
  // Y); K slices of >= 256 rows, partials <= 16M doubles.
  const long long T = ((w + 127) / 128) * ((c_other + 63) / 64);
  int best = 1;
  double bt = 1e300;
  for (int S = 1; S <= kMaxKSplit; ++S) {
    if (S > 1 && rows_y / S < 256) break;
    if (S > 1 && (long long)S * w * c_other > (16LL << 20)) break;
    const double waves = (double)((T * S + sms - 1) / sms);
    const double t = waves * ((double)rows_y / S * 65e-9 + 2e-6);
    if (t < bt * 0.99) {
      bt = t;
      best = S;
    }
  }
  return best;
}

// G = Y^T Y (w x w output, K = the reflector rows) gets its own split: with
// one or two 128 x 64 tiles it needs ~74 K-slices to fill the GPU on the TMA
// GEMM (it ran on 64 x 64 cp.async tiles at ~10 % of peak before).
constexpr int kMaxGSplit = 74;
int g_cwy_gsplit = 1;  // debug: 0 = G shares the Z split
int g_qr_outer = 0;    // debug: outer CWY block width of GEQRF (0 = 128; 64: C3 GEQRF 15.0 -> 16.2 ms, 32: 20.2)
static int cwy_gsplit(int sms, int w, long long rows_y, int S) {
  if (!g_cwy_gsplit) return S;
  const long long tg = ((w + 127) / 128) * ((w + 63) / 64);
  long long sg = (sms + tg - 1) / tg;
  sg = std::min<long long>(sg, kMaxGSplit);
  sg = std::min<long long>(sg, std::max<long long>(1, rows_y / 64));
  return (int)std::max<long long>(sg, S > 1 ? 1 : 1);
}

static size_t cwy_scratch_doubles(int sms, long long rows_y, long long c_other, int w) {
  const int S = cwy_split(sms, w, c_other, rows_y);
  const int SG = std::max(S, kMaxGSplit);
  return (size_t)S * (size_t)w * (size_t)c_other + (size_t)SG * w * w + 2 * (size_t)w * w + 64;
}

__global__ void copy_tinv_kernel(const double* __restrict__ src, long long lds, int w, double* __restrict__ dst,
                                 int* err) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= w * w) return;
  const int i = idx % w, j = idx / w;
  const double v = src[i + (long long)j * lds];
  if (i == j && v == 0.0) raise_dev(err, kDevSingularT);
  dst[idx] = i <= j ? v : 0.0;
}

// `utinv` (optional): caller-provided Tinv (w x w, ld ldt) instead of the one
// built from Y and tau (apply_block_reflector_*, qrblock.py:103-119).
static int cwy_apply(dcsvd_ctx* h, cudaStream_t st, char side, bool trans, bool ytrans, const double* Y,
                     long long ldy, const double* tau, int w, long long rows_y, double* C, long long ldc,
                     long long c_other, double* scratch, const double* utinv = nullptr, long long ldt = 0,
                     const double* utop = nullptr) {
  if (rows_y <= 0 || c_other <= 0 || w <= 0) return 0;
  // split-K so that Z's tiles x S fill the GPU
  if (w > kCwyMaxW) return set_error(h, DCSVD_EINVAL, "CWY block width %d exceeds %d", w, kCwyMaxW);
  const int S = cwy_split(h->sms, w, c_other, rows_y);
  const int SG = utinv ? 1 : cwy_gsplit(h->sms, w, rows_y, S);
  double* Zp = scratch;
  double* Gp = Zp + (size_t)S * w * c_other;
  double* Top = Gp + (size_t)std::max(S, kMaxGSplit) * w * w;
  double* TinvT = Top + (size_t)w * w;
  // slices of a multiple of 16 rows: every slice base keeps the operands' 16-byte alignment
  const long long kchunk = (((rows_y + S - 1) / S) + 15) & ~15LL;
  const long long gchunk = (((rows_y + SG - 1) / SG) + 15) & ~15LL;
  // one descriptor each, split over K inside the kernel (slice s -> partial s)
  GemmBatch zb, gb;
  zb.count = 1;
  gb.count = 1;
  zb.ksplit = S;
  gb.ksplit = SG;
  zb.kchunk = (int)kchunk;
  gb.kchunk = (int)gchunk;
  zb.cslice = (long long)w * c_other;
  gb.cslice = (long long)w * w;
  {
    GemmDesc z, g;
    z.acol = nullptr; z.ccol = nullptr; z.alpha = 1.0; z.beta = 0.0;
    g = z;
    if (side == 'L') {
      z.m = w; z.n = (int)c_other; z.k = (int)rows_y;
      z.A = Y; z.lda = ldy;
      z.B = C; z.ldb = ldc;
      z.C = Zp; z.ldc = w;
    } else {
      z.m = (int)c_other; z.n = w; z.k = (int)rows_y;
      z.A = C; z.lda = ldc;
      z.B = Y; z.ldb = ldy;
      z.C = Zp; z.ldc = c_other;
    }
    g.m = w; g.n = w; g.k = (int)rows_y;
    g.A = Y; g.lda = ldy; g.B = Y; g.ldb = ldy;
    g.C = Gp; g.ldc = w;
    zb.d[0] = z;
    gb.d[0] = g;
  }
  int rc;
  if (side == 'L') rc = gemm_launch_batch(st, /*ta=*/!ytrans, /*tb=*/false, zb);
  else rc = gemm_launch_batch(st, false, /*tb=*/ytrans, zb);
  if (rc) return rc;
  if (utop) {
    Top = const_cast<double*>(utop);  // op(T) precomputed by the caller (ormbr_run)
  } else if (utinv) {
    copy_tinv_kernel<<<(w * w + 255) / 256, 256, 0, st>>>(utinv, ldt, w, TinvT, h->d_err);
  } else {
    rc = gemm_launch_batch(st, !ytrans, ytrans, gb);
    if (rc) return rc;
    cwy_tinv_build_kernel<<<(w * w + 255) / 256, 256, 0, st>>>(Gp, SG, w, tau, TinvT, h->d_err);
  }
  if (!utop) {
    note_launch();
    rc = tinv_solve_launch(st, TinvT, w, trans, Top);
    if (rc) return rc;
  }
  const long long zc = (long long)w * c_other;
  if (S > 1) {
    if (S >= 16 && zc <= (1 << 16))
      splitk_reduce_warp_kernel<<<(unsigned)((zc * 32 + 255) / 256), 256, 0, st>>>(Zp, zc, S);
    else
      splitk_reduce_kernel<<<grid_for(zc), 256, 0, st>>>(Zp, zc, S);
    note_launch();
  }
  // X = op(T) Z  (left, w x c_other) or Z op(T) (right, c_other x w); in place
  // is not possible, so write X into the second partial slot (or a tail slot).
  double* X = (S > 1) ? Zp + zc : TinvT + (size_t)w * w;  // scratch tail when S == 1
  GemmDesc xd;
  xd.acol = nullptr; xd.ccol = nullptr; xd.alpha = 1.0; xd.beta = 0.0;
  if (side == 'L') {
    xd.m = w; xd.n = (int)c_other; xd.k = w;
    xd.A = Top; xd.lda = w; xd.B = Zp; xd.ldb = w; xd.C = X; xd.ldc = w;
  } else {
    xd.m = (int)c_other; xd.n = w; xd.k = w;
    xd.A = Zp; xd.lda = c_other; xd.B = Top; xd.ldb = w; xd.C = X; xd.ldc = c_other;
  }
  rc = gemm_launch(st, false, false, xd);
  if (rc) return rc;
  GemmDesc ud;
  ud.acol = nullptr; ud.ccol = nullptr; ud.alpha = -1.0; ud.beta = 1.0;
  if (side == 'L') {
    // C -= Y X : op(A) = Y
    ud.m = (int)rows_y; ud.n = (int)c_other; ud.k = w;
    ud.A = Y; ud.lda = ldy; ud.B = X; ud.ldb = w; ud.C = C; ud.ldc = ldc;
    return gemm_launch(st, /*ta=*/ytrans, false, ud);
  }
  // C -= X Y^T : op(B) = Y^T
  ud.m = (int)c_other; ud.n = (int)rows_y; ud.k = w;
  ud.A = X; ud.lda = c_other; ud.B = Y; ud.ldb = ldy; ud.C = C; ud.ldc = ldc;
  return gemm_launch(st, false, /*tb=*/!ytrans, ud);
}

static size_t cwy_total_scratch(int sms, long long rows_y, long long c_other, int w) {
  // Z partials + G partials + Top + Tinv + X (when S == 1)
  return cwy_scratch_doubles(sms, rows_y, c_other, w) + (size_t)w * c_other + 64;
}

// ---------------------------------------------------------------------------
// GEQR2 panel (qrblock.py:51-71): cooperative, each CTA keeps its row slab of
// the m x w panel in shared memory (ld = slab rows).
struct Geqr2Args {
  double* A;
  long long lda;
  int m, w;
  double* tau;
  double* part;    // 2 x G x 64 partials (double-buffered by column parity)
  double* rowbuf;  // 2 x 64: the pivot row of the current / next column
  unsigned* bar;
  int R1;        // rows per CTA
  unsigned long long* tlog;
};

constexpr int kGeqr2Threads = 512;
constexpr int kGeqr2Warps = kGeqr2Threads / 32;
static_assert(kGeqr2Warps * 4 >= 64, "four partial slots per warp cover a 64-wide panel");
extern unsigned long long* g_labrd_tlog;  // debug phase timestamps (gebrd.cu)

// debug: per-CTA timestamps of columns 5 and 6 (4 marks each, 256 slots per mark)
__device__ __forceinline__ void tmark_g(const Geqr2Args& a, int j, int m) {
  if (a.tlog && threadIdx.x == 0 && (j == 5 || j == 6)) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.tlog[((j == 6 ? 4 : 0) + m) * 256 + blockIdx.x] = t;
    a.tlog[(8 + (j == 6 ? 4 : 0) + m) * 256 + blockIdx.x] = clock64();
  }
}

// One grid barrier per column.  With v = [1; x/den] (LARFG, densecore.py:
// 114-128) the reflector's w_t = v^T a[:, t] = a[j, t] + (sum_{r>j} x_r a[r, t]) / den,
// so the norm of x and the cross sums sum_{r>j} x_r a[r, t] are reduced in the
// same phase, before den is known.  Each CTA keeps its R1-row slab of the
// panel in shared memory; the owner of row j+1 publishes that row (double
// buffered, like the partials) for everyone's w.
// SM = false: panels too tall for shared memory keep each CTA's row slab in
// place in global memory (same arithmetic, L2-resident for tall-skinny panels).
template <bool SM>
__global__ void __launch_bounds__(kGeqr2Threads, 1) geqr2_coop_kernel(Geqr2Args a) {
  extern __shared__ double smem_slab[];  // R1 x w when SM
  __shared__ double sh_w[64];
  __shared__ double sh_row[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int g = blockIdx.x, G = gridDim.x;
  const int r0 = g * a.R1, r1 = min(a.m, r0 + a.R1), nr = max(0, r1 - r0);
  const int w = a.w;
  double* slab = SM ? smem_slab : a.A + r0;
  const long long R1 = SM ? (long long)a.R1 : a.lda;  // slab column stride
  unsigned epoch = 0;
  if (SM) {
    for (int idx = tid; idx < nr * w; idx += blockDim.x) {
      const int rr = idx % nr, t = idx / nr;
      slab[rr + t * R1] = a.A[(r0 + rr) + (long long)t * a.lda];
    }
  }
  __syncthreads();
  // partials of column c over this CTA's rows r > c into buffer (c & 1):
  // slot 0 = sum x^2, slot t = sum x * a[r, t] (t > c); row c published.
  // Slot-major (part[slot * G + cta]) so one warp reads a slot's G <= 160
  // partials with five coalesced loads per lane.
  auto partials = [&](int c) {
    double* part = a.part + (size_t)(c & 1) * G * 64 + g;
    const int lo = max(0, c + 1 - r0);  // first local row > c
    for (int t = c + warp; t < w; t += nw) {  // warp per slot (t == c: the norm)
      double s = 0.0;
      for (int rr = lo + lane; rr < nr; rr += 32) s += slab[rr + c * R1] * slab[rr + t * R1];
      s = warp_sum(s);
      if (lane == 0) part[(size_t)(t == c ? 0 : t) * G] = s;
    }
    if (c >= r0 && c < r1)
      for (int t = c + tid; t < w; t += blockDim.x) a.rowbuf[(c & 1) * 64 + t] = slab[(c - r0) + t * R1];
  };
  partials(0);
  grid_barrier(a.bar, G, epoch);
  for (int j = 0; j < w; ++j) {
    const double* part = a.part + (size_t)(j & 1) * G * 64;
    const double* rowj = a.rowbuf + (j & 1) * 64;
    // Every load of this column is issued before any is consumed: the
    // partials of up to four slots per warp (w <= 64, 16 warps) and the
    // pivot row -- one L2 round trip after the barrier instead of one per
    // strided load.
    tmark_g(a, j, 0);
    double v[4][5];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = j + warp + kGeqr2Warps * q;
      const double* ps = part + (size_t)(t == j ? 0 : t) * G;
#pragma unroll
      for (int i = 0; i < 5; ++i) v[q][i] = (t < w && lane + 32 * i < G) ? ps[lane + 32 * i] : 0.0;
    }
    const double rowv = (tid >= j && tid < w) ? rowj[tid] : 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = j + warp + kGeqr2Warps * q;
      const double s = warp_sum(((v[q][0] + v[q][1]) + (v[q][2] + v[q][3])) + v[q][4]);
      if (t < w && lane == 0) sh_w[t] = s;
    }
    if (tid >= j && tid < w) sh_row[tid] = rowv;
    __syncthreads();
    tmark_g(a, j, 1);
    const double alpha = sh_row[j];
    double tau, beta;
    {
      const double xn = sqrt(sh_w[j]);
      if (xn == 0.0) { tau = 0.0; beta = alpha; }
      else { beta = -copysign(hypot(alpha, xn), alpha); tau = (beta - alpha) / beta; }
    }
    const double den = alpha - beta;
    if (g == 0 && tid == 0) a.tau[j] = tau;
    __syncthreads();  // everyone has read sh_w[j]
    if (tid > j && tid < w) sh_w[tid] = tau != 0.0 ? sh_row[tid] + sh_w[tid] / den : 0.0;  // w_t
    // column j of the slab: beta on row j, essential part x / den below
    for (int rr = tid; rr < nr; rr += blockDim.x) {
      const int r = r0 + rr;
      if (r == j) slab[rr + j * R1] = beta;
      else if (r > j && tau != 0.0) slab[rr + j * R1] /= den;
    }
    __syncthreads();
    if (tau != 0.0 && j + 1 < w) {  // a[r, t] -= tau v_r w_t, rows r >= j, columns t > j
      const int lo = max(0, j - r0);
      for (int t = j + 1 + warp; t < w; t += nw) {
        const double tw = tau * sh_w[t];
        for (int rr = lo + lane; rr < nr; rr += 32) {
          const int r = r0 + rr;
          const double v = r == j ? 1.0 : slab[rr + j * R1];
          slab[rr + t * R1] -= v * tw;
        }
      }
      __syncthreads();
    }
    tmark_g(a, j, 2);
    if (j + 1 < w) {
      partials(j + 1);
      tmark_g(a, j, 3);
      grid_barrier(a.bar, G, epoch);
    }
  }
  if (SM) {
    for (int idx = tid; idx < nr * w; idx += blockDim.x) {
      const int rr = idx % nr, t = idx / nr;
      a.A[(r0 + rr) + (long long)t * a.lda] = slab[rr + t * R1];
    }
  }
}

static int geqr2_launch(dcsvd_ctx* h, cudaStream_t st, double* A, long long lda, int m, int w, double* tau,
                        double* part) {
  int G = h->sms;
  int R1 = (m + G - 1) / G;
  if (R1 < 32) {
    R1 = 32;
    G = (m + R1 - 1) / R1;
  }
  const bool in_smem = sizeof(double) * (size_t)R1 * w <= 200 * 1024;
  const size_t smem = in_smem ? sizeof(double) * (size_t)R1 * w : 0;
  if (G > 160 || w > 64) return set_error(h, DCSVD_EINVAL, "QR panel kernel supports <= 160 CTAs and 64 columns");
  DC_CUDA_TRY((cudaError_t)func_attr(geqr2_coop_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  DC_CUDA_TRY(cudaMemsetAsync(h->d_bar, 0, sizeof(unsigned), st));
  Geqr2Args a;
  a.A = A; a.lda = lda; a.m = m; a.w = w; a.tau = tau; a.part = part; a.rowbuf = part + (size_t)2 * G * 64;
  a.bar = h->d_bar; a.R1 = R1; a.tlog = g_labrd_tlog;
  void* args[] = {&a};
  void* fn = in_smem ? (void*)geqr2_coop_kernel<true> : (void*)geqr2_coop_kernel<false>;
  DC_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kGeqr2Threads), args, smem, st));
  note_launch();
  return 0;
}

int geqrf_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda, double* tau,
              int nb) {
  if (n < 1) return set_error(h, DCSVD_EINVAL, "matrix must have at least one column");
  if (m < n) return set_error(h, DCSVD_EINVAL, "QR factorization requires m >= n, got %lldx%lld", m, n);
  if (nb < 1) return set_error(h, DCSVD_EINVAL, "block width must be >= 1, got %d", nb);
  if (nb > 64) nb = 64;  // panel width of the GPU kernel; wider blocks give the same reflectors
  // Two-level blocking (same reflectors, LAPACK dgeqrf order): nb-wide panels
  // are factored and applied inside an outer block of W = nb*ceil(128/nb)
  // columns; the far trailing matrix then takes one W-wide CWY block (DMMA
  // GEMMs with K = W instead of K = nb).
  const int W = g_qr_outer > 0 ? std::min(kCwyMaxW, std::max(nb, g_qr_outer / nb * nb))
                               : std::min(kCwyMaxW, nb * std::max(1, kCwyMaxW / nb));
  const size_t need = pool_bytes((size_t)m * W, 8) + pool_bytes((size_t)h->sms * 128 + 128, 8) +
                      pool_bytes(cwy_total_scratch(h->sms, m, n, W), 8);
  int rc = pool_reserve(h, 0, need, st);
  if (rc) return rc;
  double* Y = pool_take<double>(h, 0, (size_t)m * W);
  double* part = pool_take<double>(h, 0, (size_t)h->sms * 128 + 128);
  double* scr = pool_take<double>(h, 0, cwy_total_scratch(h->sms, m, n, W));
  for (long long off = 0; off < n; off += W) {
    const int wW = (int)std::min<long long>(W, n - off);
    for (int ip = 0; ip < wW; ip += nb) {
      const int w = std::min(nb, wW - ip);
      const long long o = off + ip;
      const long long rows = m - o;
      rc = geqr2_launch(h, st, A + o + o * lda, lda, (int)rows, w, tau + o, part);
      if (rc) return rc;
      if (ip + w < wW) {
        build_y_kernel<<<grid_for(rows * w), 256, 0, st>>>(0, A + o + o * lda, lda, tau + o, (int)rows, w, Y);
        note_launch();
        rc = cwy_apply(h, st, 'L', /*trans=*/true, false, Y, rows, tau + o, w, rows, A + o + (o + w) * lda, lda,
                       wW - ip - w, scr);
        if (rc) return rc;
      }
    }
    if (off + wW < n) {
      const long long rows = m - off;
      build_y_kernel<<<grid_for(rows * wW), 256, 0, st>>>(0, A + off + off * lda, lda, tau + off, (int)rows, wW, Y);
      note_launch();
      rc = cwy_apply(h, st, 'L', /*trans=*/true, false, Y, rows, tau + off, wW, rows, A + off + (off + wW) * lda, lda,
                     n - off - wW, scr);
      if (rc) return rc;
    }
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

__global__ void eye_kernel(double* Q, long long ldq, long long m, long long k) {
  const long long total = m * k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = idx % m, j = idx / m;
    Q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
  }
}

int orgqr_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long nrefl, long long k, const double* A,
              long long lda, const double* tau, double* Q, long long ldq, int nb) {
  if (k < 1 || k > m) return set_error(h, DCSVD_EINVAL, "need 1 <= k <= %lld columns of Q, got %lld", m, k);
  if (nb < 1) return set_error(h, DCSVD_EINVAL, "block width must be >= 1, got %d", nb);
  if (nb > kCwyMaxW) nb = kCwyMaxW;  // T^-1 = triu(Y^T Y, 1) + diag(1/tau) is exact for any grouping
  const size_t need = pool_bytes((size_t)m * nb, 8) + pool_bytes(cwy_total_scratch(h->sms, m, k, nb), 8);
  int rc = pool_reserve(h, 0, need, st);
  if (rc) return rc;
  double* Y = pool_take<double>(h, 0, (size_t)m * nb);
  double* scr = pool_take<double>(h, 0, cwy_total_scratch(h->sms, m, k, nb));
  eye_kernel<<<grid_for(m * k), 256, 0, st>>>(Q, ldq, m, k);
  note_launch();
  long long last = ((nrefl - 1) / nb) * nb;
  for (long long off = last; off >= 0; off -= nb) {
    const int w = (int)std::min<long long>(nb, nrefl - off);
    const long long rows = m - off;
    if (off >= k) continue;  // columns >= off are all that change; none exist
    build_y_kernel<<<grid_for(rows * w), 256, 0, st>>>(0, A + off + off * lda, lda, tau + off, (int)rows, w, Y);
    note_launch();
    // columns < off of Q stay exactly e_i (zero in rows >= off)
    rc = cwy_apply(h, st, 'L', false, false, Y, rows, tau + off, w, rows, Q + off + off * ldq, ldq, k - off, scr);
    if (rc) return rc;
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// op(T) of every full-width block depends only on the packed reflectors, so
// ormbr builds all blocks' Y once and computes G_b = Y_b^T Y_b (batched DMMA
// GEMM, kPreGSplit K-slices), Tinv_b and op(T_b) in one launch each before the
// apply loop, instead of three launches per block on the loop's critical path.
constexpr int kPreGSplit = 4;
constexpr size_t kOrmbrPreMaxBytes = size_t(4) << 30;  // resident Y of all blocks (n ~ 32 000)
int g_ormbr_pre = 1;  // debug: 0 = per-block T inside the apply loop

// ormbr_run = ormbr_prepare (pool, Y of every block, batched op(T); depends only
// on the packed reflectors) + ormbr_apply (the block loop on C).  The driver
// runs the prepare step of both sides on a side stream while BDC runs.
int ormbr_prepare(dcsvd_ctx* h, cudaStream_t st, char vect, bool trans, long long m, long long n, const double* A,
                  long long lda, const double* tau, long long c_rows, long long c_cols, int nb, OrmbrPlan& P) {
  if (nb < 1) return set_error(h, DCSVD_EINVAL, "block width must be >= 1, got %d", nb);
  if (nb > kCwyMaxW) nb = kCwyMaxW;  // same product, grouped in 128-wide compact-WY blocks
  if (vect != 'Q' && vect != 'P') return set_error(h, DCSVD_EINVAL, "vect must be 'Q' or 'P'");
  const bool isq = vect == 'Q';
  if (isq && c_rows != m) return set_error(h, DCSVD_EINVAL, "C has %lld rows, sequence acts on %lld", c_rows, m);
  if (!isq && c_cols != n) return set_error(h, DCSVD_EINVAL, "C has %lld columns, sequence acts on %lld", c_cols, n);
  P = OrmbrPlan();
  P.isq = isq; P.trans = trans; P.nb = nb; P.A = A; P.lda = lda; P.tau = tau;
  P.c_rows = c_rows; P.c_cols = c_cols;
  P.count = isq ? n : (n > 0 ? n - 1 : 0);  // reflectors
  P.rows0 = isq ? m : n - 1;                 // rows of block 0's reflectors
  const long long c_other = isq ? c_cols : c_rows;
  P.nblk = (P.count + nb - 1) / nb;
  if (P.nblk == 0) return 0;
  P.yoff.assign(P.nblk + 1, 0);
  for (long long b = 0; b < P.nblk; ++b) P.yoff[b + 1] = P.yoff[b] + (P.rows0 - b * nb) * nb;
  // every block's Y stays resident (n^2/2 doubles per side): above kOrmbrPreMaxBytes
  // (inputs of tens of GB) the blocks are built one at a time into one buffer
  // and op(T) is formed per block inside cwy_apply, as before the precompute
  P.pre = g_ormbr_pre && (size_t)P.yoff[P.nblk] * sizeof(double) <= kOrmbrPreMaxBytes;
  if (!P.pre) std::fill(P.yoff.begin(), P.yoff.end(), 0LL);
  const long long ylen = P.pre ? P.yoff[P.nblk] : P.rows0 * nb;
  P.nfull = P.pre ? P.count / nb : 0;  // blocks with precomputed op(T)
  const size_t ww = (size_t)nb * nb;
  const size_t need = pool_bytes((size_t)ylen, 8) + pool_bytes(cwy_total_scratch(h->sms, P.rows0, c_other, nb), 8) +
                      (P.nfull ? pool_bytes((size_t)P.nfull * kPreGSplit * ww, 8) + 2 * pool_bytes((size_t)P.nfull * ww, 8)
                               : 0);
  int rc = pool_reserve(h, 0, need, st);
  if (rc) return rc;
  P.Yall = pool_take<double>(h, 0, (size_t)ylen);
  P.scr = pool_take<double>(h, 0, cwy_total_scratch(h->sms, P.rows0, c_other, nb));
  double* Gall = P.nfull ? pool_take<double>(h, 0, (size_t)P.nfull * kPreGSplit * ww) : nullptr;
  double* Tinv = P.nfull ? pool_take<double>(h, 0, (size_t)P.nfull * ww) : nullptr;
  P.Top = P.nfull ? pool_take<double>(h, 0, (size_t)P.nfull * ww) : nullptr;
  if (!P.pre) return 0;
  for (long long bi = 0; bi < P.nblk; ++bi) ormbr_build_y(st, P, bi);
  if (P.nfull) {
    for (long long b0 = 0; b0 < P.nfull; b0 += kMaxBatchDesc) {
      GemmBatch gb;
      gb.count = (int)std::min<long long>(kMaxBatchDesc, P.nfull - b0);
      gb.ksplit = kPreGSplit;
      gb.kchunk = (int)((((P.rows0 - b0 * nb + kPreGSplit - 1) / kPreGSplit) + 15) & ~15LL);
      gb.cslice = (long long)ww;
      for (int i = 0; i < gb.count; ++i) {
        const long long bi = b0 + i;
        const long long rows = P.rows0 - bi * nb;
        GemmDesc g;
        g.acol = nullptr; g.ccol = nullptr; g.alpha = 1.0; g.beta = 0.0;
        g.m = nb; g.n = nb; g.k = (int)rows;
        g.A = P.Yall + P.yoff[bi]; g.B = P.Yall + P.yoff[bi];
        g.lda = g.ldb = isq ? rows : nb;
        g.C = Gall + (size_t)bi * kPreGSplit * ww; g.ldc = nb;
        gb.d[i] = g;
      }
      rc = isq ? gemm_launch_batch(st, true, false, gb) : gemm_launch_batch(st, false, true, gb);
      if (rc) return rc;
    }
    cwy_tinv_build_kernel<<<dim3((unsigned)((ww + 255) / 256), (unsigned)P.nfull), 256, 0, st>>>(
        Gall, kPreGSplit, nb, tau, Tinv, h->d_err, (long long)kPreGSplit * ww, nb);
    note_launch();
    rc = tinv_solve_launch(st, Tinv, nb, trans, P.Top, (int)P.nfull);
    if (rc) return rc;
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

void ormbr_build_y(cudaStream_t st, const OrmbrPlan& P, long long bi) {
  const long long off = bi * P.nb, rows = P.rows0 - bi * P.nb;
  const int w = (int)std::min<long long>(P.nb, P.count - off);
  const double* src = P.isq ? P.A + off + off * P.lda : P.A + off + (off + 1) * P.lda;
  build_y_kernel<<<grid_for(rows * w), 256, 0, st>>>(P.isq ? 0 : 1, src, P.lda, P.tau + off, (int)rows, w,
                                                    P.Yall + P.yoff[bi]);
  note_launch();
}

int ormbr_apply(dcsvd_ctx* h, cudaStream_t st, const OrmbrPlan& P, double* C, long long ldc) {
  const int nb = P.nb;
  const size_t ww = (size_t)nb * nb;
  int rc = 0;
  for (long long b = 0; b < P.nblk; ++b) {
    // 'Q': U1^T front-to-back, U1 back-to-front; 'P': V1^T back-to-front, V1 front-to-back
    const long long bi = (P.isq == P.trans) ? b : P.nblk - 1 - b;
    const long long off = bi * nb, rows = P.rows0 - bi * nb;
    const int w = (int)std::min<long long>(nb, P.count - off);
    const double* utop = bi < P.nfull ? P.Top + (size_t)bi * ww : nullptr;
    if (!P.pre) ormbr_build_y(st, P, bi);  // yoff == 0: the single block buffer
    if (P.isq)
      rc = cwy_apply(h, st, 'L', P.trans, false, P.Yall + P.yoff[bi], rows, P.tau + off, w, rows, C + off, ldc,
                     P.c_cols, P.scr, nullptr, 0, utop);
    else
      rc = cwy_apply(h, st, 'R', P.trans, true, P.Yall + P.yoff[bi], w, P.tau + off, w, rows, C + (off + 1) * ldc,
                     ldc, P.c_rows, P.scr, nullptr, 0, utop);
    if (rc) return rc;
  }
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

int ormbr_run(dcsvd_ctx* h, cudaStream_t st, char vect, bool trans, long long m, long long n, const double* A,
              long long lda, const double* tau, double* C, long long c_rows, long long c_cols, long long ldc,
              int nb) {
  OrmbrPlan P;
  int rc = ormbr_prepare(h, st, vect, trans, m, n, A, lda, tau, c_rows, c_cols, nb, P);
  if (rc || P.nblk == 0) return rc;
  return ormbr_apply(h, st, P, C, ldc);
}

// ---------------------------------------------------------------------------
// Standalone pieces of the reference API (qrblock.py / densecore.py).

// build_tinv (qrblock.py:90-100): Tinv = triu(Y^T Y, 1) + diag(1/tau).
int build_tinv_run(dcsvd_ctx* h, cudaStream_t st, long long rows, int w, const double* Y, long long ldy,
                   const double* tau, double* Tinv, long long ldt) {
  if (w < 1 || w > kCwyMaxW) return set_error(h, DCSVD_EINVAL, "block width must be 1..%d, got %d", kCwyMaxW, w);
  int rc = pool_reserve(h, 0, pool_bytes((size_t)2 * w * w, 8), st);
  if (rc) return rc;
  double* G = pool_take<double>(h, 0, (size_t)w * w);
  double* T = pool_take<double>(h, 0, (size_t)w * w);
  GemmDesc g;
  g.m = w; g.n = w; g.k = (int)rows;
  g.A = Y; g.lda = ldy; g.acol = nullptr; g.B = Y; g.ldb = ldy;
  g.C = G; g.ldc = w; g.ccol = nullptr; g.alpha = 1.0; g.beta = 0.0;
  if (rows > 0) {
    rc = gemm_launch(st, true, false, g);
    if (rc) return rc;
  } else {
    DC_CUDA_TRY(cudaMemsetAsync(G, 0, sizeof(double) * w * w, st));
  }
  cwy_tinv_build_kernel<<<(w * w + 255) / 256, 256, 0, st>>>(G, 1, w, tau, T, h->d_err);
  note_launch();
  DC_CUDA_TRY(cudaMemcpy2DAsync(Tinv, sizeof(double) * ldt, T, sizeof(double) * w, sizeof(double) * w, w,
                                cudaMemcpyDeviceToDevice, st));
  return 0;
}

// apply_block_reflector_left/right (qrblock.py:103-119) with a given (Y, Tinv).
int block_reflector_run(dcsvd_ctx* h, cudaStream_t st, char side, bool trans, long long rows_y, int w, const double* Y,
                        long long ldy, const double* Tinv, long long ldt, double* C, long long ldc, long long c_other) {
  if (w < 1 || w > kCwyMaxW) return set_error(h, DCSVD_EINVAL, "block width must be 1..%d, got %d", kCwyMaxW, w);
  const size_t need = pool_bytes(cwy_total_scratch(h->sms, rows_y, c_other, w), 8);
  int rc = pool_reserve(h, 0, need, st);
  if (rc) return rc;
  double* scr = pool_take<double>(h, 0, cwy_total_scratch(h->sms, rows_y, c_other, w));
  return cwy_apply(h, st, side, trans, false, Y, ldy, nullptr, w, rows_y, C, ldc, c_other, scr, Tinv, ldt);
}

// geqrf_panel (qrblock.py:51-71): unblocked QR of one tall panel (w <= 64).
int geqr2_run(dcsvd_ctx* h, cudaStream_t st, long long m, int w, double* A, long long lda, double* tau) {
  if (m < w) return set_error(h, DCSVD_EINVAL, "panel must be tall, got %lldx%d", m, w);
  if (w < 1 || w > 64) return set_error(h, DCSVD_EINVAL, "GPU panel width must be 1..64, got %d", w);
  int rc = pool_reserve(h, 0, pool_bytes((size_t)h->sms * 128 + 128, 8), st);
  if (rc) return rc;
  double* part = pool_take<double>(h, 0, (size_t)h->sms * 128 + 128);
  return geqr2_launch(h, st, A, lda, (int)m, w, tau, part);
}

// householder_generate (densecore.py:114-128): tau, beta, essential = x/(alpha-beta).
__global__ void larfg_kernel(int n, const double* __restrict__ alpha_p, const double* __restrict__ x, long long incx,
                             double* __restrict__ out /* tau, beta */, double* __restrict__ ess) {
  __shared__ double sh[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += x[i * incx] * x[i * incx];
  v = block_sum(v, sh);
  const double alpha = *alpha_p;
  const double xn = sqrt(v);
  double tau = 0.0, beta = alpha;
  if (xn != 0.0) {
    beta = -copysign(hypot(alpha, xn), alpha);
    tau = (beta - alpha) / beta;
  }
  const double den = alpha - beta;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ess[i] = xn != 0.0 ? x[i * incx] / den : x[i * incx];
  if (threadIdx.x == 0) {
    out[0] = tau;
    out[1] = beta;
  }
}

int larfg_run(dcsvd_ctx* h, cudaStream_t st, long long n, const double* alpha, const double* x, long long incx,
              double* out, double* ess) {
  larfg_kernel<<<1, 512, 0, st>>>((int)n, alpha, x, incx, out, ess);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// givens_generate (densecore.py:131-140) for a batch of (a, b) pairs: out = (c, s, r).
__global__ void lartg_kernel(long long cnt, const double* __restrict__ a, const double* __restrict__ b, double* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  double c, s, r;
  lartg(a[i], b[i], c, s, r);
  out[3 * i + 0] = c;
  out[3 * i + 1] = s;
  out[3 * i + 2] = r;
}

int lartg_run(dcsvd_ctx* h, cudaStream_t st, long long cnt, const double* a, const double* b, double* out) {
  if (cnt <= 0) return 0;
  lartg_kernel<<<(int)((cnt + 255) / 256), 256, 0, st>>>(cnt, a, b, out);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// triangular_solve (densecore.py:143-171), T upper n x n.  left: B <- T^-1 B
// (or T^-T B), thread per column of B; right: B <- B T^-1 (or B T^-T), thread
// per row of B.
__global__ void trsm_kernel(int n, const double* __restrict__ T, long long ldt, double* __restrict__ B, long long ldb,
                            long long other, int right, int trans, int* err) {
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= other) return;
  // element stride along the solved dimension and base of this vector
  double* x = right ? B + v : B + v * ldb;
  const long long inc = right ? ldb : 1;
  // left, !trans: T x = b (back substitution);  left, trans: T^T x = b (forward)
  // right, !trans: x^T T = b^T -> T^T x = b (forward); right, trans: x^T T^T = b^T -> T x = b (back)
  const bool upper_solve = (right != 0) == (trans != 0);
  if (upper_solve) {
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i * inc];
      for (int l = i + 1; l < n; ++l) s -= T[i + l * ldt] * x[l * inc];
      const double dg = T[i + i * ldt];
      if (dg == 0.0) { raise_dev(err, kDevSingularT); return; }
      x[i * inc] = s / dg;
    }
  } else {
    for (int i = 0; i < n; ++i) {
      double s = x[i * inc];
      for (int l = 0; l < i; ++l) s -= T[l + i * ldt] * x[l * inc];
      const double dg = T[i + i * ldt];
      if (dg == 0.0) { raise_dev(err, kDevSingularT); return; }
      x[i * inc] = s / dg;
    }
  }
}

int trsm_run(dcsvd_ctx* h, cudaStream_t st, int n, const double* T, long long ldt, double* B, long long ldb,
             long long other, bool right, bool trans) {
  if (other <= 0 || n <= 0) return 0;
  trsm_kernel<<<(int)((other + 127) / 128), 128, 0, st>>>(n, T, ldt, B, ldb, other, right ? 1 : 0, trans ? 1 : 0,
                                                          h->d_err);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace dc
