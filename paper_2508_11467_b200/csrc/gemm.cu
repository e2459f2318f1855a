// DMMA GEMM kernels (see gemm.cuh).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <unordered_map>
#include <vector>

#include "ctx.cuh"
#include "gemm.cuh"
#include "launch.cuh"

namespace dc {

extern thread_local dcsvd_ctx* t_cur;  // api.cu: handle of the current API call

int g_gemm_route = 0;  // debug: 0 default, 1 no streaming rank-k, 2 also 64x128 C-prefetch tiles, 5 8-byte staging

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__constant__ int g_rankk_prefetch = 1;
__constant__ int g_bulk_a = 1;  // rank-k A tiles by TMA bulk copies (debug: 0 = cp.async)
int set_rankk_bulk(int on) { return cudaMemcpyToSymbol(g_bulk_a, &on, sizeof(int)) == cudaSuccess ? 0 : -1; }
int set_rankk_prefetch(int on) {  // debug: L2 prefetch of the next C tile in the rank-k kernel
  return cudaMemcpyToSymbol(g_rankk_prefetch, &on, sizeof(int)) == cudaSuccess ? 0 : -1;
}
// TMA bulk copies (cp.async.bulk, async proxy) completing on an mbarrier.
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool TA, bool TB, int BM, int BN, int BK_, int WARPS_M, int WARPS_N, int STAGES_>
struct GemmCfg {
  static constexpr int BK = BK_;
  static constexpr int STAGES = STAGES_;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  // A stage: TA ? [BM][BK+4] : [BK][BM+4];  B stage: TB ? [BK][BN+4] : [BN][BK+4]
  // (row pitch = 4 mod 16 doubles -> conflict-free m8n8k4 fragment reads)
  static constexpr int LDA_S = TA ? (BK + 4) : (BM + 4);
  static constexpr int LDB_S = TB ? (BN + 4) : (BK + 4);
  static constexpr int A_ELEMS = TA ? BM * (BK + 4) : BK * (BM + 4);
  static constexpr int B_ELEMS = TB ? BK * (BN + 4) : BN * (BK + 4);
  static constexpr int C_ELEMS = BM * BN;  // optional C-tile prefetch (beta != 0)
  static constexpr int SMEM_BYTES = STAGES * (A_ELEMS + B_ELEMS) * 8;
  // pairs of consecutive doubles along the contiguous global dimension
  static constexpr int A_PAIRS = BM * BK / 2, B_PAIRS = BN * BK / 2;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}

// Copy the pair (x, x+1) along the contiguous dimension; `valid` in {0,1,2}.
__device__ __forceinline__ void copy_pair(double* dst, const double* src, int valid, bool vec) {
  if (vec) {
    cp_async16(dst, src, valid * 8);
  } else {
    cp_async8(dst, src, valid > 0);
    cp_async8(dst + 1, valid > 1 ? src + 1 : src, valid > 1);
  }
}

template <bool TA, bool TB, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int MINB, bool PFC,
          bool VEC, bool GATHER>
__global__ void __launch_bounds__(32 * WARPS_M * WARPS_N, MINB)
    dgemm_kernel(GemmBatch batch, const GemmDesc* __restrict__ ddesc) {
  // GATHER (device descriptors of the BDC merges): A columns gathered and C
  // columns scattered through index lists; compiled away otherwise.
  constexpr bool gather = GATHER;
  using Cfg = GemmCfg<TA, TB, BM, BN, BK, WARPS_M, WARPS_N, STAGES>;
  constexpr int THREADS = Cfg::THREADS;
  const int ks = ddesc ? 1 : batch.ksplit;
  GemmDesc P = ddesc ? ddesc[blockIdx.z] : batch.d[blockIdx.z / ks];
  if (ks > 1) {  // split-K slice of this descriptor
    const int sl = blockIdx.z % ks;
    const long long k0 = (long long)sl * batch.kchunk;
    P.k = (int)max(0LL, min((long long)batch.kchunk, (long long)P.k - k0));
    P.A += TA ? k0 : k0 * P.lda;
    P.B += TB ? k0 * P.ldb : k0;
    P.C += sl * batch.cslice;
  }
  const int M = P.m, N = P.n, K = P.k;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  if (m0 >= M || n0 >= N) return;

  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * Cfg::A_ELEMS;
  const double* __restrict__ A = P.A;
  const double* __restrict__ B = P.B;
  const long long lda = P.lda, ldb = P.ldb;
  const int* __restrict__ acol = P.acol;
  const int tid = threadIdx.x;
  // VEC (host-checked: 16-byte aligned bases, even leading dimensions) selects
  // 16-byte cp.async for every pair at compile time.
  // GATHER (device descriptors): alignment is known only here, per descriptor
  // (uniform per CTA): 16-byte copies when the base and leading dimension allow.
  const bool vecA = VEC || (gather && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((lda & 1) == 0));
  const bool vecB = VEC || (gather && ((reinterpret_cast<uintptr_t>(B) & 15) == 0) && ((ldb & 1) == 0));

  auto load_tile = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * Cfg::A_ELEMS;
    double* bs = Bs + stage * Cfg::B_ELEMS;
#pragma unroll
    for (int p = tid; p < Cfg::A_PAIRS; p += THREADS) {
      if (TA) {  // op(A)[i][kk] = A[kk + i*lda], pairs along kk
        const int kk = 2 * (p % (BK / 2)), i = p / (BK / 2);
        const int gm = m0 + i, gk = k0 + kk;
        const int valid = gm < M ? max(0, min(2, K - gk)) : 0;
        const double* src = valid ? A + (long long)gk + (long long)gm * lda : A;
        copy_pair(as + i * Cfg::LDA_S + kk, src, valid, vecA);
      } else {   // op(A)[i][kk] = A[i + col(kk)*lda], pairs along i
        const int i = 2 * (p % (BM / 2)), kk = p / (BM / 2);
        const int gm = m0 + i, gk = k0 + kk;
        const int valid = gk < K ? max(0, min(2, M - gm)) : 0;
        long long col = gk;
        if (gather) col = acol[min(gk, K - 1)];
        const double* src = valid ? A + (long long)gm + col * lda : A;
        copy_pair(as + kk * Cfg::LDA_S + i, src, valid, vecA);
      }
    }
#pragma unroll
    for (int p = tid; p < Cfg::B_PAIRS; p += THREADS) {
      if (TB) {  // op(B)[kk][j] = B[j + kk*ldb], pairs along j
        const int j = 2 * (p % (BN / 2)), kk = p / (BN / 2);
        const int gn = n0 + j, gk = k0 + kk;
        const int valid = gk < K ? max(0, min(2, N - gn)) : 0;
        const double* src = valid ? B + (long long)gn + (long long)gk * ldb : B;
        copy_pair(bs + kk * Cfg::LDB_S + j, src, valid, vecB);
      } else {   // op(B)[kk][j] = B[kk + j*ldb], pairs along kk
        const int kk = 2 * (p % (BK / 2)), j = p / (BK / 2);
        const int gn = n0 + j, gk = k0 + kk;
        const int valid = gn < N ? max(0, min(2, K - gk)) : 0;
        const double* src = valid ? B + (long long)gk + (long long)gn * ldb : B;
        copy_pair(bs + j * Cfg::LDB_S + kk, src, valid, vecB);
      }
    }
  };

  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int lr = lane >> 2, lc = lane & 3;
  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // C tile prefetch (PFC, beta != 0): issued first so it lands with stage 0
  // and the read-modify-write epilogue never waits on HBM.
  double* Cs = smem + STAGES * (Cfg::A_ELEMS + Cfg::B_ELEMS);
  const bool pfc = PFC && P.beta != 0.0;
  if (pfc) {
    const double* C0 = P.C;
    const long long ldc0 = P.ldc;
    const bool vecC = !P.ccol && ((reinterpret_cast<uintptr_t>(C0) & 15) == 0) && ((ldc0 & 1) == 0);
#pragma unroll
    for (int p = tid; p < BM * BN / 2; p += THREADS) {
      const int i = 2 * (p % (BM / 2)), j = p / (BM / 2);
      const int gm = m0 + i, gn = n0 + j;
      const int valid = gn < N ? max(0, min(2, M - gm)) : 0;
      const double* src = C0;
      if (valid) {
        const long long col = P.ccol ? (long long)P.ccol[gn] : (long long)gn;
        src = C0 + (long long)gm + col * ldc0;
      }
      copy_pair(Cs + i + j * BM, src, valid, vecC);
    }
  }
  const int KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < KT) load_tile((kt + STAGES - 1) % STAGES, kt + STAGES - 1);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * Cfg::A_ELEMS;
    const double* bs = Bs + (kt % STAGES) * Cfg::B_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int m = wm * Cfg::WTM + i * 8 + lr;
        af[i] = TA ? as[m * Cfg::LDA_S + ks + lc] : as[(ks + lc) * Cfg::LDA_S + m];
      }
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int n = wn * Cfg::WTN + j * 8 + lr;
        bf[j] = TB ? bs[(ks + lc) * Cfg::LDB_S + n] : bs[n * Cfg::LDB_S + ks + lc];
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  double* __restrict__ C = P.C;
  const long long ldc = P.ldc;
  const double alpha = P.alpha, beta = P.beta;
  const int* __restrict__ ccol = P.ccol;
#pragma unroll
  for (int j = 0; j < Cfg::FN; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
      if (gn >= N) continue;
      const long long col = gather ? (long long)ccol[gn] : (long long)gn;
      double* cc = C + col * ldc;
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int lm = wm * Cfg::WTM + i * 8 + lr;
        const int gm = m0 + lm;
        if (gm < M) {
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * (pfc ? Cs[lm + (gn - n0) * BM] : cc[gm]);
          cc[gm] = v;
        }
      }
    }
  }
}

static bool batch_vec_ok(const GemmBatch* b, const GemmDesc* dd) {
  if (dd || !b) return false;  // device descriptors: alignment unknown on the host
  for (int i = 0; i < b->count; ++i) {
    const GemmDesc& d = b->d[i];
    if ((reinterpret_cast<uintptr_t>(d.A) & 15) || (reinterpret_cast<uintptr_t>(d.B) & 15) || (d.lda & 1) ||
        (d.ldb & 1))
      return false;
    if (d.beta != 0.0 && ((reinterpret_cast<uintptr_t>(d.C) & 15) || (d.ldc & 1) || d.ccol)) return false;
  }
  return true;
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, bool PFC, bool VEC,
          bool GATHER>
static int launch_cfg_v(cudaStream_t st, const GemmBatch* b, const GemmDesc* dd, int nz, int max_m,
                        int max_n) {
  using Cfg = GemmCfg<TA, TB, BM, BN, BK, WM, WN, STAGES>;
  auto kern = dgemm_kernel<TA, TB, BM, BN, BK, WM, WN, STAGES, MINB, PFC, VEC, GATHER>;
  constexpr int smem = Cfg::SMEM_BYTES + (PFC ? Cfg::C_ELEMS * 8 : 0);
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid((max_m + BM - 1) / BM, (max_n + BN - 1) / BN, nz);
  GemmBatch empty;
  empty.count = 0;
  kern<<<grid, Cfg::THREADS, smem, st>>>(b ? *b : empty, dd);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

template <bool TA, bool TB, int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, bool PFC>
static int launch_cfg(cudaStream_t st, const GemmBatch* b, const GemmDesc* dd, int nz, int max_m,
                      int max_n) {
  if (dd) {
    if constexpr (!TA && !PFC)  // BDC merge products only
      return launch_cfg_v<TA, TB, BM, BN, BK, WM, WN, STAGES, MINB, PFC, false, true>(st, b, dd, nz, max_m, max_n);
    return -1;
  }
  if (batch_vec_ok(b, dd) && g_gemm_route != 5)  // route 5 (debug): force 8-byte copies
    return launch_cfg_v<TA, TB, BM, BN, BK, WM, WN, STAGES, MINB, PFC, true, false>(st, b, dd, nz, max_m, max_n);
  return launch_cfg_v<TA, TB, BM, BN, BK, WM, WN, STAGES, MINB, PFC, false, false>(st, b, dd, nz, max_m, max_n);
}

template <bool TA, bool TB>
static int launch_sized(cudaStream_t st, const GemmBatch* b, const GemmDesc* dd, int nz, int max_m,
                        int max_n, int max_k, bool beta_nz) {
  // Large tiles (16 warps, 128x128x32, 1 CTA/SM) when the output fills the
  // GPU and K is long enough to amortize the pipeline; otherwise 64x64 tiles
  // with several CTAs per SM so load / MMA / epilogue of different CTAs overlap.
  // 64x128x16 tiles, 4 warps of 32x64, 3 stages, 2 CTAs/SM: two independent
  // CTAs per SM keep the DMMA pipe fed across each other's barriers.
  const long long tiles64x128 = (long long)((max_m + 63) / 64) * ((max_n + 127) / 128) * nz;
  if (g_gemm_route == 2 && beta_nz)  // debug routing experiments (dcsvd_debug_gemm_route)
    return launch_cfg<TA, TB, 64, 128, 16, 2, 2, 3, 2, true>(st, b, dd, nz, max_m, max_n);
  if (tiles64x128 >= 2 * 148 && max_k >= 128)
    return launch_cfg<TA, TB, 64, 128, 16, 2, 2, 3, 2, false>(st, b, dd, nz, max_m, max_n);
  if (beta_nz && max_k <= 64)  // rank-k updates: C read-modify-write dominates -> prefetch C
    return launch_cfg<TA, TB, 64, 64, 16, 2, 2, 3, 2, true>(st, b, dd, nz, max_m, max_n);
  return launch_cfg<TA, TB, 64, 64, 16, 2, 2, 3, 3, false>(st, b, dd, nz, max_m, max_n);
}


// ---------------------------------------------------------------------------
// Streaming rank-k update  C <- alpha * A * op(B) + beta * C  for small K
// (<= 128): the GEBRD trailing update A -= P Q^T (bidiag.py:195-197) and the
// CWY updates C -= Y X (qrblock.py:103-119).  Each CTA owns 64-column strips
// of C: the K x 64 slice of op(B) is loaded once per strip and stays in shared
// memory while MT-row tiles of A stream through a double buffer: one TMA bulk
// copy (cp.async.bulk, SASS UBLKCP) per tile column, issued by K threads spread
// over the 8 warps and completing on the buffer's mbarrier (K arrivals + tx
// bytes); tiles with an odd row count fall back to 16-byte cp.async pairs.
// Bulk A copies: 8160^2 K=64 20.4 -> 21.6 TFLOP/s, 8192^2 K=128 22.3 -> 23.8
// (tools/rankk_bulk_ab.py); issuing all of them from one warp was 25 % slower
// than cp.async.  Bulk B strips on top: K=128 23.8 -> 24.1 (ORMBR 91.2 -> 90.0 ms).  Each thread loads its C fragment into registers at the start of
// a tile, so the HBM latency of the read-modify-write is covered by that
// tile's DMMAs.  Persistent grid, 1 CTA / SM, 8 warps.
template <bool TB, int KMAX, int MT, int WARPS_M>
struct RankkCfg {
  static constexpr int NW = 64;
  static constexpr int THREADS = 256;
  static constexpr int WARPS_N = 8 / WARPS_M;
  static constexpr int WTM = MT / WARPS_M, WTN = NW / WARPS_N;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int LDB_S = TB ? (NW + 4) : (KMAX + 4);
  static constexpr int B_ELEMS = TB ? KMAX * (NW + 4) : NW * (KMAX + 4);
  static constexpr int LDA_S = MT + 4;
  static constexpr int A_ELEMS = KMAX * (MT + 4);
  static constexpr int SMEM_BYTES = (B_ELEMS + 2 * A_ELEMS) * 8;
  static constexpr int CHUNK = 8;  // most row tiles per work unit (B strip reuse)
};

template <bool TB, int KMAX, int MT, int WARPS_M, bool VEC>
__global__ void __launch_bounds__(256, 1) rankk_stream_kernel(GemmDesc P, int chunk) {
  using Cfg = RankkCfg<TB, KMAX, MT, WARPS_M>;
  constexpr int THREADS = Cfg::THREADS, NW = Cfg::NW;
  extern __shared__ __align__(16) double smem[];
  double* Bs = smem;
  double* As = Bs + Cfg::B_ELEMS;  // 2 buffers
  const int M = P.m, N = P.n, K = P.k;
  const double* __restrict__ A = P.A;
  const double* __restrict__ B = P.B;
  double* __restrict__ C = P.C;
  const long long lda = P.lda, ldb = P.ldb, ldc = P.ldc;
  const double alpha = P.alpha, beta = P.beta;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int lr = lane >> 2, lc = lane & 3;
  const int Kp = (K + 3) & ~3;
  const int strips = (N + NW - 1) / NW;
  const int tiles = (M + MT - 1) / MT;
  const int chunks = (tiles + chunk - 1) / chunk;
  const int units = strips * chunks;

  // A tiles by TMA bulk copies (one per column of the tile, issued by warp 0,
  // completing on the buffer's mbarrier) when the rows allow 16-byte sizes;
  // otherwise per-thread cp.async pairs (dcsvd_debug_rankk_bulk(0): cp.async only).
  // The B strip of a unit likewise: one bulk copy per row (TB, K arrivals) or
  // per column (K even, 64 arrivals) on abar[2].
  __shared__ __align__(8) uint64_t abar[3];
  unsigned aphase = 0;  // bit b: parity of barrier b's next phase
  if (tid == 0) {
    mbar_init(&abar[0], K);
    mbar_init(&abar[1], K);
    mbar_init(&abar[2], TB ? K : NW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (Kp > K)  // pad rows/columns K..Kp-1 of the B strip: zero once (bulk copies never write them)
    for (int p = tid; p < (Kp - K) * NW; p += THREADS) {
      const int kk = K + p / NW, j = p % NW;
      Bs[TB ? kk * Cfg::LDB_S + j : j * Cfg::LDB_S + kk] = 0.0;
    }
  if (Kp > K)  // pad columns K..Kp-1 of both A buffers are never copied: zero them once
    for (int p = tid; p < 2 * (Kp - K) * MT; p += THREADS) {
      const int b = p / ((Kp - K) * MT), r = p % ((Kp - K) * MT);
      As[b * Cfg::A_ELEMS + (K + r / MT) * Cfg::LDA_S + r % MT] = 0.0;
    }
  __syncthreads();
  auto bulk_ok = [&](int m0) { return VEC && g_bulk_a && ((min(MT, M - m0) & 1) == 0); };
  auto load_a_bulk = [&](int buf, int m0) {  // thread kk < K copies column kk (K arrivals per phase)
    const int rows = min(MT, M - m0);
    const unsigned bytes = (unsigned)rows * 8u;
    const int kk = (tid & 7) * 32 + (tid >> 3);  // spread the issuing threads over the 8 warps
    if (kk < K) {
      mbar_expect_tx(&abar[buf], bytes);
      bulk_g2s(As + buf * Cfg::A_ELEMS + kk * Cfg::LDA_S, A + (long long)m0 + (long long)kk * lda, bytes, &abar[buf]);
    }
  };
  auto load_a = [&](int buf, int m0) {
    if (bulk_ok(m0)) {
      load_a_bulk(buf, m0);
      return;
    }
    double* as = As + buf * Cfg::A_ELEMS;
#pragma unroll
    for (int p0 = 0; p0 < MT * KMAX / 2; p0 += THREADS) {  // A: [k][m], pairs along m (compile-time trip count)
      const int p = p0 + tid;
      const int i = 2 * (p % (MT / 2)), kk = p / (MT / 2);
      if (kk >= Kp) break;
      const int gm = m0 + i;
      const int valid = kk < K ? max(0, min(2, M - gm)) : 0;
      const double* src = valid ? A + (long long)gm + (long long)kk * lda : A;
      copy_pair(as + kk * Cfg::LDA_S + i, src, valid, VEC);
    }
  };

  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int s = u / chunks, ch = u % chunks;
    const int n0 = s * NW;
    const int t0 = ch * chunk, t1 = min(tiles, t0 + chunk);
    const bool bbulk = VEC && g_bulk_a && (TB ? ((min(NW, N - n0) & 1) == 0) : ((K & 1) == 0));
    if (bbulk) {
      const int q = (tid & 7) * 32 + (tid >> 3);  // issuing threads spread over the warps
      if (TB) {  // row kk of the strip: min(64, N - n0) contiguous doubles
        if (q < K) {
          const unsigned bytes = (unsigned)min(NW, N - n0) * 8u;
          mbar_expect_tx(&abar[2], bytes);
          bulk_g2s(Bs + q * Cfg::LDB_S, B + (long long)n0 + (long long)q * ldb, bytes, &abar[2]);
        }
      } else if (q < NW) {  // column j of the strip: K contiguous doubles
        if (n0 + q < N) {
          mbar_expect_tx(&abar[2], (unsigned)K * 8u);
          bulk_g2s(Bs + q * Cfg::LDB_S, B + (long long)(n0 + q) * ldb, (unsigned)K * 8u, &abar[2]);
        } else {
          mbar_arrive(&abar[2]);
        }
      }
    } else if (TB) {
      for (int p = tid; p < Kp * NW / 2; p += THREADS) {  // B[n + k*ldb]: pairs along n
        const int j = 2 * (p % (NW / 2)), kk = p / (NW / 2);
        const int gn = n0 + j;
        const int valid = kk < K ? max(0, min(2, N - gn)) : 0;
        const double* src = valid ? B + (long long)gn + (long long)kk * ldb : B;
        copy_pair(Bs + kk * Cfg::LDB_S + j, src, valid, VEC);
      }
    } else {
      for (int p = tid; p < Kp * NW / 2; p += THREADS) {  // B[k + n*ldb]: pairs along k
        const int kk = 2 * (p % (Kp / 2)), j = p / (Kp / 2);
        const int gn = n0 + j;
        const int valid = gn < N ? max(0, min(2, K - kk)) : 0;
        const double* src = valid ? B + (long long)kk + (long long)gn * ldb : B;
        copy_pair(Bs + j * Cfg::LDB_S + kk, src, valid, VEC);
      }
    }
    load_a(0, t0 * MT);
    cp_async_commit();
    for (int t = t0; t < t1; ++t) {
      const int buf = (t - t0) & 1;
      const int m0 = t * MT;
      // C fragment of this tile into registers (consumed in the epilogue)
      double cv[Cfg::FM][Cfg::FN][2];
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i) {
            const int gm = m0 + wm * Cfg::WTM + i * 8 + lr;
            cv[i][j][h] = (beta != 0.0 && gn < N && gm < M) ? C[(long long)gm + (long long)gn * ldc] : 0.0;
          }
        }
      if (t + 1 < t1) {
        load_a(buf ^ 1, (t + 1) * MT);
        // C lines of the next tile into L2: its register loads at the next
        // tile's start then return at L2 latency, not HBM latency under load
        // (g_rankk_prefetch = how many tiles ahead; the unit's first tile
        // also covers the tiles before that distance)
        const int dist = g_rankk_prefetch;
        if (beta != 0.0 && dist > 0) {
          constexpr int LINES = MT * 8 / 128;  // 128-byte lines per C column of a tile
          for (int d = (t == t0 ? 1 : dist); d <= dist && t + d < t1; ++d)
            for (int q = tid; q < NW * LINES; q += THREADS) {
              const int gn = n0 + q / LINES, gm = (t + d) * MT + (q % LINES) * 16;
              if (gn < N && gm < M) prefetch_l2(C + (long long)gm + (long long)gn * ldc);
            }
        }
      }
      cp_async_commit();
      cp_async_wait<1>();
      if (bulk_ok(m0)) {
        mbar_wait(&abar[buf], (aphase >> buf) & 1u);
        aphase ^= 1u << buf;
      }
      if (t == t0 && bbulk) {
        mbar_wait(&abar[2], (aphase >> 2) & 1u);
        aphase ^= 4u;
      }
      __syncthreads();
      const double* as = As + buf * Cfg::A_ELEMS;
      double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
      for (int ks = 0; ks < Kp; ks += 4) {
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(ks + lc) * Cfg::LDA_S + wm * Cfg::WTM + i * 8 + lr];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          const int n = wn * Cfg::WTN + j * 8 + lr;
          bf[j] = TB ? Bs[(ks + lc) * Cfg::LDB_S + n] : Bs[n * Cfg::LDB_S + ks + lc];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
          if (gn >= N) continue;
          double* cc = C + (long long)gn * ldc;
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i) {
            const int gm = m0 + wm * Cfg::WTM + i * 8 + lr;
            if (gm < M) cc[gm] = alpha * acc[i][j][h] + beta * cv[i][j][h];
          }
        }
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Warp-specialized rank-k update (same contract as rankk_stream_kernel, for
// operands whose leading dimensions / bases allow 2-D TMA tensor maps): one
// producer warp (one elected lane) moves every operand with TMA tensor copies
// (cp.async.bulk.tensor.2d, SASS UTMALDG) -- ONE instruction per A tile and
// per B strip -- into a ring of S A-tile stages and a B-strip buffer, each
// completing on its own "full" mbarrier, and prefetches the tile's C block
// into L2 with one cp.async.bulk.prefetch.tensor.  The boxes are 4 elements
// wider than the tile along the contiguous dimension, so the shared-memory
// pitch is 4 mod 16 doubles and the m8n8k4 fragment reads stay bank-conflict
// free (the 4 extra rows are ignored; out-of-range elements are zero-filled
// by the TMA unit, which also supplies the K -> multiple-of-4 padding).
// NG consumer groups of 4 warps (one warp per SM sub-partition) take the
// row tiles of a unit round-robin and run only LDS + DMMA, release the A
// stage on its "empty" mbarrier after their last fragment read, then do the
// C read-modify-write epilogue.  The groups never synchronise with each
// other, so one group's epilogue / stage wait overlaps the other's DMMAs (the
// per-tile CTA barriers are what kept rankk_stream_kernel at ~60 % DMMA-pipe
// activity), and the producer's copy issue is off the math warps entirely
// (per-column 1-D bulk copies from one warp were issue-bound: 13 TF/s).
int rankk_chunk(int m, int strips, int tiles, int mt, int kmax, int cmax, int sms);
__constant__ int g_ws_flags = 0;  // debug: bit 0 = no C prefetch
int g_ws_flags_host = 0;
int set_ws_flags(int f) {
  g_ws_flags_host = f;
  return cudaMemcpyToSymbol(g_ws_flags, &f, sizeof(int)) == cudaSuccess ? 0 : -1;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(d), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(b) : "memory");
}
// TMA gather4 (sm_100): four rows (outer coordinates c[0..3]) of a box {inner, 1}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int x, const int (&c)[4], uint64_t* bar) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];\n" ::"r"(d), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(c[0]), "r"(c[1]), "r"(c[2]),
      "r"(c[3]), "r"(b) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1) : "memory");
}

template <bool TB, int KMAX, int MT, int NG, int S>
struct RankkWsCfg {
  static constexpr int NW = 64;
  static constexpr int THREADS = 32 + 128 * NG;
  static constexpr int WARPS_M = MT >= 32 ? 2 : 1, WARPS_N = 4 / WARPS_M;  // per group
  static constexpr int WTM = MT / WARPS_M, WTN = NW / WARPS_N;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  static constexpr int LDA_S = MT + 4;  // [k][m]: TMA box {MT + 4, Kp}
  static constexpr int A_ELEMS = KMAX * LDA_S;
  static constexpr int LDB_S = TB ? (NW + 4) : (KMAX + 4);  // box {68, Kp} or {KMAX + 4, 64}
  static constexpr int B_ELEMS = TB ? KMAX * LDB_S : NW * LDB_S;
  static constexpr int NBUF = 2;  // B strips double-buffered: the groups flow across unit boundaries
  static constexpr int SMEM_BYTES = (NBUF * B_ELEMS + S * A_ELEMS) * 8 + 128;  // +128: manual alignment
  static constexpr int CHUNK = 64;
};

__device__ __forceinline__ double neg_bits(double x) {  // -x on the integer pipe (not a DADD)
  double r;
  asm("{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %1;\nxor.b32 hi, hi, 0x80000000;\nmov.b64 %0, {lo, hi};\n}"
      : "=d"(r) : "d"(x));
  return r;
}

template <bool TB, int KMAX, int MT, int NG, int S>
__global__ void __launch_bounds__(32 + 128 * NG, 1)
    rankk_ws_kernel(GemmDesc P, int chunk, const __grid_constant__ CUtensorMap tA,
                    const __grid_constant__ CUtensorMap tB, const __grid_constant__ CUtensorMap tC) {
  using Cfg = RankkWsCfg<TB, KMAX, MT, NG, S>;
  constexpr int NW = Cfg::NW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 128-byte alignment by pointer arithmetic (keeps the shared address space: LDS, not generic LD)
  double* Bs = reinterpret_cast<double*>(smem_raw + ((128u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u));
  double* As = Bs + Cfg::NBUF * Cfg::B_ELEMS;
  __shared__ __align__(8) uint64_t a_full[S], a_empty[S], b_full[Cfg::NBUF], b_empty[Cfg::NBUF];
  const int M = P.m, N = P.n, K = P.k;
  double* __restrict__ C = P.C;
  const long long ldc = P.ldc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Kp = (K + 3) & ~3;
  const int strips = (N + NW - 1) / NW;
  const int tiles = (M + MT - 1) / MT;
  const int chunks = (tiles + chunk - 1) / chunk;
  const int units = strips * chunks;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], 4);
    }
    for (int b = 0; b < Cfg::NBUF; ++b) {
      mbar_init(&b_full[b], 1);
      mbar_init(&b_empty[b], 4 * NG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------ producer (one lane)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tB)) : "memory");
      const unsigned a_bytes = (unsigned)(Cfg::LDA_S * Kp * 8);
      const unsigned b_bytes = (unsigned)((TB ? Cfg::LDB_S * Kp : Cfg::LDB_S * NW) * 8);
      const bool pfc = P.beta != 0.0 && !(g_ws_flags & 1);
      unsigned seq = 0, useq = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++useq) {
        const int n0 = (u / chunks) * NW;
        const int t0 = (u % chunks) * chunk, t1 = min(tiles, t0 + chunk);
        const int bb = useq % Cfg::NBUF;
        if (useq >= (unsigned)Cfg::NBUF) mbar_wait(&b_empty[bb], ((useq / Cfg::NBUF) - 1) & 1u);
        mbar_expect_tx(&b_full[bb], b_bytes);
        if (TB) tma_load_2d(Bs + bb * Cfg::B_ELEMS, &tB, n0, 0, &b_full[bb]);
        else tma_load_2d(Bs + bb * Cfg::B_ELEMS, &tB, 0, n0, &b_full[bb]);
        for (int t = t0; t < t1; ++t, ++seq) {
          const int st = seq % S;
          if ((g_ws_flags & 4) && seq >= (unsigned)S) continue;  // debug: stages loaded once
          if (seq >= (unsigned)S) mbar_wait(&a_empty[st], ((seq / S) - 1) & 1u);
          mbar_expect_tx(&a_full[st], a_bytes);
          tma_load_2d(As + st * Cfg::A_ELEMS, &tA, t * MT, 0, &a_full[st]);
          if (pfc) tma_prefetch_2d(&tC, t * MT, n0);
        }
      }
    }
    return;
  }
  // ------------------------------ consumers
  const double* smem_b = Bs;
  const int ct = tid - 32;
  const int grp = ct >> 7;       // consumer group
  const int gw = (ct >> 5) & 3;  // warp within the group
  const int wm = gw % Cfg::WARPS_M, wn = gw / Cfg::WARPS_M;
  const int lr = lane >> 2, lc = lane & 3;
  const double alpha = P.alpha, beta = P.beta;
  // C -= A op(B) (alpha = -1, beta = 1: every rank-k update of the pipeline) and
  // C += A op(B): the accumulators start from the C fragment (C -= AB runs as
  // -((-C) + AB), the sign flips by integer XORs on the load and the store),
  // so the epilogue is plain stores -- no FP64 instruction competes with the
  // DMMAs for the shared FP64/tensor pipe.  Other (alpha, beta): general epilogue.
  const bool fold = beta == 1.0 && (alpha == 1.0 || alpha == -1.0);
  const bool noc = g_ws_flags & 2;  // debug: no C traffic (pipeline bound)
  const bool negb = alpha == -1.0;
  unsigned seqb = 0, useq = 0;
  double cn[Cfg::FM][Cfg::FN][2];
  bool have_next = false;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++useq) {
    const int n0 = (u / chunks) * NW;
    const int t0 = (u % chunks) * chunk, t1 = min(tiles, t0 + chunk);
    auto load_c = [&](int tt, double (&dst)[Cfg::FM][Cfg::FN][2]) {
      const int mm = tt * MT;
      const bool fl = mm + MT <= M && n0 + NW <= N;
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
          const double* cc = C + (long long)gn * ldc + mm + wm * Cfg::WTM + lr;
#pragma unroll
          for (int i = 0; i < Cfg::FM; ++i)
            dst[i][j][h] = (fl || (gn < N && mm + wm * Cfg::WTM + i * 8 + lr < M)) ? __ldcg(cc + i * 8) : 0.0;
        }
    };
    have_next = false;
    const int bb = useq % Cfg::NBUF;
    mbar_wait(&b_full[bb], (useq / Cfg::NBUF) & 1u);
    const double* Bs = smem_b + bb * Cfg::B_ELEMS;
    for (int t = t0 + grp; t < t1; t += NG) {
      const unsigned seq = seqb + (unsigned)(t - t0);
      const int st = seq % S;
      const int m0 = t * MT;
      const bool full = m0 + MT <= M && n0 + NW <= N;  // no bounds predicates
      double acc[Cfg::FM][Cfg::FN][2];
      if (fold && !noc) {
        // C fragment (L2-prefetched by the producer) as the accumulator init;
        // the group's next tile of the unit is loaded now into cn, one tile
        // ahead of its use, so only a unit's first tile waits on C
        if (!have_next) load_c(t, cn);
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[i][j][h] = negb ? neg_bits(cn[i][j][h]) : cn[i][j][h];
        have_next = t + NG < t1;
        if (have_next) load_c(t + NG, cn);
      } else {
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      }
      if (!(g_ws_flags & 4) || seq < (unsigned)S) mbar_wait(&a_full[st], (seq / S) & 1u);
      const double* as = As + st * Cfg::A_ELEMS;
#pragma unroll 4
      for (int ks = 0; ks < Kp; ks += 4) {
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(ks + lc) * Cfg::LDA_S + wm * Cfg::WTM + i * 8 + lr];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          const int n = wn * Cfg::WTN + j * 8 + lr;
          bf[j] = TB ? Bs[(ks + lc) * Cfg::LDB_S + n] : Bs[n * Cfg::LDB_S + ks + lc];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0 && !(g_ws_flags & 4)) mbar_arrive(&a_empty[st]);
      if (fold) {
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
            double* cc = C + (long long)gn * ldc + m0 + wm * Cfg::WTM + lr;
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i)
              if ((full || (gn < N && m0 + wm * Cfg::WTM + i * 8 + lr < M)) && (!noc || acc[i][j][h] == 1.2345e300))
                cc[i * 8] = negb ? neg_bits(acc[i][j][h]) : acc[i][j][h];
          }
        continue;
      }
      // general (alpha, beta): C read after the math, in two halves of the column
      // blocks (bounded registers); every load of a half in flight before its stores
      constexpr int EPI = Cfg::FN >= 2 ? 2 : 1;
#pragma unroll
      for (int e = 0; e < EPI; ++e) {
        double cv[Cfg::FM][Cfg::FN / EPI][2];
#pragma unroll
        for (int jj = 0; jj < Cfg::FN / EPI; ++jj)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gn = n0 + wn * Cfg::WTN + (e * (Cfg::FN / EPI) + jj) * 8 + lc * 2 + h;
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i) {
              const int gm = m0 + wm * Cfg::WTM + i * 8 + lr;
              cv[i][jj][h] = (beta != 0.0 && gn < N && gm < M) ? __ldcg(C + (long long)gm + (long long)gn * ldc) : 0.0;
            }
          }
#pragma unroll
        for (int jj = 0; jj < Cfg::FN / EPI; ++jj) {
          const int j = e * (Cfg::FN / EPI) + jj;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
            if (gn >= N) continue;
            double* cc = C + (long long)gn * ldc;
#pragma unroll
            for (int i = 0; i < Cfg::FM; ++i) {
              const int gm = m0 + wm * Cfg::WTM + i * 8 + lr;
              if (gm < M) cc[gm] = alpha * acc[i][j][h] + beta * cv[i][jj][h];
            }
          }
        }
      }
    }
    seqb += (unsigned)(t1 - t0);
    __syncwarp();
    if (lane == 0) mbar_arrive(&b_empty[bb]);  // this warp is done with the unit's B strip
  }
}

int g_rankk_ws = 1;  // debug: 0 = rankk_stream_kernel only

// 2-D fp64 tensor map: `inner` contiguous elements per line, `outer` lines
// `ld` elements apart; box {box_inner, box_outer}; out-of-range -> zero.
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
int make_tmap_2d(CUtensorMap* map, const double* base, long long inner, long long outer, long long ld,
                 int box_inner, int box_outer) {
  auto fn = tmap_encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

template <bool TB, int KMAX, int MT, int NG, int S>
static int launch_rankk_ws(cudaStream_t st, const GemmDesc& d, int sms, int kmax_cost) {
  using Cfg = RankkWsCfg<TB, KMAX, MT, NG, S>;
  const int Kp = (d.k + 3) & ~3;
  CUtensorMap tA, tB, tC;
  if (make_tmap_2d(&tA, d.A, d.m, d.k, d.lda, Cfg::LDA_S, Kp)) return -1;
  if (TB) {
    if (make_tmap_2d(&tB, d.B, d.n, d.k, d.ldb, Cfg::LDB_S, Kp)) return -1;
  } else if (make_tmap_2d(&tB, d.B, d.k, d.n, d.ldb, Cfg::LDB_S, Cfg::NW)) {
    return -1;
  }
  if (make_tmap_2d(&tC, d.C, d.m, d.n, d.ldc, MT, Cfg::NW)) return -1;
  auto kern = rankk_ws_kernel<TB, KMAX, MT, NG, S>;
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
  const int strips = (d.n + 63) / 64;
  const int tiles = (d.m + MT - 1) / MT;
  // at least one tile per consumer group in a unit (the groups share its B strip)
  const int chunk =
      std::min(tiles, std::max(NG, rankk_chunk(d.m, strips, tiles, MT, kmax_cost, Cfg::CHUNK, sms)));
  const int units = strips * ((tiles + chunk - 1) / chunk);
  const int grid = std::max(1, std::min(units, sms));
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(d, chunk, tA, tB, tC);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// Warp-specialized general DMMA GEMM (host descriptor, optional split-K over
// blockIdx.z): C = alpha op(A) op(B) + beta C on 128 x 64 tiles.  One producer
// lane streams BK = 32 k-slices of op(A) and op(B) into an S-stage ring with
// ONE TMA tensor-map load per operand per stage (boxes 4 elements wider than
// the tile along the contiguous dimension: conflict-free fragment pitch; the
// TMA unit zero-fills past K); 8 consumer warps (2 per SM sub-partition, 32 x
// 32 each) run LDS + DMMA only and release each stage on its "empty"
// mbarrier.  Used for the CWY inner products Z = Y^T C / C Y (K = the
// reflector rows), X = T Z, the TS recombination U = Q U0 and other
// long-K GEMMs.
template <bool TA, bool TB, int S>
struct DgemmWsCfg {
  static constexpr int BM = 128, BN = 64, BK = 32;
  static constexpr int WARPS_M = 4, WARPS_N = 2;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int FM = WTM / 8, FN = WTN / 8;
  // op(A) stage: !TA [k][m] pitch BM+4 (box {BM+4, BK});  TA [m][k] pitch BK+4 (box {BK+4, BM})
  static constexpr int LDA_S = TA ? (BK + 4) : (BM + 4);
  static constexpr int A_ELEMS = TA ? BM * LDA_S : BK * LDA_S;
  // op(B) stage: TB [k][n] pitch BN+4 (box {BN+4, BK});  !TB [n][k] pitch BK+4 (box {BK+4, BN})
  static constexpr int LDB_S = TB ? (BN + 4) : (BK + 4);
  static constexpr int B_ELEMS = TB ? BK * LDB_S : BN * LDB_S;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int THREADS = 32 + 256;
  static constexpr int SMEM_BYTES = S * STAGE * 8 + 128;
};

template <bool TA, bool TB, int S>
__global__ void __launch_bounds__(288, 1)
    dgemm_ws_kernel(GemmDesc P, int ksplit, int kchunk, long long cslice, const __grid_constant__ CUtensorMap tA,
                    const __grid_constant__ CUtensorMap tB) {
  using Cfg = DgemmWsCfg<TA, TB, S>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw + ((128u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int sl = blockIdx.z;
  const int kbeg = ksplit > 1 ? sl * kchunk : 0;
  const int kend = ksplit > 1 ? min(P.k, kbeg + kchunk) : P.k;
  const int KT = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tB)) : "memory");
      const unsigned bytes = (unsigned)Cfg::STAGE * 8u;
      for (int kt = 0; kt < KT; ++kt) {
        const int st = kt % S;
        if (kt >= S) mbar_wait(&empty[st], ((kt / S) - 1) & 1u);
        double* as = sm + st * Cfg::STAGE;
        double* bs = as + Cfg::A_ELEMS;
        const int k0 = kbeg + kt * BK;
        mbar_expect_tx(&full[st], bytes);
        if (TA) tma_load_2d(as, &tA, k0, m0, &full[st]);
        else tma_load_2d(as, &tA, m0, k0, &full[st]);
        if (TB) tma_load_2d(bs, &tB, n0, k0, &full[st]);
        else tma_load_2d(bs, &tB, k0, n0, &full[st]);
      }
    }
    return;
  }
  const int cw = warp - 1;
  const int wm = cw % Cfg::WARPS_M, wn = cw / Cfg::WARPS_M;
  const int lr = lane >> 2, lc = lane & 3;
  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt % S;
    mbar_wait(&full[st], (kt / S) & 1u);
    const double* as = sm + st * Cfg::STAGE;
    const double* bs = as + Cfg::A_ELEMS;
    // slice ends are multiples of 4 (split-K chunks of 16); past K the TMA zero-fills
    const int kl = min(BK, ((kend - (kbeg + kt * BK)) + 3) & ~3);
    if (kl == BK) {
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) {
          const int m = wm * Cfg::WTM + i * 8 + lr;
          af[i] = TA ? as[m * Cfg::LDA_S + ks + lc] : as[(ks + lc) * Cfg::LDA_S + m];
        }
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          const int n = wn * Cfg::WTN + j * 8 + lr;
          bf[j] = TB ? bs[(ks + lc) * Cfg::LDB_S + n] : bs[n * Cfg::LDB_S + ks + lc];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    } else {
      for (int ks = 0; ks < kl; ks += 4) {
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) {
          const int m = wm * Cfg::WTM + i * 8 + lr;
          af[i] = TA ? as[m * Cfg::LDA_S + ks + lc] : as[(ks + lc) * Cfg::LDA_S + m];
        }
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          const int n = wn * Cfg::WTN + j * 8 + lr;
          bf[j] = TB ? bs[(ks + lc) * Cfg::LDB_S + n] : bs[n * Cfg::LDB_S + ks + lc];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  double* __restrict__ C = P.C + (ksplit > 1 ? sl * cslice : 0);
  const long long ldc = P.ldc;
  const double alpha = P.alpha, beta = P.beta;
  const int M = P.m, N = P.n;
#pragma unroll
  for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
      if (gn >= N) continue;
      double* cc = C + (long long)gn * ldc;
      double cv[Cfg::FM];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int gm = m0 + wm * Cfg::WTM + i * 8 + lr;
        cv[i] = (beta != 0.0 && gm < M) ? cc[gm] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int gm = m0 + wm * Cfg::WTM + i * 8 + lr;
        if (gm < M) cc[gm] = beta != 0.0 ? fma(beta, cv[i], alpha * acc[i][j][h]) : alpha * acc[i][j][h];
      }
    }
}

int g_dgemm_ws_min_split_tiles = 148;  // debug knob (dcsvd_debug_dgemm_ws_min)
int g_dgemm_ws_min_tiles = 148;        // debug knob (dcsvd_debug_dgemm_ws_min_nosplit)
int g_dgemm_ws = 1;  // debug: 0 = cp.async kernels only, 2 = rank-k (K > 64) on the non-persistent TMA GEMM, 3 = register-C rank-k tile kernel

// Persistent rank-k update on the TMA GEMM tiles (C <- C -+ A op(B), K <= 128,
// beta = 1, alpha = +-1): 128 x 64 output tiles taken round-robin; the
// producer lane streams every tile's BK = 32 k-slices of A and op(B) through
// the S-stage ring without stopping between tiles, so the next tile's first
// stages are resident when its math starts; the 8 consumer warps hold the
// current tile's accumulators (initialised from C, the sign of alpha applied
// by integer XOR) and the NEXT tile's C fragment (loaded at the start of the
// current tile's math), so the per-tile epilogue is plain stores.
template <bool TB, int S>
__global__ void __launch_bounds__(288, 1)
    rankk_tile_kernel(GemmDesc P, const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB) {
  using Cfg = DgemmWsCfg<false, TB, S>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw + ((128u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = P.m, N = P.n, K = P.k;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN, ntiles = tm * tn;
  const int KT = (K + BK - 1) / BK;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tB)) : "memory");
      const unsigned bytes = (unsigned)Cfg::STAGE * 8u;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t % tm) * BM, n0 = (t / tm) * BN;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int st = it % S;
          if (it >= S) mbar_wait(&empty[st], ((it / S) - 1) & 1u);
          double* as = sm + st * Cfg::STAGE;
          double* bs = as + Cfg::A_ELEMS;
          mbar_expect_tx(&full[st], bytes);
          tma_load_2d(as, &tA, m0, kt * BK, &full[st]);
          if (TB) tma_load_2d(bs, &tB, n0, kt * BK, &full[st]);
          else tma_load_2d(bs, &tB, kt * BK, n0, &full[st]);
        }
      }
    }
    return;
  }
  const int cw = warp - 1;
  const int wm = cw % Cfg::WARPS_M, wn = cw / Cfg::WARPS_M;
  const int lr = lane >> 2, lc = lane & 3;
  double* __restrict__ C = P.C;
  const long long ldc = P.ldc;
  const bool negb = P.alpha == -1.0;
  auto load_c = [&](int t, double (&dst)[Cfg::FM][Cfg::FN][2]) {
    const int m0 = (t % tm) * BM, n0 = (t / tm) * BN;
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
        const double* cc = C + (long long)gn * ldc + m0 + wm * Cfg::WTM + lr;
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
          dst[i][j][h] = (gn < N && m0 + wm * Cfg::WTM + i * 8 + lr < M) ? __ldcg(cc + i * 8) : 0.0;
      }
  };
  double cn[Cfg::FM][Cfg::FN][2];
  if ((int)blockIdx.x < ntiles) load_c(blockIdx.x, cn);
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int m0 = (t % tm) * BM, n0 = (t / tm) * BN;
    double acc[Cfg::FM][Cfg::FN][2];
    // C -= A op(B) runs as -((-C) + A op(B)): sign flips by integer XOR on the load / store
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[i][j][h] = negb ? neg_bits(cn[i][j][h]) : cn[i][j][h];
    if (t + (int)gridDim.x < ntiles) load_c(t + gridDim.x, cn);  // next tile's C, in flight during the math
    for (int kt = 0; kt < KT; ++kt, ++it) {
      const int st = it % S;
      mbar_wait(&full[st], (it / S) & 1u);
      const double* as = sm + st * Cfg::STAGE;
      const double* bs = as + Cfg::A_ELEMS;
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {  // past K the TMA zero-filled both operands
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(ks + lc) * Cfg::LDA_S + wm * Cfg::WTM + i * 8 + lr];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          const int n = wn * Cfg::WTN + j * 8 + lr;
          bf[j] = TB ? bs[(ks + lc) * Cfg::LDB_S + n] : bs[n * Cfg::LDB_S + ks + lc];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
        double* cc = C + (long long)gn * ldc + m0 + wm * Cfg::WTM + lr;
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
          if (gn < N && m0 + wm * Cfg::WTM + i * 8 + lr < M) cc[i * 8] = negb ? neg_bits(acc[i][j][h]) : acc[i][j][h];
      }
  }
}

// Variant of rankk_tile_kernel with the C tile staged in shared memory by the
// producer (TMA box {130, 64}: pitch 130 makes the (row, 2-column) fragment
// reads conflict-free), one tile ahead behind a c_full / c_empty pair of
// mbarriers, so the consumers need registers for the accumulators only (no
// next-tile C fragment: the register-resident version spills at the 168-register
// cap of 9 warps, and its reloads stalled the K = 64 update).
template <bool TB, int S>
struct RankkTileCCfg {
  using G = DgemmWsCfg<false, TB, S>;
  static constexpr int LDC_S = 130;
  static constexpr int C_ELEMS = LDC_S * G::BN;
  static constexpr int SMEM_BYTES = (S * G::STAGE + C_ELEMS) * 8 + 128;
};

template <bool TB, int S>
__global__ void __launch_bounds__(288, 1)
    rankk_tilec_kernel(GemmDesc P, const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                       const __grid_constant__ CUtensorMap tC) {
  using Cfg = DgemmWsCfg<false, TB, S>;
  using CC = RankkTileCCfg<TB, S>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw + ((128u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u));
  double* cs = sm + S * Cfg::STAGE;  // C tile [n][m], pitch 130
  __shared__ __align__(8) uint64_t full[S], empty[S], c_full, c_empty;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = P.m, N = P.n, K = P.k;
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN, ntiles = tm * tn;
  const int KT = (K + BK - 1) / BK;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    mbar_init(&c_full, 1);
    mbar_init(&c_empty, 8);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tB)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tC)) : "memory");
      const unsigned bytes = (unsigned)Cfg::STAGE * 8u;
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tc) {
        const int m0 = (t % tm) * BM, n0 = (t / tm) * BN;
        // C of this tile once the consumers have read the previous one
        if (tc > 0) mbar_wait(&c_empty, (tc - 1) & 1u);
        mbar_expect_tx(&c_full, (unsigned)CC::C_ELEMS * 8u);
        tma_load_2d(cs, &tC, m0, n0, &c_full);
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int st = it % S;
          if (it >= S) mbar_wait(&empty[st], ((it / S) - 1) & 1u);
          double* as = sm + st * Cfg::STAGE;
          double* bs = as + Cfg::A_ELEMS;
          mbar_expect_tx(&full[st], bytes);
          tma_load_2d(as, &tA, m0, kt * BK, &full[st]);
          if (TB) tma_load_2d(bs, &tB, n0, kt * BK, &full[st]);
          else tma_load_2d(bs, &tB, kt * BK, n0, &full[st]);
        }
      }
    }
    return;
  }
  const int cw = warp - 1;
  const int wm = cw % Cfg::WARPS_M, wn = cw / Cfg::WARPS_M;
  const int lr = lane >> 2, lc = lane & 3;
  double* __restrict__ C = P.C;
  const long long ldc = P.ldc;
  const bool negb = P.alpha == -1.0;
  int it = 0, tc = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tc) {
    const int m0 = (t % tm) * BM, n0 = (t / tm) * BN;
    double acc[Cfg::FM][Cfg::FN][2];
    mbar_wait(&c_full, tc & 1u);
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* cc = cs + (wn * Cfg::WTN + j * 8 + lc * 2 + h) * CC::LDC_S + wm * Cfg::WTM + lr;
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) acc[i][j][h] = negb ? neg_bits(cc[i * 8]) : cc[i * 8];
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&c_empty);
    for (int kt = 0; kt < KT; ++kt, ++it) {
      const int st = it % S;
      mbar_wait(&full[st], (it / S) & 1u);
      const double* as = sm + st * Cfg::STAGE;
      const double* bs = as + Cfg::A_ELEMS;
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(ks + lc) * Cfg::LDA_S + wm * Cfg::WTM + i * 8 + lr];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) {
          const int n = wn * Cfg::WTN + j * 8 + lr;
          bf[j] = TB ? bs[(ks + lc) * Cfg::LDB_S + n] : bs[n * Cfg::LDB_S + ks + lc];
        }
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
        double* cc = C + (long long)gn * ldc + m0 + wm * Cfg::WTM + lr;
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
          if (gn < N && m0 + wm * Cfg::WTM + i * 8 + lr < M) cc[i * 8] = negb ? neg_bits(acc[i][j][h]) : acc[i][j][h];
      }
  }
}

template <bool TB>
static int launch_rankk_tilec(cudaStream_t st, const GemmDesc& d, int sms) {
  constexpr int S = 3;
  using Cfg = DgemmWsCfg<false, TB, S>;
  using CC = RankkTileCCfg<TB, S>;
  CUtensorMap tA, tB, tC;
  if (make_tmap_2d(&tA, d.A, d.m, d.k, d.lda, Cfg::LDA_S, Cfg::BK)) return -1;
  if (TB) {
    if (make_tmap_2d(&tB, d.B, d.n, d.k, d.ldb, Cfg::LDB_S, Cfg::BK)) return -1;
  } else if (make_tmap_2d(&tB, d.B, d.k, d.n, d.ldb, Cfg::LDB_S, Cfg::BN)) {
    return -1;
  }
  if (make_tmap_2d(&tC, d.C, d.m, d.n, d.ldc, CC::LDC_S, Cfg::BN)) return -1;
  auto kern = rankk_tilec_kernel<TB, S>;
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM_BYTES));
  const long long ntiles = (long long)((d.m + Cfg::BM - 1) / Cfg::BM) * ((d.n + Cfg::BN - 1) / Cfg::BN);
  const int grid = (int)std::max(1LL, std::min<long long>(ntiles, sms));
  kern<<<grid, Cfg::THREADS, CC::SMEM_BYTES, st>>>(d, tA, tB, tC);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

template <bool TB>
static int launch_rankk_tile(cudaStream_t st, const GemmDesc& d, int sms) {
  constexpr int S = 4;
  using Cfg = DgemmWsCfg<false, TB, S>;
  CUtensorMap tA, tB;
  if (make_tmap_2d(&tA, d.A, d.m, d.k, d.lda, Cfg::LDA_S, Cfg::BK)) return -1;
  if (TB) {
    if (make_tmap_2d(&tB, d.B, d.n, d.k, d.ldb, Cfg::LDB_S, Cfg::BK)) return -1;
  } else if (make_tmap_2d(&tB, d.B, d.k, d.n, d.ldb, Cfg::LDB_S, Cfg::BN)) {
    return -1;
  }
  auto kern = rankk_tile_kernel<TB, S>;
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
  const long long ntiles = (long long)((d.m + Cfg::BM - 1) / Cfg::BM) * ((d.n + Cfg::BN - 1) / Cfg::BN);
  const int grid = (int)std::max(1LL, std::min<long long>(ntiles, sms));
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(d, tA, tB);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}



template <bool TA, bool TB>
static int launch_dgemm_ws(cudaStream_t st, const GemmDesc& d, int ksplit, int kchunk, long long cslice) {
  constexpr int S = 4;
  using Cfg = DgemmWsCfg<TA, TB, S>;
  CUtensorMap tA, tB;
  // op(A): !TA -> A is m x k (m contiguous); TA -> A is k x m (k contiguous)
  if (TA) {
    if (make_tmap_2d(&tA, d.A, d.k, d.m, d.lda, Cfg::LDA_S, Cfg::BM)) return -1;
  } else if (make_tmap_2d(&tA, d.A, d.m, d.k, d.lda, Cfg::LDA_S, Cfg::BK)) {
    return -1;
  }
  if (TB) {
    if (make_tmap_2d(&tB, d.B, d.n, d.k, d.ldb, Cfg::LDB_S, Cfg::BK)) return -1;
  } else if (make_tmap_2d(&tB, d.B, d.k, d.n, d.ldb, Cfg::LDB_S, Cfg::BN)) {
    return -1;
  }
  auto kern = dgemm_ws_kernel<TA, TB, S>;
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
  dim3 grid((d.m + Cfg::BM - 1) / Cfg::BM, (d.n + Cfg::BN - 1) / Cfg::BN, std::max(1, ksplit));
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(d, ksplit, kchunk, cslice, tA, tB);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// Route a single host descriptor (optionally split over K) to the TMA GEMM when
// its operands allow tensor maps and it is big enough; -1 = not taken.
static int try_dgemm_ws(cudaStream_t st, bool ta, bool tb, const GemmBatch* b) {
  if (!g_dgemm_ws || !b || b->count != 1) return -1;
  const GemmDesc& d = b->d[0];
  if (d.acol || d.ccol || d.m <= 0 || d.n <= 0 || d.k < 64) return -1;
  if ((reinterpret_cast<uintptr_t>(d.A) & 15) || (reinterpret_cast<uintptr_t>(d.B) & 15) || (d.lda & 1) ||
      (d.ldb & 1))
    return -1;
  const int ks = std::max(1, b->ksplit);
  if (ks > 1 && (b->kchunk & 3)) return -1;
  const long long tiles = (long long)((d.m + 127) / 128) * ((d.n + 63) / 64) * ks;
  // too few tiles for one CTA per SM (split-K products with long slices still
  // beat the 64x64 cp.async config from half a wave: g_dgemm_ws_min_tiles)
  if (tiles < (ks > 1 ? g_dgemm_ws_min_split_tiles : g_dgemm_ws_min_tiles)) return -1;
  if (!ta && !tb) return launch_dgemm_ws<false, false>(st, d, ks, b->kchunk, b->cslice);
  if (!ta && tb) return launch_dgemm_ws<false, true>(st, d, ks, b->kchunk, b->cslice);
  if (ta && !tb) return launch_dgemm_ws<true, false>(st, d, ks, b->kchunk, b->cslice);
  return launch_dgemm_ws<true, true>(st, d, ks, b->kchunk, b->cslice);
}

// ---------------------------------------------------------------------------
// The BDC merge products (bdc.py:701-747) on the TMA GEMM: device descriptors
// (one per blockIdx.z) whose A columns are gathered through `acol` and whose C
// columns are scattered through `ccol`.  All operands live in one stack of
// equally shaped ld x ld workspaces (W, Q, Us, Vs, S3, S4 carved back to back),
// so ONE pair of tensor maps over that stack serves every descriptor: op(A)
// stage column kk is one TMA box {BM + 4, 1} at (row0 + m0, stack column of
// acol[k0 + kk]), issued four columns per TMA gather4 instruction (BK / 4 per
// stage from the producer lane), and op(B) one box {BK + 4, BN}.  Past a descriptor's K the stage holds other data, so
// the consumers zero both fragments there (NaN-safe).
template <int S>
__global__ void __launch_bounds__(288, 1)
    dgemm_ws_gather_kernel(const GemmDesc* __restrict__ ddesc, const double* base, long long ld,
                           const __grid_constant__ CUtensorMap tAg, const __grid_constant__ CUtensorMap tB) {
  using Cfg = DgemmWsCfg<false, false, S>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  const GemmDesc P = ddesc[blockIdx.z];
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  if (m0 >= P.m || n0 >= P.n) return;
  if (P.k <= 0) {  // empty class block: the product is zero (beta = 0 overwrites)
    for (int idx = threadIdx.x; idx < BM * BN; idx += blockDim.x) {
      const int i = m0 + idx % BM, j = n0 + idx / BM;
      if (i < P.m && j < P.n) P.C[i + (long long)(P.ccol ? P.ccol[j] : j) * P.ldc] = 0.0;
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sm = reinterpret_cast<double*>(smem_raw + ((128u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 127u)) & 127u));
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = P.k;
  const int KT = (K + BK - 1) / BK;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      const long long offA = P.A - base, offB = P.B - base;
      const int rowA = (int)(offA % ld), colA = (int)(offA / ld);
      const int rowB = (int)(offB % ld), colB = (int)(offB / ld);
      const int* __restrict__ acol = P.acol;
      for (int kt = 0; kt < KT; ++kt) {
        const int st = kt % S;
        if (kt >= S) mbar_wait(&empty[st], ((kt / S) - 1) & 1u);
        double* as = sm + st * Cfg::STAGE;
        double* bs = as + Cfg::A_ELEMS;
        const int k0 = kt * BK;
        const int nk = min(BK, K - k0);
        const int ng = (nk + 3) >> 2;  // gather4 groups (a group's dst is 4 x 1056 B: 128-byte aligned)
        mbar_expect_tx(&full[st], (unsigned)(4 * ng * Cfg::LDA_S + Cfg::B_ELEMS) * 8u);
        for (int q = 0; q < ng; ++q) {
          int c[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) c[i] = colA + acol[k0 + min(4 * q + i, nk - 1)];  // tail: repeat (masked)
          // the box's inner start must be 16-byte aligned: odd rows start one row early
          tma_gather4(as + 4 * q * Cfg::LDA_S, &tAg, (rowA & ~1) + m0, c, &full[st]);
        }
        tma_load_2d(bs, &tB, (rowB & ~1) + k0, colB + n0, &full[st]);
      }
    }
    return;
  }
  const int cw = warp - 1;
  const int wm = cw % Cfg::WARPS_M, wn = cw / Cfg::WARPS_M;
  const int lr = lane >> 2, lc = lane & 3;
  // odd operand row offsets were loaded one row early (16-byte aligned box starts)
  const int shA = (int)((P.A - base) % ld) & 1, shB = (int)((P.B - base) % ld) & 1;
  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt % S;
    mbar_wait(&full[st], (kt / S) & 1u);
    const double* as = sm + st * Cfg::STAGE + shA;
    const double* bs = sm + st * Cfg::STAGE + Cfg::A_ELEMS + shB;
    const int kl = K - kt * BK;  // valid k of this stage (>= BK: full)
    if (kl >= BK) {
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(ks + lc) * Cfg::LDA_S + wm * Cfg::WTM + i * 8 + lr];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[j] = bs[(wn * Cfg::WTN + j * 8 + lr) * Cfg::LDB_S + ks + lc];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    } else {
      for (int ks = 0; ks < kl; ks += 4) {
        const bool ok = ks + lc < kl;
        double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = ok ? as[(ks + lc) * Cfg::LDA_S + wm * Cfg::WTM + i * 8 + lr] : 0.0;
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[j] = ok ? bs[(wn * Cfg::WTN + j * 8 + lr) * Cfg::LDB_S + ks + lc] : 0.0;
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  double* __restrict__ C = P.C;
  const long long ldc = P.ldc;
  const int* __restrict__ ccol = P.ccol;
  const double alpha = P.alpha;
  const int M = P.m, N = P.n;
#pragma unroll
  for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gn = n0 + wn * Cfg::WTN + j * 8 + lc * 2 + h;
      if (gn >= N) continue;
      double* cc = C + (long long)(ccol ? ccol[gn] : gn) * ldc;
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int gm = m0 + wm * Cfg::WTM + i * 8 + lr;
        if (gm < M) cc[gm] = alpha * acc[i][j][h];  // beta = 0 (merge products overwrite)
      }
    }
}

// Grouped merge products on the TMA GEMM when the workspaces form one stack
// (`base`, `nbuf` ld x ld buffers back to back, 16-byte aligned, ld even);
// -1 = not taken (caller falls back to dgemm_kernel with gather).
int gemm_launch_device_stack(cudaStream_t st, const GemmDesc* ddesc, int ndesc, int max_m, int max_n,
                             const double* base, long long ld, int nbuf) {
  if (!g_dgemm_ws || (ld & 1) || (reinterpret_cast<uintptr_t>(base) & 15) || ld * nbuf > (1LL << 31)) {
    if (g_ws_flags_host & 8) fprintf(stderr, "stack: precondition %d %lld %p\n", g_dgemm_ws, ld, (const void*)base);
    return -1;
  }
  constexpr int S = 4;
  using Cfg = DgemmWsCfg<false, false, S>;
  CUtensorMap tAg, tB;
  if (make_tmap_2d(&tAg, base, ld, ld * nbuf, ld, Cfg::LDA_S, 1)) {
    if (g_ws_flags_host & 8) fprintf(stderr, "stack: tAg encode failed\n");
    return -1;
  }
  if (make_tmap_2d(&tB, base, ld, ld * nbuf, ld, Cfg::LDB_S, Cfg::BN)) {
    if (g_ws_flags_host & 8) fprintf(stderr, "stack: tB encode failed\n");
    return -1;
  }
  auto kern = dgemm_ws_gather_kernel<S>;
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
  dim3 grid((max_m + Cfg::BM - 1) / Cfg::BM, (max_n + Cfg::BN - 1) / Cfg::BN, ndesc);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(ddesc, base, ld, tAg, tB);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

// Row tiles per work unit.  The CTAs take units round-robin, so the kernel's
// time is the largest per-CTA sum of unit costs: the unit's rows in tiles
// (the last tile may be short) plus a fixed start cost `s` for loading its B
// strip (measured: s ~ 0.05 tile for the K = 64 / 128-row config, ~0.25 for
// the K = 128 / 64-row one, i.e. s = KMAX / (8 MT)).  Candidates CHUNK,
// CHUNK/2, ..., 1; the largest within 2 % of the best makespan wins (large
// trailing matrices keep 8-tile units, small ones get short units that fill
// the 148 SMs).  g_rankk_chunk > 0 forces it (debug).
static int g_rankk_chunk = 0;
// Smallest C (m*n) routed to the streaming kernel: 512^2 (tools/rankk_min_ab.py: ORMBR of 1024^2
// 0.99 -> 0.95 ms; 256^2 no better).
static long long g_rankk_min_mn = 512LL * 512;
int set_rankk_min(long long mn) {
  g_rankk_min_mn = mn > 0 ? mn : 512LL * 512;
  return 0;
}
int set_rankk_chunk(int c) {
  g_rankk_chunk = c;
  return 0;
}
int rankk_chunk(int m, int strips, int tiles, int mt, int kmax, int cmax, int sms) {
  if (g_rankk_chunk > 0) return std::min(g_rankk_chunk, cmax);
  const unsigned long long key = ((unsigned long long)m << 40) ^ ((unsigned long long)strips << 20) ^
                                 ((unsigned long long)kmax << 8) ^ (unsigned long long)sms;
  thread_local std::unordered_map<unsigned long long, int> cache;
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const double s = (double)kmax / (8.0 * mt);
  const double last = (double)(m - (tiles - 1) * mt) / mt;  // rows of the short last tile, in tiles
  std::vector<double> load;
  double cost[8] = {0};
  double best = 1e300;
  int ci = 0;
  for (int c = cmax; c >= 1; c >>= 1, ++ci) {
    const int chunks = (tiles + c - 1) / c;
    const long long units = (long long)strips * chunks;
    const int grid = (int)std::max(1LL, std::min(units, (long long)sms));
    load.assign(grid, 0.0);
    for (long long u = 0; u < units; ++u) {
      const int ch = (int)(u % chunks);
      const int nt = std::min(c, tiles - ch * c);
      const bool has_last = ch == chunks - 1;
      load[u % grid] += (has_last ? nt - 1 + last : nt) + s;
    }
    cost[ci] = *std::max_element(load.begin(), load.end());
    best = std::min(best, cost[ci]);
  }
  int pick = 1;
  ci = 0;
  for (int c = cmax; c >= 1; c >>= 1, ++ci)
    if (cost[ci] <= 1.02 * best) {
      pick = c;
      break;
    }
  cache.emplace(key, pick);
  return pick;
}

template <bool TB, int KMAX, int MT, int WARPS_M, bool VEC>
static int launch_rankk_v(cudaStream_t st, const GemmDesc& d, int sms) {
  using Cfg = RankkCfg<TB, KMAX, MT, WARPS_M>;
  auto kern = rankk_stream_kernel<TB, KMAX, MT, WARPS_M, VEC>;
  DC_CUDA_TRY((cudaError_t)func_attr(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
  const int strips = (d.n + 63) / 64;
  const int tiles = (d.m + MT - 1) / MT;
  const int chunk = rankk_chunk(d.m, strips, tiles, MT, KMAX, Cfg::CHUNK, sms);
  const int units = strips * ((tiles + chunk - 1) / chunk);
  const int grid = std::max(1, std::min(units, sms));
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(d, chunk);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

template <bool TB, int KMAX, int MT, int WARPS_M>
static int launch_rankk(cudaStream_t st, const GemmDesc& d, int sms) {
  const bool vec = !((reinterpret_cast<uintptr_t>(d.A) & 15) || (reinterpret_cast<uintptr_t>(d.B) & 15) ||
                     (d.lda & 1) || (d.ldb & 1));
  if (vec) return launch_rankk_v<TB, KMAX, MT, WARPS_M, true>(st, d, sms);
  return launch_rankk_v<TB, KMAX, MT, WARPS_M, false>(st, d, sms);
}

static int g_sms = 0;
static int sm_count() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

// Route rank-k updates (K <= 128, M x N >= 512^2, plain strided operands) to the
// streaming kernel.  Returns -1 when the shape does not qualify.
static int try_dgemm_ws(cudaStream_t st, bool ta, bool tb, const GemmBatch* b);
static int try_rankk(cudaStream_t st, bool ta, bool tb, const GemmDesc& d) {
  if (g_gemm_route != 0) return -1;
  if (ta || d.acol || d.ccol || d.k < 1 || d.k > 128 || d.beta == 0.0) return -1;
  if ((long long)d.m * d.n < g_rankk_min_mn || d.m < 256) return -1;
  const int sms = sm_count();
  if (g_dgemm_ws == 2 && d.k > 64) {  // debug: rank-k updates on the (non-persistent) general TMA GEMM
    GemmBatch b;
    b.d[0] = d;
    b.count = 1;
    const int r = try_dgemm_ws(st, ta, tb, &b);
    if (r >= 0) return r;
  }
  // Every rank-k update with beta = 1, alpha = +-1 (GEBRD A -= P Q^T at K = 64,
  // the 128-wide CWY updates of ORMBR / GEQRF / ORGQR at K = 128): the
  // persistent 128 x 64-tile TMA kernel with the C tile staged in shared memory
  // (8160^2 K = 64: 21.5 -> 29.7 TFLOP/s; 8192^2 K = 128: 24.9 -> 32.9; C2
  // 639 -> 626 ms; tools/rankk_tile_ab.py).  dcsvd_debug_dgemm_ws(3): the
  // register-prefetch variant; (0): the cp.async streaming kernel.
  const bool fold_ok = d.beta == 1.0 && (d.alpha == 1.0 || d.alpha == -1.0);
  if (g_dgemm_ws && g_dgemm_ws != 3 && fold_ok &&
      !((reinterpret_cast<uintptr_t>(d.A) & 15) || (reinterpret_cast<uintptr_t>(d.B) & 15) ||
        (reinterpret_cast<uintptr_t>(d.C) & 15) || (d.lda & 1) || (d.ldb & 1) || (d.ldc & 1))) {
    const int r = tb ? launch_rankk_tilec<true>(st, d, sms) : launch_rankk_tilec<false>(st, d, sms);
    if (r >= 0) return r;
  }
  if (g_dgemm_ws && (d.k > 64 || g_dgemm_ws == 3) && d.beta == 1.0 && (d.alpha == 1.0 || d.alpha == -1.0) &&
      !((reinterpret_cast<uintptr_t>(d.A) & 15) || (reinterpret_cast<uintptr_t>(d.B) & 15) || (d.lda & 1) || (d.ldb & 1))) {
    const int r = tb ? launch_rankk_tile<true>(st, d, sms) : launch_rankk_tile<false>(st, d, sms);
    if (r >= 0) return r;
  }
  // TMA tensor maps need 16-byte-aligned bases and leading dimensions.  The
  // warp-specialized kernel wins for K > 64 (8192^2 K = 128: 24.0 -> 24.9
  // TFLOP/s, C2 ORMBR 90.0 -> 87.3 ms); at K <= 64 (GEBRD trailing update)
  // the streaming kernel stays ahead (21.6 vs 19.9 at 8160^2), see DESIGN.md.
  const bool ws_ok = g_rankk_ws && d.k > 64 &&
                     !((reinterpret_cast<uintptr_t>(d.A) & 15) || (reinterpret_cast<uintptr_t>(d.B) & 15) ||
                       (reinterpret_cast<uintptr_t>(d.C) & 15) || (d.lda & 1) || (d.ldb & 1) || (d.ldc & 1));
  if (ws_ok) {
    const int r = tb ? launch_rankk_ws<true, 128, 16, 3, 4>(st, d, sms, 64)
                     : launch_rankk_ws<false, 128, 16, 3, 4>(st, d, sms, 64);
    if (r >= 0) return r;  // -1: tensor map not encodable -> streaming kernel
  }
  if (d.k <= 64) return tb ? launch_rankk<true, 64, 128, 4>(st, d, sms) : launch_rankk<false, 64, 128, 4>(st, d, sms);
  return tb ? launch_rankk<true, 128, 64, 2>(st, d, sms) : launch_rankk<false, 128, 64, 2>(st, d, sms);
}

static int dispatch(cudaStream_t st, bool ta, bool tb, const GemmBatch* b, const GemmDesc* dd, int nz,
                    int max_m, int max_n, int max_k, bool beta_nz) {
  if (max_m <= 0 || max_n <= 0 || nz <= 0) return 0;
  if (!ta && !tb) return launch_sized<false, false>(st, b, dd, nz, max_m, max_n, max_k, beta_nz);
  if (!ta && tb) return launch_sized<false, true>(st, b, dd, nz, max_m, max_n, max_k, beta_nz);
  if (ta && !tb) return launch_sized<true, false>(st, b, dd, nz, max_m, max_n, max_k, beta_nz);
  return launch_sized<true, true>(st, b, dd, nz, max_m, max_n, max_k, beta_nz);
}

int gemm_launch(cudaStream_t st, bool ta, bool tb, const GemmDesc& d) {
  if (d.m <= 0 || d.n <= 0) return 0;
  // kernel-family timing (dcsvd_set_stats, kind 1 = DMMA GEMM flops)
  const int sidx = t_cur ? stat_begin(t_cur, 1, 2.0 * d.m * d.n * d.k, st) : -1;
  int r = try_rankk(st, ta, tb, d);
  if (r < 0) {
    GemmBatch b;
    b.d[0] = d;
    b.count = 1;
    r = try_dgemm_ws(st, ta, tb, &b);
    if (r < 0) r = dispatch(st, ta, tb, &b, nullptr, 1, d.m, d.n, d.k, d.beta != 0.0);
  }
  if (t_cur) stat_end(t_cur, sidx, st);
  return r;
}

int gemm_launch_batch(cudaStream_t st, bool ta, bool tb, const GemmBatch& b) {
  int mm = 0, nn = 0, kk = 0;
  bool bnz = false;
  double flops = 0.0;
  for (int i = 0; i < b.count; ++i) {
    bnz = bnz || b.d[i].beta != 0.0;
    mm = b.d[i].m > mm ? b.d[i].m : mm;
    nn = b.d[i].n > nn ? b.d[i].n : nn;
    kk = b.d[i].k > kk ? b.d[i].k : kk;
    flops += 2.0 * b.d[i].m * b.d[i].n * b.d[i].k;
  }
  const int sidx = t_cur ? stat_begin(t_cur, 1, flops, st) : -1;
  int r = try_dgemm_ws(st, ta, tb, &b);
  if (r < 0)
    r = dispatch(st, ta, tb, &b, nullptr, b.count * std::max(1, b.ksplit), mm, nn, b.ksplit > 1 ? b.kchunk : kk, bnz);
  if (t_cur) stat_end(t_cur, sidx, st);
  return r;
}

int gemm_launch_device(cudaStream_t st, bool ta, bool tb, const GemmDesc* ddesc, int ndesc, int max_m,
                       int max_n) {
  return dispatch(st, ta, tb, nullptr, ddesc, ndesc, max_m, max_n, max_m, false);
}

// ---------------------------------------------------------------------------
// GEMV (densecore.matvec_accumulate); not on the SVD hot path, exported for
// API completeness.  y <- alpha op(A) x + beta y.
__global__ void dgemv_t_kernel(int m, int n, double alpha, const double* __restrict__ A, long long lda,
                               const double* __restrict__ x, double beta, double* __restrict__ y) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  double s = 0.0;
  const double* a = A + (long long)j * lda;
  for (int i = lane; i < m; i += 32) s += a[i] * x[i];
  s = warp_sum(s);
  if (lane == 0) y[j] = alpha * s + (beta != 0.0 ? beta * y[j] : 0.0);
}
__global__ void dgemv_n_kernel(int m, int n, double alpha, const double* __restrict__ A, long long lda,
                               const double* __restrict__ x, double beta, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int j = 0; j < n; ++j) s += A[i + (long long)j * lda] * x[j];
  y[i] = alpha * s + (beta != 0.0 ? beta * y[i] : 0.0);
}

int gemv_launch(cudaStream_t st, bool ta, int m, int n, double alpha, const double* A, long long lda,
                const double* x, double beta, double* y) {
  if (ta) {
    if (n <= 0) return 0;
    dgemv_t_kernel<<<(n + 7) / 8, 256, 0, st>>>(m, n, alpha, A, lda, x, beta, y);
  } else {
    if (m <= 0) return 0;
    dgemv_n_kernel<<<(m + 255) / 256, 256, 0, st>>>(m, n, alpha, A, lda, x, beta, y);
  }
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace dc
