// C ABI of libdcsvd_b200 (include/dcsvd_b200.h) and the gesdd driver.
//
// Driver reference: pkg/src/dcsvd/driver.py:97-170 (_square_core,
// _gesdd_impl, gesdd, phase_profile).
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>
#include <functional>
#include <atomic>
#include <mutex>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ctx.cuh"
#include "gemm.cuh"
#include "launch.cuh"

namespace dc {
std::atomic<long long> g_launch_count{0};
extern unsigned long long* g_labrd_tlog;
extern int g_labrd_gmax;
extern int g_labrd_skip_zero;
extern int g_labrd2_rpl;
extern int g_labrd4_rpl;
extern double g_labrd_l2keep;
extern double g_labrd_l2keep_min;
extern int g_gebd2_cluster;
extern int g_g2c_max_cols;
int set_rankk_prefetch(int on);
int set_rankk_chunk(int c);
int set_rankk_bulk(int on);
int set_rankk_min(long long mn);
extern bool g_labrd_last_two_phase;
extern int g_labrd_halfwidth;
extern int g_ormbr_pre;
extern long long g_labrd_halfwidth_max;
extern int g_gemm_route;
extern int g_rankk_ws;
extern int g_dgemm_ws;
extern int g_dgemm_ws_min_split_tiles;
extern int g_dgemm_ws_min_tiles;
extern int g_cwy_split_mode;
extern int g_cwy_gsplit;
extern int g_qr_outer;
int g_ts_qr_nb = 0;   // debug: QR panel width of the TS pre-step (0 = options.qr_block)
int g_ormbr_overlap = 1;  // debug: 0 = ORMBR preparation after BDC (no overlap)
int g_ts_orgqr_overlap = 1;  // debug: 0 = TS-path ORGQR after the core SVD of R on the call's stream
int g_ts_literal = 1;  // TS recombination: 1 = ORGQR + GEMM (driver.py:141-142), 0 = fused reflector apply
int set_ws_flags(int f);
thread_local dcsvd_ctx* t_cur = nullptr;

int func_attr(const void* fn, int attr, int value) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, long long>, int>> done;  // ((fn, dev<<8|attr), value)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  const long long key = ((long long)dev << 8) | attr;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& r : done)
    if (r.first.first == fn && r.first.second == key && r.second == value) return 0;
  e = cudaFuncSetAttribute(fn, (cudaFuncAttribute)attr, value);
  if (e != cudaSuccess) return (int)e;
  for (auto& r : done)
    if (r.first.first == fn && r.first.second == key) {
      r.second = value;
      return 0;
    }
  done.push_back({{fn, key}, value});
  return 0;
}

int set_error(dcsvd_ctx* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (h) h->last_error = buf;
  return code;
}

int pool_reserve(dcsvd_ctx* h, int p, size_t bytes, cudaStream_t st) {
  DevPool& pl = h->pool[p];
  pl.used = 0;
  if (bytes <= pl.cap) return 0;
  if (pl.ptr) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(h, DCSVD_ECUDA, "CUDA error before regrow: %s", cudaGetErrorString(e));
    cudaFree(pl.ptr);
    pl.ptr = nullptr;
    pl.cap = 0;
  }
  size_t cap = bytes + bytes / 8 + (1 << 20);
  cudaError_t e = cudaMalloc(&pl.ptr, cap);
  if (e != cudaSuccess) {
    pl.ptr = nullptr;
    return set_error(h, DCSVD_ECUDA, "cudaMalloc(%zu) failed: %s", cap, cudaGetErrorString(e));
  }
  pl.cap = cap;
  return 0;
}

int stat_begin(dcsvd_ctx* h, int kind, double work, cudaStream_t st) {
  if (!h || !h->stats_on) return -1;
  dcsvd_ctx::StatRec r;
  r.kind = kind;
  r.work = work;
  for (cudaEvent_t* e : {&r.a, &r.b}) {
    if (!h->ev_free.empty()) {
      *e = h->ev_free.back();
      h->ev_free.pop_back();
    } else {
      cudaEventCreate(e);
    }
  }
  cudaEventRecord(r.a, st);
  h->stats.push_back(r);
  return (int)h->stats.size() - 1;
}
void stat_end(dcsvd_ctx* h, int idx, cudaStream_t st) {
  if (idx < 0) return;
  cudaEventRecord(h->stats[idx].b, st);
}

int check_device_status(dcsvd_ctx* h, cudaStream_t st, const char* stage) {
  cudaError_t e = cudaMemcpyAsync(h->h_err, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_error(h, DCSVD_ECUDA, "%s: CUDA error %s", stage, cudaGetErrorString(e));
  const int code = *h->h_err;
  if (code == kDevOk) return 0;
  cudaMemsetAsync(h->d_err, 0, sizeof(int), st);
  switch (code) {
    case kDevNoConvergeQR:
      return set_error(h, DCSVD_ENOCONV, "%s: bidiagonal QR iteration exceeded its rotation budget", stage);
    case kDevNoConvergeSecular:
      return set_error(h, DCSVD_ENOCONV, "%s: secular solver did not converge in 100 iterations", stage);
    case kDevInterlacing:
      return set_error(h, DCSVD_EARITH, "%s: root interlacing violated: non-positive radicand in z update", stage);
    case kDevSingularT:
      return set_error(h, DCSVD_ESINGULAR, "%s: triangular factor has a zero diagonal entry", stage);
    case kDevBadDeflate:
      return set_error(h, DCSVD_EINVAL, "%s: deflate expects one zero d entry (the border row)", stage);
    default:
      return set_error(h, DCSVD_EINVAL, "%s: device status %d", stage, code);
  }
}
}  // namespace dc

int dc_cuda_fail(cudaError_t e, const char* what) {
  if (dc::t_cur) dc::set_error(dc::t_cur, DCSVD_ECUDA, "CUDA error %s in %s", cudaGetErrorString(e), what);
  return DCSVD_ECUDA;
}

using namespace dc;

extern "C" {
static dcsvd_ctx* make_sub(dcsvd_ctx* h, int sms);
}

namespace {
struct Guard {
  Guard(dcsvd_ctx* h) {
    t_cur = h;
    if (h) cudaSetDevice(h->device);
  }
  ~Guard() { t_cur = nullptr; }
};
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__global__ void transpose_kernel(int rows, int cols, const double* __restrict__ A, long long lda, double* __restrict__ B,
                                 long long ldb) {
  // B (cols x rows) = A^T
  // 32x32 tiles, grid-strided over both dimensions (any rows/cols < 2^31)
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const long long tr = (rows + 31) / 32, tc = (cols + 31) / 32;
  for (long long t = blockIdx.x; t < tr * tc; t += gridDim.x) {
    const int bx = (int)(t % tr) * 32, by = (int)(t / tr) * 32;
    for (int k = ty; k < 32; k += 8) {
      const int r = bx + tx, c = by + k;
      tile[k][tx] = (r < rows && c < cols) ? A[r + (long long)c * lda] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int r = bx + k, c = by + tx;
      if (r < rows && c < cols) B[c + (long long)r * ldb] = tile[tx][k];
    }
    __syncthreads();
  }
}
int transpose(cudaStream_t st, int rows, int cols, const double* A, long long lda, double* B, long long ldb) {
  if (rows <= 0 || cols <= 0) return 0;
  const long long tiles = ((rows + 31LL) / 32) * ((cols + 31LL) / 32);
  transpose_kernel<<<(unsigned)std::min<long long>(tiles, 148LL * 16), 256, 0, st>>>(rows, cols, A, lda, B, ldb);
  note_launch();
  DC_CUDA_TRY(cudaGetLastError());
  return 0;
}

__global__ void triu_copy_kernel(int n, const double* __restrict__ A, long long lda, double* __restrict__ R,
                                 long long ldr) {
  const long long total = (long long)n * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    R[i + (long long)j * ldr] = i <= j ? A[i + (long long)j * lda] : 0.0;
  }
}

// Per-phase CUDA events (phase_profile) and NVTX ranges named after the
// reference's PHASE_NAMES (driver.py:31) around each phase's enqueue, so an
// nsys / ncu --nvtx timeline shows the pipeline stages.
struct PhaseTimer {
  bool on;
  cudaStream_t st;
  cudaEvent_t ev[16];
  int idx[16];
  int cnt = 0;
  bool nvtx_open = false;
  PhaseTimer(bool on_, cudaStream_t s) : on(on_), st(s) {}
  ~PhaseTimer() {
    if (nvtx_open) nvtxRangePop();
    for (int i = 0; i < cnt; ++i) cudaEventDestroy(ev[i]);
  }
  void mark(int phase) {  // phase = index into the profile struct (0..5), -1 = end marker
    static const char* kNames[6] = {"dcsvd:geqrf", "dcsvd:orgqr", "dcsvd:gebrd", "dcsvd:bdcdc", "dcsvd:ormqr+ormlq",
                                    "dcsvd:gemm"};
    if (nvtx_open) nvtxRangePop();
    nvtx_open = phase >= 0 && phase < 6;
    if (nvtx_open) nvtxRangePushA(kNames[phase]);
    if (!on || cnt >= 16) return;
    cudaEventCreate(&ev[cnt]);
    cudaEventRecord(ev[cnt], st);
    idx[cnt] = phase;
    ++cnt;
  }
  void collect(dcsvd_phase_times* p) {
    if (!on || !p) return;
    double* f[6] = {&p->geqrf, &p->orgqr, &p->gebrd, &p->bdcdc, &p->ormbr, &p->gemm};
    for (int i = 0; i + 1 < cnt; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      if (idx[i] >= 0) *f[idx[i]] += ms * 1e-3;
    }
    if (cnt >= 2) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0], ev[cnt - 1]);
      p->total = ms * 1e-3;
    }
  }
};
// device status of a side/sub context folded into the parent's (stream-ordered)
__global__ void merge_err_kernel(int* dst, int* src) {
  if (*src != 0 && *dst == 0) *dst = *src;
  *src = 0;
}

// Lazily created side context (whole-GPU handles only; batch sub-contexts
// already share the GPU).
static dcsvd_ctx* side_ctx(dcsvd_ctx* h) {
  if (h->is_sub) return nullptr;
  if (!h->side) {
    h->side = make_sub(h, h->sms);
    if (!h->side) return nullptr;
    if (cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_prep, cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
  }
  h->side->stats_on = h->stats_on;
  return h->side;
}
// Second lazily created side context (TS path: ORGQR of the tall QR runs on it
// while the core SVD of R does its BDC and back-transforms).
static dcsvd_ctx* side2_ctx(dcsvd_ctx* h) {
  if (h->is_sub) return nullptr;
  if (!h->side2) {
    h->side2 = make_sub(h, h->sms);
    if (!h->side2) return nullptr;
    if (cudaEventCreateWithFlags(&h->ev_fork2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_join2, cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
  }
  h->side2->stats_on = h->stats_on;
  return h->side2;
}
constexpr int kDriverCwyWidth = 128;
enum { PH_GEQRF = 0, PH_ORGQR, PH_GEBRD, PH_BDC, PH_ORMBR, PH_GEMM, PH_END = -1 };

// _square_core (driver.py:97-118) for m >= n.  A consumed.
int square_core(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda, double* S,
                double* U, long long ldu, double* VT, long long ldvt, const dcsvd_opts& o, PhaseTimer& pt,
                double* dbuf, const std::function<int()>* after_gebrd = nullptr) {
  double* d = dbuf;
  double* e = d + n;
  double* tq = e + n;
  double* tp = tq + n;
  pt.mark(PH_GEBRD);
  int rc = gebrd_run(h, st, m, n, A, lda, d, e, tq, tp, o.bidiag_block);
  if (rc) return rc;
  if (after_gebrd) {  // caller's independent work forked here (gesdd_tall: ORGQR on a third stream)
    rc = (*after_gebrd)();
    if (rc) return rc;
  }
  const bool vec = o.want_vectors != 0;
  // The U and V^T back-transforms are independent: on a whole-GPU handle the
  // V^T one runs on a side stream with its own workspace, so the small
  // kernels and wave tails of one fill the other's gaps.  Their preparation
  // (every CWY block's Y and op(T), qr.cu ormbr_prepare) needs only the
  // packed reflectors, so the side stream does it for both sides while BDC
  // runs on `st` (BDC uses pool 2 only; the U plan lives in pool 0 of h).
  dcsvd_ctx* sd = vec ? side_ctx(h) : nullptr;
  OrmbrPlan planU, planV;
  const bool overlap = sd && g_ormbr_overlap;
  auto join_side = [&]() {
    h->last_error = sd->last_error;
    cudaStreamSynchronize(sd->own_stream);
  };
  if (overlap) {
    DC_CUDA_TRY(cudaEventRecord(h->ev_fork, st));
    DC_CUDA_TRY(cudaStreamWaitEvent(sd->own_stream, h->ev_fork, 0));
    rc = ormbr_prepare(sd, sd->own_stream, 'P', true, m, n, A, lda, tp, n, n, kDriverCwyWidth, planV);
    if (!rc) rc = ormbr_prepare(h, sd->own_stream, 'Q', false, m, n, A, lda, tq, m, n, kDriverCwyWidth, planU);
    if (rc) {
      if (h->last_error.empty()) h->last_error = sd->last_error;
      cudaStreamSynchronize(sd->own_stream);
      return rc;
    }
    DC_CUDA_TRY(cudaEventRecord(h->ev_prep, sd->own_stream));
  }
  pt.mark(PH_BDC);
  rc = bdsdc_run(h, st, n, d, e, false, vec, o.leaf_size, o.deflation_multiple, S, nullptr, vec ? U : nullptr, ldu,
                 m, nullptr, 0, vec ? VT : nullptr, ldvt);
  if (rc) {
    if (overlap) cudaStreamSynchronize(sd->own_stream);
    return rc;
  }
  if (!vec) return 0;
  pt.mark(PH_ORMBR);
  // The driver groups reflectors into the widest CWY panels the GPU kernels
  // take (kDriverCwyWidth): T^-1 = triu(Y^T Y) + diag(1/tau) is exact for any
  // width, so this is the same product as the reference's 64-wide blocks
  // (backtransform.py:90-131) with fewer, larger DMMA GEMMs.
  if (!sd) {
    rc = ormbr_run(h, st, 'Q', false, m, n, A, lda, tq, U, m, n, ldu, kDriverCwyWidth);
    if (rc) return rc;
    return ormbr_run(h, st, 'P', true, m, n, A, lda, tp, VT, n, n, ldvt, kDriverCwyWidth);
  }
  DC_CUDA_TRY(cudaEventRecord(h->ev_fork, st));  // BDC done (U, V^T initialised)
  DC_CUDA_TRY(cudaStreamWaitEvent(sd->own_stream, h->ev_fork, 0));
  rc = overlap ? ormbr_apply(sd, sd->own_stream, planV, VT, ldvt)
               : ormbr_run(sd, sd->own_stream, 'P', true, m, n, A, lda, tp, VT, n, n, ldvt, kDriverCwyWidth);
  if (rc) {
    // join the side stream before reporting: its enqueued kernels may still
    // read A / tp and write VT, which the caller frees after an error
    join_side();
    return rc;
  }
  if (overlap) {
    DC_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_prep, 0));
    rc = planU.nblk ? ormbr_apply(h, st, planU, U, ldu) : 0;
  } else {
    rc = ormbr_run(h, st, 'Q', false, m, n, A, lda, tq, U, m, n, ldu, kDriverCwyWidth);
  }
  DC_CUDA_TRY(cudaEventRecord(h->ev_join, sd->own_stream));
  DC_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
  merge_err_kernel<<<1, 1, 0, st>>>(h->d_err, sd->d_err);
  note_launch();
  return rc;
}

int gesdd_tall(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda, double* S,
               double* U, long long ldu, double* VT, long long ldvt, const dcsvd_opts& o, PhaseTimer& pt) {
  const bool vec = o.want_vectors != 0;
  const bool ts = (double)m >= o.ts_crossover * (double)n && m > n;
  const bool literal = ts && vec && g_ts_literal;
  size_t need = pool_bytes(4 * n + 8, 8);
  if (ts) need += pool_bytes(n, 8) + pool_bytes((size_t)n * n, 8);
  if (literal) need += pool_bytes((size_t)n * n, 8) + pool_bytes((size_t)m * n, 8);
  int rc = pool_reserve(h, 1, need, st);
  if (rc) return rc;
  double* dbuf = pool_take<double>(h, 1, 4 * n + 8);
  if (!ts) return square_core(h, st, m, n, A, lda, S, U, ldu, VT, ldvt, o, pt, dbuf);
  // TS path (driver.py:132-143)
  double* tau = pool_take<double>(h, 1, n);
  double* R = pool_take<double>(h, 1, (size_t)n * n);
  pt.mark(PH_GEQRF);
  rc = geqrf_run(h, st, m, n, A, lda, tau, g_ts_qr_nb > 0 ? g_ts_qr_nb : o.qr_block);
  if (rc) return rc;
  triu_copy_kernel<<<std::min<long long>(148 * 8, (n * n + 255) / 256), 256, 0, st>>>((int)n, A, lda, R, n);
  note_launch();
  if (literal) {
    // the reference's own order (driver.py:133-142): core SVD of R -> U0;
    // Q = orgqr(QR, n) (m x n, 128-wide CWY blocks); U = Q U0 (one DMMA GEMM)
    double* U0 = pool_take<double>(h, 1, (size_t)n * n);
    double* Qw = pool_take<double>(h, 1, (size_t)m * n);
    // ORGQR needs only the QR reflectors: outside phase profiling it runs on a
    // third stream (own workspace) once the cooperative GEBRD of R is done, beside
    // R's BDC and back-transforms; phase_profile keeps the sequential order so
    // every PHASE_NAMES phase is timed on the call's stream.
    dcsvd_ctx* s2 = (!pt.on && g_ts_orgqr_overlap) ? side2_ctx(h) : nullptr;
    bool forked = false;
    const std::function<int()> fork_orgqr = [&]() -> int {
      DC_CUDA_TRY(cudaEventRecord(h->ev_fork2, st));
      DC_CUDA_TRY(cudaStreamWaitEvent(s2->own_stream, h->ev_fork2, 0));
      forked = true;
      const int r2 = orgqr_run(s2, s2->own_stream, m, n, n, A, lda, tau, Qw, m, kDriverCwyWidth);
      if (r2) {
        h->last_error = s2->last_error;
        return r2;
      }
      DC_CUDA_TRY(cudaEventRecord(h->ev_join2, s2->own_stream));
      return 0;
    };
    rc = square_core(h, st, n, n, R, n, S, U0, n, VT, ldvt, o, pt, dbuf, s2 ? &fork_orgqr : nullptr);
    if (rc) {
      if (forked) cudaStreamSynchronize(s2->own_stream);  // its kernels read A / tau and write Qw
      return rc;
    }
    pt.mark(PH_ORGQR);
    if (s2) {
      DC_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join2, 0));
      merge_err_kernel<<<1, 1, 0, st>>>(h->d_err, s2->d_err);
      note_launch();
    } else {
      rc = orgqr_run(h, st, m, n, n, A, lda, tau, Qw, m, kDriverCwyWidth);
      if (rc) return rc;
    }
    pt.mark(PH_GEMM);
    GemmDesc gd{(int)m, (int)n, (int)n, Qw, m, nullptr, U0, n, U, ldu, nullptr, 1.0, 0.0};
    return gemm_launch(st, false, false, gd);
  }
  // the core SVD of R writes its left vectors U0 straight into the top n rows of U
  rc = square_core(h, st, n, n, R, n, S, vec ? U : nullptr, ldu, VT, ldvt, o, pt, dbuf);
  if (rc || !vec) return rc;
  // Fused recombination (dcsvd_debug_ts_literal(0)): U = Q [U0; 0] as the n QR
  // reflectors applied to [U0; 0] in 128-wide CWY blocks -- the same product
  // with 4mn^2 - 2n^3 flops and no m x n Q.
  pt.mark(PH_GEMM);
  if (m > n) DC_CUDA_TRY(cudaMemset2DAsync(U + n, sizeof(double) * ldu, 0, sizeof(double) * (m - n), n, st));
  return ormbr_run(h, st, 'Q', false, m, n, A, lda, tau, U, m, n, ldu, kDriverCwyWidth);
}

int validate_opts(dcsvd_ctx* h, const dcsvd_opts& o) {
  if (o.bidiag_block < 1 || o.qr_block < 1 || o.orgqr_block < 1 || o.apply_block < 1 || o.leaf_size < 1)
    return set_error(h, DCSVD_EINVAL, "block sizes must be >= 1");
  if (!(o.ts_crossover >= 1.0)) return set_error(h, DCSVD_EINVAL, "ts_crossover must be >= 1");
  if (!(o.deflation_multiple > 0.0)) return set_error(h, DCSVD_EINVAL, "deflation_multiple must be > 0");
  return 0;
}

dcsvd_opts default_opts() {
  dcsvd_opts o;
  o.want_vectors = 1; o.bidiag_block = 32; o.qr_block = 32; o.orgqr_block = 64; o.apply_block = 64;
  o.leaf_size = 32; o.ts_crossover = 5.0 / 3.0; o.deflation_multiple = 8.0;
  return o;
}

int gesdd_impl(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda, double* S,
               double* U, long long ldu, double* VT, long long ldvt, const dcsvd_opts& o, PhaseTimer& pt) {
  if (m < 1 || n < 1) return set_error(h, DCSVD_EINVAL, "matrix must be nonempty, got %lldx%lld", m, n);
  if (m >= n) return gesdd_tall(h, st, m, n, A, lda, S, U, ldu, VT, ldvt, o, pt);
  // wide: SVD of A^T (driver.py:125-131)
  const bool vec = o.want_vectors != 0;
  // At (n x m), U' (n x m), VT' (m x m) live in pool 1's tail: reserve separately
  // through a dedicated allocation (pool 1 is re-reserved by gesdd_tall).
  double *At = nullptr, *Up = nullptr, *VTp = nullptr;
  size_t bytes = sizeof(double) * ((size_t)n * m + (vec ? (size_t)n * m + (size_t)m * m : 0));
  char* blk = nullptr;
  DC_CUDA_TRY(cudaMallocAsync((void**)&blk, bytes, st));
  At = (double*)blk;
  if (vec) {
    Up = At + (size_t)n * m;
    VTp = Up + (size_t)n * m;
  }
  int rc = transpose(st, (int)m, (int)n, A, lda, At, n);
  if (!rc) rc = gesdd_tall(h, st, n, m, At, n, S, Up, n, VTp, m, o, pt);
  if (!rc && vec) {
    rc = transpose(st, (int)m, (int)m, VTp, m, U, ldu);          // U = VT'^T (m x m)
    if (!rc) rc = transpose(st, (int)n, (int)m, Up, n, VT, ldvt);  // VT = U'^T (m x n)
  }
  cudaFreeAsync(blk, st);
  return rc;
}
}  // namespace

extern "C" {

int dcsvd_version(void) { return 100; }

// Debug hook (not in the public header): record per-phase timestamps of the
// next LABRD launch into a device buffer of >= 1 + 10*nb u64.
int dcsvd_debug_labrd_tlog(unsigned long long* dev_buf) {
  dc::g_labrd_tlog = dev_buf;
  return 0;
}

/* 1 when the last LABRD panel launch used the two-phase kernel (debug). */
/* number of concurrent batch sub-contexts (streams) of a handle (debug) */
int dcsvd_debug_batch_streams(dcsvd_handle h) { return h ? (int)h->subs.size() : 0; }

int dcsvd_debug_gemm_route(int mode) {
  dc::g_gemm_route = mode;
  return 0;
}

int dcsvd_debug_ts_qr_nb(int nb) {
  dc::g_ts_qr_nb = nb;
  return 0;
}
int dcsvd_debug_ts_literal(int on) {
  dc::g_ts_literal = on;
  return 0;
}
int dcsvd_debug_ws_flags(int f) { return dc::set_ws_flags(f); }
// debug: grouped stack GEMM on host-built descriptors (copied to the device here)
int dcsvd_debug_gemm_stack(dcsvd_handle h, const void* descs, int ndesc, int max_m, int max_n, const double* base,
                           int64_t ld, int nbuf, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  dc::GemmDesc* dd = nullptr;
  DC_CUDA_TRY(cudaMalloc(&dd, sizeof(dc::GemmDesc) * ndesc));
  DC_CUDA_TRY(cudaMemcpy(dd, descs, sizeof(dc::GemmDesc) * ndesc, cudaMemcpyHostToDevice));
  int rc = dc::gemm_launch_device_stack(S(stream), dd, ndesc, max_m, max_n, base, ld, nbuf);
  cudaError_t e = cudaStreamSynchronize(S(stream));
  cudaFree(dd);
  if (rc) return rc;
  return e == cudaSuccess ? 0 : dc_cuda_fail(e, "gemm_stack");
}
int dcsvd_debug_qr_outer(int w) {
  dc::g_qr_outer = w;
  return 0;
}
int dcsvd_debug_cwy_gsplit(int on) {
  dc::g_cwy_gsplit = on;
  return 0;
}
int dcsvd_debug_cwy_split(int mode) {
  dc::g_cwy_split_mode = mode;
  return 0;
}
int dcsvd_debug_dgemm_ws_min_nosplit(int tiles) {
  dc::g_dgemm_ws_min_tiles = tiles;
  return 0;
}
int dcsvd_debug_dgemm_ws_min(int tiles) {
  dc::g_dgemm_ws_min_split_tiles = tiles;
  return 0;
}
int dcsvd_debug_dgemm_ws(int on) {
  dc::g_dgemm_ws = on;
  return 0;
}
int dcsvd_debug_rankk_ws(int on) {
  dc::g_rankk_ws = on;
  return 0;
}
int dcsvd_debug_labrd_variant(void) { return dc::g_labrd_last_two_phase ? 2 : 4; }

/* GEBD2 tail on one thread-block cluster (1, default; 8 = force 8-CTA clusters) or the panel path only (0); debug */
/* largest trailing block (columns) handed to the cluster GEBD2 kernel (debug / tuning; default 512) */
int dcsvd_debug_gebd2_max_cols(int n) {
  dc::g_g2c_max_cols = n > 0 ? n : 512;
  return 0;
}

int dcsvd_debug_gebd2_cluster(int on) {
  dc::g_gebd2_cluster = on;
  return 0;
}

/* L2 prefetch of the next C tile in the streaming rank-k kernel (debug / tuning) */
int dcsvd_debug_rankk_prefetch(int on) { return dc::set_rankk_prefetch(on); }

/* row tiles per work unit of the streaming rank-k kernel (0 = automatic; debug / tuning) */
int dcsvd_debug_rankk_chunk(int c) { return dc::set_rankk_chunk(c); }

/* A tiles of the streaming rank-k kernel by TMA bulk copies (1, default) or cp.async (0); debug */
int dcsvd_debug_rankk_bulk(int on) { return dc::set_rankk_bulk(on); }

/* smallest C size (m*n) routed to the streaming rank-k kernel (<= 0: default 512^2); debug */
int dcsvd_debug_rankk_min(long long mn) { return dc::set_rankk_min(mn); }

/* L2 bytes of each large-panel GEMV pass loaded evict_last (0 = plain loads; debug / tuning) */
int dcsvd_debug_labrd_l2keep(double bytes) {
  dc::g_labrd_l2keep = bytes;
  return 0;
}

/* smallest panel matrix (bytes) that uses the L2 hints (debug / tuning) */
int dcsvd_debug_labrd_l2keep_min(double bytes) {
  dc::g_labrd_l2keep_min = bytes;
  return 0;
}

/* half-width GEBRD panels where they let the two-phase LABRD kernel run (1, default) or never (0);
   max_elems bounds the view size (m'*n') that gets them (<= 0: no bound); debug / tuning */
int dcsvd_debug_labrd_halfwidth(int on, long long max_elems) {
  dc::g_labrd_halfwidth = on;
  dc::g_labrd_halfwidth_max = max_elems > 0 ? max_elems : (1LL << 62);
  return 0;
}

/* TS path: ORGQR on a third stream beside the core SVD of R (1, default) or after it (0); debug */
int dcsvd_debug_ts_orgqr_overlap(int on) {
  dc::g_ts_orgqr_overlap = on;
  return 0;
}

/* ORMBR preparation on the side stream during BDC (1, default) or after it (0); debug */
int dcsvd_debug_ormbr_overlap(int on) {
  dc::g_ormbr_overlap = on;
  return 0;
}

/* ORMBR: op(T) of all full CWY blocks precomputed in batched launches (1, default) or per block (0); debug */
int dcsvd_debug_ormbr_pre(int on) {
  dc::g_ormbr_pre = on;
  return 0;
}

/* force the two-phase LABRD geometry (rows per lane 2/4/8/16; 0 = automatic; debug / tuning) */
int dcsvd_debug_labrd4_rpl(int rpl) {
  dc::g_labrd4_rpl = rpl;
  return 0;
}

int dcsvd_debug_labrd2_rpl(int rpl) {
  dc::g_labrd2_rpl = rpl;
  return 0;
}

/* GEBRD panels skip the P / Q zero fill (1, default) or zero them like labrd_panel (0); debug */
int dcsvd_debug_labrd_skip_zero(int on) {
  dc::g_labrd_skip_zero = on;
  return 0;
}

/* cap the LABRD panel grid at gmax CTAs (0 = all SMs; debug / tuning) */
int dcsvd_debug_labrd_gmax(int gmax) {
  dc::g_labrd_gmax = gmax;
  return 0;
}

int dcsvd_create(dcsvd_handle* out, int device) {
  if (!out) return DCSVD_EINVAL;
  *out = nullptr;
  dcsvd_ctx* h = new dcsvd_ctx();
  h->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete h;
    return DCSVD_ECUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    delete h;
    return DCSVD_ECUDA;
  }
  h->sms = prop.multiProcessorCount;
  h->coop_ok = prop.cooperativeLaunch;
  if (cudaMalloc(&h->d_err, sizeof(int)) != cudaSuccess || cudaMalloc(&h->d_bar, sizeof(unsigned) * kNumBars) != cudaSuccess ||
      cudaMallocHost(&h->h_err, sizeof(int)) != cudaSuccess || cudaMalloc(&h->d_flops, 2 * sizeof(double)) != cudaSuccess) {
    delete h;
    return DCSVD_ECUDA;
  }
  cudaMemset(h->d_err, 0, sizeof(int));
  cudaMemset(h->d_bar, 0, sizeof(unsigned) * kNumBars);
  cudaDeviceSynchronize();
  *out = h;
  return 0;
}

static void free_ctx_resources(dcsvd_ctx* h);

int dcsvd_destroy(dcsvd_handle h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  free_ctx_resources(h);
  delete h;
  return 0;
}

int dcsvd_set_stats(dcsvd_handle h, int enable) {
  if (!h) return DCSVD_EINVAL;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (auto& r : h->stats) {
    h->ev_free.push_back(r.a);
    h->ev_free.push_back(r.b);
  }
  h->stats.clear();
  h->stats_on = enable != 0;
  if (h->d_flops) cudaMemset(h->d_flops, 0, 2 * sizeof(double));
  if (!h->ev_stats0) cudaEventCreate(&h->ev_stats0);
  cudaEventRecord(h->ev_stats0, 0);  // after the device synchronize above: precedes every record
  cudaEventSynchronize(h->ev_stats0);
  for (auto* sub : h->subs) dcsvd_set_stats(sub, enable);  // batched sub-contexts record too
  if (h->side) dcsvd_set_stats(h->side, enable);
  if (h->side2) dcsvd_set_stats(h->side2, enable);
  return 0;
}

// Debug (not in the public header): per-launch records of a kernel family.
int dcsvd_debug_stat_records(dcsvd_handle h, int kind, double* ms, double* work, int cap) {
  if (!h) return -1;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  int c = 0;
  for (auto& r : h->stats) {
    if (r.kind != kind) continue;
    if (c < cap) {
      float x = 0.f;
      cudaEventElapsedTime(&x, r.a, r.b);
      ms[c] = x;
      work[c] = r.work;
    }
    ++c;
  }
  return c;
}

// Kernel-family timing: `ms` = wall-clock time during which at least one
// launch of the family was running (union of the launch intervals over this
// handle's streams, its side stream and batch sub-contexts), `work` = summed
// algorithmic work, `launches` = count.
static void collect_stats(dcsvd_ctx* h, cudaEvent_t origin, int kind, std::vector<std::pair<double, double>>& iv,
                          double& work, long long& count) {
  for (auto& r : h->stats) {
    if (r.kind != kind) continue;
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, origin, r.a) == cudaSuccess && cudaEventElapsedTime(&b, origin, r.b) == cudaSuccess)
      iv.emplace_back(a, b);
    work += r.work;
    ++count;
  }
  if ((kind == 2 || kind == 3) && h->d_flops) {  // device-counted BDC merge flops / deflated-column bytes
    double f = 0.0;
    cudaMemcpy(&f, h->d_flops + (kind - 2), sizeof(double), cudaMemcpyDeviceToHost);
    work += f;
  }
  for (auto* sub : h->subs) collect_stats(sub, origin, kind, iv, work, count);
  if (h->side) collect_stats(h->side, origin, kind, iv, work, count);
  if (h->side2) collect_stats(h->side2, origin, kind, iv, work, count);
}

int dcsvd_get_stats(dcsvd_handle h, int kind, double* ms, double* work, long long* launches) {
  if (!h) return DCSVD_EINVAL;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  std::vector<std::pair<double, double>> iv;
  double w = 0.0;
  long long c = 0;
  if (h->ev_stats0) collect_stats(h, h->ev_stats0, kind, iv, w, c);
  std::sort(iv.begin(), iv.end());
  double t = 0.0, cur_a = 0.0, cur_b = -1.0;
  for (auto& p : iv) {
    if (p.first > cur_b) {
      if (cur_b > cur_a) t += cur_b - cur_a;
      cur_a = p.first;
      cur_b = p.second;
    } else if (p.second > cur_b) {
      cur_b = p.second;
    }
  }
  if (cur_b > cur_a) t += cur_b - cur_a;
  if (ms) *ms = t;
  if (work) *work = w;
  if (launches) *launches = c;
  return 0;
}

const char* dcsvd_last_error(dcsvd_handle h) { return h ? h->last_error.c_str() : "null handle"; }

long long dcsvd_launch_count(dcsvd_handle) { return g_launch_count.load(); }

int dcsvd_dgemm(dcsvd_handle h, int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
                int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  if (m < 0 || n < 0 || k < 0) return set_error(h, DCSVD_EINVAL, "negative GEMM dimension");
  if (m == 0 || n == 0) return 0;
  GemmDesc d;
  d.m = (int)m; d.n = (int)n; d.k = (int)k;
  d.A = A; d.lda = lda; d.acol = nullptr;
  d.B = B; d.ldb = ldb;
  d.C = C; d.ldc = ldc; d.ccol = nullptr;
  d.alpha = alpha; d.beta = beta;
  return gemm_launch(S(stream), transa != 0, transb != 0, d);
}

int dcsvd_dgemv(dcsvd_handle h, int transa, int64_t m, int64_t n, double alpha, const double* A, int64_t lda,
                const double* x, double beta, double* y, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return gemv_launch(S(stream), transa != 0, (int)m, (int)n, alpha, A, lda, x, beta, y);
}

int dcsvd_gebrd(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* d, double* e, double* tauq,
                double* taup, int nb, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return gebrd_run(h, S(stream), m, n, A, lda, d, e, tauq, taup, nb);
}

int dcsvd_labrd(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* d, double* e, double* tauq,
                double* taup, int nb, double* P, int64_t ldp, double* Q, int64_t ldq, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return labrd_run(h, S(stream), m, n, A, lda, nb, d, e, tauq, taup, P, ldp, Q, ldq);
}

int dcsvd_bdsdc(dcsvd_handle h, int64_t n, const double* d, const double* e, int bordered, int want_vectors, int leaf,
                double tol_multiple, double* dvals, double* W, int64_t ldw, double* Q, int64_t ldq, double* edge,
                void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  cudaStream_t st = S(stream);
  int rc = bdsdc_run(h, st, n, d, e, bordered != 0, want_vectors != 0, leaf, tol_multiple, dvals, edge,
                     want_vectors ? W : nullptr, ldw, n, want_vectors ? Q : nullptr, ldq, nullptr, 0);
  if (rc) return rc;
  return check_device_status(h, st, "bdsdc");
}

int dcsvd_geqrf(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* tau, int nb, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return geqrf_run(h, S(stream), m, n, A, lda, tau, nb);
}

int dcsvd_orgqr(dcsvd_handle h, int64_t m, int64_t nrefl, int64_t k, const double* A, int64_t lda, const double* tau,
                double* Q, int64_t ldq, int nb, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  int rc = orgqr_run(h, S(stream), m, nrefl, k, A, lda, tau, Q, ldq, nb);
  if (rc) return rc;
  return check_device_status(h, S(stream), "orgqr");
}

int dcsvd_ormbr(dcsvd_handle h, char vect, int trans, int64_t m, int64_t n, const double* A, int64_t lda,
                const double* tau, double* C, int64_t c_rows, int64_t c_cols, int64_t ldc, int nb, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  int rc = ormbr_run(h, S(stream), vect, trans != 0, m, n, A, lda, tau, C, c_rows, c_cols, ldc, nb);
  if (rc) return rc;
  return check_device_status(h, S(stream), "ormbr");
}

int dcsvd_gesdd(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* Sg, double* U, int64_t ldu,
                double* VT, int64_t ldvt, const dcsvd_opts* opts, dcsvd_phase_times* prof, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  dcsvd_opts o = opts ? *opts : default_opts();
  int rc = validate_opts(h, o);
  if (rc) return rc;
  cudaStream_t st = S(stream);
  if (prof) *prof = dcsvd_phase_times{0, 0, 0, 0, 0, 0, 0};
  PhaseTimer pt(prof != nullptr, st);
  pt.mark(PH_END);
  rc = gesdd_impl(h, st, m, n, A, lda, Sg, U, ldu, VT, ldvt, o, pt);
  pt.mark(PH_END);
  if (rc) return rc;
  rc = check_device_status(h, st, "gesdd");
  if (rc) return rc;
  pt.collect(prof);
  return 0;
}

static dcsvd_ctx* make_sub(dcsvd_ctx* h, int sms) {
  dcsvd_ctx* s = new dcsvd_ctx();
  s->device = h->device;
  s->sms = sms;
  s->coop_ok = h->coop_ok;
  s->is_sub = true;
  if (cudaMalloc(&s->d_err, sizeof(int)) != cudaSuccess || cudaMalloc(&s->d_bar, sizeof(unsigned) * kNumBars) != cudaSuccess ||
      cudaMalloc(&s->d_flops, 2 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&s->h_err, sizeof(int)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete s;
    return nullptr;
  }
  cudaMemset(s->d_err, 0, sizeof(int));
  cudaMemset(s->d_bar, 0, sizeof(unsigned) * kNumBars);
  cudaMemset(s->d_flops, 0, 2 * sizeof(double));
  return s;
}

static void free_ctx_resources(dcsvd_ctx* h) {
  for (auto* s : h->subs) {
    free_ctx_resources(s);
    delete s;
  }
  h->subs.clear();
  if (h->side) {
    free_ctx_resources(h->side);
    delete h->side;
    h->side = nullptr;
    cudaEventDestroy(h->ev_fork);
    cudaEventDestroy(h->ev_join);
    if (h->ev_prep) cudaEventDestroy(h->ev_prep);
  }
  if (h->side2) {
    free_ctx_resources(h->side2);
    delete h->side2;
    h->side2 = nullptr;
    if (h->ev_fork2) cudaEventDestroy(h->ev_fork2);
    if (h->ev_join2) cudaEventDestroy(h->ev_join2);
  }
  for (auto& p : h->pool)
    if (p.ptr) cudaFree(p.ptr);
  if (h->h_stage) cudaFreeHost(h->h_stage);
  if (h->ev_stage) cudaEventDestroy(h->ev_stage);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  cudaFree(h->d_err);
  cudaFree(h->d_bar);
  cudaFreeHost(h->h_err);
  if (h->d_flops) cudaFree(h->d_flops);
}

// Independent SVDs run concurrently: `conc` host threads each drive one
// sub-context (own stream, workspace, barrier counters) through its share of
// the batch; each sub-context's cooperative kernels use sms/conc CTAs, so the
// matrices in flight partition the GPU.  No data moves between them.
int dcsvd_gesdd_batched(dcsvd_handle h, int batch, int64_t m, int64_t n, double* const* A, int64_t lda,
                        double* const* Sg, double* const* U, int64_t ldu, double* const* VT, int64_t ldvt,
                        const dcsvd_opts* opts, int concurrency, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  dcsvd_opts o = opts ? *opts : default_opts();
  int rc = validate_opts(h, o);
  if (rc) return rc;
  if (batch <= 0) return 0;
  cudaStream_t st = S(stream);
  int conc = concurrency;
  if (conc <= 0) {
    const long long k = std::min(m, n);
    conc = k <= 2560 ? 8 : (k <= 4096 ? 4 : (k <= 6144 ? 2 : 1));
  }
  conc = std::max(1, std::min(conc, std::min(batch, 16)));
  {
    // each sub-context's cooperative LABRD grid needs sms/conc >= ceil(rows/512)
    // (gebrd.cu labrd_launch): clamp the concurrency to the GEBRD row count
    const long long M = std::max(m, n), K = std::min(m, n);
    const long long rows = (M >= o.ts_crossover * K && M > K) ? K : M;
    while (conc > 1 && (long long)(h->sms / conc) * 512 < rows) --conc;
  }
  if (conc == 1) {
    for (int b = 0; b < batch; ++b) {
      PhaseTimer pt(false, st);
      rc = gesdd_impl(h, st, m, n, A[b], lda, Sg[b], U ? U[b] : nullptr, ldu, VT ? VT[b] : nullptr, ldvt, o, pt);
      if (rc) return rc;
    }
    return check_device_status(h, st, "gesdd_batched");
  }
  const int sub_sms = std::max(1, h->sms / conc);
  while ((int)h->subs.size() < conc) {
    dcsvd_ctx* s = make_sub(h, sub_sms);
    if (!s) return set_error(h, DCSVD_ECUDA, "could not create a batch sub-context");
    h->subs.push_back(s);
  }
  for (int t = 0; t < conc; ++t) h->subs[t]->sms = sub_sms;
  // inputs are ready on `st`: sub-streams wait for it
  cudaEvent_t ready;
  DC_CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  DC_CUDA_TRY(cudaEventRecord(ready, st));
  for (int t = 0; t < conc; ++t) DC_CUDA_TRY(cudaStreamWaitEvent(h->subs[t]->own_stream, ready, 0));
  std::vector<int> codes(conc, 0);
  std::vector<std::thread> workers;
  for (int t = 0; t < conc; ++t) {
    workers.emplace_back([&, t]() {
      dcsvd_ctx* s = h->subs[t];
      Guard gg(s);
      int c = 0;
      for (int b = t; b < batch && c == 0; b += conc) {
        PhaseTimer pt(false, s->own_stream);
        c = gesdd_impl(s, s->own_stream, m, n, A[b], lda, Sg[b], U ? U[b] : nullptr, ldu, VT ? VT[b] : nullptr,
                       ldvt, o, pt);
      }
      if (c == 0)
        c = check_device_status(s, s->own_stream, "gesdd_batched");
      else
        cudaStreamSynchronize(s->own_stream);  // no enqueued work outlives the failed call
      codes[t] = c;
    });
  }
  for (auto& w : workers) w.join();
  cudaEventDestroy(ready);
  for (int t = 0; t < conc; ++t) {
    if (codes[t]) {
      h->last_error = h->subs[t]->last_error;
      return codes[t];
    }
  }
  // later work on `st` sees the results (all sub-streams were synchronized)
  return 0;
}

int dcsvd_larfg(dcsvd_handle h, int64_t n, const double* alpha, const double* x, int64_t incx, double* tau_beta,
                double* essential, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return larfg_run(h, S(stream), n, alpha, x, incx, tau_beta, essential);
}

int dcsvd_lartg(dcsvd_handle h, int64_t count, const double* a, const double* b, double* csr, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return lartg_run(h, S(stream), count, a, b, csr);
}

int dcsvd_trsm(dcsvd_handle h, char side, int trans, int64_t n, const double* T, int64_t ldt, double* B, int64_t ldb,
               int64_t other, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  if (side != 'L' && side != 'R') return set_error(h, DCSVD_EINVAL, "side must be 'left' or 'right'");
  int rc = trsm_run(h, S(stream), (int)n, T, ldt, B, ldb, other, side == 'R', trans != 0);
  if (rc) return rc;
  return check_device_status(h, S(stream), "triangular_solve");
}

int dcsvd_build_tinv(dcsvd_handle h, int64_t rows, int w, const double* Y, int64_t ldy, const double* tau, double* Tinv,
                     int64_t ldt, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return build_tinv_run(h, S(stream), rows, w, Y, ldy, tau, Tinv, ldt);
}

int dcsvd_block_reflector(dcsvd_handle h, char side, int trans, int64_t rows_y, int w, const double* Y, int64_t ldy,
                          const double* Tinv, int64_t ldt, double* C, int64_t ldc, int64_t c_other, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  if (side != 'L' && side != 'R') return set_error(h, DCSVD_EINVAL, "side must be 'L' or 'R'");
  int rc = block_reflector_run(h, S(stream), side, trans != 0, rows_y, w, Y, ldy, Tinv, ldt, C, ldc, c_other);
  if (rc) return rc;
  return check_device_status(h, S(stream), "apply_block_reflector");
}

int dcsvd_geqrf_panel(dcsvd_handle h, int64_t m, int w, double* A, int64_t lda, double* tau, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return geqr2_run(h, S(stream), m, w, A, lda, tau);
}

int dcsvd_secular_roots(dcsvd_handle h, int K, const double* d, const double* z, double* omega, int* anchor,
                        double* mu, int max_iterations, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  int rc = secular_run(h, S(stream), K, d, z, omega, anchor, mu, max_iterations);
  if (rc) return rc;
  return check_device_status(h, S(stream), "solve_all_roots");
}

int dcsvd_recompute_z(dcsvd_handle h, int K, const double* d, const double* z, const int* anchor, const double* mu,
                      double* ztilde, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  int rc = loewner_run(h, S(stream), K, d, z, anchor, mu, ztilde);
  if (rc) return rc;
  return check_device_status(h, S(stream), "recompute_z");
}

int dcsvd_secular_vectors(dcsvd_handle h, int K, const double* d, const int* anchor, const double* mu,
                          const double* ztilde, double* U, int64_t ldu, double* V, int64_t ldv, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return secvec_run(h, S(stream), K, d, anchor, mu, ztilde, U, ldu, V, ldv);
}

}  // extern "C"

int dcsvd_build_z(dcsvd_handle h, int nl, int nr, int bordered, double alpha, double beta, const double* left_dvals,
                  const double* left_edge, int64_t lde_l, const double* right_dvals, const double* right_edge,
                  int64_t lde_r, double* d, double* z, double* coupling, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return build_z_run(h, S(stream), nl, nr, bordered, alpha, beta, left_dvals, left_edge, lde_l, right_dvals,
                     right_edge, lde_r, d, z, coupling);
}

int dcsvd_deflate(dcsvd_handle h, int n, const double* d, const double* z, double tol_multiple, double* left,
                  int64_t rows_l, int64_t ldl, double* right, int64_t rows_r, int64_t ldr, double* edge, int64_t lde,
                  int* left_classes, int* right_classes, int64_t* perm, double* d_out, double* z_out, int64_t* kept,
                  int64_t* deflated, double* deflated_values, int64_t* rot_pq, double* rot_cs, int64_t* counts,
                  void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  static_assert(sizeof(long long) == sizeof(int64_t), "int64");
  int rc = deflate_run(h, S(stream), n, d, z, tol_multiple, left, rows_l, ldl, right, rows_r, ldr, edge, lde,
                       left_classes, right_classes, reinterpret_cast<long long*>(perm), d_out, z_out,
                       reinterpret_cast<long long*>(kept), reinterpret_cast<long long*>(deflated), deflated_values,
                       reinterpret_cast<long long*>(rot_pq), rot_cs, reinterpret_cast<long long*>(counts));
  if (rc) return rc;
  return check_device_status(h, S(stream), "deflate");
}

int dcsvd_gather(dcsvd_handle h, int64_t rows, int64_t cols, const double* src, int64_t lds, const int64_t* row_idx,
                 const int64_t* col_idx, double* dst, int64_t ldd, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return gather2d_run(h, S(stream), rows, cols, src, lds, reinterpret_cast<const long long*>(row_idx),
                      reinterpret_cast<const long long*>(col_idx), dst, ldd);
}

int dcsvd_philox(dcsvd_handle h, uint64_t key_lo, uint64_t key_hi, uint64_t word_offset, int64_t count, int normal,
                 double* out, int64_t rows, int64_t ld, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return philox_run(h, S(stream), key_lo, key_hi, word_offset, count, normal, out, rows, ld);
}

int dcsvd_prescribed_singular_values(dcsvd_handle h, int kind, int64_t n, double cond, uint64_t key_lo,
                                     uint64_t key_hi, double* sigma, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  return prescribed_sigma_run(h, S(stream), kind, (int)n, cond, key_lo, key_hi, sigma);
}

int dcsvd_generate_matrix(dcsvd_handle h, int kind, int64_t m, int64_t n, double cond, uint64_t key_lo,
                          uint64_t key_hi, double* A, int64_t lda, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  int rc = generate_run(h, S(stream), kind, m, n, cond, key_lo, key_hi, A, lda);
  if (rc) return rc;
  return kind == 0 ? 0 : check_device_status(h, S(stream), "generate_matrix");
}

int dcsvd_accuracy(dcsvd_handle h, int64_t m, int64_t n, const double* A, int64_t lda, const double* S_,
                   const double* U, int64_t ldu, const double* VT, int64_t ldvt, const double* ref_sigma,
                   double* report, void* stream) {
  Guard g(h);
  if (!h) return DCSVD_EINVAL;
  if (m < 1 || n < 1) return set_error(h, DCSVD_EINVAL, "accuracy: empty matrix");
  return accuracy_run(h, S(stream), m, n, A, lda, S_, U, ldu, VT, ldvt, ref_sigma, report);
}
