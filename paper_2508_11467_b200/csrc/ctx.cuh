// Handle state: device, scratch pools, status word, barrier counters.
#pragma once
#include <string>
#include <vector>

#include "common.cuh"

struct DevPool {
  char* ptr = nullptr;
  size_t cap = 0;
  size_t used = 0;
};

struct dcsvd_ctx {
  // concurrent sub-contexts for batched SVDs (own stream, pools, status word,
  // barrier counters, SM budget); created lazily by dcsvd_gesdd_batched
  std::vector<dcsvd_ctx*> subs;
  dcsvd_ctx* side = nullptr;    // second stream + workspace for independent stages (V^T back-transform)
  bool is_sub = false;          // batch / side sub-context (no further splitting)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // side-stream fork/join
  cudaEvent_t ev_prep = nullptr;  // side stream: ORMBR preparation done
  dcsvd_ctx* side2 = nullptr;     // third stream + workspace (TS path: ORGQR beside the core SVD of R)
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  cudaStream_t own_stream = nullptr;
  int device = 0;
  int sms = 148;
  int coop_ok = 1;
  std::string last_error;
  int* d_err = nullptr;         // device status word (dc::DevErr)
  unsigned* d_bar = nullptr;    // grid-barrier counters (kNumBars)
  int* h_err = nullptr;         // pinned mirror of d_err
  double* d_flops = nullptr;    // device-side counters: [0] BDC merge GEMM flops (stats kind 2), [1] deflated-column bytes (kind 3)
  DevPool pool[3];              // 0: stage scratch, 1: driver buffers, 2: bdc
  // optional per-kernel-family timing (bench roofline): CUDA events around
  // each launch of a family, with its algorithmic bytes/flops
  bool stats_on = false;
  struct StatRec {
    int kind;
    cudaEvent_t a, b;
    double work;
  };
  std::vector<StatRec> stats;
  std::vector<cudaEvent_t> ev_free;  // recycled timing events (no create/destroy per launch)
  cudaEvent_t ev_stats0 = nullptr;    // recorded when stats are (re)enabled: time origin of the records
  // pinned staging for small host->device uploads (BDC tree descriptors): the
  // copies stay asynchronous; ev_stage guards reuse of the buffer
  char* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  cudaEvent_t ev_stage = nullptr;
  bool stage_pending = false;
};

namespace dc {
constexpr int kNumBars = 64;

// Ensure pool `p` holds at least `bytes` (synchronizes `st` before a regrow so
// in-flight kernels never see a freed buffer), reset its bump pointer.
int pool_reserve(dcsvd_ctx* h, int p, size_t bytes, cudaStream_t st);
// Carve `count` doubles (256-byte aligned) from pool `p`.
template <typename T>
inline T* pool_take(dcsvd_ctx* h, int p, size_t count) {
  DevPool& pl = h->pool[p];
  size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
  if (pl.used + bytes > pl.cap) return nullptr;
  T* r = reinterpret_cast<T*>(pl.ptr + pl.used);
  pl.used += bytes;
  return r;
}
inline size_t pool_bytes(size_t count, size_t elem) { return (count * elem + 255) & ~size_t(255); }

int set_error(dcsvd_ctx* h, int code, const char* fmt, ...);
// stats helpers: stat_begin returns an index (or -1 when disabled)
int stat_begin(dcsvd_ctx* h, int kind, double work, cudaStream_t st);
void stat_end(dcsvd_ctx* h, int idx, cudaStream_t st);
// Read and reset the device status word (synchronizes the stream); maps it
// to an API status code with a message.
int check_device_status(dcsvd_ctx* h, cudaStream_t st, const char* stage);

// stage entry points (all stream-ordered on `st`)
int gebrd_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda,
              double* d, double* e, double* tauq, double* taup, int nb);
int labrd_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda, int nb, double* d,
              double* e, double* tauq, double* taup, double* P, long long ldp, double* Q, long long ldq);
int geqrf_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, double* A, long long lda,
              double* tau, int nb);
int orgqr_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long nrefl, long long k, const double* A,
              long long lda, const double* tau, double* Q, long long ldq, int nb);
// Left apply of column reflectors stored below the diagonal of A (rows >= j of
// reflector j, offset `roff` = 0) or right apply of row reflectors stored right
// of the superdiagonal (offset 1).  See qr.cu.
// ORMBR in two steps (qr.cu): the prepare step (pool 0 of h, every block's Y,
// batched op(T)) reads only the packed reflectors; apply runs the block loop.
struct OrmbrPlan {
  bool isq = true, trans = false, pre = false;
  int nb = 0;
  const double* A = nullptr;
  long long lda = 0;
  const double* tau = nullptr;
  long long c_rows = 0, c_cols = 0, count = 0, rows0 = 0, nblk = 0, nfull = 0;
  std::vector<long long> yoff;
  double *Yall = nullptr, *scr = nullptr, *Top = nullptr;
};
int ormbr_prepare(dcsvd_ctx* h, cudaStream_t st, char vect, bool trans, long long m, long long n, const double* A,
                  long long lda, const double* tau, long long c_rows, long long c_cols, int nb, OrmbrPlan& P);
void ormbr_build_y(cudaStream_t st, const OrmbrPlan& P, long long bi);
int ormbr_apply(dcsvd_ctx* h, cudaStream_t st, const OrmbrPlan& P, double* C, long long ldc);
int ormbr_run(dcsvd_ctx* h, cudaStream_t st, char vect, bool trans, long long m, long long n,
              const double* A, long long lda, const double* tau, double* C, long long c_rows,
              long long c_cols, long long ldc, int nb);
// Bidiagonal D&C.  Outputs (all optional except dvals): edge_out (2 x ncols),
// Wout = [W_desc; 0] with wrows >= n rows, Qout (ncols x ncols), VT = Q_desc^T
// (n x n, square problems).
int bdsdc_run(dcsvd_ctx* h, cudaStream_t st, long long n, const double* d, const double* e, bool bordered,
              bool vectors, int leaf, double tol_mult, double* dvals, double* edge_out, double* Wout,
              long long ldwo, long long wrows, double* Qout, long long ldqo, double* VT, long long ldvt);
// standalone pieces (reference API rows)
int build_tinv_run(dcsvd_ctx* h, cudaStream_t st, long long rows, int w, const double* Y, long long ldy,
                   const double* tau, double* Tinv, long long ldt);
int block_reflector_run(dcsvd_ctx* h, cudaStream_t st, char side, bool trans, long long rows_y, int w, const double* Y,
                        long long ldy, const double* Tinv, long long ldt, double* C, long long ldc, long long c_other);
int geqr2_run(dcsvd_ctx* h, cudaStream_t st, long long m, int w, double* A, long long lda, double* tau);
int larfg_run(dcsvd_ctx* h, cudaStream_t st, long long n, const double* alpha, const double* x, long long incx,
              double* out, double* ess);
int lartg_run(dcsvd_ctx* h, cudaStream_t st, long long cnt, const double* a, const double* b, double* out);
int trsm_run(dcsvd_ctx* h, cudaStream_t st, int n, const double* T, long long ldt, double* B, long long ldb,
             long long other, bool right, bool trans);
int build_z_run(dcsvd_ctx* h, cudaStream_t st, int nl, int nr, int bordered, double alpha, double beta,
                const double* ldv, const double* ledge, long long lde_l, const double* rdv, const double* redge,
                long long lde_r, double* d, double* z, double* coupling);
int deflate_run(dcsvd_ctx* h, cudaStream_t st, int n, const double* d_in, const double* z_in, double tol_multiple,
                double* left, long long rows_l, long long ldl, double* right, long long rows_r, long long ldr,
                double* edge, long long lde, int* lcls, int* rcls, long long* perm, double* d, double* z,
                long long* kept, long long* deflated, double* dvals, long long* rot_pq, double* rot_cs,
                long long* counts);
int gather2d_run(dcsvd_ctx* h, cudaStream_t st, long long rows, long long cnt, const double* src, long long lds,
                 const long long* ridx, const long long* cidx, double* dst, long long ldd);
int philox_run(dcsvd_ctx* h, cudaStream_t st, unsigned long long k0, unsigned long long k1, unsigned long long off,
               long long count, int normal, double* out, long long rows, long long ld);
int prescribed_sigma_run(dcsvd_ctx* h, cudaStream_t st, int kind, int n, double cond, unsigned long long k0,
                         unsigned long long k1, double* sigma);
int generate_run(dcsvd_ctx* h, cudaStream_t st, int kind, long long m, long long n, double cond, unsigned long long k0,
                 unsigned long long k1, double* A, long long lda);
int accuracy_run(dcsvd_ctx* h, cudaStream_t st, long long m, long long n, const double* A, long long lda,
                 const double* S, const double* U, long long ldu, const double* VT, long long ldvt,
                 const double* ref, double* out_host);
int secular_run(dcsvd_ctx* h, cudaStream_t st, int K, const double* d, const double* z, double* omega, int* anc,
                double* mu, int max_iter);
int loewner_run(dcsvd_ctx* h, cudaStream_t st, int K, const double* d, const double* z, const int* anc, const double* mu,
                double* zt);
int secvec_run(dcsvd_ctx* h, cudaStream_t st, int K, const double* d, const int* anc, const double* mu, const double* zt,
               double* U, long long ldu, double* V, long long ldv);
}  // namespace dc
