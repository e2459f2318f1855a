/* libdcsvd_b200 — B200-native (sm_100a) fp64 divide-and-conquer SVD.
 *
 * C ABI.  Every matrix is float64 column-major with an explicit leading
 * dimension; every pointer is a DEVICE pointer (e.g. torch `data_ptr()`),
 * except the option/profile structs which live on the host.  Calls enqueue on
 * the caller's stream; the handle owns scratch workspace and a device status
 * word, so use one handle per stream/thread.  Return codes:
 *   0 ok, 1 invalid argument (ValueError), 2 no convergence
 *   (ConvergenceError), 3 interlacing violated (ArithmeticError), 4 singular
 *   triangular factor (LinAlgError), 5 CUDA error (RuntimeError);
 * dcsvd_last_error() gives the message.
 *
 * The reference exposes no FFI: its boundary is the Python module API of the
 * `dcsvd` package (/root/reference/pkg/src/dcsvd/__init__.py:18-129).  Each
 * entry point below cites the reference function it replaces; the Python
 * package paper_2508_11467_b200 keeps those names/signatures and calls these
 * through ctypes.
 */
#ifndef DCSVD_B200_H
#define DCSVD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dcsvd_ctx* dcsvd_handle;

/* status codes */
#define DCSVD_OK 0
#define DCSVD_EINVAL 1
#define DCSVD_ENOCONV 2
#define DCSVD_EARITH 3
#define DCSVD_ESINGULAR 4
#define DCSVD_ECUDA 5

/* SVDOptions (pkg/src/dcsvd/driver.py:34-63). */
typedef struct dcsvd_opts {
  int want_vectors;        /* 1 = U and Vt, 0 = values only              */
  int bidiag_block;        /* GEBRD panel width (default 32)             */
  int qr_block;            /* GEQRF panel width (default 32)             */
  int orgqr_block;         /* ORGQR block width (default 64)             */
  int apply_block;         /* ORMBR block width (default 64)             */
  int leaf_size;           /* BDC leaf bound, 1..32 (default 32)         */
  double ts_crossover;     /* QR-first when m >= ts_crossover*n (5/3)    */
  double deflation_multiple; /* deflation tolerance multiple (8)         */
} dcsvd_opts;

/* PhaseProfile (driver.py:76-82): seconds per PHASE_NAMES entry (driver.py:31),
 * measured with CUDA events on the call's stream. */
typedef struct dcsvd_phase_times {
  double geqrf, orgqr, gebrd, bdcdc, ormbr, gemm, total;
} dcsvd_phase_times;

/* lifecycle ---------------------------------------------------------------- */
int dcsvd_create(dcsvd_handle* h, int device);
int dcsvd_destroy(dcsvd_handle h);
const char* dcsvd_last_error(dcsvd_handle h);
int dcsvd_version(void);
/* Number of this library's kernels launched through `h` since creation. */
long long dcsvd_launch_count(dcsvd_handle h);

/* Kernel-family timing for roofline reporting.  When enabled, CUDA events
 * bracket every launch of a family on its stream.  kind 0 = LABRD panel kernel
 * (work = algorithmic GEMV bytes), kind 1 = DMMA GEMM (work = flops).
 * dcsvd_set_stats also clears previous records; dcsvd_get_stats synchronizes. */
int dcsvd_set_stats(dcsvd_handle h, int enable);
int dcsvd_get_stats(dcsvd_handle h, int kind, double* ms, double* work, long long* launches);

/* GEMM: C <- alpha*op(A)*op(B) + beta*C (beta == 0 does not read C).
 * Replaces densecore.matmul_accumulate (pkg/src/dcsvd/densecore.py:73-93).
 * Hand-written DMMA (mma.sync m8n8k4 f64) kernel. */
int dcsvd_dgemm(dcsvd_handle h, int transa, int transb, int64_t m, int64_t n, int64_t k,
                double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                double beta, double* C, int64_t ldc, void* stream);

/* GEMV: y <- alpha*op(A)*x + beta*y (densecore.py:96-111). */
int dcsvd_dgemv(dcsvd_handle h, int transa, int64_t m, int64_t n, double alpha, const double* A,
                int64_t lda, const double* x, double beta, double* y, void* stream);

/* Blocked bidiagonalization in place, m >= n (bidiag.py:168-204, merged
 * rank-2b LABRD panel bidiag.py:113-165 + single trailing GEMM).
 * d[n], e[n-1], tauq[n], taup[n] (taup[n-1] = 0). */
int dcsvd_gebrd(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* d, double* e,
                double* tauq, double* taup, int nb, void* stream);

/* One merged rank-2b LABRD panel on the m x n view A (bidiag.py:113-165):
 * factors the leading nb rows/columns, writes d/e/tauq/taup[0..nb) and the
 * panel matrices P (m x 2nb, ldp) and Q (n x 2nb, ldq); requires
 * 1 <= nb < n <= m, nb <= 32.  The trailing update is left to the caller. */
int dcsvd_labrd(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* d, double* e,
                double* tauq, double* taup, int nb, double* P, int64_t ldp, double* Q, int64_t ldq,
                void* stream);

/* Bidiagonal divide and conquer (bdc.py:861-880).  d[n], e[n] (e[n-1] used
 * only when bordered).  Outputs: dvals[n] descending; edge[2 x ncols]
 * (ld 2, column-major, i.e. edge[2*j + r]); when want_vectors: W[n x n]
 * (ldw), Q[ncols x ncols] (ldq), ncols = n + bordered.  W/Q may be NULL when
 * want_vectors == 0. */
int dcsvd_bdsdc(dcsvd_handle h, int64_t n, const double* d, const double* e, int bordered,
                int want_vectors, int leaf, double tol_multiple, double* dvals, double* W,
                int64_t ldw, double* Q, int64_t ldq, double* edge, void* stream);

/* Blocked Householder QR in place, m >= n (qrblock.py:122-144). */
int dcsvd_geqrf(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* tau, int nb,
                void* stream);

/* First k columns of Q from a packed QR of an m x nrefl matrix
 * (qrblock.py:147-164).  Q is m x k (ldq), overwritten. */
int dcsvd_orgqr(dcsvd_handle h, int64_t m, int64_t nrefl, int64_t k, const double* A, int64_t lda,
                const double* tau, double* Q, int64_t ldq, int nb, void* stream);

/* Back-transformation with the bidiagonalization reflectors of the m x n
 * packed matrix A (backtransform.py:90-131).
 *   vect = 'Q': C (m x ncols) <- U1 C   (trans = 0)  or U1^T C (trans = 1)
 *   vect = 'P': C (nrows x n) <- C V1   (trans = 0)  or C V1^T (trans = 1)
 * tau = tauq (for 'Q') or taup (for 'P'). */
int dcsvd_ormbr(dcsvd_handle h, char vect, int trans, int64_t m, int64_t n, const double* A,
                int64_t lda, const double* tau, double* C, int64_t c_rows, int64_t c_cols,
                int64_t ldc, int nb, void* stream);

/* Economy SVD A = U diag(S) VT of an m x n matrix (driver.py:121-157).
 * A is consumed as workspace (the Python layer copies first, like the
 * reference, driver.py:154).  S[min(m,n)] descending; U m x k (ldu), VT k x n
 * (ldvt) with k = min(m, n); U/VT ignored when opts->want_vectors == 0.
 * `prof` (optional, host) receives per-phase device seconds. */
int dcsvd_gesdd(dcsvd_handle h, int64_t m, int64_t n, double* A, int64_t lda, double* S, double* U,
                int64_t ldu, double* VT, int64_t ldvt, const dcsvd_opts* opts,
                dcsvd_phase_times* prof, void* stream);

/* Batched independent SVDs of equally sized m x n matrices (BASELINE config
 * 5).  Arrays of `batch` device pointers (host arrays of device pointers);
 * leading dimensions shared.  Executes in waves of up to `concurrency`
 * matrices (0 = automatic). */
int dcsvd_gesdd_batched(dcsvd_handle h, int batch, int64_t m, int64_t n, double* const* A,
                        int64_t lda, double* const* S, double* const* U, int64_t ldu,
                        double* const* VT, int64_t ldvt, const dcsvd_opts* opts, int concurrency,
                        void* stream);

/* ---- stage pieces of the reference API (single calls, device pointers) ---- */

/* householder_generate (densecore.py:114-128): x[n] (stride incx), *alpha ->
 * tau_beta[0] = tau, tau_beta[1] = beta, essential[n] = x/(alpha-beta). */
int dcsvd_larfg(dcsvd_handle h, int64_t n, const double* alpha, const double* x, int64_t incx,
                double* tau_beta, double* essential, void* stream);
/* givens_generate (densecore.py:131-140) for `count` pairs: csr[3i..3i+2] = c, s, r. */
int dcsvd_lartg(dcsvd_handle h, int64_t count, const double* a, const double* b, double* csr, void* stream);
/* triangular_solve (densecore.py:143-171), T upper n x n: side 'L': B (n x other)
 * <- T^-1 B (T^-T B when trans); side 'R': B (other x n) <- B T^-1 (B T^-T). */
int dcsvd_trsm(dcsvd_handle h, char side, int trans, int64_t n, const double* T, int64_t ldt, double* B,
               int64_t ldb, int64_t other, void* stream);
/* build_tinv (qrblock.py:90-100): Tinv (w x w) = triu(Y^T Y, 1) + diag(1/tau), w <= 128. */
int dcsvd_build_tinv(dcsvd_handle h, int64_t rows, int w, const double* Y, int64_t ldy, const double* tau,
                     double* Tinv, int64_t ldt, void* stream);
/* apply_block_reflector_left/right (qrblock.py:103-119) with a given (Y, Tinv):
 * side 'L': C (rows_y x c_other) <- (I - Y T Y^T) C (T^T when trans);
 * side 'R': C (c_other x rows_y) <- C (I - Y T Y^T) (T^T when trans). */
int dcsvd_block_reflector(dcsvd_handle h, char side, int trans, int64_t rows_y, int w, const double* Y,
                          int64_t ldy, const double* Tinv, int64_t ldt, double* C, int64_t ldc,
                          int64_t c_other, void* stream);
/* geqrf_panel (qrblock.py:51-71): unblocked QR of an m x w panel in place, w <= 64. */
int dcsvd_geqrf_panel(dcsvd_handle h, int64_t m, int w, double* A, int64_t lda, double* tau, void* stream);
/* solve_all_roots (bdc.py:515-641) of one secular system (d ascending, d[0] = 0):
 * omega[K], anchor[K] (int32), mu[K]; max_iterations = the reference's budget
 * (100 in bdsdc); a root not converged within it -> DCSVD_ENOCONV
 * (ConvergenceError, bdc.py:636-639). */
int dcsvd_secular_roots(dcsvd_handle h, int K, const double* d, const double* z, double* omega,
                        int* anchor, double* mu, int max_iterations, void* stream);
/* recompute_z (bdc.py:644-673): Loewner update vector ztilde[K]. */
int dcsvd_recompute_z(dcsvd_handle h, int K, const double* d, const double* z, const int* anchor,
                      const double* mu, double* ztilde, void* stream);
/* secular_vectors (bdc.py:676-694): U, V (K x K) column-normalised. */
int dcsvd_secular_vectors(dcsvd_handle h, int K, const double* d, const int* anchor, const double* mu,
                          const double* ztilde, double* U, int64_t ldu, double* V, int64_t ldv,
                          void* stream);

/* ---- standalone merge stages of the divide and conquer (bdc.py:382-747) ---- */

/* build_z (bdc.py:382-412): middle-row data of a merge in pre-sort order.
 * left/right child values (nl / nr entries) and edge rows (2 x (n_child+1),
 * leading dimension lde_*).  Outputs d[n], z[n] with n = nl + nr + 1 and
 * coupling[2] = (c, s) of the bordered null-direction rotation ((1, 0) when
 * square). */
int dcsvd_build_z(dcsvd_handle h, int nl, int nr, int bordered, double alpha, double beta,
                  const double* left_dvals, const double* left_edge, int64_t lde_l,
                  const double* right_dvals, const double* right_edge, int64_t lde_r, double* d,
                  double* z, double* coupling, void* stream);

/* deflate (bdc.py:423-508): stable ascending sort of (d, z) (d[0] must be the
 * zero border entry after sorting), tolerance tol_multiple * eps * max(|d|,|z|),
 * z0 clamp, tiny-z and close-pair (Givens) deflation against the last kept
 * entry.  The optional column matrices left (rows_l x n), right (rows_r x n),
 * edge (2 x n) and int32 class arrays are permuted and rotated IN PLACE
 * (pairs with entry 0 rotate only right/edge).  Outputs: perm[n], d_out[n],
 * z_out[n] (sorted working copies after the rotations), kept[n], deflated[n],
 * deflated_values[n], rot_pq[2n] (p, j pairs), rot_cs[2n] (c, s pairs) and
 * counts[3] = {#kept, #deflated, #rotations}.  Synchronizes the stream. */
int dcsvd_deflate(dcsvd_handle h, int n, const double* d, const double* z, double tol_multiple,
                  double* left, int64_t rows_l, int64_t ldl, double* right, int64_t rows_r, int64_t ldr,
                  double* edge, int64_t lde, int* left_classes, int* right_classes, int64_t* perm,
                  double* d_out, double* z_out, int64_t* kept, int64_t* deflated,
                  double* deflated_values, int64_t* rot_pq, double* rot_cs, int64_t* counts,
                  void* stream);

/* Gather dst[r, c] = src[row_idx ? row_idx[r] : r, col_idx ? col_idx[c] : c]
 * (rows x cols), used by merge_vectors (bdc.py:701-747) to assemble the class
 * blocks of its structured DMMA products (dcsvd_dgemm). */
int dcsvd_gather(dcsvd_handle h, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 const int64_t* row_idx, const int64_t* col_idx, double* dst, int64_t ldd, void* stream);

/* ---- harness pieces on the GPU (harness.py:69-187) ---- */

/* Philox-4x64-10 word stream of numpy's Philox(key=seed) (key = 128-bit seed
 * as key_lo, key_hi): `count` outputs starting at stream word `word_offset`,
 * written column-major into a rows x * matrix (ld).  normal = 0: uniforms
 * ((w >> 11) + 0.5) 2^-53, bit-identical to harness._Stream.uniforms;
 * normal = 1: Box-Muller pairs as harness._Stream.normals (consumes
 * 2 ceil(count/2) words). */
int dcsvd_philox(dcsvd_handle h, uint64_t key_lo, uint64_t key_hi, uint64_t word_offset, int64_t count,
                 int normal, double* out, int64_t rows, int64_t ld, void* stream);

/* prescribed_singular_values (harness.py:108-114); kind 1 logrand, 2 arith, 3 geo. */
int dcsvd_prescribed_singular_values(dcsvd_handle h, int kind, int64_t n, double cond, uint64_t key_lo,
                                     uint64_t key_hi, double* sigma, void* stream);

/* generate_matrix (harness.py:131-146): kind 0 random (uniforms column-major),
 * 1 logrand / 2 arith / 3 geo = U diag(sigma) V^T with Haar factors from the
 * GPU blocked QR of Philox normals (harness.py:117-128). */
int dcsvd_generate_matrix(dcsvd_handle h, int kind, int64_t m, int64_t n, double cond, uint64_t key_lo,
                          uint64_t key_hi, double* A, int64_t lda, void* stream);

/* accuracy (harness.py:149-187): report[4] (HOST) = {e_sigma, e_svd, orth_u,
 * orth_v}; NaN where the reference leaves None (no ref_sigma / no U,VT). */
int dcsvd_accuracy(dcsvd_handle h, int64_t m, int64_t n, const double* A, int64_t lda, const double* S,
                   const double* U, int64_t ldu, const double* VT, int64_t ldvt, const double* ref_sigma,
                   double* report, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DCSVD_B200_H */
