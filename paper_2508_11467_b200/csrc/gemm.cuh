// FP64 tensor-core (DMMA) GEMM for sm_100a.
//
// On Blackwell the FP64 tensor path is the warp-level DMMA (tcgen05 has no
// f64 kind): `mma.sync.aligned.m8n8k4.row.col.f64` -> SASS DMMA.8x8x4.
// Operand tiles are staged global->shared by a 3-stage cp.async pipeline
// (8-byte granules, so arbitrary sub-view offsets/leading dimensions work),
// with shared layouts chosen per transpose so the global side is always
// contiguous and the fragment reads are bank-conflict free (pad 4 doubles).
//
// One kernel serves every GEMM-shaped stage of the pipeline:
// the GEBRD trailing update A -= P Q^T, the CWY block-reflector applies of
// ORMBR/GEQRF/ORGQR, the TS recombination U = Q U0, and the BDC merge
// products, which additionally gather A's columns and scatter C's columns
// through index lists and read (m, n, k) from device descriptors.
#pragma once
#include "common.cuh"

namespace dc {

struct GemmDesc {
  int m, n, k;
  const double* A;
  long long lda;
  const int* acol;  // optional gather: op(A) column kk -> physical column (non-transposed A only)
  const double* B;
  long long ldb;
  double* C;
  long long ldc;
  const int* ccol;  // optional scatter: C column j -> physical column
  double alpha, beta;
};

constexpr int kMaxBatchDesc = 32;
struct GemmBatch {
  GemmDesc d[kMaxBatchDesc];
  int count;
  // split-K of every descriptor over blockIdx.z: slice s covers k in
  // [s*kchunk, (s+1)*kchunk) and writes C + s*cslice (partials for a reduce)
  int ksplit = 1;
  int kchunk = 0;
  long long cslice = 0;
};

// Host launchers (stream-ordered).  `ta`/`tb` select op(A)=A^T / op(B)=B^T.
int gemm_launch(cudaStream_t st, bool ta, bool tb, const GemmDesc& d);
int gemm_launch_batch(cudaStream_t st, bool ta, bool tb, const GemmBatch& b);
// Grouped: `ndesc` descriptors in device memory (built by device code); the
// grid covers max_m x max_n tiles per descriptor, extra CTAs exit.
// Same for descriptors whose operands all live in one stack of `nbuf` equally
// shaped ld x ld buffers starting at `base` (TMA GEMM, beta = 0, no transposes);
// returns -1 when not applicable.
int gemm_launch_device_stack(cudaStream_t st, const GemmDesc* ddesc, int ndesc, int max_m, int max_n,
                             const double* base, long long ld, int nbuf);
int gemm_launch_device(cudaStream_t st, bool ta, bool tb, const GemmDesc* ddesc, int ndesc,
                       int max_m, int max_n);

}  // namespace dc
