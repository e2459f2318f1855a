// Shared device helpers for libdcsvd_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "dcsvd_b200.h"

#define DC_EPS 2.220446049250313e-16
#define DC_TINY 2.2250738585072014e-308

namespace dc {

// ---------------------------------------------------------------------------
// status words written by kernels (checked once per stage by the host)
enum DevErr : int {
  kDevOk = 0,
  kDevNoConvergeQR = 1,       // leaf QR iteration budget (bdc.py:309-312)
  kDevNoConvergeSecular = 2,  // secular solver 100 iterations (bdc.py:636-639)
  kDevInterlacing = 3,        // non-positive Loewner radicand (bdc.py:669-672)
  kDevSingularT = 4,          // zero diagonal in Tinv (densecore.py:152-153)
  kDevBadDeflate = 5,         // d[0] != 0 after sort (bdc.py:450-451)
};

__device__ __forceinline__ void raise_dev(int* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_prod(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v *= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum with a fixed reduction tree (deterministic).  `sh` needs
// blockDim.x/32 doubles.  Result valid in all threads.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// Plane rotation, reference convention (densecore.py:131-140):
// r = hypot(f, g) >= 0, c = f/r, s = g/r; (0,0) -> identity.
__device__ __forceinline__ void lartg(double f, double g, double& c, double& s, double& r) {
  r = hypot(f, g);
  if (r == 0.0) {
    c = 1.0; s = 0.0;
  } else {
    c = f / r; s = g / r;
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier for cooperative launches: monotone counter, reset by the
// host before each launch.  `epoch` counts barriers passed by this CTA.  One
// release-add per CTA, acquire polling by one thread, then a CTA barrier.
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  epoch += 1;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    const unsigned target = epoch * nblocks;
    while (ld_acquire(ctr) < target) {
    }
  }
  __syncthreads();
}

}  // namespace dc

// host-side helpers -----------------------------------------------------------
#define DC_CUDA_TRY(expr)                                 \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return dc_cuda_fail(_e, #expr); \
  } while (0)

int dc_cuda_fail(cudaError_t e, const char* what);
int dc_fail(int code, const char* fmt, ...);
