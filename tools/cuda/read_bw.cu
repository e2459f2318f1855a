// Read-only HBM bandwidth (the GEMV roofline): each CTA streams a contiguous
// chunk with 16-byte loads and reduces it.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (; i < n2; i += stride) { double2 v = __ldcs(p + i); s += v.x + v.y; }
  if (s == 1234.5) out[0] = s;
}
__global__ void rd_chunk(const double2* __restrict__ p, size_t n2, double* out) {
  // contiguous chunk per CTA (like a row-block GEMV)
  const size_t per = (n2 + gridDim.x - 1) / gridDim.x;
  const size_t b = per * blockIdx.x, e = min(n2, b + per);
  double s = 0.0;
#pragma unroll 8
  for (size_t i = b + threadIdx.x; i < e; i += blockDim.x) { double2 v = __ldcs(p + i); s += v.x + v.y; }
  if (s == 1234.5) out[0] = s;
}
int main() {
  const size_t bytes = (size_t)1 << 30;
  double2* p; double* o;
  cudaMalloc(&p, bytes); cudaMalloc(&o, 8);
  cudaMemset(p, 0, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int k : {1, 2, 4, 8}) for (int thr : {256, 512, 1024}) {
    for (int variant = 0; variant < 2; ++variant) {
      for (int w = 0; w < 2; ++w) variant ? rd_chunk<<<sms * k, thr>>>(p, bytes / 16, o) : rd<<<sms * k, thr>>>(p, bytes / 16, o);
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r) variant ? rd_chunk<<<sms * k, thr>>>(p, bytes / 16, o) : rd<<<sms * k, thr>>>(p, bytes / 16, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%s grid %4d x %4d: %.0f GB/s\n", variant ? "chunked " : "strided ", sms * k, thr, bytes * 10.0 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
