// Dependent-chain latency (cycles) of FP64 scalar ops, shuffles, shared
// loads and __syncthreads on one SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sh[256];
  sh[threadIdx.x] = x0 + threadIdx.x;
  __syncthreads();
  double x = x0;
  long long t0, t1;
#define BENCH(slot, body)                 \
  t0 = clock64();                         \
  for (int i = 0; i < n; ++i) { body; }   \
  t1 = clock64();                         \
  if (threadIdx.x == 0) cyc[slot] = (t1 - t0) / n;
  BENCH(0, x = fma(x, 1.0000001, 1e-9))
  BENCH(1, x = 1.0 / (x + 1.0))
  BENCH(2, x = sqrt(x + 2.0))
  BENCH(3, x = hypot(x, 0.5))
  BENCH(4, x = __shfl_xor_sync(~0u, x, 1) + 1e-9)
  BENCH(5, x = sh[(int)x & 7] * 0.5 + x)
  BENCH(6, __syncthreads(); x += 1e-9)
  BENCH(7, x = x * 1.0000001)
  BENCH(8, x = (x > 1.5 ? x : x + 1e-9) * 0.999)
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64 * 8);
  const char* nm[] = {"DFMA", "DDIV (1/x)", "DSQRT", "hypot", "SHFL f64 + DADD", "LDS f64 dep + DFMA", "__syncthreads (256 thr)", "DMUL", "DSETP+SEL+DMUL"};
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(o, c, 1.25, 1000); cudaDeviceSynchronize();
    lat<<<1, threads>>>(o, c, 1.25, 1000); cudaDeviceSynchronize();
    printf("block %d threads:\n", threads);
    for (int i = 0; i < 9; ++i) printf("  %-26s %lld cyc\n", nm[i], c[i]);
  }
  return 0;
}
