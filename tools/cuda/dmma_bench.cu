// Micro-benchmark: DMMA.8x8x4 throughput vs warps per SM and independent
// accumulator chains per warp (no memory traffic).
#include <cstdio>
template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double c[NACC][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
template <int NACC>
void run(int warps_per_sm) {
  double* out;
  cudaMalloc(&out, 8);
  int iters = 4096 / NACC * 16;
  int threads = 32 * warps_per_sm;
  int blocks = 148;
  if (threads > 1024) { blocks = 148 * (threads / 1024); threads = 1024; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_loop<NACC><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e0);
  dmma_loop<NACC><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * (double)NACC * iters * (blocks * threads / 32);
  printf("warps/SM %2d  acc/warp %2d : %6.2f TF/s\n", warps_per_sm, NACC, flops / ms / 1e9);
  cudaFree(out);
}
int main() {
  for (int w : {4, 8, 12, 16, 32}) { run<4>(w); run<8>(w); run<16>(w); run<32>(w); }
  return 0;
}
