// Micro-benchmark: DMMA.8x8x4 fed from shared memory fragments (FM x FN warp
// tile per k-step of 4), no global memory traffic.
#include <cstdio>
template <int FM, int FN>
__global__ void loop(double* out, int iters) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 1e-6;
  __syncthreads();
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int LD = 68;  // as in the kernels: pitch = 4 mod 16
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int ks = 0; ks < 32; ks += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = sm[(ks + lc) * LD + (warp & 1) * 32 + i * 8 + lr];
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = sm[4096 + (ks + lc) * LD + (warp >> 1) * 8 + j * 8 + lr];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 12345.0) out[0] = s;
}
template <int FM, int FN>
void run(int warps) {
  double* out; cudaMalloc(&out, 8);
  int iters = 2048 / (FM * FN) * 8;
  cudaFuncSetAttribute(loop<FM, FN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  loop<FM, FN><<<148, 32 * warps, 65536>>>(out, iters);
  cudaEventRecord(e0);
  loop<FM, FN><<<148, 32 * warps, 65536>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  double flops = 2.0 * 256 * FM * FN * 8.0 * iters * 148 * warps;
  printf("warps %2d FMxFN %dx%d : %6.2f TF/s %s\n", warps, FM, FN, flops / ms / 1e9, e ? cudaGetErrorString(e) : "");
}
int main() {
  for (int w : {4, 8, 16}) { run<2, 2>(w); run<4, 2>(w); run<4, 4>(w); run<8, 4>(w); run<4, 8>(w); }
  return 0;
}
