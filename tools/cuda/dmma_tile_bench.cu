// Micro-benchmark: DMMA.8x8x4 from shared-memory fragments in "tiles" of
// KSTEPS k-steps (accumulators consumed + reset per tile, as in a rank-k
// update), W warps per CTA, one CTA per SM.  Separates the DMMA issue limits
// (FM x FN per warp, warps per SM sub-partition, tile length) from data
// movement.
#include <cstdio>
template <int FM, int FN, int KSTEPS>
__global__ void loop(double* out, int tiles) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  for (int i = threadIdx.x; i < 24576; i += blockDim.x) sm[i] = i * 1e-6;
  __syncthreads();
  const int LD = 132;
  double sink = 0;
  for (int t = 0; t < tiles; ++t) {
    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* as = sm + (t & 1) * 4224;
#pragma unroll 4
    for (int ks = 0; ks < KSTEPS * 4; ks += 4) {
      double af[FM], bf[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) af[i] = as[((ks & 124) + lc) * 36 + (warp & 1) * 16 + i * 8 + lr];
#pragma unroll
      for (int j = 0; j < FN; ++j) bf[j] = sm[8448 + ((warp >> 1) & 1) * 32 * LD + (j * 8 + lr) * LD + (ks & 124) + lc];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) if (acc[i][j][0] == 1.2345e300) sink += acc[i][j][1];
  }
  if (sink == 12345.0) out[0] = sink;
}
template <int FM, int FN, int KSTEPS>
void run(int warps) {
  double* out; cudaMalloc(&out, 8);
  int tiles = 65536 / (FM * FN * KSTEPS);
  cudaFuncSetAttribute(loop<FM, FN, KSTEPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 24576 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  loop<FM, FN, KSTEPS><<<148, 32 * warps, 24576 * 8>>>(out, tiles);
  cudaEventRecord(e0);
  loop<FM, FN, KSTEPS><<<148, 32 * warps, 24576 * 8>>>(out, tiles);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  double flops = 2.0 * 256 * FM * FN * KSTEPS * (double)tiles * 148 * warps;
  printf("warps %2d FMxFN %dx%d ksteps %3d : %6.2f TF/s %s\n", warps, FM, FN, KSTEPS, flops / ms / 1e9, e ? cudaGetErrorString(e) : "");
}
int main() {
  for (int w : {4, 8, 12, 16}) {
    run<2, 4, 32>(w); run<2, 4, 16>(w); run<4, 4, 16>(w); run<4, 4, 32>(w); run<2, 4, 256>(w); run<4, 2, 32>(w);
  }
  return 0;
}
