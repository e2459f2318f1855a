// Micro-benchmark: grid barrier latency vs CTA count and barrier flavour.
#include <cstdio>
#include <cooperative_groups.h>
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__global__ void flat(unsigned* ctr, int iters) {
  unsigned epoch = 0;
  for (int it = 0; it < iters; ++it) {
    __syncthreads(); epoch++;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      while (ld_acquire(ctr) < epoch * gridDim.x) {}
    }
    __syncthreads();
  }
}
// two-level: groups of 8 CTAs arrive at a group counter; the last of a group
// arrives at the root; everyone polls a generation word written by the last root arriver
__global__ void tree(unsigned* ctr, unsigned* gen, int iters) {
  const int grp = blockIdx.x / 8, ngrp = (gridDim.x + 7) / 8;
  const int gsize = min(8, (int)gridDim.x - grp * 8);
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr + 1 + grp * 32) : "memory");
      if (old % gsize == (unsigned)gsize - 1) {
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
        if (old % ngrp == (unsigned)ngrp - 1) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(it + 1) : "memory");
      }
      while (ld_acquire(gen) < (unsigned)(it + 1)) {}
    }
    __syncthreads();
  }
}
int main() {
  unsigned *ctr, *gen;
  cudaMalloc(&ctr, 4096 * 4); cudaMalloc(&gen, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2000;
  for (int g : {16, 37, 74, 144, 148}) {
    for (int kind = 0; kind < 2; ++kind) {
      cudaMemset(ctr, 0, 4096 * 4); cudaMemset(gen, 0, 4);
      void* args0[] = {&ctr, (void*)&iters};
      void* args1[] = {&ctr, &gen, (void*)&iters};
      cudaEventRecord(a);
      if (kind == 0) cudaLaunchCooperativeKernel((void*)flat, g, 512, args0, 0, 0);
      else cudaLaunchCooperativeKernel((void*)tree, g, 512, args1, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("G=%3d %s barrier: %.3f us\n", g, kind ? "tree" : "flat", ms * 1e3 / iters);
    }
  }
  return 0;
}
