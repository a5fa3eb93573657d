// VIADD (ALU) vs IMAD (FMA pipe) throughput for the int->fp32 magic add.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
template <int OP>
__global__ void k(int* out, int x, int one) {
  int a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 8 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(x));
      if (OP == 1) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(one), "r"(x));
      if (OP == 2) { asm volatile("add.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(x)); asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[(i + 4) & 7]) : "r"(one), "r"(x)); }
    }
  }
  int s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345) out[0] = s;
}
template <int OP> void run(const char* name, int ops) {
  int* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 grid(sms * 4), blk(256);
  k<OP><<<grid, blk>>>(out, 3, 1); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<OP><<<grid, blk>>>(out, 3, 1); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double n = double(grid.x) * blk.x * ITERS * ops;
  printf("%-34s %8.3f ms  %7.1f thread-ops/clk/SM\n", name, ms, n / (ms * 1e-3) / sms / 1965e6);
}
int main() { run<0>("add.s32 (VIADD/IADD3)", 8); run<1>("mad.lo.s32 x*1+c (IMAD)", 8); run<2>("mixed add + mad", 16); }
