// Throughput microbenchmark of the softmax building blocks on sm_100a.
// Each thread runs 8 independent chains; 4 CTAs x 256 threads per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
template <int OP>
__global__ void k(float* out, int seed) {
  float f[8]; int a[8]; uint64_t p[4];
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 8 + i; f[i] = a[i] * 1e-7f; }
  for (int i = 0; i < 4; ++i) p[i] = (uint64_t(__float_as_uint(f[2*i+1])) << 32) | __float_as_uint(f[2*i]);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { float r; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(r) : "r"(a[i])); a[i] ^= __float_as_int(r); }
      if (OP == 1) { a[i] = a[i] + 0x4B400000; }
      if (OP == 2) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[i])); f[i] = r; }
      if (OP == 3 && i < 4) { uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(p[i]), "l"(p[(i+1)&3]), "l"(p[i])); p[i] = r; }
      if (OP == 4) { f[i] = fmaf(f[i], 1.0001f, 0.5f); }
      if (OP == 5 && i < 4) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[2*i]), "f"(f[2*i+1])); f[2*i] = __uint_as_float(r); }
      if (OP == 6) { asm volatile("max.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i+1)&7])); }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += f[i] + a[i]; for (int i = 0; i < 4; ++i) s += __uint_as_float(uint32_t(p[i]));
  if (s == 123.f) out[0] = s;
}
template <int OP> void run(const char* name, int ops_per_iter) {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  dim3 grid(sms * 4), blk(256);
  k<OP><<<grid, blk>>>(out, 1); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<OP><<<grid, blk>>>(out, 1); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = double(grid.x) * blk.x * ITERS * ops_per_iter;
  double per_clk_sm = ops / (ms * 1e-3) / sms / (1965e6);
  printf("%-28s %8.3f ms  %7.1f thread-ops/clk/SM (at 1965 MHz)\n", name, ms, per_clk_sm);
}
int main() {
  run<0>("cvt.rn.f32.s32 (I2FP)", 8);
  run<1>("iadd (magic)", 8);
  run<2>("ex2.approx (MUFU)", 8);
  run<3>("fma.rn.f32x2 (FFMA2) [x2]", 8);
  run<4>("fma.rn.f32 (FFMA)", 8);
  run<5>("cvt.rn.bf16x2.f32 (F2FP)", 4);
  run<6>("max.s32", 8);
  return 0;
}
