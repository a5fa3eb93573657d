// Packed-half MUFU.EX2 throughput: elements/clk/SM for ex2.approx.ftz.f32,
// ex2.approx.f16x2 and ex2.approx.ftz.bf16x2 (each packed op = 2 elements).
// Also F2FP.F16 packs and HADD2 as companions of a half-precision exp path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE, int NIND>
__global__ void k(float* out, float s) {
  uint32_t f[NIND];
  for (int i = 0; i < NIND; ++i) {
    float x = -s * (threadIdx.x + i) * 1e-3f;
    f[i] = __float_as_uint(x);
    if (MODE != 0) asm("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(f[i]) : "f"(x));
    if (MODE == 2) asm("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(f[i]) : "f"(x));
  }
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < NIND; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(f[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(f[i]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(f[i]));
      if (MODE == 3) asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(f[i]) : "f"(__uint_as_float(f[i])));
    }
  }
  uint32_t acc = 0; for (int i = 0; i < NIND; ++i) acc ^= f[i];
  if (acc == 12345u) out[0] = acc;
}
template <int MODE, int NIND> void run(int warps, const char* name) {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  k<MODE, NIND><<<sms, warps * 32>>>(out, 1.f); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<MODE, NIND><<<sms, warps * 32>>>(out, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = double(sms) * warps * 32 * 2048 * NIND;
  double per = ops / (ms * 1e-3) / sms / (clk * 1e3);
  printf("%-22s warps/SM %2d chains %2d: %6.2f instr-lanes/clk/SM  (%s %.2f elem/clk/SM)\n", name, warps,
         NIND, per, MODE == 1 || MODE == 2 ? "x2 =" : "=", (MODE == 1 || MODE == 2 ? 2 : 1) * per);
}
int main() {
  run<0, 16>(16, "ex2.f32");
  run<1, 16>(16, "ex2.f16x2");
  run<2, 16>(16, "ex2.bf16x2");
  run<3, 16>(16, "cvt.f16x2.f32");
  run<0, 16>(8, "ex2.f32");
  run<1, 16>(8, "ex2.f16x2");
}
