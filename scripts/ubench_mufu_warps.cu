// MUFU.EX2 throughput vs resident warps per SM, with an exp-loop-like body:
// per element IADD(magic) + FFMA + EX2 + FADD(sum) + F2FP-pack every 2.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 256
__global__ void k(float* out, float c, float b) {
  int a[64];
  for (int i = 0; i < 64; ++i) a[i] = (threadIdx.x * 131 + i * 7919) & 0xffff;
  float s0 = 0, s1 = 0; uint32_t pk = 0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      float x0 = fmaf(__int_as_float(a[i] + 0x4B400000), c, b);
      float x1 = fmaf(__int_as_float(a[i + 1] + 0x4B400000), c, b);
      float e0, e1;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(x0));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(x1));
      s0 += e0; s1 += e1;
      uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(e1), "f"(e0)); pk ^= r;
    }
#pragma unroll
    for (int i = 0; i < 64; ++i) a[i] ^= it;
  }
  if (s0 + s1 == 1.234f || pk == 77) out[0] = s0;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 12, 16, 32}) {
    k<<<sms, warps * 32>>>(out, 1e-9f, -12582912e-9f); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<<<sms, warps * 32>>>(out, 1e-9f, -12582912e-9f); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ex = double(sms) * warps * 32 * ITERS * 64;
    printf("warps/SM %2d: %6.3f ms  ex2 %5.2f /clk/SM (at 1965 MHz)  = %3.0f%% of 16\n", warps, ms,
           ex / (ms * 1e-3) / sms / 1965e6, 100 * ex / (ms * 1e-3) / sms / 1965e6 / 16);
  }
}
