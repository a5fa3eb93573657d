// Per-warp MUFU.EX2 issue rate: one warp per SMSP (4 warps/SM), NIND
// independent ex2 chains per thread, no other work.
#include <cstdio>
#include <cuda_runtime.h>
template <int NIND>
__global__ void k(float* out, float s) {
  float f[NIND];
  for (int i = 0; i < NIND; ++i) f[i] = s * (threadIdx.x + i) * 1e-6f;
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < NIND; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
  }
  float acc = 0; for (int i = 0; i < NIND; ++i) acc += f[i];
  if (acc == 1.2345f) out[0] = acc;
}
template <int NIND> void run(int warps) {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k<NIND><<<sms, warps * 32>>>(out, 1.f); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<NIND><<<sms, warps * 32>>>(out, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ex = double(sms) * warps * 32 * 2048 * NIND;
  printf("warps/SM %2d  independent chains %2d: ex2 %5.2f /clk/SM (%3.0f%% of 16)\n", warps, NIND,
         ex / (ms * 1e-3) / sms / 1965e6, 100 * ex / (ms * 1e-3) / sms / 1965e6 / 16);
}
int main() {
  run<4>(4); run<8>(4); run<16>(4); run<32>(4); run<64>(4);
  run<8>(8); run<32>(8); run<32>(12);
}
