// Does the bf16x2 pack (F2FP.BF16.F32.PACK_AB) share the XU pipe with
// MUFU.EX2?  Per "pair" of fp32 values: two ex2.approx plus
//   mode 0: nothing else            (MUFU alone)
//   mode 1: cvt.rn.bf16x2.f32       (F2FP: the attention kernel's P~ pack)
//   mode 2: two IADD (+0x8000) and one PRMT (pack by integer ops, round
//           half up -- differs from RNE only on exact ties)
// Reports cycles per pair per SMSP-warp slot (SM clock from the attribute).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE, int NIND>
__global__ void k(uint32_t* out, float s, long long* cyc) {
  const long long c0 = clock64();
  float x[NIND];
  uint32_t acc = 0;
  for (int i = 0; i < NIND; ++i) x[i] = -s * (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < 1024; ++it) {
#pragma unroll
    for (int i = 0; i < NIND; i += 2) {
      float e0, e1;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(x[i]));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(x[i + 1]));
      uint32_t p;
      if (MODE == 1) {
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(e1), "f"(e0));
      } else if (MODE == 2) {
        const uint32_t r0 = __float_as_uint(e0) + 0x8000u, r1 = __float_as_uint(e1) + 0x8000u;
        p = __byte_perm(r0, r1, 0x7632);
      } else {
        p = __float_as_uint(e0) ^ __float_as_uint(e1);
      }
      acc += p;
      x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (p & 1u));   // keep the chain live
    }
  }
  if (acc == 12345u) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = clock64() - c0;
}
template <int MODE, int NIND> void run(int warps) {
  uint32_t* out; cudaMalloc(&out, 4);
  long long* dc; cudaMalloc(&dc, 8);
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  k<MODE, NIND><<<sms, warps * 32>>>(out, 1.f, dc); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<MODE, NIND><<<sms, warps * 32>>>(out, 1.f, dc); cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double pairs_per_smsp = double(warps) / 4 * 1024 * (NIND / 2);   // warp-pairs per SMSP
  long long kc; cudaMemcpy(&kc, dc, 8, cudaMemcpyDeviceToHost);
  const double cyc = double(kc);   // SM clocks of CTA 0 (clock64)
  printf("  (event %.3f ms; attribute clock %d kHz; clock64 %lld -> %.0f MHz)\n", ms, clk, kc, kc / (ms * 1e3));
  printf("mode %d warps/SM %2d: %.2f cycles per warp-pair per SMSP (MUFU-only floor 16)\n", MODE, warps,
         cyc / pairs_per_smsp);
  cudaFree(out);
}
int main() {
  for (int w : {8, 16}) { run<0, 16>(w); run<1, 16>(w); run<2, 16>(w); }
  return 0;
}
