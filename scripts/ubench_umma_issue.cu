// Issue-rate microbenchmark of tcgen05.mma on sm_100a: back-to-back MMAs
// with loop-invariant descriptors (the compiler keeps them in uniform
// registers) vs descriptors that change every iteration.  1 CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_18137_b200/csrc/sm100.cuh"
using namespace sparge;
#define ITERS 4000
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// whole-warp (converged) issue: one elected lane executes the MMA inside the asm
__device__ __forceinline__ void mma_i8_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\t"
               "elect.sync _|e, 0xffffffff;\n\t"
               "setp.ne.and.b32 p, %4, 0, e;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_f16_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\t"
               "elect.sync _|e, 0xffffffff;\n\t"
               "setp.ne.and.b32 p, %4, 0, e;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// four kind::i8 MMAs in ONE asm statement (descriptor steps of 2 = 32 B)
__device__ __forceinline__ void mma_i8_x4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
               "setp.ne.b32 p, 1, 0;\n\t"
               "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
               "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, p;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %3, p;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
template <int MODE>
__global__ void __launch_bounds__(128) k(unsigned long long* out, int salt) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 65536 + 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(bars, 1); mbar_init(bars + 1, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = *slot;
  if (MODE >= 8 && MODE < 12 && warp == 1) {
    // converged warp, elect.sync inside the asm
    const uint64_t dQ = umma_desc_kmajor(smem_u32(sm), 128);
    const uint64_t dK = umma_desc_kmajor(smem_u32(sm + 16384), 128);
    const uint64_t dV = umma_desc_kmajor(smem_u32(sm + 32768), 128);
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
      if (MODE == 8) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8_elect(tm, dQ + 2 * kk, dK + 2 * kk, idesc_i8(128, 64), 1u);
      } else if (MODE == 9) {
        mma_i8_elect(tm, dQ, dK, idesc_i8(128, 16), 1u);
      } else if (MODE == 10) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_f16_ts_elect(tm + 128, tm + 8 * kk, dV + 2 * kk, idesc_bf16(128, 128), 1u);
      } else if (MODE == 11) {
        const uint64_t dKv = umma_desc_kmajor(smem_u32(sm + 16384 + (it & 3) * 8192), 128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8_elect(tm + (it & 1) * 64, dQ + 2 * kk, dKv + 2 * kk, idesc_i8(128, 64), 1u);
      }
    }
    if (lane == 0) { tc_commit(bars); mbar_wait(bars, 0); }
    __syncwarp();
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  } else if ((MODE < 8 || MODE >= 12) && warp == 1 && lane == 0) {
    const uint64_t dQ = umma_desc_kmajor(smem_u32(sm), 128);
    const uint64_t dK = umma_desc_kmajor(smem_u32(sm + 16384), 128);
    const uint64_t dV = umma_desc_kmajor(smem_u32(sm + 32768), 128);
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
      if (MODE == 0) {   // 4 x i8 N64, invariant descriptors
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8(tm, dQ + 2 * kk, dK + 2 * kk, idesc_i8(128, 64), 1u);
      } else if (MODE == 1) {   // 4 x i8 N64, K descriptor varies with it (ring of 4 slots)
        const uint64_t dKv = umma_desc_kmajor(smem_u32(sm + 16384 + (it & 3) * 8192), 128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8(tm, dQ + 2 * kk, dKv + 2 * kk, idesc_i8(128, 64), 1u);
      } else if (MODE == 2) {   // 1 x i8 N64 invariant
        mma_i8(tm, dQ, dK, idesc_i8(128, 64), 1u);
      } else if (MODE == 3) {   // 4 x PV TS N128 invariant
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_f16_ts(tm + 128, tm + 8 * kk, dV + 2 * kk, idesc_bf16(128, 128), 1u);
      } else if (MODE == 4) {   // 4 x i8 N128 invariant
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8(tm, dQ + 2 * kk, dK + 2 * kk, idesc_i8(128, 128), 1u);
      } else if (MODE == 5) {   // 1 x i8 N16 invariant
        mma_i8(tm, dQ, dK, idesc_i8(128, 16), 1u);
      } else if (MODE == 6) {   // 4 x i8 N64 + commit per iteration
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8(tm, dQ + 2 * kk, dK + 2 * kk, idesc_i8(128, 64), 1u);
        tc_commit(bars);
      } else if (MODE == 12) {   // 4 x i8 M64 N8 K32 (tiny: issue-bound)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_i8(tm, dQ + 2 * kk, dK + 2 * kk, idesc_i8(64, 8), 1u);
      } else if (MODE == 14) {   // 4 x i8 M64 N8 in one asm statement
        mma_i8_x4(tm, dQ, dK, idesc_i8(64, 8));
      } else if (MODE == 15) {   // 4 x i8 N64 in one asm statement
        mma_i8_x4(tm, dQ, dK, idesc_i8(128, 64));
      } else if (MODE == 13) {   // 4 x commits
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tc_commit(bars + 1);
      } else if (MODE == 7) {   // 1 x i8 N64, destination varies (2 buffers)
        mma_i8(tm + (it & 1) * 64, dQ, dK, idesc_i8(128, 64), 1u);
      }
    }
    tc_commit(bars);
    mbar_wait(bars, MODE == 6 ? (ITERS & 1) : 0);
    long long t1 = clock64();
    out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { __syncwarp(); tc_fence_after(); tmem_dealloc<512>(tm); }
}
template <int MODE> void run(const char* name, double mmas_per_iter) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 65536 + 2048;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* out; cudaMalloc(&out, sizeof(unsigned long long) * sms);
  k<MODE><<<sms, 128, smem>>>(out, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
  unsigned long long h[160]; cudaMemcpy(h, out, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < sms; ++i) s += h[i];
  s /= sms;
  printf("%-44s %8.1f cycles/iter  %6.1f cycles/MMA\n", name, s / ITERS, s / ITERS / mmas_per_iter);
}
int main() {
  run<0>("4x i8 N64 K32, invariant descriptors", 4);
  run<1>("4x i8 N64 K32, K slot varies (ring of 4)", 4);
  run<2>("1x i8 N64 K32, invariant", 1);
  run<3>("4x f16 TS N128 K16, invariant", 4);
  run<4>("4x i8 N128 K32, invariant", 4);
  run<5>("1x i8 N16 K32, invariant", 1);
  run<6>("4x i8 N64 K32 + commit", 4);
  run<7>("1x i8 N64, D alternates", 1);
  run<8>("[warp+elect] 4x i8 N64 K32 invariant", 4);
  run<9>("[warp+elect] 1x i8 N16 K32 invariant", 1);
  run<10>("[warp+elect] 4x f16 TS N128 K16", 4);
  run<11>("[warp+elect] 4x i8 N64, K slot + D vary", 4);
  run<12>("4x i8 M64 N8 K32 (tiny)", 4);
  run<13>("4x tcgen05.commit", 4);
  run<14>("4x i8 M64 N8 in one asm", 4);
  run<15>("4x i8 N64 in one asm", 4);
  return 0;
}
