// Latency / throughput microbenchmark of the tcgen05 MMA groups and the
// mbarrier round trips of k_sparse_attn (sm_100a).  One CTA per SM (or two:
// argv[1]), 192 threads: warps 0-3 "softmax" relay, warp 5 MMA issuer.
//   mode 0  QK group (4 x kind::i8 M128 N64 K32) issue -> commit -> wait, latency
//   mode 1  PV group (4 x kind::f16 TS M128 N128 K16) issue -> commit -> wait
//   mode 2  QK groups back to back (throughput), mode 3 PV groups back to back
//   mode 4  QK group -> commit s_full -> relay warps wait + arrive p_full -> issuer wait
//   mode 5  mbarrier ping-pong issuer <-> relay warps, no MMA
//   mode 6  QK N=128 group latency, mode 7 bias(N64)+QK N64 group latency
//   mode 8  QK, PV, QK, PV ... back to back (kind switch every group)
//   mode 9  PV, bias, QK ... back to back (the kernel's per-tile sequence)
//   mode 10 QK, QK, PV, PV ... back to back (pairs)
//   mode 11 QK N=128 groups back to back, mode 12 bias N=128 + QK N=128 + 2 PV
//   mode 13-16 single kind::i8 M128 K32 MMAs back to back, N = 16 / 64 / 128 / 256
//   mode 17 PV TS N=256 groups back to back (4 MMAs), mode 18 commits back to back
// Operand contents are irrelevant (uninitialised smem): timing only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_18137_b200/csrc/sm100.cuh"
using namespace sparge;
#define ITERS 2000
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__global__ void __launch_bounds__(192) k(int mode, unsigned long long* out) {
  extern __shared__ unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 65536 + 64);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(bars, 1); mbar_init(bars + 1, 4); mbar_init(bars + 2, 1); fence_mbar_init(); }
  if (warp == 5) tmem_alloc<512>(slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = *slot;
  const uint64_t dQ = umma_desc_kmajor(smem_u32(sm), 128);
  const uint64_t dK = umma_desc_kmajor(smem_u32(sm + 16384), 128);
  const uint64_t dV = umma_desc_kmajor(smem_u32(sm + 32768), 128);
  const uint32_t iqk = idesc_i8(128, 64), iqk2 = idesc_i8(128, 128), ipv = idesc_bf16(128, 128), ib = idesc_bf16(128, 64);
  auto qk = [&](uint32_t n128) {
    for (int kk = 0; kk < 4; ++kk) mma_i8(tm, dQ + 2 * kk, dK + 2 * kk, n128 ? iqk2 : iqk, kk > 0);
  };
  auto pv = [&]() {
    for (int kk = 0; kk < 4; ++kk) mma_f16_ts(tm + 128, tm + 8 * kk, dV + 2 * kk, ipv, 1u);
  };
  if (warp == 5 && lane == 0) {
    long long t0 = clock64();
    if (mode == 0 || mode == 1 || mode == 6 || mode == 7) {
      for (int it = 0; it < ITERS; ++it) {
        if (mode == 7) mma_f16(tm, dQ, dK, ib, 0u);
        if (mode == 1) pv(); else qk(mode == 6);
        tc_commit(bars);
        mbar_wait(bars, it & 1);
      }
    } else if (mode == 2 || mode == 3 || mode >= 8) {
      for (int it = 0; it < ITERS; ++it) {
        if (mode == 3) pv();
        else if (mode == 2) qk(0);
        else if (mode == 8) { qk(0); pv(); }
        else if (mode == 9) { pv(); mma_f16(tm, dQ, dK, ib, 0u); qk(0); }
        else if (mode == 10) { qk(0); qk(0); pv(); pv(); }
        else if (mode == 11) qk(1);
        else if (mode == 12) { mma_f16(tm, dQ, dK, idesc_bf16(128, 128), 0u); qk(1); pv(); pv(); }
        else if (mode >= 13 && mode <= 16) {
          const uint32_t n = mode == 13 ? 16 : mode == 14 ? 64 : mode == 15 ? 128 : 256;
          mma_i8(tm, dQ, dK, idesc_i8(128, n), 1u);
        }
        else if (mode == 17) { for (int kk = 0; kk < 4; ++kk) mma_f16_ts(tm, tm + 256 + 8 * kk, dV + 2 * kk, idesc_bf16(128, 256), 1u); }
        else if (mode == 18) tc_commit(bars + 2);
      }
      tc_commit(bars);
      mbar_wait(bars, 0);
    } else if (mode == 4) {
      for (int it = 0; it < ITERS; ++it) {
        qk(0);
        tc_commit(bars);
        mbar_wait(bars + 1, it & 1);
      }
    } else if (mode == 5) {
      for (int it = 0; it < ITERS; ++it) {
        mbar_arrive(bars);
        mbar_wait(bars + 1, it & 1);
      }
    }
    long long t1 = clock64();
    out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  } else if (warp < 4 && (mode == 4 || mode == 5)) {
    for (int it = 0; it < ITERS; ++it) {
      mbar_wait(bars, it & 1);
      tc_fence_after();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bars + 1);
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 5) { __syncwarp(); tc_fence_after(); tmem_dealloc<512>(tm); }
}
int main(int argc, char** argv) {
  int per_sm = argc > 1 ? atoi(argv[1]) : 1;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 65536 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* out; cudaMalloc(&out, sizeof(unsigned long long) * sms * 2);
  const char* names[] = {"QK group latency (4x i8 N64 K32)", "PV group latency (4x f16 TS N128 K16)",
                         "QK groups back to back", "PV groups back to back",
                         "QK + relay round trip (4 warps)", "mbarrier ping-pong (no MMA)",
                         "QK N128 group latency", "bias + QK N64 group latency",
                         "QK,PV alternating (per QK+PV)", "PV,bias,QK (per tile)", "QK,QK,PV,PV (per 2 tiles)",
                         "QK N128 back to back", "biasN128,QKN128,PV,PV (per 2 tiles)",
                         "i8 M128 N16 K32 single MMA", "i8 M128 N64 K32 single MMA", "i8 M128 N128 K32 single MMA",
                         "i8 M128 N256 K32 single MMA", "PV TS N256 group (4 MMAs)", "tcgen05.commit alone"};
  for (int mode = 0; mode < 19; ++mode) {
    k<<<sms * per_sm, 192, smem>>>(mode, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    unsigned long long h[296]; cudaMemcpy(h, out, sizeof(unsigned long long) * sms * per_sm, cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < sms * per_sm; ++i) s += h[i];
    printf("%d CTA/SM  %-40s %8.1f cycles/iter\n", per_sm, names[mode], s / (sms * per_sm) / ITERS);
  }
  return 0;
}
