// k_l1_sums -- the accuracy metric of §3.6: relative L1
//   L1 = sum |O - O'| / sum |O'|        (reading R17: the reference O' in
//                                         the denominator)
// used by the hyper-parameter tuner (scope row f2) and the permutation study
// (f3) to score a sparse output O against the dense reference O' without
// leaving the device.  Two 16-bit tensors of n elements (bf16 or fp16, same
// dtype, contiguous); fp64 accumulation; deterministic (fixed grid, fixed
// per-block tree, then one block folds the partials in order).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "sparge_internal.h"

namespace sparge {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float h2f(uint16_t b, bool f16) {
  return f16 ? __half2float(__ushort_as_half(b)) : __uint_as_float(static_cast<uint32_t>(b) << 16);
}

__device__ __forceinline__ void block_sum2(double& a, double& b, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[2 * w] = a; sh[2 * w + 1] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0.0; b = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) { a += sh[2 * k]; b += sh[2 * k + 1]; }
  }
}

__global__ void __launch_bounds__(kThreads)
k_l1_partial(const uint16_t* __restrict__ o, const uint16_t* __restrict__ r, int64_t n, int f16,
             double* __restrict__ part) {
  __shared__ double sh[2 * kThreads / 32];
  double a = 0.0, b = 0.0;
  // 8 elements (16 B) per thread per step; tail element-wise
  const int64_t n8 = n / 8;
  const uint4* o8 = reinterpret_cast<const uint4*>(o);
  const uint4* r8 = reinterpret_cast<const uint4*>(r);
  for (int64_t k = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; k < n8;
       k += static_cast<int64_t>(gridDim.x) * kThreads) {
    const uint4 x = __ldg(o8 + k), y = __ldg(r8 + k);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
    float fa = 0.f, fb = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float x0 = h2f(static_cast<uint16_t>(xs[e]), f16), x1 = h2f(static_cast<uint16_t>(xs[e] >> 16), f16);
      const float y0 = h2f(static_cast<uint16_t>(ys[e]), f16), y1 = h2f(static_cast<uint16_t>(ys[e] >> 16), f16);
      fa += fabsf(x0 - y0) + fabsf(x1 - y1);   // 8-term fp32 partial, then fp64
      fb += fabsf(y0) + fabsf(y1);
    }
    a += fa;
    b += fb;
  }
  if (blockIdx.x == 0)
    for (int64_t k = n8 * 8 + threadIdx.x; k < n; k += kThreads) {
      const float x = h2f(o[k], f16), y = h2f(r[k], f16);
      a += fabsf(x - y);
      b += fabsf(y);
    }
  block_sum2(a, b, sh);
  if (threadIdx.x == 0) { part[2 * blockIdx.x] = a; part[2 * blockIdx.x + 1] = b; }
}

__global__ void __launch_bounds__(kThreads) k_l1_final(const double* __restrict__ part, int nb,
                                                       double* __restrict__ out) {
  __shared__ double sh[2 * kThreads / 32];
  double a = 0.0, b = 0.0;
  for (int k = threadIdx.x; k < nb; k += kThreads) { a += part[2 * k]; b += part[2 * k + 1]; }
  block_sum2(a, b, sh);
  if (threadIdx.x == 0) { out[0] = a; out[1] = b; }
}

}  // namespace

cudaError_t launch_l1_sums(const void* o, const void* o_ref, int f16, int64_t n, double* out,
                           cudaStream_t stream) {
  double* part = out + 2;
  k_l1_partial<<<kL1Blocks, kThreads, 0, stream>>>(static_cast<const uint16_t*>(o),
                                                   static_cast<const uint16_t*>(o_ref), n, f16, part);
  k_l1_final<<<1, kThreads, 0, stream>>>(part, kL1Blocks, out);
  return cudaGetLastError();
}

}  // namespace sparge
