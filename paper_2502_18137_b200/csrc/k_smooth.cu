// K smoothing, scope row f4 (SageAttention-style "smooth K", footnote
// P:L44; reading R28): mu[b, h_kv, c] = the token mean of K per channel, in
// the fixed fp64 summation order of R28 -- tokens in index order within
// chunks of 128 (a sequential sum per chunk), the chunk sums added in chunk
// order, / N, rounded to fp32 -- so the oracle reproduces it bit for bit.
// k_smooth_partial: one thread per (chunk, channel), reading 16-bit K rows
// (coalesced: consecutive threads, consecutive channels); k_smooth_final:
// one thread per channel over the chunk sums.  The quantiser then uses
// fl32(K - mu) for the INT8 path (k_quant.cu).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "sparge_internal.h"

namespace sparge {

namespace {

constexpr int kChunk = 128;

template <typename T>
__device__ __forceinline__ double widen(T v);
template <>
__device__ __forceinline__ double widen<__nv_bfloat16>(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}
template <>
__device__ __forceinline__ double widen<__half>(__half v) {
  return static_cast<double>(__half2float(v));
}

template <typename T>
__global__ void k_smooth_partial(const T* __restrict__ k, int64_t sb, int64_t sh, int64_t sn,
                                 int Hkv, int N, int d, int n_chunks, double* __restrict__ part) {
  const int chunk = blockIdx.x, bh = blockIdx.y, c = threadIdx.x;
  const int h = bh % Hkv, b = bh / Hkv;
  const T* x = k + b * sb + h * sh + c;
  const int t0 = chunk * kChunk, t1 = min(N, t0 + kChunk);
  double s = 0.0;
  for (int t = t0; t < t1; ++t) s += widen<T>(x[static_cast<int64_t>(t) * sn]);
  part[(static_cast<int64_t>(bh) * n_chunks + chunk) * d + c] = s;
}

__global__ void k_smooth_final(const double* __restrict__ part, int N, int d, int n_chunks,
                               float* __restrict__ mean) {
  const int bh = blockIdx.x, c = threadIdx.x;
  const double* p = part + static_cast<int64_t>(bh) * n_chunks * d + c;
  double s = 0.0;
  for (int q = 0; q < n_chunks; ++q) s += p[static_cast<int64_t>(q) * d];
  mean[static_cast<int64_t>(bh) * d + c] = static_cast<float>(s / static_cast<double>(N));
}

}  // namespace

size_t smooth_partial_bytes(const sparge_shape& s) {
  const size_t n_chunks = (s.N + kChunk - 1) / kChunk;
  return sizeof(double) * static_cast<size_t>(s.B) * s.Hkv * n_chunks * s.d;
}

cudaError_t launch_smooth_mean(const sparge_shape& s, const void* k, sparge_strides st,
                               double* part, float* mean, cudaStream_t stream) {
  const int n_chunks = (s.N + kChunk - 1) / kChunk;
  dim3 g1(n_chunks, s.B * s.Hkv);
  if (s.in_dtype == SPARGE_FP16)
    k_smooth_partial<__half><<<g1, s.d, 0, stream>>>(static_cast<const __half*>(k), st.b, st.h,
                                                     st.n, s.Hkv, s.N, s.d, n_chunks, part);
  else
    k_smooth_partial<__nv_bfloat16><<<g1, s.d, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(k), st.b, st.h, st.n, s.Hkv, s.N, s.d, n_chunks, part);
  k_smooth_final<<<s.B * s.Hkv, s.d, 0, stream>>>(part, s.N, s.d, n_chunks, mean);
  return cudaGetLastError();
}

}  // namespace sparge
