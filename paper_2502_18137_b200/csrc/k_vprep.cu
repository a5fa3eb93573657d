// k_vprep -- V staging for the P~V product of step a3.
//
// Writes V^T[b, hkv, r / 64, c, r % 64] = V[b, hkv, perm[r], c] (zero for
// r >= N; tile-major, kVtTiled) so that every 64-key tile of V is a K-major
// UMMA B operand (64 keys = 128 bytes per row, SWIZZLE_128B) stored as one
// contiguous block and loaded by one TMA box per kept tile.  The Hilbert
// gather of §3.7 is fused here.  Bound: HBM (2 B read + 2 B write
// per element).
#include <cuda_fp16.h>
#include <cstdint>

#include "sm100.cuh"
#include "sparge_internal.h"

namespace sparge {

namespace {

template <int D>
__global__ void __launch_bounds__(256)
k_vprep(const uint16_t* __restrict__ v, int64_t sb, int64_t sh, int64_t sn,
        const int32_t* __restrict__ perm, int Hkv, int N, int n_pad,
        uint16_t* __restrict__ vt, int early) {
  constexpr int BK = 64;
  constexpr int PAD = 8;
  __shared__ __align__(16) uint16_t tile[BK][D + PAD];
  const int jb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x;
  const uint16_t* vbh = v + b * sb + h * sh;
  // PDL (sparge_internal.h).  early = 1 when launched right after k_order
  // inside one attention call (sparge_attn_fwd): V and V^T are touched by no
  // kernel after the caller's last one before the call (complete: k_order_head
  // waited for it before k_order_groups let this grid start), so the staging
  // overlaps the launch-order kernels and waits for them only at its end --
  // the attention kernel's wait on this grid then covers k_order too
  if (!early) griddep_wait();
  griddep_launch();
  // load 64 rows x D (16 B per thread per step), gathered through perm; the
  // source rows are looked up first so their loads are all in flight at once
  constexpr int CPR = D / 8;
  constexpr int NL = BK * CPR / 256;
  int src[NL];
#pragma unroll
  for (int q = 0; q < NL; ++q) {
    const int row = jb * BK + (tid + q * 256) / CPR;
    src[q] = row < N ? (perm ? __ldg(perm + row) : row) : -1;
  }
  uint4 val[NL];
#pragma unroll
  for (int q = 0; q < NL; ++q) {
    const int c8 = (tid + q * 256) % CPR;
    val[q] = src[q] >= 0
                 ? __ldg(reinterpret_cast<const uint4*>(vbh + static_cast<int64_t>(src[q]) * sn + c8 * 8))
                 : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int q = 0; q < NL; ++q) {
    const int e = tid + q * 256;
    *reinterpret_cast<uint4*>(&tile[e / CPR][(e % CPR) * 8]) = val[q];
  }
  __syncthreads();
  // write D rows x 64 keys: thread (c, k16) packs 16 keys (32 B); lanes run
  // over consecutive c, so the column reads of the tile are conflict-free
  // tile-major: this CTA's 64-key tile is one contiguous [D][64] block
  uint16_t* out = kVtTiled ? vt + ((static_cast<int64_t>(b) * Hkv + h) * (n_pad / BK) + jb) * D * BK
                           : vt + ((static_cast<int64_t>(b) * Hkv + h) * D) * n_pad + jb * BK;
  const int64_t row_stride = kVtTiled ? BK : n_pad;
#pragma unroll
  for (int e = tid; e < D * (BK / 16); e += 256) {
    const int c = e % D, k16 = e / D;
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      w[q] = static_cast<uint32_t>(tile[k16 * 16 + 2 * q][c]) |
             (static_cast<uint32_t>(tile[k16 * 16 + 2 * q + 1][c]) << 16);
    uint4* o4 = reinterpret_cast<uint4*>(out + static_cast<int64_t>(c) * row_stride + k16 * 16);
    o4[0] = make_uint4(w[0], w[1], w[2], w[3]);
    o4[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
  if (early) griddep_wait();   // this grid completes only after k_order has
}

}  // namespace

cudaError_t launch_vprep(const sparge_shape& s, const void* v, sparge_strides st,
                         const int32_t* perm, void* vt, int n_pad, bool early,
                         cudaStream_t stream) {
  dim3 grid(n_pad / 64, s.Hkv, s.B);
  return launch_k(kPdlVprep, s.d == 128 ? k_vprep<128> : k_vprep<64>, grid, dim3(256), 0, stream,
                  static_cast<const uint16_t*>(v), st.b, st.h, st.n, perm, s.Hkv, s.N, n_pad,
                  static_cast<uint16_t*>(vt), early ? 1 : 0);
}

}  // namespace sparge

// ---------------------------------------------------------------------------
// f4 (FP8 P~V, SageAttention2-style, footnote P:L44; reading R27): V is
// quantised per channel over all N tokens of its (b, kv-head): amax_c =
// max_r |V[r, c]|, V^ = e4m3_rn_satfinite(fl32(V * fl32(448 / amax_c))),
// s_c = fl32(amax_c / 448) (all-zero channel: 1, 1).  Two passes: k_vamax
// (atomicMax of the non-negative fp32 bits -- order-independent, so
// deterministic) and k_vprep_fp8 (gather + quantise + transpose to
// [b, hkv, c, r] bytes: 64 keys = 64 B per row, a SWIZZLE_64B UMMA operand).
namespace sparge {

namespace {

template <int D>
__global__ void __launch_bounds__(256)
k_vamax(const uint16_t* __restrict__ v, int64_t sb, int64_t sh, int64_t sn, int N, int f16,
        unsigned int* __restrict__ amax_bits) {
  constexpr int EPL = D / 32;
  __shared__ float s_m[8][D];
  const int h = blockIdx.y, b = blockIdx.z, Hkv = gridDim.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint16_t* vbh = v + b * sb + h * sh;
  float m[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) m[e] = 0.f;
  for (int r = blockIdx.x * 256 + wid; r < min(N, (blockIdx.x + 1) * 256); r += 8) {
    const uint16_t* row = vbh + static_cast<int64_t>(r) * sn + lane * EPL;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const uint32_t bits = row[e];
      const float f = f16 ? __half2float(__ushort_as_half(static_cast<unsigned short>(bits)))
                          : __uint_as_float(bits << 16);
      m[e] = fmaxf(m[e], fabsf(f));
    }
  }
#pragma unroll
  for (int e = 0; e < EPL; ++e) s_m[wid][lane * EPL + e] = m[e];
  __syncthreads();
  if (threadIdx.x < D) {
    float mm = s_m[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < 8; ++w) mm = fmaxf(mm, s_m[w][threadIdx.x]);
    atomicMax(amax_bits + (static_cast<int64_t>(b) * Hkv + h) * D + threadIdx.x, __float_as_uint(mm));
  }
}

template <int D>
__global__ void __launch_bounds__(256)
k_vprep_fp8(const uint16_t* __restrict__ v, int64_t sb, int64_t sh, int64_t sn,
            const int32_t* __restrict__ perm, int Hkv, int N, int n_pad, int f16,
            const unsigned int* __restrict__ amax_bits, uint8_t* __restrict__ vt8,
            float* __restrict__ v_scale) {
  constexpr int BK = 64;
  constexpr int PAD = 8;
  __shared__ __align__(16) uint16_t tile[BK][D + PAD];
  __shared__ float s_inv[D];
  const int jb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x;
  const int64_t bh = static_cast<int64_t>(b) * Hkv + h;
  const uint16_t* vbh = v + b * sb + h * sh;
  if (tid < D) {
    const float amax = __uint_as_float(__ldg(amax_bits + bh * D + tid));
    s_inv[tid] = (amax > 0.f) ? __fdiv_rn(448.f, amax) : 1.f;
    if (jb == 0) v_scale[bh * D + tid] = (amax > 0.f) ? __fdiv_rn(amax, 448.f) : 1.f;
  }
  constexpr int CPR = D / 8;
  for (int e = tid; e < BK * CPR; e += 256) {
    const int r = e / CPR, c8 = e % CPR;
    const int row = jb * BK + r;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (row < N) {
      const int src = perm ? __ldg(perm + row) : row;
      val = __ldg(reinterpret_cast<const uint4*>(vbh + static_cast<int64_t>(src) * sn + c8 * 8));
    }
    *reinterpret_cast<uint4*>(&tile[r][c8 * 8]) = val;
  }
  __syncthreads();
  // D rows x 64 keys of bytes: 8 keys (8 B) per thread per step
  uint8_t* out = vt8 + (bh * D) * n_pad + jb * BK;
  for (int e = tid; e < D * (BK / 8); e += 256) {
    const int c = e / (BK / 8), k8 = e % (BK / 8);
    const float inv = s_inv[c];
    uint32_t w[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t word = 0;
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        float f[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t bits = tile[k8 * 8 + q * 4 + pp * 2 + u][c];
          const float x = f16 ? __half2float(__ushort_as_half(static_cast<unsigned short>(bits)))
                              : __uint_as_float(bits << 16);
          f[u] = __fmul_rn(x, inv);
        }
        unsigned short r2;
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r2) : "f"(f[1]), "f"(f[0]));
        word |= static_cast<uint32_t>(r2) << (16 * pp);
      }
      w[q] = word;
    }
    *reinterpret_cast<uint2*>(out + static_cast<int64_t>(c) * n_pad + k8 * 8) = make_uint2(w[0], w[1]);
  }
}

}  // namespace

cudaError_t launch_vprep_fp8(const sparge_shape& s, const void* v, sparge_strides st,
                             const int32_t* perm, uint8_t* vt8, unsigned int* amax_bits,
                             float* v_scale, int n_pad, cudaStream_t stream) {
  const int f16 = s.in_dtype == SPARGE_FP16;
  cudaError_t e = cudaMemsetAsync(amax_bits, 0, sizeof(unsigned int) * s.B * s.Hkv * s.d, stream);
  if (e != cudaSuccess) return e;
  dim3 ga((s.N + 255) / 256, s.Hkv, s.B);
  dim3 gp(n_pad / 64, s.Hkv, s.B);
  const uint16_t* vv = static_cast<const uint16_t*>(v);
  if (s.d == 128) {
    k_vamax<128><<<ga, 256, 0, stream>>>(vv, st.b, st.h, st.n, s.N, f16, amax_bits);
    k_vprep_fp8<128><<<gp, 256, 0, stream>>>(vv, st.b, st.h, st.n, perm, s.Hkv, s.N, n_pad, f16,
                                             amax_bits, vt8, v_scale);
  } else {
    k_vamax<64><<<ga, 256, 0, stream>>>(vv, st.b, st.h, st.n, s.N, f16, amax_bits);
    k_vprep_fp8<64><<<gp, 256, 0, stream>>>(vv, st.b, st.h, st.n, perm, s.Hkv, s.N, n_pad, f16,
                                            amax_bits, vt8, v_scale);
  }
  return cudaGetLastError();
}

}  // namespace sparge
