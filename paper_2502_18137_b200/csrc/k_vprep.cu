// k_vprep -- V staging for the P~V product of step a3.
//
// Writes V^T[b, hkv, c, r] = V[b, hkv, perm[r], c] (zero for r >= N) so that
// every 64-key tile of V is a K-major UMMA B operand (64 keys = 128 bytes per
// row, SWIZZLE_128B), loaded by one TMA box per kept tile.  The Hilbert
// gather of §3.7 is fused here.  Bound: HBM (2 B read + 2 B write
// per element).
#include <cstdint>

#include "sparge_internal.h"

namespace sparge {

namespace {

template <int D>
__global__ void __launch_bounds__(256)
k_vprep(const uint16_t* __restrict__ v, int64_t sb, int64_t sh, int64_t sn,
        const int32_t* __restrict__ perm, int Hkv, int N, int n_pad,
        uint16_t* __restrict__ vt) {
  constexpr int BK = 64;
  constexpr int PAD = 8;
  __shared__ __align__(16) uint16_t tile[BK][D + PAD];
  const int jb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x;
  const uint16_t* vbh = v + b * sb + h * sh;
  // load 64 rows x D (16 B per thread per step), gathered through perm
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
  // write D rows x 64 keys: 8 keys (16 B) per thread per step
  uint16_t* out = vt + ((static_cast<int64_t>(b) * Hkv + h) * D) * n_pad + jb * BK;
  for (int e = tid; e < D * (BK / 8); e += 256) {
    const int c = e / (BK / 8), k8 = e % (BK / 8);
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      w[q] = static_cast<uint32_t>(tile[k8 * 8 + 2 * q][c]) |
             (static_cast<uint32_t>(tile[k8 * 8 + 2 * q + 1][c]) << 16);
    *reinterpret_cast<uint4*>(out + static_cast<int64_t>(c) * n_pad + k8 * 8) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

}  // namespace

cudaError_t launch_vprep(const sparge_shape& s, const void* v, sparge_strides st,
                         const int32_t* perm, void* vt, int n_pad, cudaStream_t stream) {
  dim3 grid(n_pad / 64, s.Hkv, s.B);
  if (s.d == 128)
    k_vprep<128><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(v), st.b, st.h, st.n,
                                           perm, s.Hkv, s.N, n_pad, static_cast<uint16_t*>(vt));
  else
    k_vprep<64><<<grid, 256, 0, stream>>>(static_cast<const uint16_t*>(v), st.b, st.h, st.n,
                                          perm, s.Hkv, s.N, n_pad, static_cast<uint16_t*>(vt));
  return cudaGetLastError();
}

}  // namespace sparge
