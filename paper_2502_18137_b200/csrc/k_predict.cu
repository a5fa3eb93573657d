// k_predict_topcdf -- step a2 of the hot path.
//
// One CTA per (query block i, q-head, batch).  From the a1 statistics it
// forms one row of the compressed attention map and the block mask M_g:
//   S^[j] = q_i . k_j / sqrt(d)                 Alg. 1 line 5, R2
//   S^[j] = -inf if s_kj < theta (strict, R5) or tile (i,j) causally dead (R8)
//   P^   = softmax(S^)                          line 6
//   M[i,:] = TopCdf(P^, tau)                    §3.2 pseudocode, R4:
//       order (P^ desc, j asc); keep rank k iff cumsum_k <= tau*cumsum_last;
//       always keep rank 0 (guard)
//   M[i,:] = 1 if s_qi < theta; M[:,j] = 1 if s_kj < theta    Eq. 5
//   all -inf row -> all ones (R7); causal: M &= live, M[i, i*bq/bk] = 1 (R8)
// and compacts the kept j (ascending) into the LUT the attention kernel
// walks.  Everything is fp64 (R15): masks are then exact versus the oracle
// up to decisions within ~1e-13 of a threshold.
// Bound: fp64 ALU + a shared-memory bitonic sort of T_n (<= 4096) entries.
#include <cstdint>
#include <cfloat>

#include "sparge_internal.h"

namespace sparge {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ bool before(double ka, int ia, double kb, int ib) {
  return (ka > kb) || (ka == kb && ia < ib);
}

// Block-wide exclusive scan of one double per thread (fixed order).
__device__ double block_excl_scan(double v, double* s_warp, double* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  double off = 0.0, tot = 0.0;
  for (int w = 0; w < kWarps; ++w) {
    if (w < wid) off += s_warp[w];
    tot += s_warp[w];
  }
  __syncthreads();
  *total = tot;
  return off + incl - v;
}

__device__ int block_excl_scan_int(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  int off = 0, tot = 0;
  for (int w = 0; w < kWarps; ++w) {
    if (w < wid) off += s_warp[w];
    tot += s_warp[w];
  }
  __syncthreads();
  *total = tot;
  return off + incl - v;
}

template <int D>
__global__ void __launch_bounds__(kThreads)
k_predict_topcdf(const double* __restrict__ q_pooled, const double* __restrict__ q_sim,
                 const double* __restrict__ k_pooled, const double* __restrict__ k_sim,
                 int Hq, int Hkv, int N, int T_m, int T_n, int sortn, int bq, int bk,
                 int causal, double tau, double theta,
                 uint8_t* __restrict__ mask, int32_t* __restrict__ lut,
                 int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_key = reinterpret_cast<double*>(smem);               // [sortn]
  int* s_idx = reinterpret_cast<int*>(s_key + sortn);            // [sortn]
  uint8_t* s_flag = reinterpret_cast<uint8_t*>(s_idx + sortn);   // [sortn]
  __shared__ double s_q[D];
  __shared__ double s_wd[kWarps];
  __shared__ int s_wi[kWarps];

  const int i = blockIdx.x, hq = blockIdx.y, b = blockIdx.z;
  const int hkv = hq / (Hq / Hkv);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t qrow = (static_cast<int64_t>(b) * Hq + hq) * T_m + i;
  const int64_t kbase = (static_cast<int64_t>(b) * Hkv + hkv) * T_n;
  const double sqrt_d = sqrt(static_cast<double>(D));
  const int last_q = min((i + 1) * bq, N) - 1;

  for (int c = tid; c < D; c += kThreads) s_q[c] = q_pooled[qrow * D + c];
  __syncthreads();

  // ---- S^ row: one warp per key block j ----
  for (int j = wid; j < T_n; j += kWarps) {
    const double* kb = k_pooled + (kbase + j) * D;
    double dot = 0.0;
#pragma unroll
    for (int c = lane; c < D; c += 32) dot = fma(s_q[c], kb[c], dot);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) {
      const bool dead = causal && (j * bk > last_q);
      const bool fix = k_sim[kbase + j] < theta;
      s_key[j] = (dead || fix) ? -INFINITY : dot / sqrt_d;
    }
  }
  __syncthreads();

  // ---- row max ----
  double mx = -INFINITY;
  for (int j = tid; j < T_n; j += kThreads) mx = fmax(mx, s_key[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_wd[wid] = mx;
  __syncthreads();
  mx = s_wd[0];
  for (int w = 1; w < kWarps; ++w) mx = fmax(mx, s_wd[w]);
  __syncthreads();
  const bool flagged = (mx == -INFINITY);   // every K block fixed / dead (R7)

  if (!flagged) {
    // ---- softmax (fp64), contiguous chunk per thread ----
    const int per = (T_n + kThreads - 1) / kThreads;
    const int j0 = tid * per, j1 = min(T_n, j0 + per);
    double part = 0.0;
    for (int j = j0; j < j1; ++j) {
      const double e = (s_key[j] == -INFINITY) ? 0.0 : exp(s_key[j] - mx);
      s_key[j] = e;
      part += e;
    }
    double total;
    block_excl_scan(part, s_wd, &total);
    for (int j = j0; j < j1; ++j) s_key[j] = s_key[j] / total;
    for (int j = tid; j < sortn; j += kThreads) {
      s_idx[j] = j;
      if (j >= T_n) s_key[j] = -1.0;   // padding sorts last (P^ >= 0)
    }
    __syncthreads();

    // ---- bitonic sort into (P^ desc, j asc) ----
    for (int k = 2; k <= sortn; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int t = tid; t < sortn / 2; t += kThreads) {
          const int a = 2 * jj * (t / jj) + (t % jj);
          const int c = a + jj;
          const double ka = s_key[a], kc = s_key[c];
          const int ia = s_idx[a], ic = s_idx[c];
          const bool up = (a & k) == 0;
          const bool swap = up ? before(kc, ic, ka, ia) : before(ka, ia, kc, ic);
          if (swap) {
            s_key[a] = kc; s_key[c] = ka;
            s_idx[a] = ic; s_idx[c] = ia;
          }
        }
        __syncthreads();
      }
    }

    // ---- inclusive cumulative sum in rank order, threshold ----
    const int pr = (sortn + kThreads - 1) / kThreads;
    const int k0 = tid * pr, k1 = min(T_n, k0 + pr);
    double loc = 0.0;
    for (int k = k0; k < k1; ++k) loc += s_key[k];
    double csum_total;
    const double off = block_excl_scan(loc, s_wd, &csum_total);
    double c = off;
    for (int k = k0; k < k1; ++k) {
      c += s_key[k];
      s_key[k] = c;
    }
    // c_last, the last element of the cumulative sum (R4).  In exact
    // arithmetic the cumsum is monotone and c_last is its maximum; taking the
    // maximum of the computed values keeps "tau = 1 keeps every rank" exact
    // when the parallel scan's rounding makes the sequence non-monotone by
    // an ulp.
    double cmax = (k1 > k0) ? c : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    if (lane == 0) s_wd[wid] = cmax;
    __syncthreads();
    cmax = s_wd[0];
    for (int w = 1; w < kWarps; ++w) cmax = fmax(cmax, s_wd[w]);
    const double thr = tau * cmax;
    for (int k = k0; k < k1; ++k) s_flag[s_idx[k]] = (s_key[k] <= thr || k == 0) ? 1 : 0;
    __syncthreads();
  }

  // ---- forcing (Eq. 5), flagged rows, causal live AND + diagonal guard ----
  const bool row_fix = q_sim[qrow] < theta;
  const int guard = (i * bq) / bk;
  for (int j = tid; j < T_n; j += kThreads) {
    uint8_t f = flagged ? 1 : s_flag[j];
    if (row_fix || k_sim[kbase + j] < theta) f = 1;
    if (causal) {
      if (j * bk > last_q) f = 0;
      if (j == guard) f = 1;
    }
    s_flag[j] = f;
  }
  __syncthreads();

  // ---- write M_g row and compact the kept j (ascending) ----
  uint8_t* mrow = mask ? mask + qrow * T_n : nullptr;
  const int per = (T_n + kThreads - 1) / kThreads;
  const int j0 = tid * per, j1 = min(T_n, j0 + per);
  int mine = 0;
  for (int j = j0; j < j1; ++j) {
    mine += s_flag[j];
    if (mrow) mrow[j] = s_flag[j];
  }
  int total_kept;
  int pos = block_excl_scan_int(mine, s_wi, &total_kept);
  int32_t* lrow = lut + qrow * T_n;
  for (int j = j0; j < j1; ++j)
    if (s_flag[j]) lrow[pos++] = j;
  if (tid == 0) cnt[qrow] = total_kept;
}

}  // namespace

cudaError_t launch_predict(const sparge_shape& s, const double* q_pooled, const double* q_sim,
                           const double* k_pooled, const double* k_sim, float tau, float theta,
                           uint8_t* mask, int32_t* lut, int32_t* cnt, cudaStream_t stream) {
  const int T_m = (s.N + s.bq - 1) / s.bq;
  const int T_n = (s.N + s.bk - 1) / s.bk;
  int sortn = 1;
  while (sortn < T_n) sortn <<= 1;
  const size_t smem = static_cast<size_t>(sortn) * (sizeof(double) + sizeof(int) + 1);
  dim3 grid(T_m, s.Hq, s.B);
  if (s.d == 128) {
    cudaFuncSetAttribute(k_predict_topcdf<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    k_predict_topcdf<128><<<grid, kThreads, smem, stream>>>(
        q_pooled, q_sim, k_pooled, k_sim, s.Hq, s.Hkv, s.N, T_m, T_n, sortn, s.bq, s.bk,
        s.causal, static_cast<double>(tau), static_cast<double>(theta), mask, lut, cnt);
  } else {
    cudaFuncSetAttribute(k_predict_topcdf<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    k_predict_topcdf<64><<<grid, kThreads, smem, stream>>>(
        q_pooled, q_sim, k_pooled, k_sim, s.Hq, s.Hkv, s.N, T_m, T_n, sortn, s.bq, s.bk,
        s.causal, static_cast<double>(tau), static_cast<double>(theta), mask, lut, cnt);
  }
  return cudaGetLastError();
}

}  // namespace sparge
