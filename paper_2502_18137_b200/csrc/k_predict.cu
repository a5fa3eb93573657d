// k_predict_topcdf -- step a2 of the hot path.
//
// One CTA per (8 query blocks, q-head, batch).  From the a1 statistics it
// forms the rows of the compressed attention map and the block mask M_g:
//   S^[j] = q_i . k_j / sqrt(d)                 Alg. 1 line 5, R2
//   S^[j] = -inf if s_kj < theta (strict, R5) or tile (i,j) causally dead (R8)
//   P^   = softmax(S^)                          line 6
//   M[i,:] = TopCdf(P^, tau)                    §3.2 pseudocode, R4:
//       order (P^ desc, j asc); keep rank k iff cumsum_k <= tau*c_last;
//       always keep rank 0 (guard)
//   M[i,:] = 1 if s_qi < theta; M[:,j] = 1 if s_kj < theta    Eq. 5
//   all -inf row -> all ones (R7); causal: M &= live, M[i, i*bq/bk] = 1 (R8)
// and compacts the kept j (ascending) into the LUT the attention kernel
// walks.  Everything is fp64 (R15).
//
// Phase A (all 8 warps): S^ for the CTA's 8 rows.  The pooled keys of the
//   kv-head stream through shared memory in 32-row chunks (cp.async, double
//   buffered, rows padded to d+1 doubles: conflict-free), so each chunk is
//   read from L2 once per 8 query blocks; warp w computes row w, lane l key
//   j0+l.
// Phase B (warp w owns row w): softmax, warp-synchronous bitonic sort of
//   (P^ desc, j asc) in shared memory, warp scan, threshold, forcing,
//   causal AND + guard, ballot compaction into the LUT.
// Bound: fp64 FMA + shared memory; no block-wide barrier in phase B.
#include <cstdint>
#include <cfloat>

#include "sparge_internal.h"

namespace sparge {

namespace {

constexpr int kThreads = 256;
constexpr int kRows = 8;         // query blocks per CTA (one per warp in phase B)
constexpr int kChunk = 32;       // pooled keys per shared-memory chunk

// Warp-synchronous bitonic sort, descending, of SORTN 64-bit keys in shared
// memory; branch-free compare-exchange, fully unrolled per stage.
template <int SORTN>
__device__ __forceinline__ void sort_desc(uint64_t* key, int lane) {
#pragma unroll 1
  for (int k = 2; k <= SORTN; k <<= 1) {
#pragma unroll 1
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
#pragma unroll
      for (int u = 0; u < (SORTN / 2 + 31) / 32; ++u) {
        const int t = lane + 32 * u;
        if (SORTN >= 64 || t < SORTN / 2) {
          // pair (a, a + jj): a = 2*jj*(t / jj) + t % jj, jj a power of two
          const int a = t + (t & ~(jj - 1));
          const int c = a + jj;
          const uint64_t ka = key[a], kc = key[c];
          const bool desc_block = (a & k) == 0;
          const bool sw = desc_block ? (kc > ka) : (ka > kc);
          key[a] = sw ? kc : ka;
          key[c] = sw ? ka : kc;
        }
      }
      __syncwarp();
    }
  }
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;"
               ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int D>
struct PredSmem {
  static constexpr int KROW = D + 1;                         // padded pooled-key row (doubles)
  static constexpr int KBUF = kChunk * KROW;                 // doubles per chunk buffer
  // layout: q[kRows][D] | kbuf[2][KBUF] (phase A) aliased by idx[kRows][sortn] u16
  //         (phase B) | key[kRows][sortn] f64 | flag[kRows][sortn] u8
  static size_t bytes(int sortn) {
    const size_t q = sizeof(double) * kRows * D;
    const size_t kb = sizeof(double) * 2 * KBUF;
    const size_t idx = sizeof(uint16_t) * kRows * sortn;
    const size_t u = kb > idx ? kb : idx;
    return q + u + sizeof(double) * kRows * sortn + static_cast<size_t>(kRows) * sortn;
  }
};

template <int D>
__global__ void __launch_bounds__(kThreads)
k_predict_topcdf(const double* __restrict__ q_pooled, const double* __restrict__ q_sim,
                 const double* __restrict__ k_pooled, const double* __restrict__ k_sim,
                 int Hq, int Hkv, int N, int T_m, int T_n, int sortn, int bq, int bk,
                 int causal, double tau, double theta,
                 uint8_t* __restrict__ mask, int32_t* __restrict__ lut,
                 int32_t* __restrict__ cnt) {
  using L = PredSmem<D>;
  extern __shared__ __align__(16) unsigned char smem[];
  double* s_q = reinterpret_cast<double*>(smem);                              // [kRows][D]
  double* s_kb = s_q + kRows * D;                                             // [2][KBUF]
  const size_t u_bytes = (sizeof(double) * 2 * L::KBUF > sizeof(uint16_t) * kRows * sortn)
                             ? sizeof(double) * 2 * L::KBUF
                             : sizeof(uint16_t) * kRows * sortn;
  double* s_key = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(s_kb) + u_bytes);
  uint8_t* s_flag = reinterpret_cast<uint8_t*>(s_key + kRows * sortn);

  const int hq = blockIdx.y, b = blockIdx.z;
  const int hkv = hq / (Hq / Hkv);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int i0 = blockIdx.x * kRows;
  const int64_t qbase = (static_cast<int64_t>(b) * Hq + hq) * T_m;
  const int64_t kbase = (static_cast<int64_t>(b) * Hkv + hkv) * T_n;
  const double sqrt_d = sqrt(static_cast<double>(D));

  // ---------------- phase A: S^ rows ----------------
  for (int e = tid; e < kRows * D; e += kThreads) {
    const int rr = e / D;
    s_q[e] = (i0 + rr < T_m) ? q_pooled[(qbase + i0 + rr) * D + (e % D)] : 0.0;
  }
  const int nchunks = (T_n + kChunk - 1) / kChunk;
  auto issue = [&](int c) {
    double* dst = s_kb + (c & 1) * L::KBUF;
    const int j0 = c * kChunk;
    for (int e = tid; e < kChunk * D; e += kThreads) {
      const int jj = e / D, dd = e % D;
      if (j0 + jj < T_n) cp_async8(dst + jj * L::KROW + dd, k_pooled + (kbase + j0 + jj) * D + dd);
    }
    cp_async_commit();
  };
  issue(0);
  const int my_row = i0 + wid;
  const int last_q = min((my_row + 1) * bq, N) - 1;
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      issue(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* kc = s_kb + (c & 1) * L::KBUF + lane * L::KROW;
    const double* qr = s_q + wid * D;
    double dot0 = 0.0, dot1 = 0.0;
#pragma unroll 8
    for (int dd = 0; dd < D; dd += 2) {
      dot0 = fma(qr[dd], kc[dd], dot0);
      dot1 = fma(qr[dd + 1], kc[dd + 1], dot1);
    }
    const int j = c * kChunk + lane;
    if (j < T_n && my_row < T_m) {
      const bool dead = causal && (j * bk > last_q);
      const bool fix = k_sim[kbase + j] < theta;
      s_key[wid * sortn + j] = (dead || fix) ? -INFINITY : (dot0 + dot1) / sqrt_d;
    }
    __syncthreads();
  }

  // ---------------- phase B: one warp per row ----------------
  if (my_row >= T_m) return;
  double* key = s_key + wid * sortn;
  uint8_t* flag = s_flag + wid * sortn;

  double mx = -INFINITY;
  for (int j = lane; j < T_n; j += 32) mx = fmax(mx, key[j]);
  mx = warp_max(mx);
  const bool flagged = (mx == -INFINITY);   // every K block fixed / dead (R7)

  if (!flagged) {
    double part = 0.0;
    for (int j = lane; j < T_n; j += 32) {
      const double e = (key[j] == -INFINITY) ? 0.0 : exp(key[j] - mx);
      key[j] = e;
      part += e;
    }
    const double total = warp_sum(part);
    // One 64-bit sort key per entry: the bits of P^ (>= 0, so integer order =
    // value order) with the low 11 mantissa bits replaced by 2047 - j.  Sorting
    // the keys descending orders (P^ desc, j asc) up to a 2^-42 relative
    // truncation of P^ -- far inside the 1e-6 near-threshold band of the
    // parity criterion; the cumulative sum below uses the truncated values.
    // Padding keys are 0 and sort last (a real entry has key >= 2047 - j > 0).
    uint64_t* ukey = reinterpret_cast<uint64_t*>(key);
    for (int j = lane; j < sortn; j += 32) {
      ukey[j] = (j < T_n)
                    ? ((static_cast<uint64_t>(__double_as_longlong(key[j] / total)) & ~0x7FFull) |
                       static_cast<uint64_t>(2047 - j))
                    : 0ull;
    }
    __syncwarp();
    switch (sortn) {
      case 32: sort_desc<32>(ukey, lane); break;
      case 64: sort_desc<64>(ukey, lane); break;
      case 128: sort_desc<128>(ukey, lane); break;
      case 256: sort_desc<256>(ukey, lane); break;
      case 512: sort_desc<512>(ukey, lane); break;
      case 1024: sort_desc<1024>(ukey, lane); break;
      default: sort_desc<2048>(ukey, lane); break;
    }
    // inclusive cumulative sum in rank order (contiguous chunk per lane):
    // pass 1 for the chunk totals and c_last, pass 2 for the decisions
    const int per = sortn / 32;
    const int k0 = lane * per, k1 = min(T_n, k0 + per);
    double loc = 0.0;
    for (int k = k0; k < k1; ++k) loc += __longlong_as_double(ukey[k] & ~0x7FFull);
    double incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double tv = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += tv;
    }
    // c_last, the last element of the cumulative sum (R4): the maximum of the
    // computed prefix sums (equal in exact arithmetic; keeps tau = 1 exact
    // when the parallel scan's rounding is non-monotone by an ulp)
    const double cmax = warp_max((k1 > k0) ? incl : 0.0);
    const double thr = tau * cmax;
    double cacc = incl - loc;
    for (int k = k0; k < k1; ++k) {
      const uint64_t kv = ukey[k];
      cacc += __longlong_as_double(kv & ~0x7FFull);
      flag[2047 - static_cast<int>(kv & 0x7FFull)] = (cacc <= thr || k == 0) ? 1 : 0;
    }
    __syncwarp();
  }

  // ---- forcing (Eq. 5), flagged rows, causal live AND + diagonal guard ----
  const int64_t row = qbase + my_row;
  const bool row_fix = q_sim[row] < theta;
  const int guard = (my_row * bq) / bk;
  uint8_t* mrow = mask ? mask + row * T_n : nullptr;
  int32_t* lrow = lut + row * T_n;
  int base = 0;
  for (int j0 = 0; j0 < T_n; j0 += 32) {
    const int j = j0 + lane;
    bool f = false;
    if (j < T_n) {
      f = flagged ? true : (flag[j] != 0);
      if (row_fix || k_sim[kbase + j] < theta) f = true;
      if (causal) {
        if (j * bk > last_q) f = false;
        if (j == guard) f = true;
      }
      if (mrow) mrow[j] = f ? 1 : 0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (f) lrow[base + __popc(bal & ((1u << lane) - 1u))] = j;
    base += __popc(bal);
  }
  if (lane == 0) cnt[row] = base;
}

}  // namespace

cudaError_t launch_predict(const sparge_shape& s, const double* q_pooled, const double* q_sim,
                           const double* k_pooled, const double* k_sim, float tau, float theta,
                           uint8_t* mask, int32_t* lut, int32_t* cnt, cudaStream_t stream) {
  const int T_m = (s.N + s.bq - 1) / s.bq;
  const int T_n = (s.N + s.bk - 1) / s.bk;
  int sortn = 32;
  while (sortn < T_n) sortn <<= 1;
  dim3 grid((T_m + kRows - 1) / kRows, s.Hq, s.B);
  if (s.d == 128) {
    const size_t smem = PredSmem<128>::bytes(sortn);
    cudaFuncSetAttribute(k_predict_topcdf<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    k_predict_topcdf<128><<<grid, kThreads, smem, stream>>>(
        q_pooled, q_sim, k_pooled, k_sim, s.Hq, s.Hkv, s.N, T_m, T_n, sortn, s.bq, s.bk,
        s.causal, static_cast<double>(tau), static_cast<double>(theta), mask, lut, cnt);
  } else {
    const size_t smem = PredSmem<64>::bytes(sortn);
    cudaFuncSetAttribute(k_predict_topcdf<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    k_predict_topcdf<64><<<grid, kThreads, smem, stream>>>(
        q_pooled, q_sim, k_pooled, k_sim, s.Hq, s.Hkv, s.N, T_m, T_n, sortn, s.bq, s.bk,
        s.causal, static_cast<double>(tau), static_cast<double>(theta), mask, lut, cnt);
  }
  return cudaGetLastError();
}

}  // namespace sparge
