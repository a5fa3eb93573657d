// k_order -- launch order of the attention work items (scheduling only).
//
// Each (batch, q-head, query block i) is one k_sparse_attn CTA whose cost is
// proportional to cnt[i], the number of key blocks M_g keeps for that row
// (Alg. 1 l.9).  On video inputs cnt varies by an order of magnitude
// across query blocks, and on causal inputs it grows with i, so dispatching
// CTAs in index order leaves a long tail (measured, scripts/cta_timeline.py:
// 17 % idle SM time on Llama 32K, 34 % on Mochi).  The attention grid maps
// blockIdx.x -> order[blockIdx.x], and the hardware block scheduler
// dispatches in blockIdx order, so this list is the schedule:
//   1. the n_long items with the largest cnt, longest first (they bound the
//      tail, so they must start in the first wave);
//   2. the remaining items GROUP by GROUP -- a group is a run of consecutive
//      kv-heads whose K^ + V^T fit an L2 budget, so the CTAs in flight share
//      L2-resident key/value tiles (a fully global longest-first order mixes
//      all heads and re-reads K^/V^T from HBM: 128K sweep 156 -> 211 ms) --
//      each group longest first.
// k_order_head (1 CTA): histogram of cnt, the cut value, the long items'
// positions and each group's base offset; k_order_groups (one CTA per
// group): counting sort of the group's remaining items.  Items with equal
// cnt land in arbitrary order (results do not depend on it: every CTA is
// independent and writes its own rows).
#include <cstdint>

#include "sm100.cuh"
#include "sparge_internal.h"

namespace sparge {

namespace {

constexpr int kThreads = 1024;

// exclusive scan of h[0..tn] in DESCENDING index order, in place
// (h[b] := sum_{b' > b} h[b']); returns the total.  All threads call it.
__device__ int scan_desc(int* h, int tn, int* warp_sum) {
  const int tid = threadIdx.x;
  const int per = (tn + 1 + kThreads - 1) / kThreads;
  const int r0 = tid * per;
  int local = 0;
  for (int r = r0; r < min(r0 + per, tn + 1); ++r) local += h[tn - r];
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((tid & 31) >= o) incl += y;
  }
  if ((tid & 31) == 31) warp_sum[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    int w = warp_sum[tid];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (tid >= o) w += y;
    }
    warp_sum[tid] = w;   // inclusive over warps
  }
  __syncthreads();
  int off = incl - local + ((tid >> 5) > 0 ? warp_sum[(tid >> 5) - 1] : 0);
  for (int r = r0; r < min(r0 + per, tn + 1); ++r) {
    const int b = tn - r;
    const int c = h[b];
    h[b] = off;
    off += c;
  }
  const int total = warp_sum[31];
  __syncthreads();
  return total;
}

__device__ __forceinline__ int cnt_of(const int32_t* cnt, int x, int tn) {
  return min(max(__ldg(cnt + x), 0), tn);
}

// meta[0] = cut: items with cnt > cut are "long"; meta[1 + g] = base offset
// of group g's remaining items in `order`.
__global__ void __launch_bounds__(kThreads)
k_order_head(const int32_t* __restrict__ cnt, int n, int tn, int per_group, int n_groups,
             int n_long_max, int32_t* __restrict__ order, int32_t* __restrict__ meta) {
  extern __shared__ int sh[];
  int* h = sh;                    // tn + 1 bucket counts
  int* gcount = sh + tn + 1;      // n_groups short-item counts
  __shared__ int warp_sum[kThreads / 32];
  __shared__ int s_cut;
  const int tid = threadIdx.x;
  griddep_wait();      // PDL (sparge_internal.h)
  griddep_launch();
  for (int b = tid; b <= tn; b += kThreads) h[b] = 0;
  for (int g = tid; g < n_groups; g += kThreads) gcount[g] = 0;
  __syncthreads();
  for (int x = tid; x < n; x += kThreads) atomicAdd(&h[cnt_of(cnt, x, tn)], 1);
  __syncthreads();
  // cut: the long items are the whole top buckets b > cut holding at most
  // n_long_max items.  #items with cnt >= b is non-increasing in b, so
  // cut = (the smallest b with #(cnt >= b) <= n_long_max) - 1, found in
  // parallel from a descending exclusive scan of a copy of the histogram
  int* ge = gcount + n_groups;            // tn + 1 scan slots
  for (int b = tid; b <= tn; b += kThreads) ge[b] = h[b];
  if (tid == 0) s_cut = tn + 1;
  __syncthreads();
  scan_desc(ge, tn, warp_sum);           // ge[b] = #(cnt > b)
  for (int b = tid; b <= tn; b += kThreads)
    if (ge[b] + h[b] <= n_long_max) atomicMin(&s_cut, b);
  __syncthreads();
  const int cut = s_cut - 1;
  if (tid == 0) meta[0] = cut;
  for (int x = tid; x < n; x += kThreads)
    if (cnt_of(cnt, x, tn) <= cut) atomicAdd(&gcount[x / per_group], 1);
  for (int b = tid; b <= cut; b += kThreads) h[b] = 0;   // only long buckets stay
  __syncthreads();
  const int n_long = scan_desc(h, tn, warp_sum);
  for (int x = tid; x < n; x += kThreads) {
    const int c = cnt_of(cnt, x, tn);
    if (c > cut) order[atomicAdd(&h[c], 1)] = x;
  }
  if (tid == 0) {
    int base = n_long;
    for (int g = 0; g < n_groups; ++g) {
      meta[1 + g] = base;
      base += gcount[g];
    }
  }
}

__global__ void __launch_bounds__(kThreads)
k_order_groups(const int32_t* __restrict__ cnt, int n_all, int tn, int per_group,
               int32_t* __restrict__ order, const int32_t* __restrict__ meta) {
  extern __shared__ int h[];      // tn + 1 bucket counts, then write offsets
  __shared__ int warp_sum[kThreads / 32];
  const int tid = threadIdx.x;
  // PDL: trigger BEFORE waiting -- the next kernel (the V stage, which needs
  // nothing from k_order and waits for this grid at its end, or the
  // attention kernel, which waits at its start) may start right away;
  // k_order_head ran its wait before triggering this launch, so everything
  // before the attention call is complete by now
  griddep_launch();
  griddep_wait();
  const int cut = meta[0];
  const int base = static_cast<int>(blockIdx.x) * per_group;
  const int n = min(per_group, n_all - base);
  for (int b = tid; b <= tn; b += kThreads) h[b] = 0;
  __syncthreads();
  for (int x = tid; x < n; x += kThreads) {
    const int c = cnt_of(cnt, base + x, tn);
    if (c <= cut) atomicAdd(&h[c], 1);
  }
  __syncthreads();
  scan_desc(h, tn, warp_sum);
  int32_t* out = order + meta[1 + blockIdx.x];
  for (int x = tid; x < n; x += kThreads) {
    const int c = cnt_of(cnt, base + x, tn);
    if (c <= cut) out[atomicAdd(&h[c], 1)] = base + x;
  }
}

}  // namespace

size_t order_meta_ints(int n, int per_group) {
  per_group = max(1, min(per_group, n));
  return 1 + static_cast<size_t>((n + per_group - 1) / per_group);
}

cudaError_t launch_order(const int32_t* cnt, int n, int tn, int per_group, int n_long,
                         int32_t* order, int32_t* meta, cudaStream_t stream) {
  per_group = max(1, min(per_group, n));
  const int n_groups = (n + per_group - 1) / per_group;
  const int smem_head = (2 * (tn + 1) + n_groups) * static_cast<int>(sizeof(int));
  const int smem_groups = (tn + 1) * static_cast<int>(sizeof(int));
  if (smem_head > 200 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_order_head, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_head);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_order_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_groups);
  if (e != cudaSuccess) return e;
  e = launch_k(kPdlOrder, k_order_head, dim3(1), dim3(kThreads), smem_head, stream, cnt, n, tn, per_group,
               n_groups, n_long, order, meta);
  if (e != cudaSuccess) return e;
  return launch_k(kPdlOrder, k_order_groups, dim3(n_groups), dim3(kThreads), smem_groups, stream, cnt, n, tn,
                  per_group, order, static_cast<const int32_t*>(meta));
}

}  // namespace sparge
