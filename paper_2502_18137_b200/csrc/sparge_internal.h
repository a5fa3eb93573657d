// Internal declarations shared by the C-ABI front end and the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <utility>

#include "../../include/sparge.h"

namespace sparge {

// Programmatic dependent launch (PDL).  The hot-path kernels are launched
// with programmatic stream serialisation and begin with griddep_wait()
// (before their first global-memory access: the kernel before them in the
// stream has then completed and its writes are visible) followed by
// griddep_launch() (sm100.cuh), so the next kernel's launch and its CTAs'
// shared-memory / TMEM / barrier set-up overlap this kernel's tail instead of
// following it.  Stream order is unchanged: every kernel still waits for its
// predecessor before touching memory.  SPARGE_PDL (A/B runs) is a bit mask
// over the launch sites below (kPdl*); a cleared bit launches that kernel
// plainly (griddepcontrol.wait is then a no-op).
enum : unsigned {
  kPdlQuantQ = 1u, kPdlQuantK = 2u, kPdlPredict = 4u, kPdlVprep = 8u, kPdlOrder = 16u,
  kPdlAttn = 32u
};
// default: every site but the two quantiser launches -- with PDL on the K
// launch (its CTAs queued behind the persistent Q grid) the quantisation
// stage measured ~11 us slower on Flux / 8K, the other sites ~1 % faster
// per step (profiles/r02/r02_s11_pdl_mask.txt)
constexpr unsigned kPdlDefault = kPdlPredict | kPdlVprep | kPdlOrder | kPdlAttn;
bool pdl_enabled(unsigned site);
template <typename... KArgs, typename... Args>
cudaError_t launch_k(unsigned site, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled(site) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// 16-bit V^T staging layout: tile-major [B, Hkv, N_pad/64, d, 64] (each
// 64-key tile one contiguous 16 KB (d=128) block: contiguous writes in
// k_vprep, one TMA box per tile), or with -DSPARGE_VT_ROWMAJOR the
// row-major [B, Hkv, d, N_pad] of v5.  The FP8 staging stays row-major.
#ifdef SPARGE_VT_ROWMAJOR
constexpr bool kVtTiled = false;
#else
constexpr bool kVtTiled = true;
#endif

// mu: nullptr, or (K only) the smoothing mean [B, Hkv, d] of k_smooth.cu:
// the INT8 path quantises fl32(x - mu), the statistics use the raw x (R28, R14)
cudaError_t launch_quant(const sparge_shape& s, const void* x, sparge_strides st, int is_key,
                         const int32_t* perm, void* xq, float* delta, double* pooled,
                         double* sim, const float* mu, cudaStream_t stream);

// K smoothing mean (row f4, R28): fixed-order fp64 chunk sums -> fp32 mean
size_t smooth_partial_bytes(const sparge_shape& s);
cudaError_t launch_smooth_mean(const sparge_shape& s, const void* k, sparge_strides st,
                               double* part, float* mean, cudaStream_t stream);

cudaError_t launch_predict(const sparge_shape& s, const double* q_pooled, const double* q_sim,
                           const double* k_pooled, const double* k_sim, float tau, float theta,
                           uint8_t* mask, int32_t* lut, int32_t* cnt, void* workspace,
                           cudaStream_t stream);
size_t predict_workspace_bytes(const sparge_shape& s);

// early: launched right after k_order within one attention call -- the
// staging overlaps k_order and waits for it at its end (PDL, k_vprep.cu)
cudaError_t launch_vprep(const sparge_shape& s, const void* v, sparge_strides st,
                         const int32_t* perm, void* vt, int n_pad, bool early,
                         cudaStream_t stream);
// f4: per-channel amax of V (into amax_bits, zeroed here), then V^T in FP8
// E4M3 (x * fl32(448/amax_c)) and the dequant scales s_c = fl32(amax_c/448).
cudaError_t launch_vprep_fp8(const sparge_shape& s, const void* v, sparge_strides st,
                             const int32_t* perm, uint8_t* vt8, unsigned int* amax_bits,
                             float* v_scale, int n_pad, cudaStream_t stream);

cudaError_t launch_attn(const sparge_shape& s, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, const float* dq, const float* dk,
                        const int32_t* lut, const int32_t* cnt, float lambda,
                        const int32_t* perm, void* o, sparge_strides o_str,
                        uint64_t* counters, unsigned int* status, const float* v_scale,
                        const int32_t* order, uint8_t* mpv, cudaStream_t stream);

int attn_smem_bytes(int d, int qk16);

// Launch order of the attention work items (b * Hq + h) * T_m + i: the
// n_long items with the largest cnt first, then groups of per_group
// consecutive items, each by descending cnt (k_order.cu; scheduling only).
// meta: order_meta_ints(n, per_group) int32 of scratch.
size_t order_meta_ints(int n, int per_group);
cudaError_t launch_order(const int32_t* cnt, int n, int tn, int per_group, int n_long,
                         int32_t* order, int32_t* meta, cudaStream_t stream);

constexpr int kL1Blocks = (SPARGE_L1_OUT_DOUBLES - 2) / 2;
cudaError_t launch_l1_sums(const void* o, const void* o_ref, int f16, int64_t n, double* out,
                           cudaStream_t stream);

int hilbert_build(int T, int H, int W, int text_prefix, int32_t* perm, int32_t* inv);

}  // namespace sparge
