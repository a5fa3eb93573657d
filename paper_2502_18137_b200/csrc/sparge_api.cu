// C-ABI front end of libsparge (include/sparge.h): argument validation,
// launch configuration, TMA descriptor encoding and workspace layout.  No
// compute happens here; every step of the path runs in the kernels.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "sparge_internal.h"

using namespace sparge;

namespace {

constexpr size_t kStatusBytes = 256;

bool shape_ok(const sparge_shape* s) {
  if (!s) return false;
  if (s->B < 1 || s->Hq < 1 || s->Hkv < 1 || s->N < 1) return false;
  if (s->Hq % s->Hkv) return false;
  if (s->d != 64 && s->d != 128) return false;
  if (s->bq != 128 || s->bk != 64 || s->cw != 4) return false;
  if (s->causal != 0 && s->causal != 1) return false;
  if (s->in_dtype != SPARGE_BF16 && s->in_dtype != SPARGE_FP16) return false;
  if (s->sim_mode != SPARGE_SIM_COSINE && s->sim_mode != SPARGE_SIM_LITERAL) return false;
  if (s->pv_dtype != SPARGE_PV_SAME_AS_INPUT && s->pv_dtype != SPARGE_PV_FP8_E4M3) return false;
  if (s->qk_dtype != SPARGE_QK_INT8 && s->qk_dtype != SPARGE_QK_INPUT) return false;
  return true;
}

bool strides_ok(sparge_strides st) {
  // 16-bit elements, 16-byte aligned rows
  return st.n > 0 && st.h >= 0 && st.b >= 0 && (st.n % 8) == 0 && (st.h % 8) == 0 &&
         (st.b % 8) == 0;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int n_pad_of(const sparge_shape* s) { return ((s->N + 63) / 64) * 64; }

// Workspace: [status 256 B][V^T: 16-bit, or e4m3 for pv_dtype FP8]
// (FP8 adds [amax bits u32 B*Hkv*d][dequant scales f32 B*Hkv*d], 256-aligned)
size_t round256(size_t x) { return (x + 255) / 256 * 256; }
size_t vt_bytes(const sparge_shape* s) {
  const size_t eb = s->pv_dtype == SPARGE_PV_FP8_E4M3 ? 1 : 2;
  return round256(static_cast<size_t>(s->B) * s->Hkv * s->d * n_pad_of(s) * eb);
}
int64_t n_items(const sparge_shape* s) {
  return static_cast<int64_t>(s->B) * s->Hq * ((s->N + 127) / 128);
}
// LPT launch order of the attention CTAs (k_order.cu)
// (the list, then the k_order scratch: cut value and per-group offsets)
size_t order_bytes(const sparge_shape* s) {
  return round256(static_cast<size_t>(n_items(s)) * 4) + round256(static_cast<size_t>(n_items(s) + 2) * 4);
}
// Scheduling knobs of k_order (debug overrides; defaults measured on B200):
// the L2 budget for one group's K^ + V^T and the number of longest items
// launched first.
int order_env(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
size_t chan_bytes(const sparge_shape* s) {
  return round256(static_cast<size_t>(s->B) * s->Hkv * s->d * 4);
}


// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

bool encode3d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1,
              uint64_t d2, uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0,
              uint32_t b1, CUtensorMapSwizzle sw) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

extern "C" {

const char* sparge_strerror(int status) {
  switch (status) {
    case SPARGE_OK: return "ok";
    case SPARGE_EINVAL: return "invalid argument";
    case SPARGE_EINTERNAL: return "internal invariant violated (a valid row ended with l = 0)";
    case SPARGE_ECUDA: return "CUDA error";
    case SPARGE_ENOTIMPL: return "option not implemented in this build";
    default: return "unknown status";
  }
}

int hilbert_permute(int T, int H, int W, int text_prefix, int32_t* perm_host,
                    int32_t* inv_host) {
  if (T < 1 || H < 1 || W < 1 || text_prefix < 0 || !perm_host || !inv_host)
    return SPARGE_EINVAL;
  const int64_t L = static_cast<int64_t>(text_prefix) + static_cast<int64_t>(T) * H * W;
  if (L > INT32_MAX) return SPARGE_EINVAL;
  return hilbert_build(T, H, W, text_prefix, perm_host, inv_host);
}

int sparge_quantize(const sparge_shape* shape, const void* x, sparge_strides x_str, int is_key,
                    const int32_t* perm, void* xq, float* delta, double* pooled, double* sim,
                    void* stream) {
  if (!shape_ok(shape) || !x || !xq || !delta || !pooled || !sim) return SPARGE_EINVAL;
  if (!strides_ok(x_str) || !aligned16(x) || !aligned16(xq)) return SPARGE_EINVAL;
  if (is_key != 0 && is_key != 1) return SPARGE_EINVAL;
  // a smoothed K goes through sparge_quantize_smooth_k (it needs the mean)
  if (shape->smooth_k && is_key) return SPARGE_EINVAL;
  cudaError_t e = launch_quant(*shape, x, x_str, is_key, perm, xq, delta, pooled, sim, nullptr,
                               static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPARGE_OK : SPARGE_ECUDA;
}

size_t sparge_smooth_k_workspace(const sparge_shape* shape) {
  if (!shape_ok(shape)) return 0;
  return smooth_partial_bytes(*shape);
}

int sparge_smooth_k_mean(const sparge_shape* shape, const void* k, sparge_strides k_str,
                         void* workspace, size_t ws_bytes, float* mean, void* stream) {
  if (!shape_ok(shape) || !k || !workspace || !mean) return SPARGE_EINVAL;
  if (!strides_ok(k_str) || (reinterpret_cast<uintptr_t>(workspace) & 7u)) return SPARGE_EINVAL;
  if (ws_bytes < smooth_partial_bytes(*shape)) return SPARGE_EINVAL;
  cudaError_t e = launch_smooth_mean(*shape, k, k_str, static_cast<double*>(workspace), mean,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPARGE_OK : SPARGE_ECUDA;
}

int sparge_quantize_smooth_k(const sparge_shape* shape, const void* k, sparge_strides k_str,
                             const int32_t* perm, const float* mean, void* kq, float* delta,
                             double* pooled, double* sim, void* stream) {
  if (!shape_ok(shape) || !k || !mean || !kq || !delta || !pooled || !sim) return SPARGE_EINVAL;
  if (!strides_ok(k_str) || !aligned16(k) || !aligned16(kq)) return SPARGE_EINVAL;
  if (shape->qk_dtype != SPARGE_QK_INT8) return SPARGE_ENOTIMPL;   // nothing to smooth
  cudaError_t e = launch_quant(*shape, k, k_str, 1, perm, kq, delta, pooled, sim, mean,
                               static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPARGE_OK : SPARGE_ECUDA;
}

size_t sparge_predict_workspace(const sparge_shape* shape) {
  if (!shape_ok(shape)) return 0;
  return predict_workspace_bytes(*shape);
}

int sparge_predict_mask(const sparge_shape* shape, const double* q_pooled, const double* q_sim,
                        const double* k_pooled, const double* k_sim, float tau, float theta,
                        uint8_t* mask, int32_t* lut, int32_t* cnt, void* workspace,
                        size_t ws_bytes, void* stream) {
  if (!shape_ok(shape) || !q_pooled || !q_sim || !k_pooled || !k_sim || !lut || !cnt)
    return SPARGE_EINVAL;
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255u) != 0 ||
      ws_bytes < predict_workspace_bytes(*shape))
    return SPARGE_EINVAL;
  if (!(tau > 0.f && tau <= 1.f)) return SPARGE_EINVAL;
  if (!(theta >= -1.f && theta <= 1.f)) return SPARGE_EINVAL;
  const int T_n = (shape->N + shape->bk - 1) / shape->bk;
  if (T_n > SPARGE_MAX_TN) return SPARGE_EINVAL;   // one compressed-map row per warp in smem
  cudaError_t e = launch_predict(*shape, q_pooled, q_sim, k_pooled, k_sim, tau, theta, mask, lut,
                                 cnt, workspace, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPARGE_OK : SPARGE_ECUDA;
}

size_t sparge_attn_workspace(const sparge_shape* shape) {
  if (!shape_ok(shape)) return 0;
  const size_t extra = shape->pv_dtype == SPARGE_PV_FP8_E4M3 ? 2 * chan_bytes(shape) : 0;
  return kStatusBytes + vt_bytes(shape) + extra + order_bytes(shape);
}

int sparge_attn_fwd(const sparge_shape* shape, const void* qq, const float* dq,
                    const void* kq, const float* dk, const void* v, sparge_strides v_str,
                    const int32_t* lut, const int32_t* cnt, float lambda, const int32_t* perm,
                    void* o, sparge_strides o_str, uint64_t* counters, void* workspace,
                    size_t ws_bytes, void* stream) {
  return sparge_attn_fwd_ex(shape, qq, dq, kq, dk, v, v_str, lut, cnt, lambda, perm, o, o_str,
                            counters, workspace, ws_bytes, stream, 0u);
}

namespace {
int attn_fwd_impl(const sparge_shape* shape, const void* qq, const float* dq,
                  const void* kq, const float* dk, const void* v, sparge_strides v_str,
                  const int32_t* lut, const int32_t* cnt, float lambda,
                  const int32_t* perm, void* o, sparge_strides o_str, uint64_t* counters,
                  void* workspace, size_t ws_bytes, void* stream, unsigned flags,
                  uint8_t* mpv) {
  if (flags > 2u) return SPARGE_EINVAL;
  if (!shape_ok(shape) || !qq || !dq || !kq || !dk || !v || !lut || !cnt || !o || !workspace)
    return SPARGE_EINVAL;
  if (!strides_ok(v_str) || !strides_ok(o_str) || !aligned16(v) || !aligned16(o))
    return SPARGE_EINVAL;
  if (!aligned16(qq) || !aligned16(kq)) return SPARGE_EINVAL;
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0) return SPARGE_EINVAL;
  if (ws_bytes < sparge_attn_workspace(shape)) return SPARGE_EINVAL;
  if (!(lambda < 0.f)) return SPARGE_EINVAL;   // lambda < 0 or -inf (§3.6)
  // causal masking is defined on token positions (R8); with a permutation the
  // kernel would apply it to permuted positions, which is not causal attention
  if (shape->causal && perm) return SPARGE_EINVAL;
  const bool pv8 = shape->pv_dtype == SPARGE_PV_FP8_E4M3;
  if (pv8 && shape->qk_dtype != SPARGE_QK_INT8) return SPARGE_ENOTIMPL;   // FP8 PV with INT8 QK only
  if (shape->smooth_k && shape->qk_dtype != SPARGE_QK_INT8) return SPARGE_ENOTIMPL;

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const sparge_shape& s = *shape;
  const int n_pad = n_pad_of(shape);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  unsigned int* status = reinterpret_cast<unsigned int*>(ws);
  void* vt = ws + kStatusBytes;
  unsigned int* amax_bits = reinterpret_cast<unsigned int*>(ws + kStatusBytes + vt_bytes(shape));
  float* v_scale = reinterpret_cast<float*>(ws + kStatusBytes + vt_bytes(shape) + chan_bytes(shape));
  int32_t* order = reinterpret_cast<int32_t*>(
      ws + kStatusBytes + vt_bytes(shape) + (pv8 ? 2 * chan_bytes(shape) : 0));

  cudaError_t e = cudaSuccess;
  // the whole call (flags 0, 16-bit V): k_order first, then the V stage,
  // which overlaps it (PDL, k_vprep.cu), then the attention kernel
  const bool vprep_after_order = flags == 0u && !pv8;
  if (!(flags & SPARGE_ATTN_SKIP_VPREP) && !vprep_after_order) {
    e = pv8 ? launch_vprep_fp8(s, v, v_str, perm, static_cast<uint8_t*>(vt), amax_bits, v_scale,
                               n_pad, st)
            : launch_vprep(s, v, v_str, perm, vt, n_pad, false, st);
    if (e != cudaSuccess) return SPARGE_ECUDA;
  }
  if (flags & SPARGE_ATTN_VPREP_ONLY) return SPARGE_OK;

  // Q and K operand maps.  INT8: one box of d bytes per row (SWIZZLE_128B at
  // d=128, 64B at d=64).  16-bit (qk_dtype INPUT): boxes of 64 elements =
  // 128 B per row, loaded d/64 times (one SWIZZLE_128B K-atom each).
  const bool qk16 = s.qk_dtype == SPARGE_QK_INPUT;
  const CUtensorMapDataType dt16 =
      s.in_dtype == SPARGE_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const CUtensorMapSwizzle sw_qk =
      (qk16 || s.d == 128) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  const CUtensorMapDataType dt_qk = qk16 ? dt16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const uint64_t eb = qk16 ? 2 : 1;
  const uint32_t box0 = qk16 ? 64u : static_cast<uint32_t>(s.d);
  CUtensorMap mq, mk, mv;
  const uint64_t d = static_cast<uint64_t>(s.d);
  const uint64_t N = static_cast<uint64_t>(s.N);
  if (!encode3d(&mq, dt_qk, qq, d, N, static_cast<uint64_t>(s.B) * s.Hq, d * eb, d * N * eb,
                box0, 128, sw_qk) ||
      !encode3d(&mk, dt_qk, kq, d, N, static_cast<uint64_t>(s.B) * s.Hkv, d * eb, d * N * eb,
                box0, 64, sw_qk) ||
      !(pv8 ? encode3d(&mv, CU_TENSOR_MAP_DATA_TYPE_UINT8, vt, static_cast<uint64_t>(n_pad), d,
                       static_cast<uint64_t>(s.B) * s.Hkv, static_cast<uint64_t>(n_pad), d * n_pad,
                       64, s.d, CU_TENSOR_MAP_SWIZZLE_64B)
            : (kVtTiled ? encode3d(&mv, dt16, vt, 64, d * static_cast<uint64_t>(n_pad / 64),
                                   static_cast<uint64_t>(s.B) * s.Hkv, 128, d * n_pad * 2, 64, s.d,
                                   CU_TENSOR_MAP_SWIZZLE_128B)
                        : encode3d(&mv, dt16, vt, static_cast<uint64_t>(n_pad), d,
                                   static_cast<uint64_t>(s.B) * s.Hkv, static_cast<uint64_t>(n_pad) * 2,
                                   d * n_pad * 2, 64, s.d, CU_TENSOR_MAP_SWIZZLE_128B))))
    return SPARGE_ECUDA;

  // launch order: the longest items first, then groups of kv-heads whose
  // K^ + V^T fit the L2 budget, each longest first (k_order.cu).  With the
  // Hilbert permutation the kept blocks are local, so a CTA touches a small
  // part of its head's K^/V^T and larger groups fit: 64 MB; in token order
  // 48 MB (profiles/r01s6_quant_ab.txt).
  static const int budget_perm_mb = order_env("SPARGE_ORDER_BUDGET_MB", 64);
  static const int budget_plain_mb = order_env("SPARGE_ORDER_BUDGET_MB", 48);
  const int budget_mb = perm ? budget_perm_mb : budget_plain_mb;
  static const int n_long = order_env("SPARGE_ORDER_LONG", 296);
  const int64_t kv_head_bytes = static_cast<int64_t>(n_pad) * s.d * ((qk16 ? 2 : 1) + (pv8 ? 1 : 2));
  // groups of equal size: ceil(kv-heads / groups) kv-heads each
  const int64_t kv_heads = static_cast<int64_t>(s.B) * s.Hkv;
  const int64_t kv_fit = std::max<int64_t>(1, (static_cast<int64_t>(budget_mb) << 20) / kv_head_bytes);
  const int64_t n_groups = (kv_heads + kv_fit - 1) / kv_fit;
  const int64_t kv_per_group = (kv_heads + n_groups - 1) / n_groups;
  const int64_t per_group = kv_per_group * (s.Hq / s.Hkv) * ((s.N + 127) / 128);
  const int n_it = static_cast<int>(n_items(shape));
  e = launch_order(cnt, n_it, (s.N + 63) / 64, static_cast<int>(std::min<int64_t>(per_group, n_it)),
                   n_long, order, order + round256(static_cast<size_t>(n_it) * 4) / 4, st);
  if (e != cudaSuccess) return SPARGE_ECUDA;
  if (vprep_after_order) {
    e = launch_vprep(s, v, v_str, perm, vt, n_pad, true, st);
    if (e != cudaSuccess) return SPARGE_ECUDA;
  }
  e = launch_attn(s, mq, mk, mv, dq, dk, lut, cnt, lambda, perm, o, o_str, counters, status,
                  pv8 ? v_scale : nullptr, order, mpv, st);
  return e == cudaSuccess ? SPARGE_OK : SPARGE_ECUDA;
}
}  // namespace

int sparge_attn_fwd_ex(const sparge_shape* shape, const void* qq, const float* dq,
                       const void* kq, const float* dk, const void* v, sparge_strides v_str,
                       const int32_t* lut, const int32_t* cnt, float lambda,
                       const int32_t* perm, void* o, sparge_strides o_str, uint64_t* counters,
                       void* workspace, size_t ws_bytes, void* stream, unsigned flags) {
  return attn_fwd_impl(shape, qq, dq, kq, dk, v, v_str, lut, cnt, lambda, perm, o, o_str,
                       counters, workspace, ws_bytes, stream, flags, nullptr);
}

int sparge_attn_fwd_mpv(const sparge_shape* shape, const void* qq, const float* dq,
                        const void* kq, const float* dk, const void* v, sparge_strides v_str,
                        const int32_t* lut, const int32_t* cnt, float lambda,
                        const int32_t* perm, void* o, sparge_strides o_str, uint64_t* counters,
                        void* workspace, size_t ws_bytes, void* stream, uint8_t* mpv) {
  if (!mpv) return SPARGE_EINVAL;
  return attn_fwd_impl(shape, qq, dq, kq, dk, v, v_str, lut, cnt, lambda, perm, o, o_str,
                       counters, workspace, ws_bytes, stream, 0u, mpv);
}

int sparge_l1_sums(const void* o, const void* o_ref, int dtype, int64_t n, double* out,
                   void* stream) {
  if (!o || !o_ref || !out || n < 1) return SPARGE_EINVAL;
  if (dtype != SPARGE_BF16 && dtype != SPARGE_FP16) return SPARGE_EINVAL;
  if (!aligned16(o) || !aligned16(o_ref) || (reinterpret_cast<uintptr_t>(out) & 7u)) return SPARGE_EINVAL;
  cudaError_t e = launch_l1_sums(o, o_ref, dtype == SPARGE_FP16, n, out,
                                 static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPARGE_OK : SPARGE_ECUDA;
}

int sparge_attn_status(void* workspace, void* stream) {
  if (!workspace) return SPARGE_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned int h = 0;
  if (cudaMemcpyAsync(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return SPARGE_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return SPARGE_ECUDA;
  if (cudaMemsetAsync(workspace, 0, sizeof(h), st) != cudaSuccess) return SPARGE_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return SPARGE_ECUDA;
  return h ? SPARGE_EINTERNAL : SPARGE_OK;
}

}  // extern "C"

namespace sparge {
// PDL on the hot-path launches (sparge_internal.h); SPARGE_PDL=0 disables
bool pdl_enabled(unsigned site) {
  static const unsigned v = [] {
    const char* e = std::getenv("SPARGE_PDL");
    return e ? static_cast<unsigned>(std::strtoul(e, nullptr, 0)) : kPdlDefault;
  }();
  return (v & site) != 0u;
}
}  // namespace sparge
