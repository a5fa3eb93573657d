// k_sparse_attn -- step a3 of the hot path.
//
// Stage 2 of Algorithm 1: for one (q-head, query block i) the
// CTA walks the kept key blocks j of M_g (the LUT from k_predict_topcdf, in
// ascending j) and runs the online-softmax recurrence of Eq. 1:
//   S   = (Q^_i K^_j^T) dq_i dk_j / sqrt(d)          line 12, R3
//   m_local = rowmax S; m_new = max(m, m_local); P~ = exp(S - m_new)
//   l   = e^{m - m_new} l + rowsum P~                 line 13
//   per warp group w (rows 32w..32w+31, c_w = 4, R10):
//     if max(m_local - m_new) > lambda:               line 15, R5
//        O[I_w] = e^{m - m_new} O[I_w] + P~[I_w] V_j  line 16
//   O_i = O / l                                       line 19
//
// sm_100a design (v4, "pair" iterations).  One CTA = 4 softmax warps + 1 TMA
// producer warp + 1 MMA warp, two CTAs per SM, 256 TMEM columns per CTA:
// S (128 columns: two 64-key tiles side by side) | O (d columns).
// The kept tiles are processed two at a time (a PAIR, tiles 2p and 2p+1 of
// the LUT), so every synchronisation round trip between the softmax warps
// and the MMA warp carries two tiles of tensor work (ablations, profiles/
// r01s2/attn_ablations.md: with one 64-key tile per round trip the MMA chain
// alone left the tensor pipe 36 % idle).  Alg. 1 stays tile-sequential: the
// two tiles keep their own row maxima, gate votes and P~V MMAs.
//   producer  Q^ once, then K^_t (ring of KST slots; the two tiles of a pair
//             land in adjacent slots, i.e. one 128-row K-major operand) and
//             V^T_t (ring of VST slots) for every kept tile.
//   MMA       one thread.  Pair p: S := 1.5*2^23 (bias MMA, INT8 only), then
//             kind::i8 Q^ K^^T for both tiles at once (N = 128) -> S; after
//             the softmax hands P~ back (p_full): kind::f16 P~ V per tile
//             with P~ read from TMEM (TS form), skipped when all four gate
//             groups vote to skip that tile.  QK(p+1) is issued right after
//             the P~V MMAs of pair p (in-order tensor pipe: P~ aliases S).
//   softmax   thread r owns row r == TMEM lane r; warp w is the gate group
//             I_w.  Per pair: both tiles' row maxima (integer domain), the
//             two gate votes in Alg. 1 order, one reference max for the pair
//             (lazy, R22), exp2 with one FFMA per pair of elements (R23),
//             P~ (16-bit or E4M3) written over the first columns of its own
//             tile in S, one arrive.
#include <cuda.h>
#include <cstdint>
#include <climits>
#include <type_traits>

#include "sm100.cuh"
#include "sparge_internal.h"

// SPARGE_CTA_TIMING (debug builds only): per-CTA globaltimer records
// {entry, softmax loop start, loop end, exit, smid, n_tiles} in a device
// array read back by sparge_debug_cta_records (scripts/cta_timeline.py).
#ifdef SPARGE_CTA_TIMING
__device__ unsigned long long g_cta_rec[1 << 16][6];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CTA_REC(slot, val)                                                               \
  do {                                                                                   \
    const unsigned cid = blockIdx.y * gridDim.x + blockIdx.x;                           \
    if (cid < (1u << 16)) g_cta_rec[cid][slot] = (val);                                  \
  } while (0)
#else
#define CTA_REC(slot, val) do { } while (0)
#endif

#ifdef SPARGE_PHASE_TIMING
#define PT_MARK(k) do { const long long _c = clock64(); ph[k] += _c - ph_last; ph_last = _c; } while (0)
#else
#define PT_MARK(k) do { } while (0)
#endif

namespace sparge {

namespace {

constexpr int BQ = 128;
constexpr int BK = 64;
constexpr int NSOFT = 4;      // softmax warps per group: one per TMEM lane quadrant
constexpr int NG = 2;         // query-tile groups per CTA (one CTA per SM)
constexpr int THREADS = (NG * NSOFT + NG + 1) * 32;
constexpr int WARP_LOAD0 = NG * NSOFT;       // producer of group g: WARP_LOAD0 + g
constexpr int WARP_MMA = WARP_LOAD0 + NG;    // one MMA issuer for both groups
#ifndef SPARGE_RESCALE_THR
#define SPARGE_RESCALE_THR 8
#endif
// lazy-rescale threshold (R22), log2 units: P~ <= 2^thr, which fp16 P~ must
// hold (max 65504 < 2^16)
constexpr float kRescaleThreshold = static_cast<float>(SPARGE_RESCALE_THR);
constexpr float kRescaleThresholdF16 = SPARGE_RESCALE_THR < 15 ? SPARGE_RESCALE_THR : 15.0f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMagic = 0x4B400000;          // bits of 1.5 * 2^23
constexpr float kMagicF = 12582912.0f;

#ifndef SPARGE_POLY_EVERY
#define SPARGE_POLY_EVERY 8
#endif
constexpr int kPolyEvery = SPARGE_POLY_EVERY;   // one pair in kPolyEvery uses exp2_poly2 (0: none)

// SPARGE_BIAS_MMA (INT8 QK): before the kind::i8 MMAs of a pair, one
// kind::f16 MMA (M128 N<=128 K16, constant operands 1.0 x 1.5*2^19 summed
// over K = 16) writes the fp32 value 1.5*2^23 into every S accumulator; the
// i8 MMAs then accumulate onto those bits as int32, so S leaves the tensor
// core as bits(1.5*2^23 + acc) -- the exact fp32 value 1.5*2^23 + acc (R23)
// without a per-element integer add in the softmax warps.
#ifndef SPARGE_BIAS_MMA
#define SPARGE_BIAS_MMA 1
#endif
constexpr bool kBiasMma = SPARGE_BIAS_MMA != 0;
constexpr uint16_t kBf16One = 0x3F80;        // bf16 1.0
constexpr uint16_t kBf16MagicPart = 0x4940;  // bf16 786432 = 1.5*2^19 (x 16 = 1.5*2^23)

// Shared-memory plan.  QK16 = the unquantised f1 kernel (16-bit Q, K tiles
// stored as d/64 SWIZZLE_128B K-atoms of 128-B rows); with d = 128 its rings
// shrink to 2 + 2 slots so that two CTAs still fit on an SM.  KST is even:
// the two tiles of a pair occupy slots (2q, 2q+1), adjacent in memory.
template <int D, bool QK16, bool PV8 = false>
struct Smem {
  static constexpr int EB = QK16 ? 2 : 1;       // bytes per Q/K element
  static constexpr int KST = (QK16 && D == 128) ? 2 : 4;
  static constexpr int VST = (QK16 && D == 128) ? 2 : (PV8 ? 4 : 3);
  static constexpr int Q_BYTES = BQ * D * EB;
  static constexpr int K_BYTES = BK * D * EB;
  static constexpr int V_BYTES = D * BK * (PV8 ? 1 : 2);    // V^T tile, 16-bit or e4m3
  static constexpr bool BIAS = kBiasMma && !QK16;
  // constant bias-MMA operands: A 128 x 16 bf16 ones, B 128 x 16 bf16 1.5*2^19
  static constexpr int CA_BYTES = BIAS ? BQ * 16 * 2 : 0;
  static constexpr int CB_BYTES = BIAS ? 2 * BK * 16 * 2 : 0;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * K_BYTES;
  static constexpr int OFF_CA = OFF_V + VST * V_BYTES;
  static constexpr int OFF_CB = OFF_CA + CA_BYTES;
  static constexpr int OFF_BAR = OFF_CB + CB_BYTES;
  static constexpr int N_BARS = 1 + 2 * KST + 2 * VST + 3;
  static constexpr int OFF_MISC = OFF_BAR + N_BARS * 8;    // [0] TMEM base, [1..8] pv flags
  static constexpr int TOTAL = OFF_MISC + 64;
  static constexpr int BYTES = (TOTAL + 1023) / 1024 * 1024;
  // INT8: one K-atom of D bytes per row (128 -> SW128, 64 -> SW64); 16-bit:
  // 128-B atoms, the second (d = 128) BQ*128 / BK*128 bytes after the first
  static constexpr int ROW_BYTES_QK = QK16 ? 128 : D;
  static constexpr int Q_ATOM = BQ * 128, K_ATOM = BK * 128;
  static_assert(KST % 2 == 0, "pairs need adjacent K slots");
  static_assert(NG * BYTES + 1024 <= 227 * 1024, "both groups must fit one CTA");
};

struct AttnParams {
  const float* dq;
  const float* dk;
  const int32_t* lut;
  const int32_t* cnt;
  const int32_t* perm;
  uint16_t* o;
  int64_t o_sb, o_sh, o_sn;
  unsigned long long* counters;
  unsigned int* status;
  const float* v_scale;   // PV8: per-(b, hkv, channel) dequant scale s_c [B*Hkv, D]
  float lam2;         // lambda * log2(e)
  float scale_log2;   // log2(e) / sqrt(d)
  int N, T_m, T_n, Hq, Hkv, group;
  unsigned long long* phase_clk;   // debug: per-phase cycle sums (SPARGE_PHASE_TIMING)
};

// ---- packed f32x2 helpers (FADD2 / FFMA2 on sm_100a) ----
__device__ __forceinline__ uint64_t pk(float lo, float hi) {
  return (static_cast<uint64_t>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }

// 2^x for a pair of floats on the FMA pipe (MUFU offload): x clamped to
// >= -125, j = rint(x) via the 1.5*2^23 rounding trick, f = x - j in
// [-0.5, 0.5], 2^f by a degree-3 polynomial (max relative error 1.0e-4, below
// the 2^-9 rounding of the bf16 P~ it feeds), 2^j added into the exponent.
constexpr float kP1 = 0.69328290224f, kP2 = 0.24221096933f, kP3 = 0.05500892922f;
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  const uint64_t xc = pk(fmaxf(lo_f(x2), -125.f), fmaxf(hi_f(x2), -125.f));
  const uint64_t r = add2(xc, pk(kMagicF, kMagicF));
  const uint64_t jf = add2(r, pk(-kMagicF, -kMagicF));
  const uint64_t f = fma2(jf, pk(-1.f, -1.f), xc);
  uint64_t q = fma2(pk(kP3, kP3), f, pk(kP2, kP2));
  q = fma2(q, f, pk(kP1, kP1));
  q = fma2(q, f, pk(1.f, 1.f));
  const uint32_t e0 = static_cast<uint32_t>(q) + (static_cast<uint32_t>(r) << 23);
  const uint32_t e1 = static_cast<uint32_t>(q >> 32) + (static_cast<uint32_t>(r >> 32) << 23);
  return (static_cast<uint64_t>(e1) << 32) | e0;
}

__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <bool F16>
__device__ __forceinline__ uint32_t pack16(float lo, float hi) {
  return F16 ? pack_f16x2(lo, hi) : pack_bf16x2(lo, hi);
}
// two fp32 -> FP8 E4M3 (round to nearest even, saturate to +-448), lo in the
// low byte
__device__ __forceinline__ uint32_t pack_e4m3x2(float lo, float hi) {
  unsigned short r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void mma_f8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// P~ = exp2(acc * c - m_ref) for the 64 columns of a row, packed to 16-bit,
// and their sum.  bits(acc + 0x4B400000) are the fp32 value M + acc,
// M = 1.5*2^23, exactly for |acc| < 2^22 (|acc| <= 127^2 d); one FFMA gives
//   (M + acc) c - (M c + m_ref) = acc c - m_ref + e,
// e = the fp32 rounding of the per-tile bias M c + m_ref: a constant shift of
// the whole tile's exponent of at most 0.75 c, i.e. under one unit of the
// integer accumulator, far below the INT8 quantisation error in acc (R23).
// MASKED: INT_MIN entries and rows without a finite reference give 0.
// QK16: a holds fp32 S accumulators (no magic constant); masked entries -inf.
// PV8: P~ packed to FP8 E4M3, four per word (pw[16]).
// S encodings (SBits): the int32 accumulator (kAdd = magic, masked INT_MIN),
// the bias-MMA fp32 bits of 1.5*2^23 + acc (kAdd = 0, masked 0), or fp32 S
// of the unquantised kernel (kAdd = 0, masked -inf).
template <bool QK16, bool BIAS>
struct SBits {
  static constexpr int kAdd = (QK16 || BIAS) ? 0 : kMagic;
  static constexpr int kMasked = QK16 ? static_cast<int>(0xFF800000u) : (BIAS ? 0 : INT_MIN);
};

template <bool MASKED, bool F16, bool QK16 = false, bool PV8 = false, bool BIAS = false>
__device__ __forceinline__ void exps64(const int32_t* a, float c, float m_ref, uint32_t* pw,
                                       float& sum) {
  constexpr int kAdd = SBits<QK16, BIAS>::kAdd;
  constexpr int kMaskedBits = SBits<QK16, BIAS>::kMasked;
  const uint64_t c2 = pk(c, c);
  const float nbias = QK16 ? -m_ref : fmaf(-kMagicF, c, -m_ref);
  const uint64_t nb2 = pk(nbias, nbias);
  const bool row_live = m_ref > -INFINITY;
  uint64_t rs2[2] = {0ull, 0ull};
#pragma unroll
  for (int k = 0; k < BK; k += 2) {
    const uint64_t x2 = fma2(pk(__int_as_float(a[k] + kAdd), __int_as_float(a[k + 1] + kAdd)),
                             c2, nb2);
    uint64_t e2;
    if (!MASKED && kPolyEvery > 0 && ((k >> 1) % (kPolyEvery > 0 ? kPolyEvery : 1)) == kPolyEvery - 1)
      e2 = exp2_poly2(x2);
    else
      e2 = pk(ex2_approx(lo_f(x2)), ex2_approx(hi_f(x2)));
    if (MASKED) {
      const float e0 = (a[k] == kMaskedBits || !row_live) ? 0.f : lo_f(e2);
      const float e1 = (a[k + 1] == kMaskedBits || !row_live) ? 0.f : hi_f(e2);
      e2 = pk(e0, e1);
    }
    rs2[(k >> 1) & 1] = add2(rs2[(k >> 1) & 1], e2);
    if (PV8) {
      const uint32_t h = pack_e4m3x2(lo_f(e2), hi_f(e2));
      if ((k & 2) == 0) pw[k >> 2] = h;
      else pw[k >> 2] |= h << 16;
    } else {
      pw[k >> 1] = pack16<F16>(lo_f(e2), hi_f(e2));
    }
  }
  const uint64_t rs = add2(rs2[0], rs2[1]);
  sum = lo_f(rs) + hi_f(rs);
}

template <int D, bool CAUSAL, bool F16, bool QK16, bool PV8>
__global__ void __launch_bounds__(THREADS, 1)
k_sparse_attn(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using L = Smem<D, QK16, PV8>;
#ifdef SPARGE_CTA_TIMING
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    CTA_REC(0, gtimer());
    CTA_REC(4, smid);
  }
#endif
  // FP8 P~ (f4) is rounded relative to the reference max: rescale eagerly so
  // the reference is the true running max (R27), as the oracle's P~ = e^{S-m}
  constexpr float kRefThreshold = PV8 ? 0.0f : (F16 ? kRescaleThresholdF16 : kRescaleThreshold);
  constexpr int KST = L::KST, VST = L::VST;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = __shfl_sync(0xffffffffu, warp_id(), 0), lane = lane_id();
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);   // group 0's
  const int bhq = blockIdx.y;
  const int b = bhq / p.Hq, hq = bhq % p.Hq;
  const int bkv = b * p.Hkv + hq / p.group;
  // Group gg handles query tile u = 2 blockIdx.x + gg (causal: longest rows
  // first); u >= T_m is an empty group.
  auto tile_of = [&](int gg, int& i_out) -> int {
    const int u = static_cast<int>(blockIdx.x) * NG + gg;
    if (u >= p.T_m) { i_out = p.T_m - 1; return 0; }
    i_out = CAUSAL ? (p.T_m - 1 - u) : u;
    return p.cnt[static_cast<int64_t>(bhq) * p.T_m + i_out];
  };
  // group of this warp (softmax warps 4g..4g+3, producer WARP_LOAD0 + g; the
  // MMA warp serves both).  `warp` comes from a shuffle, so g and every
  // address derived from it are warp-uniform.
  const int g = warp < WARP_LOAD0 ? (warp >> 2) : (warp < WARP_MMA ? warp - WARP_LOAD0 : 0);
  int i = 0;
  const int n_tiles = tile_of(g, i);
  const int64_t row_id = static_cast<int64_t>(bhq) * p.T_m + i;
  const int n_pairs = (n_tiles + 1) >> 1;
  const int32_t* lut_row = p.lut + row_id * p.T_n;

  auto gsm = [&](int gg) { return smem + gg * L::BYTES; };
  unsigned char* sg = gsm(g);
  int8_t* sQ = reinterpret_cast<int8_t*>(sg + L::OFF_Q);
  int8_t* sK = reinterpret_cast<int8_t*>(sg + L::OFF_K);
  unsigned char* sV = sg + L::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sg + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + KST;
  uint64_t* v_full = k_empty + KST;
  uint64_t* v_empty = v_full + VST;
  uint64_t* s_full = v_empty + VST;   // QK of the pair done
  uint64_t* p_full = s_full + 1;      // P~ of the pair in TMEM (4 softmax warps)
  uint64_t* o_done = p_full + 1;      // last P~V done (epilogue)
  uint32_t* pv_flag = reinterpret_cast<uint32_t*>(sg + L::OFF_MISC) + 1;   // [2 tiles][4 warps]

  if (threadIdx.x == 0) {
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) {
      uint64_t* bg = reinterpret_cast<uint64_t*>(gsm(gg) + L::OFF_BAR);
      mbar_init(bg, 1);
      for (int s = 0; s < KST; ++s) { mbar_init(bg + 1 + s, 1); mbar_init(bg + 1 + KST + s, 1); }
      for (int s = 0; s < VST; ++s) { mbar_init(bg + 1 + 2 * KST + s, 1); mbar_init(bg + 1 + 2 * KST + VST + s, 1); }
      mbar_init(bg + 1 + 2 * KST + 2 * VST, 1);          // s_full
      mbar_init(bg + 2 + 2 * KST + 2 * VST, NSOFT);      // p_full
      mbar_init(bg + 3 + 2 * KST + 2 * VST, 1);          // o_done
    }
    fence_mbar_init();
  }
  if constexpr (L::BIAS) {
    // constant operands of the bias MMA (every element equal, so the core
    // matrix layout of the descriptor is immaterial)
    constexpr uint32_t kOnes = kBf16One | (static_cast<uint32_t>(kBf16One) << 16);
    constexpr uint32_t kParts = kBf16MagicPart | (static_cast<uint32_t>(kBf16MagicPart) << 16);
#pragma unroll
    for (int gg = 0; gg < NG; ++gg) {
      uint32_t* cw = reinterpret_cast<uint32_t*>(gsm(gg) + L::OFF_CA);
      for (int x = threadIdx.x; x < (L::CA_BYTES + L::CB_BYTES) / 4; x += blockDim.x)
        cw[x] = x < L::CA_BYTES / 4 ? kOnes : kParts;
    }
    fence_proxy_async_smem();   // generic-proxy writes -> visible to the tensor core
  }
  if (warp == WARP_MMA) tmem_alloc<256 * NG>(tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const uint32_t tS = tmem_base + g * 256, tO = tS + 2 * BK;

  if (warp >= WARP_LOAD0 && warp < WARP_MMA) {
    // ============================ TMA producer ============================
    if (lane == 0 && n_tiles > 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_arrive_expect_tx(q_full, L::Q_BYTES);
      if (QK16) {
#pragma unroll
        for (int h = 0; h < D / 64; ++h) tma_load_3d(sQ + h * L::Q_ATOM, &tmQ, q_full, h * 64, i * BQ, bhq);
      } else {
        tma_load_3d(sQ, &tmQ, q_full, 0, i * BQ, bhq);
      }
      int j_next = __ldg(lut_row);
      for (int t = 0; t < n_tiles; ++t) {
        const int j = j_next;
        if (t + 1 < n_tiles) j_next = __ldg(lut_row + t + 1);
        const int ks = t % KST;
        mbar_wait(k_empty + ks, ((t / KST) & 1) ^ 1);
        mbar_arrive_expect_tx(k_full + ks, L::K_BYTES);
        if (QK16) {
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
            tma_load_3d(sK + ks * L::K_BYTES + h * L::K_ATOM, &tmK, k_full + ks, h * 64, j * BK, bkv);
        } else {
          tma_load_3d(sK + ks * L::K_BYTES, &tmK, k_full + ks, 0, j * BK, bkv);
        }
        const int vs = t % VST;
        mbar_wait(v_empty + vs, ((t / VST) & 1) ^ 1);
        mbar_arrive_expect_tx(v_full + vs, L::V_BYTES);
        tma_load_3d(sV + vs * L::V_BYTES, &tmV, v_full + vs, j * BK, 0, bkv);
      }
    }
  } else if (warp == WARP_MMA) {
    // ============================ MMA issuer ==============================
    // One thread serves both groups in a fixed alternation (QK(A,0), QK(B,0),
    // then per pair: P~V(A,p), QK(A,p+1), P~V(B,p), QK(B,p+1)), which keeps
    // the two groups' softmax phases staggered: while one group's softmax
    // works on its S, the tensor pipe runs the other group's MMAs.
    if (lane == 0) {
      constexpr uint32_t IDESC_PV = (F16 || PV8) ? idesc_f16(BQ, D) : idesc_bf16(BQ, D);
      int nt[NG], np[NG];
      int np_max = 0;
#pragma unroll
      for (int gg = 0; gg < NG; ++gg) {
        int ii;
        nt[gg] = tile_of(gg, ii);
        np[gg] = (nt[gg] + 1) >> 1;
        np_max = max(np_max, np[gg]);
      }
      unsigned long long issued[NG] = {};
#ifdef SPARGE_PHASE_TIMING
      long long mw[3] = {0, 0, 0};   // cycles waiting: p_full, k_full, v_full
      const long long m_start = clock64();
#define MMA_WAIT(k, bar, par) do { const long long _c0 = clock64(); mbar_wait(bar, par); mw[k] += clock64() - _c0; } while (0)
#else
#define MMA_WAIT(k, bar, par) mbar_wait(bar, par)
#endif
      auto bar_of = [&](int gg, int k) { return reinterpret_cast<uint64_t*>(gsm(gg) + L::OFF_BAR) + k; };
      // QK of pair pp of group gg (Alg. 1 l.12)
      auto issue_qk = [&](int gg, int pp) {
        unsigned char* sgg = gsm(gg);
        const uint32_t tSg = tmem_base + gg * 256;
        const int t0 = 2 * pp;
        const bool two = t0 + 1 < nt[gg];
        const int ks = t0 % KST;                     // even: the pair's slots are ks, ks + 1
        const uint32_t kpar = (t0 / KST) & 1;
        MMA_WAIT(1, bar_of(gg, 1 + ks), kpar);
        if (two) MMA_WAIT(1, bar_of(gg, 2 + ks), kpar);
        // S holds P~ of pair pp-1, read by its P~V MMAs, which this thread
        // issued before this QK: tcgen05.mma from one thread execute in issue
        // order.
        tc_fence_after();
        const uint64_t dQ = umma_desc_kmajor(smem_u32(sgg + L::OFF_Q), L::ROW_BYTES_QK);
        if (QK16) {
          // per tile: K = 16 per kind::f16 MMA (32 B), 4 steps per 128-B
          // atom, then the next atom (fp32 S accumulators)
          constexpr uint32_t IDESC_QK = F16 ? idesc_f16(BQ, BK) : idesc_bf16(BQ, BK);
          for (int h = 0; h < (two ? 2 : 1); ++h) {
            const uint64_t dK = umma_desc_kmajor(smem_u32(sgg + L::OFF_K + (ks + h) * L::K_BYTES), 128);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
              mma_f16(tSg + h * BK, dQ + (((kk >> 2) * L::Q_ATOM + (kk & 3) * 32) >> 4),
                      dK + (((kk >> 2) * L::K_ATOM + (kk & 3) * 32) >> 4), IDESC_QK, kk > 0 ? 1u : 0u);
          }
        } else {
          // both tiles at once: the two K slots are one 128-row operand
          const uint64_t dK = umma_desc_kmajor(smem_u32(sgg + L::OFF_K + ks * L::K_BYTES), L::ROW_BYTES_QK);
          const uint32_t idesc_qk = two ? idesc_i8(BQ, 2 * BK) : idesc_i8(BQ, BK);
          if (L::BIAS)   // S := 1.5*2^23 (fp32 bits), then += acc as int32
            mma_f16(tSg, umma_desc_noswz(smem_u32(sgg + L::OFF_CA), 128, 256),
                    umma_desc_noswz(smem_u32(sgg + L::OFF_CB), 128, 256),
                    two ? idesc_bf16(BQ, 2 * BK) : idesc_bf16(BQ, BK), 0u);
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk)       // K = 32 per kind::i8 MMA (32 B)
            mma_i8(tSg, dQ + 2 * kk, dK + 2 * kk, idesc_qk, (L::BIAS || kk > 0) ? 1u : 0u);
        }
        tc_commit(bar_of(gg, 1 + 2 * KST + 2 * VST));          // s_full
        tc_commit(bar_of(gg, 1 + KST + ks));                   // k_empty
        if (two) tc_commit(bar_of(gg, 2 + KST + ks));
      };
      // P~V of pair pp of group gg, per tile (Alg. 1 l.15-16)
      auto issue_pv = [&](int gg, int pp) {
        unsigned char* sgg = gsm(gg);
        const uint32_t tSg = tmem_base + gg * 256, tOg = tSg + 2 * BK;
        const uint32_t* fl0 = reinterpret_cast<const uint32_t*>(sgg + L::OFF_MISC) + 1;
        const int t0 = 2 * pp;
        const bool two = t0 + 1 < nt[gg];
        MMA_WAIT(0, bar_of(gg, 2 + 2 * KST + 2 * VST), pp & 1);   // p_full
        tc_fence_after();
        for (int h = 0; h < (two ? 2 : 1); ++h) {
          const int t = t0 + h;
          const int vs = t % VST;
          MMA_WAIT(2, bar_of(gg, 1 + 2 * KST + vs), (t / VST) & 1);   // v_full
          tc_fence_after();
          const uint32_t* fl = fl0 + h * 4;
          if ((fl[0] | fl[1] | fl[2] | fl[3]) != 0) {
            const uint32_t tP = tSg + h * BK;     // P~ 16-bit (32 cols) or e4m3 (16 cols)
            if (PV8) {
              // K = 32 e4m3 per kind::f8f6f4 MMA: 8 TMEM cols of P~, 32 B of V^T rows
              const uint64_t dV = umma_desc_kmajor(smem_u32(sgg + L::OFF_V + vs * L::V_BYTES), 64);
#pragma unroll
              for (int kk = 0; kk < BK / 32; ++kk)
                mma_f8_ts(tOg, tP + 8 * kk, dV + 2 * kk, IDESC_PV, 1u);
            } else {
              const uint64_t dV = umma_desc_kmajor(smem_u32(sgg + L::OFF_V + vs * L::V_BYTES), 128);
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)   // K = 16 per kind::f16 MMA: 8 TMEM cols
                mma_f16_ts(tOg, tP + 8 * kk, dV + 2 * kk, IDESC_PV, 1u);
            }
            ++issued[gg];
          }
          tc_commit(bar_of(gg, 1 + 2 * KST + VST + vs));    // v_empty
        }
      };
#pragma unroll
      for (int gg = 0; gg < NG; ++gg) {
        if (np[gg] > 0) {
          mbar_wait(bar_of(gg, 0), 0);   // q_full
          issue_qk(gg, 0);
        }
      }
      for (int pp = 0; pp < np_max; ++pp) {
#pragma unroll
        for (int gg = 0; gg < NG; ++gg) {
          if (pp < np[gg]) {
            issue_pv(gg, pp);
            if (pp + 1 < np[gg]) issue_qk(gg, pp + 1);
            else tc_commit(bar_of(gg, 3 + 2 * KST + 2 * VST));   // o_done
          }
        }
      }
      if (p.counters) {
#pragma unroll
        for (int gg = 0; gg < NG; ++gg)
          if (nt[gg] > 0) atomicAdd(p.counters + bhq * 3 + 2, issued[gg]);
      }
#undef MMA_WAIT
#ifdef SPARGE_PHASE_TIMING
      if (p.phase_clk) {
        for (int k = 0; k < 3; ++k) atomicAdd(p.phase_clk + 8 + k, static_cast<unsigned long long>(mw[k]));
        atomicAdd(p.phase_clk + 11, static_cast<unsigned long long>(clock64() - m_start));
        atomicAdd(p.phase_clk + 12, 1ull);
      }
#endif
    }
  } else {
    // ============================ softmax warps ===========================
    const int quad = warp & 3;                 // TMEM lane quadrant = gate group I_w
    const int r = quad * 32 + lane;            // row within the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const int row_g = i * BQ + r;
    // an empty group (u >= T_m, odd T_m) writes nothing
    const bool group_live = static_cast<int>(blockIdx.x) * NG + g < p.T_m;
    const bool row_valid = group_live && row_g < p.N;
    const bool tile_tail = (i * BQ + BQ > p.N);
    using SB = SBits<QK16, L::BIAS>;
    constexpr int kMaskedBits = SB::kMasked;   // -inf / INT_MIN / 0 (bias MMA)
    constexpr float kPvShift = PV8 ? 7.0f : 0.0f;   // P~' = 2^7 P~ in E4M3 (R27)
    {
      uint32_t z[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) z[k] = 0u;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) tmem_st32(tO + lane_base + cc * 32, z);
      tmem_wait_st();
    }
    const float* dk_row = p.dk + static_cast<int64_t>(bkv) * p.T_n;
    const float dq_scale = __ldg(p.dq + row_id) * p.scale_log2;
    float m_true = -INFINITY, m_ref = -INFINITY, l = 0.f;
    unsigned int slices = 0;
    // Lane u caches j and the dequant scale c = dq*dk*log2e/sqrt(d) of tile
    // 32*chunk + u; they are broadcast with shuffles, so no global load sits
    // on the per-pair path.  The next chunk's j is loaded when a chunk starts
    // and its dk sixteen tiles later (by then j has arrived).
    int cj = 0, nj = 0;
    float cc_ = 0.f, ndk = 0.f;
    if (lane < n_tiles) {
      cj = __ldg(lut_row + lane);
      cc_ = dq_scale * __ldg(dk_row + cj);
    }
    // boundary tiles: keys >= N, causal keys > query, rows >= N
    auto needs_mask = [&](int k0) {
      return tile_tail || (k0 + BK > p.N) || (CAUSAL && (k0 + BK - 1 > i * BQ));
    };
    auto apply_mask = [&](int32_t* a, int k0) {
      const int kmax = CAUSAL ? min(p.N - 1, row_g) : p.N - 1;
#pragma unroll
      for (int k = 0; k < BK; ++k)
        if (!row_valid || k0 + k > kmax) a[k] = kMaskedBits;
    };
    // row max m_local of one tile (Alg. 1 l.14)
    auto row_max = [&](const int32_t* a, float c, float& m_loc, bool& row_has) {
      if (QK16) {
        // fp32 row max of S (masked entries -inf), eight chains
        const float* af = reinterpret_cast<const float*>(a);
        float f8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) f8[u] = fmaxf(af[u], af[u + 8]);
#pragma unroll
        for (int k = 16; k < BK; k += 16)
#pragma unroll
          for (int u = 0; u < 8; ++u) f8[u] = fmaxf(f8[u], fmaxf(af[k + u], af[k + 8 + u]));
        const float mxf = fmaxf(fmaxf(fmaxf(f8[0], f8[1]), fmaxf(f8[2], f8[3])),
                                fmaxf(fmaxf(f8[4], f8[5]), fmaxf(f8[6], f8[7])));
        row_has = mxf > -INFINITY;
        m_loc = row_has ? mxf * c : -INFINITY;
      } else {
        // integer-domain row max over the int32 accumulators, or over the
        // positive fp32 bits 1.5*2^23 + acc (bias MMA): both monotone in acc,
        // and the dequant scale c > 0; eight independent chains
        int m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = max(a[u], a[u + 8]);
#pragma unroll
        for (int k = 16; k < BK; k += 16)
#pragma unroll
          for (int u = 0; u < 8; ++u) m8[u] = max(m8[u], max(a[k + u], a[k + 8 + u]));
        const int mx = max(max(max(m8[0], m8[1]), max(m8[2], m8[3])),
                           max(max(m8[4], m8[5]), max(m8[6], m8[7])));
        // S = acc * dq * dk / sqrt(d) in log2 units; exact int -> fp32
        // through the magic constant (I2F runs on the slow XU pipe)
        row_has = mx != kMaskedBits;
        m_loc = row_has ? (__int_as_float(mx + SB::kAdd) - kMagicF) * c : -INFINITY;
      }
    };
    // P~ of one tile: exps, row sum into l (R9: skipped groups still add their
    // mass), zero rows when the warp skips, store over the tile's S columns
    auto softmax_tile = [&](const int32_t* a, bool masked, float c, bool compute, uint32_t tcol) {
      uint32_t pw[BK / 2];
      float rsum;
      if (masked) exps64<true, F16, QK16, PV8, L::BIAS>(a, c, m_ref - kPvShift, pw, rsum);
      else exps64<false, F16, QK16, PV8, L::BIAS>(a, c, m_ref - kPvShift, pw, rsum);
      l += rsum;
      if (!compute) {
#pragma unroll
        for (int k = 0; k < (PV8 ? BK / 4 : BK / 2); ++k) pw[k] = 0u;
      }
      if (PV8) tmem_st16(tcol, pw);
      else tmem_st32(tcol, pw);
    };
#ifdef SPARGE_PHASE_TIMING
    long long ph[7] = {0, 0, 0, 0, 0, 0, 0};
    long long ph_last = clock64();
#endif
#ifdef SPARGE_CTA_TIMING
    if (threadIdx.x == 0) { CTA_REC(1, gtimer()); CTA_REC(5, n_tiles); }
#endif
    const uint32_t tSa = tS + lane_base, tSb = tS + BK + lane_base;
    for (int pp = 0; pp < n_pairs; ++pp) {
      const int t0 = 2 * pp;
      const bool two = t0 + 1 < n_tiles;
      // ---- LUT entries of the pair ----
      const int tl = t0 & 31;
      if (tl == 0) {
        if (t0 > 0) { cj = nj; cc_ = dq_scale * ndk; }
        if (t0 + 32 + lane < n_tiles) nj = __ldg(lut_row + t0 + 32 + lane);
      } else if (tl == 16) {
        if (t0 + 16 + lane < n_tiles) ndk = __ldg(dk_row + nj);
      }
      const int k0a = __shfl_sync(0xffffffffu, cj, tl) * BK;
      const float ca = __shfl_sync(0xffffffffu, cc_, tl);
      const int k0b = __shfl_sync(0xffffffffu, cj, tl + 1) * BK;
      const float cb = __shfl_sync(0xffffffffu, cc_, tl + 1);
      const bool nma = needs_mask(k0a);
      const bool nmb = two && needs_mask(k0b);

      mbar_wait(s_full, pp & 1);
      tc_fence_after();
#ifdef SPARGE_ABL_NOSOFT   // timing ablation only (wrong results): MMA/sync pipeline floor
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        pv_flag[quad] = 1u;
        pv_flag[4 + quad] = 1u;
        mbar_arrive(p_full);
      }
      continue;
#endif
      PT_MARK(0);
      int32_t a[BK];
      // ---- tile b: row max only (reloaded for its exps below) ----
      float mlb = -INFINITY;
      bool hasb = false;
      if (two) {
        tmem_ld32(tSb, reinterpret_cast<uint32_t*>(a));
        tmem_ld32(tSb + 32, reinterpret_cast<uint32_t*>(a) + 32);
        tmem_wait_ld();
        if (nmb) apply_mask(a, k0b);
        row_max(a, cb, mlb, hasb);
      }
      PT_MARK(1);
      // ---- tile a: row max, kept in registers ----
      tmem_ld32(tSa, reinterpret_cast<uint32_t*>(a));
      tmem_ld32(tSa + 32, reinterpret_cast<uint32_t*>(a) + 32);
      tmem_wait_ld();
      if (nma) apply_mask(a, k0a);
      float mla;
      bool hasa;
      row_max(a, ca, mla, hasa);
      // ---- gates in Alg. 1 order: tile a, then tile b (l.14-15) ----
      const float mn0 = fmaxf(m_true, mla);
      const bool comp0 = __any_sync(0xffffffffu, hasa && (mla - mn0 > p.lam2));
      const float mn1 = fmaxf(mn0, mlb);
      const bool comp1 = two && __any_sync(0xffffffffu, hasb && (mlb - mn1 > p.lam2));
      // one reference for the pair (R22): move it only when a computing tile
      // pushes the true max more than the threshold above it
      const bool need = (comp0 || comp1) && (mn1 > m_ref + kRefThreshold);
      const bool rescale_o = __any_sync(0xffffffffu, need && (m_ref > -INFINITY));
      float alpha = 1.f;
      if (need) {
        alpha = ex2_approx(m_ref - mn1);   // 0 when m_ref = -inf (l, O are 0 then)
        l *= alpha;
        m_ref = mn1;
      }
      m_true = mn1;
      PT_MARK(2);
      if (rescale_o) {
        // O rows of this warp hold P~V of earlier pairs, all complete (s_full
        // of this pair was committed after them): rescale in TMEM before
        // p_full releases this pair's P~V.
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t ov[32];
          tmem_ld32(tO + lane_base + cc * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) ov[k] = __float_as_uint(__uint_as_float(ov[k]) * alpha);
          tmem_st32(tO + lane_base + cc * 32, ov);
        }
      }
      PT_MARK(3);
      // ---- P~ of tile a, then tile b ----
      softmax_tile(a, nma, ca, comp0, tSa);
      PT_MARK(4);
      if (two) {
        tmem_ld32(tSb, reinterpret_cast<uint32_t*>(a));
        tmem_ld32(tSb + 32, reinterpret_cast<uint32_t*>(a) + 32);
        tmem_wait_ld();
        if (nmb) apply_mask(a, k0b);
        softmax_tile(a, nmb, cb, comp1, tSb);
      }
      PT_MARK(5);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(pv_flag + quad)),
                     "r"(comp0 ? 1u : 0u) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(pv_flag + 4 + quad)),
                     "r"(comp1 ? 1u : 0u) : "memory");
        mbar_arrive(p_full);
      }
      slices += (comp0 ? 1u : 0u) + (comp1 ? 1u : 0u);
      PT_MARK(6);
    }
#ifdef SPARGE_PHASE_TIMING
    if (lane == 0 && p.phase_clk)
      for (int k = 0; k < 7; ++k) atomicAdd(p.phase_clk + k, static_cast<unsigned long long>(ph[k]));
    if (quad == 0 && lane == 0 && p.phase_clk)
      atomicAdd(p.phase_clk + 7, static_cast<unsigned long long>(n_tiles));
#endif

#ifdef SPARGE_CTA_TIMING
    if (threadIdx.x == 0) CTA_REC(2, gtimer());
#endif
    // ---- epilogue: O_i = O / l (line 19), scattered back through perm ----
    if (n_tiles > 0) mbar_wait(o_done, 0);
    tc_fence_after();
    if (row_valid && !(l > 0.f)) atomicOr(p.status, 1u);
    const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
    const int dst_row = row_valid ? (p.perm ? __ldg(p.perm + row_g) : row_g) : 0;
    const float* vsc = PV8 ? p.v_scale + static_cast<int64_t>(bkv) * D : nullptr;
    uint16_t* orow = p.o + b * p.o_sb + hq * p.o_sh + static_cast<int64_t>(dst_row) * p.o_sn;
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t ov[32];
      tmem_ld32(tO + lane_base + cc * 32, ov);
      tmem_wait_ld();
      if (PV8) {
#pragma unroll
        for (int k = 0; k < 32; ++k)
          ov[k] = __float_as_uint(__uint_as_float(ov[k]) * __ldg(vsc + cc * 32 + k));
      }
      if (row_valid) {
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          uint4 w;
          const float* f = reinterpret_cast<const float*>(ov) + qq * 8;
          w.x = pack16<F16>(f[0] * inv_l, f[1] * inv_l);
          w.y = pack16<F16>(f[2] * inv_l, f[3] * inv_l);
          w.z = pack16<F16>(f[4] * inv_l, f[5] * inv_l);
          w.w = pack16<F16>(f[6] * inv_l, f[7] * inv_l);
          *reinterpret_cast<uint4*>(orow + cc * 32 + qq * 8) = w;
        }
      }
    }
    if (p.counters) {
      if (lane == 0) atomicAdd(p.counters + bhq * 3 + 1, static_cast<unsigned long long>(slices));
      if (quad == 0 && lane == 0)
        atomicAdd(p.counters + bhq * 3 + 0, static_cast<unsigned long long>(n_tiles));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<256 * NG>(tmem_base);
  }
#ifdef SPARGE_CTA_TIMING
  if (threadIdx.x == 0) CTA_REC(3, gtimer());
#endif
}

template <int D, bool CAUSAL, bool F16, bool QK16, bool PV8 = false>
cudaError_t launch_t(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                     const AttnParams& p, int B, cudaStream_t stream) {
  auto kern = k_sparse_attn<D, CAUSAL, F16, QK16, PV8>;
  const int smem = NG * Smem<D, QK16, PV8>::BYTES + 1024;   // + slack for 1024-B alignment
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((p.T_m + NG - 1) / NG, B * p.Hq);
  kern<<<grid, THREADS, smem, stream>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn(const sparge_shape& s, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, const float* dq, const float* dk,
                        const int32_t* lut, const int32_t* cnt, float lambda,
                        const int32_t* perm, void* o, sparge_strides o_str,
                        uint64_t* counters, unsigned int* status, const float* v_scale,
                        cudaStream_t stream) {
  AttnParams p;
  p.v_scale = v_scale;
  p.dq = dq; p.dk = dk; p.lut = lut; p.cnt = cnt; p.perm = perm;
  p.o = static_cast<uint16_t*>(o);
  p.o_sb = o_str.b; p.o_sh = o_str.h; p.o_sn = o_str.n;
  p.counters = reinterpret_cast<unsigned long long*>(counters);
  p.status = status;
  p.lam2 = lambda * kLog2e;     // -inf stays -inf
  p.scale_log2 = kLog2e / sqrtf(static_cast<float>(s.d));
  p.N = s.N;
  p.T_m = (s.N + BQ - 1) / BQ;
  p.T_n = (s.N + BK - 1) / BK;
  p.Hq = s.Hq; p.Hkv = s.Hkv; p.group = s.Hq / s.Hkv;
  p.phase_clk = reinterpret_cast<unsigned long long*>(status + 8);   // debug builds only
  const bool f16 = s.in_dtype == SPARGE_FP16;
  const bool qk16 = s.qk_dtype == SPARGE_QK_INPUT;
  const bool pv8 = s.pv_dtype == SPARGE_PV_FP8_E4M3;   // INT8 QK only (validated)
#define SPARGE_A(D, C, F)                                                      \
  return qk16 ? launch_t<D, C, F, true>(mq, mk, mv, p, s.B, stream)            \
              : (pv8 ? launch_t<D, C, F, false, true>(mq, mk, mv, p, s.B, stream) \
                     : launch_t<D, C, F, false>(mq, mk, mv, p, s.B, stream))
  if (s.d == 128) {
    if (s.causal) { if (f16) SPARGE_A(128, true, true); else SPARGE_A(128, true, false); }
    else          { if (f16) SPARGE_A(128, false, true); else SPARGE_A(128, false, false); }
  } else {
    if (s.causal) { if (f16) SPARGE_A(64, true, true); else SPARGE_A(64, true, false); }
    else          { if (f16) SPARGE_A(64, false, true); else SPARGE_A(64, false, false); }
  }
#undef SPARGE_A
}

#ifdef SPARGE_CTA_TIMING
}  // namespace sparge
extern "C" int sparge_debug_cta_records(void* host_dst, size_t bytes) {
  return cudaMemcpyFromSymbol(host_dst, g_cta_rec, bytes) == cudaSuccess ? 0 : 4;
}
namespace sparge {
#endif

int attn_smem_bytes(int d, int qk16) {
  if (qk16) return NG * (d == 128 ? Smem<128, true>::BYTES : Smem<64, true>::BYTES) + 1024;
  return NG * (d == 128 ? Smem<128, false>::BYTES : Smem<64, false>::BYTES) + 1024;
}

}  // namespace sparge
