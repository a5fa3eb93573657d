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
// sm_100a design.  A CTA = 4 softmax warps + 1 TMA producer warp + 1 MMA
// warp, 256 TMEM columns (S0 | S1, 64 cols each | O, d cols), two CTAs per
// SM; the grid is the launch order of k_order (longest work items first).
//   producer  Q^ once, then K^_j (4-stage ring) and V^T_j (3-stage ring) for
//             every kept j; SWIZZLE_128B/64B tiles.
//   MMA       one thread: per tile a bias MMA (S := fp32 bits of 1.5*2^23),
//             then tcgen05.mma kind::i8 Q^K^^T accumulating onto it ->
//             S[t%2] (kind::f16 for the unquantised f1 kernel), then
//             kind::f16 P~ V -> O with P~ read from TMEM (TS form).  QK(t+1)
//             is issued right after P~V(t-1) (in-order tensor pipe).  The
//             P~V MMA is skipped when all four row groups vote to skip
//             (their P~ rows are zero otherwise: exact).
//   softmax   thread r owns row r == TMEM lane r; warp w is the gate group
//             I_w (rows 32w..32w+31).  exp2 domain (lambda compared as
//             lambda*log2e); the gate max is a warp vote (max_r gap_r >
//             lambda <=> any_r gap_r > lambda); integer row max over the
//             biased fp32 bits; one FFMA per element dequantises and applies
//             the reference (R23); packed f32x2 arithmetic; all exponentials
//             on the MUFU (SPARGE_POLY_EVERY=k moves 1 pair in k to the FMA
//             pipe, exp2_poly2: slower, the MUFU is not the bound); P~
//             (16-bit) written back into the first 32 columns of its own S
//             buffer; lazy O rescale (R22: the reference max moves only when
//             the true max grows by > 16 in log2 units, 15 for fp16 P~; O/l is
//             invariant to the reference, the gate always uses the true
//             running max).
//   (Experiments -- two query tiles per CTA with ping-pong exp bursts, rows
//   split over 8 softmax warps, 128-key pair iterations, speculative exps --
//   are in profiles/experiments/ and the git history.)
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
constexpr int NSOFT = 4;      // softmax warps per query tile: one per TMEM lane quadrant
#ifndef SPARGE_RESCALE_THR
#define SPARGE_RESCALE_THR 16
#endif
// lazy-rescale threshold (R22), log2 units: P~ <= 2^thr, which fp16 P~ must
// hold (max 65504 < 2^16)
constexpr float kRescaleThreshold = static_cast<float>(SPARGE_RESCALE_THR);
constexpr float kRescaleThresholdF16 = SPARGE_RESCALE_THR < 15 ? SPARGE_RESCALE_THR : 15.0f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMagic = 0x4B400000;          // bits of 1.5 * 2^23
constexpr float kMagicF = 12582912.0f;

#ifndef SPARGE_POLY_EVERY
#define SPARGE_POLY_EVERY 0
#endif
// one pair in kPolyEvery uses exp2_poly2 (0: none).  d = 128 is chain-bound
// (the MUFU is not the limit: 0); the d = 64 kernel has half the tensor work
// per tile and is softmax-bound, where offloading 1 pair in 8 measured ~1 %
// faster (CogVideoX) and 1 in 4 slower
#ifndef SPARGE_POLY_EVERY64
#define SPARGE_POLY_EVERY64 8
#endif
constexpr int kPolyEvery = SPARGE_POLY_EVERY;
constexpr int kPolyEvery64 = SPARGE_POLY_EVERY64;

// CTA roles: softmax warps 0-3 (one per TMEM lane quadrant), TMA producer
// warp 4, MMA issuer warp 5.  (Experiments with two query tiles per CTA, a
// speculative exp pass and timing ablations live in the git history and
// profiles/experiments/; DESIGN.md §6 has their measurements.)
//
// SPARGE_ATTN_8W=1 (round 2 option, off by default): two idle warps pad the CTA to 8 warps =
// two warpgroups, launched at 128 registers per thread; the softmax
// warpgroup raises its budget to kRegSoftmax and the producer / MMA / idle
// warpgroup lowers its to kRegOther with setmaxnreg.  Why: with 6 warps at
// ~160 registers a CTA puts 2 warps on two SM sub-partitions and 1 on the
// other two, so a second CTA fits only in the complementary placement --
// per-CTA timelines (scripts/cta_timeline.py) showed an SM whose YOUNGER CTA
// exited first was never refilled until the older one exited too (Mochi 22K:
// ~85 % of SMs at one CTA for 135 us, 12 % of slot time idle).  With 8 warps
// every CTA puts exactly two warps (one per warpgroup) on each sub-partition
// and fits next to any other.  Measured (profiles/r02/r02_s19_attn_8w.txt):
// the refill gaps vanish (Mochi 22K 80 -> 10 us per slot: step -3.7 %) but
// a tile costs ~2 % more (786 -> 805 ns/tile on Llama), so Llama, CogVideoX,
// Flux and the sweep are 1-2 % slower -- not the default.  (A 6-warp CTA
// cannot use setmaxnreg: it needs whole warpgroups; that variant hung.)
#ifndef SPARGE_ATTN_8W
#define SPARGE_ATTN_8W 0
#endif
constexpr bool kPad8 = SPARGE_ATTN_8W == 1;
constexpr int kMaxSms = 256;
__device__ unsigned g_sm_slots[kMaxSms];     // per-SM CTA-slot bits (kPad8)
constexpr int WARP_LOAD = NSOFT, WARP_MMA = NSOFT + 1;
constexpr int THREADS = (kPad8 ? 2 * NSOFT : NSOFT + 2) * 32;
#ifndef SPARGE_REG_SOFTMAX
#define SPARGE_REG_SOFTMAX 168
#endif
constexpr int kRegSoftmax = SPARGE_REG_SOFTMAX;      // setmaxnreg budgets: (softmax + other) / 2
constexpr int kRegOther = 256 - SPARGE_REG_SOFTMAX;  // = 128 registers per warp pair
static_assert(!kPad8 || (kRegSoftmax + kRegOther) / 2 * THREADS * 2 <= 65536, "two CTAs per SM");

// Shared-memory plan of a CTA.  QK16 = the unquantised f1 kernel (16-bit Q,
// K tiles stored as d/64 SWIZZLE_128B K-atoms of 128 B rows); with d = 128
// its rings shrink to 2 + 2 stages so that two CTAs still fit on an SM.
// SPARGE_BIAS_MMA (INT8 QK): before the kind::i8 MMAs of a tile, one
// kind::f16 MMA (M128 N64 K16, constant operands 1.0 x 1.5*2^19 summed over
// K = 16) writes the fp32 value 1.5*2^23 into every S accumulator; the i8
// MMAs then accumulate onto those bits as int32, so S leaves the tensor core
// as bits(1.5*2^23 + acc) -- the exact fp32 value 1.5*2^23 + acc (R23)
// without a per-element integer add in the softmax warps.
#ifndef SPARGE_BIAS_MMA
#define SPARGE_BIAS_MMA 1
#endif
constexpr bool kBiasMma = SPARGE_BIAS_MMA != 0;
constexpr uint16_t kBf16One = 0x3F80;        // bf16 1.0
constexpr uint16_t kBf16MagicPart = 0x4940;  // bf16 786432 = 1.5*2^19 (x 16 = 1.5*2^23)

#ifndef SPARGE_NSB64
#define SPARGE_NSB64 2
#endif
template <int D, bool QK16, bool PV8 = false>
struct Smem {
  static constexpr int EB = QK16 ? 2 : 1;       // bytes per Q/K element
  static constexpr int KST = (QK16 && D == 128) ? 2 : 4;   // K stages
  static constexpr int VST = (QK16 && D == 128) ? 2 : (PV8 ? 4 : 3);   // V^T stages
  static constexpr int Q_BYTES = BQ * D * EB;
  static constexpr int K_BYTES = BK * D * EB;
  static constexpr int V_BYTES = D * BK * (PV8 ? 1 : 2);    // V^T tile, 16-bit or e4m3
  static constexpr bool BIAS = kBiasMma && !QK16;
  // constant bias-MMA operands: A 128 x 16 bf16 ones, B 64 x 16 bf16 1.5*2^19
  static constexpr int CA_BYTES = BIAS ? BQ * 16 * 2 : 0;
  static constexpr int CB_BYTES = BIAS ? BK * 16 * 2 : 0;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * K_BYTES;
  static constexpr int OFF_CA = OFF_V + VST * V_BYTES;
  static constexpr int OFF_CB = OFF_CA + CA_BYTES;
  static constexpr int OFF_BAR = OFF_CB + CB_BYTES;
  // S ring depth: d = 128 fits two 64-column S buffers next to O in 256
  // TMEM columns (2*64 + 128); d = 64 would fit three (3*64 + 64), but the
  // third buffer measured no faster on CogVideoX (1.067 vs 1.058 ms: the
  // d = 64 kernel is softmax-bound), so SPARGE_NSB64 = 3 is an option only
  static constexpr int NSB = SPARGE_NSB64 > 0 && D == 64 ? SPARGE_NSB64 : 2;
  static constexpr int N_BARS = 1 + 2 * KST + VST + 2 * 3;
  // [0] TMEM base, [16..] P~V flags [NSB][4]
  static constexpr int OFF_MISC = (OFF_BAR + N_BARS * 8 + 15) / 16 * 16;
  static constexpr int TOTAL = OFF_MISC + 16 + 16 * NSB;
  static constexpr int BYTES = (TOTAL + 1023) / 1024 * 1024;
  static_assert(VST >= NSB, "the V-slot release waits on QK(t - VST + NSB) <= QK(t)");
  // INT8: one K-atom of D bytes per row (128 -> SW128, 64 -> SW64); 16-bit:
  // 128-B atoms, the second (d = 128) BQ*128 / BK*128 bytes after the first
  static constexpr int ROW_BYTES_QK = QK16 ? 128 : D;
  static constexpr int Q_ATOM = BQ * 128, K_ATOM = BK * 128;
  static_assert(2 * (BYTES + 1024) <= 227 * 1024, "two CTAs must fit one SM");
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
  const int32_t* order;   // work items (bhq * T_m + i), the launch order of k_order
  uint8_t* mpv;           // debug: M_pv decisions [B*Hq*T_m, T_n, 4] (nullptr = off)
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
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
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
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}"
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

template <bool MASKED, bool F16, bool QK16 = false, bool PV8 = false, bool BIAS = false,
          int POLY = 0>
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
    if (!MASKED && POLY > 0 && ((k >> 1) % (POLY > 0 ? POLY : 1)) == POLY - 1)
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
// SPARGE_ATTN_MAXNREG=R (A/B option): cap the 6-warp kernel at R registers
// per thread instead of the launch bound's 170; at R <= 128 two CTAs fit an
// SM in any warp placement (no refill gaps, see SPARGE_ATTN_8W above)
#if defined(SPARGE_ATTN_MAXNREG) && !SPARGE_ATTN_8W
__global__ void __maxnreg__(SPARGE_ATTN_MAXNREG)
#else
__global__ void __launch_bounds__(THREADS, 2)
#endif
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

  // `warp` comes from a shuffle, so the compiler treats it (and every smem /
  // barrier / TMEM address derived from it) as warp-uniform
  const int warp = __shfl_sync(0xffffffffu, warp_id(), 0), lane = lane_id();
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  // kPad8: which of its SM's two CTA slots this CTA holds (a per-SM bit mask
  // in global memory, claimed here and released at exit).  Slot 0 runs the
  // producer / MMA roles on warps 4 / 5 (sub-partitions 0 / 1), slot 1 on
  // warps 6 / 7 (2 / 3), so two co-resident CTAs split the single-thread
  // tcgen05 / TMA issue over the four sub-partitions.  A mask left stale by
  // an aborted launch only costs balance: both bits taken -> slot 0.
  // OFF_MISC + 4: the slot (0/1); + 8: the claimed bit (-1: none); + 12: smid
  int* slot_smem = reinterpret_cast<int*>(smem + L::OFF_MISC + 4);
  if (kPad8 && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned* w = g_sm_slots + (smid & (kMaxSms - 1));
    int my_bit = -1;
    if (!(atomicOr(w, 1u) & 1u)) my_bit = 0;
    else if (!(atomicOr(w, 2u) & 2u)) my_bit = 1;
    slot_smem[0] = my_bit > 0 ? 1 : 0;
    slot_smem[1] = my_bit;
    slot_smem[2] = static_cast<int>(smid);
  }

  int8_t* sQ = reinterpret_cast<int8_t*>(smem + L::OFF_Q);
  int8_t* sK = reinterpret_cast<int8_t*>(smem + L::OFF_K);
  unsigned char* sV = smem + L::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  // s_full[ks]: QK of the tile in K slot ks is done -- S is ready for the
  // softmax AND the K slot is free for the producer (one commit, not two)
  uint64_t* s_full = k_full + KST;           // [KST]
  uint64_t* v_full = s_full + KST;
  constexpr int NSB = L::NSB;
  uint64_t* p_full = v_full + VST;           // [NSB]
  uint64_t* o_tail = p_full + NSB;           // [NSB], each completes once
  // P~V flags [NSB][4] (16-B aligned rows: one ld.shared.v4 per tile)
  uint32_t* pv_flag = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC + 16);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) { mbar_init(k_full + s, 1); mbar_init(s_full + s, 1); }
    for (int s = 0; s < VST; ++s) mbar_init(v_full + s, 1);
    for (int s = 0; s < NSB; ++s) {
      mbar_init(p_full + s, NSOFT);
      mbar_init(o_tail + s, 1);
    }
    fence_mbar_init();
  }
  if constexpr (L::BIAS) {
    // constant operands of the bias MMA (every element equal, so the core
    // matrix layout of the descriptor is immaterial)
    constexpr uint32_t kOnes = kBf16One | (static_cast<uint32_t>(kBf16One) << 16);
    constexpr uint32_t kParts = kBf16MagicPart | (static_cast<uint32_t>(kBf16MagicPart) << 16);
    uint32_t* cw = reinterpret_cast<uint32_t*>(smem + L::OFF_CA);
    for (int x = threadIdx.x; x < (L::CA_BYTES + L::CB_BYTES) / 4; x += blockDim.x)
      cw[x] = x < L::CA_BYTES / 4 ? kOnes : kParts;
    fence_proxy_async_smem();   // generic-proxy writes -> visible to the tensor core
  }
  if (warp == WARP_MMA) tmem_alloc<256>(tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const int slot2 = kPad8 ? 2 * *slot_smem : 0;
  const int warp_load = WARP_LOAD + slot2, warp_mma = WARP_MMA + slot2;
  // PDL (sparge_internal.h): the set-up above (barriers, bias operands, TMEM)
  // overlapped the previous kernel's tail; its outputs are visible from here
  griddep_wait();
  griddep_launch();
  // this CTA's work item from the launch order of k_order (the items with
  // the most kept blocks launch first)
  const int item = __ldg(p.order + blockIdx.x);
  const int bhq = item / p.T_m, i = item - bhq * p.T_m;
  const int b = bhq / p.Hq, hq = bhq % p.Hq;
  const int bkv = b * p.Hkv + hq / p.group;

  const int64_t row_id = static_cast<int64_t>(bhq) * p.T_m + i;
  const int n_tiles = p.cnt[row_id];
  const int32_t* lut_row = p.lut + row_id * p.T_n;
  const uint32_t tS0 = tmem_base, tO = tS0 + NSB * BK;
  // P~V(u) of the last NSB tiles, u >= n - NSB, completes o_tail[u - max(0,
  // n - NSB)] -- a barrier used once, so its parity-0 wait is unambiguous
  auto wait_tail = [&](int u) { mbar_wait(o_tail + (u - max(0, n_tiles - NSB)), 0); };
  // register budgets per warpgroup (kPad8), set at the top of each role's
  // branch so the compiler allocates each role's code under its own budget
  auto regs_other = [] {
    if constexpr (kPad8) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegOther));
  };

  if (warp == warp_load) {
    regs_other();
    // ============================ TMA producer ============================
    // (the whole warp runs the loop, one elected lane issues: see sm100.cuh)
    if (n_tiles > 0) {
      if (lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
      }
      mbar_arrive_expect_tx_ew(q_full, L::Q_BYTES);
      if (QK16) {
#pragma unroll
        for (int h = 0; h < D / 64; ++h) tma_load_3d_ew(sQ + h * L::Q_ATOM, &tmQ, q_full, h * 64, i * BQ, bhq);
      } else {
        tma_load_3d_ew(sQ, &tmQ, q_full, 0, i * BQ, bhq);
      }
      int j_next = __ldg(lut_row);
      for (int t = 0; t < n_tiles; ++t) {
        const int j = j_next;
        if (t + 1 < n_tiles) j_next = __ldg(lut_row + t + 1);
        const int ks = t % KST;
        mbar_wait_backoff(s_full + ks, ((t / KST) & 1) ^ 1);   // QK(t - KST) done: slot free
        mbar_arrive_expect_tx_ew(k_full + ks, L::K_BYTES);
        if (QK16) {
#pragma unroll
          for (int h = 0; h < D / 64; ++h)
            tma_load_3d_ew(sK + ks * L::K_BYTES + h * L::K_ATOM, &tmK, k_full + ks, h * 64, j * BK, bkv);
        } else {
          tma_load_3d_ew(sK + ks * L::K_BYTES, &tmK, k_full + ks, 0, j * BK, bkv);
        }
        const int vs = t % VST;
        // V slot of tile t - VST is free once P~V(t - VST) is done, i.e. once
        // QK(t - VST + NSB) -- the next QK issued after it (issue order:
        // QK(u + NSB - 1), P~V(u), QK(u + NSB)) -- is (its s_full commit
        // covers every earlier MMA; a skipped P~V needs nothing).  u <= t
        // because VST >= NSB, so that QK's K tile is already in flight.
        if (t >= VST) {
          const int u = t - VST + L::NSB;
          mbar_wait_backoff(s_full + u % KST, (u / KST) & 1);
        }
        mbar_arrive_expect_tx_ew(v_full + vs, L::V_BYTES);
        if (kVtTiled && !PV8) tma_load_3d_ew(sV + vs * L::V_BYTES, &tmV, v_full + vs, 0, j * D, bkv);
        else tma_load_3d_ew(sV + vs * L::V_BYTES, &tmV, v_full + vs, j * BK, 0, bkv);
      }
    }
  } else if (warp == warp_mma) {
    regs_other();
    // ============================ MMA issuer ==============================
    // (the whole warp runs the loop, one elected lane issues: see sm100.cuh)
    if (n_tiles > 0) {
      constexpr uint32_t IDESC_QK =
          QK16 ? (F16 ? idesc_f16(BQ, BK) : idesc_bf16(BQ, BK)) : idesc_i8(BQ, BK);
      // (kind::f8f6f4 with E4M3 A/B and fp32 D has the f16 field values)
      constexpr uint32_t IDESC_PV = (F16 || PV8) ? idesc_f16(BQ, D) : idesc_bf16(BQ, D);
      const uint64_t dQ = umma_desc_kmajor(smem_u32(sQ), L::ROW_BYTES_QK);
      const uint64_t dK0 = umma_desc_kmajor(smem_u32(sK), L::ROW_BYTES_QK);
      const uint64_t dV0 = umma_desc_kmajor(smem_u32(sV), PV8 ? 64 : 128);
      constexpr uint32_t IDESC_BIAS = idesc_bf16(BQ, BK);
      const uint64_t dCA = umma_desc_noswz(smem_u32(smem + L::OFF_CA), 128, 256);
      const uint64_t dCB = umma_desc_noswz(smem_u32(smem + L::OFF_CB), 128, 256);
      unsigned long long issued = 0;
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto do_pv = [&](int u) {
        const int pb = u % NSB, vs = u % VST;
        mbar_wait(p_full + pb, (u / NSB) & 1);
        mbar_wait(v_full + vs, (u / VST) & 1);
        tc_fence_after();
        uint32_t f0, f1, f2, f3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(f0), "=r"(f1), "=r"(f2), "=r"(f3) : "r"(smem_u32(pv_flag + pb * 4))
                     : "memory");
        const bool any = (f0 | f1 | f2 | f3) != 0;
        if (any) {
          const uint32_t tP = tS0 + pb * BK;     // P~ 16-bit (32 cols) or e4m3 (16 cols)
          if (PV8) {
            // K = 32 e4m3 per kind::f8f6f4 MMA: 8 TMEM cols of P~, 32 B of V^T rows
            const uint64_t dV = dV0 + static_cast<uint64_t>((vs * L::V_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk)
              mma_f8_ts(tO, tP + 8 * kk, dV + 2 * kk, IDESC_PV, 1u);
          } else {
            const uint64_t dV = dV0 + static_cast<uint64_t>((vs * L::V_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)   // K = 16 per kind::f16 MMA: 8 TMEM cols
              mma_f16_ts(tO, tP + 8 * kk, dV + 2 * kk, IDESC_PV, 1u);
          }
          ++issued;
        }
        // only the last NSB P~V signal completion (o_tail): the softmax's
        // rare O rescale at tile t waits on s_full(t+NSB-1) instead (QK(t+NSB-1)
        // is issued after P~V(t-1)) while that tile exists, else on o_tail, as
        // does the epilogue -- one tcgen05.commit (~44 issue cycles) less per
        // tile
        if (u + NSB >= n_tiles) tc_commit_ew(o_tail + (u - max(0, n_tiles - NSB)));
      };
      // QK(t) into S[t % NSB]: issued right after P~V(t - NSB), the previous
      // reader of that buffer (tcgen05.mma from one thread execute in issue
      // order; the softmax warps finished reading S(t-NSB) before they
      // arrived on its p_full).  Order: QK(0..NSB-2), then per t: QK(t+NSB-1),
      // P~V(t) -- the S ring runs NSB-1 tiles ahead of the P~V.
      auto issue_qk = [&](int t) {
        const int ks = t % KST, sb = t % NSB;
        mbar_wait(k_full + ks, (t / KST) & 1);
        tc_fence_after();
        // slot descriptors = the slot-0 descriptor + the slot offset in the
        // 14-bit start-address field (smem < 256 KB: no carry out of it)
        const uint64_t dK = dK0 + static_cast<uint64_t>((ks * L::K_BYTES) >> 4);
        if (QK16) {
          // K = 16 per kind::f16 MMA (32 B): 4 steps per 128-B atom, then
          // the next atom (fp32 S accumulators)
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_f16_ew(tS0 + sb * BK, dQ + (((kk >> 2) * L::Q_ATOM + (kk & 3) * 32) >> 4),
                    dK + (((kk >> 2) * L::K_ATOM + (kk & 3) * 32) >> 4), IDESC_QK, kk > 0 ? 1u : 0u);
        } else {
          if (L::BIAS)   // S := 1.5*2^23 (fp32 bits), then += acc as int32
            mma_f16_ew(tS0 + sb * BK, dCA, dCB, IDESC_BIAS, 0u);
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk)       // K = 32 per kind::i8 MMA (32 B)
            mma_i8_ew(tS0 + sb * BK, dQ + 2 * kk, dK + 2 * kk, IDESC_QK, (L::BIAS || kk > 0) ? 1u : 0u);
        }
        tc_commit_ew(s_full + ks);
      };
      for (int t = 0; t < NSB - 1 && t < n_tiles; ++t) issue_qk(t);
      for (int t = 0; t < n_tiles; ++t) {
        if (t + NSB - 1 < n_tiles) issue_qk(t + NSB - 1);
        do_pv(t);
      }
      if (p.counters && lane == 0) atomicAdd(p.counters + bhq * 3 + 2, issued);
    }
  } else if (warp >= NSOFT) {
    regs_other();               // kPad8: the two idle warps
  } else {
    if constexpr (kPad8) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    // ============================ softmax warps ===========================
    const int quad = warp & 3;                 // TMEM lane quadrant = gate group I_w
    const int r = quad * 32 + lane;            // row within the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const int row_g = i * BQ + r;
    const bool row_valid = row_g < p.N;
    const bool tile_tail = (i * BQ + BQ > p.N);
    using SB = SBits<QK16, L::BIAS>;
    constexpr int kMaskedBits = SB::kMasked;   // -inf / INT_MIN / 0 (bias MMA)
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
    // on the per-tile path.  The next chunk's j is loaded at t%32 == 0 and
    // its dk at t%32 == 16 (by then j has arrived).
    int cj = 0, nj = 0;
    float cc_ = 0.f, ndk = 0.f;
    if (lane < n_tiles) {
      cj = __ldg(lut_row + lane);
      cc_ = dq_scale * __ldg(dk_row + cj);
    }
#ifdef SPARGE_PHASE_TIMING
    long long ph[7] = {0, 0, 0, 0, 0, 0, 0};
    long long ph_last = clock64();
#endif
#ifdef SPARGE_CTA_TIMING
    if (threadIdx.x == 0) { CTA_REC(1, gtimer()); CTA_REC(5, n_tiles); }
#endif
    for (int t = 0; t < n_tiles; ++t) {
      const int sb = t % NSB;
      const uint32_t tS = tS0 + sb * BK + lane_base;
      int32_t a[BK];
      uint32_t pw[BK / 2];
      float c = 0.f;
      bool need_mask = false, compute = false, need = false, rescale_o = false;
      float alpha = 1.f;
      {
        const int tl = t & 31;
        if (tl == 0) {
          if (t > 0) { cj = nj; cc_ = dq_scale * ndk; }
          if (t + 32 + lane < n_tiles) nj = __ldg(lut_row + t + 32 + lane);
        } else if (tl == 16) {
          if (t + 16 + lane < n_tiles) ndk = __ldg(dk_row + nj);
        }
        const int j = __shfl_sync(0xffffffffu, cj, tl);
        c = __shfl_sync(0xffffffffu, cc_, tl);

        PT_MARK(0);
        mbar_wait(s_full + t % KST, (t / KST) & 1);
        PT_MARK(1);
        tc_fence_after();
        tmem_ld32(tS, reinterpret_cast<uint32_t*>(a));
        tmem_ld32(tS + 32, reinterpret_cast<uint32_t*>(a) + 32);
        tmem_wait_ld();
        PT_MARK(6);

        // ---- masking of boundary tiles: keys >= N, causal keys > query, rows >= N
        const int k0 = j * BK;
        need_mask = tile_tail || (k0 + BK > p.N) || (CAUSAL && (k0 + BK - 1 > i * BQ));
        if (need_mask) {
          const int kmax = CAUSAL ? min(p.N - 1, row_g) : p.N - 1;
#pragma unroll
          for (int k = 0; k < BK; ++k)
            if (!row_valid || k0 + k > kmax) a[k] = kMaskedBits;
        }
        // row max m_local (Alg. 1 l.14)
        auto row_max = [&](float& m_loc, bool& row_has) {
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
            // positive fp32 bits 1.5*2^23 + acc (bias MMA): both monotone in
            // acc, and the dequant scale c > 0; eight independent chains
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
        // PV8: P~' = 2^7 P~ (E4M3 range and precision; l carries the same
        // factor, so O = acc * s_c / l needs no extra scale)
        constexpr float kPvShift = PV8 ? 7.0f : 0.0f;
        float m_loc, rsum = 0.f;
        bool row_has;
        row_max(m_loc, row_has);
        const float m_new = fmaxf(m_true, m_loc);
        // Alg. 1 line 15: max_{r in I_w}(m_local - m_new) > lambda, as a vote
        compute = __any_sync(0xffffffffu, row_has && (m_loc - m_new > p.lam2));
        // debug dump of the gate decision of (tile j, warp quad): 2 = P~V
        // computed, 1 = skipped by the lambda gate (0 stays: block not kept)
        if (p.mpv != nullptr && lane == 0)
          p.mpv[(row_id * p.T_n + j) * NSOFT + quad] = compute ? 2 : 1;
        // lazy rescale (R22): move the reference max only when it lags the
        // true max by more than the threshold (always when it is -inf)
        need = compute && (m_new > m_ref + kRefThreshold);
        rescale_o = __any_sync(0xffffffffu, need && (m_ref > -INFINITY));
        if (need) {
          alpha = ex2_approx(m_ref - m_new);   // 0 when m_ref = -inf (l, O are 0 then)
          l *= alpha;
          m_ref = m_new;
        }
        m_true = m_new;
        PT_MARK(2);

        // ---- P~ = exp2(S*log2e - m_ref), row sum, 16-bit P~ (l.13) ----
        constexpr int kPoly = D == 64 ? kPolyEvery64 : kPolyEvery;
        if (need_mask) exps64<true, F16, QK16, PV8, L::BIAS, kPoly>(a, c, m_ref - kPvShift, pw, rsum);
        else exps64<false, F16, QK16, PV8, L::BIAS, kPoly>(a, c, m_ref - kPvShift, pw, rsum);
        l += rsum;           // R9: skipped groups still add their mass to l
      }

      {
        if (!compute) {
#pragma unroll
          for (int k = 0; k < (PV8 ? BK / 4 : BK / 2); ++k) pw[k] = 0u;
        }
        PT_MARK(4);

        if (rescale_o) {
          // O rows of this warp hold P~V of earlier tiles: wait for the last
          // issued P~V, then rescale in TMEM (before p_full(t) releases P~V(t)).
          if (t >= 1) {
            const int tq = t + NSB - 1;
            if (tq < n_tiles) mbar_wait(s_full + tq % KST, (tq / KST) & 1);
            else wait_tail(t - 1);   // P~V(t-1)
          }
          tc_fence_after();
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

        // P~(t) overwrites the first 32 columns of S[sb]: S(t) is already in
        // registers, and QK(t) -- complete, per s_full -- executed after
        // P~V(t-2), the previous reader of this buffer.
        if (PV8) tmem_st16(tS, pw);
        else tmem_st32(tS, pw);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(pv_flag + sb * 4 + quad)),
                       "r"(compute ? 1u : 0u) : "memory");
          mbar_arrive(p_full + sb);
        }
        if (compute) ++slices;
        PT_MARK(5);
      }
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
    if (n_tiles > 0) wait_tail(n_tiles - 1);   // P~V(n-1)
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
  if (warp == WARP_MMA) {     // the allocating warp (MMA or idle role)
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<256>(tmem_base);
  }
  if (kPad8 && threadIdx.x == 0 && slot_smem[1] >= 0) {
    // release the slot; the returned value is consumed so the atomic has
    // completed before this CTA exits and the SM takes the next one
    const unsigned r = atomicAnd(g_sm_slots + (slot_smem[2] & (kMaxSms - 1)), ~(1u << slot_smem[1]));
    asm volatile("" ::"r"(r));
  }
#ifdef SPARGE_CTA_TIMING
  if (threadIdx.x == 0) CTA_REC(3, gtimer());
#endif
}

template <int D, bool CAUSAL, bool F16, bool QK16, bool PV8 = false>
cudaError_t launch_t(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                     const AttnParams& p, int B, cudaStream_t stream) {
  auto kern = k_sparse_attn<D, CAUSAL, F16, QK16, PV8>;
  const int smem = Smem<D, QK16, PV8>::BYTES + 1024;   // + slack for 1024-B alignment
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  return launch_k(kPdlAttn, kern, dim3(p.T_m * B * p.Hq), dim3(THREADS), smem, stream, mq, mk, mv, p);
}


}  // namespace

cudaError_t launch_attn(const sparge_shape& s, const CUtensorMap& mq, const CUtensorMap& mk,
                        const CUtensorMap& mv, const float* dq, const float* dk,
                        const int32_t* lut, const int32_t* cnt, float lambda,
                        const int32_t* perm, void* o, sparge_strides o_str,
                        uint64_t* counters, unsigned int* status, const float* v_scale,
                        const int32_t* order, uint8_t* mpv, cudaStream_t stream) {
  AttnParams p;
  p.mpv = mpv;
  p.v_scale = v_scale;
  p.order = order;
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
  if (qk16) return (d == 128 ? Smem<128, true>::BYTES : Smem<64, true>::BYTES) + 1024;
  return (d == 128 ? Smem<128, false>::BYTES : Smem<64, false>::BYTES) + 1024;
}

}  // namespace sparge
