// Experiment (slower: Llama 32K 4.99 ms vs 3.40 for the two-CTA kernel): one CTA per SM,
// eight softmax warps splitting each pair of tiles by columns, N=128 QK.  Not built.

// ============================================================================
// v5 ("column-split pairs", INT8 QK with 16-bit P~V; the default for those):
// one CTA per SM, EIGHT softmax warps, 512 TMEM columns:
//   SP[0] | SP[1]  two pair buffers of 128 columns (tiles 2p | 2p+1 of the
//                  LUT side by side), double-buffered across pairs
//   O              d columns
// The kept tiles go two at a time: one kind::i8 QK MMA group with N = 128
// covers both tiles of a pair (the two K slots are adjacent, one 128-row
// operand), so a pair costs ~9 tensor instructions per tile instead of 13
// (profiles/r01s2/attn_ablations.md: the single MMA thread issues one
// tcgen05 op per ~48 cycles, and with one 64-key tile per synchronisation
// round trip the MMA chain alone left the tensor pipe 36 % idle).  Softmax
// warp w owns TMEM lane quadrant q = w & 3 and HALF h = w >> 2 of each pair
// (tile 2p + h): warps q and q+4 hold the same 32 rows, exchange their tile
// row maxima through shared memory (named barrier 1 + q), and then both
// evaluate the identical Alg. 1 recurrence for the pair -- tile 2p first,
// then tile 2p+1 (gates l.14-15 per tile, one lazy reference max for the
// pair, R22) -- each keeping its own partial row sum; the epilogue adds them.
// ============================================================================
#ifndef SPARGE_ATTN_V5
#define SPARGE_ATTN_V5 1
#endif
constexpr bool kV5 = SPARGE_ATTN_V5 != 0;
constexpr int V5_SOFT = 8;
constexpr int V5_THREADS = (V5_SOFT + 2) * 32;
constexpr int V5_LOAD = V5_SOFT, V5_MMA = V5_SOFT + 1;

template <int D>
struct Smem5 {
  static constexpr int KST = 8;                 // K slots (4 pairs)
  static constexpr int VST = 6;                 // V^T slots
  static constexpr int Q_BYTES = BQ * D;
  static constexpr int K_BYTES = BK * D;
  static constexpr int V_BYTES = D * BK * 2;
  static constexpr int CA_BYTES = BQ * 16 * 2;  // bias MMA A: 128 x 16 bf16 ones
  static constexpr int CB_BYTES = 2 * BK * 16 * 2;   // bias MMA B: 128 x 16 bf16 1.5*2^19
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + KST * K_BYTES;
  static constexpr int OFF_CA = OFF_V + VST * V_BYTES;
  static constexpr int OFF_CB = OFF_CA + CA_BYTES;
  static constexpr int OFF_XM = OFF_CB + CB_BYTES;            // float [2 bufs][2 halves][128 rows]
  static constexpr int OFF_XL = OFF_XM + 2 * 2 * BQ * 4;      // float [2][128]: half-1 partial l, total l
  static constexpr int OFF_BAR = OFF_XL + 2 * BQ * 4;
  // q_full, k_full[KST], k_empty[KST/2], v_full[VST], v_empty[VST], s_full[2], p_full[2], o_done[2]
  static constexpr int N_BARS = 1 + KST + KST / 2 + 2 * VST + 6;
  static constexpr int OFF_MISC = OFF_BAR + N_BARS * 8;      // [0] TMEM base, [1..16] pv flags [2][2][4]
  static constexpr int TOTAL = OFF_MISC + 128;
  static constexpr int BYTES = (TOTAL + 1023) / 1024 * 1024;
  static_assert(BYTES + 1024 <= 227 * 1024, "one CTA per SM");
};

template <int D, bool CAUSAL, bool F16>
__global__ void __launch_bounds__(V5_THREADS, 1)
k_sparse_attn_v5(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using L = Smem5<D>;
  constexpr int KST = L::KST, VST = L::VST;
  constexpr float kRefThreshold = F16 ? kRescaleThresholdF16 : kRescaleThreshold;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
#ifdef SPARGE_CTA_TIMING
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    CTA_REC(0, gtimer());
    CTA_REC(4, smid);
  }
#endif
  const int warp = __shfl_sync(0xffffffffu, warp_id(), 0), lane = lane_id();
  // this CTA's work item from the launch order (k_order: longest first)
  const int item = __ldg(p.order + blockIdx.x);
  const int bhq = item / p.T_m, i = item - bhq * p.T_m;
  const int b = bhq / p.Hq, hq = bhq % p.Hq;
  const int bkv = b * p.Hkv + hq / p.group;
  const int64_t row_id = static_cast<int64_t>(bhq) * p.T_m + i;
  const int n_tiles = p.cnt[row_id];
  const int n_pairs = (n_tiles + 1) >> 1;
  const int32_t* lut_row = p.lut + row_id * p.T_n;

  int8_t* sQ = reinterpret_cast<int8_t*>(smem + L::OFF_Q);
  int8_t* sK = reinterpret_cast<int8_t*>(smem + L::OFF_K);
  unsigned char* sV = smem + L::OFF_V;
  float* xm = reinterpret_cast<float*>(smem + L::OFF_XM);
  float* xl = reinterpret_cast<float*>(smem + L::OFF_XL);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + KST;         // per slot PAIR
  uint64_t* v_full = k_empty + KST / 2;
  uint64_t* v_empty = v_full + VST;
  uint64_t* s_full = v_empty + VST;         // [2] QK of the pair done
  uint64_t* p_full = s_full + 2;            // [2] P~ of the pair in TMEM (8 softmax warps)
  uint64_t* o_done = p_full + 2;            // [2] P~V of the pair done
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_MISC);
  uint32_t* pv_flag = tmem_base_slot + 1;   // [2 bufs][2 tiles][4 quads]

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) mbar_init(k_full + s, 1);
    for (int s = 0; s < KST / 2; ++s) mbar_init(k_empty + s, 1);
    for (int s = 0; s < VST; ++s) { mbar_init(v_full + s, 1); mbar_init(v_empty + s, 1); }
    for (int s = 0; s < 2; ++s) {
      mbar_init(s_full + s, 1);
      mbar_init(p_full + s, V5_SOFT);
      mbar_init(o_done + s, 1);
    }
    fence_mbar_init();
  }
  {
    // constant operands of the bias MMA (every element equal, so the core
    // matrix layout of the descriptor is immaterial)
    constexpr uint32_t kOnes = kBf16One | (static_cast<uint32_t>(kBf16One) << 16);
    constexpr uint32_t kParts = kBf16MagicPart | (static_cast<uint32_t>(kBf16MagicPart) << 16);
    uint32_t* cw = reinterpret_cast<uint32_t*>(smem + L::OFF_CA);
    for (int x = threadIdx.x; x < (L::CA_BYTES + L::CB_BYTES) / 4; x += blockDim.x)
      cw[x] = x < L::CA_BYTES / 4 ? kOnes : kParts;
    fence_proxy_async_smem();
  }
  if (warp == V5_MMA) tmem_alloc<512>(tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  const uint32_t tO = tmem_base + 4 * BK;    // after SP[0], SP[1]

  if (warp == V5_LOAD) {
    // ============================ TMA producer ============================
    if (lane == 0 && n_tiles > 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_arrive_expect_tx(q_full, L::Q_BYTES);
      tma_load_3d(sQ, &tmQ, q_full, 0, i * BQ, bhq);
      int j_next = __ldg(lut_row);
      for (int t = 0; t < n_tiles; ++t) {
        const int j = j_next;
        if (t + 1 < n_tiles) j_next = __ldg(lut_row + t + 1);
        const int ks = t % KST;
        if ((t & 1) == 0) mbar_wait(k_empty + (ks >> 1), ((t / KST) & 1) ^ 1);
        mbar_arrive_expect_tx(k_full + ks, L::K_BYTES);
        tma_load_3d(sK + ks * L::K_BYTES, &tmK, k_full + ks, 0, j * BK, bkv);
        const int vs = t % VST;
        mbar_wait(v_empty + vs, ((t / VST) & 1) ^ 1);
        mbar_arrive_expect_tx(v_full + vs, L::V_BYTES);
        tma_load_3d(sV + vs * L::V_BYTES, &tmV, v_full + vs, j * BK, 0, bkv);
      }
    }
  } else if (warp == V5_MMA) {
    // ============================ MMA issuer ==============================
    if (lane == 0 && n_tiles > 0) {
      constexpr uint32_t IDESC_PV = F16 ? idesc_f16(BQ, D) : idesc_bf16(BQ, D);
      const uint64_t dQ = umma_desc_kmajor(smem_u32(sQ), D);
      const uint64_t dCA = umma_desc_noswz(smem_u32(smem + L::OFF_CA), 128, 256);
      const uint64_t dCB = umma_desc_noswz(smem_u32(smem + L::OFF_CB), 128, 256);
      unsigned long long issued = 0;
      mbar_wait(q_full, 0);
      tc_fence_after();
      // P~V of pair u (Alg. 1 l.15-16), per tile, skipped when all four gate
      // groups of the tile vote to skip
      auto do_pv = [&](int u) {
        const int ub = u & 1;
        mbar_wait(p_full + ub, (u >> 1) & 1);
        tc_fence_after();
        const int t0 = 2 * u;
        for (int h = 0; h < ((t0 + 1 < n_tiles) ? 2 : 1); ++h) {
          const int t = t0 + h;
          const int vs = t % VST;
          mbar_wait(v_full + vs, (t / VST) & 1);
          tc_fence_after();
          const uint32_t* fl = pv_flag + ub * 8 + h * 4;
          if ((fl[0] | fl[1] | fl[2] | fl[3]) != 0) {
            const uint32_t tP = tmem_base + ub * 2 * BK + h * BK;
            const uint64_t dV = umma_desc_kmajor(smem_u32(sV + vs * L::V_BYTES), 128);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              mma_f16_ts(tO, tP + 8 * kk, dV + 2 * kk, IDESC_PV, 1u);
            ++issued;
          }
          tc_commit(v_empty + vs);
        }
        tc_commit(o_done + ub);
      };
      for (int pp = 0; pp < n_pairs; ++pp) {
        const int sb = pp & 1;
        const int t0 = 2 * pp;
        const bool two = t0 + 1 < n_tiles;
        const int ks = t0 % KST;
        const uint32_t kpar = (t0 / KST) & 1;
        mbar_wait(k_full + ks, kpar);
        if (two) mbar_wait(k_full + ks + 1, kpar);
        // SP[sb] holds P~ of pair pp-2, read by its P~V MMAs, issued by this
        // thread before this QK (in-order tensor pipe)
        tc_fence_after();
        const uint32_t tS = tmem_base + sb * 2 * BK;
        const uint64_t dK = umma_desc_kmajor(smem_u32(sK + ks * L::K_BYTES), D);
        const uint32_t idesc_qk = two ? idesc_i8(BQ, 2 * BK) : idesc_i8(BQ, BK);
        mma_f16(tS, dCA, dCB, two ? idesc_bf16(BQ, 2 * BK) : idesc_bf16(BQ, BK), 0u);
#pragma unroll
        for (int kk = 0; kk < D / 32; ++kk) mma_i8(tS, dQ + 2 * kk, dK + 2 * kk, idesc_qk, 1u);
        tc_commit(s_full + sb);
        tc_commit(k_empty + (ks >> 1));
        if (pp > 0) do_pv(pp - 1);
      }
      do_pv(n_pairs - 1);
      if (p.counters) atomicAdd(p.counters + bhq * 3 + 2, issued);
    }
  } else {
    // ============================ softmax warps ===========================
    const int quad = warp & 3, half = warp >> 2;
    const int r = quad * 32 + lane;            // row within the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const int row_g = i * BQ + r;
    const bool row_valid = row_g < p.N;
    const bool tile_tail = (i * BQ + BQ > p.N);
    using SB = SBits<false, true>;
    constexpr int kMaskedBits = SB::kMasked;   // 0: bias-MMA fp32 bits
    {
      // O is zeroed by the half-0 warps (their rows), before any P~V
      if (half == 0) {
        uint32_t z[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) z[k] = 0u;
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) tmem_st32(tO + lane_base + cc * 32, z);
        tmem_wait_st();
      }
    }
    const float* dk_row = p.dk + static_cast<int64_t>(bkv) * p.T_n;
    const float dq_scale = __ldg(p.dq + row_id) * p.scale_log2;
    float m_true = -INFINITY, m_ref = -INFINITY, l = 0.f;   // l: this half's partial row sum
    unsigned int slices = 0;
    // Lane u caches j and c = dq*dk*log2e/sqrt(d) of this half's tile of pair
    // 32*chunk + u (tile 2*(32 chunk + u) + half); broadcast by shuffles.
    int cj = 0, nj = 0;
    float cc_ = 0.f, ndk = 0.f;
    if (2 * lane + half < n_tiles) {
      cj = __ldg(lut_row + 2 * lane + half);
      cc_ = dq_scale * __ldg(dk_row + cj);
    }
    const uint32_t nbar = 1 + quad;            // named barrier of warps quad, quad+4
#ifdef SPARGE_CTA_TIMING
    if (threadIdx.x == 0) { CTA_REC(1, gtimer()); CTA_REC(5, n_tiles); }
#endif
    for (int pp = 0; pp < n_pairs; ++pp) {
      const int sb = pp & 1;
      const int t = 2 * pp + half;             // this warp's tile
      const bool mine = t < n_tiles;
      const bool two = 2 * pp + 1 < n_tiles;
      const int tl = pp & 31;
      if (tl == 0) {
        if (pp > 0) { cj = nj; cc_ = dq_scale * ndk; }
        const int tn = 2 * (pp + 32 + lane) + half;
        if (tn < n_tiles) nj = __ldg(lut_row + tn);
      } else if (tl == 16) {
        const int tn = 2 * (pp + 16 + lane) + half;
        if (tn < n_tiles) ndk = __ldg(dk_row + nj);
      }
      const int j = __shfl_sync(0xffffffffu, cj, tl);
      const float c = __shfl_sync(0xffffffffu, cc_, tl);
      const uint32_t tS = tmem_base + sb * 2 * BK + half * BK + lane_base;

      mbar_wait(s_full + sb, (pp >> 1) & 1);
      tc_fence_after();
      int32_t a[BK];
      float m_mine = -INFINITY;
      bool need_mask = false;
      if (mine) {
        tmem_ld32(tS, reinterpret_cast<uint32_t*>(a));
        tmem_ld32(tS + 32, reinterpret_cast<uint32_t*>(a) + 32);
        tmem_wait_ld();
        // boundary tiles: keys >= N, causal keys > query, rows >= N
        const int k0 = j * BK;
        need_mask = tile_tail || (k0 + BK > p.N) || (CAUSAL && (k0 + BK - 1 > i * BQ));
        if (need_mask) {
          const int kmax = CAUSAL ? min(p.N - 1, row_g) : p.N - 1;
#pragma unroll
          for (int k = 0; k < BK; ++k)
            if (!row_valid || k0 + k > kmax) a[k] = kMaskedBits;
        }
        // integer-domain row max over the positive fp32 bits 1.5*2^23 + acc
        // (monotone in acc; c > 0), eight independent chains
        int m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = max(a[u], a[u + 8]);
#pragma unroll
        for (int k = 16; k < BK; k += 16)
#pragma unroll
          for (int u = 0; u < 8; ++u) m8[u] = max(m8[u], max(a[k + u], a[k + 8 + u]));
        const int mx = max(max(max(m8[0], m8[1]), max(m8[2], m8[3])),
                           max(max(m8[4], m8[5]), max(m8[6], m8[7])));
        if (mx != kMaskedBits) m_mine = (__int_as_float(mx) - kMagicF) * c;
      }
      // exchange the tile maxima of the pair with the partner warp
      xm[(sb * 2 + half) * BQ + r] = m_mine;
      named_bar_sync(nbar, 64);
      const float m_other = xm[(sb * 2 + (half ^ 1)) * BQ + r];
      const float mA = half == 0 ? m_mine : m_other;
      const float mB = half == 0 ? m_other : m_mine;
      // Alg. 1 l.14-15 for tile 2p, then tile 2p+1 (both warps, identically)
      const float mn0 = fmaxf(m_true, mA);
      const bool comp0 = __any_sync(0xffffffffu, (mA > -INFINITY) && (mA - mn0 > p.lam2));
      const float mn1 = fmaxf(mn0, mB);
      const bool comp1 = two && __any_sync(0xffffffffu, (mB > -INFINITY) && (mB - mn1 > p.lam2));
      // one reference for the pair (R22): it moves only when a computing tile
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
      const bool comp_mine = half == 0 ? comp0 : comp1;
      if (rescale_o && half == 0) {
        // O rows hold P~V of earlier pairs: wait for the last one (pp-1),
        // then rescale in TMEM before p_full releases this pair's P~V
        if (pp >= 1) mbar_wait(o_done + ((pp - 1) & 1), ((pp - 1) >> 1) & 1);
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
      if (mine) {
        // P~ = exp2(S*log2e - m_ref), row sum (R9: skipped groups still add
        // their mass), 16-bit P~ over the first 32 columns of this tile
        uint32_t pw[BK / 2];
        float rsum;
        if (need_mask) exps64<true, F16, false, false, true>(a, c, m_ref, pw, rsum);
        else exps64<false, F16, false, false, true>(a, c, m_ref, pw, rsum);
        l += rsum;
        if (!comp_mine) {
#pragma unroll
          for (int k = 0; k < BK / 2; ++k) pw[k] = 0u;
        }
        tmem_st32(tS, pw);
        tmem_wait_st();
        if (comp_mine) ++slices;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (mine)
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(pv_flag + sb * 8 + half * 4 + quad)),
                       "r"(comp_mine ? 1u : 0u) : "memory");
        mbar_arrive(p_full + sb);
      }
    }
#ifdef SPARGE_CTA_TIMING
    if (threadIdx.x == 0) CTA_REC(2, gtimer());
#endif
    // ---- epilogue: O_i = O / l (line 19), scattered back through perm ----
    // l = the two halves' partial sums; warp quad+4*half writes columns
    // [half*D/2, (half+1)*D/2) of its rows
    if (half == 1) xl[r] = l;                  // partial sum of half 1
    named_bar_sync(nbar, 64);
    if (half == 0) xl[BQ + r] = l + xl[r];     // total
    named_bar_sync(nbar, 64);
    const float lt = xl[BQ + r];
    if (n_tiles > 0) mbar_wait(o_done + ((n_pairs - 1) & 1), ((n_pairs - 1) >> 1) & 1);
    tc_fence_after();
    if (half == 0 && row_valid && !(lt > 0.f)) atomicOr(p.status, 1u);
    const float inv_l = (lt > 0.f) ? 1.f / lt : 0.f;
    const int dst_row = row_valid ? (p.perm ? __ldg(p.perm + row_g) : row_g) : 0;
    uint16_t* orow = p.o + b * p.o_sb + hq * p.o_sh + static_cast<int64_t>(dst_row) * p.o_sn;
#pragma unroll
    for (int cq = 0; cq < D / 64; ++cq) {
      const int cc = half * (D / 64) + cq;     // 32-column chunk
      uint32_t ov[32];
      tmem_ld32(tO + lane_base + cc * 32, ov);
      tmem_wait_ld();
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
      if (warp == 0 && lane == 0)
        atomicAdd(p.counters + bhq * 3 + 0, static_cast<unsigned long long>(n_tiles));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == V5_MMA) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
#ifdef SPARGE_CTA_TIMING
  if (threadIdx.x == 0) CTA_REC(3, gtimer());
#endif
}

template <int D, bool CAUSAL, bool F16>
cudaError_t launch_t5(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                      const AttnParams& p, int B, cudaStream_t stream) {
  auto kern = k_sparse_attn_v5<D, CAUSAL, F16>;
  const int smem = Smem5<D>::BYTES + 1024;   // + slack for 1024-B alignment
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(p.T_m * B * p.Hq), V5_THREADS, smem, stream>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

