// Stage 1 of Algorithm 1 -- step a2 of the hot path.
//
//   S^[i,j] = q_i . k_j / sqrt(d)                 Alg. 1 line 5, R2
//   S^[i,j] = -inf if s_kj < theta (strict, R5) or tile (i,j) causally dead (R8)
//   P^[i]  = softmax(S^[i])                       line 6
//   M[i,:] = TopCdf(P^[i], tau)                   §3.2 pseudocode, R4:
//       order (P^ desc, j asc); keep rank k iff cumsum_k <= tau*c_last;
//       always keep rank 0 (guard)
//   M[i,:] = 1 if s_qi < theta; M[:,j] = 1 if s_kj < theta    Eq. 5
//   all -inf row -> all ones (R7); causal: M &= live, M[i, i*bq/bk] = 1 (R8)
// plus the compaction of the kept j (ascending) into the LUT the attention
// kernel walks.  Everything is fp64 (R15).
//
// k_shat_dmma   S^ = Q^-bar K^-bar^T / sqrt(d) per head on the fp64 tensor
//               cores (mma.sync m8n8k4 f64, DMMA): 64 query blocks x 64 key
//               blocks per CTA staged in shared memory (rows padded to d+4
//               doubles: the A/B fragment loads are bank-conflict free), one
//               8-row strip per warp; written to the workspace with -inf in
//               the fixed K columns (s_kj < theta), so the TopCdf kernels
//               bulk-copy a row into shared memory and read the forced
//               columns back from it (no per-row k_sim reads).
// k_topcdf_rows one warp per (head, query block): masks, softmax, the
//               sort-free binned TopCdf selection (topcdf_binned: fixed-point
//               integer bin masses, only the boundary bin sorted), forcing,
//               causal AND + guard, ballot compaction into the LUT.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cfloat>

#include "sm100.cuh"
#include "sparge_internal.h"

namespace sparge {

namespace {

// ---------------------------------------------------------------- S^ GEMM
// v2 (round 2): 64 query blocks x 64 key blocks per CTA, the d axis staged in
// chunks of kKC doubles through a double-buffered cp.async ring (loads of
// chunk c+1 overlap the DMMAs of chunk c; 37 KB per stage, so several CTAs
// share an SM -- v1 staged all of d at once, 135 KB, one CTA per SM, and the
// SM idled during every load: 25 % occupancy, ncu r02_pred128k); 8 warps,
// each a 16-row x 32-key register tile (2 x 4 DMMA fragments per k-step:
// 6 fragment loads per 8 DMMAs).  SPARGE_SHAT_TN (A/B knob) widens or
// narrows the CTA's key tile: 128 (2 CTAs/SM) and 32 (4 CTAs/SM) measured
// 4 % / 2 % slower at 128K (profiles/r02/r02_s8_shat_tile_ab.txt).
#ifndef SPARGE_SHAT_TN
#define SPARGE_SHAT_TN 64
#endif
constexpr int kTile = 64;          // query blocks per CTA
constexpr int kTileN = SPARGE_SHAT_TN;   // key blocks per CTA
constexpr int kFragN = kTileN / 16;      // 8-key fragments per warp (two key halves)
constexpr int kKC = 32;            // d chunk (doubles) per stage
constexpr int kKR = kKC + 4;       // padded chunk row: kKR % 16 == 4 (conflict-free fragments)
constexpr int kGemmThreads = 256;
constexpr size_t kGemmSmem = sizeof(double) * 2 /*stages*/ * (kTile + kTileN) * kKR;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
               ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int D>
__global__ void __launch_bounds__(kGemmThreads)
k_shat_dmma(const double* __restrict__ q_pooled, const double* __restrict__ k_pooled,
            const double* __restrict__ k_sim, double theta,
            int Hq, int Hkv, int T_m, int T_n, int N, int bq, int bk, int causal,
            double* __restrict__ shat) {
  constexpr int NCH = D / kKC;
  extern __shared__ __align__(16) unsigned char smem[];
  double* stage = reinterpret_cast<double*>(smem);       // [2][kTile + kTileN][kKR]
  const int j0 = blockIdx.x * kTileN, i0 = blockIdx.y * kTile, bhq = blockIdx.z;
  // causal: a tile whose every key block is dead for every query block of
  // the tile (R8-i) is never read by k_topcdf_rows -- skip it
  if (causal && j0 * bk > min((min(i0 + kTile, T_m)) * bq, N) - 1) return;
  griddep_wait();      // PDL (sparge_internal.h)
  griddep_launch();
  const int hq = bhq % Hq, b = bhq / Hq;
  const int hkv = hq / (Hq / Hkv);
  const int64_t qbase = static_cast<int64_t>(bhq) * T_m;
  const int64_t kbase = (static_cast<int64_t>(b) * Hkv + hkv) * T_n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  // chunk c of 64 pooled-Q rows and 64 pooled-K rows (zero beyond T_m / T_n)
  auto issue = [&](int c, int buf) {
    double* sq = stage + buf * (kTile + kTileN) * kKR;
    double* sk = sq + kTile * kKR;
    constexpr int CH = kKC / 2;      // 16-B pieces per chunk row
    for (int e = tid; e < (kTile + kTileN) * CH; e += kGemmThreads) {
      const int which = e >= kTile * CH;
      const int rr = which ? e / CH - kTile : e / CH, cc = e % CH;
      double* dst = (which ? sk : sq) + rr * kKR + 2 * cc;
      const bool ok = which ? (j0 + rr < T_n) : (i0 + rr < T_m);
      if (ok) {
        const double* src = which ? k_pooled + (kbase + j0 + rr) * D + c * kKC + 2 * cc
                                  : q_pooled + (qbase + i0 + rr) * D + c * kKC + 2 * cc;
        cp_async16(dst, src);
      } else {
        dst[0] = 0.0;
        dst[1] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // warp w: rows 16*(w%4)..+15 (two 8-row fragments) x keys 32*(w/4)..+31
  // (four 8-key fragments); fragments (m8n8k4, f64): A row = lane/4,
  // k = lane%4; B k = lane%4, n = lane/4; C row = lane/4, cols 2*(lane%4)+{0,1}
  const int rs = wid & 3, kh = wid >> 2;
  const int g = lane >> 2, t4 = lane & 3;
  double acc[2][kFragN][2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int kt = 0; kt < kFragN; ++kt) acc[r][kt][0] = acc[r][kt][1] = 0.0;

  issue(0, 0);
  for (int c = 0; c < NCH; ++c) {
    if (c + 1 < NCH) {
      issue(c + 1, (c + 1) & 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* sq = stage + (c & 1) * (kTile + kTileN) * kKR;
    const double* sk = sq + kTile * kKR;
    const double* a0 = sq + (16 * rs + g) * kKR + t4;
    const double* b0 = sk + (8 * kFragN * kh + g) * kKR + t4;
#pragma unroll
    for (int ks = 0; ks < kKC / 4; ++ks) {
      const double a_lo = a0[4 * ks], a_hi = a0[8 * kKR + 4 * ks];
#pragma unroll
      for (int kt = 0; kt < kFragN; ++kt) {
        const double bv = b0[8 * kt * kKR + 4 * ks];
        dmma_884(acc[0][kt][0], acc[0][kt][1], a_lo, bv);
        dmma_884(acc[1][kt][0], acc[1][kt][1], a_hi, bv);
      }
    }
    __syncthreads();          // the buffer is refilled two chunks later
  }
  // epilogue: S^ / sqrt(d), and -inf in the columns of the fixed K blocks
  // (s_kj < theta, strict, R5) -- the TopCdf kernels read the forced
  // columns back as the -inf entries of a live column (a finite q.k never is
  // -inf), so they need not re-read k_sim for every row.  Pairs of keys as one
  // 16-B store when the row offset is even (T_n even).
  const double inv_sqrt_d = 1.0 / sqrt(static_cast<double>(D));
  bool fk[kFragN][2];
#pragma unroll
  for (int kt = 0; kt < kFragN; ++kt) {
    const int key = j0 + 8 * kFragN * kh + 8 * kt + 2 * t4;
    fk[kt][0] = key < T_n && __ldg(k_sim + kbase + key) < theta;
    fk[kt][1] = key + 1 < T_n && __ldg(k_sim + kbase + key + 1) < theta;
  }
  const bool pair_ok = (T_n & 1) == 0;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = i0 + 16 * rs + 8 * r + g;
    if (row >= T_m) continue;
    double* out = shat + (qbase + row) * T_n;
#pragma unroll
    for (int kt = 0; kt < kFragN; ++kt) {
      const int key = j0 + 8 * kFragN * kh + 8 * kt + 2 * t4;
      const double v0 = fk[kt][0] ? -INFINITY : acc[r][kt][0] * inv_sqrt_d;
      const double v1 = fk[kt][1] ? -INFINITY : acc[r][kt][1] * inv_sqrt_d;
      if (pair_ok && key + 1 < T_n) {
        *reinterpret_cast<double2*>(out + key) = make_double2(v0, v1);
      } else {
        if (key < T_n) out[key] = v0;
        if (key + 1 < T_n) out[key + 1] = v1;
      }
    }
  }
}

// e^x for x <= 0 in fp64 without the library's special-case paths: 2^t,
// t = x log2(e), split t = n + f (n = rint t by the 1.5 * 2^52 trick,
// |f| <= 1/2), 2^f by its degree-12 Taylor polynomial in f (relative error
// < 5e-16 on [-1/2, 1/2]), 2^n added into the exponent; e^x < 2^-1000 -> 0
// (such an entry carries no P^ mass at fp64 resolution).  Relative error
// ~|t| 2^-53 from rounding t: < 1e-13 for |t| < 1000, far below the 1e-6
// near-threshold band (R4, R15).
__device__ __forceinline__ double exp_nonpos(double x) {
  const double t = x * 1.4426950408889634;
  if (!(t > -1000.0)) return 0.0;
  const double r = t + 6755399441055744.0;            // 1.5 * 2^52: rounds t to an integer
  const int n = static_cast<int>(__double2loint(r));  // low word = n (two's complement)
  const double f = t - (r - 6755399441055744.0);
  double p = 2.5678435993488196e-11;
  p = fma(p, f, 4.44553827187081e-10);
  p = fma(p, f, 7.054911620801121e-09);
  p = fma(p, f, 1.0178086009239696e-07);
  p = fma(p, f, 1.3215486790144305e-06);
  p = fma(p, f, 1.5252733804059838e-05);
  p = fma(p, f, 0.00015403530393381606);
  p = fma(p, f, 0.0013333558146428441);
  p = fma(p, f, 0.009618129107628477);
  p = fma(p, f, 0.055504108664821576);
  p = fma(p, f, 0.2402265069591007);
  p = fma(p, f, 0.6931471805599453);
  p = fma(p, f, 1.0);
  return __hiloint2double(__double2hiint(p) + (n << 20), __double2loint(p));
}

// ---------------------------------------------------------------- TopCdf rows
// k_topcdf_rows: up to kMaxRowWarps rows (one warp each) per CTA, each warp
// holding its row in shared memory: pow2ceil(T_n) 64-bit keys (the boundary
// bin is sorted in place by a power-of-two bitonic sort), T_n flags and the
// bin sums.  T_n <= kMaxTn (N <= 2^20 tokens) keeps one row within a CTA's
// shared memory; the key's low kIdxBits mantissa bits carry the index.
constexpr int kMaxRowWarps = 4;
constexpr int kIdxBits = 16;
constexpr uint64_t kIdxMask = (1ull << kIdxBits) - 1;
constexpr size_t kRowSmemMax = 200 * 1024;
// rows longer than this use k_topcdf_cta (env SPARGE_TOPCDF_CTA_MIN_TN
// overrides for A/B runs; default measured on B200)
int cta_row_min_tn() {
  static const int v = [] {
    const char* e = std::getenv("SPARGE_TOPCDF_CTA_MIN_TN");
    return e ? std::atoi(e) : 1024;
  }();
  return v;
}
// first-level bins: 32 binades below the row max x SUB mantissa sub-bins
// (the last bin is the catch-all for entries >= 31 binades down), 256 bins
// (SUB 8); 1024 bins (SUB 32) measured slower in the CTA kernel (the bin
// clearing and scan outweigh the smaller boundary sort)
constexpr int kNB = 256;
constexpr int kNBCta = 256;
__host__ __device__ inline int pow2ceil(int n) {
  int p = 32;
  while (p < n) p <<= 1;
  return p;
}
// bin masses: three 32-bit partial sums per bin (bits 0-16, 17-33, 34-) of
// the fixed-point masses, so each entry is three native shared-memory atomic
// adds (a 64-bit shared atomicAdd is a CAS loop on sm_100: ATOMS.CAST.SPIN.64,
// 20 % of the r02 TopCdf instructions); q < 2^51 per entry and T_n <= 2^14
// keep every partial sum below 2^32
__host__ __device__ inline size_t bins_bytes(int nb) { return static_cast<size_t>(nb) * 12; }
__device__ __forceinline__ void bin_add(uint32_t* c, int nb, int b, unsigned long long q) {
  atomicAdd(c + b, static_cast<uint32_t>(q & 0x1FFFFu));
  atomicAdd(c + nb + b, static_cast<uint32_t>((q >> 17) & 0x1FFFFu));
  atomicAdd(c + 2 * nb + b, static_cast<uint32_t>(q >> 34));
}
__device__ __forceinline__ unsigned long long bin_mass(const uint32_t* c, int nb, int b) {
  return static_cast<unsigned long long>(c[b]) + (static_cast<unsigned long long>(c[nb + b]) << 17) +
         (static_cast<unsigned long long>(c[2 * nb + b]) << 34);
}
// per row: pow2ceil(T_n) keys, the bins, T_n flags, the forced-column bits
__host__ __device__ inline size_t forced_bytes(int T_n) { return static_cast<size_t>((T_n + 127) / 128) * 16; }
__host__ __device__ inline size_t row_smem_bytes(int T_n) {
  return static_cast<size_t>(pow2ceil(T_n)) * 8 + 16 * kNB + ((T_n + 15) / 16) * 16 +
         forced_bytes(T_n);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Warp-synchronous bitonic sort, descending, of n (a power of two) 64-bit
// keys in shared memory, runtime n.
__device__ __forceinline__ void sort_desc_n(uint64_t* key, int n, int lane) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = lane; t < n / 2; t += 32) {
        const int a = t + (t & ~(jj - 1));
        const int c = a + jj;
        const uint64_t ka = key[a], kc = key[c];
        const bool desc_block = (a & k) == 0;
        const bool sw = desc_block ? (kc > ka) : (ka > kc);
        key[a] = sw ? kc : ka;
        key[c] = sw ? ka : kc;
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// TopCdf selection without a full sort (v4).  Keys as in the sort path
// (truncated P^ bits | kIdxMask - j).  The selected set is a prefix of the
// descending order, so only the entries of the BOUNDARY bin need ordering:
//   * P^ (here e = exp(S^ - max), the unnormalised P^) is put in fixed
//     point, q_j = floor(e_j * 2^s) (fixed_point_scale: the sum < 2^64):
//     integer sums are exact and order-free, so
//     the result is deterministic and equals the sequential fp64 cumsum up
//     to ~2^-52 relative (inside the 1e-6 near-threshold band);
//   * bins by (binade below the max, top 3 mantissa bits): NB = 256 bins in
//     descending key order, counts and integer mass per bin;
//   * the boundary bin b* = the first whose cumulative mass exceeds
//     tau * total; bins before it are selected, bins after it are not, and
//     the entries of b* are sorted and scanned from the mass above it.
// tau >= 1 selects everything (c_k <= c_last for every k, R4).  Rank 0 is
// always selected (guard).  ukey: the keys, entry j at ukey[j] (room for
// pow2ceil(T_n) keys), overwritten: the boundary bin is compacted in place to
// ukey[0, m) and sorted there; bsum: NB bin sums; flag: [T_n].
template <int NB, int SUB = 8>
__device__ __forceinline__ int bin_of(uint64_t key, int emax) {
  constexpr int SB = SUB == 8 ? 3 : 5, NBIN = NB / SUB;   // binades covered
  const int e = static_cast<int>(key >> 52) & 0x7FF;
  const int db = emax - e;
  if (db >= NBIN) return NB - 1;
  return db * SUB + (SUB - 1 - static_cast<int>((key >> (52 - SB)) & (SUB - 1)));
}
// q_j = floor(e_j 2^sc): the largest entry (e_max = 1, emax its exponent)
// lands in [2^50, 2^51) unless T_n * 2^51 could overflow the 64-bit sum,
// then sc drops to 63 - ceil(log2 T_n) (T_n <= 2^14: sc >= 49; entries below
// 2^-sc of the max become 0 -- a cumulative error <= T_n 2^-sc, far inside
// the 1e-6 band)
__device__ __forceinline__ int fixed_point_scale(int emax, int T_n) {
  const int lg = T_n > 1 ? 32 - __clz(T_n - 1) : 0;     // ceil(log2 T_n)
  return min(50 - (emax - 1023), 63 - lg);
}
// The boundary bin over NB bins (warp-parallel, NB/32 bins per lane in
// order): the first bin whose cumulative mass exceeds thr, and the mass of
// the bins before it; NB when none does.
template <int NB>
__device__ __forceinline__ int boundary_bin(const uint32_t* c, double thr, int lane,
                                            unsigned long long& a_star) {
  constexpr int PER = NB / 32;
  unsigned long long lsum = 0;
#pragma unroll 8
  for (int u = 0; u < PER; ++u) lsum += bin_mass(c, NB, lane * PER + u);
  unsigned long long incl = lsum;
#pragma unroll 8
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  unsigned long long above = incl - lsum;   // mass of the bins before this lane's first
  int bstar = NB;
  unsigned long long as = 0;
#pragma unroll 8
  for (int u = 0; u < PER; ++u) {
    const int b = lane * PER + u;
    const unsigned long long nxt = above + bin_mass(c, NB, b);
    if (bstar == NB && static_cast<double>(nxt) > thr) { bstar = b; as = above; }
    above = nxt;
  }
  int bmin = bstar;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
  const unsigned int owner = __ballot_sync(0xffffffffu, bstar == bmin && bmin < NB);
  a_star = (bmin < NB) ? __shfl_sync(0xffffffffu, as, __ffs(owner) - 1) : 0ull;
  return bmin;
}
// descending bitonic sort of one 64-bit key per lane across a warp
__device__ __forceinline__ uint64_t warp_sort_desc(uint64_t k, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int st = size >> 1; st > 0; st >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, k, st);
      const bool desc = ((lane & size) == 0);      // this lane's block sorts descending
      const bool lower = ((lane & st) == 0);
      // keep the larger on the lower lane of a descending block
      const bool take_max = (desc == lower);
      k = take_max ? max(k, o) : min(k, o);
    }
  }
  return k;
}

__device__ void topcdf_binned(uint64_t* ukey, uint32_t* bins, uint8_t* flag, int T_n,
                              double tau, int lane) {
  auto kix = [](int j) { return j; };
  uint64_t* list = ukey;
  // max key -> its exponent; fixed-point scale
  uint64_t kmax = 0;
  for (int j = lane; j < T_n; j += 32) kmax = max(kmax, ukey[kix(j)]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  const int emax = static_cast<int>(kmax >> 52) & 0x7FF;
  const int sc = fixed_point_scale(emax, T_n);
  for (int b = lane; b < 3 * kNB; b += 32) bins[b] = 0u;
  __syncwarp();
  // the catch-all bin (>= 32 binades below the max: most entries of a
  // peaked row) is summed in registers -- 32-way atomic conflicts otherwise
  const double scale = ldexp(1.0, sc);
  unsigned long long part = 0, q_last = 0;
  for (int j = lane; j < T_n; j += 32) {
    const uint64_t k = ukey[kix(j)];
    const unsigned long long qj = __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale);
    const int b = bin_of<kNB>(k, emax);
    if (b == kNB - 1) q_last += qj;
    else if (qj) bin_add(bins, kNB, b, qj);
    part += qj;
  }
  const unsigned long long total = warp_sum_u64(part);
  q_last = warp_sum_u64(q_last);
  __syncwarp();
  if (lane == 0) bin_add(bins, kNB, kNB - 1, q_last);
  __syncwarp();
  const double thr = (tau >= 1.0) ? INFINITY : tau * static_cast<double>(total);
  unsigned long long a_star;
  const int bmin = boundary_bin<kNB>(bins, thr, lane, a_star);
  // flags outside the boundary bin; compact the boundary bin's keys in place
  // (write index m + rank <= j0 + lane <= kix(j0 + lane): never ahead of an
  // unread key, and the reads of a chunk precede its writes)
  int m = 0;
  for (int j0 = 0; j0 < T_n; j0 += 32) {
    const int j = j0 + lane;
    const uint64_t k = (j < T_n) ? ukey[kix(j)] : 0ull;
    const int b = (j < T_n) ? bin_of<kNB>(k, emax) : kNB;
    const bool inb = (j < T_n) && (b == bmin);
    if (j < T_n) flag[j] = (b < bmin) ? 1 : 0;
    const unsigned int bal = __ballot_sync(0xffffffffu, inb);
    __syncwarp();
    if (inb) list[m + __popc(bal & ((1u << lane) - 1u))] = k;
    m += __popc(bal);
    __syncwarp();
  }
  // radix refinement of the boundary bin by 8 key bits per level (ordered
  // in-place compaction of the crossing sub-bin) down to <= 32 entries
  unsigned long long above = a_star;
  int shift = 52 - 3 - 8;                       // key bits 48..41 first
  int bcur = bmin;
  while (bcur < kNB && m > 32 && shift >= 0) {
    for (int b = lane; b < 4 * kNB; b += 32) bins[b] = 0u;
    __syncwarp();
    for (int t = lane; t < m; t += 32) {
      const uint64_t k = list[t];
      const int d = 255 - static_cast<int>((k >> shift) & 255u);
      const unsigned long long q = __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale);
      if (q) bin_add(bins, kNB, d, q);
      atomicAdd(bins + 3 * kNB + d, 1u);
    }
    __syncwarp();
    unsigned long long as;
    bcur = boundary_bin<kNB>(bins, thr - static_cast<double>(above), lane, as);
    above += as;
    int mm = 0;
    for (int t0 = 0; t0 < m; t0 += 32) {
      const int t = t0 + lane;
      const uint64_t k = (t < m) ? list[t] : 0ull;
      const int d = 255 - static_cast<int>((k >> shift) & 255u);
      if (t < m) flag[kIdxMask - static_cast<int>(k & kIdxMask)] = (d < bcur) ? 1 : 0;
      const bool inb = (t < m) && (d == bcur);
      const unsigned int bal = __ballot_sync(0xffffffffu, inb);
      __syncwarp();
      if (inb) list[mm + __popc(bal & ((1u << lane) - 1u))] = k;
      mm += __popc(bal);
      __syncwarp();
    }
    m = mm;
    shift -= 8;
  }
  if (bcur < kNB && m <= 32) {
    // <= 32 boundary entries: order in registers, scan from `above`
    uint64_t k = (lane < m) ? list[lane] : 0ull;
    k = warp_sort_desc(k, lane);
    unsigned long long qv =
        (lane < m) ? __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale) : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, qv, o);
      if (lane >= o) qv += y;
    }
    __syncwarp();
    if (lane < m)
      flag[kIdxMask - static_cast<int>(k & kIdxMask)] = (static_cast<double>(above + qv) <= thr) ? 1 : 0;
  } else if (bcur < kNB) {
    int n2 = 2;
    while (n2 < m) n2 <<= 1;
    for (int t = m + lane; t < n2; t += 32) list[t] = 0ull;
    __syncwarp();
    sort_desc_n(list, n2, lane);
    // sequential scan of the bin (in chunks of 32, integer prefix sums)
    unsigned long long carry = above;
    for (int t0 = 0; t0 < m; t0 += 32) {
      const int t = t0 + lane;
      const uint64_t k = (t < m) ? list[t] : 0ull;
      unsigned long long qv =
          (t < m) ? __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale) : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, qv, o);
        if (lane >= o) qv += y;
      }
      const unsigned long long c = carry + qv;
      if (t < m) flag[kIdxMask - static_cast<int>(k & kIdxMask)] = (static_cast<double>(c) <= thr) ? 1 : 0;
      carry = __shfl_sync(0xffffffffu, c, 31);
    }
  }
  __syncwarp();
  // guard: the top entry
  if (lane == 0) flag[kIdxMask - static_cast<int>(kmax & kIdxMask)] = 1;
  __syncwarp();
}

template <int D>
__global__ void __launch_bounds__(kMaxRowWarps * 32)
k_topcdf_rows(const double* __restrict__ shat, const double* __restrict__ q_sim,
              int Hq, int Hkv, int N, int T_m, int T_n,
              int rows_total, int bq, int bk, int causal, double tau, double theta,
              uint8_t* __restrict__ mask, int32_t* __restrict__ lut, int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int row_warps = blockDim.x >> 5;
  const int row = blockIdx.x * row_warps + wid;          // (b*Hq + hq)*T_m + i
  griddep_wait();      // PDL (sparge_internal.h)
  griddep_launch();
  if (row >= rows_total) return;
  // per warp: T_n keys (8 B), T_n flags, kNB bin sums (8 B)
  const size_t per_warp = row_smem_bytes(T_n);
  unsigned char* base_w = smem + wid * per_warp;
  uint64_t* ukey = reinterpret_cast<uint64_t*>(base_w);
  double* key = reinterpret_cast<double*>(ukey);
  const size_t nk = static_cast<size_t>(pow2ceil(T_n));
  uint32_t* bins = reinterpret_cast<uint32_t*>(base_w + nk * 8);         // [4][kNB]
  uint8_t* flag = base_w + nk * 8 + 16 * kNB;
  uint32_t* forced = reinterpret_cast<uint32_t*>(flag + ((T_n + 15) / 16) * 16);   // s_k < theta

  const int i = row % T_m;
  const int last_q = min((i + 1) * bq, N) - 1;
  // causal: key blocks j >= n_live are dead for this row (R8-i) -- never
  // loaded (k_shat_dmma does not compute tiles that are dead for a whole CTA)
  const int n_live = causal ? min(T_n, last_q / bk + 1) : T_n;
  const double* srow = shat + static_cast<int64_t>(row) * T_n;

  // ---- S^ row (k_shat_dmma already wrote -inf in the fixed K columns) ----
  // one bulk copy of the row's live entries into the key array (T_n even:
  // 16-B aligned rows), completing on this warp's mbarrier; entries j >=
  // n_live (causally dead, possibly never written) become -inf here.  A
  // forced column is a live -inf entry.
  __shared__ __align__(8) uint64_t s_bar[kMaxRowWarps];
  const bool bulk = (T_n & 1) == 0;
  if (bulk) {
    if (lane == 0) {
      mbar_init(s_bar + wid, 1);
      fence_mbar_init();
      const uint32_t bytes = static_cast<uint32_t>((n_live + 1) & ~1) * 8u;
      mbar_arrive_expect_tx(s_bar + wid, bytes);
      bulk_g2s(key, srow, bytes, s_bar + wid);
    }
    __syncwarp();
    mbar_wait(s_bar + wid, 0);
  }
  double mx = -INFINITY;
  for (int j0 = 0; j0 < T_n; j0 += 32) {                  // warp-uniform bound (ballots below)
    const int j = j0 + lane;
    double sv = -INFINITY;
    if (j < n_live) sv = bulk ? key[j] : __ldg(srow + j);
    const unsigned int fb = __ballot_sync(0xffffffffu, j < n_live && sv == -INFINITY);
    if (lane == 0) forced[j0 >> 5] = fb;
    if (j < T_n) {
      if (!bulk || j >= n_live) key[j] = sv;
      mx = fmax(mx, sv);
    }
  }
  mx = warp_max(mx);
  const bool flagged = (mx == -INFINITY);   // every K block fixed / dead (R7)

  if (!flagged) {
    // One 64-bit sort key per entry: the bits of e_j = exp(S^_j - max) (>= 0,
    // so integer order = value order) with the low kIdxBits mantissa bits
    // replaced by kIdxMask - j.  TopCdf's rule c_k <= tau c_last is
    // homogeneous, so selecting on e is selecting on P^ = e / sum(e) (R4):
    // the normalisation (a division per entry) is skipped.  Ordering the keys
    // descending orders (P^ desc, j asc) up to a 2^-36 relative truncation --
    // far inside the 1e-6 near-threshold band; the cumulative sums use the
    // truncated values.
    for (int j = lane; j < T_n; j += 32) {
      const double kv = key[j];
      const double e = (kv == -INFINITY) ? 0.0 : exp_nonpos(kv - mx);
      ukey[j] = (static_cast<uint64_t>(__double_as_longlong(e)) & ~kIdxMask) |
                static_cast<uint64_t>(kIdxMask - j);
    }
    __syncwarp();
    topcdf_binned(ukey, bins, flag, T_n, tau, lane);
  }

  // ---- forcing (Eq. 5), flagged rows, causal live AND + diagonal guard ----
  const bool row_fix = q_sim[row] < theta;
  const int guard = (i * bq) / bk;
  uint8_t* mrow = mask ? mask + static_cast<int64_t>(row) * T_n : nullptr;
  int32_t* lrow = lut + static_cast<int64_t>(row) * T_n;
  int base = 0;
  for (int j0 = 0; j0 < T_n; j0 += 32) {
    const int j = j0 + lane;
    bool f = false;
    if (j < T_n) {
      f = flagged ? true : (flag[j] != 0);
      if (row_fix || ((forced[j >> 5] >> (j & 31)) & 1u)) f = true;
      if (causal) {
        if (j >= n_live) f = false;
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

// ---------------------------------------------------------------- TopCdf, CTA per row
// The same selection as k_topcdf_rows with one CTA of kCtaWarps warps per
// row, for long rows (T_n large): a row's keys take pow2ceil(T_n) * 8 bytes of
// shared memory, so one warp per row left an SM with 8 warps at T_n = 2048
// (12.5 % occupancy, ncu r02_pred128k); a CTA per row keeps ~40 warps busy.
// Streaming phases split j across the warps; reductions go through shared
// memory in a fixed order (deterministic); the boundary bin (usually small)
// is compacted, sorted and scanned by warp 0.  The binning pass caches each
// entry's bin (u8), so the gather and mask passes decide "bin < b*" without
// the key; the boundary entries' decisions are bits set by the refinement.
constexpr int kCtaWarps = 4;
constexpr int kCtaThreads = kCtaWarps * 32;
#ifndef SPARGE_LISTCAP
#define SPARGE_LISTCAP 256
#endif
// boundary entries gathered outside the key array; a larger boundary bin
// falls back to in-place compaction + a warp-0 sort (rare).  256 keeps
// ~26 KB per CTA (8 CTAs/SM at T_n = 2048): 128K prediction 1.69 -> 1.55 ms
// vs 1024 (r02)
constexpr int kListCap = SPARGE_LISTCAP;

// keys, bins (3 mass chunks + a count per bin), two boundary lists, the
// entries' bin indices, forced-column bits, boundary-decision bits
__host__ __device__ inline size_t cta_row_smem_bytes(int T_n) {
  return static_cast<size_t>(pow2ceil(T_n)) * 8 + 4 * 4 * kNBCta + 2 * kListCap * 8 +
         ((T_n + 15) / 16) * 16 + 2 * forced_bytes(T_n);
}

__device__ __forceinline__ double block_max(double v, double* red) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int w = 1; w < kCtaWarps; ++w) r = fmax(r, red[w]);
  return r;
}
template <int D>
__global__ void __launch_bounds__(kCtaThreads)
k_topcdf_cta(const double* __restrict__ shat, const double* __restrict__ q_sim,
             int Hq, int Hkv, int N, int T_m, int T_n,
             int bq, int bk, int causal, double tau, double theta,
             uint8_t* __restrict__ mask, int32_t* __restrict__ lut, int32_t* __restrict__ cnt) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[kCtaWarps];
  __shared__ unsigned long long red_u[kCtaWarps];
  __shared__ int s_info[4];                 // bmin, m (boundary entries), refinement bin, count
  __shared__ unsigned long long s_astar;
  __shared__ int s_wcount[kCtaWarps];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int row = blockIdx.x;               // (b*Hq + hq)*T_m + i
  griddep_wait();      // PDL (sparge_internal.h)
  griddep_launch();
  uint64_t* ukey = reinterpret_cast<uint64_t*>(smem);
  double* key = reinterpret_cast<double*>(ukey);
  const size_t nk = static_cast<size_t>(pow2ceil(T_n));
  uint32_t* bins = reinterpret_cast<uint32_t*>(smem + nk * 8);           // [4][kNBCta]
  uint64_t* list = reinterpret_cast<uint64_t*>(smem + nk * 8 + 16 * kNBCta);
  uint64_t* list2 = list + kListCap;
  // bin of each entry (u8; kNBCta = 256 bins) -- pass 4 and the mask pass
  // read it instead of recomputing bin_of from the key
  uint8_t* ebin = smem + nk * 8 + 16 * kNBCta + 2 * kListCap * 8;
  uint32_t* forced = reinterpret_cast<uint32_t*>(ebin + ((T_n + 15) / 16) * 16);   // s_k < theta
  // kept bits of the boundary bin's entries (and the guard), set by the
  // refinement / final scan; every other entry is kept iff its bin < bmin
  uint32_t* dec = forced + forced_bytes(T_n) / 4;
  static_assert(kNBCta == 256, "bin indices stored as u8");

  const int i = row % T_m;
  const int last_q = min((i + 1) * bq, N) - 1;
  const int n_live = causal ? min(T_n, last_q / bk + 1) : T_n;
  const double* srow = shat + static_cast<int64_t>(row) * T_n;

  // ---- S^ row (k_shat_dmma already wrote -inf in the fixed K columns):
  // one bulk copy of the live entries into the key array (T_n even), as in
  // k_topcdf_rows; the bins are cleared while it lands ----
  __shared__ __align__(8) uint64_t s_bar;
  const bool bulk = (T_n & 1) == 0;
  if (bulk && tid == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
    const uint32_t bytes = static_cast<uint32_t>((n_live + 1) & ~1) * 8u;
    mbar_arrive_expect_tx(&s_bar, bytes);
    bulk_g2s(key, srow, bytes, &s_bar);
  }
  for (int t = tid; t < 3 * kNBCta; t += kCtaThreads) bins[t] = 0u;
  for (int t = tid; t < static_cast<int>(forced_bytes(T_n) / 4); t += kCtaThreads) dec[t] = 0u;
  __syncthreads();                           // s_bar initialised
  if (bulk) mbar_wait(&s_bar, 0);
  double mx = -INFINITY;
  for (int j0 = 0; j0 < T_n; j0 += kCtaThreads) {   // uniform bound (ballots)
    const int j = j0 + tid;
    double sv = -INFINITY;
    if (j < n_live) sv = bulk ? key[j] : __ldg(srow + j);
    const unsigned int fb = __ballot_sync(0xffffffffu, j < n_live && sv == -INFINITY);
    if (lane == 0 && j - lane < T_n) forced[(j - lane) >> 5] = fb;
    if (j < T_n) {
      if (!bulk || j >= n_live) key[j] = sv;
      mx = fmax(mx, sv);
    }
  }
  mx = block_max(mx, red);
  const bool flagged = (mx == -INFINITY);   // every K block fixed / dead (R7)
  int bmin = kNBCta;                         // entries of bins < bmin are kept
  auto keep_bit = [&](int j) { atomicOr(dec + (j >> 5), 1u << (j & 31)); };

  if (!flagged) {
    // keys (bits of e = exp(S^ - max), low kIdxBits replaced by kIdxMask - j;
    // unnormalised as in k_topcdf_rows) and the max key
    uint64_t kmax = 0;
    for (int j = tid; j < T_n; j += kCtaThreads) {
      const double kv = key[j];
      const double e = (kv == -INFINITY) ? 0.0 : exp_nonpos(kv - mx);
      const uint64_t k = (static_cast<uint64_t>(__double_as_longlong(e)) & ~kIdxMask) |
                         static_cast<uint64_t>(kIdxMask - j);
      ukey[j] = k;
      kmax = max(kmax, k);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    __syncthreads();
    if (lane == 0) red_u[wid] = kmax;
    __syncthreads();
    kmax = red_u[0];
#pragma unroll
    for (int w = 1; w < kCtaWarps; ++w) kmax = max(kmax, static_cast<uint64_t>(red_u[w]));
    const int emax = static_cast<int>(kmax >> 52) & 0x7FF;
    const int sc = fixed_point_scale(emax, T_n);
    const double scale = ldexp(1.0, sc);
    unsigned long long qpart = 0, q_last = 0;
    for (int j = tid; j < T_n; j += kCtaThreads) {
      const uint64_t k = ukey[j];
      const unsigned long long qj = __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale);
      const int bb = bin_of<kNBCta>(k, emax);
      ebin[j] = static_cast<uint8_t>(bb);
      if (bb == kNBCta - 1) q_last += qj;           // catch-all bin in registers
      else if (qj) bin_add(bins, kNBCta, bb, qj);
      qpart += qj;
    }
    qpart = warp_sum_u64(qpart);
    q_last = warp_sum_u64(q_last);
    if (lane == 0 && q_last) bin_add(bins, kNBCta, kNBCta - 1, q_last);
    __syncthreads();                                 // bins complete; red_u reuse
    if (lane == 0) red_u[wid] = qpart;
    __syncthreads();
    unsigned long long qtotal = 0;
#pragma unroll
    for (int w = 0; w < kCtaWarps; ++w) qtotal += red_u[w];
    const double thr = (tau >= 1.0) ? INFINITY : tau * static_cast<double>(qtotal);
    // boundary bin by warp 0 (lane-parallel prefix over the bins)
    if (wid == 0) {
      unsigned long long a_star;
      const int bmin = boundary_bin<kNBCta>(bins, thr, lane, a_star);
      if (lane == 0) {
        s_info[0] = bmin;
        s_info[1] = 0;
        s_astar = a_star;
      }
    }
    __syncthreads();
    bmin = s_info[0];
    // the boundary entries gathered into `list` (order irrelevant: sorted
    // below) while they fit kListCap; the other entries are decided by bin
    for (int j0 = wid * 32; j0 < T_n; j0 += kCtaThreads) {
      const int j = j0 + lane;
      const bool inb = (j < T_n) && (static_cast<int>(ebin[j]) == bmin);
      const unsigned int bal = __ballot_sync(0xffffffffu, inb);
      if (bal == 0u) continue;
      int base = 0;
      if (lane == 0) base = atomicAdd(&s_info[1], __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int pos = base + __popc(bal & ((1u << lane) - 1u));
      if (inb && pos < kListCap) list[pos] = ukey[j];
    }
    __syncthreads();
    int m = s_info[1];
    // radix refinement of the boundary bin (it fits the lists): histogram its
    // entries by the next 8 key bits, keep the sub-bins above the crossing
    // one, recurse into that sub-bin until <= 32 entries remain, which warp 0
    // orders in registers and scans (a large boundary bin -- a smooth P^
    // near the cut -- made the warp-0 bitonic sort the critical path)
    unsigned long long above = s_astar;
    uint64_t* la = list;
    uint64_t* lb = list2;
    int shift = 52 - 3 - 8;                     // key bits 48..41 first
    while (bmin < kNBCta && m > 32 && m <= kListCap && shift >= 0) {
      for (int t = tid; t < 4 * kNBCta; t += kCtaThreads) bins[t] = 0u;
      __syncthreads();
      for (int t = tid; t < m; t += kCtaThreads) {
        const uint64_t k = la[t];
        const int d = 255 - static_cast<int>((k >> shift) & 255u);
        const unsigned long long q = __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale);
        if (q) bin_add(bins, kNBCta, d, q);
        atomicAdd(bins + 3 * kNBCta + d, 1u);
      }
      __syncthreads();
      if (wid == 0) {
        unsigned long long as;
        const int b2 = boundary_bin<kNBCta>(bins, thr - static_cast<double>(above), lane, as);
        if (lane == 0) {
          s_info[2] = b2;
          s_info[3] = 0;
          s_astar = as;
        }
      }
      __syncthreads();
      const int b2 = s_info[2];
      above += s_astar;
      for (int t0 = wid * 32; t0 < m; t0 += kCtaThreads) {   // warp-aggregated gather
        const int t = t0 + lane;
        const uint64_t k = (t < m) ? la[t] : 0ull;
        const int d = 255 - static_cast<int>((k >> shift) & 255u);
        if (t < m && d < b2) keep_bit(kIdxMask - static_cast<int>(k & kIdxMask));
        const bool inb = (t < m) && (d == b2);
        const unsigned int bal = __ballot_sync(0xffffffffu, inb);
        int pos = 0;
        if (lane == 0 && bal) pos = atomicAdd(&s_info[3], __popc(bal));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (inb) lb[pos + __popc(bal & ((1u << lane) - 1u))] = k;
      }
      __syncthreads();
      m = s_info[3];
      uint64_t* tmp = la;
      la = lb;
      lb = tmp;
      shift -= 8;
      __syncthreads();                          // s_info / s_astar reuse
    }
    if (wid == 0 && bmin < kNBCta && m <= 32) {
      // <= 32 boundary entries: order in registers, scan from `above`
      uint64_t k = (lane < m) ? la[lane] : 0ull;
      k = warp_sort_desc(k, lane);
      unsigned long long qv =
          (lane < m) ? __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale) : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, qv, o);
        if (lane >= o) qv += y;
      }
      if (lane < m && static_cast<double>(above + qv) <= thr)
        keep_bit(kIdxMask - static_cast<int>(k & kIdxMask));
    } else if (wid == 0 && bmin < kNBCta) {
      const unsigned long long carry0 = above;
      uint64_t* lst = la;
      if (m > kListCap) {
        // rare (a huge boundary bin, e.g. near-uniform P^): warp 0 alone
        // compacts the bin in place in the key array, as topcdf_binned does
        lst = ukey;
        int mm = 0;
        for (int j0 = 0; j0 < T_n; j0 += 32) {
          const int j = j0 + lane;
          const uint64_t k = (j < T_n) ? ukey[j] : 0ull;
          const bool inb = (j < T_n) && (static_cast<int>(ebin[j]) == bmin);
          const unsigned int bal = __ballot_sync(0xffffffffu, inb);
          __syncwarp();
          if (inb) lst[mm + __popc(bal & ((1u << lane) - 1u))] = k;
          mm += __popc(bal);
          __syncwarp();
        }
      }
      int n2 = 2;
      while (n2 < m) n2 <<= 1;
      for (int t = m + lane; t < n2; t += 32) lst[t] = 0ull;
      __syncwarp();
      sort_desc_n(lst, n2, lane);
      unsigned long long carry = carry0;
      for (int t0 = 0; t0 < m; t0 += 32) {
        const int t = t0 + lane;
        const uint64_t k = (t < m) ? lst[t] : 0ull;
        unsigned long long qv =
            (t < m) ? __double2ull_rz(__longlong_as_double(k & ~kIdxMask) * scale) : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xffffffffu, qv, o);
          if (lane >= o) qv += y;
        }
        const unsigned long long c = carry + qv;
        if (t < m && static_cast<double>(c) <= thr) keep_bit(kIdxMask - static_cast<int>(k & kIdxMask));
        carry = __shfl_sync(0xffffffffu, c, 31);
      }
    }
    if (tid == 0) keep_bit(kIdxMask - static_cast<int>(kmax & kIdxMask));   // guard
  }
  __syncthreads();

  // ---- forcing (Eq. 5), flagged rows, causal live AND + diagonal guard;
  // LUT in ascending j: warp w owns the contiguous chunk [w*ch, (w+1)*ch) ----
  const bool row_fix = q_sim[row] < theta;
  const int guard = (i * bq) / bk;
  uint8_t* mrow = mask ? mask + static_cast<int64_t>(row) * T_n : nullptr;
  int32_t* lrow = lut + static_cast<int64_t>(row) * T_n;
  const int ch = ((T_n + kCtaWarps - 1) / kCtaWarps + 31) / 32 * 32;
  const int c0 = wid * ch, c1 = min(T_n, c0 + ch);
  auto kept = [&](int j) {
    bool f = flagged || static_cast<int>(ebin[j]) < bmin || ((dec[j >> 5] >> (j & 31)) & 1u);
    if (row_fix || ((forced[j >> 5] >> (j & 31)) & 1u)) f = true;
    if (causal) {
      if (j >= n_live) f = false;
      if (j == guard) f = true;
    }
    return f;
  };
  // pass 1: the kept bits of each 32-entry word (overwriting that word's
  // forced bits, already read by every lane before the ballot), the mask
  // and the warp's count; pass 2: the LUT from the words
  int wc = 0;
  for (int j0 = c0; j0 < c1; j0 += 32) {
    const int j = j0 + lane;
    const bool f = (j < c1) && kept(j);
    if (j < c1 && mrow) mrow[j] = f ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) forced[j0 >> 5] = bal;
    wc += __popc(bal);
  }
  if (lane == 0) s_wcount[wid] = wc;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < wid; ++w) base += s_wcount[w];
  for (int j0 = c0; j0 < c1; j0 += 32) {
    const unsigned bal = forced[j0 >> 5];
    if ((bal >> lane) & 1u) lrow[base + __popc(bal & ((1u << lane) - 1u))] = j0 + lane;
    base += __popc(bal);
  }
  if (tid == 0) {
    int total = 0;
    for (int w = 0; w < kCtaWarps; ++w) total += s_wcount[w];
    cnt[row] = total;
  }
}

template <int D>
cudaError_t launch_d(const sparge_shape& s, const double* q_pooled, const double* q_sim,
                     const double* k_pooled, const double* k_sim, float tau, float theta,
                     uint8_t* mask, int32_t* lut, int32_t* cnt, double* shat,
                     cudaStream_t stream) {
  const int T_m = (s.N + s.bq - 1) / s.bq;
  const int T_n = (s.N + s.bk - 1) / s.bk;
  const size_t smem_g = kGemmSmem;
  cudaError_t e = cudaFuncSetAttribute(k_shat_dmma<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_g));
  if (e != cudaSuccess) return e;
  dim3 g1((T_n + kTileN - 1) / kTileN, (T_m + kTile - 1) / kTile, s.B * s.Hq);
  const int rows = s.B * s.Hq * T_m;
  const double tau_d = static_cast<double>(tau), theta_d = static_cast<double>(theta);
  e = launch_k(kPdlPredict, k_shat_dmma<D>, g1, dim3(kGemmThreads), smem_g, stream, q_pooled, k_pooled, k_sim,
               theta_d, s.Hq, s.Hkv, T_m, T_n, s.N, s.bq, s.bk, s.causal, shat);
  if (e != cudaSuccess) return e;
  // long rows: one CTA of kCtaWarps warps per row (occupancy); short rows:
  // one warp per row, up to kMaxRowWarps rows per CTA
  if (T_n > cta_row_min_tn()) {
    const size_t smem_c = cta_row_smem_bytes(T_n);
    e = cudaFuncSetAttribute(k_topcdf_cta<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_c));
    if (e != cudaSuccess) return e;
    return launch_k(kPdlPredict, k_topcdf_cta<D>, dim3(rows), dim3(kCtaThreads), smem_c, stream, shat, q_sim,
                    s.Hq, s.Hkv, s.N, T_m, T_n, s.bq, s.bk, s.causal, tau_d, theta_d, mask, lut,
                    cnt);
  }
  // rows per CTA: up to kMaxRowWarps, as many as fit the shared memory
  const size_t per_warp = row_smem_bytes(T_n);
  const int warps = static_cast<int>(std::min<size_t>(kMaxRowWarps, kRowSmemMax / per_warp));
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem_r = per_warp * warps;
  e = cudaFuncSetAttribute(k_topcdf_rows<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem_r));
  if (e != cudaSuccess) return e;
  return launch_k(kPdlPredict, k_topcdf_rows<D>, dim3((rows + warps - 1) / warps), dim3(warps * 32), smem_r,
                  stream, shat, q_sim, s.Hq, s.Hkv, s.N, T_m, T_n, rows, s.bq, s.bk, s.causal,
                  tau_d, theta_d, mask, lut, cnt);
}

}  // namespace

size_t predict_workspace_bytes(const sparge_shape& s) {
  const size_t T_m = (s.N + s.bq - 1) / s.bq;
  const size_t T_n = (s.N + s.bk - 1) / s.bk;
  return sizeof(double) * static_cast<size_t>(s.B) * s.Hq * T_m * T_n;
}

cudaError_t launch_predict(const sparge_shape& s, const double* q_pooled, const double* q_sim,
                           const double* k_pooled, const double* k_sim, float tau, float theta,
                           uint8_t* mask, int32_t* lut, int32_t* cnt, void* workspace,
                           cudaStream_t stream) {
  double* shat = static_cast<double*>(workspace);
  if (s.d == 128)
    return launch_d<128>(s, q_pooled, q_sim, k_pooled, k_sim, tau, theta, mask, lut, cnt, shat,
                         stream);
  return launch_d<64>(s, q_pooled, q_sim, k_pooled, k_sim, tau, theta, mask, lut, cnt, shat,
                      stream);
}

}  // namespace sparge
