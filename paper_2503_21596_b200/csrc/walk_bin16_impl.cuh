// Hot binary Gray walk, packed 16-bit variant: L_1, L_marg, L_2.
//
// Same decomposition and Gray control as walk_bin_impl.cuh (units = prefixes,
// warp-uniform local suffix walk, Eq. 9 / Eq. 12), but two column sums share one
// 32-bit register (s16x2) and the value uses the identity
//     |m| = 2 max(m, 0) - m   =>   sum_y |m_y| = 2 sum_y max(m_y, 0) - sum_y m_y,
// so that per PAIR of columns a step costs
//     VIADD.16x2   (m += delta, FMA-heavy pipe)  and
//     VIADDMNMX.S16x2 (acc = max(acc + m, acc) = acc + max(m, 0), ALU pipe)
// i.e. one instruction per column update instead of two, split over both pipes.
// The scalar q carries the linear part:  L_1: q = -sum_y m_y;
// L_marg: column 0 is kept out of the packed words and q = m_0 - sum_{y>=1} m_y
// (Eq. 2);  L_2: m_1 = T - m_0 is packed too and q = -sum_y T_y.  Per step
//     value = 2 (acc.lo + acc.hi) + q  =  IDP.2A(acc, {2,2}, q).
// Exactness: every partial sum stays inside s16 when,
// for each column parity class, sum_y sum_x |M_xy| <= 32767 (checked on the host;
// otherwise the int32 kernels run).
#include "common.cuh"

#ifndef LN_BIN_MODE
#error "define LN_BIN_MODE before including walk_bin16_impl.cuh"
#endif

namespace lnorm {

namespace {

constexpr int kTabWords = 16384;   // smem table limit (words); scratch buffer is 32768 ints
constexpr int kBlock = 32;

// ctz for the unrolled step index j in [1, 16): a ternary chain that folds at compile time
__host__ __device__ constexpr int cctz(int j) { return (j & 1) ? 0 : (j & 2) ? 1 : (j & 4) ? 2 : 3; }

// Unrolled low suffix digits: as many as keep the unrolled block under ~800
// instructions (instruction-cache footprint; see walk_pair16_impl.cuh).
// (measured: with plain loads and K = 4 the 42x42 L_1 walk ran 3.80 s vs 4.18 s with
// K = 3 and volatile loads, so the budget here is larger than the paired kernel's)
__host__ __device__ constexpr int unroll_digits(int step_instr) {
  return step_instr * 16 <= 1800 ? 4 : step_instr * 8 <= 1800 ? 3 : step_instr * 4 <= 1800 ? 2 : 1;
}

// Record strides are padded to 4 words so every row starts 16-byte aligned for LDS.128.
__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }

template <int MODE, int W>
struct Layout {
  static constexpr int Wt = (MODE == MODE_LD ? 2 * W : W);     // packed words per delta record
  static constexpr int RWd = pad4(Wt + 1);                     // delta record: Wt words, q at RWd-1
  static constexpr int RWp = pad4(W + 1);                      // prefix record: W words, q at W
  static constexpr int RWb = pad4(Wt + 1);                     // base record: W (+ W totals), q at Wt
};

template <int MODE, int W, int P>
struct Walker16 {
  static constexpr int RWd = Layout<MODE, W>::RWd;
  // Apply the delta record at sT + off (one warp-uniform broadcast LDS.128 per 4 words,
  // shared by the lane's P units); returns nothing, updates ub[] with the new values.
  static __device__ __forceinline__ void step(uint32_t (&m)[P][W], uint32_t (&m1)[P][W], int32_t (&q)[P],
                                              int32_t (&ub)[P], const uint32_t* sT, int off) {
    uint32_t r[RWd];
    const uint4* src = reinterpret_cast<const uint4*>(sT + off);
#pragma unroll
    for (int v = 0; v < RWd / 4; ++v) {
      const uint4 x = src[v];   // plain loads: ptxas keeps the block's few distinct rows in registers
      r[4 * v] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      uint32_t a0, a1 = 0u;
#pragma unroll
      for (int i = 0; i < W; ++i) {
        m[j][i] = __vadd2(m[j][i], r[i]);
        if (i == 0) a0 = __vmaxs2(m[j][0], 0u);
        else if (i & 1) a1 = __viaddmax_s16x2(a1, m[j][i], a1);
        else a0 = __viaddmax_s16x2(a0, m[j][i], a0);
      }
      if (MODE == MODE_LD) {
#pragma unroll
        for (int i = 0; i < W; ++i) {
          m1[j][i] = __vadd2(m1[j][i], r[W + i]);
          if (i & 1) a1 = __viaddmax_s16x2(a1, m1[j][i], a1);
          else a0 = __viaddmax_s16x2(a0, m1[j][i], a0);
        }
      }
      q[j] += (int32_t)r[RWd - 1];
      ub[j] = max(ub[j], __dp2a_lo((int)__vadd2(a0, a1), 0x0202, q[j]));
    }
  }
  static __device__ __forceinline__ int32_t value(const uint32_t (&m)[W], const uint32_t (&m1)[W], int32_t q) {
    uint32_t a0 = 0u, a1 = 0u;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      if (i & 1) a1 = __viaddmax_s16x2(a1, m[i], a1);
      else a0 = __viaddmax_s16x2(a0, m[i], a0);
      if (MODE == MODE_LD) {
        if (i & 1) a1 = __viaddmax_s16x2(a1, m1[i], a1);
        else a0 = __viaddmax_s16x2(a0, m1[i], a0);
      }
    }
    return __dp2a_lo((int)__vadd2(a0, a1), 0x0202, q);
  }
};

template <int MODE, int W, int P>
__host__ __device__ constexpr int bin16_unroll() {
  // wide rows: keep the unrolled block near 1000 instructions (instruction cache)
  return (Layout<MODE, W>::Wt > 40 && unroll_digits(P * (2 * Layout<MODE, W>::Wt + 5) + Layout<MODE, W>::RWd / 4) > 2)
             ? 2 : unroll_digits(P * (2 * Layout<MODE, W>::Wt + 5) + Layout<MODE, W>::RWd / 4);
}

template <int MODE, int W, int P>
__global__ void __launch_bounds__(kBlock) walk_bin16_kernel(const WalkParams p, const uint32_t* __restrict__ gTab) {
  using LY = Layout<MODE, W>;
  constexpr int K = bin16_unroll<MODE, W, P>();
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int s = p.s, k = p.k;
  const int preOff = 2 * s * LY::RWd;
  const int baseOff = preOff + (k + 1) * LY::RWp;
  const int total = baseOff + LY::RWb;
  for (int i = threadIdx.x; i < total; i += blockDim.x) sT[i] = gTab[i];
  __syncthreads();
  const uint32_t nblk = 1u << (s - K);
  int32_t best = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  // Static warp-chunk schedule (block = one warp): chunk ch holds units
  // [ch*32P, ch*32P + 32P); lane l owns units ch*32P + j*32 + l, j < P.
  const int64_t nchunks = (p.unit_count + 32 * P - 1) / (32 * P);
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    uint32_t m[P][W], m1[P][W];
    int32_t q[P], ub[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = ch * 32 * P + j * 32 + lane;
      const int64_t u = p.unit_begin + (rel < p.unit_count ? rel : 0);
      q[j] = (int32_t)sT[baseOff + LY::Wt];
#pragma unroll
      for (int i = 0; i < W; ++i) m[j][i] = sT[baseOff + i];
      for (int x = 0; x <= k; ++x) {
        const int dig = prefix_digit(p, u, x);
        const int po = preOff + x * LY::RWp;
        if (MODE == MODE_LD) {
          if (dig == 0) {
#pragma unroll
            for (int i = 0; i < W; ++i) m[j][i] = __vadd2(m[j][i], sT[po + i]);
          }
        } else {
          if (dig == 0) {
#pragma unroll
            for (int i = 0; i < W; ++i) m[j][i] = __vadd2(m[j][i], sT[po + i]);
            q[j] += (int32_t)sT[po + W];
          } else {
#pragma unroll
            for (int i = 0; i < W; ++i) m[j][i] = __vsub2(m[j][i], sT[po + i]);
            q[j] -= (int32_t)sT[po + W];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < W; ++i) m1[j][i] = (MODE == MODE_LD) ? __vsub2(sT[baseOff + W + i], m[j][i]) : 0u;
      ub[j] = Walker16<MODE, W, P>::value(m[j], m1[j], q[j]);
    }
    for (uint32_t t = 0; t < nblk; ++t) {
      if (t != 0) {
        const int tz = __ffs((int)t) - 1;
        const int b = K + tz;
        const int sg = 1 ^ (int)((t >> (tz + 1)) & 1u);
        Walker16<MODE, W, P>::step(m, m1, q, ub, sT, (2 * b + sg) * LY::RWd);
      }
#pragma unroll
      for (int jj = 1; jj < (1 << K); ++jj) {
        const int b = cctz(jj);
        const int sg = (b < K - 1) ? (1 ^ ((jj >> (b + 1)) & 1)) : (1 ^ (int)(t & 1u));
        Walker16<MODE, W, P>::step(m, m1, q, ub, sT, (2 * b + sg) * LY::RWd);
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = ch * 32 * P + j * 32 + lane;
      if (rel < p.unit_count) {
        if (p.unit_max) p.unit_max[rel] = ub[j];
        // units of a lane are visited in increasing order: strict '>' keeps the smallest
        if (!have || ub[j] > best) { best = ub[j]; best_u = (uint32_t)(p.unit_begin + rel); have = true; }
      }
    }
  }
  unsigned long long key = have ? make_key(best, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key) atomicMax(p.key, key);
}

__device__ __forceinline__ uint32_t pack2(int32_t lo, int32_t hi) {
  return (uint32_t)(lo & 0xFFFF) | ((uint32_t)(hi & 0xFFFF) << 16);
}

// One thread per record: builds the packed table from the oriented matrix.
template <int MODE>
__global__ void build_table16_kernel(const int32_t* M, int r, int c, int W, int k, int s, uint32_t* tab) {
  const int Wt = (MODE == MODE_LD ? 2 * W : W);
  const int RWd = pad4(Wt + 1), RWp = pad4(W + 1), RWb = pad4(Wt + 1);
  const int preOff = 2 * s * RWd, baseOff = preOff + (k + 1) * RWp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < baseOff + RWb; i += gridDim.x * blockDim.x) tab[i] = 0u;
  __syncthreads();
  const int c0 = (MODE == MODE_MARG) ? 1 : 0;      // first packed column
  const int nrec = 2 * s + (k + 1) + 1;
  const int scale = (MODE == MODE_LD) ? 1 : 2;
  for (int rec = blockIdx.x * blockDim.x + threadIdx.x; rec < nrec; rec += gridDim.x * blockDim.x) {
    if (rec < 2 * s) {                                 // delta record (2b + sign)
      const int b = rec >> 1, sg = rec & 1;
      const int32_t* row = M + (int64_t)(r - 1 - b) * c;
      const int f = sg ? -scale : scale;
      uint32_t* out = tab + rec * RWd;
      int32_t qd = 0;
      for (int i = 0; i < W; ++i) {
        const int y0 = c0 + 2 * i, y1 = y0 + 1;
        const int32_t lo = y0 < c ? f * row[y0] : 0, hi = y1 < c ? f * row[y1] : 0;
        out[i] = pack2(lo, hi);
        if (MODE == MODE_LD) out[W + i] = pack2(-lo, -hi);
        qd -= lo + hi;
      }
      if (MODE == MODE_MARG) qd += f * row[0];
      if (MODE == MODE_LD) qd = 0;
      out[RWd - 1] = (uint32_t)qd;
    } else if (rec < 2 * s + k + 1) {                  // prefix record x (raw row)
      const int x = rec - 2 * s;
      const int32_t* row = M + (int64_t)x * c;
      uint32_t* out = tab + preOff + x * RWp;
      int32_t qd = 0;
      for (int i = 0; i < W; ++i) {
        const int y0 = c0 + 2 * i, y1 = y0 + 1;
        const int32_t lo = y0 < c ? row[y0] : 0, hi = y1 < c ? row[y1] : 0;
        out[i] = pack2(lo, hi);
        qd -= lo + hi;
      }
      if (MODE == MODE_MARG) qd += row[0];
      out[W] = (uint32_t)qd;
    } else {                                           // base record: suffix rows at digit 0
      uint32_t* out = tab + baseOff;
      int32_t qd = 0, qT = 0;
      for (int i = 0; i < W; ++i) {
        int32_t bl = 0, bh = 0, tl = 0, th = 0;
        const int y0 = c0 + 2 * i, y1 = y0 + 1;
        for (int x = 0; x < r; ++x) {
          const int32_t vl = y0 < c ? M[(int64_t)x * c + y0] : 0, vh = y1 < c ? M[(int64_t)x * c + y1] : 0;
          tl += vl; th += vh;
          if (x > k) { bl += vl; bh += vh; }
        }
        out[i] = pack2(bl, bh);
        if (MODE == MODE_LD) out[W + i] = pack2(tl, th);
        qd -= bl + bh;
        qT -= tl + th;
      }
      if (MODE == MODE_MARG) { int32_t b0 = 0; for (int x = k + 1; x < r; ++x) b0 += M[(int64_t)x * c]; qd += b0; }
      out[Wt] = (uint32_t)(MODE == MODE_LD ? qT : qd);
    }
  }
}

template <int MODE, int W>
size_t smem16(int k, int s) {
  using LY = Layout<MODE, W>;
  return sizeof(uint32_t) * (size_t)(2 * s * LY::RWd + (k + 1) * LY::RWp + LY::RWb);
}

// units per lane: 2 while the packed state stays small, else 1 (register budget)
template <int MODE, int W>
__host__ __device__ constexpr int units_per_lane() { return (MODE == MODE_LD ? 2 * W : W) <= 24 ? 2 : 1; }

template <int MODE, int W>
cudaError_t launch_one16(const WalkParams& p, const uint32_t* tab, int grid, cudaStream_t st) {
  constexpr int P = units_per_lane<MODE, W>();
  const size_t sm = smem16<MODE, W>(p.k, p.s);
  cudaError_t e = ensure_dyn_smem((const void*)walk_bin16_kernel<MODE, W, P>, sm);
  if (e != cudaSuccess) return e;
  walk_bin16_kernel<MODE, W, P><<<grid, kBlock, sm, st>>>(p, tab);
  return cudaGetLastError();
}

template <int MODE, int W>
int upl_one16() { return units_per_lane<MODE, W>(); }

template <int MODE, int W>
int occ_one16(int k, int s) {
  constexpr int P = units_per_lane<MODE, W>();
  const size_t sm = smem16<MODE, W>(k, s);
  const int nb = occupancy_cached((const void*)walk_bin16_kernel<MODE, W, P>, kBlock, sm);
  return nb;
}

#define LN_W16_SWITCH(MODE, W_, FN, ...)                                                     \
  switch (W_) {                                                                              \
    case 1: return FN<MODE, 1>(__VA_ARGS__);   case 2: return FN<MODE, 2>(__VA_ARGS__);      \
    case 3: return FN<MODE, 3>(__VA_ARGS__);   case 4: return FN<MODE, 4>(__VA_ARGS__);      \
    case 5: return FN<MODE, 5>(__VA_ARGS__);   case 6: return FN<MODE, 6>(__VA_ARGS__);      \
    case 7: return FN<MODE, 7>(__VA_ARGS__);   case 8: return FN<MODE, 8>(__VA_ARGS__);      \
    case 9: return FN<MODE, 9>(__VA_ARGS__);   case 10: return FN<MODE, 10>(__VA_ARGS__);    \
    case 11: return FN<MODE, 11>(__VA_ARGS__); case 12: return FN<MODE, 12>(__VA_ARGS__);    \
    case 13: return FN<MODE, 13>(__VA_ARGS__); case 14: return FN<MODE, 14>(__VA_ARGS__);    \
    case 15: return FN<MODE, 15>(__VA_ARGS__); case 16: return FN<MODE, 16>(__VA_ARGS__);    \
    case 17: return FN<MODE, 17>(__VA_ARGS__); case 18: return FN<MODE, 18>(__VA_ARGS__);    \
    case 19: return FN<MODE, 19>(__VA_ARGS__); case 20: return FN<MODE, 20>(__VA_ARGS__);    \
    case 21: return FN<MODE, 21>(__VA_ARGS__); case 22: return FN<MODE, 22>(__VA_ARGS__);    \
    case 23: return FN<MODE, 23>(__VA_ARGS__); case 24: return FN<MODE, 24>(__VA_ARGS__);    \
    case 26: return FN<MODE, 26>(__VA_ARGS__); case 28: return FN<MODE, 28>(__VA_ARGS__);    \
    case 30: return FN<MODE, 30>(__VA_ARGS__); case 32: return FN<MODE, 32>(__VA_ARGS__);    \
    case 40: return FN<MODE, 40>(__VA_ARGS__); case 48: return FN<MODE, 48>(__VA_ARGS__);    \
    case 56: return FN<MODE, 56>(__VA_ARGS__); case 64: return FN<MODE, 64>(__VA_ARGS__);    \
    case 72: return FN<MODE, 72>(__VA_ARGS__); case 80: return FN<MODE, 80>(__VA_ARGS__);    \
    case 88: return FN<MODE, 88>(__VA_ARGS__); case 96: return FN<MODE, 96>(__VA_ARGS__);    \
    default: break;                                                                          \
  }

}  // namespace

template <>
int walk_bin16_words<LN_BIN_MODE>(int c) {
  const int cp = (LN_BIN_MODE == MODE_MARG) ? c - 1 : c;
  int W = (cp + 1) / 2;
  if (W < 1) W = 1;
  if (W > 24) W = (W + 1) & ~1;
  if (W > 32) W = (W + 7) & ~7;            // wide matrices (m up to 4n, SURVEY config 5a): W in 40..96
  return W <= 96 ? W : 0;
}

template <>
cudaError_t walk_bin16_launch_mode<LN_BIN_MODE>(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st) {
  const int W = walk_bin16_words<LN_BIN_MODE>(p.c);
  if (W == 0) return cudaErrorInvalidValue;
  const int Wt = (LN_BIN_MODE == MODE_LD ? 2 * W : W);
  const int total = 2 * p.s * pad4(Wt + 1) + (p.k + 1) * pad4(W + 1) + pad4(Wt + 1);
  if (total > kTabWords) return cudaErrorInvalidValue;
  uint32_t* tab = reinterpret_cast<uint32_t*>(scratch_tab);
  build_table16_kernel<LN_BIN_MODE><<<1, 128, 0, st>>>(p.M, p.r, p.c, W, p.k, p.s, tab);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  LN_W16_SWITCH(LN_BIN_MODE, W, launch_one16, p, tab, grid, st)
  return cudaErrorInvalidValue;
}

template <int MODE, int W>
int unroll_one16() { return bin16_unroll<MODE, W, units_per_lane<MODE, W>()>(); }

template <>
int walk_bin16_unroll_mode<LN_BIN_MODE>(int c) {
  const int W = walk_bin16_words<LN_BIN_MODE>(c);
  LN_W16_SWITCH(LN_BIN_MODE, W, unroll_one16)
  return 4;
}

template <>
int64_t walk_bin16_table_words_mode<LN_BIN_MODE>(int c, int k, int s) {
  const int W = walk_bin16_words<LN_BIN_MODE>(c);
  if (W == 0) return INT64_MAX;
  const int Wt = (LN_BIN_MODE == MODE_LD ? 2 * W : W);
  return (int64_t)2 * s * pad4(Wt + 1) + (int64_t)(k + 1) * pad4(W + 1) + pad4(Wt + 1);
}

template <>
int walk_bin16_units_per_lane_mode<LN_BIN_MODE>(int c) {
  const int W = walk_bin16_words<LN_BIN_MODE>(c);
  LN_W16_SWITCH(LN_BIN_MODE, W, upl_one16)
  return 1;
}

template <>
int walk_bin16_occupancy_mode<LN_BIN_MODE>(int c, int k, int s) {
  const int W = walk_bin16_words<LN_BIN_MODE>(c);
  LN_W16_SWITCH(LN_BIN_MODE, W, occ_one16, k, s)
  return 0;
}

}  // namespace lnorm
