// Hot d-ary Gray walk for L_3 and L_4, column sums packed four per register as offset bytes,
// the LAST PR rows (L_3: 3-5, L_4: 3-4) evaluated for all D^PR labellings at every walked word,
// with every group's 2^PR bias sums kept as plain |.|-sums ("all-H" form) and the bias words
// staged in shared memory.
//
// Same units, restricted-growth prefixes, warp-uniform reflected D-ary walk (PAPER.md
// Eqs. 13-17) and byte encoding as walk_ldu8_impl.cuh (read its header first): group g's
// column sum m_g,y lives in [N_y, N_y + W_y], a_g,y = m_g,y - N_y is one unsigned byte
// when every W_y <= 255, one 32-bit add of a packed row moves a row between two groups
// (Eqs. 18-19), and VABSDIFF4.U8.ACC accumulates four |.| per instruction.
//
// What differs.  For a subset T of the paired rows let
//     H[T][g] = sum_y |m_g,y + sum_{i in T} rho_i,y|        (T = {} is the plain ||m_g||_1)
// = sum_y |a_g,y - B_T,y| + kappa_T  with B_T = clamp(-N - sum_{i in T} rho_i, 0, 255).  A
// labelling of the paired rows is the partition (T_0, .., T_{D-1}) of them by label, and by
// Eq. (6) the strategy's value is exactly
//     L*(walked word, labelling) = sum_g H[T_g][g]
// -- D non-negative terms, no running S or differences to maintain.  A move p -> q
// re-accumulates the 2^PR sums of the two changed groups (2 * 2^PR * NW VABSDIFF4 on the ALU
// pipe); the best labelling of the word is a max-plus subset convolution over the H (LdW::
// conv_best: G_2(U) = max_{T subset U} H[T][1] + H[U \ T][0], for L_4 G_3(U) likewise from
// G_2, then the last label's term), 3^PR (+ 3^PR for L_4) + 2^PR additions as subnormal-float
// FADDs (FMA pipes) and about D^PR / 2 three-input maxes (ALU).  At 24 columns that is 2.96
// ALU instructions per strategy at PR = 4 and 2.14 at PR = 5 (round 1's all-E walk: 4.07).
//
// The 2^PR * NW bias words do not fit the register file next to the H sums, so they are read per
// move from shared memory with warp-uniform LDS.128 broadcasts (four bias sets of one word each,
// shared by the two moved groups); the kappa sums stay in registers, or at five paired rows in
// shared memory as well (LdW::KS).
//
// Control: a move of the reflected D-ary walk is between adjacent labels lo and lo + 1; the
// kernel holds D - 1 sum bodies (the direction only picks which of the delta record's +row /
// -row each group adds, a uniform shared-memory offset) and ONE copy of the convolution, so the
// hot code stays small for the instruction cache.  The changed digit, old and new label come
// from the uniform word counter: inside a block of D words the low digit moves 0 -> D-1 (even
// block) or back (odd block), the block start is dary_block_start (Eq. 17).
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace lnorm {

namespace {

constexpr int kBlockW = 32;
// most paired rows an instance is compiled for (5: 243 labellings per walked word, 2 x 32 bias
// sums per move; 4: 81, 2 x 16)
#ifndef LN_LDU8W_MAXPR
#define LN_LDU8W_MAXPR 5
#endif
// resident warps per SM asked of ptxas: 16 (<= 128 registers, four warps per SMSP) where that
// needs no spills (L_3 up to four paired rows except NW = 10 and 12), else 12 (<= 168 registers:
// L_3 with five paired rows, 96 H sums per unit; L_4 with four, 64 H sums + the convolution levels)
#ifndef LN_LDU8W_MINB
#define LN_LDU8W_MINB 16
#endif
#ifndef LN_LDU8W_MINB5
#define LN_LDU8W_MINB5 12
#endif
// paired rows from which the kappa sums live in shared memory instead of registers (LdW::KS)
#ifndef LN_LDU8W_KSMEM_PR
#define LN_LDU8W_KSMEM_PR 5
#endif
template <int D, int NW, int PR>
__host__ __device__ constexpr int w_minb() {
  return (PR == 5 || (D == 4 && PR >= 4)) ? LN_LDU8W_MINB5 : (PR == 4 && (NW == 10 || NW == 12)) ? 12 : LN_LDU8W_MINB;
}
constexpr int kTabWordsW = 16384;

__host__ __device__ constexpr int w_pad4(int x) { return (x + 3) & ~3; }
__host__ __device__ constexpr int w_pow(int d, int e) { return e == 0 ? 1 : d * w_pow(d, e - 1); }
__host__ __device__ constexpr int w_popc(int x) { return x == 0 ? 0 : (x & 1) + w_popc(x >> 1); }
// the i-th submask of U in increasing order (i < 2^popc(U)): bit j of i -> j-th set bit of U
__host__ __device__ constexpr int w_submask(int U, int i) {
  return U == 0 ? 0 : ((U & 1) ? ((i & 1) | (w_submask(U >> 1, i >> 1) << 1)) : (w_submask(U >> 1, i) << 1));
}
// bitmask of the paired rows labelled g in labelling L (base-D digits of L, paired row b = digit b)
__host__ __device__ constexpr int w_mask(int L, int g, int PR, int D) {
  return PR == 0 ? 0 : ((L % D == g) ? 1 : 0) | (w_mask(L / D, g, PR - 1, D) << 1);
}

__device__ __forceinline__ uint32_t w_sad4(uint32_t a, uint32_t b, uint32_t acc) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(acc));
  return d;
}
// The candidate sums and their max.  Every value here is a non-negative integer below 2^23
// (at most 3 * sum |M| <= 3 * 255 * 48 under the byte guard), and read as IEEE-754 single
// bits such an integer v is the subnormal v * 2^-149: subnormal addition is exact and
// bit-additive while the sum stays below 2^23 (a carry into the exponent field at 2^23 is
// still the integer v), and subnormal max orders like the integers.  So, with denormals
// kept (add.f32 / max.f32 without .ftz -- no fast-math in this build), FADD computes the
// integer sum on EITHER FMA pipe (full rate, where IMAD runs on the FMA-heavy pipe only at
// half rate) and FMNMX3 the integer max.  LN_LDU8W_FP=0 keeps integer IMAD / VIMNMX3.
#ifndef LN_LDU8W_FP
#define LN_LDU8W_FP 1
#endif
__device__ __forceinline__ int32_t w_fadd(int32_t a, int32_t b, uint32_t one) {
#if LN_LDU8W_FP
  (void)one;
  float r;
  asm("add.f32 %0, %1, %2;" : "=f"(r) : "f"(__int_as_float(a)), "f"(__int_as_float(b)));
  return __float_as_int(r);
#else
  int32_t r;   // IMAD with a uniform operand ptxas cannot fold: stays on the FMA-heavy pipe
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
  return r;
#endif
}
__device__ __forceinline__ int32_t w_max3(int32_t a, int32_t b, int32_t c) {
#if LN_LDU8W_FP
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(__int_as_float(a)), "f"(__int_as_float(b)), "f"(__int_as_float(c)));
  return __float_as_int(r);
#else
  return __vimax3_s32(a, b, c);
#endif
}
__device__ __forceinline__ int32_t w_max2(int32_t a, int32_t b) {
#if LN_LDU8W_FP
  float r;
  asm("max.f32 %0, %1, %2;" : "=f"(r) : "f"(__int_as_float(a)), "f"(__int_as_float(b)));
  return __float_as_int(r);
#else
  return max(a, b);
#endif
}

// max of N non-negative values with three-input maxes: ceil((N - 1) / 2) ALU instructions
template <int N>
__device__ __forceinline__ int32_t w_max_tree(const int32_t (&v)[N]) {
  if constexpr (N == 1) {
    return v[0];
  } else if constexpr (N == 2) {
    return w_max2(v[0], v[1]);
  } else {
    constexpr int M = (N + 2) / 3;
    int32_t w[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (3 * i + 2 < N) w[i] = w_max3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
      else if (3 * i + 1 < N) w[i] = w_max2(v[3 * i], v[3 * i + 1]);
      else w[i] = v[3 * i];
    }
    return w_max_tree<M>(w);
  }
}

// PK (two units per lane, every H / convolution value of the two units packed as unsigned 16-bit
// halves): VIADD.16x2 (FMA pipe) adds both units' candidates in one instruction and VIMNMX3.U16x2
// (ALU) takes the max of three pairs -- half the convolution's max instructions per unit.  Exact:
// every H, convolution value and strategy value is a partial sum of one labelling's value, which
// is <= sum |M| <= 255 * 48 < 2^16 under the byte guard (every column's sum_x |M_xy| <= 255).
// LN_LDU8W_PK_IMAD: the packed add as a 32-bit IMAD a * one + b (no half ever carries: both halves
// stay below 2^16), which ptxas cannot fuse with the following max into an ALU-pipe VIADDMNMX.U16x2
// the way it fuses VIADD.16x2.  Measured 2.5 % slower (24x24 L_3 5.90 vs 5.75 ms, 26x26 58.1 vs
// 57.5 ms; profiles/r02/ab_l3_pk_imad.log): the fused form needs fewer issue slots, off by default
#ifndef LN_LDU8W_PK_IMAD
#define LN_LDU8W_PK_IMAD 0
#endif
// LN_LDU8W_PK_IMAD_LV: bit l-1 set = the adds of convolution level l (1: G_2 from H, 2: L_4's G_3,
// 3: the last step) use the unfusable IMAD form (A/B knob; LN_LDU8W_PK_IMAD = all levels)
#ifndef LN_LDU8W_PK_IMAD_LV
#define LN_LDU8W_PK_IMAD_LV (LN_LDU8W_PK_IMAD ? 7 : 0)
#endif
template <bool PK, int LV = 1>
__device__ __forceinline__ int32_t op_add(int32_t a, int32_t b, uint32_t one) {
  if constexpr (PK) {
    if constexpr (((LN_LDU8W_PK_IMAD_LV >> (LV - 1)) & 1) != 0) {
      uint32_t r;
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"((uint32_t)a), "r"(one), "r"((uint32_t)b));
      return (int32_t)r;
    } else {
      (void)one;
      return (int32_t)__vadd2((uint32_t)a, (uint32_t)b);
    }
  } else {
    return w_fadd(a, b, one);
  }
}
template <bool PK>
__device__ __forceinline__ int32_t op_max3(int32_t a, int32_t b, int32_t c) {
  if constexpr (PK) return (int32_t)__vimax3_u16x2((uint32_t)a, (uint32_t)b, (uint32_t)c);
  else return w_max3(a, b, c);
}
template <bool PK>
__device__ __forceinline__ int32_t op_max2(int32_t a, int32_t b) {
  if constexpr (PK) return (int32_t)__vmaxu2((uint32_t)a, (uint32_t)b);
  else return w_max2(a, b);
}
template <bool PK, int N>
__device__ __forceinline__ int32_t op_max_tree(const int32_t (&v)[N]) {
  if constexpr (N == 1) {
    return v[0];
  } else if constexpr (N == 2) {
    return op_max2<PK>(v[0], v[1]);
  } else {
    constexpr int M = (N + 2) / 3;
    int32_t w[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (3 * i + 2 < N) w[i] = op_max3<PK>(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
      else if (3 * i + 1 < N) w[i] = op_max2<PK>(v[3 * i], v[3 * i + 1]);
      else w[i] = v[3 * i];
    }
    return op_max_tree<PK, M>(w);
  }
}

template <int D, int NW, int PR, bool PK = false>
struct LdW {
  static constexpr int RW = w_pad4(NW);
  static constexpr int RD = 2 * RW;          // delta record: +row at [0, NW), -row at [RW, RW + NW)
  static constexpr int NS = 1 << PR;         // bias sets (subsets of the paired rows)
  static constexpr int NL = w_pow(D, PR);    // labellings of the paired rows

  // Direct form (LN_LDU8W_CONV = 0, L_3 only): the value of labelling L is
  // sum_g H[T_g][g] (masks forced to compile time), D - 1 FADD per labelling.
  template <int L>
  static __device__ __forceinline__ int32_t cand(const int32_t (&H)[NS][D], uint32_t one) {
    constexpr int m0 = std::integral_constant<int, w_mask(L, 0, PR, D)>::value;
    constexpr int m1 = std::integral_constant<int, w_mask(L, 1, PR, D)>::value;
    constexpr int m2 = std::integral_constant<int, w_mask(L, 2, PR, D)>::value;
    return op_add<PK>(op_add<PK>(H[m0][0], H[m1][1], one), H[m2][2], one);
  }
  template <int... Ls>
  static __device__ __forceinline__ int32_t best_seq(const int32_t (&H)[NS][D], int32_t best, uint32_t one,
                                                     std::integer_sequence<int, Ls...>) {
    int32_t v[NL + 1] = {cand<Ls>(H, one)..., best};
    return op_max_tree<PK, NL + 1>(v);
  }
  // Max-plus subset convolution form of the same maximum (LN_LDU8W_CONV = 1).  A labelling of the
  // paired rows is a partition (T_0, .., T_{D-1}) of them by label, valued sum_g H[T_g][g]; with
  //     G_1(U) = H[U][0],   G_{g+1}(U) = max over T subset of U of  H[T][g] + G_g(U \ T)
  // the best labelling is G_D(all paired rows) = max over T of H[T][D-1] + G_{D-1}(rest).  Additions: 3^PR per intermediate level (sum over
  // U of 2^|U|) plus 2^PR for the last one -- L_3, PR = 4: 97 FADD instead of 2 * 81 = 162; L_4,
  // PR = 4: 178 instead of 3 * 256 = 768 -- with about as many maxes as the direct form.
  // L_01(U) = max over T subset of U of H[T][1] + H[U \ T][0]  (= G_2(U), streamed)
  template <int U, int I>
  static __device__ __forceinline__ int32_t term01(const int32_t (&H)[NS][D], uint32_t one) {
    constexpr int T = std::integral_constant<int, w_submask(U, I)>::value;
    return op_add<PK>(H[T][1], H[U ^ T][0], one);
  }
  template <int U, int... Is>
  static __device__ __forceinline__ int32_t L01(const int32_t (&H)[NS][D], uint32_t one, std::integer_sequence<int, Is...>) {
    int32_t v[sizeof...(Is)] = {term01<U, Is>(H, one)...};
    return op_max_tree<PK, (int)sizeof...(Is)>(v);
  }
  template <int U>
  static __device__ __forceinline__ int32_t G2(const int32_t (&H)[NS][D], uint32_t one) {
    return L01<U>(H, one, std::make_integer_sequence<int, (1 << w_popc(U))>{});
  }
  // L_4's middle level from the stored G_2 values: G_3(U) = max over T subset of U of H[T][2] + G_2(U \ T)
  template <int U, int I>
  static __device__ __forceinline__ int32_t term2(const int32_t (&H)[NS][D], const int32_t (&g2)[NS], uint32_t one) {
    constexpr int T = std::integral_constant<int, w_submask(U, I)>::value;
    return op_add<PK, 2>(H[T][2], g2[U ^ T], one);
  }
  template <int U, int... Is>
  static __device__ __forceinline__ int32_t L2(const int32_t (&H)[NS][D], const int32_t (&g2)[NS], uint32_t one,
                                               std::integer_sequence<int, Is...>) {
    int32_t v[sizeof...(Is)] = {term2<U, Is>(H, g2, one)...};
    return op_max_tree<PK, (int)sizeof...(Is)>(v);
  }
  // last level, one term per label-(D-1) set T (the complement is the rest of the paired rows);
  // the intermediate level is streamed (L_3) or read from the stored G_2 (L_4), so at most NS
  // intermediate values are live next to the H sums
  template <int T>
  static __device__ __forceinline__ int32_t last(const int32_t (&H)[NS][D], const int32_t (&g2)[NS], uint32_t one) {
    constexpr int U = (NS - 1) ^ T;
    if constexpr (D == 3) return op_add<PK, 3>(H[T][2], G2<U>(H, one), one);
    else return op_add<PK, 3>(H[T][3], L2<U>(H, g2, one, std::make_integer_sequence<int, (1 << w_popc(U))>{}), one);
  }
  template <int... Us>
  static __device__ __forceinline__ void fill_g2(const int32_t (&H)[NS][D], int32_t (&g2)[NS], uint32_t one,
                                                 std::integer_sequence<int, Us...>) {
    ((g2[Us] = G2<Us>(H, one)), ...);
  }
  template <int... Ts>
  static __device__ __forceinline__ int32_t conv_seq(const int32_t (&H)[NS][D], const int32_t (&g2)[NS], int32_t best,
                                                     uint32_t one, std::integer_sequence<int, Ts...>) {
    int32_t v[NS + 1] = {last<Ts>(H, g2, one)..., best};
    return op_max_tree<PK, NS + 1>(v);
  }
  static __device__ __forceinline__ int32_t conv_best(const int32_t (&H)[NS][D], int32_t best, uint32_t one) {
    int32_t g2[NS];
    if constexpr (D == 4) fill_g2(H, g2, one, std::make_integer_sequence<int, NS>{});
    return conv_seq(H, g2, best, one, std::make_integer_sequence<int, NS>{});
  }
  // max(best, every labelling's value of the current word)
  static __device__ __forceinline__ int32_t best_of(const int32_t (&H)[NS][D], int32_t best, uint32_t one) {
#ifndef LN_LDU8W_CONV
#define LN_LDU8W_CONV 1
#endif
    static_assert(D == 3 || D == 4, "L_3 and L_4");
    if constexpr (LN_LDU8W_CONV || D != 3) return conv_best(H, best, one);
    else return best_seq(H, best, one, std::make_integer_sequence<int, NL>{});
  }

  // A move between groups GA < GB (either direction): the lower group adds the packed row at
  // shared address rowA, the higher one the row at rowB (the +row or the -row of the walked
  // digit's delta record, chosen by the direction), then both groups' 2^PR bias sums are
  // re-accumulated.  The max over the labellings follows at the single call site.
  // Shared-memory bias layout: word-major, sBias[i * NS + m] = B_m word i, so the 2^PR bias
  // words of one packed word are NS / 4 LDS.128.  Instruction order: per packed word i and per
  // half of the bias sets, all VABSDIFF4 of one group back to back -- they share the byte
  // operand A[g][i] (operand reuse cache), so each reads two registers (bias word, accumulator)
  // instead of three; the register-file read ports, not the ALU pipe, bound a 3-source mix.
  // KS: the kappa sums (accumulator starts) are read from shared memory (after the bias words)
  // instead of living in NS registers -- frees 32 registers at five paired rows, where every
  // instance but 24 columns otherwise spills 30-430 bytes (26x26 L_3: 79.0 -> 75.5 ms; 24x24,
  // spill-free either way: 7.89 vs 7.96 ms, so it keeps its kappas in registers;
  // profiles/r02/ab_l3_ksmem.jsonl)
  static constexpr bool KS = PR >= LN_LDU8W_KSMEM_PR && NW != 6;
  template <int GA, int GB, int P>
  static __device__ __forceinline__ void sums(uint32_t (&A)[P][D][NW], int32_t (&H)[P][NS][D], const uint32_t (&Ks)[NS],
                                              uint32_t rowA, uint32_t rowB, uint32_t sbias) {
#ifndef LN_LDU8W_HB
#define LN_LDU8W_HB 8
#endif
    constexpr int HB = NS >= LN_LDU8W_HB ? LN_LDU8W_HB : NS;     // bias sets per batch of loads
#pragma unroll
    for (int v = 0; v < RW / 4; ++v) {
      const uint4 xa = lds128(rowA + 16u * (uint32_t)v);
      const uint4 xb = lds128(rowB + 16u * (uint32_t)v);
      const uint32_t ra[4] = {xa.x, xa.y, xa.z, xa.w}, rb[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * v + e;
        if (i < NW) {
#pragma unroll
          for (int j = 0; j < P; ++j) {
            A[j][GA][i] += ra[e];
            A[j][GB][i] += rb[e];
          }
#pragma unroll
          for (int h = 0; h < NS / HB; ++h) {
            uint32_t bb[HB];
#pragma unroll
            for (int q = 0; q < HB / 4; ++q) {
              const uint4 bq = lds128(sbias + 4u * (uint32_t)(i * NS + h * HB + 4 * q));
              bb[4 * q] = bq.x; bb[4 * q + 1] = bq.y; bb[4 * q + 2] = bq.z; bb[4 * q + 3] = bq.w;
            }
            uint32_t kk[HB];                           // accumulator starts of this batch of bias sets
#pragma unroll
            for (int m = 0; m < HB; ++m) kk[m] = KS ? 0u : Ks[h * HB + m];
            if (KS && i == 0) {
#pragma unroll
              for (int q = 0; q < HB / 4; ++q) {
                const uint4 kq = lds128(sbias + 4u * (uint32_t)(NW * NS + h * HB + 4 * q));
                kk[4 * q] = kq.x; kk[4 * q + 1] = kq.y; kk[4 * q + 2] = kq.z; kk[4 * q + 3] = kq.w;
              }
            }
#pragma unroll
            for (int j = 0; j < P; ++j) {
#pragma unroll
              for (int m = 0; m < HB; ++m)
                H[j][h * HB + m][GA] =
                    (int32_t)w_sad4(A[j][GA][i], bb[m], i == 0 ? kk[m] : (uint32_t)H[j][h * HB + m][GA]);
#pragma unroll
              for (int m = 0; m < HB; ++m)
                H[j][h * HB + m][GB] =
                    (int32_t)w_sad4(A[j][GB][i], bb[m], i == 0 ? kk[m] : (uint32_t)H[j][h * HB + m][GB]);
            }
          }
        }
      }
    }
  }
};

// Packed variant (PK instances): the two units of a lane move the same rows; their bias sums are
// accumulated in 32 bits (four independent VABSDIFF4 chains per bias set: two units x two groups,
// all reading the same bias word from the operand-reuse cache) and packed by one IMAD each.  Bias
// words set-major in shared memory (sbias + 4 (m RW + i)), kappa sums after them (sbias + 4 (NS RW + m)).
template <int D, int NW, int PR, int GA, int GB>
__device__ __forceinline__ void sums_pk(uint32_t (&A)[2][D][NW], int32_t (&H)[1 << PR][D], uint32_t rowA,
                                        uint32_t rowB, uint32_t sbias, uint32_t k16) {
  constexpr int RW = w_pad4(NW), NS = 1 << PR;
#pragma unroll
  for (int v = 0; v < RW / 4; ++v) {
    const uint4 xa = lds128(rowA + 16u * (uint32_t)v);
    const uint4 xb = lds128(rowB + 16u * (uint32_t)v);
    const uint32_t ra[4] = {xa.x, xa.y, xa.z, xa.w}, rb[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * v + e;
      if (i < NW) {
        A[0][GA][i] += ra[e]; A[1][GA][i] += ra[e];
        A[0][GB][i] += rb[e]; A[1][GB][i] += rb[e];
      }
    }
  }
#pragma unroll
  for (int m4 = 0; m4 < NS; m4 += 4) {
    const uint4 kq = lds128(sbias + 4u * (uint32_t)(NS * RW + m4));
    const uint32_t kk[4] = {kq.x, kq.y, kq.z, kq.w};
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      const int m = m4 + mm;
      uint32_t b[RW];
#pragma unroll
      for (int v = 0; v < RW / 4; ++v) {
        const uint4 q = lds128(sbias + 4u * (uint32_t)(m * RW + 4 * v));
        b[4 * v] = q.x; b[4 * v + 1] = q.y; b[4 * v + 2] = q.z; b[4 * v + 3] = q.w;
      }
      uint32_t a0 = kk[mm], a1 = kk[mm], c0 = kk[mm], c1 = kk[mm];
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        a0 = w_sad4(A[0][GA][i], b[i], a0);
        a1 = w_sad4(A[1][GA][i], b[i], a1);
        c0 = w_sad4(A[0][GB][i], b[i], c0);
        c1 = w_sad4(A[1][GB][i], b[i], c1);
      }
      uint32_t pa, pc;
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(pa) : "r"(a1), "r"(k16), "r"(a0));
      asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(pc) : "r"(c1), "r"(k16), "r"(c0));
      H[m][GA] = (int32_t)pa;
      H[m][GB] = (int32_t)pc;
    }
  }
}

// Init records: as build_ldu8_kernel writes them (prefix rows 0..k, the walked base, -N,
// then NS * NW bias words and the NS kappa sums), stride CW = 4 NW.
// Units per lane: P units of a lane move the same rows at every word, so one shared-memory
// load of a row or bias quad serves all P and the P max trees of a word can overlap the other
// units' VABSDIFF4 streams.  Measured on 24x24 L_3 (profiles/r02): P = 2 needs 212 registers
// (two warps per SMSP) and runs 2 % slower than P = 1 at 128 registers; default 1.
#ifndef LN_LDU8W_P
#define LN_LDU8W_P 1
#endif
template <int NW, int PR>
__host__ __device__ constexpr int w_units() { return (NW <= 6) ? LN_LDU8W_P : 1; }

template <int D, int NW, int PR, bool BAT = false>
__global__ void __launch_bounds__(kBlockW, (w_minb<D, NW, PR>()))
walk_ldu8w_kernel(const WalkParams p, const uint32_t* __restrict__ gTab, const int32_t* __restrict__ gInit) {
  using WK = LdW<D, NW, PR>;
  constexpr int P = w_units<NW, PR>();
  constexpr int RD = WK::RD, RW = WK::RW, CW = 4 * NW, NS = WK::NS;
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int sw = p.s - PR;                         // walked digits
  uint32_t* sBias = sT + sw * RD;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sT);
  const uint32_t sbias = (uint32_t)__cvta_generic_to_shared(sBias);
  // LN_LDU8W_KVEC: XOR with threadIdx.y (always 0 in these one-dimensional blocks, but not
  // provably uniform) keeps the kappa sums in vector registers, where VABSDIFF4 reads them,
  // instead of uniform registers copied over at every use (IMAD.U32 on the FMA pipe)
#ifndef LN_LDU8W_KVEC
#define LN_LDU8W_KVEC 1
#endif
  uint32_t Ks[NS];
  uint32_t nwords = 1;
  for (int i = 0; i < sw; ++i) nwords *= D;
  int32_t best_all = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  // matrix mb's delta table and word-major bias words -> shared memory, its kappas -> registers
  auto stage = [&](int mb) {
    __syncwarp();
    const int32_t* gM = gInit + mb * p.init_stride;
    const uint32_t* src = gTab + mb * p.tab_stride;
    const uint32_t* biasRec = reinterpret_cast<const uint32_t*>(gM + (p.k + 3) * CW);
    for (int i = lane; i < sw * RD; i += 32) sT[i] = src[i];
    for (int i = lane; i < NS * NW; i += 32) {     // word-major: sBias[q * NS + m]
      const int q = i / NS, m = i % NS;
      sBias[i] = biasRec[m * NW + q];
    }
    for (int m = lane; m < NS; m += 32) sBias[NS * NW + m] = biasRec[NS * NW + m];   // kappas (WK::KS)
    if constexpr (!WK::KS) {
#pragma unroll
      for (int m = 0; m < NS; ++m) Ks[m] = __ldg(biasRec + NS * NW + m) ^ (LN_LDU8W_KVEC ? (uint32_t)threadIdx.y : 0u);
    }
    __syncwarp();
  };
  // BAT (batched launches, f3): chunk ch -> matrix mb = ch / CPM (units_per units per matrix,
  // the launch's range unless batched); a warp restages the tables when it moves to the next
  // matrix.  The single-search instance stages them once.
  const int64_t CPM = (p.units_per + 32 * P - 1) / (32 * P);
  const int64_t nchunks = BAT ? CPM * p.batch : CPM;
  int cur_b = BAT ? -1 : 0;
  if constexpr (!BAT) stage(0);
  for (int64_t ch = blockIdx.x; ch < nchunks; ch = next_chunk(ch, p.chunk_ctr, lane)) {
    int64_t lc = ch;
    const int32_t* gI = gInit;
    if constexpr (BAT) {
      const int mb = (int)(ch / CPM);
      lc = ch - (int64_t)mb * CPM;
      gI = gInit + mb * p.init_stride;
      if (mb != cur_b) {
        if (cur_b >= 0) {
          unsigned long long key = have ? make_key(best_all, best_u) : 0ull;
          key = warp_max_u64(key);
          if (lane == 0 && key) atomicMax(p.key + cur_b, key);
          best_all = INT32_MIN; have = false;
        }
        stage(mb);
        cur_b = mb;
      }
    }
    uint32_t A[P][D][NW];
    int32_t H[P][NS][D];
    int32_t best[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      // ---- unit init: prefix labels -> the D groups' bytes at the start word (suffix all 0)
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      const int64_t u = p.unit_begin + (rel < p.units_per ? rel : 0);
      uint64_t lab = 0;
      if (p.prefix_table) lab = p.prefix_table[u - p.unit_begin];
      else for (int x = 0; x <= p.k; ++x) lab |= (uint64_t)prefix_digit(p, u, x) << (p.pbits * x);
      const uint64_t lmask = (1ull << p.pbits) - 1ull;
      // packed start bytes, then every prefix row's packed word added to the group of its label
      // (build_ldu8_kernel's packed records: 2 instructions per row, word and group)
      const uint32_t* pkRec = reinterpret_cast<const uint32_t*>(gI + (p.k + 3) * CW) + NS * NW + NS;
      const uint32_t* stRec = pkRec + (p.k + 1) * NW;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        A[j][0][q] = __ldg(stRec + q);
        const uint32_t sg = __ldg(stRec + NW + q);
#pragma unroll
        for (int g = 1; g < D; ++g) A[j][g][q] = sg;
      }
      for (int x = 0; x <= p.k; ++x) {
        const int dig = (int)((lab >> (p.pbits * x)) & lmask);
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          const uint32_t w = __ldg(pkRec + x * NW + q);
#pragma unroll
          for (int g = 0; g < D; ++g) A[j][g][q] += (dig == g) ? w : 0u;
        }
      }
#pragma unroll
      for (int g = 0; g < D; ++g)
#pragma unroll
        for (int m = 0; m < NS; ++m) {
          uint32_t h = WK::KS ? sBias[NS * NW + m] : Ks[m];
#pragma unroll
          for (int q = 0; q < NW; ++q) h = w_sad4(A[j][g][q], sBias[q * NS + m], h);
          H[j][m][g] = (int32_t)h;
        }
      best[j] = WK::best_of(H[j], 0, p.one);          // every value is >= 0 (a sum of |.|)
    }
    // ---- the walk: words 1 .. D^sw - 1, one dispatch site per pair of adjacent labels
    uint32_t t = 0, jj = 0;
    for (uint32_t w = 1; w < nwords; ++w) {
      uint32_t i, from, to;
      if (++jj == D) { jj = 0; ++t; }
      if (jj == 0) {
        dary_block_start<D>(t, &i, &from, &to);
      } else {                                       // low digit: 0 -> D-1 (even block) or back (odd)
        i = 0;
        const bool odd = (t & 1u) != 0;
        from = odd ? D - jj : jj - 1;
        to = odd ? D - 1 - jj : jj;
      }
      // walked digit i's delta record: +row at srow, -row at srow + 4 RW bytes; the group the
      // row leaves (from) adds the -row, the group it joins (to) the +row
      const uint32_t srow = sbase + 4u * i * (uint32_t)RD;
      const uint32_t rlo = from < to ? srow + 4u * (uint32_t)RW : srow;   // row for the lower group
      const uint32_t rhi = from < to ? srow : srow + 4u * (uint32_t)RW;   // row for the higher group
      const uint32_t lo = from < to ? from : to;       // the move is between labels lo and lo + 1
      if (lo == 0) WK::template sums<0, 1, P>(A, H, Ks, rlo, rhi, sbias);
      else if (D == 3 || lo == 1) WK::template sums<1, 2, P>(A, H, Ks, rlo, rhi, sbias);
      else if constexpr (D >= 4) WK::template sums<2, 3, P>(A, H, Ks, rlo, rhi, sbias);
#pragma unroll
      for (int j = 0; j < P; ++j) best[j] = WK::best_of(H[j], best[j], p.one);
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      if (rel < p.units_per) {
        if (p.unit_max) p.unit_max[rel] = best[j];
        if (!have || best[j] > best_all) { best_all = best[j]; best_u = (uint32_t)(p.unit_begin + rel); have = true; }
      }
    }
  }
  unsigned long long key = have ? make_key(best_all, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key) atomicMax(p.key + (BAT && cur_b > 0 ? cur_b : 0), key);
}

// Packed two-unit instances (single searches; LN_LDU8W_PK): L_3 with five paired rows and L_4 with
// four, up to 24 columns.
#ifndef LN_LDU8W_PK
#define LN_LDU8W_PK 1
#endif
#ifndef LN_LDU8W_PK_PR4
#define LN_LDU8W_PK_PR4 0            // L_3 with four paired rows (short suffixes: small searches)
#endif
#ifndef LN_LDU8W_PK_L4PR3
#define LN_LDU8W_PK_L4PR3 1          // L_4 with three paired rows (short suffixes, batches of small matrices)
#endif
#ifndef LN_LDU8W_PK_BAT
#define LN_LDU8W_PK_BAT 1
#endif
#ifndef LN_LDU8W_PK_MAXNW
#define LN_LDU8W_PK_MAXNW 8
#endif
template <int D, int NW, int PR>
__host__ __device__ constexpr bool w_has_pk() {
  return LN_LDU8W_PK && NW <= LN_LDU8W_PK_MAXNW &&
         ((D == 3 && PR == 5) || (D == 4 && PR == 4) || (LN_LDU8W_PK_PR4 && D == 3 && PR == 4) ||
          (LN_LDU8W_PK_L4PR3 && D == 4 && PR == 3));
}

// The walk with two units per lane and packed H (see sums_pk / op_add): same units, chunks, Gray
// control and reduction key as walk_ldu8w_kernel; a chunk is 64 consecutive units (unit j of lane l
// = chunk base + 32 j + l).
// batched packed instances (f3, up to 24 columns): L_3 with four or five paired rows, L_4 with four
template <int D, int NW, int PR>
__host__ __device__ constexpr bool w_has_pk_bat() {
  return LN_LDU8W_PK && LN_LDU8W_PK_BAT && NW <= 6 &&
         ((D == 3 && (PR == 5 || PR == 4)) || (D == 4 && (PR == 4 || (LN_LDU8W_PK_L4PR3 && PR == 3))));
}

template <int D, int NW, int PR, bool BAT = false>
__global__ void __launch_bounds__(kBlockW, (w_minb<D, NW, PR>()))
walk_ldu8w_pk_kernel(const WalkParams p, const uint32_t* __restrict__ gTab, const int32_t* __restrict__ gInit) {
  using WK = LdW<D, NW, PR, true>;
  constexpr int P = 2;
  constexpr int RD = WK::RD, RW = WK::RW, CW = 4 * NW, NS = WK::NS;
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int sw = p.s - PR;
  uint32_t* sBias = sT + sw * RD;                 // set-major: sBias[m * RW + q], kappas at NS * RW
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sT);
  const uint32_t sbias = (uint32_t)__cvta_generic_to_shared(sBias);
  const uint32_t k16 = p.one << 16;
  uint32_t nwords = 1;
  for (int i = 0; i < sw; ++i) nwords *= D;
  // matrix mb's delta table, set-major bias words and kappa sums -> shared memory
  auto stage = [&](int mb) {
    __syncwarp();
    const uint32_t* biasRec = reinterpret_cast<const uint32_t*>(gInit + mb * p.init_stride + (p.k + 3) * CW);
    const uint32_t* src = gTab + mb * p.tab_stride;
    for (int i = lane; i < sw * RD; i += 32) sT[i] = src[i];
    for (int i = lane; i < NS * RW; i += 32) {
      const int m = i / RW, q = i % RW;
      sBias[i] = q < NW ? biasRec[m * NW + q] : 0u;
    }
    for (int m = lane; m < NS; m += 32) sBias[NS * RW + m] = biasRec[NS * NW + m];
    __syncwarp();
  };
  int32_t best_all = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  // BAT (batched launches): chunk ch -> matrix ch / CPM, as walk_ldu8w_kernel
  const int64_t CPM = (p.units_per + 32 * P - 1) / (32 * P);
  const int64_t nchunks = BAT ? CPM * p.batch : CPM;
  int cur_b = BAT ? -1 : 0;
  if constexpr (!BAT) stage(0);
  for (int64_t ch = blockIdx.x; ch < nchunks; ch = next_chunk(ch, p.chunk_ctr, lane)) {
    int64_t lc = ch;
    const int32_t* gI = gInit;
    if constexpr (BAT) {
      const int mb = (int)(ch / CPM);
      lc = ch - (int64_t)mb * CPM;
      gI = gInit + mb * p.init_stride;
      if (mb != cur_b) {
        if (cur_b >= 0) {                          // flush the previous matrix's key
          unsigned long long key = have ? make_key(best_all, best_u) : 0ull;
          key = warp_max_u64(key);
          if (lane == 0 && key) atomicMax(p.key + cur_b, key);
          best_all = INT32_MIN; have = false;
        }
        stage(mb);
        cur_b = mb;
      }
    }
    uint32_t A[P][D][NW];
    int32_t H[NS][D];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      const int64_t u = p.unit_begin + (rel < p.units_per ? rel : 0);
      uint64_t lab = 0;
      if (p.prefix_table) lab = p.prefix_table[u - p.unit_begin];
      else for (int x = 0; x <= p.k; ++x) lab |= (uint64_t)prefix_digit(p, u, x) << (p.pbits * x);
      const uint64_t lmask = (1ull << p.pbits) - 1ull;
      const uint32_t* pkRec = reinterpret_cast<const uint32_t*>(gI + (p.k + 3) * CW) + NS * NW + NS;
      const uint32_t* stRec = pkRec + (p.k + 1) * NW;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        A[j][0][q] = __ldg(stRec + q);
        const uint32_t sg = __ldg(stRec + NW + q);
#pragma unroll
        for (int g = 1; g < D; ++g) A[j][g][q] = sg;
      }
      for (int x = 0; x <= p.k; ++x) {
        const int dig = (int)((lab >> (p.pbits * x)) & lmask);
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          const uint32_t w = __ldg(pkRec + x * NW + q);
#pragma unroll
          for (int g = 0; g < D; ++g) A[j][g][q] += (dig == g) ? w : 0u;
        }
      }
#pragma unroll
      for (int g = 0; g < D; ++g)
#pragma unroll
        for (int m = 0; m < NS; ++m) {
          uint32_t h = sBias[NS * RW + m];
#pragma unroll
          for (int q = 0; q < NW; ++q) h = w_sad4(A[j][g][q], sBias[m * RW + q], h);
          H[m][g] = j == 0 ? (int32_t)h : (int32_t)((uint32_t)H[m][g] | (h << 16));   // unit j in half j
        }
    }
    int32_t best = WK::best_of(H, 0, p.one);       // both units' start words (every value >= 0)
    uint32_t t = 0, jj = 0;
    for (uint32_t w = 1; w < nwords; ++w) {
      uint32_t i, from, to;
      if (++jj == D) { jj = 0; ++t; }
      if (jj == 0) {
        dary_block_start<D>(t, &i, &from, &to);
      } else {
        i = 0;
        const bool odd = (t & 1u) != 0;
        from = odd ? D - jj : jj - 1;
        to = odd ? D - 1 - jj : jj;
      }
      const uint32_t srow = sbase + 4u * i * (uint32_t)RD;
      const uint32_t rlo = from < to ? srow + 4u * (uint32_t)RW : srow;
      const uint32_t rhi = from < to ? srow : srow + 4u * (uint32_t)RW;
      const uint32_t lo = from < to ? from : to;
      if (lo == 0) sums_pk<D, NW, PR, 0, 1>(A, H, rlo, rhi, sbias, k16);
      else if (D == 3 || lo == 1) sums_pk<D, NW, PR, 1, 2>(A, H, rlo, rhi, sbias, k16);
      else if constexpr (D >= 4) sums_pk<D, NW, PR, 2, 3>(A, H, rlo, rhi, sbias, k16);
      best = WK::best_of(H, best, p.one);
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      const int32_t bj = (int32_t)(j == 0 ? ((uint32_t)best & 0xFFFFu) : ((uint32_t)best >> 16));
      if (rel < p.units_per) {
        if (p.unit_max) p.unit_max[rel] = bj;
        if (!have || bj > best_all) { best_all = bj; best_u = (uint32_t)(p.unit_begin + rel); have = true; }
      }
    }
  }
  unsigned long long key = have ? make_key(best_all, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key) atomicMax(p.key + (BAT && cur_b > 0 ? cur_b : 0), key);
}

template <int NW, int PR>
size_t w_smem(int s) { return sizeof(uint32_t) * (size_t)((s - PR) * 2 * w_pad4(NW) + (1 << PR) * (w_pad4(NW) + 1)); }

template <int D, int NW, int PR>
cudaError_t launch_w(const WalkParams& p, const uint32_t* tab, const int32_t* init, int grid, cudaStream_t st) {
  const size_t sm = w_smem<NW, PR>(p.s);
  if (p.batch > 1) {                     // batched instances: <= 24 columns (the small-matrix regime)
    if constexpr (w_has_pk_bat<D, NW, PR>()) {
      cudaError_t e = ensure_dyn_smem((const void*)walk_ldu8w_pk_kernel<D, NW, PR, true>, sm);
      if (e != cudaSuccess) return e;
      walk_ldu8w_pk_kernel<D, NW, PR, true><<<grid, kBlockW, sm, st>>>(p, tab, init);
      return cudaGetLastError();
    }
    if constexpr (NW <= 6) {
      cudaError_t e = ensure_dyn_smem((const void*)walk_ldu8w_kernel<D, NW, PR, true>, sm);
      if (e != cudaSuccess) return e;
      walk_ldu8w_kernel<D, NW, PR, true><<<grid, kBlockW, sm, st>>>(p, tab, init);
      return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
  }
  if constexpr (w_has_pk<D, NW, PR>()) {
    cudaError_t e = ensure_dyn_smem((const void*)walk_ldu8w_pk_kernel<D, NW, PR>, sm);
    if (e != cudaSuccess) return e;
    walk_ldu8w_pk_kernel<D, NW, PR><<<grid, kBlockW, sm, st>>>(p, tab, init);
    return cudaGetLastError();
  }
  cudaError_t e = ensure_dyn_smem((const void*)walk_ldu8w_kernel<D, NW, PR>, sm);
  if (e != cudaSuccess) return e;
  walk_ldu8w_kernel<D, NW, PR><<<grid, kBlockW, sm, st>>>(p, tab, init);
  return cudaGetLastError();
}

template <int D, int NW, int PR>
int occ_w(int s) {
  const size_t sm = w_smem<NW, PR>(s);
  const int nb = occupancy_cached((const void*)walk_ldu8w_kernel<D, NW, PR>, kBlockW, sm);
  return nb;
}

template <int D, int NW, int PR>
int upl_w() { return w_units<NW, PR>(); }

template <int D, int NW, int PR>
int pk_w() { return w_has_pk<D, NW, PR>() ? 1 : 0; }

}  // namespace

#ifdef LN_LDU8W_PART
// One translation unit per label count (LN_LDU8W_D) and half of the column range
// (LN_LDU8W_PART 0: 1-6 packed words, <= 24 columns; 1: 7-12), compiled in parallel.
#define LN_LDU8W_SWITCH(NW_, FN, PR, ...)                                                          \
  if constexpr (LN_LDU8W_PART == 0) {                                                              \
    switch (NW_) {                                                                                 \
      case 1: return FN<LN_LDU8W_D, 1, PR>(__VA_ARGS__); case 2: return FN<LN_LDU8W_D, 2, PR>(__VA_ARGS__); \
      case 3: return FN<LN_LDU8W_D, 3, PR>(__VA_ARGS__); case 4: return FN<LN_LDU8W_D, 4, PR>(__VA_ARGS__); \
      case 5: return FN<LN_LDU8W_D, 5, PR>(__VA_ARGS__); case 6: return FN<LN_LDU8W_D, 6, PR>(__VA_ARGS__); \
      default: break;                                                                              \
    }                                                                                              \
  } else {                                                                                         \
    switch (NW_) {                                                                                 \
      case 7: return FN<LN_LDU8W_D, 7, PR>(__VA_ARGS__);   case 8: return FN<LN_LDU8W_D, 8, PR>(__VA_ARGS__);   \
      case 9: return FN<LN_LDU8W_D, 9, PR>(__VA_ARGS__);   case 10: return FN<LN_LDU8W_D, 10, PR>(__VA_ARGS__); \
      case 11: return FN<LN_LDU8W_D, 11, PR>(__VA_ARGS__); case 12: return FN<LN_LDU8W_D, 12, PR>(__VA_ARGS__); \
      default: break;                                                                              \
    }                                                                                              \
  }
// paired rows compiled per label count: L_3 3-5, L_4 3-4 (64 H sums per unit at four)
#if LN_LDU8W_D == 3 && LN_LDU8W_MAXPR >= 5
#define LN_LDU8W_PRS(FN, ...)                                                                      \
  if (pr == 5) { LN_LDU8W_SWITCH(NW, FN, 5, __VA_ARGS__) }                                         \
  else if (pr == 4) { LN_LDU8W_SWITCH(NW, FN, 4, __VA_ARGS__) }                                    \
  else if (pr == 3) { LN_LDU8W_SWITCH(NW, FN, 3, __VA_ARGS__) }
#else
#define LN_LDU8W_PRS(FN, ...)                                                                      \
  if (pr == 4) { LN_LDU8W_SWITCH(NW, FN, 4, __VA_ARGS__) }                                         \
  else if (pr == 3) { LN_LDU8W_SWITCH(NW, FN, 3, __VA_ARGS__) }
#endif

template <>
cudaError_t walk_ldu8w_launch_part<LN_LDU8W_D, LN_LDU8W_PART>(const WalkParams& p, const uint32_t* tab,
                                                               const int32_t* init, int grid, cudaStream_t st, int NW,
                                                               int pr) {
  LN_LDU8W_PRS(launch_w, p, tab, init, grid, st)
  return cudaErrorInvalidValue;
}

template <>
int walk_ldu8w_upl_part<LN_LDU8W_D, LN_LDU8W_PART>(int NW, int pr) {
  LN_LDU8W_PRS(upl_w)
  return 1;
}

template <>
int walk_ldu8w_pk_part<LN_LDU8W_D, LN_LDU8W_PART>(int NW, int pr) {
  LN_LDU8W_PRS(pk_w)
  return 0;
}

template <>
int walk_ldu8w_occ_part<LN_LDU8W_D, LN_LDU8W_PART>(int NW, int pr, int s) {
  LN_LDU8W_PRS(occ_w, s)
  return 0;
}
#endif

}  // namespace lnorm
