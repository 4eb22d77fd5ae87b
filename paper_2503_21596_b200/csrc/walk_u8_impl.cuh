// Hot binary Gray walk with the column sums packed FOUR per register as offset
// bytes: L_1, L_marg, L_2.
//
// Same units, warp-uniform Gray control and lexicographic reduction key as the
// other binary walks (walk_pair16_impl.cuh): a unit fixes rows 0..k and walks its
// s suffix rows (digit b <-> row r-1-b) in reflected Gray order (Eq. 9,
// Table 1), each step adding ONE row of M to the column sums (Eq. 12: +-2 M_rho
// for L_1 / L_marg; Eqs. 18-19 with d = 2: m_0 -/+= M_rho for L_2).
//
// Byte encoding.  Within one unit column y only moves inside a window fixed by
// the unit's prefix part P_y (rows 0..k) and the suffix rows' W_y = sum_{suffix x}
// |M_xy|:  L_1: m_y in [P_y - W_y, P_y + W_y];  L_2: m_0y in [P_y + N_y, P_y + N_y + W_y]
// with N_y = sum_{suffix x} min(M_xy, 0).  With Lo_y the window's low end, the lane
// keeps a_y = m_y - Lo_y in [0, 2 W_y] (L_1) or [0, W_y] (L_2): one unsigned byte as
// long as the window is at most 255 wide (the exactness guard, checked on the host).
// Four bytes share a 32-bit register and ONE 32-bit add of the packed step delta
// sum_e 256^e delta_e updates all four exactly (no byte ever leaves [0, 255], so no
// carry or borrow crosses a byte).  Every |.| is then one byte of
//     |m_y| = |a_y - B_y| + kappa_y,   B_y = clamp(c_y, 0, 255),  kappa_y = |c_y - B_y|,
// with c_y = -Lo_y (for |m_y|) or T_y - Lo_y (for |m_1y| = |T_y - m_0y|, L_2), because a_y
// stays on one side of c_y whenever c_y is outside [0, 255].  VABSDIFF4.U8.ACC adds the
// four |a - B| of a register to a 32-bit accumulator in one instruction, so a Gray
// step costs one IADD (FMA-heavy pipe) + one VABSDIFF4 (ALU pipe) per FOUR columns
// (L_2: + one more VABSDIFF4 for m_1), and the unit's value is acc + K, K = sum kappa.
// L_marg's column 0 is linear (Eq. 2): it is kept as a byte too with B_0 = 0 and
// kappa_0 = Lo_0, so that |a_0 - 0| + Lo_0 = m_0.  Per unit, B and K are computed once
// (the paper's per-thread initial product) and the start bytes a_y are
// the same for every unit (a uniform table).
#include "common.cuh"

#ifndef LN_BIN_MODE
#error "define LN_BIN_MODE before including walk_u8_impl.cuh"
#endif

namespace lnorm {

namespace {

constexpr int kBlockU8 = 32;

#ifndef LN_U8_BUDGET
#define LN_U8_BUDGET 1800
#endif
#ifndef LN_U8_MINB
#define LN_U8_MINB 16
#endif

__host__ __device__ constexpr int u8_cctz(int j) { return (j & 1) ? 0 : (j & 2) ? 1 : (j & 4) ? 2 : 3; }
__host__ __device__ constexpr int u8_pad4(int x) { return (x + 3) & ~3; }

// d = acc + sum over the 4 bytes of |a_b - b_b| (unsigned bytes): VABSDIFF4.U8.ACC
__device__ __forceinline__ uint32_t sad4(uint32_t a, uint32_t b, uint32_t acc) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(acc));
  return d;
}

// Per-byte |a_b - b_b| (no accumulate): VABSDIFF4.U8 with the full byte mask
__device__ __forceinline__ uint32_t absdiff4_bytes(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(0u));
  return d;
}
// acc + sum_b x_b * w_b over unsigned bytes: IDP.4A (FMA-heavy pipe), used with a 0/1 byte mask w
__device__ __forceinline__ uint32_t dp4a_u(uint32_t x, uint32_t w, uint32_t acc) {
  uint32_t d;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(w), "r"(acc));
  return d;
}

// Merged last word (MRG, LN_U8_MERGE): when the last packed word holds only one or two live
// columns (c mod 4 = 1 or 2 -- e.g. 42 columns = 10 full words + 2), units 2i and 2i+1 of a lane
// group keep those columns in ONE register (unit 2i in bytes 0-1, unit 2i+1 in bytes 2-3; their
// bias bytes are shared, the delta record's last word is duplicated into bytes 2-3).  One
// per-byte VABSDIFF4 (ALU) then serves both units, and two IDP.4A with the byte masks 0x0101 /
// 0x01010000 (FMA-heavy pipe) add each unit's two bytes to its own sum -- the ALU pipe, which
// binds, does 21 instead of 22 VABSDIFF4 per unit and word at 42 columns.  Measured 3.4 % SLOWER
// on 42x42 L_1 (1490 vs 1441 ms, profiles/r02/ab_u8_merge.log): off by default (no instances).
#ifndef LN_U8_MERGE
#define LN_U8_MERGE 0
#endif

// Self-check build (`python -m paper_2503_21596_b200.build --selfcheck`): after
// every Gray step, unit 0 of every lane recomputes its word's NS strategy values FROM SCRATCH
// (Eq. 1 / Eq. 2 / Eq. 6 over all r rows of the oriented M, no bytes, no Gray state) and counts
// any difference in p.counter (unused by this kernel otherwise); the host turns a nonzero count
// into LNORM_EINTERNAL.  The product build compiles it out (LN_SELFCHECK = 0).
#ifndef LN_SELFCHECK
#define LN_SELFCHECK 0
#endif

template <int MODE>
__device__ int32_t u8_scratch_value(const WalkParams& p, int64_t u, uint32_t w, int PR, int h) {
  const uint32_t g = w ^ (w >> 1);
  int32_t val = 0;
  for (int y = 0; y < p.c; ++y) {
    int32_t m0 = 0, m1 = 0;                   // L_1 / L_marg: sum a_x M_xy; L_2: the two groups
    for (int x = 0; x < p.r; ++x) {
      int dig;
      if (x <= p.k) dig = prefix_digit(p, u, x);
      else if (x < p.r - PR) dig = (int)((g >> (p.r - 1 - PR - x)) & 1u);   // walked digit b <-> row r-1-PR-b
      else dig = (h >> (p.r - 1 - x)) & 1;                                   // paired row r-1-i <-> bit i of h
      const int32_t v = p.M[(int64_t)x * p.c + y];
      if (MODE == MODE_LD) { if (dig) m1 += v; else m0 += v; }
      else m0 += dig ? -v : v;
    }
    if (MODE == MODE_LD) val += abs(m0) + abs(m1);
    else if (MODE == MODE_MARG && y == 0) val += m0;
    else val += abs(m0);
  }
  return val;
}

template <int MODE, int NW>
struct U8Layout {
  static constexpr int G = (MODE == MODE_LD) ? 2 : 1;   // bias sets: |m_0| (and |m_1| for L_2)
  static constexpr int RW = u8_pad4(NW);                // words per packed delta record
  static constexpr int CW = 4 * NW;                     // int32 columns per init row
};

#ifndef LN_U8_P
#define LN_U8_P 4
#endif
#ifndef LN_U8_MAD
#define LN_U8_MAD 0
#endif
#ifndef LN_U8_CHAINS
#define LN_U8_CHAINS 2
#endif
// LN_U8_PAIR: the last row r-1 is not walked; every walked word evaluates both of its
// signs (strategies A: a_{r-1} = +1 / group 0, B: -1 / group 1) against a second set
// of bias words, B'_y = clamp(c_y + scale rho_y): one IADD per four columns serves two
// strategies (walk_ldu8.cu applies the same pairing to the d-ary walk).
#ifndef LN_U8_PAIR
#define LN_U8_PAIR 1
#endif
// paired rows per mode (L_2 holds two bias sets per strategy already: at most one row)
template <int MODE>
__host__ __device__ constexpr int u8_pr() { return MODE == MODE_LD ? (LN_U8_PAIR < 1 ? LN_U8_PAIR : 1) : LN_U8_PAIR; }

// units per lane: the row quad loaded once per step is shared by P units
#ifndef LN_U8_PWIDE
#define LN_U8_PWIDE 1
#endif
// Lanes per unit: wide L_1 / L_marg rows (more than 128 columns) split over a lane PAIR
// (each lane holds half of the words of the same units; the two partial sums of a strategy
// are combined with one SHFL), so a lane keeps two units sharing one bias set instead of one
// unit with its own (measured +7-9 % on 144-190 columns).  The second unit adds a prefix
// row to the byte window, so the planner falls back to the one-lane instance where that row
// no longer fits (48x192: k would exceed 31).  The 192-column lane-pair instance spills a
// few registers in its unit init (none inside the walk loop).
#ifndef LN_U8_LPU2
#define LN_U8_LPU2 1
#endif
#ifndef LN_U8_WIDE_EVEN
#define LN_U8_WIDE_EVEN 1
#endif
// resident blocks asked of ptxas for the wide lane-pair instances (10: 168 registers, a few
// spills in the unit init only; measured 3-4 % faster than the unbounded 244-register build on
// 144-160 columns, profiles/r02/ab_wide_rows.jsonl)
#ifndef LN_U8_MINB_LP
#define LN_U8_MINB_LP 10
#endif
// lanes per unit an instance can run with (the planner picks 2 where the byte guard allows
// the extra window row, else 1; both instances are compiled for those NW)
template <int MODE, int NW>
#ifndef LN_U8_LPU_FROM
#define LN_U8_LPU_FROM 33                // smallest word count with a lane-pair instance
#endif
__host__ __device__ constexpr int u8_lpu_max() { return (U8Layout<MODE, NW>::G == 1 && NW >= LN_U8_LPU_FROM && LN_U8_LPU2 && u8_pr<MODE>() >= 1) ? 2 : 1; }
template <int MODE, int NW, int LPU = 1>
__host__ __device__ constexpr int u8_units_per_lane() {
  return LPU == 2 ? (NW / 2 <= 8 ? 4 : 2)
       : U8Layout<MODE, NW>::G * NW <= 16 ? LN_U8_P
       : (U8Layout<MODE, NW>::G * NW <= 32 ? 2 : (U8Layout<MODE, NW>::G == 1 ? LN_U8_PWIDE : 1));
}

// packed byte update A + D; LN_U8_MAD: as IMAD D * one + A with `one` a kernel
// parameter (uniform register operand), pinning the add to the FMA-heavy pipe
__device__ __forceinline__ uint32_t u8_add(uint32_t a, uint32_t d, uint32_t one) {
#if LN_U8_MAD
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(d), "r"(one), "r"(a));
  return r;
#else
  (void)one;
  return a + d;
#endif
}

template <int MODE, int NW, int P>
__host__ __device__ constexpr int u8_step_instr() {
  return P * ((1 << u8_pr<MODE>()) * U8Layout<MODE, NW>::G + 1) * NW + P + U8Layout<MODE, NW>::RW / 4;
}

template <int MODE, int NW, int P>
__host__ __device__ constexpr int u8_unroll() {
  return u8_step_instr<MODE, NW, P>() * 16 <= LN_U8_BUDGET ? 4
       : u8_step_instr<MODE, NW, P>() * 8 <= LN_U8_BUDGET ? 3
       : u8_step_instr<MODE, NW, P>() * 4 <= LN_U8_BUDGET ? 2 : 1;
}

// PK: the running maxima of two units share one register as unsigned 16-bit halves (every value
// is a non-negative integer <= sum |M| <= 65535: L_1 and L_2, host-checked), so ONE VIMNMX3.U16x2
// serves the four strategies (two units x the paired row's two signs) of a walked word; the two
// values are packed by an IMAD (FMA-heavy pipe) -- half the epilogue's ALU instructions.
template <int MODE, int NW, int P, int LPU = 1, bool PK = false, bool MRG = false>
struct U8Step {
  // NW here = the words THIS lane holds (half of the unit's words when LPU = 2)
  static constexpr int PR = u8_pr<MODE>(), NS = 1 << PR;   // paired rows, bias sets
  static_assert(LPU == 1 || PR >= 1, "lane pairs need the paired epilogue");
  static constexpr int G = U8Layout<MODE, NW>::G, RW = U8Layout<MODE, NW>::RW;
  static constexpr int NB = NS * G * NW;        // bias words: set h (paired-row signs h) x group
  static_assert(!MRG || (G == 1 && LPU == 1 && PR >= 1 && P % 2 == 0 && NW >= 2 && !PK), "merged last word");
  // One Gray step: add the packed delta record at sbase + off to every unit's bytes,
  // re-accumulate sum |a - B| (and sum |a - B'| for the paired strategy), keep the max.
  // vout (self-check builds only, LN_SELFCHECK): receives unit 0's NS strategy values of the word
  static __device__ __forceinline__ void run(uint32_t (&A)[P][NW], const uint32_t (&B)[NB],
                                             const uint32_t (&K)[NS], int32_t (&best)[P], uint32_t sbase, int off,
                                             uint32_t one, int32_t* vout = nullptr) {
    uint32_t a0[P], a1[P], hs[P][NS][G];
#pragma unroll
    for (int v = 0; v < RW / 4; ++v) {
      const uint4 x4 = lds128(sbase + 4u * (uint32_t)(off + 4 * v));
      const uint32_t rq[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * v + e;
        if (MRG && i == NW - 1) {                  // the merged last word of unit pairs (2i, 2i+1)
#pragma unroll
          for (int j = 0; j < P; j += 2) {
            A[j][i] = u8_add(A[j][i], rq[e], one);
#pragma unroll
            for (int h = 0; h < NS; ++h) {
              const uint32_t x = absdiff4_bytes(A[j][i], B[h * NW + i]);
              hs[j][h][0] = dp4a_u(x, 0x00000101u, hs[j][h][0]);
              hs[j + 1][h][0] = dp4a_u(x, 0x01010000u, hs[j + 1][h][0]);
            }
          }
        } else if (i < NW) {
#pragma unroll
          for (int j = 0; j < P; ++j) {
            A[j][i] = u8_add(A[j][i], rq[e], one);
            if (PR >= 1) {
#pragma unroll
              for (int h = 0; h < NS; ++h)
#pragma unroll
                for (int gg = 0; gg < G; ++gg)
                  hs[j][h][gg] = sad4(A[j][i], B[(h * G + gg) * NW + i], i == 0 ? (gg == 0 ? K[h] : 0u) : hs[j][h][gg]);
            } else if (G == 2) {
              a0[j] = sad4(A[j][i], B[i], i == 0 ? K[0] : a0[j]);
              a1[j] = sad4(A[j][i], B[NW + i], i == 0 ? 0u : a1[j]);
            } else if (i == 0) {
              a0[j] = sad4(A[j][0], B[0], K[0]);
            } else if (LN_U8_CHAINS == 1) {
              a0[j] = sad4(A[j][i], B[i], a0[j]);
            } else if (i == 1) {
              a1[j] = sad4(A[j][1], B[1], 0u);
            } else if (i & 1) {
              a1[j] = sad4(A[j][i], B[i], a1[j]);
            } else {
              a0[j] = sad4(A[j][i], B[i], a0[j]);
            }
          }
        }
      }
    }
    if constexpr (PK && LPU == 2) {
      // lane pairs (PKL): the unit's two strategy values (paired row +/-) as u16 halves -> ONE SHFL and
      // one packed add join the two lanes' partial sums, one VIMNMX.U16x2 keeps both running maxima
      static_assert(PR == 1 && MODE == MODE_L1 && G == 1, "packed lane-pair join");
      const uint32_t k16 = one << 16;
#pragma unroll
      for (int j = 0; j < P; ++j) {
        uint32_t w;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(w) : "r"(hs[j][1][0]), "r"(k16), "r"(hs[j][0][0]));
        w += __shfl_xor_sync(0xffffffffu, w, 1);     // halves never carry: each is <= sum |M| <= 65535
        best[j] = (int32_t)__vmaxu2((uint32_t)best[j], w);
      }
    } else if constexpr (PK) {
      static_assert(!PK || (PR == 1 && LPU == 1 && P % 2 == 0 && MODE != MODE_MARG), "packed maxima");
      const uint32_t k16 = one << 16;                 // 65536 from a kernel parameter: IMAD, not LEA
#pragma unroll
      for (int j = 0; j < P; j += 2) {
        uint32_t w[NS];
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          const uint32_t lo = (G == 2) ? hs[j][h][0] + hs[j][h][1] : hs[j][h][0];
          const uint32_t hi = (G == 2) ? hs[j + 1][h][0] + hs[j + 1][h][1] : hs[j + 1][h][0];
          if (LN_SELFCHECK && j == 0 && vout) vout[h] = (int32_t)lo;
          asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(w[h]) : "r"(hi), "r"(k16), "r"(lo));
        }
        best[j / 2] = (int32_t)__vimax3_u16x2((uint32_t)best[j / 2], w[0], w[1]);
      }
    } else if (PR >= 1) {
#pragma unroll
      for (int j = 0; j < P; ++j) {
        int32_t v[NS];
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          v[h] = (G == 2) ? (int32_t)(hs[j][h][0] + hs[j][h][1]) : (int32_t)hs[j][h][0];
          if (LPU == 2) v[h] += __shfl_xor_sync(0xffffffffu, v[h], 1);   // partner lane: other half of the words
          if (LN_SELFCHECK && j == 0 && vout) vout[h] = v[h];
        }
#pragma unroll
        for (int h = 0; h < NS; h += 2) best[j] = __vimax3_s32(best[j], v[h], v[h + 1]);
      }
    } else if (G == 1 && (NW == 1 || LN_U8_CHAINS == 1)) {
#pragma unroll
      for (int j = 0; j < P; ++j) best[j] = max(best[j], (int32_t)a0[j]);
    } else {
#pragma unroll
      for (int j = 0; j < P; ++j) best[j] = __viaddmax_s32((int32_t)a0[j], (int32_t)a1[j], best[j]);
    }
  }
};

// Lane groups.  The P units of a lane are the P consecutive units of one aligned
// group g (units gP .. gP+P-1), which differ only in the last L = log2 P prefix rows
// k-L+1 .. k.  Those rows are counted in the byte window together with the suffix
// (window rows = the last s + L rows), so the P units share ONE set of bias words B
// and one K: consecutive VABSDIFF4 of the P units then read B from the operand
// reuse cache (two register-file reads per VABSDIFF4 instead of three, the
// register-bank limit measured in profiles/r01), and B costs NW registers per lane,
// not P*NW.  Slices that do not start or end on a group boundary (Algorithm 1 ranks,
// checkpoint chunks) mask the units outside [unit_begin, unit_begin + unit_count).
//
// Init records (global, int32), per matrix:
//   [0, (k+1)*CW)          prefix rows 0..k, columns padded to CW with zeros
//   [(k+1)*CW, +CW)        Lo_y - Ph_y over the window rows: -W_y (L_1, L_marg) or N_y (L_2)
//   [(k+2)*CW, +CW)        T_y = sum_x M_xy (L_2 only)
//   [(k+3)*CW, +CW)        a_y - delta_y at the start word: sum_suffix M_xy + W_y (L_1, L_marg)
//                          or sum_suffix M_xy - N_y (L_2); delta = the unit's low prefix rows
//   [(k+4)*CW, +CW)        scale * rho_y, rho = row r-1 (the paired row; scale 2 for L_1 / L_marg)
// resident warps per SM asked of ptxas: 16 (128 registers) where the lane's bytes and
// biases leave room for it without spilling, else 14 or 12, else no bound
#ifndef LN_U8_MINB_MID
#define LN_U8_MINB_MID 14
#endif
template <int MODE, int NW, int P>
__host__ __device__ constexpr int u8_foot() { return U8Layout<MODE, NW>::G * NW * (P + (1 << u8_pr<MODE>())); }
template <int MODE, int NW, int P, int LPU>
__host__ __device__ constexpr int u8_min_blocks() {
  return LPU == 2 ? (u8_foot<MODE, NW / 2, P>() <= 40 ? 12 : LN_U8_MINB_LP)
       : (U8Layout<MODE, NW>::G == 1 && u8_foot<MODE, NW, P>() <= 56) ? LN_U8_MINB
       : (U8Layout<MODE, NW>::G == 1 && u8_foot<MODE, NW, P>() <= 70) ? LN_U8_MINB_MID
       : ((u8_foot<MODE, NW, P>() <= 96 && P >= 4) || u8_foot<MODE, NW, P>() <= 54) ? 12 : 1;
}

// BAT: batched instance (f3, one launch over many matrices: chunk ch -> matrix mb = ch / CPM,
// local chunk lc; chunks never straddle matrices and a warp restages the delta table when it
// moves to the next matrix).  The single-search instance (BAT = false) keeps the table staged
// once and no per-chunk bookkeeping (the batch state costs registers the hot loop needs).
template <int MODE, int NW, int P, int LPU, bool BAT = false, bool PK = false, bool MRG = false>
__global__ void __launch_bounds__(kBlockU8, u8_min_blocks<MODE, NW, P, LPU>())
walk_u8_kernel(const WalkParams p, const uint32_t* __restrict__ gTab, const int32_t* __restrict__ gInit) {
  using LY = U8Layout<MODE, NW>;
  constexpr int G = LY::G, CW = LY::CW;
  constexpr int LG = (P >= 8) ? 3 : (P >= 4) ? 2 : (P == 2 ? 1 : 0);
  constexpr int NWL = NW / LPU;                    // LPU = lanes per unit; words held by one lane
  constexpr int RWL = u8_pad4(NWL);                // its slice of a delta record (16B aligned)
  constexpr int RREC = LPU * RWL;                  // words per delta record
  constexpr int GPW = 32 / LPU;                    // lane groups per warp
  constexpr int K = u8_unroll<MODE, NWL, P>();
  using STEP = U8Step<MODE, NWL, P, LPU, PK, MRG>;
  constexpr int NB = STEP::NB;
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int half = (LPU == 2) ? (lane & 1) : 0, slot = lane / LPU;
  constexpr int PR = STEP::PR, NS = STEP::NS;
  const int sw = p.s - PR;                         // walked digits (the last PR rows are paired, not walked)
  const int total = 2 * sw * RREC;
  if constexpr (!BAT) {
    for (int i = lane; i < total; i += 32) sT[i] = gTab[i];
    __syncwarp();
  }
  const uint32_t nblk = 1u << (sw - K);
  const int kh = p.k - LG;                         // last row of the shared (high) prefix part
  int32_t best_all = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  // units of one matrix: [unit_begin, unit_begin + units_per) (= the launch's range unless batched)
  const int64_t u_end = p.unit_begin + p.units_per;
  const int64_t g0 = p.unit_begin / P, g_end = (u_end + P - 1) / P;
  const int64_t CPM = (g_end - g0 + GPW - 1) / GPW;
  const int64_t nchunks = BAT ? CPM * p.batch : CPM;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sT);
  int cur_b = BAT ? -1 : 0;
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
        __syncwarp();
        const uint32_t* src = gTab + mb * p.tab_stride;
        for (int i = lane; i < total; i += 32) sT[i] = src[i];
        __syncwarp();
        cur_b = mb;
      }
    }
    const int32_t* loRec = gI + (p.k + 1) * CW;
    const int32_t* tRec = loRec + CW;
    const int32_t* abRec = tRec + CW;
    const int32_t* rhoRec = abRec + CW;
    const int64_t g = g0 + lc * GPW + slot;
    const int64_t uh = min(max(g * P, p.unit_begin), u_end - 1);   // a valid unit of the group
    uint32_t A[P][NWL];
    uint32_t B[NB];
    uint32_t Kc[NS];
    int32_t best[P];
    // ---- lane init (PAPER.md:253's per-thread product): shared high part -> B, K;
    //      per unit: its low prefix rows -> start bytes
    {
      uint64_t neg = 0;                            // bit x: digit of row x (0..kh) is 1
      for (int x = 0; x <= kh; ++x) neg |= (uint64_t)(prefix_digit(p, uh, x) != 0) << x;
      int32_t kap[NS];
#pragma unroll
      for (int h = 0; h < NS; ++h) kap[h] = 0;
#pragma unroll
      for (int ql = 0; ql < NWL; ++ql) {
        const int q = half * NWL + ql;             // global word of this lane's column slice
        int32_t Pv[4] = {0, 0, 0, 0};              // high prefix part of columns 4q..4q+3
        for (int x = 0; x <= kh; ++x) {
          // L_1 / L_marg: a_x = +1 (digit 0) or -1; L_2: only rows in group 0 count
          const int dig = (int)((neg >> x) & 1ull);
          const int32_t f = (MODE == MODE_LD) ? 1 - dig : 1 - 2 * dig;
          const int4 v = __ldg(reinterpret_cast<const int4*>(gI + x * CW) + q);
          Pv[0] += f * v.x; Pv[1] += f * v.y; Pv[2] += f * v.z; Pv[3] += f * v.w;
        }
        uint32_t w[NS][2];                         // [paired-row signs][bias set]
#pragma unroll
        for (int h = 0; h < NS; ++h) w[h][0] = w[h][1] = 0u;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int y = 4 * q + e;
          const int32_t lo = Pv[e] + __ldg(loRec + y);
          int32_t srho[PR > 0 ? PR : 1];
#pragma unroll
          for (int i = 0; i < PR; ++i) srho[i] = __ldg(rhoRec + i * CW + y);
#pragma unroll
          for (int h = 0; h < NS; ++h) {           // bit i of h: paired row r-1-i flipped (m -= scale rho_i)
            int32_t sh = 0;
#pragma unroll
            for (int i = 0; i < PR; ++i) sh += ((h >> i) & 1) ? srho[i] : 0;
            int32_t& kk = kap[h];
            const int32_t c0 = -lo + sh;
            int32_t b0;
            if (MODE == MODE_MARG && y == 0) {     // linear column: m_0 = a_0 + Lo_0 (- 2 rho_0)
              b0 = 0;
              kk += lo - sh;
            } else {
              b0 = min(max(c0, 0), 255);
              kk += abs(c0 - b0);
            }
            w[h][0] |= (uint32_t)b0 << (8 * e);
            if (G == 2) {
              const int32_t c1 = __ldg(tRec + y) - lo + sh;
              const int32_t b1 = min(max(c1, 0), 255);
              kk += abs(c1 - b1);
              w[h][1] |= (uint32_t)b1 << (8 * e);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          B[h * G * NWL + ql] = w[h][0];
          if (G == 2) B[h * G * NWL + NWL + ql] = w[h][1];
        }
      }
#pragma unroll
      for (int h = 0; h < NS; ++h) Kc[h] = (uint32_t)kap[h];
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      int64_t u = g * P + j;
      if (u < p.unit_begin || u >= u_end) u = uh; // masked unit: walk a valid copy
      int lowdig[LG > 0 ? LG : 1];
#pragma unroll
      for (int b = 0; b < LG; ++b) lowdig[b] = prefix_digit(p, u, kh + 1 + b);
#pragma unroll
      for (int ql = 0; ql < NWL; ++ql) {
        const int q = half * NWL + ql;
        int32_t a[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) a[e] = __ldg(abRec + 4 * q + e);
#pragma unroll
        for (int b = 0; b < LG; ++b) {
          const int dig = lowdig[b];
          const int32_t f = (MODE == MODE_LD) ? 1 - dig : 1 - 2 * dig;
          const int4 v = __ldg(reinterpret_cast<const int4*>(gI + (kh + 1 + b) * CW) + q);
          a[0] += f * v.x; a[1] += f * v.y; a[2] += f * v.z; a[3] += f * v.w;
        }
        A[j][ql] = (uint32_t)(a[0] & 0xFF) | ((uint32_t)(a[1] & 0xFF) << 8) | ((uint32_t)(a[2] & 0xFF) << 16) |
                   ((uint32_t)(a[3] & 0xFF) << 24);
      }
      // value of the unit's start word (strategy A, and B when paired)
      int32_t v0 = 0;
#pragma unroll
      for (int h = 0; h < NS; ++h) {
        uint32_t acc = Kc[h];
#pragma unroll
        for (int q = 0; q < NWL; ++q) {
          acc = sad4(A[j][q], B[h * G * NWL + q], acc);
          if (G == 2) acc = sad4(A[j][q], B[h * G * NWL + NWL + q], acc);
        }
        if (LPU == 2) acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if constexpr (PK && LPU == 2) v0 = h == 0 ? (int32_t)acc : (int32_t)((uint32_t)v0 | (acc << 16));
        else v0 = h == 0 ? (int32_t)acc : max(v0, (int32_t)acc);
      }
      best[j] = v0;
    }
    if constexpr (MRG) {                               // merge the last words: unit 2i+1's bytes 0-1 -> 2i's bytes 2-3
#pragma unroll
      for (int h = 0; h < NS; ++h) {
        const uint32_t b = B[h * NWL + NWL - 1] & 0xFFFFu;
        B[h * NWL + NWL - 1] = b | (b << 16);
      }
#pragma unroll
      for (int j = 0; j < P; j += 2) A[j][NWL - 1] = (A[j][NWL - 1] & 0xFFFFu) | (A[j + 1][NWL - 1] << 16);
    }
    if constexpr (PK && LPU == 1) {                    // two units' maxima per register (lo: unit 2i)
#pragma unroll
      for (int i = 0; i < P / 2; ++i) best[i] = (int32_t)(((uint32_t)best[2 * i + 1] << 16) | (uint32_t)best[2 * i]);
    }
    // ---- the walk: 2^s - 1 Gray steps (low K digits unrolled, Table 1's ruler pattern)
    for (uint32_t t = 0; t < nblk; ++t) {
#if LN_SELFCHECK
      int32_t vchk[NS];
      const int64_t u0 = [&] { int64_t u = g * P; return (u < p.unit_begin || u >= u_end) ? uh : u; }();
      auto check = [&](uint32_t w) {
        if (BAT) return;                           // (batched instances: not self-checked)
        for (int h = 0; h < NS; ++h)
          if (u8_scratch_value<MODE>(p, u0, w, PR, h) + p.selfcheck_delta != vchk[h]) atomicAdd(p.counter, 1ull);
      };
#endif
      if (t != 0) {                                    // block start: digit K + ctz(t)
        const int tz = __ffs((int)t) - 1;
        const int b = K + tz;
        const int sg = 1 ^ (int)((t >> (tz + 1)) & 1u);
#if LN_SELFCHECK
        STEP::run(A, B, Kc, best, sbase, (2 * b + sg) * RREC + half * RWL, p.one, vchk);
        check(t << K);
#else
        STEP::run(A, B, Kc, best, sbase, (2 * b + sg) * RREC + half * RWL, p.one);
#endif
      }
#pragma unroll
      for (int jj = 1; jj < (1 << K); ++jj) {
        const int b = u8_cctz(jj);
        const int sg = (b < K - 1) ? (1 ^ ((jj >> (b + 1)) & 1)) : (1 ^ (int)(t & 1u));
#if LN_SELFCHECK
        STEP::run(A, B, Kc, best, sbase, (2 * b + sg) * RREC + half * RWL, p.one, vchk);
        check((t << K) | (uint32_t)jj);
#else
        STEP::run(A, B, Kc, best, sbase, (2 * b + sg) * RREC + half * RWL, p.one);
#endif
      }
    }
    if constexpr (PK && LPU == 1) {                    // unpack (back to front: slot i holds units 2i, 2i+1)
#pragma unroll
      for (int i = P / 2 - 1; i >= 0; --i) {
        const uint32_t w = (uint32_t)best[i];
        best[2 * i + 1] = (int32_t)(w >> 16);
        best[2 * i] = (int32_t)(w & 0xFFFFu);
      }
    } else if constexpr (PK) {                         // lane pairs: the max of the two signs' maxima
#pragma unroll
      for (int j = 0; j < P; ++j) best[j] = (int32_t)max((uint32_t)best[j] & 0xFFFFu, (uint32_t)best[j] >> 16);
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t u = g * P + j;
      if (u >= p.unit_begin && u < u_end && half == 0) {
        if (p.unit_max) p.unit_max[u - p.unit_begin] = best[j];
        if (!have || best[j] > best_all) { best_all = best[j]; best_u = (uint32_t)(u >> p.key_shift); have = true; }
      }
    }
  }
  unsigned long long key = have ? make_key(best_all, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key) atomicMax(p.key + (BAT && cur_b > 0 ? cur_b : 0), key);
}

// Delta table (walked digit b <-> row r-1-b, sign sg = new digit value) and init
// records; the byte window covers the last s + lg rows (lg = log2 of the lane group).
template <int MODE>
__global__ void build_u8_kernel(const int32_t* M, int r, int c, int NW, int k, int s, int lg, int lpu, uint32_t* tab,
                                int32_t* init, int64_t m_stride, int64_t tab_stride, int64_t init_stride,
                                unsigned long long* chunk_ctr, int mrg) {
  if (chunk_ctr && blockIdx.x == 0 && threadIdx.x == 0) *chunk_ctr = 0ull;   // the next walk's chunk schedule
  M += blockIdx.x * m_stride;              // one block per matrix of a batch
  tab += blockIdx.x * tab_stride;
  init += blockIdx.x * init_stride;
  // a record holds lpu slices of pad4(NW / lpu) words (one per lane of a lane pair)
  const int NWL = NW / lpu, RWL = u8_pad4(NWL), RW = lpu * RWL, CW = 4 * NW;
  const int scale = (MODE == MODE_LD) ? 1 : 2;
  const int tid = threadIdx.x;
  const int PR = u8_pr<MODE>();
  const int sw = s - PR;
  for (int rec = tid; rec < 2 * sw; rec += blockDim.x) {
    const int b = rec >> 1, sg = rec & 1;
    const int32_t* row = M + (int64_t)(r - 1 - PR - b) * c;   // walked digit b
    const int f = sg ? -scale : scale;     // digit -> 1: a_x = -1 (m -= 2M) or group 1 (m_0 -= M)
    for (int i = 0; i < RW; ++i) {
      const int h = i / RWL, ql = i % RWL, q = h * NWL + ql;   // slice h, word q of the row
      uint32_t w = 0;
      for (int e = 0; e < 4; ++e) {
        const int y = 4 * q + e;
        const int32_t v = (ql < NWL && y < c) ? f * row[y] : 0;
        w += (uint32_t)v << (8 * e);       // packed signed delta sum_e 256^e delta_e (mod 2^32)
      }
      if (mrg && q == NW - 1) w *= 65537u;   // merged last word: the same delta for bytes 2-3 (D + 2^16 D)
      tab[rec * RW + i] = w;
    }
  }
  for (int i = tid; i < (k + 1) * CW; i += blockDim.x) {
    const int x = i / CW, y = i % CW;
    init[i] = y < c ? M[(int64_t)x * c + y] : 0;
  }
  for (int y = tid; y < CW; y += blockDim.x) {
    int32_t W = 0, N = 0, T = 0, Ssuf = 0;
    if (y < c)
      for (int x = 0; x < r; ++x) {
        const int32_t v = M[(int64_t)x * c + y];
        T += v;
        if (x >= r - s - lg) { W += abs(v); N += min(v, 0); }   // window rows
        if (x >= r - s) Ssuf += v;                             // suffix rows (all digit 0 at the start)
      }
    init[(k + 1) * CW + y] = (MODE == MODE_LD) ? N : -W;
    init[(k + 2) * CW + y] = (MODE == MODE_LD) ? T : 0;
    init[(k + 3) * CW + y] = (MODE == MODE_LD) ? Ssuf - N : Ssuf + W;
    for (int i = 0; i < PR; ++i) init[(k + 4 + i) * CW + y] = y < c ? scale * M[(int64_t)(r - 1 - i) * c + y] : 0;
  }
}

template <int MODE, int NW, int LPU>
size_t u8_smem(int s) { return sizeof(uint32_t) * (size_t)(2 * (s - u8_pr<MODE>()) * LPU * u8_pad4(NW / LPU)); }

// batched instances exist for the small-matrix regime only (<= 32 columns, one lane per unit)
constexpr int kU8BatchMaxNW = 8;
// packed-maxima instances (LN_U8_PACKMAX, U8Step PK) for up to 64 columns (four units per lane).
// Off: measured 5.6 % SLOWER on 42x42 L_1 (1583 vs 1499 ms, profiles/r02/ab_u8_packmax.jsonl) --
// the halved VIMNMX3 count does not pay for the packing IMADs and the longer dependency chain
#ifndef LN_U8_PACKMAX
#define LN_U8_PACKMAX 0
#endif
constexpr int kU8PackMaxNW = LN_U8_PACKMAX ? 16 : 0;
// packed lane-pair join (U8Step PK with LPU = 2, L_1 wide rows with sum |M| <= 65535): one SHFL and
// one VIMNMX.U16x2 per unit instead of two SHFL + two VIADDMNMX.  Measured 1 % slower on 36x144
// (81.7 vs 80.9 ms) and 2 % on 40x160 (1439 vs 1411 ms; profiles/r02/ab_u8_pkl.log): off
#ifndef LN_U8_PKL
#define LN_U8_PKL 0
#endif

// merged-last-word instances (MRG): 33-48 columns (the m = n sweep and the 42x42 headline)
template <int MODE, int NW, int LPU>
__host__ __device__ constexpr bool u8_has_mrg() {
  return LN_U8_MERGE && LPU == 1 && MODE != MODE_LD && NW >= 9 && NW <= 12 && u8_units_per_lane<MODE, NW, LPU>() % 2 == 0 &&
         u8_pr<MODE>() >= 1;
}
inline bool u8_mrg_cols(int c) { return (c & 3) == 1 || (c & 3) == 2; }

template <int MODE, int NW, int LPU>
cudaError_t launch_u8_l(const WalkParams& p, const uint32_t* tab, const int32_t* init, int grid, cudaStream_t st) {
  constexpr int P = u8_units_per_lane<MODE, NW, LPU>();
  const size_t sm = u8_smem<MODE, NW, LPU>(p.s);
  if constexpr (u8_has_mrg<MODE, NW, LPU>()) {
    if (p.batch == 1 && u8_mrg_cols(p.c)) {
      cudaError_t e = ensure_dyn_smem((const void*)walk_u8_kernel<MODE, NW, P, LPU, false, false, true>, sm);
      if (e != cudaSuccess) return e;
      walk_u8_kernel<MODE, NW, P, LPU, false, false, true><<<grid, kBlockU8, sm, st>>>(p, tab, init);
      return cudaGetLastError();
    }
  }
  if (p.batch > 1) {
    if constexpr (NW <= kU8BatchMaxNW && LPU == 1) {
      cudaError_t e = ensure_dyn_smem((const void*)walk_u8_kernel<MODE, NW, P, LPU, true>, sm);
      if (e != cudaSuccess) return e;
      walk_u8_kernel<MODE, NW, P, LPU, true><<<grid, kBlockU8, sm, st>>>(p, tab, init);
      return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
  }
  if constexpr (MODE == MODE_L1 && LPU == 2 && LN_U8_PKL) {
    if (p.u8_pack_max) {                 // every value <= sum |M| <= 65535 (host): packed lane-pair join
      cudaError_t e = ensure_dyn_smem((const void*)walk_u8_kernel<MODE, NW, P, LPU, false, true>, sm);
      if (e != cudaSuccess) return e;
      walk_u8_kernel<MODE, NW, P, LPU, false, true><<<grid, kBlockU8, sm, st>>>(p, tab, init);
      return cudaGetLastError();
    }
  }
  if constexpr (MODE != MODE_MARG && LPU == 1 && P % 2 == 0 && NW <= kU8PackMaxNW && u8_pr<MODE>() == 1) {
    if (p.u8_pack_max) {                 // every value <= sum |M| <= 65535 (host): packed maxima
      cudaError_t e = ensure_dyn_smem((const void*)walk_u8_kernel<MODE, NW, P, LPU, false, true>, sm);
      if (e != cudaSuccess) return e;
      walk_u8_kernel<MODE, NW, P, LPU, false, true><<<grid, kBlockU8, sm, st>>>(p, tab, init);
      return cudaGetLastError();
    }
  }
  cudaError_t e = ensure_dyn_smem((const void*)walk_u8_kernel<MODE, NW, P, LPU>, sm);
  if (e != cudaSuccess) return e;
  walk_u8_kernel<MODE, NW, P, LPU><<<grid, kBlockU8, sm, st>>>(p, tab, init);
  return cudaGetLastError();
}

template <int MODE, int NW>
cudaError_t launch_u8(const WalkParams& p, const uint32_t* tab, const int32_t* init, int grid, cudaStream_t st) {
  if constexpr (u8_lpu_max<MODE, NW>() == 2) {
    if (p.u8_lpu == 2) return launch_u8_l<MODE, NW, 2>(p, tab, init, grid, st);
  }
  return launch_u8_l<MODE, NW, 1>(p, tab, init, grid, st);
}

template <int MODE, int NW, int LPU>
int occ_u8_l(int s) {
  constexpr int P = u8_units_per_lane<MODE, NW, LPU>();
  const size_t sm = u8_smem<MODE, NW, LPU>(s);
  const int nb = occupancy_cached((const void*)walk_u8_kernel<MODE, NW, P, LPU>, kBlockU8, sm);
  return nb;
}

template <int MODE, int NW>
int occ_u8(int s, int lpu) {
  if constexpr (u8_lpu_max<MODE, NW>() == 2) {
    if (lpu == 2) return occ_u8_l<MODE, NW, 2>(s);
  }
  return occ_u8_l<MODE, NW, 1>(s);
}

template <int MODE, int NW>
int upl_u8(int lpu) {
  if constexpr (u8_lpu_max<MODE, NW>() == 2) {
    if (lpu == 2) return u8_units_per_lane<MODE, NW, 2>();
  }
  return u8_units_per_lane<MODE, NW, 1>();
}

template <int MODE, int NW>
int lpu_u8() { return u8_lpu_max<MODE, NW>(); }

template <int MODE, int NW>
int mrg_u8(int lpu) { return lpu == 1 && u8_has_mrg<MODE, NW, 1>() ? 1 : 0; }

template <int MODE, int NW>
int unroll_u8(int lpu) {
  if constexpr (u8_lpu_max<MODE, NW>() == 2) {
    if (lpu == 2) return u8_unroll<MODE, NW / 2, u8_units_per_lane<MODE, NW, 2>()>();
  }
  return u8_unroll<MODE, NW, u8_units_per_lane<MODE, NW, 1>()>();
}

// Wide rows (more than 128 columns, lane pairs): L_1 / L_marg instances for every EVEN word
// count, so a 144-column row is 36 words, not 40 (round 1 rounded to multiples of 8: up to
// 15 % padding VABSDIFF4 on the m = 4n sweep); L_2 (two bias sets, one lane per unit) keeps
// multiples of 8.
#if LN_BIN_MODE != 2 && LN_U8_WIDE_EVEN
#define LN_U8_WIDE_CASES(MODE, FN, ...)                                                              \
    case 34: return FN<MODE, 34>(__VA_ARGS__); case 36: return FN<MODE, 36>(__VA_ARGS__);            \
    case 38: return FN<MODE, 38>(__VA_ARGS__); case 42: return FN<MODE, 42>(__VA_ARGS__);            \
    case 44: return FN<MODE, 44>(__VA_ARGS__); case 46: return FN<MODE, 46>(__VA_ARGS__);
#else
#define LN_U8_WIDE_CASES(MODE, FN, ...)
#endif

#ifdef LN_U8_ONLY_NW   // experiment builds (tools/build_variant.py): one instance only
#define LN_U8_SWITCH(MODE, NW_, FN, ...)                                                             \
  if ((NW_) == LN_U8_ONLY_NW) return FN<MODE, LN_U8_ONLY_NW>(__VA_ARGS__);
#else
#define LN_U8_SWITCH(MODE, NW_, FN, ...)                                                             \
  switch (NW_) {                                                                                     \
    case 1: return FN<MODE, 1>(__VA_ARGS__);   case 2: return FN<MODE, 2>(__VA_ARGS__);              \
    case 3: return FN<MODE, 3>(__VA_ARGS__);   case 4: return FN<MODE, 4>(__VA_ARGS__);              \
    case 5: return FN<MODE, 5>(__VA_ARGS__);   case 6: return FN<MODE, 6>(__VA_ARGS__);              \
    case 7: return FN<MODE, 7>(__VA_ARGS__);   case 8: return FN<MODE, 8>(__VA_ARGS__);              \
    case 9: return FN<MODE, 9>(__VA_ARGS__);   case 10: return FN<MODE, 10>(__VA_ARGS__);            \
    case 11: return FN<MODE, 11>(__VA_ARGS__); case 12: return FN<MODE, 12>(__VA_ARGS__);            \
    case 13: return FN<MODE, 13>(__VA_ARGS__); case 14: return FN<MODE, 14>(__VA_ARGS__);            \
    case 15: return FN<MODE, 15>(__VA_ARGS__); case 16: return FN<MODE, 16>(__VA_ARGS__);            \
    case 20: return FN<MODE, 20>(__VA_ARGS__); case 24: return FN<MODE, 24>(__VA_ARGS__);            \
    case 28: return FN<MODE, 28>(__VA_ARGS__); case 32: return FN<MODE, 32>(__VA_ARGS__);            \
    case 40: return FN<MODE, 40>(__VA_ARGS__); case 48: return FN<MODE, 48>(__VA_ARGS__);            \
    LN_U8_WIDE_CASES(MODE, FN, __VA_ARGS__)                                                          \
    default: break;                                                                                  \
  }
#endif

}  // namespace

// packed words for c columns (0 = unsupported)
template <>
int walk_u8_words_mode<LN_BIN_MODE>(int c) {
  int nw = (c + 3) / 4;
#ifdef LN_U8_ONLY_NW
  if (nw != LN_U8_ONLY_NW) return 0;
#endif
  if (nw < 1) return 0;
  if (nw > 32) nw = (LN_BIN_MODE != 2 && LN_U8_WIDE_EVEN) ? (nw + 1) & ~1 : (nw + 7) & ~7;
  else if (nw > 16) nw = (nw + 3) & ~3;
  return nw <= 48 ? nw : 0;
}

template <>
cudaError_t walk_u8_launch_mode<LN_BIN_MODE>(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init,
                                             int grid, cudaStream_t st) {
  const int NW = walk_u8_words_mode<LN_BIN_MODE>(p.c);
  if (NW == 0) return cudaErrorInvalidValue;
  uint32_t* tab = reinterpret_cast<uint32_t*>(scratch_tab);
  const int lmax = [&]() -> int { LN_U8_SWITCH(LN_BIN_MODE, NW, lpu_u8) return 1; }();
  const int lpu = (p.u8_lpu == 2 && lmax == 2) ? 2 : 1;
  const int P = [&]() -> int { LN_U8_SWITCH(LN_BIN_MODE, NW, upl_u8, lpu) return 1; }();
  const int mrg = [&]() -> int { LN_U8_SWITCH(LN_BIN_MODE, NW, mrg_u8, lpu) return 0; }() && p.batch == 1 && u8_mrg_cols(p.c);
  build_u8_kernel<LN_BIN_MODE><<<p.batch, 256, 0, st>>>(p.M, p.r, p.c, NW, p.k, p.s, P >= 8 ? 3 : P >= 4 ? 2 : (P == 2 ? 1 : 0),
                                                        lpu, tab, scratch_init, p.m_stride, p.tab_stride, p.init_stride,
                                                        p.chunk_ctr, mrg);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  LN_U8_SWITCH(LN_BIN_MODE, NW, launch_u8, p, tab, scratch_init, grid, st)
  return cudaErrorInvalidValue;
}

// per-matrix scratch of a launch (batched launches: the strides): delta records, init records
template <>
void walk_u8_table_sizes_mode<LN_BIN_MODE>(int c, int k, int s, int lpu, int64_t* tab_words, int64_t* init_ints) {
  const int NW = walk_u8_words_mode<LN_BIN_MODE>(c), PR = u8_pr<LN_BIN_MODE>();
  *tab_words = (int64_t)2 * (s - PR) * lpu * u8_pad4(NW / lpu);
  *init_ints = (int64_t)(k + 4 + PR) * 4 * NW;
}

template <>
int walk_u8_occupancy_mode<LN_BIN_MODE>(int c, int s, int lpu) {
  LN_U8_SWITCH(LN_BIN_MODE, walk_u8_words_mode<LN_BIN_MODE>(c), occ_u8, s, lpu)
  return 0;
}

template <>
int walk_u8_units_per_lane_mode<LN_BIN_MODE>(int c, int lpu) {
  LN_U8_SWITCH(LN_BIN_MODE, walk_u8_words_mode<LN_BIN_MODE>(c), upl_u8, lpu)
  return 1;
}

template <>
int walk_u8_paired_rows_mode<LN_BIN_MODE>() { return u8_pr<LN_BIN_MODE>(); }

template <>
int walk_u8_lanes_per_unit_mode<LN_BIN_MODE>(int c) {
  LN_U8_SWITCH(LN_BIN_MODE, walk_u8_words_mode<LN_BIN_MODE>(c), lpu_u8)
  return 1;
}

template <>
int walk_u8_unroll_mode<LN_BIN_MODE>(int c, int lpu) {
  LN_U8_SWITCH(LN_BIN_MODE, walk_u8_words_mode<LN_BIN_MODE>(c), unroll_u8, lpu)
  return 4;
}

}  // namespace lnorm
