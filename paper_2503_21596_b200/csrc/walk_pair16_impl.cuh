// Hot binary Gray walk, "strategy-paired" 16-bit layout: L_1, L_marg, L_2.
//
// Same units and warp-uniform Gray control as walk_bin_impl.cuh, but the LAST
// suffix row (row r-1, the digit that flips every other step of the binary
// reflected code, Table 1) is not walked: every register holds ONE
// column for the TWO strategies that differ only in that row,
//     R_y = ( m_y(A) , m_y(B) )  as s16x2,  A: a_{r-1} = +1 (label 0), B: a_{r-1} = -1 (label 1).
// A step of the walk flips a row rho among rows k+1..r-2 and changes both halves
// by the same delta (Eq. 12), so one VIADD.16x2 updates column y of both
// strategies and one VIADDMNMX.S16x2 accumulates max(m_y, 0) for both:
//     |m| = 2 max(m, 0) - m,    value = 2 H + q,   H = sum_y max(m_y, 0)
// with the linear part q carried per strategy (L_1: q = -sum m; L_marg: q =
// m_0 - sum_{y>=1} m_y, column 0 kept out of the packed registers; L_2: m_1 =
// T - m_0 is held too and q = -sum T).  The running maximum is kept packed:
//     t = H + Q ;  best2 = max(H + t, best2)   (= max(2H + Q, best2), both halves)
// where Q is the warp-uniform sum of q-deltas since the unit start, so the
// epilogue costs two instructions per PAIR of strategies.  Per strategy
// and column this is (1 + 1/c) instructions split over the FMA-heavy and ALU pipes.
// Exactness guard: every 16-bit intermediate is bounded
// by 2S with S = sum_ij |M_ij| (2H + Q = value - q(0), |value|, |q(0)| <= S), so
// S <= 16383 is required and checked on the host.
#include "common.cuh"

#ifndef LN_BIN_MODE
#error "define LN_BIN_MODE before including walk_pair16_impl.cuh"
#endif

namespace lnorm {

namespace {

constexpr int kBlock = 32;

__host__ __device__ constexpr int cctz(int j) { return (j & 1) ? 0 : (j & 2) ? 1 : (j & 4) ? 2 : 3; }

// Unrolled low walked digits: as many as keep the unrolled block under ~800
// instructions (~13 KB): a larger body thrashes the instruction cache (ncu showed
// 'no_instruction' as the dominant stall with 16 unrolled steps at C = 42, P = 2).
#ifndef LN_PAIR_PMAX
#define LN_PAIR_PMAX 2
#endif
#ifndef LN_PAIR_MINB
#define LN_PAIR_MINB 12
#endif
#ifndef LN_PAIR_CHUNKED
#define LN_PAIR_CHUNKED 1
#endif
#ifndef LN_PAIR_VOLATILE
#define LN_PAIR_VOLATILE 0
#endif
#ifndef LN_PAIR_ACC
#define LN_PAIR_ACC 2
#endif
#ifndef LN_PAIR_BUDGET
#define LN_PAIR_BUDGET 1800
#endif
__host__ __device__ constexpr int unroll_digits(int step_instr) {
  return step_instr * 16 <= LN_PAIR_BUDGET ? 4 : step_instr * 8 <= LN_PAIR_BUDGET ? 3 : step_instr * 4 <= LN_PAIR_BUDGET ? 2 : 1;
}
__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }

template <int MODE, int C>
struct PairLayout {
  static constexpr int G = (MODE == MODE_LD) ? 2 : 1;   // packed register groups (m_0, m_1 for L_2)
  static constexpr int RW = pad4(G * C + 1);            // delta record: G*C duplicated words + q word
};

// Init data (global memory, packed s16x2 words), per record of IW = G*C + 2 words:
//   prefix rows x = 0..k : row duplicated in both halves (+ its negation for L_2's m_1), q part
//   base                 : suffix rows k+1..r-1 at digit 0 (strategy A) duplicated [+ T - base], q
//   pair                 : the change A -> B (flip of row r-1) in the HIGH half only, and its q part
template <int MODE, int C>
struct InitLayout {
  static constexpr int IW = (MODE == MODE_LD ? 2 * C : C) + 2;
};

template <int MODE, int C, int P>
struct PairStep {
  static constexpr int G = PairLayout<MODE, C>::G, RW = PairLayout<MODE, C>::RW;
  // One walked word: apply the delta record at sbase + off to both strategies of each
  // unit.  Q is the warp-uniform running sum of the q deltas since the unit start
  // (identical for every unit: the walk is lockstep), so per unit the epilogue is
  //     t = H + Q ; best2 = max(H + t, best2)  =  max(2H + Q, best2)
  // and the unit's own q at its start word is added once at the end.
  static __device__ __forceinline__ void run(uint32_t (&R)[P][G * C], uint32_t& Q, uint32_t (&best2)[P],
                                             uint32_t sbase, int off) {
#if LN_PAIR_CHUNKED
    // row consumed 4 words at a time (one LDS.128 per quad, applied to every unit
    // before the next quad is loaded): keeps only a quad of the row live
    uint32_t a0[P], a1[P];
#pragma unroll
    for (int v = 0; v < RW / 4; ++v) {
      const uint4 x4 = lds128(sbase + 4u * (uint32_t)(off + 4 * v));
      const uint32_t rq[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * v + e;
        if (i < G * C) {
#pragma unroll
          for (int j = 0; j < P; ++j) {
            R[j][i] = __vadd2(R[j][i], rq[e]);
            if (i == 0) a0[j] = __vmaxs2(R[j][0], 0u);
            else if (i == 1) a1[j] = __vmaxs2(R[j][1], 0u);
            else if (i & 1) a1[j] = __viaddmax_s16x2(a1[j], R[j][i], a1[j]);
            else a0[j] = __viaddmax_s16x2(a0[j], R[j][i], a0[j]);
          }
        } else if (i == RW - 1 && MODE != MODE_LD) {
          Q = __vadd2(Q, rq[e]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const uint32_t a = (G * C > 1) ? __vadd2(a0[j], a1[j]) : a0[j];
      best2[j] = __viaddmax_s16x2(a, __vadd2(a, Q), best2[j]);
    }
#else
    uint32_t r[RW];
#if LN_PAIR_VOLATILE
#pragma unroll
    for (int v = 0; v < RW / 4; ++v) {
      const uint4 x4 = lds128(sbase + 4u * (uint32_t)(off + 4 * v));
#else
    const uint4* src = reinterpret_cast<const uint4*>(__cvta_shared_to_generic(sbase) ) + off / 4;
#pragma unroll
    for (int v = 0; v < RW / 4; ++v) {
      const uint4 x4 = src[v];
#endif
      r[4 * v] = x4.x; r[4 * v + 1] = x4.y; r[4 * v + 2] = x4.z; r[4 * v + 3] = x4.w;
    }
    if (MODE != MODE_LD) Q = __vadd2(Q, r[RW - 1]);
#pragma unroll
    for (int j = 0; j < P; ++j) {
#if LN_PAIR_ACC == 2
      uint32_t a0, a1 = 0u;
#pragma unroll
      for (int i = 0; i < G * C; ++i) {
        R[j][i] = __vadd2(R[j][i], r[i]);
        if (i == 0) a0 = __vmaxs2(R[j][0], 0u);
        else if (i & 1) a1 = __viaddmax_s16x2(a1, R[j][i], a1);
        else a0 = __viaddmax_s16x2(a0, R[j][i], a0);
      }
      const uint32_t a = __vadd2(a0, a1);
#else
      uint32_t a = 0u;
#pragma unroll
      for (int i = 0; i < G * C; ++i) {
        R[j][i] = __vadd2(R[j][i], r[i]);
        a = (i == 0) ? __vmaxs2(R[j][0], 0u) : __viaddmax_s16x2(a, R[j][i], a);
      }
#endif
      best2[j] = __viaddmax_s16x2(a, __vadd2(a, Q), best2[j]);
    }
#endif
  }
};

template <int MODE, int C, int P>
__host__ __device__ constexpr int pair_unroll() { return unroll_digits(P * (2 * PairLayout<MODE, C>::G * C + 4) + PairLayout<MODE, C>::RW / 4); }

template <int MODE, int C, int P>
__global__ void __launch_bounds__(kBlock, (PairLayout<MODE, C>::G * C * P <= 96 ? LN_PAIR_MINB : 1)) walk_pair16_kernel(const WalkParams p, const uint32_t* __restrict__ gTab,
                                                             const int32_t* __restrict__ gInit) {
  using LY = PairLayout<MODE, C>;
  constexpr int G = LY::G, RW = LY::RW, IW = InitLayout<MODE, C>::IW;
  constexpr int K = pair_unroll<MODE, C, P>();
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int sw = p.s - 1;                          // walked digits (rows k+1 .. r-2)
  const int total = 2 * sw * RW;
  const uint32_t nblk = 1u << (sw - K);
  int32_t best = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  // Static warp-chunk schedule (block = one warp).  Chunks never straddle matrices
  // (batched launches): chunk ch -> matrix b = ch / CPM, local chunk lc = ch % CPM.
  const int64_t CPM = (p.units_per + 32 * P - 1) / (32 * P);
  const int64_t nchunks = CPM * p.batch;
  int64_t cur_b = -1;
  const int32_t* gI = gInit;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t b = ch / CPM, lc = ch - b * CPM;
    if (b != cur_b) {                              // (re)stage this matrix's delta table
      if (cur_b >= 0) {
        unsigned long long key = have ? make_key(best, best_u) : 0ull;
        key = warp_max_u64(key);
        if (lane == 0 && key) atomicMax(p.key + cur_b, key);
        best = INT32_MIN; have = false;
      }
      __syncwarp();
      const uint32_t* src = gTab + b * p.tab_stride;
      for (int i = lane; i < total; i += 32) sT[i] = src[i];
      __syncwarp();
      gI = gInit + b * p.init_stride;
      cur_b = b;
    }
    const int32_t* baseRec = gI + (p.k + 1) * IW;
    const int32_t* pairRec = baseRec + IW;
    uint32_t R[P][G * C];
    uint32_t q[P], best2[P];
    uint32_t Q = 0u;                                   // uniform: q(t) - q(0), both halves
    // ---- unit init: column sums of strategies A and B (the paper's per-thread product)
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      const int64_t u = p.unit_begin + (rel < p.units_per ? rel : 0);
      // packed init (no int32 temporaries): base, +-prefix rows, then the pair row's
      // contribution to the high (strategy B) half only
      const uint32_t* bR = reinterpret_cast<const uint32_t*>(baseRec);
      const uint32_t* pR = reinterpret_cast<const uint32_t*>(pairRec);
#pragma unroll
      for (int i = 0; i < G * C; ++i) R[j][i] = __ldg(bR + i);
      q[j] = __ldg(bR + G * C);
      for (int x = 0; x <= p.k; ++x) {
        const int dig = prefix_digit(p, u, x);
        const uint32_t* rec = reinterpret_cast<const uint32_t*>(gI + x * IW);
        if (dig == 0) {
#pragma unroll
          for (int i = 0; i < G * C; ++i) R[j][i] = __vadd2(R[j][i], __ldg(rec + i));
          q[j] = __vadd2(q[j], __ldg(rec + G * C));
        } else if (MODE != MODE_LD) {
#pragma unroll
          for (int i = 0; i < G * C; ++i) R[j][i] = __vsub2(R[j][i], __ldg(rec + i));
          q[j] = __vsub2(q[j], __ldg(rec + G * C));
        }
      }
#pragma unroll
      for (int i = 0; i < G * C; ++i) R[j][i] = __vadd2(R[j][i], __ldg(pR + i));
      q[j] = __vadd2(q[j], __ldg(pR + G * C));
      // value of the starting pair
      uint32_t a0 = __vmaxs2(R[j][0], 0u), a1 = 0u;
#pragma unroll
      for (int i = 1; i < G * C; ++i) {
        if (i & 1) a1 = __viaddmax_s16x2(a1, R[j][i], a1);
        else a0 = __viaddmax_s16x2(a0, R[j][i], a0);
      }
      const uint32_t h = __vadd2(a0, a1);
      best2[j] = __vadd2(h, h);                         // 2H + Q at the start word (Q = 0); + q[j] at the end
    }
    // ---- the walk: 2^(s-1) words, each evaluating the pair (A, B)
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sT);
    for (uint32_t t = 0; t < nblk; ++t) {
      if (t != 0) {                                    // block start: walked digit K + ctz(t)
        const int tz = __ffs((int)t) - 1;
        const int b = K + tz;
        const int sg = 1 ^ (int)((t >> (tz + 1)) & 1u);
        PairStep<MODE, C, P>::run(R, Q, best2, sbase, (2 * b + sg) * RW);
      }
#pragma unroll
      for (int jj = 1; jj < (1 << K); ++jj) {
        const int b = cctz(jj);
        const int sg = (b < K - 1) ? (1 ^ ((jj >> (b + 1)) & 1)) : (1 ^ (int)(t & 1u));
        PairStep<MODE, C, P>::run(R, Q, best2, sbase, (2 * b + sg) * RW);
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      if (rel < p.units_per) {
        // add the unit's own start-word q (per strategy) back: value = 2H + Q + q(0)
        const int32_t lo = (int32_t)(int16_t)(best2[j] & 0xFFFF) + (int32_t)(int16_t)(q[j] & 0xFFFF);
        const int32_t hi = (int32_t)(int16_t)(best2[j] >> 16) + (int32_t)(int16_t)(q[j] >> 16);
        const int32_t ub = max(lo, hi);
        if (p.unit_max) p.unit_max[rel] = ub;
        if (!have || ub > best) { best = ub; best_u = (uint32_t)(p.unit_begin + rel); have = true; }
      }
    }
  }
  unsigned long long key = have ? make_key(best, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key && cur_b >= 0) atomicMax(p.key + cur_b, key);
}

// Tables from the oriented matrix: packed duplicated delta records (walked digit b
// <-> row r-2-b, sign 1 = flip to -1 / label 1) and the int32 init records.
template <int MODE>
__global__ void build_pair16_kernel(const int32_t* M, int r, int c, int C, int k, int s,
                                    uint32_t* tab, int32_t* init, int64_t m_stride, int64_t tab_stride,
                                    int64_t init_stride) {
  M += blockIdx.x * m_stride;            // one block per matrix of a batch
  tab += blockIdx.x * tab_stride;
  init += blockIdx.x * init_stride;
  const int G = (MODE == MODE_LD) ? 2 : 1;
  const int RW = pad4(G * C + 1), IW = G * C + 2;
  const int c0 = (MODE == MODE_MARG) ? 1 : 0;
  const int scale = (MODE == MODE_LD) ? 1 : 2;
  const int sw = s - 1;
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * sw * RW; i += blockDim.x) tab[i] = 0u;
  for (int i = tid; i < (k + 3) * IW; i += blockDim.x) init[i] = 0;
  __syncthreads();
  for (int rec = tid; rec < 2 * sw; rec += blockDim.x) {
    const int b = rec >> 1, sg = rec & 1;
    const int32_t* row = M + (int64_t)(r - 2 - b) * c;
    const int f = sg ? -scale : scale;
    int32_t qd = 0;
    for (int j = 0; j < C; ++j) {
      const int y = c0 + j;
      const int32_t v = y < c ? f * row[y] : 0;
      tab[rec * RW + j] = (uint32_t)(v & 0xFFFF) * 0x10001u;
      if (MODE == MODE_LD) tab[rec * RW + C + j] = (uint32_t)((-v) & 0xFFFF) * 0x10001u;
      qd -= v;
    }
    if (MODE == MODE_MARG) qd += f * row[0];
    tab[rec * RW + RW - 1] = MODE == MODE_LD ? 0u : (uint32_t)(qd & 0xFFFF) * 0x10001u;
  }
  // init records (packed s16x2): prefix rows 0..k, base, pair
  auto dup = [](int32_t v) { return (uint32_t)(v & 0xFFFF) * 0x10001u; };
  auto hi = [](int32_t v) { return (uint32_t)(v & 0xFFFF) << 16; };
  uint32_t* initw = reinterpret_cast<uint32_t*>(init);
  for (int rec = tid; rec < k + 3; rec += blockDim.x) {
    uint32_t* out = initw + rec * IW;
    if (rec <= k) {                                // +row (m_0 part), -row (m_1 = T - m_0 part), q
      const int32_t* row = M + (int64_t)rec * c;
      int32_t qd = 0;
      for (int j = 0; j < C; ++j) {
        const int y = c0 + j;
        const int32_t v = y < c ? row[y] : 0;
        out[j] = dup(v);
        if (MODE == MODE_LD) out[C + j] = dup(-v);
        qd -= v;
      }
      if (MODE == MODE_MARG) qd += row[0];
      out[G * C] = MODE == MODE_LD ? 0u : dup(qd);
    } else if (rec == k + 1) {                     // base: suffix rows k+1..r-1 at digit 0 (strategy A)
      int32_t qd = 0, tsum = 0;
      for (int j = 0; j < C; ++j) {
        const int y = c0 + j;
        int32_t bv = 0, tv = 0;
        if (y < c)
          for (int x = 0; x < r; ++x) {
            const int32_t v = M[(int64_t)x * c + y];
            tv += v;
            if (x > k) bv += v;
          }
        out[j] = dup(bv);
        if (MODE == MODE_LD) out[C + j] = dup(tv - bv);
        qd -= bv;
        tsum += tv;
      }
      if (MODE == MODE_MARG) {
        int32_t b0 = 0;
        for (int x = k + 1; x < r; ++x) b0 += M[(int64_t)x * c];
        qd += b0;
      }
      out[G * C] = dup(MODE == MODE_LD ? -tsum : qd);
    } else {                                       // pair row r-1: strategy B = A with a_{r-1} flipped
      const int32_t* row = M + (int64_t)(r - 1) * c;
      int32_t s1 = 0;
      for (int j = 0; j < C; ++j) {
        const int y = c0 + j;
        const int32_t v = y < c ? row[y] : 0;
        out[j] = hi(MODE == MODE_LD ? -v : -2 * v);          // m_B = m_A - 2 M_{r-1} (L_2: - M_{r-1})
        if (MODE == MODE_LD) out[C + j] = hi(v);             // m_1 = T - m_0
        s1 += v;
      }
      int32_t dq = 2 * s1;                                   // L_1: q = -sum m
      if (MODE == MODE_MARG) dq -= 2 * row[0];
      out[G * C] = MODE == MODE_LD ? 0u : hi(dq);
    }
  }
}

template <int MODE, int C>
__host__ __device__ constexpr int pair_units_per_lane() { return (MODE == MODE_LD ? 2 * C : C) <= 48 ? LN_PAIR_PMAX : 1; }

template <int MODE, int C>
size_t pair_smem(int s) { return sizeof(uint32_t) * (size_t)(2 * (s - 1) * PairLayout<MODE, C>::RW); }

template <int MODE, int C>
cudaError_t launch_pair(const WalkParams& p, const uint32_t* tab, const int32_t* init, int grid, cudaStream_t st) {
  constexpr int P = pair_units_per_lane<MODE, C>();
  const size_t sm = pair_smem<MODE, C>(p.s);
  cudaError_t e = ensure_dyn_smem((const void*)walk_pair16_kernel<MODE, C, P>, sm);
  if (e != cudaSuccess) return e;
  walk_pair16_kernel<MODE, C, P><<<grid, kBlock, sm, st>>>(p, tab, init);
  return cudaGetLastError();
}

template <int MODE, int C>
int occ_pair(int s) {
  constexpr int P = pair_units_per_lane<MODE, C>();
  const size_t sm = pair_smem<MODE, C>(s);
  const int nb = occupancy_cached((const void*)walk_pair16_kernel<MODE, C, P>, kBlock, sm);
  return nb;
}

template <int MODE, int C>
int upl_pair() { return pair_units_per_lane<MODE, C>(); }

#define LN_PAIR_SWITCH(MODE, C_, FN, ...)                                                            \
  switch (C_) {                                                                                      \
    case 2: return FN<MODE, 2>(__VA_ARGS__);   case 4: return FN<MODE, 4>(__VA_ARGS__);              \
    case 6: return FN<MODE, 6>(__VA_ARGS__);   case 8: return FN<MODE, 8>(__VA_ARGS__);              \
    case 10: return FN<MODE, 10>(__VA_ARGS__); case 12: return FN<MODE, 12>(__VA_ARGS__);            \
    case 14: return FN<MODE, 14>(__VA_ARGS__); case 16: return FN<MODE, 16>(__VA_ARGS__);            \
    case 18: return FN<MODE, 18>(__VA_ARGS__); case 20: return FN<MODE, 20>(__VA_ARGS__);            \
    case 22: return FN<MODE, 22>(__VA_ARGS__); case 24: return FN<MODE, 24>(__VA_ARGS__);            \
    case 26: return FN<MODE, 26>(__VA_ARGS__); case 28: return FN<MODE, 28>(__VA_ARGS__);            \
    case 30: return FN<MODE, 30>(__VA_ARGS__); case 32: return FN<MODE, 32>(__VA_ARGS__);            \
    case 34: return FN<MODE, 34>(__VA_ARGS__); case 36: return FN<MODE, 36>(__VA_ARGS__);            \
    case 38: return FN<MODE, 38>(__VA_ARGS__); case 40: return FN<MODE, 40>(__VA_ARGS__);            \
    case 42: return FN<MODE, 42>(__VA_ARGS__); case 44: return FN<MODE, 44>(__VA_ARGS__);            \
    case 46: return FN<MODE, 46>(__VA_ARGS__); case 48: return FN<MODE, 48>(__VA_ARGS__);            \
    case 52: return FN<MODE, 52>(__VA_ARGS__); case 56: return FN<MODE, 56>(__VA_ARGS__);            \
    case 60: return FN<MODE, 60>(__VA_ARGS__); case 64: return FN<MODE, 64>(__VA_ARGS__);            \
    default: break;                                                                                  \
  }

}  // namespace

template <>
int walk_pair16_cols<LN_BIN_MODE>(int c) {
  const int cp = (LN_BIN_MODE == MODE_MARG) ? c - 1 : c;
  int C = cp < 2 ? 2 : (cp + 1) & ~1;
  if (C > 48) C = (C + 3) & ~3;
  return C <= 64 ? C : 0;
}

template <>
cudaError_t walk_pair16_launch_mode<LN_BIN_MODE>(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init,
                                                 int grid, cudaStream_t st) {
  const int C = walk_pair16_cols<LN_BIN_MODE>(p.c);
  if (C == 0) return cudaErrorInvalidValue;
  uint32_t* tab = reinterpret_cast<uint32_t*>(scratch_tab);
  build_pair16_kernel<LN_BIN_MODE><<<p.batch, 128, 0, st>>>(p.M, p.r, p.c, C, p.k, p.s, tab, scratch_init,
                                                             p.m_stride, p.tab_stride, p.init_stride);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  LN_PAIR_SWITCH(LN_BIN_MODE, C, launch_pair, p, tab, scratch_init, grid, st)
  return cudaErrorInvalidValue;
}

template <>
int walk_pair16_occupancy_mode<LN_BIN_MODE>(int c, int s) {
  LN_PAIR_SWITCH(LN_BIN_MODE, walk_pair16_cols<LN_BIN_MODE>(c), occ_pair, s)
  return 0;
}

template <int MODE, int C>
int unroll_pair() { return pair_unroll<MODE, C, pair_units_per_lane<MODE, C>()>(); }

template <int MODE, int C>
int tabw_pair() { return PairLayout<MODE, C>::RW; }

// words of the delta table / ints of the init records for one matrix
template <>
void walk_pair16_table_sizes_mode<LN_BIN_MODE>(int c, int k, int s, int64_t* tab_words, int64_t* init_ints) {
  const int C = walk_pair16_cols<LN_BIN_MODE>(c);
  const int G = (LN_BIN_MODE == MODE_LD) ? 2 : 1;
  const int RW = (G * C + 1 + 3) & ~3, IW = G * C + 2;
  *tab_words = (int64_t)2 * (s - 1) * RW;
  *init_ints = (int64_t)(k + 3) * IW;
}

template <>
int walk_pair16_unroll_mode<LN_BIN_MODE>(int c) {
  LN_PAIR_SWITCH(LN_BIN_MODE, walk_pair16_cols<LN_BIN_MODE>(c), unroll_pair)
  return 4;
}

template <>
int walk_pair16_units_per_lane_mode<LN_BIN_MODE>(int c) {
  LN_PAIR_SWITCH(LN_BIN_MODE, walk_pair16_cols<LN_BIN_MODE>(c), upl_pair)
  return 1;
}

}  // namespace lnorm
