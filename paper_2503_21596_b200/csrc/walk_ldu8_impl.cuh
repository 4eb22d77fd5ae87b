// Hot d-ary Gray walk for L_d, d in {3, 4}, column sums packed four per register
// as offset bytes, the LAST TWO rows evaluated for all d^2 labellings at every walked
// word (LN_LDU8_ROWS = 2; 1 = last row only, used when the suffix is too short).
//
// Units and control as in walk_ldpair16.cu (restricted-growth prefixes, warp-uniform
// d-ary reflected walk, Eqs. 13-17; walked rows k+1..r-1-PR, rows r-PR..r-1
// paired).
// Group g's column sum m_g,y = sum_{x labelled g} M_xy is a subset sum of column y,
// so it always lies in [N_y, N_y + W_y] with N_y = sum_x min(M_xy, 0) and
// W_y = sum_x |M_xy|.  When every W_y <= 255 (the exactness guard, checked on the
// host) the lane keeps a_g,y = m_g,y - N_y as one unsigned byte, four columns per
// register, and one 32-bit add of the packed row moves a row between groups exactly
// (Eqs. 18-19: m_p -= M_rho, m_q += M_rho; no byte leaves [0, 255]).  The window is
// the same for every unit, so the biases are global constants:
//     |m_g,y|          = |a_g,y - B_y|,            B_y  = -N_y            (in [0, 255])
//     |m_g,y + rho_y|  = |a_g,y - B'_y| + kappa'_y, B'_y = clamp(c_y, 0, 255),
//                                                   c_y = -N_y - rho_y, kappa'_y = |c_y - B'_y|
// and VABSDIFF4.U8.ACC accumulates four |.| per instruction.  With H_g = sum_y |m_g,y|
// and H'_g = sum_y |m_g,y + rho_y| the value of the strategy that puts row r-1 in
// group a is (Eq. 6)  L*(a) = sum_g H_g + (H'_a - H_a),  so a walked word evaluates
// all d labels of the last row; with two paired rows (below) all d^2 labellings.
#include "common.cuh"

// Included by walk_ldu8.cu (dispatch + table builder, LN_LDU8_PART undefined) and by the
// walk_ldu8_d{3,4}{a,b}.cu translation units, each instantiating the kernels of one label
// count and half of the column range (LN_LDU8_D, LN_LDU8_PART) so they compile in parallel.

namespace lnorm {

namespace {

constexpr int kBlockLU = 32;
constexpr int kTabWordsLU = 16384;
#ifndef LN_LDU8_MINB
#define LN_LDU8_MINB 12
#endif
#ifndef LN_LDU8_MINB3
#define LN_LDU8_MINB3 14                 // d = 3, three paired rows, <= 28 columns: measured +2-3 %
#endif

__host__ __device__ constexpr int lu_pad4(int x) { return (x + 3) & ~3; }

#ifndef LN_LDU8_EPI
#define LN_LDU8_EPI 2
#endif
// a + b as IMAD (FMA-heavy pipe) with `one` a uniform operand ptxas cannot fold: keeps the
// epilogue's adds off the ALU pipe, which the VABSDIFF4s saturate
__device__ __forceinline__ int32_t lu_fadd(int32_t a, int32_t b, uint32_t one) {
  int32_t r;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
  return r;
}

__device__ __forceinline__ uint32_t lu_sad4(uint32_t a, uint32_t b, uint32_t acc) {
  uint32_t d;
  asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(acc));
  return d;
}

// PR = number of paired last rows (1: row r-1; 2: rows r-1 and r-2).  Bias set m
// (bitmask over the paired rows) serves |m_g,y + sum_{i in m} rho_i,y|; with
// E_m,g = H_m,g - H_g the value for paired-row labels (a_1 for row r-1, a_2 for r-2) is
//   PR = 1:  S + E_1,a1;     PR = 2:  S + E_1,a1 + E_2,a2 (a1 != a2),  S + E_3,a1 (a1 == a2)
// with S = sum_g H_g.  PR = 2 evaluates d^2 strategies per walked word from 8 sums of the
// two groups a move changes: 2 IADD + 8 VABSDIFF4 per four columns for d^2 strategies.
template <int D, int NW, int P, int PR>
struct LdU8 {
  static constexpr int RW = lu_pad4(NW);
  static constexpr int RD = 2 * RW;        // delta record: +row at [0, NW), -row at [RW, RW + NW)
  static constexpr int NS = 1 << PR;       // bias sets
  struct Unit {
    uint32_t A[D][NW];
    int32_t H[D], E[NS - 1][D];
    int32_t S, best;
  };
  static __device__ __forceinline__ int32_t max_of(const int32_t (&v)[D]) {
    if constexpr (D == 3) return __vimax3_s32(v[0], v[1], v[2]);
    else return max(__vimax3_s32(v[0], v[1], v[2]), v[3]);
  }
  // best paired-row extension of the current word, relative to S
  // max over a != b of X[a] + Y[b]
  static __device__ __forceinline__ int32_t pairmax(const int32_t (&X)[D], const int32_t (&Y)[D]) {
    int32_t m[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      int32_t o;
      if constexpr (D == 3) o = max(Y[(a + 1) % 3], Y[(a + 2) % 3]);
      else o = __vimax3_s32(Y[(a + 1) % 4], Y[(a + 2) % 4], Y[(a + 3) % 4]);
      m[a] = X[a] + o;
    }
    return max_of(m);
  }
  // max over pairwise distinct a, b, c of X[a] + Y[b] + Z[c]
  static __device__ __forceinline__ int32_t triplemax(const int32_t (&X)[D], const int32_t (&Y)[D], const int32_t (&Z)[D]) {
    int32_t m[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      int32_t o;
      if constexpr (D == 3) {
        const int b = (a + 1) % 3, c = (a + 2) % 3;
        o = max(Y[b] + Z[c], Y[c] + Z[b]);
      } else {
        const int b = (a + 1) % 4, c = (a + 2) % 4, e = (a + 3) % 4;
        o = __vimax3_s32(Y[b] + max(Z[c], Z[e]), Y[c] + max(Z[b], Z[e]), Y[e] + max(Z[b], Z[c]));
      }
      m[a] = X[a] + o;
    }
    return max_of(m);
  }
  // best paired-row extension of the current word, relative to S.  E[m - 1] serves the
  // subset m of paired rows (bit 0 = row r-1, bit 1 = row r-2, bit 2 = row r-3); the
  // labellings of the paired rows are the set partitions of them into distinct groups.
  // max of n candidate values with 3-input maxes (VIMNMX3): (n - 1) / 2 ALU instructions
  template <int N>
  static __device__ __forceinline__ int32_t max_tree(const int32_t (&v)[N]) {
    if constexpr (N == 1) {
      return v[0];
    } else if constexpr (N == 2) {
      return max(v[0], v[1]);
    } else {
      constexpr int M = (N + 2) / 3;
      int32_t w[M];
#pragma unroll
      for (int i = 0; i < M; ++i) {
        if (3 * i + 2 < N) w[i] = __vimax3_s32(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
        else if (3 * i + 1 < N) w[i] = max(v[3 * i], v[3 * i + 1]);
        else w[i] = v[3 * i];
      }
      return max_tree<M>(w);
    }
  }
  // d = 3: every labelling of the paired rows as an explicit candidate (sums on the FMA
  // pipe), then one max tree on the ALU pipe
  static __device__ __forceinline__ int32_t ext_flat(const Unit& U, uint32_t one) {
    if constexpr (PR == 2) {
      int32_t v[9];
      int n = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          if (a != b) v[n++] = lu_fadd(U.E[0][a], U.E[1][b], one);
#pragma unroll
      for (int a = 0; a < 3; ++a) v[n++] = U.E[2][a];
      return max_tree<9>(v);
    } else {
      int32_t v[27];
      int n = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)                                    // {1}{2}{3}
#pragma unroll
        for (int b = 0; b < 3; ++b)
          if (a != b) v[n++] = lu_fadd(lu_fadd(U.E[0][a], U.E[1][b], one), U.E[3][3 - a - b], one);
#pragma unroll
      for (int a = 0; a < 3; ++a)                                    // {12}{3}, {13}{2}, {23}{1}
#pragma unroll
        for (int b = 0; b < 3; ++b)
          if (a != b) {
            v[n++] = lu_fadd(U.E[2][a], U.E[3][b], one);
            v[n++] = lu_fadd(U.E[4][a], U.E[1][b], one);
            v[n++] = lu_fadd(U.E[5][a], U.E[0][b], one);
          }
#pragma unroll
      for (int a = 0; a < 3; ++a) v[n++] = U.E[6][a];                // {123}
      return max_tree<27>(v);
    }
  }
  static __device__ __forceinline__ int32_t ext(const Unit& U, uint32_t one) {
    if constexpr (D == 3 && PR >= 2 && LN_LDU8_EPI == 2) {
      return ext_flat(U, one);
    } else if constexpr (PR == 1) {
      return max_of(U.E[0]);
    } else if constexpr (PR == 2) {
      return max(pairmax(U.E[0], U.E[1]), max_of(U.E[2]));
    } else {
      const int32_t t1 = triplemax(U.E[0], U.E[1], U.E[3]);          // {1}{2}{3}
      const int32_t t2 = __vimax3_s32(pairmax(U.E[2], U.E[3]),       // {12}{3}
                                      pairmax(U.E[4], U.E[1]),       // {13}{2}
                                      pairmax(U.E[5], U.E[0]));      // {23}{1}
      return __vimax3_s32(t1, t2, max_of(U.E[6]));                  // {123}
    }
  }
  static __device__ __forceinline__ void refresh(Unit& U, int g, const uint32_t (&h)[NS], uint32_t one) {
    if (LN_LDU8_EPI == 2 && D == 3) {
      U.S = lu_fadd(U.S, lu_fadd((int32_t)h[0], -U.H[g], one), one);
      U.H[g] = (int32_t)h[0];
#pragma unroll
      for (int m = 1; m < NS; ++m) U.E[m - 1][g] = lu_fadd((int32_t)h[m], -(int32_t)h[0], one);
    } else {
      U.S += (int32_t)h[0] - U.H[g];
      U.H[g] = (int32_t)h[0];
#pragma unroll
      for (int m = 1; m < NS; ++m) U.E[m - 1][g] = (int32_t)h[m] - (int32_t)h[0];
    }
  }
  // move the walked row of record `off` from group PG to group QG in every unit
  template <int PG, int QG>
  static __device__ __forceinline__ void move(Unit (&U)[P], const uint32_t (&Bs)[NS * NW], const uint32_t (&Ks)[NS],
                                              uint32_t sbase, int off, uint32_t one) {
    uint32_t hp[P][NS], hq[P][NS];
#pragma unroll
    for (int v = 0; v < RW / 4; ++v) {
      const uint4 pq = lds128(sbase + 4u * (uint32_t)(off + 4 * v));        // +row quad
      const uint4 nq = lds128(sbase + 4u * (uint32_t)(off + RW + 4 * v));   // -row quad
      const uint32_t pp[4] = {pq.x, pq.y, pq.z, pq.w}, nn[4] = {nq.x, nq.y, nq.z, nq.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 4 * v + e;
        if (i < NW) {
#pragma unroll
          for (int j = 0; j < P; ++j) {
            U[j].A[PG][i] += nn[e];
            U[j].A[QG][i] += pp[e];
#pragma unroll
            for (int m = 0; m < NS; ++m) {
              hp[j][m] = lu_sad4(U[j].A[PG][i], Bs[m * NW + i], i == 0 ? Ks[m] : hp[j][m]);
              hq[j][m] = lu_sad4(U[j].A[QG][i], Bs[m * NW + i], i == 0 ? Ks[m] : hq[j][m]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      refresh(U[j], PG, hp[j], one);
      refresh(U[j], QG, hq[j], one);
      U[j].best = __viaddmax_s32(U[j].S, ext(U[j], one), U[j].best);
    }
  }
  static __device__ __forceinline__ void move_dyn(Unit (&U)[P], const uint32_t (&Bs)[NS * NW], const uint32_t (&Ks)[NS],
                                                  uint32_t sbase, int off, int p, int q, uint32_t one) {
    switch (p * D + q) {
      case 0 * D + 1: move<0, 1>(U, Bs, Ks, sbase, off, one); return;
      case 1 * D + 0: move<1, 0>(U, Bs, Ks, sbase, off, one); return;
      case 1 * D + 2: move<1, 2>(U, Bs, Ks, sbase, off, one); return;
      case 2 * D + 1: move<2, 1>(U, Bs, Ks, sbase, off, one); return;
      default: break;
    }
    if constexpr (D >= 4) {
      switch (p * D + q) {
        case 2 * D + 3: move<2, 3>(U, Bs, Ks, sbase, off, one); return;
        case 3 * D + 2: move<3, 2>(U, Bs, Ks, sbase, off, one); return;
        default: break;
      }
    }
  }
};

#ifndef LN_LDU8_ROWS
#define LN_LDU8_ROWS 3
#endif

// Init records (global int32, stride CW = 4 NW): prefix rows 0..k, the base (walked
// rows at label 0), -N_y, then the packed bias words of the NS sets and their K_m.
template <int D, int NW, int P, int PR, bool BAT = false>
__global__ void __launch_bounds__(kBlockLU, ((PR == 3 && D == 3 && D * NW * P * PR <= 63) ? LN_LDU8_MINB3 : (D * NW * P * (PR >= 2 ? PR : 1) <= 72 ? LN_LDU8_MINB : 1)))
walk_ldu8_kernel(const WalkParams p, const uint32_t* __restrict__ gTab, const int32_t* __restrict__ gInit) {
  using WK = LdU8<D, NW, P, PR>;
  constexpr int RD = WK::RD, CW = 4 * NW, NS = WK::NS;
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int sw = p.s - PR;                         // walked digits
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sT);
  uint32_t Bs[NS * NW], Ks[NS];
  uint32_t nblk = 1;
  for (int i = 1; i < sw; ++i) nblk *= D;
  int32_t best = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  // matrix mb's delta table -> shared memory, its bias words and kappas -> registers
  auto stage = [&](int mb) {
    __syncwarp();
    const uint32_t* src = gTab + mb * p.tab_stride;
    for (int i = lane; i < sw * RD; i += 32) sT[i] = src[i];
    __syncwarp();
    const uint32_t* biasRec = reinterpret_cast<const uint32_t*>(gInit + mb * p.init_stride + (p.k + 3) * CW);
#pragma unroll
    for (int i = 0; i < NS * NW; ++i) Bs[i] = __ldg(biasRec + i);
#pragma unroll
    for (int m = 0; m < NS; ++m) Ks[m] = __ldg(biasRec + NS * NW + m);
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
          unsigned long long key = have ? make_key(best, best_u) : 0ull;
          key = warp_max_u64(key);
          if (lane == 0 && key) atomicMax(p.key + cur_b, key);
          best = INT32_MIN; have = false;
        }
        stage(mb);
        cur_b = mb;
      }
    }
    const int32_t* baseRec = gI + (p.k + 1) * CW;
    const int32_t* negRec = baseRec + CW;
    typename WK::Unit U[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      const int64_t u = p.unit_begin + (rel < p.units_per ? rel : 0);
      // prefix labels, pbits per row (the RGS table word; arithmetic prefixes repacked)
      uint64_t lab = 0;
      if (p.prefix_table) lab = p.prefix_table[u - p.unit_begin];
      else for (int x = 0; x <= p.k; ++x) lab |= (uint64_t)prefix_digit(p, u, x) << (p.pbits * x);
      const uint64_t lmask = (1ull << p.pbits) - 1ull;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        int32_t a[D][4];
#pragma unroll
        for (int g = 0; g < D; ++g)
#pragma unroll
          for (int e = 0; e < 4; ++e) a[g][e] = __ldg(negRec + 4 * q + e) + (g == 0 ? __ldg(baseRec + 4 * q + e) : 0);
        for (int x = 0; x <= p.k; ++x) {
          const int dig = (int)((lab >> (p.pbits * x)) & lmask);
          const int4 v = __ldg(reinterpret_cast<const int4*>(gI + x * CW) + q);
#pragma unroll
          for (int g = 0; g < D; ++g) {
            const int32_t f = dig == g ? 1 : 0;
            a[g][0] += f * v.x; a[g][1] += f * v.y; a[g][2] += f * v.z; a[g][3] += f * v.w;
          }
        }
#pragma unroll
        for (int g = 0; g < D; ++g)
          U[j].A[g][q] = (uint32_t)(a[g][0] & 0xFF) | ((uint32_t)(a[g][1] & 0xFF) << 8) |
                         ((uint32_t)(a[g][2] & 0xFF) << 16) | ((uint32_t)(a[g][3] & 0xFF) << 24);
      }
      U[j].S = 0;
#pragma unroll
      for (int g = 0; g < D; ++g) {
        uint32_t h[NS];
#pragma unroll
        for (int m = 0; m < NS; ++m) {
          h[m] = Ks[m];
#pragma unroll
          for (int q = 0; q < NW; ++q) h[m] = lu_sad4(U[j].A[g][q], Bs[m * NW + q], h[m]);
        }
        U[j].H[g] = (int32_t)h[0];
        U[j].S += (int32_t)h[0];
#pragma unroll
        for (int m = 1; m < NS; ++m) U[j].E[m - 1][g] = (int32_t)h[m] - (int32_t)h[0];
      }
      U[j].best = U[j].S + WK::ext(U[j], p.one);
    }
    for (uint32_t t = 0; t < nblk; ++t) {
      if (t != 0) {
        uint32_t i, from, to;
        dary_block_start<D>(t, &i, &from, &to);
        WK::move_dyn(U, Bs, Ks, sbase, (int)i * RD, (int)from, (int)to, p.one);
      }
      if ((t & 1u) == 0) {
        WK::template move<0, 1>(U, Bs, Ks, sbase, 0, p.one);
        WK::template move<1, 2>(U, Bs, Ks, sbase, 0, p.one);
        if constexpr (D >= 4) WK::template move<2, 3>(U, Bs, Ks, sbase, 0, p.one);
      } else {
        if constexpr (D >= 4) WK::template move<3, 2>(U, Bs, Ks, sbase, 0, p.one);
        WK::template move<2, 1>(U, Bs, Ks, sbase, 0, p.one);
        WK::template move<1, 0>(U, Bs, Ks, sbase, 0, p.one);
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = lc * 32 * P + j * 32 + lane;
      if (rel < p.units_per) {
        const int32_t ub = U[j].best;
        if (p.unit_max) p.unit_max[rel] = ub;
        if (!have || ub > best) { best = ub; best_u = (uint32_t)(p.unit_begin + rel); have = true; }
      }
    }
  }
  unsigned long long key = have ? make_key(best, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key) atomicMax(p.key + (BAT && cur_b > 0 ? cur_b : 0), key);
}

__global__ void build_ldu8_kernel(const int32_t* M, int r, int c, int NW, int k, int s, int pr, uint32_t* tab,
                                  int32_t* init, int64_t m_stride, int64_t tab_stride, int64_t init_stride,
                                  unsigned long long* chunk_ctr) {
  if (chunk_ctr && blockIdx.x == 0 && threadIdx.x == 0) *chunk_ctr = 0ull;   // the next walk's chunk schedule
  M += blockIdx.x * m_stride;              // one block per matrix of a batch
  tab += blockIdx.x * tab_stride;
  init += blockIdx.x * init_stride;
  const int RW = lu_pad4(NW), RD = 2 * RW, CW = 4 * NW, sw = s - pr, NS = 1 << pr;
  auto pack = [](const int32_t* v) {
    uint32_t w = 0;
    for (int e = 0; e < 4; ++e) w += (uint32_t)v[e] << (8 * e);   // sum_e 256^e v_e (mod 2^32)
    return w;
  };
  for (int rec = threadIdx.x; rec < sw; rec += blockDim.x) {      // walked digit rec <-> row r-1-pr-rec
    const int32_t* row = M + (int64_t)(r - 1 - pr - rec) * c;
    for (int i = 0; i < RW; ++i) {
      int32_t vp[4], vn[4];
      for (int e = 0; e < 4; ++e) {
        const int y = 4 * i + e;
        vp[e] = (i < NW && y < c) ? row[y] : 0;
        vn[e] = -vp[e];
      }
      tab[rec * RD + i] = pack(vp);
      tab[rec * RD + RW + i] = pack(vn);
    }
  }
  for (int i = threadIdx.x; i < (k + 1) * CW; i += blockDim.x) {
    const int x = i / CW, y = i % CW;
    init[i] = y < c ? M[(int64_t)x * c + y] : 0;
  }
  for (int y = threadIdx.x; y < CW; y += blockDim.x) {
    int32_t b = 0, N = 0;
    if (y < c)
      for (int x = 0; x < r; ++x) {
        const int32_t v = M[(int64_t)x * c + y];
        N += min(v, 0);
        if (x > k && x < r - pr) b += v;
      }
    init[(k + 1) * CW + y] = b;
    init[(k + 2) * CW + y] = -N;
  }
  if (threadIdx.x < NS) {
    const int m = threadIdx.x;                   // bias set: paired rows in bitmask m
    uint32_t* bias = reinterpret_cast<uint32_t*>(init + (k + 3) * CW);
    int32_t kap = 0;
    for (int i = 0; i < NW; ++i) {
      uint32_t w = 0;
      for (int e = 0; e < 4; ++e) {
        const int y = 4 * i + e;
        int32_t cb = 0;
        if (y < c) {
          int32_t N = 0, add = 0;
          for (int x = 0; x < r; ++x) N += min(M[(int64_t)x * c + y], 0);
          for (int b = 0; b < pr; ++b)
            if ((m >> b) & 1) add += M[(int64_t)(r - 1 - b) * c + y];
          cb = -N - add;
        }
        const int32_t bb = min(max(cb, 0), 255);
        kap += abs(cb - bb);
        w |= (uint32_t)bb << (8 * e);
      }
      bias[m * NW + i] = w;
    }
    bias[NS * NW + m] = (uint32_t)kap;
  }
  // packed prefix rows (signed deltas, sum_e 256^e M_xy mod 2^32) and the packed start bytes of
  // group 0 (base - N) and of the other groups (-N): the all-H kernel's unit init adds whole
  // packed rows to its groups (every partial sum is a subset sum of the column, so no byte
  // leaves [0, 255]) instead of summing int32 columns
  uint32_t* pk = reinterpret_cast<uint32_t*>(init + (k + 3) * CW) + NS * NW + NS;
  for (int i = threadIdx.x; i < (k + 1) * NW; i += blockDim.x) {
    const int x = i / NW, q = i % NW;
    int32_t v[4];
    for (int e = 0; e < 4; ++e) v[e] = (4 * q + e < c) ? M[(int64_t)x * c + 4 * q + e] : 0;
    pk[i] = pack(v);
  }
  __syncthreads();                             // the base / -N records above are read back here
  for (int q = threadIdx.x; q < NW; q += blockDim.x) {
    int32_t v0[4], vg[4];
    for (int e = 0; e < 4; ++e) {
      vg[e] = init[(k + 2) * CW + 4 * q + e];                  // -N
      v0[e] = vg[e] + init[(k + 1) * CW + 4 * q + e];          // base - N
    }
    pk[(k + 1) * NW + q] = pack(v0);
    pk[(k + 2) * NW + q] = pack(vg);
  }
}

#ifndef LN_LDU8_PMAX
#define LN_LDU8_PMAX 4
#endif
// units per lane: the row quad loaded once per move is shared by P units (fewer when the
// per-unit bytes and the 2^PR bias sets would not fit the register budget)
template <int D, int NW, int PR>
constexpr int ldu8_units_per_lane() {
#ifndef LN_LDU8_P3
#define LN_LDU8_P3 12
#endif
  return PR == 3 ? (D * NW <= LN_LDU8_P3 ? 2 : 1)
       : D * NW * (PR == 2 ? 2 : 1) <= 24 ? LN_LDU8_PMAX : (D * NW <= 48 ? (LN_LDU8_PMAX < 2 ? LN_LDU8_PMAX : 2) : 1);
}

// paired rows for a unit of s suffix digits (at least one walked digit stays)
int ldu8_rows(int s) { return s >= LN_LDU8_ROWS + 1 ? LN_LDU8_ROWS : (s >= 3 ? 2 : 1); }

size_t ldu8_smem(int NW, int s) { return sizeof(uint32_t) * (size_t)((s - ldu8_rows(s)) * 2 * lu_pad4(NW)); }

template <int D, int NW, int PR>
cudaError_t launch_lu_pr(const WalkParams& p, const uint32_t* tab, const int32_t* init, int grid, cudaStream_t st) {
  constexpr int P = ldu8_units_per_lane<D, NW, PR>();
  const size_t sm = ldu8_smem(NW, p.s);
  if (p.batch > 1) {                     // batched instances: <= 24 columns (the small-matrix regime)
    if constexpr (NW <= 6) {
      cudaError_t e = ensure_dyn_smem((const void*)walk_ldu8_kernel<D, NW, P, PR, true>, sm);
      if (e != cudaSuccess) return e;
      walk_ldu8_kernel<D, NW, P, PR, true><<<grid, kBlockLU, sm, st>>>(p, tab, init);
      return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
  }
  cudaError_t e = ensure_dyn_smem((const void*)walk_ldu8_kernel<D, NW, P, PR>, sm);
  if (e != cudaSuccess) return e;
  walk_ldu8_kernel<D, NW, P, PR><<<grid, kBlockLU, sm, st>>>(p, tab, init);
  return cudaGetLastError();
}

template <int D, int NW>
cudaError_t launch_lu(const WalkParams& p, const uint32_t* tab, const int32_t* init, int grid, cudaStream_t st) {
  switch (ldu8_rows(p.s)) {
#if LN_LDU8_ROWS >= 3
    case 3: return launch_lu_pr<D, NW, 3>(p, tab, init, grid, st);
#endif
    case 2: return launch_lu_pr<D, NW, 2>(p, tab, init, grid, st);
    default: return launch_lu_pr<D, NW, 1>(p, tab, init, grid, st);
  }
}

template <int D, int NW, int PR>
int occ_lu_pr(int s) {
  constexpr int P = ldu8_units_per_lane<D, NW, PR>();
  const size_t sm = ldu8_smem(NW, s);
  const int nb = occupancy_cached((const void*)walk_ldu8_kernel<D, NW, P, PR>, kBlockLU, sm);
  return nb;
}

template <int D, int NW>
int occ_lu(int s) {
  switch (ldu8_rows(s)) {
#if LN_LDU8_ROWS >= 3
    case 3: return occ_lu_pr<D, NW, 3>(s);
#endif
    case 2: return occ_lu_pr<D, NW, 2>(s);
    default: return occ_lu_pr<D, NW, 1>(s);
  }
}

template <int D, int NW>
int upl_lu(int s) {
  switch (ldu8_rows(s)) {
#if LN_LDU8_ROWS >= 3
    case 3: return ldu8_units_per_lane<D, NW, 3>();
#endif
    case 2: return ldu8_units_per_lane<D, NW, 2>();
    default: return ldu8_units_per_lane<D, NW, 1>();
  }
}

int words_of(int c) { return (c + 3) / 4; }

}  // namespace

#ifdef LN_LDU8_PART
// part 0: 1-6 words (<= 24 columns), part 1: 7-12 words
#define LN_LDU8_PSWITCH(D, NW_, FN, ...)                                                     \
  if constexpr (LN_LDU8_PART == 0) {                                                         \
    switch (NW_) {                                                                           \
      case 1: return FN<D, 1>(__VA_ARGS__); case 2: return FN<D, 2>(__VA_ARGS__);            \
      case 3: return FN<D, 3>(__VA_ARGS__); case 4: return FN<D, 4>(__VA_ARGS__);            \
      case 5: return FN<D, 5>(__VA_ARGS__); case 6: return FN<D, 6>(__VA_ARGS__);            \
      default: break;                                                                        \
    }                                                                                        \
  } else {                                                                                   \
    switch (NW_) {                                                                           \
      case 7: return FN<D, 7>(__VA_ARGS__);   case 8: return FN<D, 8>(__VA_ARGS__);          \
      case 9: return FN<D, 9>(__VA_ARGS__);   case 10: return FN<D, 10>(__VA_ARGS__);        \
      case 11: return FN<D, 11>(__VA_ARGS__); case 12: return FN<D, 12>(__VA_ARGS__);        \
      default: break;                                                                        \
    }                                                                                        \
  }

template <>
int walk_ldu8_upl_part<LN_LDU8_D, LN_LDU8_PART>(int NW, int s) {
  LN_LDU8_PSWITCH(LN_LDU8_D, NW, upl_lu, s)
  return 1;
}

template <>
int walk_ldu8_occ_part<LN_LDU8_D, LN_LDU8_PART>(int NW, int s) {
  LN_LDU8_PSWITCH(LN_LDU8_D, NW, occ_lu, s)
  return 0;
}

template <>
cudaError_t walk_ldu8_launch_part<LN_LDU8_D, LN_LDU8_PART>(const WalkParams& p, const uint32_t* tab, const int32_t* init,
                                                             int grid, cudaStream_t st, int NW) {
  LN_LDU8_PSWITCH(LN_LDU8_D, NW, launch_lu, p, tab, init, grid, st)
  return cudaErrorInvalidValue;
}
#endif

}  // namespace lnorm
