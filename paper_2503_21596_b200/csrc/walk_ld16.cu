// Hot d-ary Gray walk for L_d, d in {3, 4}, packed 16-bit variant.
//
// Decomposition and Gray control are those of walk_ld.cu (restricted-growth
// prefixes, warp-uniform d-ary reflected suffix walk, Eqs. 13-17).  The group
// sums m_a are packed two columns per register (s16x2) and the value uses
//     ||m_a||_1 = 2 sum_y max(m_a,y, 0) - sum_y m_a,y,   sum_a sum_y m_a,y = sum_y T_y,
// so  L*_d = 2 sum_a H_a - sum_y T_y  with H_a = sum_y max(m_a,y, 0).
// A step moving row rho from group p to q (Eqs. 18-19) costs, per pair of
// columns, two VIADD.16x2 (m_p -= M_rho, m_q += M_rho) and two VIADDMNMX.S16x2
// (recompute H_p, H_q), i.e. one instruction per column update (2c updates per
// step), split over the FMA-heavy and ALU pipes.  Rows are read from shared
// memory with warp-uniform LDS.128 broadcasts.  Exactness guard: as for the
// binary packed walk (every |m_a,y| <= sum_x |M_xy|), checked on the host.
#include "common.cuh"

namespace lnorm {

namespace {

constexpr int kBlock = 32;
constexpr int kTabWords = 8448;

__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }

template <int W>
struct LdLayout {
  static constexpr int RD = pad4(2 * W);   // delta record: +row (W words) then -row (W words)
  static constexpr int RP = pad4(W);       // prefix / base record: raw row (W words)
};

template <int D, int W, int P>
struct Ld16 {
  static constexpr int RD = LdLayout<W>::RD;
  static __device__ __forceinline__ int32_t half_sum(const uint32_t (&v)[W]) {
    uint32_t a0 = __vmaxs2(v[0], 0u), a1 = 0u;
#pragma unroll
    for (int i = 1; i < W; ++i) {
      if (i & 1) a1 = __viaddmax_s16x2(a1, v[i], a1);
      else a0 = __viaddmax_s16x2(a0, v[i], a0);
    }
    return __dp2a_lo((int)__vadd2(a0, a1), 0x0101, 0);   // H = lo + hi
  }
  // move suffix row (record at sT + off) from group PG to group QG for all P units
  template <int PG, int QG>
  static __device__ __forceinline__ void move(uint32_t (&m)[P][D][W], int32_t (&H)[P][D], int32_t (&Hs)[P],
                                              int32_t (&ub)[P], const uint32_t* sT, int off, int32_t q0) {
    uint32_t r[RD];
    const uint4* src = reinterpret_cast<const uint4*>(sT + off);
#pragma unroll
    for (int v = 0; v < RD / 4; ++v) {
      const uint4 x = src[v];
      r[4 * v] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
#pragma unroll
      for (int i = 0; i < W; ++i) {
        m[j][PG][i] = __vadd2(m[j][PG][i], r[W + i]);   // -row
        m[j][QG][i] = __vadd2(m[j][QG][i], r[i]);       // +row
      }
      const int32_t hp = half_sum(m[j][PG]), hq = half_sum(m[j][QG]);
      Hs[j] += (hp - H[j][PG]) + (hq - H[j][QG]);
      H[j][PG] = hp;
      H[j][QG] = hq;
      ub[j] = max(ub[j], 2 * Hs[j] + q0);
    }
  }
  static __device__ __forceinline__ void move_dyn(uint32_t (&m)[P][D][W], int32_t (&H)[P][D], int32_t (&Hs)[P],
                                                  int32_t (&ub)[P], const uint32_t* sT, int off, int p, int q,
                                                  int32_t q0) {
    switch (p * D + q) {
      case 0 * D + 1: move<0, 1>(m, H, Hs, ub, sT, off, q0); return;
      case 1 * D + 0: move<1, 0>(m, H, Hs, ub, sT, off, q0); return;
      case 1 * D + 2: move<1, 2>(m, H, Hs, ub, sT, off, q0); return;
      case 2 * D + 1: move<2, 1>(m, H, Hs, ub, sT, off, q0); return;
      default: break;
    }
    if constexpr (D >= 4) {
      switch (p * D + q) {
        case 2 * D + 3: move<2, 3>(m, H, Hs, ub, sT, off, q0); return;
        case 3 * D + 2: move<3, 2>(m, H, Hs, ub, sT, off, q0); return;
        default: break;
      }
    }
  }
};

template <int D, int W, int P>
__global__ void __launch_bounds__(kBlock) walk_ld16_kernel(const WalkParams p, const uint32_t* __restrict__ gTab) {
  using LY = LdLayout<W>;
  using WK = Ld16<D, W, P>;
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int s = p.s, k = p.k;
  const int preOff = s * LY::RD;
  const int baseOff = preOff + (k + 1) * LY::RP;
  const int total = baseOff + LY::RP + 4;
  for (int i = threadIdx.x; i < total; i += blockDim.x) sT[i] = gTab[i];
  __syncthreads();
  const int32_t q0 = (int32_t)sT[baseOff + LY::RP];   // -sum_y T_y
  uint32_t nblk = 1;
  for (int i = 1; i < s; ++i) nblk *= D;
  int32_t best = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  const int64_t nchunks = (p.unit_count + 32 * P - 1) / (32 * P);
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    uint32_t m[P][D][W];
    int32_t H[P][D], Hs[P], ub[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = ch * 32 * P + j * 32 + lane;
      const int64_t u = p.unit_begin + (rel < p.unit_count ? rel : 0);
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int i = 0; i < W; ++i) m[j][a][i] = (a == 0) ? sT[baseOff + i] : 0u;
      for (int x = 0; x <= k; ++x) {
        const int dig = prefix_digit(p, u, x);
        const int po = preOff + x * LY::RP;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const uint32_t msk = (dig == a) ? 0xFFFFFFFFu : 0u;
#pragma unroll
          for (int i = 0; i < W; ++i) m[j][a][i] = __vadd2(m[j][a][i], sT[po + i] & msk);
        }
      }
      Hs[j] = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) { H[j][a] = WK::half_sum(m[j][a]); Hs[j] += H[j][a]; }
      ub[j] = 2 * Hs[j] + q0;
    }
    for (uint32_t t = 0; t < nblk; ++t) {
      if (t != 0) {
        uint32_t i, from, to;
        dary_block_start<D>(t, &i, &from, &to);
        WK::move_dyn(m, H, Hs, ub, sT, (int)i * LY::RD, (int)from, (int)to, q0);
      }
      if ((t & 1u) == 0) {
        WK::template move<0, 1>(m, H, Hs, ub, sT, 0, q0);
        WK::template move<1, 2>(m, H, Hs, ub, sT, 0, q0);
        if constexpr (D >= 4) WK::template move<2, 3>(m, H, Hs, ub, sT, 0, q0);
      } else {
        if constexpr (D >= 4) WK::template move<3, 2>(m, H, Hs, ub, sT, 0, q0);
        WK::template move<2, 1>(m, H, Hs, ub, sT, 0, q0);
        WK::template move<1, 0>(m, H, Hs, ub, sT, 0, q0);
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = ch * 32 * P + j * 32 + lane;
      if (rel < p.unit_count) {
        if (p.unit_max) p.unit_max[rel] = ub[j];
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

// table: s delta records [+row | -row] for suffix digit i (row r-1-i), k+1 prefix
// records (raw rows 0..k), the base record (suffix rows at label 0), then -sum T.
__global__ void build_table_ld16_kernel(const int32_t* M, int r, int c, int W, int k, int s, uint32_t* tab) {
  const int RD = pad4(2 * W), RP = pad4(W);
  const int preOff = s * RD, baseOff = preOff + (k + 1) * RP;
  const int total = baseOff + RP + 4;
  for (int i = threadIdx.x; i < total; i += blockDim.x) tab[i] = 0u;
  __syncthreads();
  for (int rec = threadIdx.x; rec < s + (k + 1) + 1; rec += blockDim.x) {
    if (rec < s) {
      const int32_t* row = M + (int64_t)(r - 1 - rec) * c;
      for (int i = 0; i < W; ++i) {
        const int32_t lo = 2 * i < c ? row[2 * i] : 0, hi = 2 * i + 1 < c ? row[2 * i + 1] : 0;
        tab[rec * RD + i] = pack2(lo, hi);
        tab[rec * RD + W + i] = pack2(-lo, -hi);
      }
    } else if (rec < s + k + 1) {
      const int x = rec - s;
      const int32_t* row = M + (int64_t)x * c;
      for (int i = 0; i < W; ++i) {
        const int32_t lo = 2 * i < c ? row[2 * i] : 0, hi = 2 * i + 1 < c ? row[2 * i + 1] : 0;
        tab[preOff + x * RP + i] = pack2(lo, hi);
      }
    } else {
      int32_t tsum = 0;
      for (int i = 0; i < W; ++i) {
        int32_t bl = 0, bh = 0;
        for (int x = 0; x < r; ++x) {
          const int32_t vl = 2 * i < c ? M[(int64_t)x * c + 2 * i] : 0;
          const int32_t vh = 2 * i + 1 < c ? M[(int64_t)x * c + 2 * i + 1] : 0;
          tsum += vl + vh;
          if (x > k) { bl += vl; bh += vh; }
        }
        tab[baseOff + i] = pack2(bl, bh);
      }
      tab[baseOff + RP] = (uint32_t)(-tsum);
    }
  }
}

template <int D, int W>
constexpr int ld16_units_per_lane() { return D * W <= 24 ? 2 : 1; }

size_t ld16_smem(int W, int k, int s) {
  return sizeof(uint32_t) * (size_t)(s * pad4(2 * W) + (k + 1) * pad4(W) + pad4(W) + 4);
}

template <int D, int W>
cudaError_t launch_one(const WalkParams& p, const uint32_t* tab, int grid, cudaStream_t st) {
  constexpr int P = ld16_units_per_lane<D, W>();
  const size_t sm = ld16_smem(W, p.k, p.s);
  cudaError_t e = ensure_dyn_smem((const void*)walk_ld16_kernel<D, W, P>, sm);
  if (e != cudaSuccess) return e;
  walk_ld16_kernel<D, W, P><<<grid, kBlock, sm, st>>>(p, tab);
  return cudaGetLastError();
}

template <int D, int W>
int occ_one(int k, int s) {
  constexpr int P = ld16_units_per_lane<D, W>();
  const size_t sm = ld16_smem(W, k, s);
  const int nb = occupancy_cached((const void*)walk_ld16_kernel<D, W, P>, kBlock, sm);
  return nb;
}

template <int D, int W>
int upl_one() { return ld16_units_per_lane<D, W>(); }

#define LN_LD16_SWITCH(D, W_, FN, ...)                                                       \
  switch (W_) {                                                                              \
    case 1: return FN<D, 1>(__VA_ARGS__);   case 2: return FN<D, 2>(__VA_ARGS__);            \
    case 3: return FN<D, 3>(__VA_ARGS__);   case 4: return FN<D, 4>(__VA_ARGS__);            \
    case 5: return FN<D, 5>(__VA_ARGS__);   case 6: return FN<D, 6>(__VA_ARGS__);            \
    case 7: return FN<D, 7>(__VA_ARGS__);   case 8: return FN<D, 8>(__VA_ARGS__);            \
    case 9: return FN<D, 9>(__VA_ARGS__);   case 10: return FN<D, 10>(__VA_ARGS__);          \
    case 11: return FN<D, 11>(__VA_ARGS__); case 12: return FN<D, 12>(__VA_ARGS__);          \
    case 13: return FN<D, 13>(__VA_ARGS__); case 14: return FN<D, 14>(__VA_ARGS__);          \
    case 15: return FN<D, 15>(__VA_ARGS__); case 16: return FN<D, 16>(__VA_ARGS__);          \
    default: break;                                                                          \
  }

int words_of(int c) { return (c + 1) / 2; }

}  // namespace

bool walk_ld16_supported(int d, int c, int s) {
  if ((d != 3 && d != 4) || c < 1 || s < 1) return false;
  const int W = words_of(c);
  if (W > 16) return false;
  const int k_max_words = s * pad4(2 * W) + 64 * pad4(W) + pad4(W) + 4;
  return k_max_words <= kTabWords;
}

int walk_ld16_units_per_lane(int d, int c) {
  const int W = words_of(c);
  if (d == 3) { LN_LD16_SWITCH(3, W, upl_one) }
  if (d == 4) { LN_LD16_SWITCH(4, W, upl_one) }
  return 1;
}

int walk_ld16_occupancy(int d, int c, int k, int s, int* block_out) {
  *block_out = kBlock;
  const int W = words_of(c);
  if (d == 3) { LN_LD16_SWITCH(3, W, occ_one, k, s) }
  if (d == 4) { LN_LD16_SWITCH(4, W, occ_one, k, s) }
  return 0;
}

cudaError_t walk_ld16_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st, int* block_out) {
  *block_out = kBlock;
  const int W = words_of(p.c);
  uint32_t* tab = reinterpret_cast<uint32_t*>(scratch_tab);
  const int total = p.s * pad4(2 * W) + (p.k + 1) * pad4(W) + pad4(W) + 4;
  if (total > kTabWords) return cudaErrorInvalidValue;
  build_table_ld16_kernel<<<1, 128, 0, st>>>(p.M, p.r, p.c, W, p.k, p.s, tab);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.d == 3) { LN_LD16_SWITCH(3, W, launch_one, p, tab, grid, st) }
  if (p.d == 4) { LN_LD16_SWITCH(4, W, launch_one, p, tab, grid, st) }
  return cudaErrorInvalidValue;
}

}  // namespace lnorm
