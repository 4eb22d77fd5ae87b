// Hot d-ary Gray walk for L_d, d in {3, 4}, with the LAST row evaluated for all
// d labels at every walked word (packed 16-bit).
//
// Units and control as in walk_ld16.cu (restricted-growth prefixes, warp-uniform
// d-ary reflected walk, Eqs. 13-17), but the walked rows are k+1..r-2 and the
// last row rho = M_{r-1} is not walked: for every group g the lane keeps
//     R_g,y = ( B_g,y , B_g,y + rho_y )        (s16x2)
// where B_g = sum of the walked/prefix rows labelled g.  With
//     ||x||_1 = 2 sum max(x, 0) - sum x,   H_g = ( sum_y max(B_g,y, 0), sum_y max(B_g,y + rho_y, 0) )
// the value of the strategy that puts row r-1 into group a is (Eq. 6)
//     L*_d(a) = 2 [ sum_g H_g.lo + (H_a.hi - H_a.lo) ] - sum_y T_y ,
// so one walked word evaluates all d labellings of the last row:
//     best = max(best, sum_g H_g.lo + max_a (H_a.hi - H_a.lo)).
// A step moving a walked row from group p to q (Eqs. 18-19) updates R_p, R_q
// (one VIADD.16x2 per column each, both versions at once) and re-accumulates
// H_p, H_q (one VIADDMNMX.S16x2 per column each): 4c instructions per word for
// d strategies, i.e. 2c/d per column update counted as in SURVEY §8 (2c per
// strategy) -- below the one-instruction-per-update bound of a plain walk.
// Exactness guard: all 16-bit halves are bounded by S = sum_ij |M_ij| <= 32767.
#include "common.cuh"

namespace lnorm {

namespace {

constexpr int kBlock = 32;
constexpr int kTabWords = 8448;
#ifndef LN_LDP_CHUNKED
#define LN_LDP_CHUNKED 1
#endif
#ifndef LN_LDP_MINB
#define LN_LDP_MINB 12
#endif

__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }

template <int D, int C, int P>
struct LdPair {
  static constexpr int C4 = pad4(C);
  static constexpr int RD = 2 * C4;        // delta record: +row at [0, C), -row at [C4, C4 + C) (16B aligned)
  static __device__ __forceinline__ uint32_t half_sums(const uint32_t (&v)[C]) {
    uint32_t a0 = __vmaxs2(v[0], 0u), a1 = 0u;
#pragma unroll
    for (int i = 1; i < C; ++i) {
      if (i & 1) a1 = __viaddmax_s16x2(a1, v[i], a1);
      else a0 = __viaddmax_s16x2(a0, v[i], a0);
    }
    return __vadd2(a0, a1);
  }
  struct Unit {
    uint32_t R[D][C];
    int32_t lo[D], dd[D];
    int32_t lsum, best;
  };
  static __device__ __forceinline__ int32_t maxd(const int32_t (&dd)[D]) {
    if constexpr (D == 3) return __vimax3_s32(dd[0], dd[1], dd[2]);
    else return max(__vimax3_s32(dd[0], dd[1], dd[2]), dd[3]);
  }
  static __device__ __forceinline__ void refresh(Unit& U, int g, uint32_t H) {
    const int32_t l = (int32_t)(H & 0xFFFFu), h = (int32_t)(H >> 16);
    U.lsum += l - U.lo[g];
    U.lo[g] = l;
    U.dd[g] = h - l;
  }
  // move the walked row of record `off` from group PG to group QG in every unit
  template <int PG, int QG>
  static __device__ __forceinline__ void move(Unit (&U)[P], uint32_t sbase, int off) {
#if LN_LDP_CHUNKED
    // consume the +row / -row records a quad at a time (one LDS.128 each), updating and
    // re-accumulating both groups column by column: only two quads of the row stay live
    uint32_t ap0[P], ap1[P], aq0[P], aq1[P];
#pragma unroll
    for (int v = 0; v < (C + 3) / 4; ++v) {
      const uint4 pq = lds128(sbase + 4u * (uint32_t)(off + 4 * v));        // +row quad
      const uint4 nq = lds128(sbase + 4u * (uint32_t)(off + C4 + 4 * v));   // -row quad
      const uint32_t pp[4] = {pq.x, pq.y, pq.z, pq.w}, nn[4] = {nq.x, nq.y, nq.z, nq.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int y = 4 * v + e;
        if (y < C) {
#pragma unroll
          for (int j = 0; j < P; ++j) {
            U[j].R[PG][y] = __vadd2(U[j].R[PG][y], nn[e]);
            U[j].R[QG][y] = __vadd2(U[j].R[QG][y], pp[e]);
            if (y == 0) { ap0[j] = __vmaxs2(U[j].R[PG][0], 0u); aq0[j] = __vmaxs2(U[j].R[QG][0], 0u); }
            else if (y == 1) { ap1[j] = __vmaxs2(U[j].R[PG][1], 0u); aq1[j] = __vmaxs2(U[j].R[QG][1], 0u); }
            else if (y & 1) { ap1[j] = __viaddmax_s16x2(ap1[j], U[j].R[PG][y], ap1[j]); aq1[j] = __viaddmax_s16x2(aq1[j], U[j].R[QG][y], aq1[j]); }
            else { ap0[j] = __viaddmax_s16x2(ap0[j], U[j].R[PG][y], ap0[j]); aq0[j] = __viaddmax_s16x2(aq0[j], U[j].R[QG][y], aq0[j]); }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      refresh(U[j], PG, C > 1 ? __vadd2(ap0[j], ap1[j]) : ap0[j]);
      refresh(U[j], QG, C > 1 ? __vadd2(aq0[j], aq1[j]) : aq0[j]);
      U[j].best = max(U[j].best, U[j].lsum + maxd(U[j].dd));
    }
#else
    uint32_t r[RD];
#pragma unroll
    for (int v = 0; v < RD / 4; ++v) {
      const uint4 x4 = lds128(sbase + 4u * (uint32_t)(off + 4 * v));
      r[4 * v] = x4.x; r[4 * v + 1] = x4.y; r[4 * v + 2] = x4.z; r[4 * v + 3] = x4.w;
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
#pragma unroll
      for (int y = 0; y < C; ++y) {
        U[j].R[PG][y] = __vadd2(U[j].R[PG][y], r[C4 + y]);  // -row
        U[j].R[QG][y] = __vadd2(U[j].R[QG][y], r[y]);       // +row
      }
      refresh(U[j], PG, half_sums(U[j].R[PG]));
      refresh(U[j], QG, half_sums(U[j].R[QG]));
      U[j].best = max(U[j].best, U[j].lsum + maxd(U[j].dd));
    }
#endif
  }
  static __device__ __forceinline__ void move_dyn(Unit (&U)[P], uint32_t sbase, int off, int p, int q) {
    switch (p * D + q) {
      case 0 * D + 1: move<0, 1>(U, sbase, off); return;
      case 1 * D + 0: move<1, 0>(U, sbase, off); return;
      case 1 * D + 2: move<1, 2>(U, sbase, off); return;
      case 2 * D + 1: move<2, 1>(U, sbase, off); return;
      default: break;
    }
    if constexpr (D >= 4) {
      switch (p * D + q) {
        case 2 * D + 3: move<2, 3>(U, sbase, off); return;
        case 3 * D + 2: move<3, 2>(U, sbase, off); return;
        default: break;
      }
    }
  }
};

// Init records (global int32, stride IW = C + 1): prefix rows 0..k, the base
// (walked rows k+1..r-2 at label 0), the paired row r-1, then [sum T].
template <int D, int C, int P>
__global__ void __launch_bounds__(kBlock, (D * C * P <= 84 ? LN_LDP_MINB : 1)) walk_ldpair16_kernel(const WalkParams p, const uint32_t* __restrict__ gTab,
                                                               const int32_t* __restrict__ gInit) {
  using WK = LdPair<D, C, P>;
  constexpr int RD = WK::RD, IW = C + 1;
  extern __shared__ __align__(16) uint32_t sT[];
  const int lane = threadIdx.x & 31;
  const int sw = p.s - 1;
  for (int i = threadIdx.x; i < sw * RD; i += blockDim.x) sT[i] = gTab[i];
  __syncthreads();
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sT);
  const int32_t* baseRec = gInit + (p.k + 1) * IW;
  const int32_t* pairRec = baseRec + IW;
  const int32_t tsum = __ldg(pairRec + IW);
  uint32_t nblk = 1;
  for (int i = 1; i < sw; ++i) nblk *= D;
  int32_t best = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  const int64_t nchunks = (p.unit_count + 32 * P - 1) / (32 * P);
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    typename WK::Unit U[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = ch * 32 * P + j * 32 + lane;
      const int64_t u = p.unit_begin + (rel < p.unit_count ? rel : 0);
      int32_t B[D][C];
#pragma unroll
      for (int g = 0; g < D; ++g)
#pragma unroll
        for (int y = 0; y < C; ++y) B[g][y] = (g == 0) ? __ldg(baseRec + y) : 0;
      for (int x = 0; x <= p.k; ++x) {
        const int dig = prefix_digit(p, u, x);
        const int32_t* rec = gInit + x * IW;
#pragma unroll
        for (int g = 0; g < D; ++g) {
          const int32_t f = (dig == g) ? 1 : 0;
#pragma unroll
          for (int y = 0; y < C; ++y) B[g][y] += f * __ldg(rec + y);
        }
      }
      U[j].lsum = 0;
#pragma unroll
      for (int g = 0; g < D; ++g) {
#pragma unroll
        for (int y = 0; y < C; ++y) {
          const int32_t b = B[g][y], bp = b + __ldg(pairRec + y);
          U[j].R[g][y] = (uint32_t)(b & 0xFFFF) | ((uint32_t)(bp & 0xFFFF) << 16);
        }
        const uint32_t H = WK::half_sums(U[j].R[g]);
        U[j].lo[g] = (int32_t)(H & 0xFFFFu);
        U[j].dd[g] = (int32_t)(H >> 16) - U[j].lo[g];
        U[j].lsum += U[j].lo[g];
      }
      U[j].best = U[j].lsum + WK::maxd(U[j].dd);
    }
    for (uint32_t t = 0; t < nblk; ++t) {
      if (t != 0) {
        uint32_t i, from, to;
        dary_block_start<D>(t, &i, &from, &to);
        WK::move_dyn(U, sbase, (int)i * RD, (int)from, (int)to);
      }
      if ((t & 1u) == 0) {
        WK::template move<0, 1>(U, sbase, 0);
        WK::template move<1, 2>(U, sbase, 0);
        if constexpr (D >= 4) WK::template move<2, 3>(U, sbase, 0);
      } else {
        if constexpr (D >= 4) WK::template move<3, 2>(U, sbase, 0);
        WK::template move<2, 1>(U, sbase, 0);
        WK::template move<1, 0>(U, sbase, 0);
      }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int64_t rel = ch * 32 * P + j * 32 + lane;
      if (rel < p.unit_count) {
        const int32_t ub = 2 * U[j].best - tsum;
        if (p.unit_max) p.unit_max[rel] = ub;
        if (!have || ub > best) { best = ub; best_u = (uint32_t)(p.unit_begin + rel); have = true; }
      }
    }
  }
  unsigned long long key = have ? make_key(best, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key) atomicMax(p.key, key);
}

__global__ void build_ldpair16_kernel(const int32_t* M, int r, int c, int C, int k, int s, uint32_t* tab,
                                      int32_t* init) {
  const int C4 = pad4(C), RD = 2 * C4, IW = C + 1, sw = s - 1;
  for (int i = threadIdx.x; i < sw * RD; i += blockDim.x) tab[i] = 0u;
  for (int i = threadIdx.x; i < (k + 3) * IW + 1; i += blockDim.x) init[i] = 0;
  __syncthreads();
  for (int rec = threadIdx.x; rec < sw; rec += blockDim.x) {           // walked digit rec <-> row r-2-rec
    const int32_t* row = M + (int64_t)(r - 2 - rec) * c;
    for (int y = 0; y < C; ++y) {
      const int32_t v = y < c ? row[y] : 0;
      tab[rec * RD + y] = (uint32_t)(v & 0xFFFF) * 0x10001u;
      tab[rec * RD + C4 + y] = (uint32_t)((-v) & 0xFFFF) * 0x10001u;
    }
  }
  for (int rec = threadIdx.x; rec < k + 3; rec += blockDim.x) {
    int32_t* out = init + rec * IW;
    if (rec <= k) {
      for (int y = 0; y < C; ++y) out[y] = y < c ? M[(int64_t)rec * c + y] : 0;
    } else if (rec == k + 1) {
      for (int y = 0; y < C; ++y) {
        int32_t b = 0;
        if (y < c) for (int x = k + 1; x < r - 1; ++x) b += M[(int64_t)x * c + y];
        out[y] = b;
      }
    } else {
      int32_t t = 0;
      for (int y = 0; y < C; ++y) out[y] = y < c ? M[(int64_t)(r - 1) * c + y] : 0;
      for (int64_t i = 0; i < (int64_t)r * c; ++i) t += M[i];
      init[(k + 3) * IW] = t;                                            // sum_y T_y
    }
  }
}

template <int D, int C>
constexpr int ldpair_units_per_lane() { return D * C <= 40 ? 2 : 1; }

size_t ldpair_smem(int C, int s) { return sizeof(uint32_t) * (size_t)((s - 1) * 2 * pad4(C)); }

template <int D, int C>
cudaError_t launch_one(const WalkParams& p, const uint32_t* tab, const int32_t* init, int grid, cudaStream_t st) {
  constexpr int P = ldpair_units_per_lane<D, C>();
  const size_t sm = ldpair_smem(C, p.s);
  cudaError_t e = ensure_dyn_smem((const void*)walk_ldpair16_kernel<D, C, P>, sm);
  if (e != cudaSuccess) return e;
  walk_ldpair16_kernel<D, C, P><<<grid, kBlock, sm, st>>>(p, tab, init);
  return cudaGetLastError();
}

template <int D, int C>
int occ_one(int s) {
  constexpr int P = ldpair_units_per_lane<D, C>();
  const size_t sm = ldpair_smem(C, s);
  const int nb = occupancy_cached((const void*)walk_ldpair16_kernel<D, C, P>, kBlock, sm);
  return nb;
}

template <int D, int C>
int upl_one() { return ldpair_units_per_lane<D, C>(); }

#define LN_LDP_SWITCH(D, C_, FN, ...)                                                        \
  switch (C_) {                                                                              \
    case 2: return FN<D, 2>(__VA_ARGS__);   case 4: return FN<D, 4>(__VA_ARGS__);            \
    case 6: return FN<D, 6>(__VA_ARGS__);   case 8: return FN<D, 8>(__VA_ARGS__);            \
    case 10: return FN<D, 10>(__VA_ARGS__); case 12: return FN<D, 12>(__VA_ARGS__);          \
    case 14: return FN<D, 14>(__VA_ARGS__); case 16: return FN<D, 16>(__VA_ARGS__);          \
    case 18: return FN<D, 18>(__VA_ARGS__); case 20: return FN<D, 20>(__VA_ARGS__);          \
    case 22: return FN<D, 22>(__VA_ARGS__); case 24: return FN<D, 24>(__VA_ARGS__);          \
    case 26: return FN<D, 26>(__VA_ARGS__); case 28: return FN<D, 28>(__VA_ARGS__);          \
    case 30: return FN<D, 30>(__VA_ARGS__); case 32: return FN<D, 32>(__VA_ARGS__);          \
    default: break;                                                                          \
  }

int cols_of(int c) { return c < 2 ? 2 : (c + 1) & ~1; }

}  // namespace

bool walk_ldpair16_supported(int d, int c, int s) {
  if ((d != 3 && d != 4) || c < 1 || s < 2) return false;
  const int C = cols_of(c);
  if (C > 32) return false;
  return (s - 1) * 2 * pad4(C) <= kTabWords;
}

int walk_ldpair16_units_per_lane(int d, int c) {
  const int C = cols_of(c);
  if (d == 3) { LN_LDP_SWITCH(3, C, upl_one) }
  if (d == 4) { LN_LDP_SWITCH(4, C, upl_one) }
  return 1;
}

int walk_ldpair16_occupancy(int d, int c, int s, int* block_out) {
  *block_out = kBlock;
  const int C = cols_of(c);
  if (d == 3) { LN_LDP_SWITCH(3, C, occ_one, s) }
  if (d == 4) { LN_LDP_SWITCH(4, C, occ_one, s) }
  return 0;
}

cudaError_t walk_ldpair16_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                                 cudaStream_t st, int* block_out) {
  *block_out = kBlock;
  const int C = cols_of(p.c);
  if ((p.s - 1) * 2 * pad4(C) > kTabWords || (p.k + 3) * (C + 1) + 1 > 16384) return cudaErrorInvalidValue;
  uint32_t* tab = reinterpret_cast<uint32_t*>(scratch_tab);
  build_ldpair16_kernel<<<1, 128, 0, st>>>(p.M, p.r, p.c, C, p.k, p.s, tab, scratch_init);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.d == 3) { LN_LDP_SWITCH(3, C, launch_one, p, tab, scratch_init, grid, st) }
  if (p.d == 4) { LN_LDP_SWITCH(4, C, launch_one, p, tab, scratch_init, grid, st) }
  return cudaErrorInvalidValue;
}

}  // namespace lnorm
