// Hot d-ary Gray walk for L_d, d in {3, 4} (Eqs. 6-7).
//
// A unit fixes rows 0..k to one restricted-growth prefix (R1: the
// canonical labelling removes the d! relabelling symmetry; the paper fixes one
// entry); the s suffix rows are walked in the d-ary reflected
// Gray code of Eqs. (13)-(15), suffix digit i <-> row r-1-i.
// All lanes of a warp walk the same suffix sequence, so the changed digit
// (Eq. 17) and the old/new labels (p, q) are warp-uniform.
//
// Per step (Eqs. 18-19): m_p -= M_rho, m_q += M_rho; only
// ||m_p||_1 and ||m_q||_1 are recomputed and value = sum_a ||m_a||_1.
// The lowest digit (row r-1) is unrolled: within a block of d words it climbs
// 0 -> d-1 (even block) or descends d-1 -> 0 (odd block) with compile-time
// (p, q); the block-start step changes digit >= 1 and dispatches on (p, q)
// with a warp-uniform switch over the 2(d-1) reflected-code cases.
#include "common.cuh"

namespace lnorm {

namespace {

constexpr int kTabInts = 8448;
constexpr int kBlock = 32;   // one warp per block (see the schedule comment in the kernel)

// Layout (ints): [0, 2sC): suffix rows, index (2i + neg) * C  (neg: -M_rho)
//                then (k+1)C prefix rows 0..k; then C suffix base sum_{x>k} M_xy.
__constant__ int32_t cTab[kTabInts];

template <int D, int C>
struct LdWalker {
  static __device__ __forceinline__ int32_t norm(const int32_t (&v)[C]) {
    int32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int y = 0; y < C; ++y) {
      int32_t& a = (y & 3) == 0 ? a0 : (y & 3) == 1 ? a1 : (y & 3) == 2 ? a2 : a3;
      a = __sad(v[y], 0, a);
    }
    return (a0 + a1) + (a2 + a3);
  }
  // move suffix row (table index i) from group P to group Q; returns new value
  template <int P, int Q>
  static __device__ __forceinline__ int32_t move(int32_t (&m)[D][C], int32_t (&n)[D], int32_t v, int i) {
    const int offPos = (2 * i) * C, offNeg = (2 * i + 1) * C;
#pragma unroll
    for (int y = 0; y < C; ++y) {
      m[P][y] += cTab[offNeg + y];
      m[Q][y] += cTab[offPos + y];
    }
    const int32_t np = norm(m[P]), nq = norm(m[Q]);
    v += (np - n[P]) + (nq - n[Q]);
    n[P] = np;
    n[Q] = nq;
    return v;
  }
  static __device__ __forceinline__ int32_t move_dyn(int32_t (&m)[D][C], int32_t (&n)[D], int32_t v, int i,
                                                     int p, int q) {
    switch (p * D + q) {
      case 0 * D + 1: return move<0, 1>(m, n, v, i);
      case 1 * D + 0: return move<1, 0>(m, n, v, i);
      case 1 * D + 2: return move<1, 2>(m, n, v, i);
      case 2 * D + 1: return move<2, 1>(m, n, v, i);
      default: break;
    }
    if constexpr (D >= 4) {
      switch (p * D + q) {
        case 2 * D + 3: return move<2, 3>(m, n, v, i);
        case 3 * D + 2: return move<3, 2>(m, n, v, i);
        default: break;
      }
    }
    return v;
  }
};

template <int D, int C>
__global__ void __launch_bounds__(kBlock) walk_ld_kernel(const WalkParams p) {
  const int lane = threadIdx.x & 31;
  const int s = p.s, k = p.k;
  const int preOff = 2 * s * C, baseOff = preOff + (k + 1) * C;
  // number of d-blocks in a unit: D^(s-1)
  uint32_t nblk = 1;
  for (int i = 1; i < s; ++i) nblk *= D;
  int32_t best = INT32_MIN;
  uint32_t best_u = 0;
  bool have = false;
  // Static warp-chunk schedule: block = one warp, so the chunk index (and every
  // Gray-control value derived from it) is provably warp-uniform and ptxas keeps
  // the walk's row addressing on the uniform datapath (LDCU + VIADD R, R, UR).
  const int64_t nchunks = (p.unit_count + 31) / 32;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t rel = ch * 32 + lane;
    const bool active = rel < p.unit_count;
    const int64_t u = p.unit_begin + (active ? rel : 0);
    int32_t m[D][C];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int y = 0; y < C; ++y) m[a][y] = (a == 0) ? cTab[baseOff + y] : 0;
    for (int x = 0; x <= k; ++x) {
      const int dig = prefix_digit(p, u, x);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const int32_t f = (dig == a) ? 1 : 0;
#pragma unroll
        for (int y = 0; y < C; ++y) m[a][y] += f * cTab[preOff + x * C + y];
      }
    }
    int32_t n[D];
    int32_t v = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) { n[a] = LdWalker<D, C>::norm(m[a]); v += n[a]; }
    int32_t ub = v;
    for (uint32_t t = 0; t < nblk; ++t) {
      if (t != 0) {
        uint32_t i, from, to;
        dary_block_start<D>(t, &i, &from, &to);
        v = LdWalker<D, C>::move_dyn(m, n, v, (int)i, (int)from, (int)to);
        ub = max(ub, v);
      }
      if ((t & 1u) == 0) {
#pragma unroll
        for (int a = 0; a + 1 < D; ++a) {
          if (a == 0) v = LdWalker<D, C>::template move<0, 1>(m, n, v, 0);
          if (a == 1) v = LdWalker<D, C>::template move<1, 2>(m, n, v, 0);
          if constexpr (D >= 4) { if (a == 2) v = LdWalker<D, C>::template move<2, 3>(m, n, v, 0); }
          ub = max(ub, v);
        }
      } else {
#pragma unroll
        for (int a = D - 1; a >= 1; --a) {
          if (a == 1) v = LdWalker<D, C>::template move<1, 0>(m, n, v, 0);
          if (a == 2) v = LdWalker<D, C>::template move<2, 1>(m, n, v, 0);
          if constexpr (D >= 4) { if (a == 3) v = LdWalker<D, C>::template move<3, 2>(m, n, v, 0); }
          ub = max(ub, v);
        }
      }
    }
    if (active) {
      if (p.unit_max) p.unit_max[rel] = ub;
      if (!have || ub > best) { best = ub; best_u = (uint32_t)u; have = true; }
    }
  }
  unsigned long long key = have ? make_key(best, best_u) : 0ull;
  key = warp_max_u64(key);
  if (lane == 0 && key) atomicMax(p.key, key);
}

__global__ void build_table_ld_kernel(const int32_t* M, int r, int c, int C, int k, int s, int32_t* tab) {
  const int preOff = 2 * s * C, baseOff = preOff + (k + 1) * C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < baseOff + C; i += gridDim.x * blockDim.x) {
    int32_t v = 0;
    if (i < preOff) {
      const int rowi = i / C, y = i % C, di = rowi >> 1, ng = rowi & 1;
      if (y < c) v = (ng ? -1 : 1) * M[(int64_t)(r - 1 - di) * c + y];
    } else if (i < baseOff) {
      const int x = (i - preOff) / C, y = (i - preOff) % C;
      if (y < c) v = M[(int64_t)x * c + y];
    } else {
      const int y = i - baseOff;
      if (y < c) for (int x = k + 1; x < r; ++x) v += M[(int64_t)x * c + y];
    }
    tab[i] = v;
  }
}

template <int D, int C>
cudaError_t launch_one(const WalkParams& p, int grid, cudaStream_t st) {
  walk_ld_kernel<D, C><<<grid, kBlock, 0, st>>>(p);
  return cudaGetLastError();
}
template <int D, int C>
int occ_one() {
  const int nb = occupancy_cached((const void*)walk_ld_kernel<D, C>, kBlock, 0);
  return nb;
}

constexpr int padC(int c) { return (c + 3) & ~3; }

#define LN_LD_SWITCH(D, C_, FN, ...)                                                \
  switch (C_) {                                                                     \
    case 4: return FN<D, 4>(__VA_ARGS__);   case 8: return FN<D, 8>(__VA_ARGS__);   \
    case 12: return FN<D, 12>(__VA_ARGS__); case 16: return FN<D, 16>(__VA_ARGS__); \
    case 20: return FN<D, 20>(__VA_ARGS__); case 24: return FN<D, 24>(__VA_ARGS__); \
    case 28: return FN<D, 28>(__VA_ARGS__); case 32: return FN<D, 32>(__VA_ARGS__); \
    default: break;                                                                 \
  }

}  // namespace

bool walk_ld_supported(int d, int c, int s) {
  return (d == 3 || d == 4) && c >= 1 && padC(c) <= 32 && s >= 1;
}

int walk_ld_occupancy(int d, int c, int* block_out) {
  *block_out = kBlock;
  const int C = padC(c);
  if (d == 3) { LN_LD_SWITCH(3, C, occ_one) }
  if (d == 4) { LN_LD_SWITCH(4, C, occ_one) }
  return 0;
}

cudaError_t walk_ld_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st, int* block_out) {
  const int C = padC(p.c);
  const int total = (2 * p.s + p.k + 2) * C;
  if (total > kTabInts) return cudaErrorInvalidValue;
  build_table_ld_kernel<<<8, 256, 0, st>>>(p.M, p.r, p.c, C, p.k, p.s, scratch_tab);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbolAsync(cTab, scratch_tab, sizeof(int32_t) * total, 0, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  *block_out = kBlock;
  if (p.d == 3) { LN_LD_SWITCH(3, C, launch_one, p, grid, st) }
  if (p.d == 4) { LN_LD_SWITCH(4, C, launch_one, p, grid, st) }
  return cudaErrorInvalidValue;
}

}  // namespace lnorm
