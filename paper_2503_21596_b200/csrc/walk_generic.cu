// Generic warp-per-unit Gray walk, argmax recovery and the trace hook.
//
// Every norm is written in the group-sum form of Eqs. (6)-(7):
// the strategy assigns each row a label, (m_a)_y = sum_{x: a_x = a} M_xy, and a
// step of the reflected Gray code moves ONE row rho from group `from` to group
// `to` (Eqs. 18-19):  m_from -= M_rho,  m_to += M_rho.
//   L_d    : value = sum_a ||m_a||_1                                  (Eq. 6)
//   L_1    : labels 0/1 <-> a_x = +1/-1, m = m_0 - m_1, value = ||m||_1   (Eq. 1;
//            moving a row between the groups is Eq. 12's m += +-2 M_rho)
//   L_marg : value = m_0[0] - m_1[0] + sum_{y>=1} |m_0 - m_1|_y        (Eq. 2)
// The lanes of a warp split the columns; the change digit (Eq. 9 / Eq. 17) is
// warp-uniform.  This kernel covers every shape (any c <= 1024, any d <= 8,
// any suffix length) and is the correctness anchor for shapes outside the
// hot kernels' template set; recover and trace reuse the same device code.
#include <algorithm>

#include "common.cuh"

namespace lnorm {

namespace {

constexpr int kGenWarps = 4;   // warps per block

__device__ __forceinline__ int groups_of(const WalkParams& p) { return p.mode == MODE_LD ? p.d : 2; }
__device__ __forceinline__ int base_of(const WalkParams& p) { return p.mode == MODE_LD ? p.d : 2; }

// Initialise the warp's group sums for unit u with suffix word `w0` (digits of
// the reflected Gray code, Eq. 8 / Eqs. 13-15; suffix digit i <-> row r-1-i).
__device__ void gen_init(const WalkParams& p, int64_t u, uint64_t w0, int32_t* G, int lane) {
  const int nG = groups_of(p), base = base_of(p);
  for (int y = lane; y < p.c; y += 32) {
    for (int a = 0; a < nG; ++a) G[a * p.c + y] = 0;
  }
  for (int x = 0; x < p.r; ++x) {
    int lab;
    if (x <= p.k) lab = prefix_digit(p, u, x);
    else lab = (int)dary_digit((uint32_t)base, (uint32_t)(p.r - 1 - x), w0);
    const int32_t* row = p.M + (int64_t)x * p.c;
    for (int y = lane; y < p.c; y += 32) G[lab * p.c + y] += row[y];
  }
}

__device__ int32_t gen_value(const WalkParams& p, const int32_t* G, int lane) {
  int32_t v = 0;
  if (p.mode == MODE_LD) {
    for (int a = 0; a < p.d; ++a)
      for (int y = lane; y < p.c; y += 32) v += abs(G[a * p.c + y]);
  } else {
    for (int y = lane; y < p.c; y += 32) {
      int32_t mm = G[y] - G[p.c + y];
      v += (p.mode == MODE_MARG && y == 0) ? mm : abs(mm);
    }
  }
  return __reduce_add_sync(0xffffffffu, v);
}

__device__ __forceinline__ void gen_move(const WalkParams& p, int32_t* G, int row, int from, int to, int lane) {
  const int32_t* R = p.M + (int64_t)row * p.c;
  for (int y = lane; y < p.c; y += 32) {
    int32_t v = R[y];
    G[from * p.c + y] -= v;
    G[to * p.c + y] += v;
  }
}

__device__ __forceinline__ uint64_t ipow64(uint32_t b, int e) {
  uint64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// Batched launches (p.batch > 1, many small matrices): work item t is unit
// t % units_per of matrix t / units_per (matrix b at M + b*m_stride, key[b]).
__global__ void __launch_bounds__(32 * kGenWarps) walk_generic_kernel(const WalkParams p) {
  extern __shared__ int32_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nG = groups_of(p);
  int32_t* G = smem + wib * nG * p.c;
  const uint32_t base = (uint32_t)base_of(p);
  const uint64_t words = ipow64(base, p.s);
  unsigned long long best_key = 0;
  WalkParams q = p;
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(p.counter, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((int64_t)t >= p.unit_count) break;
    int64_t lu = (int64_t)t, b = 0;
    if (p.batch > 1) { b = lu / p.units_per; lu -= b * p.units_per; q.M = p.M + b * p.m_stride; }
    const int64_t u = p.unit_begin + lu;
    gen_init(q, u, 0, G, lane);
    int32_t best = gen_value(q, G, lane);
    for (uint64_t w = 1; w < words; ++w) {
      uint32_t i, from, to;
      dary_change_values(base, w, &i, &from, &to);
      gen_move(q, G, p.r - 1 - (int)i, (int)from, (int)to, lane);
      int32_t v = gen_value(q, G, lane);
      best = v > best ? v : best;
    }
    if (p.unit_max && lane == 0) p.unit_max[t] = best;
    unsigned long long kk = make_key(best, (uint32_t)u);
    if (p.batch > 1) { if (lane == 0) atomicMax(p.key + b, kk); }
    else best_key = kk > best_key ? kk : best_key;
  }
  if (lane == 0 && best_key) atomicMax(p.key, best_key);
}

// Recovery: the words of the winning unit are split into contiguous chunks
// (Algorithm 1), one per warp; each warp starts from its
// chunk's first word by the closed form and walks it, keeping the smallest
// lexicographic suffix key among words whose value equals the optimum.  The
// re-walk recomputes every value with independent int32 group sums, so it also
// checks the hot kernels: the largest value it sees goes to rmax_out (biased like
// the key) and must equal the key's value (host check, LNORM_EINTERNAL otherwise).
__device__ void recover_one(const WalkParams& p, unsigned long long* lex_out, unsigned long long* rmax_out,
                            int32_t* G, int lane, int wib) {
  const uint32_t base = (uint32_t)base_of(p);
  const uint64_t words = ipow64(base, p.s);
  const unsigned long long key = *p.key;
  const int32_t target = key_value(key);
  const int64_t g0 = (int64_t)key_unit(key) << p.key_shift;    // first unit of the winning key group
  const int64_t gcount = 1LL << p.key_shift;
  const uint64_t T = (uint64_t)gridDim.x * kGenWarps;
  const uint64_t t = (uint64_t)blockIdx.x * kGenWarps + wib;
  const uint64_t J = words / T, R = words % T;
  const uint64_t lo = t * J + (t < R ? t : R);
  const uint64_t hi = lo + J + (t < R ? 1 : 0);
  if (lo >= hi) return;
  if (key == 0ull || g0 < p.unit_begin || g0 >= p.unit_begin + p.unit_count) return;   // no valid key: report nothing
  unsigned long long bestlex = ~0ull;
  int32_t vmax = INT32_MIN;
  for (int64_t o = 0; o < gcount; ++o) {
    const int64_t u = g0 + o;
    if (u >= p.unit_begin + p.unit_count) break;              // (a group may run past the last unit)
    gen_init(p, u, lo, G, lane);
    uint64_t lex = 0;
    for (int i = 0; i < p.s; ++i) lex += (uint64_t)dary_digit(base, (uint32_t)i, lo) * ipow64(base, i);
    const unsigned long long hiword = (unsigned long long)o << 32;
    int32_t v = gen_value(p, G, lane);
    vmax = max(vmax, v);
    if (v == target && (hiword | lex) < bestlex) bestlex = hiword | lex;
    for (uint64_t w = lo + 1; w < hi; ++w) {
      uint32_t i, from, to;
      dary_change_values(base, w, &i, &from, &to);
      gen_move(p, G, p.r - 1 - (int)i, (int)from, (int)to, lane);
      lex = lex + (uint64_t)to * ipow64(base, (int)i) - (uint64_t)from * ipow64(base, (int)i);
      v = gen_value(p, G, lane);
      vmax = max(vmax, v);
      if (v == target && (hiword | lex) < bestlex) bestlex = hiword | lex;
    }
    if (bestlex != ~0ull) break;                              // an earlier unit of the group wins
  }
  if (lane == 0) {
    if (bestlex != ~0ull) atomicMin(lex_out, bestlex);
    atomicMax(rmax_out, (unsigned long long)((uint32_t)vmax ^ 0x80000000u));
  }
}

// Batched launches: matrices b = blockIdx.y, blockIdx.y + gridDim.y, ... (any batch size).
// stage_m: the block first copies the (oriented) matrix into shared memory, so every Gray step
// reads its row there instead of through L2 (the recovery is latency-bound: one unit, short
// chunks per warp).
__global__ void __launch_bounds__(32 * kGenWarps) recover_kernel(const WalkParams pin, unsigned long long* lex_out,
                                                                 unsigned long long* rmax_out, int stage_m) {
  extern __shared__ int32_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int rc = pin.r * pin.c;
  int32_t* G = smem + (stage_m ? rc : 0) + wib * groups_of(pin) * pin.c;
  const int nb = pin.batch > 0 ? pin.batch : 1;
  for (int b = blockIdx.y; b < nb; b += gridDim.y) {
    WalkParams p = pin;
    p.M = pin.M + (int64_t)b * pin.m_stride;
    p.key = pin.key + b;
    if (stage_m) {
      __syncthreads();
      for (int i = threadIdx.x; i < rc; i += blockDim.x) smem[i] = p.M[i];
      __syncthreads();
      p.M = smem;
    }
    recover_one(p, lex_out + b, rmax_out + b, G, lane, wib);
  }
}

// Trace: one warp walks unit p.unit_begin and records every step.
__global__ void trace_kernel(const WalkParams p, int64_t max_steps, int64_t* values, int8_t* digits) {
  extern __shared__ int32_t smem[];
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)base_of(p);
  const uint64_t words = ipow64(base, p.s);
  int32_t* G = smem;
  const int64_t u = p.unit_begin;
  gen_init(p, u, 0, G, lane);
  int8_t dig[kMaxRows];
  for (int x = 0; x < p.r; ++x) dig[x] = (int8_t)(x <= p.k ? prefix_digit(p, u, x) : 0);
  for (uint64_t w = 0; w < words && (int64_t)w < max_steps; ++w) {
    if (w > 0) {
      uint32_t i, from, to;
      dary_change_values(base, w, &i, &from, &to);
      gen_move(p, G, p.r - 1 - (int)i, (int)from, (int)to, lane);
      dig[p.r - 1 - i] = (int8_t)to;
    }
    int32_t v = gen_value(p, G, lane);
    if (lane == 0) {
      values[w] = v;
      if (digits)
        for (int x = 0; x < p.r; ++x) digits[w * p.r + x] = dig[x];
    }
  }
}

size_t gen_smem(int nG, int c, int warps) { return (size_t)nG * c * warps * sizeof(int32_t); }

}  // namespace

bool walk_generic_supported(int d, int c) {
  const int nG = d < 2 ? 2 : d;
  return c >= 1 && c <= kMaxCols && (size_t)nG * c * sizeof(int32_t) * kGenWarps <= 200 * 1024;
}

int walk_generic_occupancy(int d, int c, int* block_out) {
  const int nG = d < 2 ? 2 : d;
  size_t sm = gen_smem(nG, c, kGenWarps);
  const int nb = occupancy_cached((const void*)walk_generic_kernel, 32 * kGenWarps, sm);
  *block_out = 32 * kGenWarps;
  return nb;
}

cudaError_t walk_generic_launch(const WalkParams& p, int grid, cudaStream_t st, int* block_out) {
  const int nG = p.mode == MODE_LD ? p.d : 2;
  size_t sm = gen_smem(nG, p.c, kGenWarps);
  cudaError_t e = ensure_dyn_smem((const void*)walk_generic_kernel, sm);
  if (e != cudaSuccess) return e;
  walk_generic_kernel<<<grid, 32 * kGenWarps, sm, st>>>(p);
  *block_out = 32 * kGenWarps;
  return cudaGetLastError();
}

cudaError_t recover_launch(const WalkParams& p, unsigned long long* lex_out, unsigned long long* rmax_out,
                           cudaStream_t st) {
  const int nG = p.mode == MODE_LD ? p.d : 2;
  const size_t gsm = gen_smem(nG, p.c, kGenWarps);
  const size_t msm = sizeof(int32_t) * (size_t)p.r * p.c;
  const int stage = gsm + msm <= 96 * 1024 ? 1 : 0;
  const size_t sm = gsm + (stage ? msm : 0);
  const int nsm = device_sms();
  cudaError_t e = ensure_dyn_smem((const void*)recover_kernel, std::max<size_t>(sm, 96 * 1024));
  if (e != cudaSuccess) return e;
  // blocks per matrix: enough warps for ~2-word chunks, at most 4 blocks per SM.  The recovery is
  // latency-bound (one warp per chunk, a d-ary step of this generic walk is a few hundred cycles
  // of dependent work, the chunk's init ~1-2k): a 20x20 search's 32-word unit took 21 us with
  // 8-word chunks on one block (ncu: 4 warps, 9 cycles per instruction), several us with 2-word
  // chunks; large units still fill 4 blocks per SM
  uint64_t words = 1;
  for (int i = 0; i < p.s; ++i) words *= (uint64_t)(p.mode == MODE_LD ? p.d : 2);
  int gx = (int)std::min<uint64_t>((uint64_t)nsm * 4, std::max<uint64_t>(1, words / (2ull * kGenWarps)));
  if (p.batch > 1) gx = std::max(1, std::min(gx, (nsm * 8 + p.batch - 1) / p.batch));
  const int gy = std::max(1, std::min(p.batch > 0 ? p.batch : 1, 65535));
  recover_kernel<<<dim3(gx, gy), 32 * kGenWarps, sm, st>>>(p, lex_out, rmax_out, stage);
  return cudaGetLastError();
}

cudaError_t trace_launch(const WalkParams& p, int64_t max_steps, int64_t* values, int8_t* digits,
                         cudaStream_t st) {
  const int nG = p.mode == MODE_LD ? p.d : 2;
  size_t sm = gen_smem(nG, p.c, 1);
  cudaError_t e = ensure_dyn_smem((const void*)trace_kernel, sm);
  if (e != cudaSuccess) return e;
  trace_kernel<<<1, 32, sm, st>>>(p, max_steps, values, digits);
  return cudaGetLastError();
}

}  // namespace lnorm
