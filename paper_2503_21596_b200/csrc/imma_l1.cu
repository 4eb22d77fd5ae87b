// the tcgen05 `kind::i8` (integer tensor-core) formulation of the L_1 search
// -- an EXPERIMENT, measured against the byte-packed Gray walk and not adopted.
//
// What it computes (Eq. 1): L_1(M) = max_a sum_y |sum_x a_x M_xy| over
// a in {+-1}^n with a_0 = +1, for the strategies it is asked to cover.  Instead of
// walking a Gray code on the ALU (Eq. 12), a tile of 512 strategies has its column sums formed
// by ONE tensor-core instruction, the product of a strategy tile with M:
//
//   D[l][(i, y)] = sum_k A[l][k] * B[(i, y)][k]                 (int8 x int8 -> int32 in TMEM)
//
//   strategy (t, i, l) of tile t: rows 1, 2 carry the two bits of i in [0, 4) (the MMA's N
//   blocks), rows 3..n-8 the bits of the reflected Gray word g(t) = t ^ (t >> 1),
//   the last 7 rows the bits of l in [0, 128) (the MMA's M = 128 lanes); set bit = -1.
//   A[l][k]  = a_{n-7+k}(l) for k < 7;  1 for k = 8..13;  0 otherwise
//   B[(i,y)][k] = M_{n-7+k, y} for k < 7;  four int8 pieces of Q_y(t) = M_0y + sum_{x=3..n-8}
//   a_x(t) M_xy for k = 8..11 (the pieces sum to Q_y exactly);  a_1(i) M_1y, a_2(i) M_2y for
//   k = 12, 13;  0 otherwise  (N = 4 * CP columns, CP = c rounded up to 4).
//
// so D holds m_y(t, i, l) = sum_x a_x M_xy exactly.  The producer warp advances Q_y along the
// Gray code (one row update per tile, Eq. 12, rows staged as 2 M in shared memory), writes its
// pieces into the B operand and issues the MMA (one elected thread, cta_group::1, M = 128,
// N = 4 CP, K = 32) into one of two TMEM stages; sixteen epilogue warps read their lane
// quadrant back with tcgen05.ld and accumulate sum_y |m_y| (one ALU |.|-accumulate per column
// per strategy) and the running max.
//
// Why it cannot win (the measurement is the point): the byte walk spends 1/4
// ALU instruction per column per strategy (VABSDIFF4 on four byte-packed columns); here every
// column arrives as a 32-bit TMEM word and costs one full ALU instruction plus its share of
// the tcgen05.ld traffic, so the ALU floor alone is 4x the byte walk's.
//
// Operand layout: K-major, no swizzle: 8-row x 16-byte core matrices; row r, K byte kb lives at
// (kb / 16) * LBO + (r / 8) * 128 + (r % 8) * 16 + kb % 16 with LBO = rows / 8 * 128 (the distance
// between the two 16-byte K halves) and SBO = 128 (between 8-row groups).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "lnorm.h"

namespace {

constexpr int kLow = 7;                  // low rows per tile: 2^7 = 128 strategies = MMA M
constexpr int kHper = 4;                 // sign patterns of rows 1, 2 per tile (N = kHper * CP)
constexpr int kEpiWarps = 16;            // 4 lane quadrants x 4 patterns
constexpr int kThreads = 32 * (1 + kEpiWarps);
constexpr int kStageCols = 256;          // TMEM columns per accumulator stage (2 stages, 512 allocated)
constexpr int kAbytes = 128 * 32;
constexpr int kMaxC = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;                // descriptor version (sm_100)
  return d;                              // base offset 0, layout type 0 = no swizzle
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, int32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}

__device__ __forceinline__ int cm_off(int row, int kb, int rows) {   // core-matrix byte offset
  return (kb >> 4) * (rows / 8) * 128 + (row >> 3) * 128 + (row & 7) * 16 + (kb & 15);
}

// Key: value in the high 22 bits (the host guarantees 0 <= value < 2^21), ~strategy in the low 42.
__device__ __forceinline__ unsigned long long imma_key(int32_t v, uint64_t idx) {
  return ((unsigned long long)(uint32_t)v << 42) | ((1ull << 42) - 1 - idx);
}

// four int8 pieces summing to q (|q| <= 508), packed little-endian
__device__ __forceinline__ uint32_t int8_pieces(int32_t q) {
  uint32_t w = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int32_t pc = max(-127, min(127, q));
    q -= pc;
    w |= ((uint32_t)(uint8_t)(int8_t)pc) << (8 * e);
  }
  return w;
}

template <int CP>
__global__ void __launch_bounds__(kThreads, 1)
imma_l1_kernel(const int32_t* __restrict__ M, int r, int c, uint64_t tile_begin, uint64_t tile_count,
               unsigned long long* key_out) {
  constexpr int N = kHper * CP;
  constexpr int Bbytes = N * 32;
  static_assert(N % 16 == 0 && N <= kStageCols && CP % 4 == 0, "MMA N for M = 128");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB0 = smem + kAbytes;                      // two stages of B
  int32_t* sD = reinterpret_cast<int32_t*>(smem + kAbytes + 2 * Bbytes);   // 2 M_x of the Gray rows
  const int HB = r - 1 - kLow;                        // rows 1..HB above the low block
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + (HB + 1) * kMaxC);     // full[2], empty[2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- tile range of this CTA (contiguous, so the producer walks one Gray run)
  const uint64_t per = tile_count / gridDim.x, rem = tile_count % gridDim.x;
  const uint64_t t0 = tile_begin + blockIdx.x * per + min((uint64_t)blockIdx.x, rem);
  const uint64_t nt = per + (blockIdx.x < rem ? 1 : 0);

  // ---- operands: A (fixed), the constant part of both B stages, the Gray rows
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int l = i >> 5, kb = i & 31;
    int8_t v = 0;
    if (kb < kLow) v = ((l >> kb) & 1) ? -1 : 1;
    else if (kb >= 8 && kb < 14) v = 1;
    sA[cm_off(l, kb, 128)] = (uint8_t)v;
  }
  for (int i = threadIdx.x; i < N * 32; i += blockDim.x) {
    const int row = i >> 5, kb = i & 31, y = row % CP, pat = row / CP;
    int8_t v = 0;
    if (y < c) {
      if (kb < kLow) v = (int8_t)M[(r - kLow + kb) * c + y];
      else if (kb == 12) v = (int8_t)((pat & 1) ? -M[c + y] : M[c + y]);            // row 1
      else if (kb == 13) v = (int8_t)((pat & 2) ? -M[2 * c + y] : M[2 * c + y]);    // row 2
    }
    sB0[cm_off(row, kb, N)] = (uint8_t)v;
    sB0[Bbytes + cm_off(row, kb, N)] = (uint8_t)v;
  }
  for (int i = threadIdx.x; i < (HB + 1) * kMaxC; i += blockDim.x) {
    const int x = i / kMaxC, y = i % kMaxC;
    sD[i] = (y < c) ? 2 * M[x * c + y] : 0;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&bar[i]), 1);                 // full: one tcgen05.commit
      mbar_init(smem_u32(&bar[2 + i]), kEpiWarps);     // empty: one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  unsigned long long best = 0;
  if (warp == 0) {
    // ===== producer: Q_y along the Gray code over rows 3..HB, its pieces, one MMA per tile
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t adesc = umma_smem_desc(smem_u32(sA), (128 / 8) * 128, 128);
    int32_t Q[2] = {0, 0};                             // columns lane, lane + 32
    {
      const uint64_t g = t0 ^ (t0 >> 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int y = lane + 32 * h;
        int32_t q = sD[y];
        for (int x = 3; x <= HB; ++x) q += ((g >> (x - 3)) & 1) ? -sD[x * kMaxC + y] : sD[x * kMaxC + y];
        Q[h] = q / 2;                                  // sD holds 2 M
      }
    }
    for (uint64_t tt = 0; tt < nt; ++tt) {
      const uint64_t t = t0 + tt;
      const int s = (int)(tt & 1);
      const uint32_t use = (uint32_t)(tt >> 1);
      if (tt != 0) {                                   // one Gray step (Eq. 9): row 3 + ctz(t)
        const int b = __ffsll((long long)t) - 1;
        const bool neg = (((t ^ (t >> 1)) >> b) & 1) != 0;
        const int32_t* row = sD + (3 + b) * kMaxC;
        Q[0] += neg ? -row[lane] : row[lane];
        Q[1] += neg ? -row[lane + 32] : row[lane + 32];
      }
      const uint32_t w0 = int8_pieces(Q[0]), w1 = int8_pieces(Q[1]);
      if (tt >= 2) mbar_wait(smem_u32(&bar[2 + s]), (use - 1) & 1);
      uint8_t* sB = sB0 + s * Bbytes;
#pragma unroll
      for (int i = 0; i < kHper; ++i) {
        if (lane < CP) *reinterpret_cast<uint32_t*>(sB + cm_off(i * CP + lane, 8, N)) = w0;
        if (lane + 32 < CP) *reinterpret_cast<uint32_t*>(sB + cm_off(i * CP + lane + 32, 8, N)) = w1;
      }
      fence_async_smem();
      __syncwarp();
      tc_fence_after();
      if (lane == 0) {
        const uint64_t bdesc = umma_smem_desc(smem_u32(sB), (N / 8) * 128, 128);
        const uint32_t dcol = tmem + (uint32_t)(s * kStageCols);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar[s]))
                     : "memory");
      }
      __syncwarp();
    }
  } else {
    // ===== epilogue: lane quadrant (warp % 4) of sign pattern i = (warp - 1) / 4 of every tile
    const int quad = warp & 3, i = (warp - 1) >> 2;
    const int l = quad * 32 + lane;
    int32_t bv = -1;
    uint64_t bidx = 0;
    for (uint64_t tt = 0; tt < nt; ++tt) {
      const int s = (int)(tt & 1);
      mbar_wait(smem_u32(&bar[s]), (uint32_t)(tt >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(s * kStageCols + i * CP);
      int32_t v[CP];
#pragma unroll
      for (int cc = 0; cc + 8 <= CP; cc += 8) tmem_ld8(taddr + cc, v + cc);
      if (CP % 8) tmem_ld4(taddr + (CP & ~7), v + (CP & ~7));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bar[2 + s]));
      uint32_t acc = 0;
#pragma unroll
      for (int y = 0; y < CP; ++y) acc = __sad(v[y], 0, acc);   // |m_y| accumulate (padding columns are 0)
      if ((int32_t)acc > bv) {
        bv = (int32_t)acc;
        bidx = ((t0 + tt) * kHper + i) * 128 + (uint64_t)l;
      }
    }
    if (nt) best = imma_key(bv, bidx);
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  if (lane == 0 && best) atomicMax(key_out, best);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int CP>
cudaError_t launch_imma(const int32_t* dM, int r, int c, uint64_t tb, uint64_t tc, unsigned long long* key, int grid,
                        cudaStream_t st) {
  const size_t sm = kAbytes + 2 * (size_t)kHper * CP * 32 + sizeof(int32_t) * (size_t)(r - kLow) * kMaxC + 64;
  cudaError_t e = cudaFuncSetAttribute(imma_l1_kernel<CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  imma_l1_kernel<CP><<<grid, kThreads, sm, st>>>(dM, r, c, tb, tc, key);
  return cudaGetLastError();
}

}  // namespace

extern "C" int lnorm_imma_l1(const int32_t* M, int32_t n, int32_t m, uint64_t tile_begin, uint64_t tile_count,
                             int64_t* value, int8_t* argmax, uint64_t* strategies, double* kernel_ms) {
  if (!M || !value || n < 2 + kLow + 1 || m < 1 || m > kMaxC) return LNORM_EINVAL;
  const int HB = n - 1 - kLow;
  if (HB > 35) return LNORM_ETOOLARGE;                 // strategy index < 2^42 (key layout)
  const uint64_t tiles_total = 1ull << (HB - 2);
  if (tile_count == 0) { tile_begin = 0; tile_count = tiles_total; }
  if (tile_begin >= tiles_total || tile_count > tiles_total - tile_begin) return LNORM_EINVAL;
  int64_t total = 0;
  for (int y = 0; y < m; ++y) {
    int64_t q = 0;
    for (int x = 0; x < n; ++x) {
      const int64_t a = llabs((long long)M[(size_t)x * m + y]);
      if ((x >= n - kLow || x == 1 || x == 2) && a > 127) return LNORM_EOVERFLOW;   // int8 B operand
      if (x == 0 || (x >= 3 && x < n - kLow)) q += a;
      total += a;
    }
    if (q > 4 * 127) return LNORM_EOVERFLOW;                     // four int8 pieces
  }
  if (total >= (1 << 21)) return LNORM_EOVERFLOW;                // key layout
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return LNORM_ENODEV;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int cp = ((m + 3) / 4) * 4;
  int32_t* dM = nullptr;
  unsigned long long* dKey = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = LNORM_OK;
  if (cudaMalloc(&dM, sizeof(int32_t) * (size_t)n * m) != cudaSuccess || cudaMalloc(&dKey, 8) != cudaSuccess) {
    cudaFree(dM);
    return LNORM_ENOMEM;
  }
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaMemcpyAsync(dM, M, sizeof(int32_t) * (size_t)n * m, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(dKey, 0, 8, st);
  const int grid = (int)((tile_count < (uint64_t)nsm) ? tile_count : (uint64_t)nsm);
  cudaEventRecord(e0, st);
  cudaError_t e = cudaErrorInvalidValue;
  switch (cp) {
#define LN_IMMA_CASE(CPV) \
  case CPV: e = launch_imma<CPV>(dM, n, m, tile_begin, tile_count, dKey, grid, st); break;
    LN_IMMA_CASE(4) LN_IMMA_CASE(8) LN_IMMA_CASE(12) LN_IMMA_CASE(16) LN_IMMA_CASE(20) LN_IMMA_CASE(24)
    LN_IMMA_CASE(28) LN_IMMA_CASE(32) LN_IMMA_CASE(36) LN_IMMA_CASE(40) LN_IMMA_CASE(44) LN_IMMA_CASE(48)
    LN_IMMA_CASE(52) LN_IMMA_CASE(56) LN_IMMA_CASE(60) LN_IMMA_CASE(64)
#undef LN_IMMA_CASE
  }
  cudaEventRecord(e1, st);
  unsigned long long key = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&key, dKey, 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    rc = LNORM_ECUDA;
  } else {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (kernel_ms) *kernel_ms = ms;
    const uint64_t idx = (1ull << 42) - 1 - (key & ((1ull << 42) - 1));
    *value = (int64_t)(key >> 42);
    if (argmax) {
      const uint64_t t = idx >> 9, i = (idx >> 7) & 3, l = idx & 127, g = t ^ (t >> 1);
      argmax[0] = 1;
      argmax[1] = (i & 1) ? -1 : 1;
      argmax[2] = (i & 2) ? -1 : 1;
      for (int x = 3; x <= HB; ++x) argmax[x] = ((g >> (x - 3)) & 1) ? -1 : 1;
      for (int k = 0; k < kLow; ++k) argmax[n - kLow + k] = ((l >> k) & 1) ? -1 : 1;
    }
    if (strategies) *strategies = tile_count * (uint64_t)kHper * 128;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(dM);
  cudaFree(dKey);
  return rc;
}
