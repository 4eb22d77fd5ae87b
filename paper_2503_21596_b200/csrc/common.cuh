// Shared device-side definitions of the walk kernels (product path).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

#include "gray.cuh"

namespace lnorm {

enum Mode : int32_t { MODE_L1 = 0, MODE_MARG = 1, MODE_LD = 2 };

// bits per packed prefix digit for a label alphabet of size `base`
__host__ __device__ __forceinline__ int prefix_bits(int base) { return base <= 2 ? 1 : (base <= 4 ? 2 : 3); }

constexpr int kMaxRows = 64;       // enumerated rows after orientation
constexpr int kMaxCols = 1024;     // columns after orientation
constexpr int kMaxD = 8;

// One launch of a walk kernel over a contiguous range of units.
// A unit = one fixed prefix (rows 0..k) whose suffix (rows k+1..r-1, s = r-1-k
// digits) is walked completely in reflected Gray order.
struct WalkParams {
  const int32_t* M;              // device, r x c row-major (oriented)
  int32_t r, c;                  // enumerated rows, columns
  int32_t mode;                  // Mode
  int32_t d;                     // 2 for +-1 strategies and L_2, else label count
  int32_t k;                     // prefix rows 1..k (row 0 fixed); unit prefix length k+1
  int32_t s;                     // suffix digits
  int64_t unit_begin;            // first global unit index of this launch
  int64_t unit_count;            // units in this launch
  int32_t pbits;                 // bits per packed prefix digit (1, 2 or 3)
  const uint64_t* prefix_table;  // packed prefix digits (pbits per row 0..k) or nullptr:
                                 //   binary arithmetic prefix, digit of row x = bit (k-x) of u
  unsigned long long* counter;   // work counter (zeroed before launch)
  // dynamic chunk schedule of the byte walks (LN_DYN_CHUNKS): chunks beyond the first wave are
  // handed out by an atomicAdd on this word, zeroed by the table-build kernel that precedes every
  // walk launch; nullptr = static round-robin chunks
  unsigned long long* chunk_ctr;
  unsigned long long* key;       // global max key (zeroed before launch)
  int64_t* unit_max;             // optional per-unit maxima (index u - unit_begin)
  // batched launches (walk_pair16 only; every other kernel uses batch == 1):
  // matrix b has its oriented matrix at M + b*m_stride, its tables at
  // table + b*tab_stride / init + b*init_stride and its key at key[b];
  // each matrix has units_per units (unit_count = batch * units_per).
  int32_t batch;
  int64_t units_per;
  int64_t m_stride, tab_stride, init_stride;
  uint32_t one;                  // = 1 (a uniform operand the compiler cannot fold)
  int32_t u8_lpu;                // byte walk: lanes per unit (1, or 2 for > 128 columns)
  // reduction keys carry unit >> key_shift (a 32-bit "key unit"): splits with more than 2^32
  // units (byte walk only) compare groups of 2^key_shift consecutive units; the recovery then
  // re-walks the whole winning group (lex order = unit order, so the smallest group holding
  // an optimum holds the smallest optimal unit)
  int32_t key_shift;
  // self-check builds (LN_SELFCHECK): added to every from-scratch value before the comparison
  // (test hook LNORM_SELFCHECK_INJECT: a nonzero delta must make the call fail)
  int32_t selfcheck_delta;
  // byte binary walk (L_1 / L_2): every strategy value <= 65535 (sum |M|), so two units' running
  // maxima may share a register as 16-bit halves (set by the host planner)
  int32_t u8_pack_max;
};

// Defaults for a single-matrix launch.
inline void walk_params_single(WalkParams& p) {
  p.one = 1;
  if (p.u8_lpu < 1) p.u8_lpu = 1;
  p.batch = 1;
  p.units_per = p.unit_count;
  p.m_stride = p.tab_stride = p.init_stride = 0;
}

// Max-reduction key: high word = value biased to unsigned order, low word =
// ~unit so that, among equal values, the SMALLEST unit index wins
// (R2: lexicographically smallest optimum).
__host__ __device__ __forceinline__ unsigned long long make_key(int32_t v, uint32_t unit) {
  return ((unsigned long long)((uint32_t)v ^ 0x80000000u) << 32) | (unsigned long long)(0xFFFFFFFFu - unit);
}
__host__ __device__ __forceinline__ int32_t key_value(unsigned long long key) {
  return (int32_t)((uint32_t)(key >> 32) ^ 0x80000000u);
}
__host__ __device__ __forceinline__ uint32_t key_unit(unsigned long long key) {
  return 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
}

// Prefix digit of row x (0..k) of unit u.
__device__ __forceinline__ int prefix_digit(const WalkParams& p, int64_t u, int x) {
  if (p.prefix_table) return (int)((p.prefix_table[u - p.unit_begin] >> (p.pbits * x)) & ((1ull << p.pbits) - 1ull));
  return x == 0 ? 0 : (int)((u >> (p.k - x)) & 1);
}

// Broadcast 16-byte shared-memory load issued as volatile PTX: every Gray step
// re-reads its row (one LDS.128 per 4 words) instead of letting ptxas keep the
// few distinct rows of an unrolled block resident in registers, which would
// cost more registers (and occupancy) than the loads cost issue slots.
__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
  return v;
}

// Dynamic chunk schedule (byte walks).  A warp's first chunk is blockIdx.x; every later one is
// gridDim.x + an atomicAdd on p.chunk_ctr by lane 0 when the warp finishes its current chunk
// (fetched at the end, not prefetched: a prefetched index would stay live across the walk and
// push the 168-register L_3 instances into stack spills).  Warps that the schedulers favour take
// more chunks, so every warp of the grid stays resident until the work runs out (static
// round-robin chunks left ~20 % of the resident warps idle at the end of L_3 searches: ncu
// sm__warps_active 9.5 of 12).  The reduction key orders by value and unit only, so the result
// does not depend on which warp walked a chunk.
#ifndef LN_DYN_CHUNKS
#define LN_DYN_CHUNKS 1
#endif
__device__ __forceinline__ int64_t next_chunk(int64_t ch, unsigned long long* ctr, int lane) {
  if (LN_DYN_CHUNKS && ctr) {
    unsigned long long nx = 0;
    if (lane == 0) nx = atomicAdd(ctr, 1ull);
    return (int64_t)gridDim.x + (int64_t)__shfl_sync(0xffffffffu, nx, 0);
  }
  return ch + gridDim.x;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Host: raise a kernel's dynamic shared-memory limit to >= bytes once per (kernel, device)
// instead of at every launch, and the SM count per device (cached; launch paths call these
// per search, so they must be cheap).
inline cudaError_t ensure_dyn_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  size_t& have = done[{fn, dev}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
// Resident blocks per SM of a kernel at (block, dynamic smem), computed once per device.
inline int occupancy_cached(const void* fn, int block, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<std::pair<const void*, int>, std::pair<int, size_t>>, int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = done.find({{fn, dev}, {block, smem}});
    if (it != done.end()) return it->second;
  }
  if (smem > 48 * 1024 && ensure_dyn_smem(fn, smem) != cudaSuccess) return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, block, smem) != cudaSuccess) { (void)cudaGetLastError(); return 0; }
  std::lock_guard<std::mutex> g(mu);
  done[{{fn, dev}, {block, smem}}] = nb;
  return nb;
}
inline int device_sms() {
  static int nsm[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!nsm[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    nsm[dev] = v > 0 ? v : 148;
  }
  return nsm[dev];
}

}  // namespace lnorm

// Kernel launchers (one per translation unit); return cudaError_t.
namespace lnorm {
struct LaunchCfg { int grid, block; size_t smem; cudaStream_t stream; };
// Hot binary walk (L_1, L_marg, L_2): r, c within the template set, s >= 4.
bool walk_bin_supported(int mode, int c, int s);
// scratch_tab: device buffer of >= 8448 int32 used to stage the constant table.
cudaError_t walk_bin_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st,
                            int* block_out);
int walk_bin_occupancy(int mode, int c, int* block_out);
template <int MODE> cudaError_t walk_bin_launch_mode(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st);
template <int MODE> int walk_bin_occupancy_mode(int c);
// Packed 16-bit binary walk (exactness guard checked by the caller).
bool walk_bin16_supported(int mode, int c, int s);
cudaError_t walk_bin16_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st, int* block_out);
int walk_bin16_occupancy(int mode, int c, int k, int s, int* block_out);
template <int MODE> int walk_bin16_words(int c);
template <int MODE> cudaError_t walk_bin16_launch_mode(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st);
template <int MODE> int walk_bin16_occupancy_mode(int c, int k, int s);
template <int MODE> int walk_bin16_units_per_lane_mode(int c);
template <int MODE> int walk_bin16_unroll_mode(int c);
template <int MODE> int64_t walk_bin16_table_words_mode(int c, int k, int s);
bool walk_bin16_table_fits(int mode, int c, int k, int s);
int walk_bin16_units_per_lane(int mode, int c);
// Hot d-ary walk (L_d, d in {3,4}).
bool walk_ld_supported(int d, int c, int s);
cudaError_t walk_ld_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st,
                           int* block_out);
int walk_ld_occupancy(int d, int c, int* block_out);
// Strategy-paired packed 16-bit binary walk (guard: sum |M| <= 16383, checked by the caller).
bool walk_pair16_supported(int mode, int c, int s);
int walk_pair16_units_per_lane(int mode, int c);
int walk_pair16_occupancy(int mode, int c, int s, int* block_out);
// scratch_init: device buffer of >= 16384 int32 for the unit-init records.
cudaError_t walk_pair16_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                               cudaStream_t st, int* block_out);
template <int MODE> int walk_pair16_cols(int c);
template <int MODE> cudaError_t walk_pair16_launch_mode(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init,
                                                        int grid, cudaStream_t st);
template <int MODE> int walk_pair16_occupancy_mode(int c, int s);
template <int MODE> int walk_pair16_units_per_lane_mode(int c);
template <int MODE> int walk_pair16_unroll_mode(int c);
template <int MODE> void walk_pair16_table_sizes_mode(int c, int k, int s, int64_t* tab_words, int64_t* init_ints);
void walk_pair16_table_sizes(int mode, int c, int k, int s, int64_t* tab_words, int64_t* init_ints);
// Packed 16-bit d-ary walk (L_d, d in {3,4}; exactness guard checked by the caller).
bool walk_ld16_supported(int d, int c, int s);
int walk_ld16_units_per_lane(int d, int c);
int walk_ld16_occupancy(int d, int c, int k, int s, int* block_out);
cudaError_t walk_ld16_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st, int* block_out);
// d-ary walk with the last row evaluated for all d labels per word (guard: sum |M| <= 32767).
bool walk_ldpair16_supported(int d, int c, int s);
int walk_ldpair16_units_per_lane(int d, int c);
int walk_ldpair16_occupancy(int d, int c, int s, int* block_out);
cudaError_t walk_ldpair16_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                                 cudaStream_t st, int* block_out);
// Byte-packed binary walk (L_1, L_marg, L_2): four column sums per register as offset
// bytes; exact when every column's suffix window fits a byte (guard checked by the caller).
bool walk_u8_supported(int mode, int c, int s, int lpu = 1);
int walk_u8_units_per_lane(int mode, int c, int lpu = 1);
int walk_u8_occupancy(int mode, int c, int s, int lpu, int* block_out);
cudaError_t walk_u8_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                           cudaStream_t st, int* block_out);
template <int MODE> int walk_u8_words_mode(int c);
template <int MODE> void walk_u8_table_sizes_mode(int c, int k, int s, int lpu, int64_t* tab_words, int64_t* init_ints);
// per-matrix delta-table words and init-record ints of a byte-walk launch (batched strides)
void walk_u8_table_sizes(int mode, int c, int k, int s, int lpu, int64_t* tab_words, int64_t* init_ints);
template <int MODE> cudaError_t walk_u8_launch_mode(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init,
                                                    int grid, cudaStream_t st);
template <int MODE> int walk_u8_occupancy_mode(int c, int s, int lpu);
template <int MODE> int walk_u8_units_per_lane_mode(int c, int lpu);
template <int MODE> int walk_u8_lanes_per_unit_mode(int c);
template <int MODE> int walk_u8_paired_rows_mode();
int walk_u8_lanes_per_unit(int mode, int c);
// packed words per unit of the byte-walk instance for c columns (0 = none)
int walk_u8_words(int mode, int c);
template <int MODE> int walk_u8_unroll_mode(int c, int lpu);
// Byte-packed d-ary walk, last row paired (L_d, d in {3,4}; guard: every column's
// sum_x |M_xy| <= 255, checked by the caller).
bool walk_ldu8_supported(int d, int c, int s);
// rows the byte d-ary walk pairs for a unit of s suffix digits (the all-H kernel's 3-4 for L_3)
int walk_ldu8_paired_rows(int d, int s);
int walk_ldu8_units_per_lane(int d, int c, int s);
int walk_ldu8_occupancy(int d, int c, int s, int* block_out);
cudaError_t walk_ldu8_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                             cudaStream_t st, int* block_out);
// per-matrix delta-table words and init-record ints of a byte d-ary launch (batched strides)
void walk_ldu8_table_sizes(int d, int c, int k, int s, int64_t* tab_words, int64_t* init_ints);
template <int D, int PART> int walk_ldu8_upl_part(int NW, int s);
template <int D, int PART> int walk_ldu8_occ_part(int NW, int s);
template <int D, int PART> cudaError_t walk_ldu8_launch_part(const WalkParams& p, const uint32_t* tab, const int32_t* init,
                                                             int grid, cudaStream_t st, int NW);
// Byte-packed L_3 / L_4 walk, 3-5 paired rows, all-H form, bias words in shared memory
// (walk_ldu8w_impl.cuh); dispatched by walk_ldu8_launch for L_3 and L_4 when the suffix allows.
template <int D, int PART> cudaError_t walk_ldu8w_launch_part(const WalkParams& p, const uint32_t* tab,
                                                              const int32_t* init, int grid, cudaStream_t st, int NW,
                                                              int pr);
template <int D, int PART> int walk_ldu8w_occ_part(int NW, int pr, int s);
template <int D, int PART> int walk_ldu8w_upl_part(int NW, int pr);
template <int D, int PART> int walk_ldu8w_pk_part(int NW, int pr);
// single-search L_3 / L_4 byte walks: 1 if the instance keeps two units per lane with packed sums
int walk_ldu8_packed(int d, int c, int s);
// Generic warp-per-unit walk (any mode, d, c, s).
bool walk_generic_supported(int d, int c);
cudaError_t walk_generic_launch(const WalkParams& p, int grid, cudaStream_t st, int* block_out);
int walk_generic_occupancy(int d, int c, int* block_out);
// Argmax recovery: re-walk the units key_unit(*key) << key_shift .. + 2^key_shift - 1 and
// write the smallest (unit offset << 32 | lexicographic suffix key) attaining
// key_value(*key) into *lex_out (atomicMin), and the largest value seen (biased as the
// key's high word) into *rmax_out (atomicMax) for the self-check.  Batched launches:
// lex_out / rmax_out / key are per matrix; the batch is passed in p.batch (<= 65535).
cudaError_t recover_launch(const WalkParams& p, unsigned long long* lex_out, unsigned long long* rmax_out,
                           cudaStream_t st);
// Trace: per-step values of one unit (test hook).
cudaError_t trace_launch(const WalkParams& p, int64_t max_steps, int64_t* values, int8_t* digits,
                         cudaStream_t st);
}  // namespace lnorm
