// C ABI (include/lnorm.h): validation, orientation, unit planning, device
// contexts, launches, the single NCCL all-reduce of the multi-GPU variants and
// the argmax recovery / finalisation kernels.  Host code here only marshals
// and plans; every step of the search runs in the kernels.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <cstdio>
#include <functional>
#include <string>
#include <map>
#include <memory>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: host ranges per phase (SURVEY.md §5 tracing)

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/lnorm.h"
#include "common.cuh"

using namespace lnorm;

namespace lnorm {
size_t reduce_scratch_ints(int n, int m);
cudaError_t reduce_launch(const int32_t* M, int n, int m, int mode, int32_t* scratch, int32_t* R, int32_t* rowsel,
                          int32_t* info_dev, cudaStream_t st);
cudaError_t mapback_launch(int n, int m, int nred, int ld, int32_t* scratch, const int32_t* rowsel,
                           const int8_t* argr, int8_t* out, int32_t* info_dev, cudaStream_t st);
}  // namespace lnorm

namespace {

// NVTX range for the lifetime of a scope: the host phases of a call (guard statistics,
// planning, walk enqueue, all-reduce, recovery) show up as named ranges in nsys / ncu's NVTX
// filter (`ncu --nvtx --nvtx-include "lnorm.walk/"`).  Costs ~100 ns per range without a tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ------------------------------------------------------------------ NCCL --
// NCCL is resolved at run time (dlopen) so the library loads on hosts without
// it and shares the process's already-loaded libnccl (e.g. torch's).
struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (h) break;
    }
    if (!h) for (const char* nm : names) { h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL); if (h) break; }
    if (!h) return;
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(h, "ncclCommInitRank");
    n.CommInitAll = (decltype(n.CommInitAll))dlsym(h, "ncclCommInitAll");
    n.AllReduce = (decltype(n.AllReduce))dlsym(h, "ncclAllReduce");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(h, "ncclCommDestroy");
    n.CommAbort = (decltype(n.CommAbort))dlsym(h, "ncclCommAbort");
    n.CommCount = (decltype(n.CommCount))dlsym(h, "ncclCommCount");
    n.CommUserRank = (decltype(n.CommUserRank))dlsym(h, "ncclCommUserRank");
    n.GroupStart = (decltype(n.GroupStart))dlsym(h, "ncclGroupStart");
    n.GroupEnd = (decltype(n.GroupEnd))dlsym(h, "ncclGroupEnd");
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommInitAll && n.AllReduce && n.CommDestroy && n.CommAbort &&
           n.CommCount && n.CommUserRank;
  });
  return n;
}

// --------------------------------------------------------------- problem --
struct Problem {
  int n = 0, m = 0, d = 1, marg = 0;
  int mode = MODE_L1;   // Mode
  int dl = 2;           // labels walked: 2 for +-1 strategies, else effective d
  bool transposed = false;
  int r = 0, c = 0;     // enumerated rows / columns
  bool fits16 = false;  // packed 16-bit column-pair path is exact
  bool fitsPair = false;  // strategy-paired path is exact: sum |M| <= 16383
  bool fitsLdPair = false;  // last-row-paired d-ary path is exact: sum |M| <= 32767
  bool fitsU16 = false;     // every strategy value fits 16 unsigned bits: sum |M| <= 65535 (packed maxima)
  // u8 guard: sufW[s] = max over columns y of sum_{x = r-s}^{r-1} |M_xy| (the last s rows)
  int64_t sufW[kMaxRows + 1] = {};
};

// Exactness-guard statistics of the oriented matrix (the data-dependent half of
// validation; the host computes them for host input, guard_stats_kernel for device
// input -- same definitions):
//   S       = sum |M_ij| (int64; > 2^31-1 => EOVERFLOW, P:259 integer exactness)
//   par[i]  = packed column-pair guard: sum over the columns y >= c0 with (y - c0) & 1 == i
//             of sum_x |M_xy| (c0 = 1 for L_marg's linear column, else 0)
//   sufW[s] = byte-path guard: max over columns y of sum over the last s enumerated rows
//             of |M_xy| (s = 1..r)
struct GuardStats {
  int64_t S = 0;
  int64_t par[2] = {0, 0};
  int64_t sufW[kMaxRows + 1] = {};
};

// Entry (x, y) of the ORIENTED r x c matrix from the caller's n x m M.
inline int64_t oriented(const int32_t* M, int m, bool transposed, int x, int y) {
  return transposed ? M[(int64_t)y * m + x] : M[(int64_t)x * m + y];
}

void host_stats(const int32_t* M, const Problem& p, GuardStats* g) {
  std::vector<int64_t> colw(p.c, 0);
  g->sufW[0] = 0;
  for (int s = 1; s <= p.r; ++s) {
    const int x = p.r - s;
    int64_t mx = 0;
    for (int y = 0; y < p.c; ++y) {
      const int64_t v = oriented(M, p.m, p.transposed, x, y);
      colw[y] += v < 0 ? -v : v;
      mx = std::max(mx, colw[y]);
    }
    g->sufW[s] = mx;
  }
  const int c0 = p.mode == MODE_MARG ? 1 : 0;
  g->S = 0; g->par[0] = g->par[1] = 0;
  for (int y = 0; y < p.c; ++y) {
    g->S += colw[y];
    if (y >= c0) g->par[(y - c0) & 1] += colw[y];
  }
}

// One block of 256 threads: each thread owns columns y = tid, tid + 256, ... (c <= 1024);
// per suffix length a warp max goes to shared memory (no block barrier per row), one barrier
// at the end combines the eight warps.
__global__ void __launch_bounds__(256) guard_stats_kernel(const int32_t* M, int m, int transposed, int r, int c,
                                                          int marg, long long* out, int64_t m_stride = 0,
                                                          int out_stride = 0) {
  M += blockIdx.x * m_stride;              // batched calls: one block per matrix
  out += blockIdx.x * out_stride;
  constexpr int kW = 8, kPer = kMaxCols / 256;
  __shared__ long long red[kMaxRows][kW];
  __shared__ long long red3[3][kW];
  long long colw[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) colw[i] = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto wmax = [](long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { const long long w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
    return v;
  };
  auto wsum = [](long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  for (int s = 1; s <= r; ++s) {
    const int x = r - s;
    long long mx = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int y = threadIdx.x + i * 256;
      if (y < c) {
        const long long v = transposed ? M[(int64_t)y * m + x] : M[(int64_t)x * m + y];
        colw[i] += v < 0 ? -v : v;
        mx = colw[i] > mx ? colw[i] : mx;
      }
    }
    mx = wmax(mx);
    if (lane == 0) red[s - 1][wid] = mx;
  }
  long long S = 0, p0 = 0, p1 = 0;
  const int c0 = marg ? 1 : 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int y = threadIdx.x + i * 256;
    if (y < c) {
      S += colw[i];
      if (y >= c0) { if ((y - c0) & 1) p1 += colw[i]; else p0 += colw[i]; }
    }
  }
  S = wsum(S); p0 = wsum(p0); p1 = wsum(p1);
  if (lane == 0) { red3[0][wid] = S; red3[1][wid] = p0; red3[2][wid] = p1; }
  __syncthreads();
  if (threadIdx.x < r) {
    long long v = red[threadIdx.x][0];
    for (int w = 1; w < kW; ++w) v = red[threadIdx.x][w] > v ? red[threadIdx.x][w] : v;
    out[3 + threadIdx.x] = v;
  }
  if (threadIdx.x < 3) {
    long long v = 0;
    for (int w = 0; w < kW; ++w) v += red3[threadIdx.x][w];
    out[threadIdx.x] = v;
  }
}

// log2 of the u8 kernel's lane group: its units differ in the last lane_bits prefix
// rows, which join the byte window (walk_u8_impl.cuh "Lane groups")
int u8_lane_bits(const Problem& p, int lpu = 1) {
  const int P = walk_u8_units_per_lane(p.mode, p.c, lpu);
  return P >= 8 ? 3 : P >= 4 ? 2 : (P == 2 ? 1 : 0);
}

// Byte-packed path guard (walk_u8_impl.cuh): a unit's window of column y spans
// 2 W_y (L_1, L_marg: +-1 on every window row) or W_y (L_2 / L_d), W_y = sum over the
// window rows of |M_xy|; it must fit an unsigned byte.
bool u8_fits(const Problem& p, int s) {
  if (s < 1 || s > p.r) return false;
  return p.mode == MODE_LD ? p.sufW[s] <= 255 : 2 * p.sufW[s] <= 255;
}

// Shape half of validation (no entries read): argument checks, orientation, limits.
int validate_shape(int n, int m, int d, int marg, Problem* pr) {
  if (n < 1 || m < 1 || d < 1 || d > kMaxD || (marg != 0 && marg != 1)) return LNORM_EINVAL;
  if (marg && d != 1) return LNORM_EINVAL;
  Problem p;
  p.n = n; p.m = m; p.d = d; p.marg = marg;
  if (d == 1) {
    p.mode = marg ? MODE_MARG : MODE_L1;
    p.dl = 2;
    p.transposed = n > m;                 // PAPER.md:144 (L_1); R5 (L_marg)
    p.r = p.transposed ? m : n;
    p.c = p.transposed ? n : m;
  } else {
    p.mode = MODE_LD;
    p.dl = std::max(2, std::min(d, n));   // L_d = L_min(d,n) (at most n labels used)
    p.r = n; p.c = m;                     // never transposed
  }
  if (p.r > kMaxRows - 1 || p.c > kMaxCols) return LNORM_ETOOLARGE;
  // search space d^(r-1) must fit a 63-bit word index
  long double space = 1;
  for (int i = 0; i < p.r - 1; ++i) space *= p.dl;
  if (space >= 9.2e18L) return LNORM_ETOOLARGE;
  *pr = p;
  return LNORM_OK;
}

// Data half: the guards that pick the exact kernel families.
int apply_stats(const GuardStats& g, Problem* p) {
  if (g.S > INT32_MAX) return LNORM_EOVERFLOW;
  p->fits16 = g.par[0] <= 32767 && g.par[1] <= 32767;
  for (int s = 0; s <= kMaxRows; ++s) p->sufW[s] = g.sufW[s];
  p->fitsPair = g.S <= 16383;
  p->fitsLdPair = g.S <= 32767;
  p->fitsU16 = g.S <= 65535;
  return LNORM_OK;
}

int validate(const int32_t* M, int n, int m, int d, int marg, Problem* pr) {
  if (!M) return LNORM_EINVAL;
  Problem p;
  int rc = validate_shape(n, m, d, marg, &p);
  if (rc) return rc;
  GuardStats g;
  host_stats(M, p, &g);
  if ((rc = apply_stats(g, &p))) return rc;
  *pr = p;
  return LNORM_OK;
}

// ------------------------------------------------------------------ plan --
enum Kernel { K_BIN = 0, K_LD = 1, K_GEN = 2, K_BIN16 = 3, K_LD16 = 4, K_PAIR16 = 5, K_LDPAIR16 = 6, K_U8 = 7, K_LDU8 = 8 };

// LNORM_KERNEL=auto|u8|pair16|packed|int32|generic forces a kernel family (benchmarks
// and tests): the named family or, where it cannot run, the next one down the
// preference order u8 > pair16 > packed > int32 > generic.
int kernel_override() {
  const char* e = getenv("LNORM_KERNEL");
  if (!e || !*e || !strcmp(e, "auto") || !strcmp(e, "u8")) return -1;
  if (!strcmp(e, "int32")) return K_BIN;
  if (!strcmp(e, "generic")) return K_GEN;
  if (!strcmp(e, "packed")) return K_BIN16;
  if (!strcmp(e, "pair16")) return K_PAIR16;
  return -1;
}

struct Plan {
  int kernel = K_GEN;
  int k = 0, s = 0;
  int u8_lpu = 1;                // byte walk: lanes per unit
  int key_shift = 0;             // reduction keys carry unit >> key_shift (units > 2^32, byte walk)
  int64_t units = 1;
  std::vector<uint64_t> table;   // packed prefixes (RGS for d >= 3, explicit for hooks); empty = arithmetic
  // RGS plans: the process-wide immutable prefix list for (k, d), shared instead of copied
  std::shared_ptr<const std::vector<uint64_t>> shared;
  const std::vector<uint64_t>& prefixes() const { return shared ? *shared : table; }
};

constexpr int64_t kNominalLanes = 148LL * 1024;   // plan is hardware-independent => identical on every rank
constexpr int kMaxKeyShift = 8;                    // byte walk: up to 2^39 units (the recovery re-walks <= 256)
constexpr int64_t kTableCap = 1LL << 22;

// All restricted-growth prefixes of length k+1 with labels < d, in lexicographic order.
void rgs_enumerate(int len, int d, std::vector<uint64_t>& out, int64_t cap) {
  const int pb = prefix_bits(d);
  std::vector<int> dig(len, 0);
  // iterative DFS in lexicographic order
  std::function<bool(int, int)> rec = [&](int pos, int mx) -> bool {
    if (pos == len) {
      uint64_t w = 0;
      for (int x = 0; x < len; ++x) w |= (uint64_t)dig[x] << (pb * x);
      out.push_back(w);
      return (int64_t)out.size() < cap;
    }
    for (int a = 0; a <= std::min(mx + 1, d - 1); ++a) {
      dig[pos] = a;
      if (!rec(pos + 1, std::max(mx, a))) return false;
    }
    return true;
  };
  dig[0] = 0;
  if (len == 1) { out.push_back(0); return; }
  rec(1, 0);
}

int64_t rgs_count(int len, int d) {
  // number of RGS strings of length len with at most d labels: sum_{j<=d} S(len, j)
  std::vector<std::vector<long double>> S(len + 1, std::vector<long double>(d + 1, 0));
  S[0][0] = 1;
  for (int i = 1; i <= len; ++i)
    for (int j = 1; j <= d; ++j) S[i][j] = j * S[i - 1][j] + S[i - 1][j - 1];
  long double t = 0;
  for (int j = 1; j <= d; ++j) t += S[len][j];
  return t > 9e18L ? INT64_MAX : (int64_t)t;
}

// shortest byte-walk suffix kept while the split still leaves ~2^21 units (LNORM_U8_SMIN: A/B hook).
// 13 (round 1: 10): the lane-pair unit init is heavier than the square instances' (34x136:
// 24.8 -> 20.8 ms, 36x144: 89.7 -> 85.7 ms, squares equal or faster; profiles/r02/ab_u8_smin.log)
int u8_min_walk() {
  static const int v = [] { const char* e = getenv("LNORM_U8_SMIN"); return (e && *e) ? atoi(e) : 13; }();
  return v;
}
constexpr double kLdInitStrategies = 500.0;   // a byte d-ary unit's init, in walked strategies (24 columns)
constexpr int kU8MinSuffix = 6;
constexpr double kU8InitWords = 8.0;
#ifndef LN_U8_SMALL_PLAN
#define LN_U8_SMALL_PLAN 1
#endif   // a byte binary unit's init, in walked words (its prefix rows summed per word)   // shortest byte-walk suffix preferred over a packed 16-bit walk

int make_plan(const Problem& pr, int world, Plan* pl, int64_t target_override = 0, bool allow_u8 = true) {
  const int f = pr.r - 1;
  const int64_t target = target_override > 0 ? target_override : kNominalLanes * 64 * std::max(1, world);
  Plan p;
  if (pr.dl == 2) {
    // kernel family first (each has its own minimal suffix length), then the split
    const int ov = kernel_override();
    auto min_s = [&](int kind) {
      for (int s_ = 1; s_ <= f; ++s_) {
        if (kind == K_PAIR16 && walk_pair16_supported(pr.mode, pr.c, s_)) return s_;
        if (kind == K_BIN16 && walk_bin16_supported(pr.mode, pr.c, s_)) return s_;
        if (kind == K_BIN && walk_bin_supported(pr.mode, pr.c, s_)) return s_;
      }
      return -1;
    };
    int kern = K_GEN, smin = 0;
    // byte-packed walk first: its guard bounds the suffix length from above, so the
    // split takes at least f - su prefix digits (units must stay below 2^32)
    if (ov < 0 && allow_u8) {
      // lane pairs (lpu 2) first where the instance offers them: their second unit per lane
      // adds a prefix row to the byte window, so fall back to one lane per unit if it no longer fits
      for (int lpu = walk_u8_lanes_per_unit(pr.mode, pr.c); lpu >= 1; --lpu) {
        const int lg = u8_lane_bits(pr, lpu);
        int su = 0;
        for (int s_ = 1; s_ <= f - lg && s_ <= 31; ++s_)
          if (u8_fits(pr, s_ + lg) && walk_u8_supported(pr.mode, pr.c, s_, lpu)) su = s_;
        int s_lo = 0;
        for (int s_ = 1; s_ <= su; ++s_) if (walk_u8_supported(pr.mode, pr.c, s_, lpu)) { s_lo = s_; break; }
        // wide entries force short suffixes, where the unit init (a prefix-row sum per unit)
        // outweighs the walk: below 6 suffix rows a packed 16-bit walk is faster whenever its
        // guard holds (42x42, entries in [-20,20]: byte walk at s = 6 3.88 s, packed 16-bit
        // 3.89 s; [-25,25] at s = 5: 6.17 s vs ~3.9 s; profiles/r02/envelope_42x42.jsonl)
        // (large searches only: below 24 rows the whole search is microseconds either way, and the
        // byte walk's guard-boundary tests run it at its shortest suffix)
        const bool short_u8 = su < kU8MinSuffix && (pr.fitsPair || pr.fits16) && f >= 24;
        if (su > 0 && s_lo > 0 && f - su <= 31 + kMaxKeyShift && !short_u8) {
          int k = std::max(lg, f - su);
          while (k < f - s_lo && k < 31 && (1LL << k) < target) ++k;
          // short suffixes spend their time in the lane init: keep s >= u8_min_walk() while the
          // split still leaves ~2^21 units (several chunks per resident warp)
          while (f - k < u8_min_walk() && k > std::max(lg, 21) && f - k < su) --k;
          if (LN_U8_SMALL_PLAN && (1LL << k) < target && target_override == 0) {
            // Small searches (below ~2^23 units: 24x24 L_2, 20-30 rows): the split above takes
            // the shortest suffix the instance allows, which can leave slightly more units than
            // one wave of resident unit slots, each paying an init for a walk of a few words.
            // Pick the prefix length minimising ceil(units / slots) * (init + walked words),
            // as the d-ary planner does (kU8InitWords: a unit's init in walked words).
            const double slots = (double)kNominalLanes / 2 * std::max(1, world) *
                                 walk_u8_units_per_lane(pr.mode, pr.c, lpu) / lpu;
            const int pr1 = pr.mode == MODE_L1 ? walk_u8_paired_rows_mode<MODE_L1>()
                          : pr.mode == MODE_MARG ? walk_u8_paired_rows_mode<MODE_MARG>() : walk_u8_paired_rows_mode<MODE_LD>();
            auto cost = [&](int kk) {
              return std::ceil(std::ldexp(1.0, kk) / slots) * (kU8InitWords + std::ldexp(1.0, f - kk - pr1));
            };
            int best_k = k;
            double best_c = cost(k);
            for (int kk = k - 1; kk >= std::max(lg, f - su); --kk) {
              const double c = cost(kk);
              if (c < best_c) { best_c = c; best_k = kk; }
            }
            k = best_k;
          }
          p.k = k; p.s = f - k; p.units = 1LL << k;
          p.kernel = K_U8;
          p.u8_lpu = lpu;
          p.key_shift = std::max(0, k - 31);
          if (const char* e = getenv("LNORM_KEY_SHIFT"))       // test hook: force coarse keys
            p.key_shift = std::max(p.key_shift, std::min(atoi(e), std::min(k, kMaxKeyShift)));
          *pl = std::move(p);
          return LNORM_OK;
        }
      }
    }
    const int sp = (pr.fitsPair && ov != K_BIN16 && ov != K_BIN && ov != K_GEN) ? min_s(K_PAIR16) : -1;
    const int sb = (pr.fits16 && ov != K_BIN && ov != K_GEN) ? min_s(K_BIN16) : -1;
    const int si = (ov != K_GEN) ? min_s(K_BIN) : -1;
    if (sp > 0) { kern = K_PAIR16; smin = sp; }
    else if (sb > 0) { kern = K_BIN16; smin = sb; }
    else if (si > 0) { kern = K_BIN; smin = si; }
    int k = 0;
    while (k < f - smin && k < 31 && (1LL << k) < target) ++k;
    // a unit's walk counts its words in 32 bits: at most 31 suffix digits (r <= 63)
    if (f - k > 31) k = std::min(31, f - 31);
    p.k = k; p.s = f - k; p.units = 1LL << k;
    p.kernel = kern;
    if (kern == K_BIN16 && !walk_bin16_table_fits(pr.mode, pr.c, p.k, p.s))
      p.kernel = walk_bin_supported(pr.mode, pr.c, p.s) ? K_BIN : K_GEN;
  } else {
    const int d = pr.dl;
    const int ov = kernel_override();
    // the fastest exact d-ary family (byte > last-row-paired 16-bit > 16-bit > int32 > generic);
    // each is checked on its own column limit (the int32 walk stops at 32 columns, the byte
    // walk at 48, the 16-bit ones at 64), LNORM_KERNEL starts the order lower
    int kern = K_GEN, smin = 0;
    if (f >= 1 && ov != K_GEN) {
      if (ov < 0 && pr.mode == MODE_LD && pr.sufW[pr.r] <= 255 && f >= 2 && walk_ldu8_supported(d, pr.c, 2)) { kern = K_LDU8; smin = 2; }
      else if (ov != K_BIN && ov != K_BIN16 && pr.fitsLdPair && f >= 2 && walk_ldpair16_supported(d, pr.c, 2)) { kern = K_LDPAIR16; smin = 2; }
      else if (ov != K_BIN && pr.fits16 && walk_ld16_supported(d, pr.c, 1)) { kern = K_LD16; smin = 1; }
      else if (walk_ld_supported(d, pr.c, 1)) { kern = K_LD; smin = 1; }
    }
    int k = 0;
    while (k < f - smin && (k + 2) * prefix_bits(d) <= 64 && rgs_count(k + 2, d) <= kTableCap && rgs_count(k + 1, d) < target) ++k;
    if (kern == K_LDU8 && target_override == 0) {
      // Small searches (L_3 below ~24 rows): the RGS table caps k, so the split above leaves
      // 2-5 suffix rows and every unit pays an init (its prefix rows summed into the byte
      // groups, the bias sums: ~kLdInitStrategies strategies' worth of work) for a walk of a
      // few hundred strategies.  Pick the prefix length minimising
      //     ceil(units / resident unit slots) * (init + d^s)
      // instead (24x24 and larger keep the split above; 20x20 L_3: s 5 -> 7).
      const double slots = (double)kNominalLanes / 2 * std::max(1, world);   // 16 warps x 32 lanes per SM
      auto cost = [&](int kk) {
        return std::ceil((double)rgs_count(kk + 1, d) / slots) * (kLdInitStrategies + std::pow((double)d, f - kk));
      };
      int best_k = k;
      double best_c = cost(k);
      for (int kk = k - 1; kk >= 0 && f - kk <= 20 && walk_ldu8_supported(d, pr.c, f - kk); --kk) {
        const double c = cost(kk);
        if (c < best_c) { best_c = c; best_k = kk; }
      }
      k = best_k;
    }
    p.k = k; p.s = f - k;
    {
      // the RGS prefix list depends only on (k, d): enumerate once per process
      static std::mutex mu;
      static std::map<std::pair<int, int>, std::shared_ptr<const std::vector<uint64_t>>> cache;
      std::shared_ptr<const std::vector<uint64_t>> tab;
      {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find({k, d});
        if (it != cache.end()) tab = it->second;
      }
      if (!tab) {
        auto v = std::make_shared<std::vector<uint64_t>>();
        rgs_enumerate(k + 1, d, *v, kTableCap + 1);
        std::lock_guard<std::mutex> g(mu);
        // a concurrent miss may have inserted the list first: keep that one (never replace
        // an entry a device context may mirror)
        tab = cache.emplace(std::make_pair(k, d), std::move(v)).first->second;
      }
      p.shared = tab;
    }
    p.units = (int64_t)p.shared->size();
    p.kernel = kern;
    // the split may leave a suffix a family cannot take: step down the order
    if (p.kernel == K_LDU8 && !walk_ldu8_supported(d, pr.c, p.s)) p.kernel = pr.fitsLdPair ? K_LDPAIR16 : K_LD16;
    if (p.kernel == K_LDPAIR16 && !walk_ldpair16_supported(d, pr.c, p.s)) p.kernel = K_LD16;
    if (p.kernel == K_LD16 && !(pr.fits16 && walk_ld16_supported(d, pr.c, p.s))) p.kernel = K_LD;
    if (p.kernel == K_LD && !walk_ld_supported(d, pr.c, p.s)) p.kernel = K_GEN;
  }
  // per-unit word count must fit 32-bit block counters
  long double words = 1;
  for (int i = 0; i < p.s; ++i) words *= pr.dl;
  if (words >= 4.0e9L || (p.units >> p.key_shift) >= (1LL << 32)) return LNORM_ETOOLARGE;
  *pl = std::move(p);
  return LNORM_OK;
}

// --------------------------------------------------------------- kernels --
// Batched launches: matrices b = blockIdx.y, blockIdx.y + gridDim.y, ... < batch.
// ctl (single searches): the search's control block is initialised here too (one launch less).
__global__ void orient_kernel(const int32_t* in, int n, int m, int transpose, int32_t* out, int batch = 1,
                              unsigned long long* ctl = nullptr) {
  if (ctl && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    ctl[0] = 0ull; ctl[1] = 0ull; ctl[2] = 0ull; ctl[3] = ~0ull; ctl[4] = 0ull; ctl[5] = 0ull;
  }
  const int64_t total = (int64_t)n * m;
  for (int b = blockIdx.y; b < batch; b += gridDim.y) {
    const int32_t* ib = in + b * total;
    int32_t* ob = out + b * total;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      if (!transpose) ob[i] = ib[i];
      else { const int64_t x = i / m, y = i % m; ob[y * n + x] = ib[i]; }
    }
  }
}

// Control block of one search (device):
//   [0] work counter (generic kernel)   [1] max reduction key   [2] error flag
//   [3] min lexicographic suffix key (recovery)   [4] max value the recovery re-walk
//   saw, biased like the key (self-check).  [5] the byte walks' dynamic chunk counter (zeroed by
//   their table-build kernel before every walk launch).  [1] and [2] are adjacent: the multi-rank
//   all-reduce(max) combines the key and the "some rank failed" flag in ONE call.
constexpr int kCtlWords = 6;
__global__ void init_ctl_kernel(unsigned long long* ctl) {
  ctl[0] = 0ull;
  ctl[1] = 0ull;
  ctl[2] = 0ull;
  ctl[3] = ~0ull;
  ctl[4] = 0ull;
  ctl[5] = 0ull;
}

// Test hook (LNORM_TEST_CORRUPT_KEY=delta): shift the reduced key's value by delta so
// that the recovery self-check must fail.
__global__ void corrupt_key_kernel(unsigned long long* key, int delta) {
  const int32_t v = key_value(*key) + delta;
  *key = make_key(v, key_unit(*key));
}

struct FinalizeArgs {
  const unsigned long long* key;   // [batch] max keys
  const unsigned long long* lex;   // [batch] smallest optimal suffix keys
  const uint64_t* table;   // full prefix table or null (binary arithmetic)
  const int32_t* Min;      // original (un-oriented) input, n x m
  int n, m, r, k, s, base, mode, transposed, pbits, key_shift;
  int64_t units;           // units per matrix (bounds the decoded winning unit)
  int64_t* value_out;      // [batch]
  int8_t* argmax_out;      // int8[batch][n]
};

// Assemble the lexicographically smallest optimum from (unit, suffix key) and
// map it back to the caller's row order (R2, R6).
__global__ void finalize_kernel(FinalizeArgs a) {
  __shared__ int8_t dig[kMaxRows];
  __shared__ int flip;
  // batched launches: blockIdx.x = matrix
  const unsigned long long key = a.key[blockIdx.x], lex = a.lex[blockIdx.x];
  a.Min += (int64_t)blockIdx.x * a.n * a.m;
  a.argmax_out += (int64_t)blockIdx.x * a.n;
  // unit = key group start + the group offset recovery found (high word of lex)
  const int64_t u = ((int64_t)key_unit(key) << a.key_shift) + (int64_t)(lex >> 32);
  if (lex == ~0ull || u < 0 || u >= a.units) {
    // the recovery found no strategy attaining the key (the host reports LNORM_EINTERNAL):
    // decode nothing
    if (threadIdx.x == 0) a.value_out[blockIdx.x] = INT64_MIN;
    for (int x = threadIdx.x; x < a.n; x += blockDim.x) a.argmax_out[x] = 0;
    return;
  }
  if (threadIdx.x == 0) {
    a.value_out[blockIdx.x] = (int64_t)key_value(key);
    for (int x = 0; x <= a.k; ++x)
      dig[x] = a.table ? (int8_t)((a.table[u] >> (a.pbits * x)) & ((1ull << a.pbits) - 1ull)) : (int8_t)(x == 0 ? 0 : (u >> (a.k - x)) & 1);
    uint64_t q = lex & 0xFFFFFFFFull;
    for (int i = 0; i < a.s; ++i) { dig[a.r - 1 - i] = (int8_t)(q % (uint64_t)a.base); q /= (uint64_t)a.base; }
  }
  __syncthreads();
  if (!a.transposed) {
    for (int x = threadIdx.x; x < a.n; x += blockDim.x)
      a.argmax_out[x] = a.mode == MODE_LD ? dig[x] : (int8_t)(dig[x] ? -1 : 1);
    return;
  }
  // searched M^T: dig is y* over the caller's columns; x_i = sgn((M y*)_i), sgn(0) = +1
  for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
    int64_t z = 0;
    for (int j = 0; j < a.m; ++j) z += (int64_t)a.Min[(int64_t)i * a.m + j] * (dig[j] ? -1 : 1);
    a.argmax_out[i] = z >= 0 ? 1 : -1;
  }
  __syncthreads();
  if (threadIdx.x == 0) flip = (a.mode == MODE_L1 && a.argmax_out[0] == -1) ? 1 : 0;
  __syncthreads();
  if (a.mode == MODE_MARG) { if (threadIdx.x == 0) a.argmax_out[0] = 1; }
  else if (flip) for (int i = threadIdx.x; i < a.n; i += blockDim.x) a.argmax_out[i] = (int8_t)-a.argmax_out[i];
}

// --------------------------------------------------------------- context --
struct DevCtx {
  int device = -1;
  std::mutex mu;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {};
  int nsm = 148;
  int32_t* dIn = nullptr; size_t capIn = 0;
  int32_t* dM = nullptr; size_t capM = 0;
  int32_t* dTab = nullptr;
  int32_t* dInit = nullptr;
  unsigned long long* dCtl = nullptr;
  uint64_t* dPre = nullptr; size_t capPre = 0;
  // the immutable process-wide RGS list dPre currently mirrors (held, so its address
  // cannot be reused by another list while this context refers to it); null = none
  std::shared_ptr<const std::vector<uint64_t>> preHold;
  long long* dStats = nullptr;      // guard_stats_kernel output (device input)
  long long* hStats = nullptr;      // pinned mirror
  unsigned long long* hCtl = nullptr;   // pinned mirror of the control block (self-check)
  cudaStream_t cur = nullptr;       // stream of the call in progress (caller's or `stream`)
  int64_t* dRes = nullptr;          // [0] value, then int8 argmax[kMaxCols]
  int64_t* dUnit = nullptr; size_t capUnit = 0;
  int32_t* dRed = nullptr; size_t capRed = 0;      // reduction scratch + reduced matrix + maps
  int64_t* dBatch = nullptr; size_t capBatch = 0;  // batched-call buffers
  long long* dBStats = nullptr; long long* hBStats = nullptr; size_t capBStats = 0;  // batched guard stats
  int64_t* hRes = nullptr;          // pinned mirror of dRes
  bool ready = false;
};

DevCtx g_ctx[64];
std::mutex g_ctx_mu;
thread_local lnorm_stats g_stats;

#define CU(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { (void)cudaGetLastError(); \
  return e_ == cudaErrorMemoryAllocation ? LNORM_ENOMEM : LNORM_ECUDA; } } while (0)

int ctx_get(int device, DevCtx** out) {
  if (device < 0 || device >= 64) return LNORM_ENODEV;
  std::lock_guard<std::mutex> g(g_ctx_mu);
  DevCtx& c = g_ctx[device];
  if (!c.ready) {
    CU(cudaSetDevice(device));
    CU(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    for (auto& e : c.ev) CU(cudaEventCreate(&e));
    CU(cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, device));
    CU(cudaMalloc(&c.dTab, sizeof(int32_t) * 32768));
    CU(cudaMalloc(&c.dInit, sizeof(int32_t) * 16384));
    CU(cudaMalloc(&c.dCtl, sizeof(unsigned long long) * kCtlWords));
    CU(cudaMalloc(&c.dRes, 8 + kMaxCols + 64));
    CU(cudaMallocHost(&c.hRes, 8 + kMaxCols + 64));
    CU(cudaMalloc(&c.dStats, sizeof(long long) * (3 + kMaxRows)));
    CU(cudaMallocHost(&c.hStats, sizeof(long long) * (3 + kMaxRows)));
    CU(cudaMallocHost(&c.hCtl, sizeof(unsigned long long) * kCtlWords));
    c.cur = c.stream;
    c.device = device;
    c.ready = true;
  }
  *out = &c;
  return LNORM_OK;
}

template <class T>
int grow(T** p, size_t* cap, size_t need) {
  if (*cap >= need) return LNORM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr; *cap = 0;
  CU(cudaMalloc(p, sizeof(T) * need));
  *cap = need;
  return LNORM_OK;
}

// Algorithm 1 verbatim: inclusive range of worker t of T over C words;
// the provisional j_max is signed (it is -1 when J = 0).
void algorithm1(uint64_t C, int64_t T, int64_t t, int64_t* j_min, int64_t* j_max) {
  const int64_t J = (int64_t)(C / (uint64_t)T), R = (int64_t)(C % (uint64_t)T);
  int64_t lo = t * J, hi = (t + 1) * J - 1;
  if (t <= R) lo += t; else lo += R;
  if (t < R) hi += t + 1; else hi += R;
  *j_min = lo;
  *j_max = hi;
}

int64_t ipow(int b, int e) { int64_t r = 1; for (int i = 0; i < e; ++i) r *= b; return r; }

struct RunOut {
  int64_t value = 0;
  std::vector<int8_t> argmax;
};

// Launch the walk over units [ub, ub+uc) of plan `pl` (params prepared by caller).
int launch_walk(DevCtx& cx, const Problem& pr, const Plan& pl, WalkParams& wp, int* grid_out, int* block_out) {
  int block = 128, occ = 0;
  if (pl.kernel == K_BIN) occ = walk_bin_occupancy(pr.mode, pr.c, &block);
  else if (pl.kernel == K_BIN16) occ = walk_bin16_occupancy(pr.mode, pr.c, pl.k, pl.s, &block);
  else if (pl.kernel == K_LD16) occ = walk_ld16_occupancy(pr.dl, pr.c, pl.k, pl.s, &block);
  else if (pl.kernel == K_PAIR16) occ = walk_pair16_occupancy(pr.mode, pr.c, pl.s, &block);
  else if (pl.kernel == K_U8) occ = walk_u8_occupancy(pr.mode, pr.c, pl.s, pl.u8_lpu, &block);
  else if (pl.kernel == K_LDPAIR16) occ = walk_ldpair16_occupancy(pr.dl, pr.c, pl.s, &block);
  else if (pl.kernel == K_LDU8) occ = walk_ldu8_occupancy(pr.dl, pr.c, pl.s, &block);
  else if (pl.kernel == K_LD) occ = walk_ld_occupancy(pr.dl, pr.c, &block);
  else occ = walk_generic_occupancy(pr.dl, pr.c, &block);
  if (occ < 1) occ = 1;
  int64_t per_block = pl.kernel == K_GEN ? block / 32 : block;   // units per block chunk
  if (pl.kernel == K_BIN16) per_block *= walk_bin16_units_per_lane(pr.mode, pr.c);
  if (pl.kernel == K_LD16) per_block *= walk_ld16_units_per_lane(pr.dl, pr.c);
  if (pl.kernel == K_PAIR16) per_block *= walk_pair16_units_per_lane(pr.mode, pr.c);
  if (pl.kernel == K_U8) per_block = per_block * walk_u8_units_per_lane(pr.mode, pr.c, pl.u8_lpu) / pl.u8_lpu;
  wp.u8_lpu = pl.u8_lpu;
  wp.u8_pack_max = pr.fitsU16 ? 1 : 0;
  if (pl.kernel == K_LDPAIR16) per_block *= walk_ldpair16_units_per_lane(pr.dl, pr.c);
  if (pl.kernel == K_LDU8) per_block *= walk_ldu8_packed(pr.dl, pr.c, pl.s) ? 2 : walk_ldu8_units_per_lane(pr.dl, pr.c, pl.s);
  int64_t want = (wp.unit_count + per_block - 1) / per_block;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)occ * cx.nsm, want));
  cudaError_t e;
  cudaStream_t st = cx.cur ? cx.cur : cx.stream;
  if (pl.kernel == K_BIN) e = walk_bin_launch(wp, cx.dTab, grid, st, &block);
  else if (pl.kernel == K_BIN16) e = walk_bin16_launch(wp, cx.dTab, grid, st, &block);
  else if (pl.kernel == K_LD16) e = walk_ld16_launch(wp, cx.dTab, grid, st, &block);
  else if (pl.kernel == K_PAIR16) e = walk_pair16_launch(wp, cx.dTab, cx.dInit, grid, st, &block);
  else if (pl.kernel == K_U8) e = walk_u8_launch(wp, cx.dTab, cx.dInit, grid, st, &block);
  else if (pl.kernel == K_LDPAIR16) e = walk_ldpair16_launch(wp, cx.dTab, cx.dInit, grid, st, &block);
  else if (pl.kernel == K_LDU8) e = walk_ldu8_launch(wp, cx.dTab, cx.dInit, grid, st, &block);
  else if (pl.kernel == K_LD) e = walk_ld_launch(wp, cx.dTab, grid, st, &block);
  else e = walk_generic_launch(wp, grid, st, &block);
  if (e != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  *grid_out = grid; *block_out = block;
  return LNORM_OK;
}

// Full search on one device.  dIn: device copy of the caller's n x m matrix.
// world > 1: this rank walks its Algorithm-1 slice and `comm` all-reduces the key.
// Checkpointed single-device search: the unit list is walked in chunks of
// `chunk_units`; after every chunk (units done, best key) is written atomically
// to `path` (tmp + rename) together with a fingerprint of the problem and plan,
// so an interrupted run resumes exactly where it stopped.
struct Checkpoint {
  const char* path = nullptr;
  int64_t chunk_units = 0;
  int32_t max_chunks = 0;        // chunks to walk in this call (<= 0: all)
  int32_t* done = nullptr;       // out: 1 when the search finished (value/argmax valid)
  int64_t* units_done = nullptr; // out
};

uint64_t fnv1a(uint64_t h, const void* p, size_t n) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ull; }
  return h;
}

struct CkState { uint64_t magic, fingerprint; int64_t next_unit; unsigned long long key; };

bool ck_load(const char* path, uint64_t fp, CkState* st) {
  FILE* f = fopen(path, "rb");
  if (!f) return false;
  CkState t{};
  const bool ok = fread(&t, sizeof(t), 1, f) == 1;
  fclose(f);
  if (!ok || t.magic != 0x4c4e4f524d434b31ull || t.fingerprint != fp) return false;
  *st = t;
  return true;
}

bool ck_save(const char* path, const CkState& st) {
  std::string tmp = std::string(path) + ".tmp";
  FILE* f = fopen(tmp.c_str(), "wb");
  if (!f) return false;
  const bool ok = fwrite(&st, sizeof(st), 1, f) == 1;
  fclose(f);
  return ok && rename(tmp.c_str(), path) == 0;
}

// Recovery self-check: the re-walk of the winning unit
// must reproduce the reduced maximum exactly -- some strategy of the unit attains
// key_value(key) (lex found) and none exceeds it (rmax == key value).  Any mismatch
// means the hot walk or the reduction is wrong: LNORM_EINTERNAL, never a silent answer.
bool recovery_consistent(unsigned long long key, unsigned long long lex, unsigned long long rmax) {
  return key != 0ull && lex != ~0ull && (uint32_t)(rmax & 0xFFFFFFFFull) == (uint32_t)(key >> 32);
}

int corrupt_key_delta() {
  const char* e = getenv("LNORM_TEST_CORRUPT_KEY");
  return (e && *e) ? atoi(e) : 0;
}

// vslices > 1 (test hook, world == 1): walk the Algorithm-1 slices of `vslices`
// virtual ranks one after the other on this device; the shared key then holds
// exactly what the multi-rank all-reduce(max) would.
// comm != null: this rank walks its Algorithm-1 slice of `world` and ONE
// ncclAllReduce(max) over {key, error flag} combines the ranks (also at world == 1).
int run_device(DevCtx& cx, const int32_t* dIn, const Problem& pr, int rank, int world, ncclComm_t comm,
               RunOut* out, lnorm_stats* st, int vslices = 1, const Checkpoint* ck = nullptr,
               const int32_t* hostM = nullptr) {
  Plan pl;
  // the plan depends only on (M, world): identical on every rank, so a planning error
  // is raised by all ranks alike before any of them reaches the collective
  int rc;
  {
    NvtxRange nr("lnorm.plan");
    rc = make_plan(pr, std::max(world, vslices), &pl);
  }
  if (rc) return rc;
  cudaStream_t s = cx.cur ? cx.cur : cx.stream;
  const bool collective = comm != nullptr;
  const std::vector<uint64_t>& ptab = pl.prefixes();
  int grid = 0, block = 0, launches = 0;
  int64_t cnt = pl.units, walked = 0;
  WalkParams wp{};
  // ---- everything up to the collective: on error the rank still joins the all-reduce
  //      with its error flag raised, so its peers return instead of hanging
  auto pre = [&]() -> int {
    int e;
    if ((e = grow(&cx.dM, &cx.capM, (size_t)pr.n * pr.m))) return e;
    const bool mirror = !ptab.empty() && pl.shared && cx.preHold.get() == pl.shared.get();
    if (!ptab.empty() && !mirror) {
      cx.preHold.reset();
      if ((e = grow(&cx.dPre, &cx.capPre, ptab.size()))) return e;
    }
    CU(cudaEventRecord(cx.ev[0], s));
    // orientation + control-block init in one launch (init_ctl_kernel's job folded in)
    orient_kernel<<<std::min(1024, (pr.n * pr.m + 255) / 256), 256, 0, s>>>(dIn, pr.n, pr.m, pr.transposed ? 1 : 0, cx.dM,
                                                                             1, cx.dCtl);
    ++launches;
    CU(cudaGetLastError());
    if (!ptab.empty() && !mirror) {
      // the RGS list for (k, d) is immutable and lives for the process: upload it once per device
      CU(cudaMemcpyAsync(cx.dPre, ptab.data(), sizeof(uint64_t) * ptab.size(), cudaMemcpyHostToDevice, s));
      if (pl.shared) cx.preHold = pl.shared;
    }
    wp.M = cx.dM; wp.r = pr.r; wp.c = pr.c; wp.mode = pr.mode; wp.d = pr.dl; wp.k = pl.k; wp.s = pl.s;
    wp.pbits = prefix_bits(pr.dl);
    wp.key_shift = pl.key_shift;
    wp.counter = cx.dCtl; wp.key = cx.dCtl + 1; wp.unit_max = nullptr; wp.chunk_ctr = cx.dCtl + 5;
#if LN_SELFCHECK
    if (const char* e = getenv("LNORM_SELFCHECK_INJECT")) wp.selfcheck_delta = atoi(e);
#endif
    CU(cudaEventRecord(cx.ev[1], s));
    if (ck && ck->path && world == 1 && vslices <= 1 && !collective) {
      // ---- checkpointed walk: chunks of the unit list, state persisted after each
      uint64_t fp = 1469598103934665603ull;
      const int32_t hdr[8] = {pr.n, pr.m, pr.d, pr.marg, pl.k, pl.s, pl.kernel, (int32_t)pr.transposed};
      fp = fnv1a(fp, hdr, sizeof(hdr));
      if (hostM) fp = fnv1a(fp, hostM, sizeof(int32_t) * (size_t)pr.n * pr.m);
      CkState cs{0x4c4e4f524d434b31ull, fp, 0, 0ull};
      ck_load(ck->path, fp, &cs);
      if (cs.key) CU(cudaMemcpyAsync(cx.dCtl + 1, &cs.key, sizeof(cs.key), cudaMemcpyHostToDevice, s));
      const int64_t chunk = ck->chunk_units > 0 ? ck->chunk_units : pl.units;
      int32_t chunks = 0;
      while (cs.next_unit < pl.units && (ck->max_chunks <= 0 || chunks < ck->max_chunks)) {
        const int64_t c0 = cs.next_unit, c1 = std::min<int64_t>(pl.units, c0 + chunk);
        wp.unit_begin = c0; wp.unit_count = c1 - c0;
        walk_params_single(wp);
        wp.prefix_table = ptab.empty() ? nullptr : cx.dPre + c0;
        if (pl.kernel == K_GEN) CU(cudaMemsetAsync(cx.dCtl, 0, sizeof(unsigned long long), s));
        if ((e = launch_walk(cx, pr, pl, wp, &grid, &block))) return e;
        launches += pl.kernel == K_GEN ? 1 : 2;
        walked += c1 - c0;
        CU(cudaMemcpyAsync(&cs.key, cx.dCtl + 1, sizeof(cs.key), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        cs.next_unit = c1;
        if (!ck_save(ck->path, cs)) return LNORM_EINVAL;
        ++chunks;
      }
      if (ck->units_done) *ck->units_done = cs.next_unit;
      if (cs.next_unit < pl.units) {               // partial: report the best so far, no recovery yet
        if (ck->done) *ck->done = 0;
        out->value = cs.key ? (int64_t)key_value(cs.key) : INT64_MIN;
        out->argmax.assign(pr.n, 0);
        lnorm_stats S{};
        S.rows = pr.r; S.cols = pr.c; S.units = walked; S.units_total = pl.units; S.launches = launches;
        S.variant = pl.kernel;
        *st = S;
        return -1;                                 // (not an error: partial result, no recovery)
      }
      if (ck->done) *ck->done = 1;
      return LNORM_OK;
    }
    const int nslices = collective ? 1 : std::max(1, vslices);
    int64_t lo = 0;
    for (int sl = 0; sl < nslices; ++sl) {
      const int T = collective ? world : nslices, t = collective ? rank : sl;
      if (T > 1) {
        int64_t jmin = 0, jmax = -1;
        algorithm1((uint64_t)pl.units, T, t, &jmin, &jmax);
        lo = jmin;
        cnt = jmax - jmin + 1;
      }
      wp.unit_begin = lo; wp.unit_count = cnt;
      walk_params_single(wp);
      wp.prefix_table = ptab.empty() ? nullptr : cx.dPre + lo;
      if (cnt > 0) {
        if (sl > 0 && pl.kernel == K_GEN) {   // the generic kernel's work counter restarts per slice
          CU(cudaMemsetAsync(cx.dCtl, 0, sizeof(unsigned long long), s));
        }
        if ((e = launch_walk(cx, pr, pl, wp, &grid, &block))) return e;
        launches += pl.kernel == K_GEN ? 1 : 2;   // table build + walk
        walked += cnt;
      }
    }
    return LNORM_OK;
  };
  int pre_rc;
  {
    NvtxRange nr("lnorm.walk");
    pre_rc = pre();
  }
  if (pre_rc == -1) return LNORM_OK;           // checkpoint: partial result already written
  cnt = walked;
  if (pre_rc != LNORM_OK) {
    if (!collective) return pre_rc;
    (void)cudaGetLastError();
    (void)cudaMemsetAsync(cx.dCtl + 2, 0xFF, sizeof(unsigned long long), s);   // raise the error flag
  }
  (void)cudaEventRecord(cx.ev[2], s);
  if (collective) {
    NvtxRange nr("lnorm.allreduce");
    Nccl& nc = nccl();
    if (!nc.ok) return LNORM_ENCCL;
    if (nc.AllReduce(cx.dCtl + 1, cx.dCtl + 1, 2, ncclUint64, ncclMax, comm, s) != ncclSuccess) return LNORM_ENCCL;
    ++launches;
    if (pre_rc != LNORM_OK) { (void)cudaStreamSynchronize(s); return pre_rc; }
  }
  if (const int delta = corrupt_key_delta()) {
    corrupt_key_kernel<<<1, 1, 0, s>>>(cx.dCtl + 1, delta);
    CU(cudaGetLastError());
    ++launches;
  }
  // recovery over the full unit space (same winning unit on every rank)
  NvtxRange nr_rec("lnorm.recover+sync");
  WalkParams rp = wp;
  rp.unit_begin = 0; rp.unit_count = pl.units;
  walk_params_single(rp);
  rp.prefix_table = ptab.empty() ? nullptr : cx.dPre;
  if (recover_launch(rp, cx.dCtl + 3, cx.dCtl + 4, s) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  ++launches;
  FinalizeArgs fa;
  fa.key = cx.dCtl + 1; fa.lex = cx.dCtl + 3; fa.table = rp.prefix_table; fa.Min = dIn; fa.n = pr.n; fa.m = pr.m; fa.r = pr.r;
  fa.k = pl.k; fa.s = pl.s; fa.base = pr.dl; fa.mode = pr.mode; fa.transposed = pr.transposed ? 1 : 0; fa.pbits = prefix_bits(pr.dl);
  fa.key_shift = pl.key_shift;
  fa.units = pl.units;
  fa.value_out = cx.dRes; fa.argmax_out = reinterpret_cast<int8_t*>(cx.dRes + 1);
  finalize_kernel<<<1, 256, 0, s>>>(fa);
  ++launches;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(cx.hRes, cx.dRes, 8 + pr.n, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(cx.hCtl, cx.dCtl, sizeof(unsigned long long) * kCtlWords, cudaMemcpyDeviceToHost, s));
  CU(cudaEventRecord(cx.ev[3], s));
  CU(cudaStreamSynchronize(s));
  if (cx.hCtl[2]) return LNORM_ENCCL;                 // a peer rank failed before the collective
#if LN_SELFCHECK
  if (pl.kernel == K_U8 && cx.hCtl[0]) return LNORM_EINTERNAL;   // a step's value differed from scratch
#endif
  if (!recovery_consistent(cx.hCtl[1], cx.hCtl[3], cx.hCtl[4])) return LNORM_EINTERNAL;
  out->value = cx.hRes[0];
  out->argmax.assign(reinterpret_cast<int8_t*>(cx.hRes + 1), reinterpret_cast<int8_t*>(cx.hRes + 1) + pr.n);
  float wms = 0, tms = 0;
  cudaEventElapsedTime(&wms, cx.ev[1], cx.ev[2]);
  cudaEventElapsedTime(&tms, cx.ev[0], cx.ev[3]);
  lnorm_stats S{};
  S.rows = pr.r; S.cols = pr.c; S.transposed = pr.transposed; S.prefix_digits = pl.k; S.suffix_digits = pl.s;
  S.d = pr.d == 1 ? 1 : pr.dl; S.units = cnt; S.units_total = pl.units;
  S.steps = (double)cnt * (double)ipow(pr.dl, pl.s);
  S.column_updates = S.steps * pr.c * (pr.mode == MODE_LD && pr.dl >= 3 ? 2 : 1);
  S.walk_ms = wms; S.total_ms = tms; S.launches = launches; S.variant = pl.kernel;
  S.block_threads = block; S.grid_blocks = grid;
  S.paired_rows = pl.kernel == K_LDU8 ? walk_ldu8_paired_rows(pr.dl, pl.s) : (pl.kernel == K_U8 ? 1 : 0);
  S.packed_units = pl.kernel == K_LDU8 && walk_ldu8_packed(pr.dl, pr.c, pl.s) ? 2 : 0;
  *st = S;
  return LNORM_OK;
}

int current_device(int* dev) {
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt < 1) { (void)cudaGetLastError(); return LNORM_ENODEV; }
  if (cudaGetDevice(dev) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ENODEV; }
  return LNORM_OK;
}

void write_out(const RunOut& ro, int64_t* value, int8_t* argmax) {
  *value = ro.value;
  if (argmax) std::memcpy(argmax, ro.argmax.data(), ro.argmax.size());
}

// Restores the context's default stream when a call that borrowed the caller's ends.
struct StreamScope {
  DevCtx* c;
  StreamScope(DevCtx* cx, cudaStream_t user) : c(cx) { c->cur = user ? user : c->stream; }
  ~StreamScope() { c->cur = c->stream; }
};

// Guard statistics of a device-resident matrix: one-block kernel on the call's stream,
// ~0.5 KB copied back (the plan depends on them: the only host round trip before the walk).
int device_stats(DevCtx& cx, const int32_t* devM, Problem* pr) {
  NvtxRange nr("lnorm.guard_stats");
  cudaStream_t s = cx.cur;
  guard_stats_kernel<<<1, 256, 0, s>>>(devM, pr->m, pr->transposed ? 1 : 0, pr->r, pr->c,
                                       pr->mode == MODE_MARG ? 1 : 0, cx.dStats);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(cx.hStats, cx.dStats, sizeof(long long) * (3 + pr->r), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  GuardStats g;
  g.S = cx.hStats[0]; g.par[0] = cx.hStats[1]; g.par[1] = cx.hStats[2];
  for (int q = 1; q <= pr->r; ++q) g.sufW[q] = cx.hStats[3 + q - 1];
  return apply_stats(g, pr);
}

int compute_on(int device, const int32_t* hostM, const int32_t* devM, int n, int m, int d, int marg,
               int rank, int world, ncclComm_t comm, cudaStream_t user_stream, int64_t* value, int8_t* argmax,
               int vslices = 1) {
  if (!value || (!hostM && !devM)) return LNORM_EINVAL;
  NvtxRange nr("lnorm.compute");
  Problem pr;
  DevCtx* cx = nullptr;
  int rc = ctx_get(device, &cx);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(cx->mu);
  CU(cudaSetDevice(device));
  StreamScope scope(cx, user_stream);
  const int32_t* dIn = devM;
  if (devM) {
    if ((rc = validate_shape(n, m, d, marg, &pr))) return rc;
    if ((rc = device_stats(*cx, devM, &pr))) return rc;
  } else {
    if ((rc = validate(hostM, n, m, d, marg, &pr))) return rc;
    if ((rc = grow(&cx->dIn, &cx->capIn, (size_t)n * m))) return rc;
    CU(cudaMemcpyAsync(cx->dIn, hostM, sizeof(int32_t) * n * m, cudaMemcpyHostToDevice, cx->cur));
    dIn = cx->dIn;
  }
  RunOut ro;
  lnorm_stats st{};
  if ((rc = run_device(*cx, dIn, pr, rank, world, comm, &ro, &st, vslices))) return rc;
  g_stats = st;
  write_out(ro, value, argmax);
  return LNORM_OK;
}

// Rank entry points: the communicator (if any) must span `world` ranks with this
// process at `rank`.
int check_comm(ncclComm_t comm, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) return LNORM_EINVAL;
  if (!comm) return world == 1 ? LNORM_OK : LNORM_EINVAL;
  Nccl& nc = nccl();
  if (!nc.ok) return LNORM_ENCCL;
  int cnt = 0, me = -1;
  if (nc.CommCount(comm, &cnt) != ncclSuccess || nc.CommUserRank(comm, &me) != ncclSuccess) return LNORM_ENCCL;
  return (cnt == world && me == rank) ? LNORM_OK : LNORM_EINVAL;
}

}  // namespace

struct lnorm_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
};

extern "C" {

const char* lnorm_status_string(int status) {
  switch (status) {
    case LNORM_OK: return "ok";
    case LNORM_EINVAL: return "invalid argument";
    case LNORM_EOVERFLOW: return "sum |M_ij| exceeds 2^31-1 (int32 exactness bound)";
    case LNORM_ETOOLARGE: return "search space or shape exceeds the supported limits";
    case LNORM_ENODEV: return "no CUDA device";
    case LNORM_ECUDA: return "CUDA runtime error";
    case LNORM_ENCCL: return "NCCL unavailable or failed";
    case LNORM_ENOMEM: return "out of device memory";
    case LNORM_EINTERNAL: return "internal self-check failed (argmax recovery did not reproduce the reduced maximum)";
    default: return "unknown status";
  }
}

// 2.0: caller-owned NCCL comm + stream in lnorm_compute_rank, EINTERNAL; 2.1: lnorm_imma_l1,
// lnorm_plan_info.words (the former reserved field)
int32_t lnorm_version(void) { return (2 << 16) | 1; }

int lnorm_compute(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                  int64_t* value, int8_t* argmax) {
  if (!M) return LNORM_EINVAL;
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  return compute_on(dev, M, nullptr, n, m, d, with_marginals, 0, 1, nullptr, nullptr, value, argmax);
}

int lnorm_compute_device(const int32_t* M_device, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                         void* cuda_stream, int64_t* value, int8_t* argmax) {
  if (!M_device) return LNORM_EINVAL;
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  return compute_on(dev, nullptr, M_device, n, m, d, with_marginals, 0, 1, nullptr,
                    static_cast<cudaStream_t>(cuda_stream), value, argmax);
}

int lnorm_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) return LNORM_EINVAL;
  Nccl& nc = nccl();
  if (!nc.ok) return LNORM_ENCCL;
  ncclUniqueId id;
  if (nc.GetUniqueId(&id) != ncclSuccess) return LNORM_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id_out, &id, 128);
  return LNORM_OK;
}

int lnorm_comm_create(const uint8_t id[128], int32_t rank, int32_t world, int32_t device, lnorm_comm** comm_out) {
  if (!comm_out || world < 1 || rank < 0 || rank >= world || device < 0) return LNORM_EINVAL;
  if (!id && world > 1) return LNORM_EINVAL;
  lnorm_comm* c = new lnorm_comm;
  c->rank = rank; c->world = world; c->device = device;
  if (id) {   // a real communicator for every world >= 1 (world 1 exercises the all-reduce path)
    Nccl& nc = nccl();
    if (!nc.ok) { delete c; return LNORM_ENCCL; }
    if (cudaSetDevice(device) != cudaSuccess) { (void)cudaGetLastError(); delete c; return LNORM_ENODEV; }
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    if (nc.CommInitRank(&c->comm, world, uid, rank) != ncclSuccess) { delete c; return LNORM_ENCCL; }
  }
  *comm_out = c;
  return LNORM_OK;
}

int lnorm_comm_nccl(lnorm_comm* comm, void** nccl_comm_out) {
  if (!comm || !nccl_comm_out) return LNORM_EINVAL;
  *nccl_comm_out = static_cast<void*>(comm->comm);
  return LNORM_OK;
}

int lnorm_comm_destroy(lnorm_comm* comm) {
  if (!comm) return LNORM_EINVAL;
  if (comm->comm) { Nccl& nc = nccl(); if (nc.ok) nc.CommDestroy(comm->comm); }
  delete comm;
  return LNORM_OK;
}

int lnorm_compute_rank(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                       void* nccl_comm, int32_t rank, int32_t world, void* cuda_stream,
                       int64_t* value, int8_t* argmax) {
  if (!M) return LNORM_EINVAL;
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int rc = check_comm(comm, rank, world);
  if (rc) return rc;
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  return compute_on(dev, M, nullptr, n, m, d, with_marginals, rank, world, comm,
                    static_cast<cudaStream_t>(cuda_stream), value, argmax);
}

int lnorm_compute_rank_device(const int32_t* M_device, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                              void* nccl_comm, int32_t rank, int32_t world, void* cuda_stream,
                              int64_t* value, int8_t* argmax) {
  if (!M_device) return LNORM_EINVAL;
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int rc = check_comm(comm, rank, world);
  if (rc) return rc;
  int dev = 0;
  if ((rc = current_device(&dev))) return rc;
  return compute_on(dev, nullptr, M_device, n, m, d, with_marginals, rank, world, comm,
                    static_cast<cudaStream_t>(cuda_stream), value, argmax);
}

int lnorm_compute_multi(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                        int32_t num_devices, const int32_t* device_ids, int64_t* value, int8_t* argmax) {
  if (!M || !value || num_devices < 1 || num_devices > 64) return LNORM_EINVAL;
  std::vector<int> devs(num_devices);
  for (int i = 0; i < num_devices; ++i) devs[i] = device_ids ? device_ids[i] : i;
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ENODEV; }
  for (int dv : devs) if (dv < 0 || dv >= cnt) return LNORM_ENODEV;
  {   // argument / shape / overflow errors are the same on every device: report them before any comm
    Problem pr;
    const int rc = validate(M, n, m, d, with_marginals, &pr);
    if (rc) return rc;
  }
  Nccl& nc = nccl();
  if (!nc.ok) return LNORM_ENCCL;
  // one communicator per device (also for a single device: the all-reduce path always runs)
  std::vector<ncclComm_t> comms(num_devices);
  if (nc.CommInitAll(comms.data(), num_devices, devs.data()) != ncclSuccess) return LNORM_ENCCL;
  std::vector<int> rcs(num_devices, 0);
  std::vector<int64_t> vals(num_devices, 0);
  std::vector<std::vector<int8_t>> args(num_devices, std::vector<int8_t>(n, 0));
  std::vector<lnorm_stats> sts(num_devices);
  std::atomic<int> finished{0}, failed{0};
  std::vector<std::thread> th;
  for (int g = 0; g < num_devices; ++g) {
    th.emplace_back([&, g] {
      rcs[g] = compute_on(devs[g], M, nullptr, n, m, d, with_marginals, g, num_devices, comms[g], nullptr, &vals[g],
                          args[g].data());
      sts[g] = g_stats;
      if (rcs[g]) failed.fetch_add(1);
      finished.fetch_add(1);
    });
  }
  // A device that fails before reaching the collective (context or allocation failure)
  // would leave its peers blocked in the all-reduce: once any device has failed and the
  // others make no progress for 2 s, abort every communicator (unblocks them with an error).
  bool aborted = false;
  auto t_fail = std::chrono::steady_clock::time_point{};
  while (finished.load() < num_devices) {
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
    if (!aborted && failed.load() > 0) {
      const auto now = std::chrono::steady_clock::now();
      if (t_fail == std::chrono::steady_clock::time_point{}) t_fail = now;
      else if (now - t_fail > std::chrono::seconds(2)) {
        for (auto& cm : comms) nc.CommAbort(cm);
        aborted = true;
      }
    }
  }
  for (auto& t : th) t.join();
  if (!aborted) for (auto& cm : comms) nc.CommDestroy(cm);
  for (int g = 0; g < num_devices; ++g) if (rcs[g]) return rcs[g];
  for (int g = 1; g < num_devices; ++g)
    if (vals[g] != vals[0] || args[g] != args[0]) return LNORM_EINTERNAL;   // ranks must agree bit-for-bit
  *value = vals[0];
  if (argmax) std::memcpy(argmax, args[0].data(), n);
  lnorm_stats S = sts[0];
  for (int g = 1; g < num_devices; ++g) {
    S.units += sts[g].units; S.steps += sts[g].steps; S.column_updates += sts[g].column_updates;
    S.walk_ms = std::max(S.walk_ms, sts[g].walk_ms); S.total_ms = std::max(S.total_ms, sts[g].total_ms);
    S.launches += sts[g].launches;
  }
  g_stats = S;
  return LNORM_OK;
}

int lnorm_compute_reduced(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                          int64_t* value, int8_t* argmax, int32_t* reduced_shape) {
  if (!M || !value) return LNORM_EINVAL;
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  Problem pr0;
  if ((rc = validate(M, n, m, d, with_marginals, &pr0))) return rc;
  DevCtx* cx = nullptr;
  if ((rc = ctx_get(dev, &cx))) return rc;
  std::lock_guard<std::mutex> g(cx->mu);
  CU(cudaSetDevice(dev));
  cudaStream_t s = cx->stream;
  const size_t nm = (size_t)n * m;
  const size_t need = reduce_scratch_ints(n, m) + nm + (size_t)n + 8 + (size_t)n;   // scratch, R, rowsel, info, argr/out
  if ((rc = grow(&cx->dRed, &cx->capRed, need))) return rc;
  if ((rc = grow(&cx->dIn, &cx->capIn, nm))) return rc;
  int32_t* scratch = cx->dRed;
  int32_t* R = scratch + reduce_scratch_ints(n, m);
  int32_t* rowsel = R + nm;
  int32_t* info = rowsel + n;
  int8_t* bytes = reinterpret_cast<int8_t*>(info + 8);        // argr (n) then out (n)
  CU(cudaMemcpyAsync(cx->dIn, M, sizeof(int32_t) * nm, cudaMemcpyHostToDevice, s));
  const int mode = with_marginals ? MODE_MARG : (d == 1 ? MODE_L1 : MODE_LD);
  if (reduce_launch(cx->dIn, n, m, mode, scratch, R, rowsel, info, s) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  int32_t hinfo[3] = {0, 0, 0};                              // reduced rows, columns, mode (reduce_kernel)
  CU(cudaMemcpyAsync(hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  const int nr = hinfo[0], mr = hinfo[1], mode2 = hinfo[2];
  if (reduced_shape) { reduced_shape[0] = nr; reduced_shape[1] = mr; }
  RunOut ro;
  lnorm_stats st{};
  if (nr > 0 && mr > 0) {
    std::vector<int32_t> hR((size_t)nr * mr);
    CU(cudaMemcpyAsync(hR.data(), R, sizeof(int32_t) * hR.size(), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    Problem pr;
    const int marg2 = mode2 == MODE_MARG ? 1 : 0;
    if ((rc = validate(hR.data(), nr, mr, d, marg2, &pr))) return rc;
    if ((rc = run_device(*cx, R, pr, 0, 1, nullptr, &ro, &st))) return rc;
    CU(cudaMemcpyAsync(bytes, ro.argmax.data(), (size_t)nr, cudaMemcpyHostToDevice, s));
  } else {
    ro.value = 0;   // everything reduced away: the zero matrix (norm 0)
  }
  if (mapback_launch(n, m, nr > 0 && mr > 0 ? nr : 0, mode == MODE_LD ? 1 : 0, scratch, rowsel, bytes, bytes + n,
                     info, s) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  std::vector<int8_t> out((size_t)n);
  CU(cudaMemcpyAsync(out.data(), bytes + n, (size_t)n, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  st.launches += 3;
  g_stats = st;
  *value = ro.value;
  if (argmax) std::memcpy(argmax, out.data(), (size_t)n);
  return LNORM_OK;
}

int lnorm_compute_checkpointed(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                               const char* path, int64_t chunk_units, int32_t max_chunks, int64_t* value,
                               int8_t* argmax, int32_t* done, int64_t* units_done) {
  if (!M || !value || !path || !done) return LNORM_EINVAL;
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  Problem pr;
  if ((rc = validate(M, n, m, d, with_marginals, &pr))) return rc;
  DevCtx* cx = nullptr;
  if ((rc = ctx_get(dev, &cx))) return rc;
  std::lock_guard<std::mutex> g(cx->mu);
  CU(cudaSetDevice(dev));
  if ((rc = grow(&cx->dIn, &cx->capIn, (size_t)n * m))) return rc;
  CU(cudaMemcpyAsync(cx->dIn, M, sizeof(int32_t) * n * m, cudaMemcpyHostToDevice, cx->stream));
  Checkpoint ck;
  ck.path = path; ck.chunk_units = chunk_units; ck.max_chunks = max_chunks; ck.done = done; ck.units_done = units_done;
  RunOut ro;
  lnorm_stats st{};
  if ((rc = run_device(*cx, cx->dIn, pr, 0, 1, nullptr, &ro, &st, 1, &ck, M))) return rc;
  g_stats = st;
  *value = ro.value;
  if (argmax && *done) std::memcpy(argmax, ro.argmax.data(), (size_t)n);
  return LNORM_OK;
}

int lnorm_compute_batch(const int32_t* M, int32_t batch, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                        int64_t* values, int8_t* argmax) {
  if (!M || !values || batch < 1) return LNORM_EINVAL;
  NvtxRange nr("lnorm.compute_batch");
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  const size_t nm = (size_t)n * m;
  Problem pr;
  if ((rc = validate_shape(n, m, d, with_marginals, &pr))) return rc;
  DevCtx* cx = nullptr;
  if ((rc = ctx_get(dev, &cx))) return rc;
  std::lock_guard<std::mutex> g(cx->mu);
  CU(cudaSetDevice(dev));
  cudaStream_t s = cx->stream;
  StreamScope scope(cx, nullptr);
  // every matrix to the device, then its guard statistics there (one block per matrix; the
  // host loop over thousands of matrices cost more than the whole batched walk)
  const int sw_ = 3 + pr.r;
  if ((rc = grow(&cx->dIn, &cx->capIn, (size_t)batch * nm))) return rc;
  if (cx->capBStats < (size_t)batch * sw_) {
    cudaFree(cx->dBStats); cudaFreeHost(cx->hBStats);
    cx->dBStats = nullptr; cx->hBStats = nullptr; cx->capBStats = 0;
    CU(cudaMalloc(&cx->dBStats, sizeof(long long) * (size_t)batch * sw_));
    CU(cudaMallocHost(&cx->hBStats, sizeof(long long) * (size_t)batch * sw_));
    cx->capBStats = (size_t)batch * sw_;
  }
  CU(cudaEventRecord(cx->ev[0], s));
  CU(cudaMemcpyAsync(cx->dIn, M, sizeof(int32_t) * batch * nm, cudaMemcpyHostToDevice, s));
  guard_stats_kernel<<<batch, 256, 0, s>>>(cx->dIn, m, pr.transposed ? 1 : 0, pr.r, pr.c, pr.mode == MODE_MARG ? 1 : 0,
                                           cx->dBStats, (int64_t)nm, sw_);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(cx->hBStats, cx->dBStats, sizeof(long long) * (size_t)batch * sw_, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  // the batched plan must be exact for every matrix, so it is made for the element-wise worst
  // case of their guard statistics (same shape, orientation and mode): sufW = max over the
  // batch, the 16-bit guards = AND over the batch; a matrix with sum |M| > 2^31-1 fails the call
  auto stats_of = [&](int b, Problem* q) {
    const long long* h = cx->hBStats + (size_t)b * sw_;
    GuardStats gs;
    gs.S = h[0]; gs.par[0] = h[1]; gs.par[1] = h[2];
    for (int x = 1; x <= pr.r; ++x) gs.sufW[x] = h[3 + x - 1];
    *q = pr;
    return apply_stats(gs, q);
  };
  {
    Problem all = pr;
    for (int b = 0; b < batch; ++b) {
      Problem q;
      if ((rc = stats_of(b, &q))) return rc;
      if (b == 0) { all = q; continue; }
      all.fits16 = all.fits16 && q.fits16;
      all.fitsPair = all.fitsPair && q.fitsPair;
      all.fitsLdPair = all.fitsLdPair && q.fitsLdPair;
      for (int i = 0; i <= kMaxRows; ++i) all.sufW[i] = std::max(all.sufW[i], q.sufW[i]);
    }
    pr = all;
  }
  // path: one launch over the units of all matrices through the byte-packed walks (L_1,
  // L_marg, L_2: walk_u8; L_3, L_4: walk_ldu8 / walk_ldu8w) or the strategy-paired 16-bit
  // walk, each restaging its per-matrix tables per chunk; else the generic warp-per-unit
  // kernel batched the same way for small search spaces (tiny shapes, any d); else one
  // search per matrix through the hot single-matrix kernels (inputs already on the device)
  Plan pl;
  const int64_t target = std::max<int64_t>(1, kNominalLanes * 8 / batch);
  int bkern = -1;
  // batched byte instances exist for the small-matrix regime: <= 32 columns with one lane per
  // unit (binary), <= 24 columns (d-ary); wider batches take the 16-bit paired walk
  auto batchable = [&](const Plan& q) {
    if (q.key_shift != 0) return false;
    if (q.kernel == K_U8) return pr.c <= 32 && q.u8_lpu == 1;
    if (q.kernel == K_LDU8) return pr.c <= 24;
    return q.kernel == K_PAIR16;
  };
  if (make_plan(pr, 1, &pl, target) == LNORM_OK && batchable(pl)) bkern = pl.kernel;
  else if (pr.dl == 2 && make_plan(pr, 1, &pl, target, /*allow_u8=*/false) == LNORM_OK && batchable(pl)) bkern = pl.kernel;
  long double space = 1;
  for (int i = 0; i < pr.r - 1; ++i) space *= pr.dl;
  if (bkern < 0 && space > (long double)(1 << 20)) {
    for (int b = 0; b < batch; ++b) {
      Problem q;
      if ((rc = stats_of(b, &q))) return rc;
      RunOut ro;
      lnorm_stats st{};
      if ((rc = run_device(*cx, cx->dIn + (size_t)b * nm, q, 0, 1, nullptr, &ro, &st))) return rc;
      g_stats = st;
      values[b] = ro.value;
      if (argmax) std::memcpy(argmax + (size_t)b * n, ro.argmax.data(), (size_t)n);
    }
    return LNORM_OK;
  }
  if (bkern < 0) {
    // generic batched plan: the smallest prefix length giving ~64 warps of work per SM
    pl = Plan{};
    pl.kernel = K_GEN;
    const int f = pr.r - 1;
    auto units_of = [&](int k) -> int64_t { return pr.dl == 2 ? (1LL << k) : rgs_count(k + 1, pr.dl); };
    int k = 0;
    while (k < f && (int64_t)batch * units_of(k) < (int64_t)cx->nsm * 64 && units_of(k + 1) <= kTableCap &&
           (k + 2) * prefix_bits(pr.dl) <= 64)
      ++k;
    pl.k = k; pl.s = f - k; pl.units = units_of(k);
    if (pr.dl > 2 && k > 0) {
      auto v = std::make_shared<std::vector<uint64_t>>();
      rgs_enumerate(k + 1, pr.dl, *v, kTableCap + 1);
      pl.shared = v;
    }
  }
  int64_t tabw = 0, initw = 0;
  if (bkern == K_PAIR16) walk_pair16_table_sizes(pr.mode, pr.c, pl.k, pl.s, &tabw, &initw);
  else if (bkern == K_U8) walk_u8_table_sizes(pr.mode, pr.c, pl.k, pl.s, pl.u8_lpu, &tabw, &initw);
  else if (bkern == K_LDU8) walk_ldu8_table_sizes(pr.dl, pr.c, pl.k, pl.s, &tabw, &initw);
  // per-matrix records start 16-byte aligned (the kernels read them as int4 / LDS.128 rows)
  tabw = (tabw + 3) & ~(int64_t)3;
  initw = (initw + 3) & ~(int64_t)3;
  auto up8 = [](size_t x) { return (x + 7) & ~(size_t)7; };
  const size_t oM = 0, oTab = oM + up8(batch * nm), oInit = oTab + up8(batch * (size_t)tabw);
  const size_t oKey = oInit + up8(batch * (size_t)initw);                 // int32 units so far
  // keys, lex, rmax, values: int64 each per matrix; then argmax bytes
  const size_t words32 = oKey + 8 * (size_t)batch + up8((size_t)batch * n) / 4 + 8;
  if ((rc = grow(&cx->dBatch, &cx->capBatch, words32 / 2 + 1))) return rc;
  const std::vector<uint64_t>& ptab = pl.prefixes();
  if (!ptab.empty()) {
    cx->preHold.reset();
    if ((rc = grow(&cx->dPre, &cx->capPre, ptab.size()))) return rc;
  }
  int32_t* base = reinterpret_cast<int32_t*>(cx->dBatch);
  int32_t* dIn = cx->dIn;
  int32_t* dMo = base + oM;
  uint32_t* dTab = reinterpret_cast<uint32_t*>(base + oTab);
  int32_t* dInit = base + oInit;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(base + oKey);
  unsigned long long* lex = keys + batch;
  unsigned long long* rmax = lex + batch;
  int64_t* vals = reinterpret_cast<int64_t*>(rmax + batch);
  int8_t* args = reinterpret_cast<int8_t*>(vals + batch);
  if (!ptab.empty()) CU(cudaMemcpyAsync(cx->dPre, ptab.data(), sizeof(uint64_t) * ptab.size(), cudaMemcpyHostToDevice, s));
  orient_kernel<<<dim3(std::min(64, (int)((nm + 255) / 256)), std::min(batch, 65535)), 256, 0, s>>>(
      dIn, n, m, pr.transposed ? 1 : 0, dMo, batch);
  CU(cudaGetLastError());
  CU(cudaMemsetAsync(keys, 0, sizeof(unsigned long long) * batch, s));
  CU(cudaMemsetAsync(lex, 0xFF, sizeof(unsigned long long) * batch, s));
  CU(cudaMemsetAsync(rmax, 0, sizeof(unsigned long long) * batch, s));
  CU(cudaMemsetAsync(cx->dCtl, 0, sizeof(unsigned long long), s));     // generic kernel's work counter
  WalkParams wp{};
  wp.M = dMo; wp.r = pr.r; wp.c = pr.c; wp.mode = pr.mode; wp.d = pr.dl; wp.k = pl.k; wp.s = pl.s;
  wp.pbits = prefix_bits(pr.dl); wp.prefix_table = ptab.empty() ? nullptr : cx->dPre;
  wp.counter = cx->dCtl; wp.key = keys; wp.unit_max = nullptr; wp.chunk_ctr = cx->dCtl + 5;
  wp.unit_begin = 0; wp.unit_count = pl.units * batch;
  wp.batch = batch; wp.units_per = pl.units; wp.m_stride = (int64_t)nm; wp.tab_stride = tabw; wp.init_stride = initw; wp.one = 1;
  wp.u8_lpu = bkern == K_U8 ? pl.u8_lpu : 1;
  wp.key_shift = 0;
  int block = 32, grid = 1;
  CU(cudaEventRecord(cx->ev[1], s));
  if (bkern >= 0) {
    // chunks of 32 lanes x P units (byte binary walk: 32 / lpu lane groups of P units)
    int occ = 0;
    int64_t per_chunk = 32;
    if (bkern == K_PAIR16) {
      occ = walk_pair16_occupancy(pr.mode, pr.c, pl.s, &block);
      per_chunk = 32 * (int64_t)walk_pair16_units_per_lane(pr.mode, pr.c);
    } else if (bkern == K_U8) {
      occ = walk_u8_occupancy(pr.mode, pr.c, pl.s, pl.u8_lpu, &block);
      per_chunk = 32 / pl.u8_lpu * (int64_t)walk_u8_units_per_lane(pr.mode, pr.c, pl.u8_lpu);
    } else {
      occ = walk_ldu8_occupancy(pr.dl, pr.c, pl.s, &block);
      per_chunk = 32 * (int64_t)walk_ldu8_units_per_lane(pr.dl, pr.c, pl.s);
    }
    const int64_t chunks = (int64_t)batch * ((pl.units + per_chunk - 1) / per_chunk);
    grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(1, occ) * cx->nsm, chunks));
    cudaError_t e = cudaErrorInvalidValue;
    int32_t* tab32 = reinterpret_cast<int32_t*>(dTab);
    if (bkern == K_PAIR16) e = walk_pair16_launch(wp, tab32, dInit, grid, s, &block);
    else if (bkern == K_U8) e = walk_u8_launch(wp, tab32, dInit, grid, s, &block);
    else e = walk_ldu8_launch(wp, tab32, dInit, grid, s, &block);
    if (e != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  } else {
    const int occ = std::max(1, walk_generic_occupancy(pr.dl, pr.c, &block));
    const int64_t want = (wp.unit_count + block / 32 - 1) / (block / 32);
    grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)occ * cx->nsm, want));
    if (walk_generic_launch(wp, grid, s, &block) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  }
  CU(cudaEventRecord(cx->ev[2], s));
  WalkParams rp = wp;
  rp.unit_count = pl.units;          // recovery: units of one matrix (blockIdx.y = matrix)
  if (recover_launch(rp, lex, rmax, s) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  FinalizeArgs fa;
  fa.key = keys; fa.lex = lex; fa.table = wp.prefix_table; fa.Min = dIn; fa.n = n; fa.m = m; fa.r = pr.r;
  fa.k = pl.k; fa.s = pl.s; fa.base = pr.dl; fa.mode = pr.mode; fa.transposed = pr.transposed ? 1 : 0;
  fa.pbits = prefix_bits(pr.dl);
  fa.key_shift = 0;
  fa.units = pl.units;
  fa.value_out = vals; fa.argmax_out = args;
  finalize_kernel<<<batch, 128, 0, s>>>(fa);
  CU(cudaGetLastError());
  std::vector<unsigned long long> hk(3 * (size_t)batch);
  std::vector<int64_t> hv((size_t)batch);
  std::vector<int8_t> ha(argmax ? (size_t)batch * n : 0);
  CU(cudaMemcpyAsync(hk.data(), keys, sizeof(unsigned long long) * 3 * batch, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(hv.data(), vals, sizeof(int64_t) * batch, cudaMemcpyDeviceToHost, s));
  if (argmax) CU(cudaMemcpyAsync(ha.data(), args, (size_t)batch * n, cudaMemcpyDeviceToHost, s));
  CU(cudaEventRecord(cx->ev[3], s));
  CU(cudaStreamSynchronize(s));
  for (int b = 0; b < batch; ++b)
    if (!recovery_consistent(hk[b], hk[batch + b], hk[2 * (size_t)batch + b])) return LNORM_EINTERNAL;
  std::memcpy(values, hv.data(), sizeof(int64_t) * batch);
  if (argmax) std::memcpy(argmax, ha.data(), (size_t)batch * n);
  float wms = 0, tms = 0;
  cudaEventElapsedTime(&wms, cx->ev[1], cx->ev[2]);
  cudaEventElapsedTime(&tms, cx->ev[0], cx->ev[3]);
  lnorm_stats S{};
  S.rows = pr.r; S.cols = pr.c; S.transposed = pr.transposed; S.prefix_digits = pl.k; S.suffix_digits = pl.s;
  S.d = pr.d == 1 ? 1 : pr.dl; S.units = pl.units * batch; S.units_total = S.units;
  S.steps = (double)S.units * (double)ipow(pr.dl, pl.s);
  S.column_updates = S.steps * pr.c * (pr.mode == MODE_LD && pr.dl >= 3 ? 2 : 1);
  S.walk_ms = wms; S.total_ms = tms; S.launches = bkern >= 0 ? 7 : 6; S.variant = pl.kernel; S.block_threads = block;
  S.grid_blocks = grid;
  S.paired_rows = pl.kernel == K_LDU8 ? walk_ldu8_paired_rows(pr.dl, pl.s) : (pl.kernel == K_U8 ? 1 : 0);
  g_stats = S;
  return LNORM_OK;
}

int lnorm_compute_sliced(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                         int32_t slices, int64_t* value, int8_t* argmax) {
  if (!M || slices < 1 || slices > 4096) return LNORM_EINVAL;
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  return compute_on(dev, M, nullptr, n, m, d, with_marginals, 0, 1, nullptr, nullptr, value, argmax, slices);
}

int lnorm_prefix_maxima(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                        int32_t nfixed, const int8_t* prefixes, int64_t count, int64_t* out) {
  if (!M || !prefixes || !out || count < 1 || nfixed < 1 || nfixed > n) return LNORM_EINVAL;
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  Problem pr;
  if ((rc = validate(M, n, m, d, with_marginals, &pr))) return rc;
  // no orientation, no label reduction: the hook walks exactly the suffix of the given rows
  pr.transposed = false; pr.r = n; pr.c = m;
  pr.dl = d == 1 ? 2 : d;
  if (pr.r > kMaxRows - 1 || pr.c > kMaxCols) return LNORM_ETOOLARGE;
  {
    GuardStats gs;
    host_stats(M, pr, &gs);
    if ((rc = apply_stats(gs, &pr))) return rc;
  }
  const int base = pr.dl;
  Plan pl;
  pl.k = nfixed - 1; pl.s = n - nfixed; pl.units = count;
  pl.table.resize(count);
  const int pb = prefix_bits(base);
  if (nfixed * pb > 64) return LNORM_EINVAL;
  for (int64_t i = 0; i < count; ++i) {
    uint64_t w = 0;
    for (int x = 0; x < nfixed; ++x) {
      int v = prefixes[i * nfixed + x];
      if (v < 0 || v >= base) return LNORM_EINVAL;
      if (x == 0 && with_marginals && v != 0) return LNORM_EINVAL;
      w |= (uint64_t)v << (pb * x);
    }
    pl.table[i] = w;
  }
  if (base == 2) {
    // same family preference as make_plan (paired > column-paired > int32 > generic)
    const int ov = kernel_override();
    pl.kernel = K_GEN;
    if (ov != K_GEN && walk_bin_supported(pr.mode, pr.c, pl.s)) pl.kernel = K_BIN;
    if (ov != K_GEN && ov != K_BIN && pr.fits16 && walk_bin16_supported(pr.mode, pr.c, pl.s) &&
        walk_bin16_table_fits(pr.mode, pr.c, pl.k, pl.s))
      pl.kernel = K_BIN16;
    if (ov != K_GEN && ov != K_BIN && ov != K_BIN16 && pr.fitsPair && walk_pair16_supported(pr.mode, pr.c, pl.s))
      pl.kernel = K_PAIR16;
    // the u8 kernel needs aligned lane groups: prefix i*P + j equals prefix i*P on rows
    // 0..k-lg and carries the bits of j on the last lg prefix rows (row k = bit 0)
    bool grouped = false;
    for (int lpu = walk_u8_lanes_per_unit(pr.mode, pr.c); lpu >= 1 && !grouped; --lpu) {
      const int lg = u8_lane_bits(pr, lpu), P = 1 << lg;
      grouped = ov < 0 && pl.k >= lg && count % P == 0 && u8_fits(pr, pl.s + lg) &&
                walk_u8_supported(pr.mode, pr.c, pl.s, lpu);
      for (int64_t i = 0; grouped && i < count; ++i) {
        const int64_t h = i - i % P;
        for (int x = 0; x <= pl.k && grouped; ++x) {
          const int v = prefixes[i * nfixed + x];
          if (x <= pl.k - lg) grouped = v == prefixes[h * nfixed + x];
          else grouped = v == (int)(((i % P) >> (pl.k - x)) & 1);
        }
      }
      if (grouped) pl.u8_lpu = lpu;
    }
    if (grouped) pl.kernel = K_U8;
  }
  else {
    // same family order as make_plan, each on its own column limit
    const int ov = kernel_override();
    pl.kernel = K_GEN;
    if (ov != K_GEN) {
      if (ov < 0 && pr.sufW[pr.r] <= 255 && walk_ldu8_supported(base, pr.c, pl.s)) pl.kernel = K_LDU8;
      else if (ov != K_BIN && ov != K_BIN16 && pr.fitsLdPair && walk_ldpair16_supported(base, pr.c, pl.s)) pl.kernel = K_LDPAIR16;
      else if (ov != K_BIN && pr.fits16 && walk_ld16_supported(base, pr.c, pl.s)) pl.kernel = K_LD16;
      else if (walk_ld_supported(base, pr.c, pl.s)) pl.kernel = K_LD;
    }
  }
  long double words = 1;
  for (int i = 0; i < pl.s; ++i) words *= base;
  if (words >= 4.0e9L) return LNORM_ETOOLARGE;
  DevCtx* cx = nullptr;
  if ((rc = ctx_get(dev, &cx))) return rc;
  std::lock_guard<std::mutex> g(cx->mu);
  CU(cudaSetDevice(dev));
  if ((rc = grow(&cx->dIn, &cx->capIn, (size_t)n * m))) return rc;
  if ((rc = grow(&cx->dM, &cx->capM, (size_t)n * m))) return rc;
  if ((rc = grow(&cx->dPre, &cx->capPre, (size_t)count))) return rc;
  if ((rc = grow(&cx->dUnit, &cx->capUnit, (size_t)count))) return rc;
  cudaStream_t s = cx->stream;
  CU(cudaMemcpyAsync(cx->dM, M, sizeof(int32_t) * n * m, cudaMemcpyHostToDevice, s));
  cx->preHold.reset();
  CU(cudaMemcpyAsync(cx->dPre, pl.table.data(), sizeof(uint64_t) * count, cudaMemcpyHostToDevice, s));
  init_ctl_kernel<<<1, 1, 0, s>>>(cx->dCtl);
  WalkParams wp{};
  wp.M = cx->dM; wp.r = n; wp.c = m; wp.mode = pr.mode; wp.d = base; wp.k = pl.k; wp.s = pl.s;
  wp.unit_begin = 0; wp.unit_count = count; wp.prefix_table = cx->dPre; wp.pbits = pb;
  walk_params_single(wp);
  wp.counter = cx->dCtl; wp.key = cx->dCtl + 1; wp.unit_max = cx->dUnit; wp.chunk_ctr = cx->dCtl + 5;
  int grid = 0, block = 0;
  CU(cudaEventRecord(cx->ev[1], s));
  if ((rc = launch_walk(*cx, pr, pl, wp, &grid, &block))) return rc;
  CU(cudaEventRecord(cx->ev[2], s));
  CU(cudaMemcpyAsync(out, cx->dUnit, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  float wms = 0;
  cudaEventElapsedTime(&wms, cx->ev[1], cx->ev[2]);
  lnorm_stats S{};
  S.rows = pr.r; S.cols = pr.c; S.prefix_digits = pl.k; S.suffix_digits = pl.s; S.d = pr.d == 1 ? 1 : base;
  S.units = count; S.units_total = count;
  S.steps = (double)count * (double)ipow(base, pl.s);
  S.column_updates = S.steps * pr.c * (pr.mode == MODE_LD && base >= 3 ? 2 : 1);
  S.walk_ms = wms; S.total_ms = wms; S.launches = pl.kernel == K_GEN ? 1 : 2; S.variant = pl.kernel;
  S.block_threads = block; S.grid_blocks = grid;
  S.paired_rows = pl.kernel == K_LDU8 ? walk_ldu8_paired_rows(pr.dl, pl.s) : (pl.kernel == K_U8 ? 1 : 0);
  S.packed_units = pl.kernel == K_LDU8 && walk_ldu8_packed(pr.dl, pr.c, pl.s) ? 2 : 0;
  g_stats = S;
  return LNORM_OK;
}

int lnorm_unit_maxima(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                      int32_t prefix_digits, const uint64_t* units, int64_t count, int32_t* unit_max) {
  if (!M || !units || !unit_max || count < 1 || prefix_digits < 0 || prefix_digits >= n) return LNORM_EINVAL;
  Problem pr;
  int rc = validate(M, n, m, d, with_marginals, &pr);
  if (rc) return rc;
  const int k = prefix_digits, nfixed = k + 1;
  std::vector<int8_t> pre((size_t)count * nfixed, 0);
  if (d == 1 || pr.dl == 2) {
    if (k > 62) return LNORM_EINVAL;
    for (int64_t i = 0; i < count; ++i) {
      if (units[i] >> k) return LNORM_EINVAL;
      for (int x = 1; x <= k; ++x) pre[(size_t)i * nfixed + x] = (int8_t)((units[i] >> (k - x)) & 1ull);
    }
  } else {
    const int dl = pr.dl, pb = prefix_bits(dl);
    if (nfixed * pb > 64 || rgs_count(nfixed, dl) > kTableCap) return LNORM_EINVAL;
    std::vector<uint64_t> list;
    rgs_enumerate(nfixed, dl, list, kTableCap + 1);
    for (int64_t i = 0; i < count; ++i) {
      if (units[i] >= list.size()) return LNORM_EINVAL;
      for (int x = 0; x < nfixed; ++x)
        pre[(size_t)i * nfixed + x] = (int8_t)((list[units[i]] >> (pb * x)) & ((1ull << pb) - 1ull));
    }
  }
  std::vector<int64_t> out((size_t)count);
  if ((rc = lnorm_prefix_maxima(M, n, m, d, with_marginals, nfixed, pre.data(), count, out.data()))) return rc;
  for (int64_t i = 0; i < count; ++i) unit_max[i] = (int32_t)out[i];
  return LNORM_OK;
}

int lnorm_walk_trace(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                     int32_t nfixed, const int8_t* prefix, int64_t max_steps, int64_t* values, int8_t* digits) {
  if (!M || !prefix || !values || nfixed < 1 || nfixed > n || max_steps < 1) return LNORM_EINVAL;
  int dev = 0, rc = current_device(&dev);
  if (rc) return rc;
  Problem pr;
  if ((rc = validate(M, n, m, d, with_marginals, &pr))) return rc;
  pr.r = n; pr.c = m; pr.dl = d == 1 ? 2 : d;
  if (n > kMaxRows - 1 || m > kMaxCols) return LNORM_ETOOLARGE;
  const int base = pr.dl, s_ = n - nfixed;
  long double words = 1;
  for (int i = 0; i < s_; ++i) words *= base;
  if (words > (long double)max_steps) return LNORM_EINVAL;
  uint64_t w = 0;
  const int pb = prefix_bits(base);
  if (nfixed * pb > 64) return LNORM_EINVAL;
  for (int x = 0; x < nfixed; ++x) {
    if (prefix[x] < 0 || prefix[x] >= base) return LNORM_EINVAL;
    w |= (uint64_t)prefix[x] << (pb * x);
  }
  DevCtx* cx = nullptr;
  if ((rc = ctx_get(dev, &cx))) return rc;
  std::lock_guard<std::mutex> g(cx->mu);
  CU(cudaSetDevice(dev));
  const int64_t nw = (int64_t)words;
  if ((rc = grow(&cx->dM, &cx->capM, (size_t)n * m))) return rc;
  if ((rc = grow(&cx->dPre, &cx->capPre, 1))) return rc;
  if ((rc = grow(&cx->dUnit, &cx->capUnit, (size_t)nw + (size_t)(nw * n + 7) / 8))) return rc;
  cudaStream_t s = cx->stream;
  CU(cudaMemcpyAsync(cx->dM, M, sizeof(int32_t) * n * m, cudaMemcpyHostToDevice, s));
  cx->preHold.reset();
  CU(cudaMemcpyAsync(cx->dPre, &w, sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  WalkParams wp{};
  wp.M = cx->dM; wp.r = n; wp.c = m; wp.mode = pr.mode; wp.d = base; wp.k = nfixed - 1; wp.s = s_;
  wp.unit_begin = 0; wp.unit_count = 1; wp.prefix_table = cx->dPre; wp.pbits = pb;
  walk_params_single(wp);
  int8_t* ddig = reinterpret_cast<int8_t*>(cx->dUnit + nw);
  if (trace_launch(wp, nw, cx->dUnit, digits ? ddig : nullptr, s) != cudaSuccess) { (void)cudaGetLastError(); return LNORM_ECUDA; }
  CU(cudaMemcpyAsync(values, cx->dUnit, sizeof(int64_t) * nw, cudaMemcpyDeviceToHost, s));
  if (digits) CU(cudaMemcpyAsync(digits, ddig, (size_t)nw * n, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return LNORM_OK;
}

int32_t lnorm_gray_digit(int32_t d, int32_t i, uint64_t j) {
  if (d < 2 || i < 0 || i > 63) return -1;
  if (d == 2) return (int32_t)brgc_digit((uint32_t)i, j);
  return (int32_t)dary_digit((uint32_t)d, (uint32_t)i, j);
}

int lnorm_gray_change(int32_t d, uint64_t j, int32_t* digit, int32_t* from, int32_t* to) {
  if (d < 2 || j < 1 || !digit || !from || !to) return LNORM_EINVAL;
  if (d == 2) {
    uint32_t i = brgc_change(j);
    *digit = (int32_t)i;
    *from = (int32_t)brgc_digit(i, j - 1);
    *to = (int32_t)brgc_digit(i, j);
    return LNORM_OK;
  }
  uint32_t i, f, t;
  dary_change_values((uint32_t)d, j, &i, &f, &t);
  *digit = (int32_t)i; *from = (int32_t)f; *to = (int32_t)t;
  return LNORM_OK;
}

int lnorm_partition(uint64_t C, int64_t T, int64_t t, int64_t* j_min, int64_t* j_max) {
  if (T < 1 || t < 0 || t >= T || !j_min || !j_max) return LNORM_EINVAL;
  algorithm1(C, T, t, j_min, j_max);
  return LNORM_OK;
}

uint64_t lnorm_reduction_key(int32_t value, uint32_t unit) { return make_key(value, unit); }

int lnorm_key_decode(uint64_t key, int32_t* value, uint32_t* unit) {
  if (!value || !unit) return LNORM_EINVAL;
  *value = key_value(key);
  *unit = key_unit(key);
  return LNORM_OK;
}

int lnorm_plan(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals, int32_t world,
               lnorm_plan_info* out) {
  if (!out || world < 1) return LNORM_EINVAL;
  Problem pr;
  int rc = validate(M, n, m, d, with_marginals, &pr);
  if (rc) return rc;
  Plan pl;
  if ((rc = make_plan(pr, world, &pl))) return rc;
  lnorm_plan_info I{};
  I.rows = pr.r; I.cols = pr.c; I.transposed = pr.transposed; I.d_walked = pr.dl;
  I.prefix_digits = pl.k; I.suffix_digits = pl.s; I.variant = pl.kernel; I.packed_ok = pr.fits16;
  I.units = pl.units;
  I.steps = (double)pl.units * (double)ipow(pr.dl, pl.s);
  I.lanes_per_unit = pl.kernel == K_U8 ? pl.u8_lpu : 1;
  I.words = pl.kernel == K_U8 ? walk_u8_words(pr.mode, pr.c) : 0;
  *out = I;
  return LNORM_OK;
}

int lnorm_last_stats(lnorm_stats* out) {
  if (!out) return LNORM_EINVAL;
  *out = g_stats;
  return LNORM_OK;
}

}  // extern "C"
