// Integer/issue-pipe throughput microbenchmark for the L_d Gray-walk roofline
// (SURVEY.md §8(d) "Roofline microbenchmark").  Measures lane-operations per
// clock per SM for each candidate hot-loop instruction and for the 1:1 mixes
// the walk kernels issue, so DESIGN.md's "alu" peak is a B200 measurement,
// not an assumption.  Standalone executable; prints one JSON object per probe.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo tools/peaks.cu -o tools/peaks
// Verify opcodes: cuobjdump -sass tools/peaks | grep -E 'VABSDIFF|IMAD|IADD3|VIADD|VIMNMX|HFMA2|HADD2'
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int CH = 8;       // independent chains per thread
constexpr int UNR = 32;     // unrolled iterations per loop trip

__constant__ int32_t cTab[1024];

struct Rec { long long t0, t1; unsigned smid; unsigned pad; };

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

// op ids
enum {
  OP_ADD = 0,        // add.s32            -> IADD3 / IMAD.IADD (ptxas choice)
  OP_MAD,            // mad.lo.s32 x,a,1,x -> IMAD (fma pipe)
  OP_SAD,            // sad.s32 acc,a,0,acc-> VABSDIFF
  OP_ADD_SAD,        // 1:1 add + sad (the int32 walk body)
  OP_MAD_SAD,        // 1:1 mad + sad
  OP_VADD2,          // __vadd2            -> VIADD.16x2
  OP_VIADDMAX2,      // __viaddmax_s16x2   -> VIADDMNMX.S16x2
  OP_VADD2_VIADDMAX2,// 1:1 (packed s16 walk body)
  OP_VMAXU2,         // __vmaxu2           -> VIMNMX.U16x2
  OP_MAD_VMAXU2_MAD, // biased-u16 body: mad + vmaxu2 + mad
  OP_HADD2,          // __hadd2            -> HADD2
  OP_HFMA2ABS,       // __hadd2(__habs2)   -> HFMA2 |a|
  OP_HADD2_HFMA2ABS, // 1:1 (fp16x2 walk body)
  OP_ADDC_SAD,       // add with __constant__ operand + sad
  OP_LDS128,         // broadcast ld.shared.v4 (+ xor to keep live)
  OP_IADD3,          // 3-input add a+b+c -> IADD3
  OP_VIADDMAX32,     // __viaddmax_s32     -> VIADDMNMX
  OP_MAD_VIADDMAX2,  // mad (packed biased update) + viaddmax s16x2
  OP_SAD4,           // vabsdiff4.add (u8x4 sum of |a_b - b_b| + acc) -> VABSDIFF4.U8.ACC
  OP_MAD_SAD4,       // 1:1 mad (packed u8x4 update) + vabsdiff4.add
  OP_ADD_SAD4,       // 1:1 add (uniform operand) + vabsdiff4.add
  OP_MAD_SAD4V,      // 1:1 mad + vabsdiff4.add with a DISTINCT bias register per chain (3 live sources)
  OP_VIMNMX3,        // __vimax3_s32       -> VIMNMX3
  OP_SAD4_VIMNMX3,   // 1:1 vabsdiff4.add + VIMNMX3
  OP_FMNMX3,         // max.f32 d,a,b,c    -> FMNMX3 (sm_100 three-input float max)
  OP_SAD4_FMNMX3,    // 1:1 vabsdiff4.add + FMNMX3 (does the float max leave the ALU pipe free?)
  OP_FMNMX,          // max.f32 d,a,b      -> FMNMX
  OP_SAD4_FMNMX,     // 1:1 vabsdiff4.add + FMNMX
  OP_SAD4_MAD_FMNMX3,// 2:1:1 vabsdiff4.add, mad, FMNMX3 (the byte d-ary walk's mix with a float max tree)
  OP_N
};
static const char* kNames[OP_N] = {
  "add.s32(uniform operand)", "mad.lo.s32", "sad.s32", "add+sad", "mad+sad", "vadd2", "viaddmax_s16x2",
  "vadd2+viaddmax_s16x2", "vmaxu2", "mad+vmaxu2+mad", "hadd2", "hfma2_abs", "hadd2+hfma2_abs",
  "add_constbank+sad", "lds128_bcast", "iadd3", "viaddmax_s32", "mad+viaddmax_s16x2", "vabsdiff4_acc",
  "mad+vabsdiff4_acc", "add+vabsdiff4_acc", "mad+vabsdiff4_acc(per-chain bias)", "vimnmx3", "vabsdiff4_acc+vimnmx3",
  "fmnmx3", "vabsdiff4_acc+fmnmx3", "fmnmx", "vabsdiff4_acc+fmnmx", "2 vabsdiff4_acc+mad+fmnmx3"};
// SASS instructions per chain per unrolled iteration, read off `cuobjdump -sass`
// (ptxas fuses two u16x2 maxes into one VIMNMX3; the constant-bank probe adds one LDCU.128 per 4 adds)
static const double kInstr[OP_N] = {1,1,1,2,2,1,1,2,0.5,3,1,1,2,2.25,1,1,1,2,1,2,2,2,1,2,1,2,1,2,4};

template <int OP>
__global__ void __launch_bounds__(256) probe(int32_t* out, Rec* rec, int trips, int32_t a_in, int32_t one_in, int32_t zero_in) {
  __shared__ int4 srow[64];
  if (threadIdx.x < 64) srow[threadIdx.x] = make_int4(threadIdx.x, a_in, one_in, zero_in);
  __syncthreads();
  int32_t x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * (c + 1) + a_in; y[c] = (int32_t)(threadIdx.x & 7) - 3 + c; }
  // per-lane registers the compiler cannot prove uniform (threadIdx.x >> 10 == 0 at 256 threads)
  const int32_t tz = (int32_t)(threadIdx.x >> 10);
  const int32_t a = a_in ^ tz, one = one_in ^ tz, zero = zero_in ^ tz;
  const unsigned au = ((unsigned)a_in * 0x00010001u) ^ (unsigned)tz;
  const unsigned bias = 0x80808080u ^ (unsigned)tz;
  unsigned bv[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) bv[c] = (0x80808080u + 0x01010101u * c) ^ (unsigned)(threadIdx.x >> (10 + c));
  long long t0 = clock64();
  for (int t = 0; t < trips; ++t) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if constexpr (OP == OP_ADD) {
          asm volatile("add.s32 %0, %0, %1;" : "+r"(x[c]) : "r"(a));
        } else if constexpr (OP == OP_MAD) {
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(one));
        } else if constexpr (OP == OP_SAD) {
          asm volatile("sad.s32 %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(zero));
        } else if constexpr (OP == OP_ADD_SAD) {
          asm volatile("add.s32 %0, %0, %1;" : "+r"(y[c]) : "r"(a));
          asm volatile("sad.s32 %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(zero));
        } else if constexpr (OP == OP_MAD_SAD) {
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(y[c]) : "r"(a), "r"(one));
          asm volatile("sad.s32 %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(zero));
        } else if constexpr (OP == OP_VADD2) {
          x[c] = __vadd2(x[c], y[c]); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_VIADDMAX2) {
          x[c] = __viaddmax_s16x2(x[c], y[c], x[c]); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_VADD2_VIADDMAX2) {
          y[c] = __vadd2(y[c], a); asm volatile("" : "+r"(y[c]));
          x[c] = __viaddmax_s16x2(x[c], y[c], x[c]); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_VMAXU2) {
          x[c] = __vmaxu2(x[c], y[c]); asm volatile("" : "+r"(x[c]));
          y[c] ^= 0; // keep form
        } else if constexpr (OP == OP_MAD_VMAXU2_MAD) {
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(y[c]) : "r"(a), "r"(one));
          int32_t t2 = __vmaxu2(y[c], au); asm volatile("" : "+r"(t2));
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(x[c]) : "r"(t2), "r"(one));
        } else if constexpr (OP == OP_HADD2) {
          __half2 h = *reinterpret_cast<__half2*>(&x[c]);
          __half2 g = *reinterpret_cast<__half2*>(&y[c]);
          h = __hadd2(h, g);
          x[c] = *reinterpret_cast<int32_t*>(&h); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_HFMA2ABS) {
          __half2 h = *reinterpret_cast<__half2*>(&x[c]);
          __half2 g = *reinterpret_cast<__half2*>(&y[c]);
          h = __hadd2(__habs2(g), h);
          x[c] = *reinterpret_cast<int32_t*>(&h); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_HADD2_HFMA2ABS) {
          __half2 g = *reinterpret_cast<__half2*>(&y[c]);
          __half2 aa = *reinterpret_cast<const __half2*>(&a);
          g = __hadd2(g, aa);
          y[c] = *reinterpret_cast<int32_t*>(&g); asm volatile("" : "+r"(y[c]));
          g = *reinterpret_cast<__half2*>(&y[c]);
          __half2 h = *reinterpret_cast<__half2*>(&x[c]);
          h = __hadd2(__habs2(g), h);
          x[c] = *reinterpret_cast<int32_t*>(&h); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_ADDC_SAD) {
          y[c] += cTab[(u * CH + c) & 1023]; asm volatile("" : "+r"(y[c]));
          asm volatile("sad.s32 %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(zero));
        } else if constexpr (OP == OP_LDS128) {
          int4 v;
          const int idx = (u * CH + c + t) & 63;
          asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "r"((unsigned)__cvta_generic_to_shared(&srow[idx])));
          x[c] ^= v.x; y[c] ^= v.w;
        } else if constexpr (OP == OP_IADD3) {
          asm volatile("add.s32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;" : "+r"(x[c]) : "r"(y[c]), "r"(a));
        } else if constexpr (OP == OP_VIADDMAX32) {
          x[c] = __viaddmax_s32(x[c], y[c], x[c]); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_MAD_VIADDMAX2) {
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(y[c]) : "r"(a), "r"(one));
          x[c] = __viaddmax_s16x2(x[c], y[c], x[c]); asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_SAD4) {
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bias));
        } else if constexpr (OP == OP_MAD_SAD4) {
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(y[c]) : "r"(a), "r"(one));
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bias));
        } else if constexpr (OP == OP_MAD_SAD4V) {
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(y[c]) : "r"(a), "r"(one));
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bv[c]));
        } else if constexpr (OP == OP_VIMNMX3) {
          const int32_t t3 = __vimax3_s32(x[c], y[c], a); y[c] = x[c]; x[c] = t3; asm volatile("" : "+r"(x[c]));
        } else if constexpr (OP == OP_SAD4_VIMNMX3) {
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bias));
          y[c] = __vimax3_s32(y[c], x[c], a); asm volatile("" : "+r"(y[c]));
        } else if constexpr (OP == OP_FMNMX3) {
          int32_t t3;
          asm volatile("max.f32 %0, %1, %2, %3;" : "=r"(t3) : "r"(x[c]), "r"(y[c]), "r"(a));
          y[c] = x[c]; x[c] = t3;
        } else if constexpr (OP == OP_SAD4_FMNMX3) {
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bias));
          asm volatile("max.f32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(x[c]), "r"(a));
        } else if constexpr (OP == OP_FMNMX) {
          int32_t t2;
          asm volatile("max.f32 %0, %1, %2;" : "=r"(t2) : "r"(x[c]), "r"(y[c]));
          y[c] = x[c]; x[c] = t2;
        } else if constexpr (OP == OP_SAD4_FMNMX) {
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bias));
          asm volatile("max.f32 %0, %0, %1;" : "+r"(y[c]) : "r"(x[c]));
        } else if constexpr (OP == OP_SAD4_MAD_FMNMX3) {
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bias));
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(y[c]) : "r"(a), "r"(one));
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bv[c]));
          asm volatile("max.f32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(x[c]), "r"(a));
        } else if constexpr (OP == OP_ADD_SAD4) {
          asm volatile("add.s32 %0, %0, %1;" : "+r"(y[c]) : "r"(a));
          asm volatile("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(x[c]) : "r"(y[c]), "r"(bias));
        }
      }
    }
  }
  long long t1 = clock64();
  int32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= x[c] ^ y[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) { rec[blockIdx.x].t0 = t0; rec[blockIdx.x].t1 = t1; rec[blockIdx.x].smid = smid(); }
}

template <int OP>
static void run(int nsm, int bps, int threads, int trips, int32_t* dout, Rec* drec, std::vector<Rec>& hrec) {
  const int blocks = nsm * bps;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  probe<OP><<<blocks, threads>>>(dout, drec, 2, 3, 1, 0);  // warm-up
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  probe<OP><<<blocks, threads>>>(dout, drec, trips, 3, 1, 0);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
  hrec.resize(blocks);
  CK(cudaMemcpy(hrec.data(), drec, sizeof(Rec) * blocks, cudaMemcpyDeviceToHost));
  // per-SM: ops of all blocks resident on it / (max t1 - min t0)
  std::vector<long long> mn(nsm * 2, LLONG_MAX), mx(nsm * 2, 0); std::vector<int> cnt(nsm * 2, 0);
  for (auto& r : hrec) { if (r.smid >= (unsigned)(nsm * 2)) continue;
    mn[r.smid] = std::min(mn[r.smid], r.t0); mx[r.smid] = std::max(mx[r.smid], r.t1); cnt[r.smid]++; }
  const double lane_instr_per_block = (double)threads * trips * UNR * CH * kInstr[OP];
  std::vector<double> per_sm; double cyc_sum = 0; int nused = 0;
  for (int s = 0; s < nsm * 2; ++s) if (cnt[s]) {
    double cyc = (double)(mx[s] - mn[s]); per_sm.push_back(lane_instr_per_block * cnt[s] / cyc); cyc_sum += cyc; nused++; }
  std::sort(per_sm.begin(), per_sm.end());
  double med = per_sm[per_sm.size() / 2];
  double mhz = (cyc_sum / nused) / (ms * 1e3);
  printf("{\"probe\": \"%s\", \"lane_instr_per_clk_per_sm_median\": %.2f, \"min\": %.2f, \"max\": %.2f, "
         "\"instr_per_chain_iter\": %.2f, \"chain_iters_per_clk_per_sm\": %.2f, \"kernel_ms\": %.3f, \"effective_mhz\": %.0f, \"sms\": %d, \"blocks_per_sm\": %d, \"threads\": %d}\n",
         kNames[OP], med, per_sm.front(), per_sm.back(), kInstr[OP], med / kInstr[OP], ms, mhz, nused, bps, threads);
  fflush(stdout);
}

template <int... OPS> struct All;
template <> struct All<> { static void go(int, int, int, int, int32_t*, Rec*, std::vector<Rec>&) {} };
template <int O, int... R> struct All<O, R...> {
  static void go(int nsm, int bps, int th, int trips, int32_t* o, Rec* r, std::vector<Rec>& h) {
    run<O>(nsm, bps, th, trips, o, r, h); All<R...>::go(nsm, bps, th, trips, o, r, h); }
};

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  int bps = argc > 1 ? atoi(argv[1]) : 4;   // 4 blocks x 256 threads = 32 warps/SM
  int trips = argc > 2 ? atoi(argv[2]) : 2000;
  const int threads = 256;
  std::vector<int32_t> tab(1024); for (int i = 0; i < 1024; ++i) tab[i] = (i * 7) % 21 - 10;
  CK(cudaMemcpyToSymbol(cTab, tab.data(), sizeof(int32_t) * 1024));
  int32_t* dout; Rec* drec; CK(cudaMalloc(&dout, sizeof(int32_t) * nsm * bps * threads)); CK(cudaMalloc(&drec, sizeof(Rec) * nsm * bps));
  std::vector<Rec> h;
  All<OP_ADD, OP_MAD, OP_SAD, OP_ADD_SAD, OP_MAD_SAD, OP_VADD2, OP_VIADDMAX2, OP_VADD2_VIADDMAX2, OP_VMAXU2,
      OP_MAD_VMAXU2_MAD, OP_HADD2, OP_HFMA2ABS, OP_HADD2_HFMA2ABS, OP_ADDC_SAD, OP_LDS128, OP_IADD3,
      OP_VIADDMAX32, OP_MAD_VIADDMAX2, OP_SAD4, OP_MAD_SAD4, OP_ADD_SAD4, OP_MAD_SAD4V, OP_VIMNMX3, OP_SAD4_VIMNMX3,
      OP_FMNMX3, OP_SAD4_FMNMX3, OP_FMNMX, OP_SAD4_FMNMX, OP_SAD4_MAD_FMNMX3>::go(nsm, bps, threads, trips, dout, drec, h);
  return 0;
}
