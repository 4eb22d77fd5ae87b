// Walk-shaped throughput probe: candidate inner loops of the Gray walk
// (one uniform row per step applied to every lane's column sums, then an
// abs-accumulate and a max), timed as column-updates per clock per SM.
// Decides the hot-loop arithmetic of the real kernels.
//
//   V_I32_LDS   int32 sums, row from shared memory (LDS.128 broadcast)
//   V_I32_CST   int32 sums, row from the constant bank at a uniform index
//   V_S16_LDS   s16x2 packed sums: VIADD.16x2 update + VIADDMNMX.S16x2 max-accumulate
//   V_B16_LDS   biased packed sums: 32-bit IADD update + LOP3 fix + VIADDMNMX.S16x2
//   V_U8_LDS    u8x4 offset sums: 32-bit IADD update + VABSDIFF4.U8.ACC against a per-unit bias word
//   V_U8S_LDS   same, the P units of a lane share their bias words (operand reuse)
//   V_U8SE_LDS  shared bias, evaluate-then-update order (A in the reuse slot of the add)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 tools/walkprobe.cu -o tools/walkprobe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <climits>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

enum { V_I32_LDS = 0, V_I32_CST, V_S16_LDS, V_B16_LDS, V_U8_LDS, V_U8S_LDS, V_U8SE_LDS, V_N };
static const char* kNames[V_N] = {"i32_lds", "i32_const", "s16x2_lds", "biased16_lds", "u8x4_lds", "u8x4_sharedB_lds", "u8x4_sharedB_evalfirst_lds"};

constexpr int NROWS = 64;
__constant__ int32_t cRows[NROWS * 64];

struct Rec { long long t0, t1; unsigned smid; unsigned pad; };
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

template <int V, int C, int P>
__global__ void __launch_bounds__(128) walk(int32_t* out, Rec* rec, int steps, const int32_t* rows) {
  constexpr int W = (V == V_U8_LDS || V == V_U8S_LDS || V == V_U8SE_LDS) ? C / 4 : (V == V_S16_LDS || V == V_B16_LDS) ? C / 2 : C;   // 32-bit words per unit
  __shared__ __align__(16) int32_t srow[NROWS * W];
  __shared__ int32_t srsum[NROWS];
  for (int i = threadIdx.x; i < NROWS * W; i += blockDim.x) srow[i] = rows[i];
  for (int i = threadIdx.x; i < NROWS; i += blockDim.x) srsum[i] = rows[NROWS * W + i];
  __syncthreads();
  int32_t m[P][W];
  uint32_t bb[P][W];
  int32_t best[P], S[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    best[p] = INT_MIN; S[p] = 0;
#pragma unroll
    for (int y = 0; y < W; ++y) { m[p][y] = (int32_t)((threadIdx.x * 13 + y * 7 + p) & 15) - 8;
                                  bb[p][y] = 0x40404040u * (uint32_t)((threadIdx.x * 5 + y + p) & 3); }
  }
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int row = (s * 7) & (NROWS - 1);
    int32_t r[W];
    if constexpr (V == V_I32_CST) {
#pragma unroll
      for (int y = 0; y < W; ++y) r[y] = cRows[row * 64 + y];
    } else {
      const int4* src = reinterpret_cast<const int4*>(srow + row * W);
#pragma unroll
      for (int q = 0; q < W / 4; ++q) { int4 v = src[q]; r[4*q] = v.x; r[4*q+1] = v.y; r[4*q+2] = v.z; r[4*q+3] = v.w; }
    }
    const int32_t rs = srsum[row];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if constexpr (V == V_I32_LDS || V == V_I32_CST) {
        int32_t a0 = 0, a1 = 0;
#pragma unroll
        for (int y = 0; y < W; y += 2) {
          m[p][y] += r[y];     a0 = __sad(m[p][y], 0, a0);
          m[p][y+1] += r[y+1]; a1 = __sad(m[p][y+1], 0, a1);
        }
        best[p] = max(best[p], a0 + a1);
      } else if constexpr (V == V_S16_LDS) {
        uint32_t a0 = 0, a1 = 0;
#pragma unroll
        for (int y = 0; y < W; y += 2) {
          m[p][y] = __vadd2(m[p][y], r[y]);       a0 = __viaddmax_s16x2(a0, m[p][y], a0);
          m[p][y+1] = __vadd2(m[p][y+1], r[y+1]); a1 = __viaddmax_s16x2(a1, m[p][y+1], a1);
        }
        S[p] += rs;
        uint32_t a = __vadd2(a0, a1);
        int32_t h = __dp2a_lo((int)a, 0x00010001, 0);   // lo16 + hi16 (signed)
        best[p] = max(best[p], 2 * h - S[p]);
      } else if constexpr (V == V_U8_LDS) {
        uint32_t a0 = (uint32_t)S[p], a1 = 0;
#pragma unroll
        for (int y = 0; y < W; y += 2) {
          m[p][y] += r[y];
          asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a0) : "r"(m[p][y]), "r"(bb[p][y]));
          if (y + 1 < W) {
            m[p][y+1] += r[y+1];
            asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a1) : "r"(m[p][y+1]), "r"(bb[p][y+1]));
          }
        }
        best[p] = __viaddmax_s32((int)a0, (int)a1, best[p]);
      } else if constexpr (V == V_U8S_LDS) {
        uint32_t a0 = (uint32_t)S[p], a1 = 0;
#pragma unroll
        for (int y = 0; y < W; y += 2) {
          m[p][y] += r[y];
          asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a0) : "r"(m[p][y]), "r"(bb[0][y]));
          if (y + 1 < W) {
            m[p][y+1] += r[y+1];
            asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a1) : "r"(m[p][y+1]), "r"(bb[0][y+1]));
          }
        }
        best[p] = __viaddmax_s32((int)a0, (int)a1, best[p]);
      } else if constexpr (V == V_U8SE_LDS) {
        uint32_t a0 = (uint32_t)S[p], a1 = 0;
#pragma unroll
        for (int y = 0; y < W; y += 2) {
          asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a0) : "r"(m[p][y]), "r"(bb[0][y]));
          m[p][y] += r[y];
          if (y + 1 < W) {
            asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %0;" : "+r"(a1) : "r"(m[p][y+1]), "r"(bb[0][y+1]));
            m[p][y+1] += r[y+1];
          }
        }
        best[p] = __viaddmax_s32((int)a0, (int)a1, best[p]);
      } else {  // V_B16_LDS: low half biased by 0x8000 so a plain 32-bit add is carry-free
        uint32_t a0 = 0, a1 = 0;
#pragma unroll
        for (int y = 0; y < W; y += 2) {
          m[p][y] += r[y];     a0 = __viaddmax_s16x2(a0, (uint32_t)m[p][y] ^ 0x8000u, a0);
          m[p][y+1] += r[y+1]; a1 = __viaddmax_s16x2(a1, (uint32_t)m[p][y+1] ^ 0x8000u, a1);
        }
        S[p] += rs;
        uint32_t a = __vadd2(a0, a1);
        int32_t h = __dp2a_lo((int)a, 0x00010001, 0);
        best[p] = max(best[p], 2 * h - S[p]);
      }
    }
  }
  long long t1 = clock64();
  int32_t acc = 0;
#pragma unroll
  for (int p = 0; p < P; ++p) { acc ^= best[p]; for (int y = 0; y < W; ++y) acc ^= m[p][y]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) { rec[blockIdx.x].t0 = t0; rec[blockIdx.x].t1 = t1; rec[blockIdx.x].smid = smid(); }
}

template <int V, int C, int P>
static void run(int nsm, int bps, int steps, int32_t* dout, Rec* drec, const int32_t* drows) {
  const int threads = 128, blocks = nsm * bps;
  walk<V, C, P><<<blocks, threads>>>(dout, drec, 8, drows);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  walk<V, C, P><<<blocks, threads>>>(dout, drec, steps, drows);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  std::vector<Rec> h(blocks);
  CK(cudaMemcpy(h.data(), drec, sizeof(Rec) * blocks, cudaMemcpyDeviceToHost));
  std::vector<long long> mn(512, LLONG_MAX), mx(512, 0); std::vector<int> cnt(512, 0);
  for (auto& r : h) { mn[r.smid] = std::min(mn[r.smid], r.t0); mx[r.smid] = std::max(mx[r.smid], r.t1); cnt[r.smid]++; }
  std::vector<double> v; double cyc = 0; int k = 0;
  for (int s = 0; s < 512; ++s) if (cnt[s]) {
    double c = (double)(mx[s] - mn[s]); cyc += c; k++;
    v.push_back((double)threads * cnt[s] * steps * P * C / c); }
  std::sort(v.begin(), v.end());
  double regs = 0; cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, walk<V, C, P>)); regs = fa.numRegs;
  printf("{\"variant\": \"%s\", \"C\": %d, \"P\": %d, \"col_updates_per_clk_per_sm\": %.2f, \"min\": %.2f, \"max\": %.2f, "
         "\"regs\": %.0f, \"local_bytes\": %zu, \"blocks_per_sm\": %d, \"kernel_ms\": %.3f, \"mhz\": %.0f}\n",
         kNames[V], C, P, v[v.size() / 2], v.front(), v.back(), regs, fa.localSizeBytes, bps, ms, cyc / k / (ms * 1e3));
  fflush(stdout);
}

int main(int argc, char** argv) {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int steps = argc > 1 ? atoi(argv[1]) : 20000;
  std::vector<int32_t> rows(NROWS * 64 + NROWS);
  for (size_t i = 0; i < rows.size(); ++i) rows[i] = (int32_t)((i * 2654435761u) % 21) - 10;
  CK(cudaMemcpyToSymbol(cRows, rows.data(), sizeof(int32_t) * NROWS * 64));
  int32_t *dout, *drows; Rec* drec;
  CK(cudaMalloc(&dout, sizeof(int32_t) * nsm * 32 * 128)); CK(cudaMalloc(&drec, sizeof(Rec) * nsm * 32));
  CK(cudaMalloc(&drows, sizeof(int32_t) * rows.size()));
  CK(cudaMemcpy(drows, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice));
  for (int bps : {4, 8}) {
    run<V_I32_LDS, 32, 1>(nsm, bps, steps, dout, drec, drows);
    run<V_I32_LDS, 32, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_I32_LDS, 48, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_I32_CST, 32, 1>(nsm, bps, steps, dout, drec, drows);
    run<V_I32_CST, 32, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_S16_LDS, 32, 1>(nsm, bps, steps, dout, drec, drows);
    run<V_S16_LDS, 32, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_S16_LDS, 48, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_S16_LDS, 64, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_B16_LDS, 32, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_B16_LDS, 48, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_U8_LDS, 48, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_U8_LDS, 32, 4>(nsm, bps, steps, dout, drec, drows);
    run<V_U8_LDS, 48, 4>(nsm, bps, steps, dout, drec, drows);
    run<V_U8_LDS, 64, 4>(nsm, bps, steps, dout, drec, drows);
    run<V_U8S_LDS, 48, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_U8S_LDS, 48, 4>(nsm, bps, steps, dout, drec, drows);
    run<V_U8SE_LDS, 48, 2>(nsm, bps, steps, dout, drec, drows);
    run<V_U8SE_LDS, 48, 4>(nsm, bps, steps, dout, drec, drows);
  }
  return 0;
}
