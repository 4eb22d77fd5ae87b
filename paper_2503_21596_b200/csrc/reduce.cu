// Norm-preserving matrix reduction (proofs
// App. A/B) and the argmax map-back, as single-block kernels.
//
// Rules, applied to a fixpoint in the order zero lines -> proportional lines ->
// sign-uniform columns:
//   zero row / column            : removed (L_1, L_d; L_marg: rows/columns >= 1 only,
//                                  row 0 + column 0 together when both vanish -> L_1)
//   rows x'' = c x'              : L_1 / L_marg (x', x'' >= 1): any c != 0, row x' becomes
//                                  M_x' + sgn(c) M_x'' = (1 + |c|) M_x' (rule A1) and
//                                  a_x'' = sgn(c) a_x' in the map-back; L_d: only c > 0 (A3),
//                                  label(x'') = label(x')
//   columns y'' = c y'           : all modes (L_marg: y', y'' >= 1), column y' becomes
//                                  M_y' + sgn(c) M_y'' (A1/A2); no argmax effect
//   sign-uniform columns (L_d)   : two columns each of one sign become |M_y1| + |M_y2| (App. B)
// Proportionality is tested exactly by int64 cross-multiplication against the
// first nonzero entry.  The reduced matrix is then searched by the usual path;
// the argmax of the reduced problem is expanded to the original rows.  The
// expanded strategy attains the norm but need not be the lexicographically
// smallest optimum of the original matrix (R11).
#include "common.cuh"

namespace lnorm {

namespace {

constexpr int kRedThreads = 256;

struct RedState {
  int32_t* A;          // n x m working copy (int32: every entry stays <= sum |M|)
  int32_t* rep;        // [n] representative row (-1: removed zero row), rep[x] == x if alive
  int32_t* rsgn;       // [n] sign relative to the representative
  int32_t* calive;     // [m] column alive
  int32_t* info;       // [0] n', [1] m', [2] mode after reduction, [3] changed flag
};

__device__ bool row_alive(const RedState& S, int x) { return S.rep[x] == x; }

// 0: not proportional; +1 / -1: v = c u with sgn(c) = +-1 (over alive columns)
__device__ int prop_rows(const RedState& S, int n, int m, int u, int v, int c0) {
  int j0 = -1;
  for (int j = c0; j < m; ++j)
    if (S.calive[j] && S.A[(int64_t)u * m + j] != 0) { j0 = j; break; }
  if (j0 < 0) return 0;
  const int64_t u0 = S.A[(int64_t)u * m + j0], v0 = S.A[(int64_t)v * m + j0];
  if (v0 == 0) return 0;
  for (int j = c0; j < m; ++j) {
    if (!S.calive[j]) continue;
    if ((int64_t)S.A[(int64_t)v * m + j] * u0 != (int64_t)S.A[(int64_t)u * m + j] * v0) return 0;
  }
  return (u0 > 0) == (v0 > 0) ? 1 : -1;
}

__device__ int prop_cols(const RedState& S, int n, int m, int u, int v, int r0) {
  int i0 = -1;
  for (int i = r0; i < n; ++i)
    if (row_alive(S, i) && S.A[(int64_t)i * m + u] != 0) { i0 = i; break; }
  if (i0 < 0) return 0;
  const int64_t u0 = S.A[(int64_t)i0 * m + u], v0 = S.A[(int64_t)i0 * m + v];
  if (v0 == 0) return 0;
  for (int i = r0; i < n; ++i) {
    if (!row_alive(S, i)) continue;
    if ((int64_t)S.A[(int64_t)i * m + v] * u0 != (int64_t)S.A[(int64_t)i * m + u] * v0) return 0;
  }
  return (u0 > 0) == (v0 > 0) ? 1 : -1;
}

// sign of a column over alive rows: 1 all >= 0, -1 all <= 0, 0 mixed (zero column: 1)
__device__ int col_sign(const RedState& S, int n, int m, int y) {
  bool pos = false, neg = false;
  for (int i = 0; i < n; ++i) {
    if (!row_alive(S, i)) continue;
    const int32_t v = S.A[(int64_t)i * m + y];
    pos |= v > 0;
    neg |= v < 0;
  }
  return (pos && neg) ? 0 : (neg ? -1 : 1);
}

// Single block; thread 0 drives the (tiny) combinatorial fixpoint, the block
// parallelises the O(m) / O(n) line operations.
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(const int32_t* M, int n, int m, int mode, RedState S) {
  __shared__ int act, a1, a2, sg;
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < (int64_t)n * m; i += blockDim.x) S.A[i] = M[i];
  for (int x = tid; x < n; x += blockDim.x) { S.rep[x] = x; S.rsgn[x] = 1; }
  for (int y = tid; y < m; y += blockDim.x) S.calive[y] = 1;
  if (tid == 0) S.info[2] = mode;
  __syncthreads();
  const bool marg = (mode == MODE_MARG), ld = (mode == MODE_LD);
  const int r0 = marg ? 1 : 0, c0 = marg ? 1 : 0;
  for (int iter = 0; iter < 4 * (n + m) + 8; ++iter) {
    // ---- find ONE applicable rule (thread 0), then apply it with the whole block
    if (tid == 0) {
      act = 0;
      for (int x = r0; x < n && !act; ++x) {                     // zero row
        if (!row_alive(S, x)) continue;
        bool z = true;
        for (int j = 0; j < m && z; ++j) z = !(S.calive[j] && S.A[(int64_t)x * m + j] != 0);
        if (z) { act = 1; a1 = x; }
      }
      for (int y = c0; y < m && !act; ++y) {                     // zero column
        if (!S.calive[y]) continue;
        bool z = true;
        for (int i = 0; i < n && z; ++i) z = !(row_alive(S, i) && S.A[(int64_t)i * m + y] != 0);
        if (z) { act = 2; a1 = y; }
      }
      for (int u = r0; u < n && !act; ++u) {                     // proportional rows
        if (!row_alive(S, u)) continue;
        for (int v = u + 1; v < n && !act; ++v) {
          if (!row_alive(S, v)) continue;
          const int s = prop_rows(S, n, m, u, v, 0);
          if (s != 0 && (!ld || s > 0)) { act = 3; a1 = u; a2 = v; sg = s; }
        }
      }
      for (int u = c0; u < m && !act; ++u) {                     // proportional columns
        if (!S.calive[u]) continue;
        for (int v = u + 1; v < m && !act; ++v) {
          if (!S.calive[v]) continue;
          const int s = prop_cols(S, n, m, u, v, 0);
          if (s != 0) { act = 4; a1 = u; a2 = v; sg = s; }
        }
      }
      if (ld) {                                                  // sign-uniform column pair
        int first = -1;
        for (int y = 0; y < m && !act; ++y) {
          if (!S.calive[y] || col_sign(S, n, m, y) == 0) continue;
          if (first < 0) first = y;
          else { act = 5; a1 = first; a2 = y; }
        }
      }
      if (!act && marg) {                                        // row 0 and column 0 both zero -> L_1
        bool z = true;
        for (int j = 0; j < m && z; ++j) z = !(S.calive[j] && S.A[j] != 0);
        for (int i = 0; i < n && z; ++i) z = !(row_alive(S, i) && S.A[(int64_t)i * m] != 0);
        if (z && n > 1 && m > 1 && S.rep[0] == 0 && S.calive[0]) act = 6;
      }
    }
    __syncthreads();
    const int a = act;
    if (a == 0) break;
    if (a == 1) { if (tid == 0) S.rep[a1] = -1; }
    else if (a == 2) { if (tid == 0) S.calive[a1] = 0; }
    else if (a == 3) {
      for (int j = tid; j < m; j += blockDim.x) S.A[(int64_t)a1 * m + j] += sg * S.A[(int64_t)a2 * m + j];
      if (tid == 0) { S.rep[a2] = a1; S.rsgn[a2] = sg; }
    } else if (a == 4) {
      for (int i = tid; i < n; i += blockDim.x) S.A[(int64_t)i * m + a1] += sg * S.A[(int64_t)i * m + a2];
      if (tid == 0) S.calive[a2] = 0;
    } else if (a == 5) {
      for (int i = tid; i < n; i += blockDim.x)
        S.A[(int64_t)i * m + a1] = abs(S.A[(int64_t)i * m + a1]) + abs(S.A[(int64_t)i * m + a2]);
      if (tid == 0) S.calive[a2] = 0;
    } else if (a == 6) {
      // L_marg with zero first row and column: solve L_1 of the rest;
      // row 0 keeps a_0 = +1 in the map-back (rep = -1 maps to +1)
      if (tid == 0) { S.rep[0] = -1; S.calive[0] = 0; S.info[2] = MODE_L1; }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    int nn = 0, mm = 0;
    for (int x = 0; x < n; ++x) nn += row_alive(S, x);
    for (int y = 0; y < m; ++y) mm += S.calive[y];
    S.info[0] = nn;
    S.info[1] = mm;
  }
}

// Compact the alive rows / columns into R (n' x m'); rowsel[i] = original row of reduced row i.
__global__ void compact_kernel(int n, int m, RedState S, int32_t* R, int32_t* rowsel) {
  __shared__ int rows[kMaxRows * 16], cols[kMaxCols];
  __shared__ int nn, mm;
  if (threadIdx.x == 0) {
    nn = 0; mm = 0;
    for (int x = 0; x < n; ++x) if (row_alive(S, x)) rows[nn++] = x;
    for (int y = 0; y < m; ++y) if (S.calive[y]) cols[mm++] = y;
    for (int i = 0; i < nn; ++i) rowsel[i] = rows[i];
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < (int64_t)nn * mm; t += blockDim.x) {
    const int i = (int)(t / mm), j = (int)(t % mm);
    R[t] = S.A[(int64_t)rows[i] * m + cols[j]];
  }
}

// Expand the reduced argmax (int8 over reduced rows, at argr) to the original rows.
__global__ void mapback_kernel(int n, int nred, int ld, RedState S, const int32_t* rowsel, const int8_t* argr,
                               int8_t* out) {
  if (threadIdx.x != 0) return;
  int8_t val[1024];
  for (int x = 0; x < n && x < 1024; ++x) val[x] = ld ? 0 : 1;
  for (int i = 0; i < nred; ++i) val[rowsel[i]] = argr[i];
  for (int x = 0; x < n; ++x) {
    // follow the representative chain to an alive row (or a removed zero row)
    int y = x, sgn = 1;
    while (y >= 0 && S.rep[y] != y) { sgn *= S.rsgn[y]; y = S.rep[y]; }
    if (y < 0) out[x] = ld ? 0 : 1;                 // removed zero row: any value attains
    else out[x] = ld ? val[y] : (int8_t)(sgn * val[y]);
  }
}

}  // namespace

size_t reduce_scratch_ints(int n, int m) { return (size_t)n * m + 2 * (size_t)n + (size_t)m + 8; }

cudaError_t reduce_launch(const int32_t* M, int n, int m, int mode, int32_t* scratch, int32_t* R, int32_t* rowsel,
                          int32_t* info_dev, cudaStream_t st) {
  RedState S;
  S.A = scratch;
  S.rep = S.A + (size_t)n * m;
  S.rsgn = S.rep + n;
  S.calive = S.rsgn + n;
  S.info = info_dev;
  reduce_kernel<<<1, kRedThreads, 0, st>>>(M, n, m, mode, S);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  compact_kernel<<<1, kRedThreads, 0, st>>>(n, m, S, R, rowsel);
  return cudaGetLastError();
}

cudaError_t mapback_launch(int n, int m, int nred, int ld, int32_t* scratch, const int32_t* rowsel,
                           const int8_t* argr, int8_t* out, int32_t* info_dev, cudaStream_t st) {
  RedState S;
  S.A = scratch;
  S.rep = S.A + (size_t)n * m;
  S.rsgn = S.rep + n;
  S.calive = S.rsgn + n;
  S.info = info_dev;
  mapback_kernel<<<1, 32, 0, st>>>(n, nred, ld, S, rowsel, argr, out);
  return cudaGetLastError();
}

}  // namespace lnorm
