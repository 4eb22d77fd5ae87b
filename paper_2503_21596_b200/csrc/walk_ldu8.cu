// Byte-packed d-ary walk: dispatch, exactness limits and the table builder (the kernels
// are instantiated in walk_ldu8_d{3,4}{a,b}.cu; see walk_ldu8_impl.cuh).
#include <algorithm>
#include <cstdlib>

#include "walk_ldu8_impl.cuh"

namespace lnorm {

namespace {
int part_of(int NW) { return NW <= 6 ? 0 : 1; }
// paired rows of the all-H kernel when the suffix allows (LNORM_LDU8W_PR caps it: A/B)
constexpr int kLdu8wMaxRows = 5;

// Paired rows of the all-H L_3 / L_4 kernel (walk_ldu8w_impl.cuh) for a unit of s suffix digits:
// 5 (L_3 only) when at least two walked digits remain, 4 with one, 3 at s = 4, else 0 (the all-E
// kernel runs).
// LNORM_LDU8W=0 disables it (A/B); LNORM_LDU8W_PR=3 or 4 caps the paired rows.
int ldu8w_rows(int d, int s) {
  if (d != 3 && d != 4) return 0;
  const char* em = getenv("LNORM_LDU8W");
  const char* ec = getenv("LNORM_LDU8W_PR");
  const int mode = (em && *em) ? atoi(em) : 1, cap = (ec && *ec) ? atoi(ec) : kLdu8wMaxRows;
  if (!mode) return 0;
  const int pr = (s >= 7 && d == 3) ? 5 : s >= 5 ? 4 : (s == 4 ? 3 : 0);
  return std::min(pr, cap) >= 3 ? std::min(pr, cap) : 0;
}
}  // namespace

int walk_ldu8_paired_rows(int d, int s) {
  const int wr = ldu8w_rows(d, s);
  return wr ? wr : ldu8_rows(s);
}

bool walk_ldu8_supported(int d, int c, int s) {
  if ((d != 3 && d != 4) || c < 1 || s < 2) return false;
  const int NW = words_of(c);
  if (NW > 12) return false;
  return (s - 1) * 2 * lu_pad4(NW) <= kTabWordsLU;
}

void walk_ldu8_table_sizes(int d, int c, int k, int s, int64_t* tab_words, int64_t* init_ints) {
  const int NW = words_of(c), pr = walk_ldu8_paired_rows(d, s);
  *tab_words = (int64_t)(s - pr) * 2 * lu_pad4(NW);
  *init_ints = (int64_t)(k + 3) * 4 * NW + (int64_t)NW * (1 << pr) + (1 << pr) + (int64_t)(k + 3) * NW;
}

int walk_ldu8_packed(int d, int c, int s) {
  const int NW = words_of(c), pt = part_of(NW);
  if (const int wr = ldu8w_rows(d, s)) {
    if (d == 4) return pt ? walk_ldu8w_pk_part<4, 1>(NW, wr) : walk_ldu8w_pk_part<4, 0>(NW, wr);
    return pt ? walk_ldu8w_pk_part<3, 1>(NW, wr) : walk_ldu8w_pk_part<3, 0>(NW, wr);
  }
  return 0;
}

int walk_ldu8_units_per_lane(int d, int c, int s) {
  const int NW = words_of(c), pt = part_of(NW);
  if (const int wr = ldu8w_rows(d, s)) {
    if (d == 4) return pt ? walk_ldu8w_upl_part<4, 1>(NW, wr) : walk_ldu8w_upl_part<4, 0>(NW, wr);
    return pt ? walk_ldu8w_upl_part<3, 1>(NW, wr) : walk_ldu8w_upl_part<3, 0>(NW, wr);
  }
  if (d == 3) return pt ? walk_ldu8_upl_part<3, 1>(NW, s) : walk_ldu8_upl_part<3, 0>(NW, s);
  if (d == 4) return pt ? walk_ldu8_upl_part<4, 1>(NW, s) : walk_ldu8_upl_part<4, 0>(NW, s);
  return 1;
}

int walk_ldu8_occupancy(int d, int c, int s, int* block_out) {
  *block_out = kBlockLU;
  const int NW = words_of(c), pt = part_of(NW);
  if (const int wr = ldu8w_rows(d, s)) {
    if (d == 4) return pt ? walk_ldu8w_occ_part<4, 1>(NW, wr, s) : walk_ldu8w_occ_part<4, 0>(NW, wr, s);
    return pt ? walk_ldu8w_occ_part<3, 1>(NW, wr, s) : walk_ldu8w_occ_part<3, 0>(NW, wr, s);
  }
  if (d == 3) return pt ? walk_ldu8_occ_part<3, 1>(NW, s) : walk_ldu8_occ_part<3, 0>(NW, s);
  if (d == 4) return pt ? walk_ldu8_occ_part<4, 1>(NW, s) : walk_ldu8_occ_part<4, 0>(NW, s);
  return 0;
}

cudaError_t walk_ldu8_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                             cudaStream_t st, int* block_out) {
  *block_out = kBlockLU;
  const int NW = words_of(p.c), pt = part_of(NW);
  const int wr = ldu8w_rows(p.d, p.s);
  const int pr = wr ? wr : ldu8_rows(p.s);
  if ((p.s - pr) * 2 * lu_pad4(NW) > kTabWordsLU || (p.k + 3) * 5 * NW + (NW + 1) * (1 << pr) > 16384)
    return cudaErrorInvalidValue;
  uint32_t* tab = reinterpret_cast<uint32_t*>(scratch_tab);
  build_ldu8_kernel<<<p.batch, 128, 0, st>>>(p.M, p.r, p.c, NW, p.k, p.s, pr, tab, scratch_init, p.m_stride,
                                             p.tab_stride, p.init_stride, p.chunk_ctr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (wr && p.d == 4) return pt ? walk_ldu8w_launch_part<4, 1>(p, tab, scratch_init, grid, st, NW, wr)
                                : walk_ldu8w_launch_part<4, 0>(p, tab, scratch_init, grid, st, NW, wr);
  if (wr) return pt ? walk_ldu8w_launch_part<3, 1>(p, tab, scratch_init, grid, st, NW, wr)
                    : walk_ldu8w_launch_part<3, 0>(p, tab, scratch_init, grid, st, NW, wr);
  if (p.d == 3) return pt ? walk_ldu8_launch_part<3, 1>(p, tab, scratch_init, grid, st, NW)
                          : walk_ldu8_launch_part<3, 0>(p, tab, scratch_init, grid, st, NW);
  if (p.d == 4) return pt ? walk_ldu8_launch_part<4, 1>(p, tab, scratch_init, grid, st, NW)
                          : walk_ldu8_launch_part<4, 0>(p, tab, scratch_init, grid, st, NW);
  return cudaErrorInvalidValue;
}

}  // namespace lnorm
