// Byte-packed d-ary walk: dispatch, exactness limits and the table builder (the kernels
// are instantiated in walk_ldu8_d{3,4}{a,b}.cu; see walk_ldu8_impl.cuh).
#include "walk_ldu8_impl.cuh"

namespace lnorm {

namespace {
int part_of(int NW) { return NW <= 6 ? 0 : 1; }
}  // namespace

bool walk_ldu8_supported(int d, int c, int s) {
  if ((d != 3 && d != 4) || c < 1 || s < 2) return false;
  const int NW = words_of(c);
  if (NW > 12) return false;
  return (s - 1) * 2 * lu_pad4(NW) <= kTabWordsLU;
}

int walk_ldu8_units_per_lane(int d, int c, int s) {
  const int NW = words_of(c), pt = part_of(NW);
  if (d == 3) return pt ? walk_ldu8_upl_part<3, 1>(NW, s) : walk_ldu8_upl_part<3, 0>(NW, s);
  if (d == 4) return pt ? walk_ldu8_upl_part<4, 1>(NW, s) : walk_ldu8_upl_part<4, 0>(NW, s);
  return 1;
}

int walk_ldu8_occupancy(int d, int c, int s, int* block_out) {
  *block_out = kBlockLU;
  const int NW = words_of(c), pt = part_of(NW);
  if (d == 3) return pt ? walk_ldu8_occ_part<3, 1>(NW, s) : walk_ldu8_occ_part<3, 0>(NW, s);
  if (d == 4) return pt ? walk_ldu8_occ_part<4, 1>(NW, s) : walk_ldu8_occ_part<4, 0>(NW, s);
  return 0;
}

cudaError_t walk_ldu8_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                             cudaStream_t st, int* block_out) {
  *block_out = kBlockLU;
  const int NW = words_of(p.c), pt = part_of(NW);
  const int pr = ldu8_rows(p.s);
  if ((p.s - pr) * 2 * lu_pad4(NW) > kTabWordsLU || (p.k + 3) * 4 * NW + (NW + 1) * (1 << pr) > 16384) return cudaErrorInvalidValue;
  uint32_t* tab = reinterpret_cast<uint32_t*>(scratch_tab);
  build_ldu8_kernel<<<1, 128, 0, st>>>(p.M, p.r, p.c, NW, p.k, p.s, pr, tab, scratch_init);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.d == 3) return pt ? walk_ldu8_launch_part<3, 1>(p, tab, scratch_init, grid, st, NW)
                          : walk_ldu8_launch_part<3, 0>(p, tab, scratch_init, grid, st, NW);
  if (p.d == 4) return pt ? walk_ldu8_launch_part<4, 1>(p, tab, scratch_init, grid, st, NW)
                          : walk_ldu8_launch_part<4, 0>(p, tab, scratch_init, grid, st, NW);
  return cudaErrorInvalidValue;
}

}  // namespace lnorm
