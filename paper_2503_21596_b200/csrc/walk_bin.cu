// Dispatch for the hot binary walk (kernels in walk_bin_impl.cuh, one TU per mode).
#include "common.cuh"

namespace lnorm {

namespace {
constexpr int padC(int c) { return (c + 3) & ~3; }
}

bool walk_bin_supported(int mode, int c, int s) {
  return (mode == MODE_L1 || mode == MODE_MARG || mode == MODE_LD) && c >= 1 && padC(c) <= 64 && s >= 4;
}

int walk_bin_occupancy(int mode, int c, int* block_out) {
  *block_out = 32;
  if (mode == MODE_L1) return walk_bin_occupancy_mode<MODE_L1>(c);
  if (mode == MODE_MARG) return walk_bin_occupancy_mode<MODE_MARG>(c);
  return walk_bin_occupancy_mode<MODE_LD>(c);
}

cudaError_t walk_bin_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st, int* block_out) {
  *block_out = 32;
  if (p.mode == MODE_L1) return walk_bin_launch_mode<MODE_L1>(p, scratch_tab, grid, st);
  if (p.mode == MODE_MARG) return walk_bin_launch_mode<MODE_MARG>(p, scratch_tab, grid, st);
  return walk_bin_launch_mode<MODE_LD>(p, scratch_tab, grid, st);
}

bool walk_bin16_supported(int mode, int c, int s) {
  if (s < 4) return false;
  if (mode == MODE_L1) return walk_bin16_words<MODE_L1>(c) > 0;
  if (mode == MODE_MARG) return c >= 2 && walk_bin16_words<MODE_MARG>(c) > 0;
  if (mode == MODE_LD) return walk_bin16_words<MODE_LD>(c) > 0;
  return false;
}

int walk_bin16_occupancy(int mode, int c, int k, int s, int* block_out) {
  *block_out = 32;
  if (mode == MODE_L1) return walk_bin16_occupancy_mode<MODE_L1>(c, k, s);
  if (mode == MODE_MARG) return walk_bin16_occupancy_mode<MODE_MARG>(c, k, s);
  return walk_bin16_occupancy_mode<MODE_LD>(c, k, s);
}

int walk_bin16_units_per_lane(int mode, int c) {
  if (mode == MODE_L1) return walk_bin16_units_per_lane_mode<MODE_L1>(c);
  if (mode == MODE_MARG) return walk_bin16_units_per_lane_mode<MODE_MARG>(c);
  return walk_bin16_units_per_lane_mode<MODE_LD>(c);
}

cudaError_t walk_bin16_launch(const WalkParams& p, int32_t* scratch_tab, int grid, cudaStream_t st, int* block_out) {
  *block_out = 32;
  if (p.mode == MODE_L1) return walk_bin16_launch_mode<MODE_L1>(p, scratch_tab, grid, st);
  if (p.mode == MODE_MARG) return walk_bin16_launch_mode<MODE_MARG>(p, scratch_tab, grid, st);
  return walk_bin16_launch_mode<MODE_LD>(p, scratch_tab, grid, st);
}

}  // namespace lnorm
