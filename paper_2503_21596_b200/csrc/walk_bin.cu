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
  if (mode == MODE_L1) return walk_bin16_words<MODE_L1>(c) > 0 && s >= walk_bin16_unroll_mode<MODE_L1>(c);
  if (mode == MODE_MARG)
    return c >= 2 && walk_bin16_words<MODE_MARG>(c) > 0 && s >= walk_bin16_unroll_mode<MODE_MARG>(c);
  if (mode == MODE_LD) return walk_bin16_words<MODE_LD>(c) > 0 && s >= walk_bin16_unroll_mode<MODE_LD>(c);
  return false;
}

bool walk_bin16_table_fits(int mode, int c, int k, int s) {
  int64_t w = 0;
  if (mode == MODE_L1) w = walk_bin16_table_words_mode<MODE_L1>(c, k, s);
  else if (mode == MODE_MARG) w = walk_bin16_table_words_mode<MODE_MARG>(c, k, s);
  else w = walk_bin16_table_words_mode<MODE_LD>(c, k, s);
  return w <= 16384;
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

bool walk_pair16_supported(int mode, int c, int s) {
  int C = 0, K = 4;
  if (mode == MODE_L1) { C = walk_pair16_cols<MODE_L1>(c); if (C) K = walk_pair16_unroll_mode<MODE_L1>(c); }
  else if (mode == MODE_MARG) { C = c >= 2 ? walk_pair16_cols<MODE_MARG>(c) : 0; if (C) K = walk_pair16_unroll_mode<MODE_MARG>(c); }
  else if (mode == MODE_LD) { C = walk_pair16_cols<MODE_LD>(c); if (C) K = walk_pair16_unroll_mode<MODE_LD>(c); }
  if (C == 0 || s < 1 + K) return false;   // one paired digit + K unrolled walked digits
  const int G = mode == MODE_LD ? 2 : 1;
  const int RW = (G * C + 1 + 3) & ~3;
  return 2 * (s - 1) * RW <= 8448;
}

void walk_pair16_table_sizes(int mode, int c, int k, int s, int64_t* tab_words, int64_t* init_ints) {
  if (mode == MODE_L1) walk_pair16_table_sizes_mode<MODE_L1>(c, k, s, tab_words, init_ints);
  else if (mode == MODE_MARG) walk_pair16_table_sizes_mode<MODE_MARG>(c, k, s, tab_words, init_ints);
  else walk_pair16_table_sizes_mode<MODE_LD>(c, k, s, tab_words, init_ints);
}

int walk_pair16_units_per_lane(int mode, int c) {
  if (mode == MODE_L1) return walk_pair16_units_per_lane_mode<MODE_L1>(c);
  if (mode == MODE_MARG) return walk_pair16_units_per_lane_mode<MODE_MARG>(c);
  return walk_pair16_units_per_lane_mode<MODE_LD>(c);
}

int walk_pair16_occupancy(int mode, int c, int s, int* block_out) {
  *block_out = 32;
  if (mode == MODE_L1) return walk_pair16_occupancy_mode<MODE_L1>(c, s);
  if (mode == MODE_MARG) return walk_pair16_occupancy_mode<MODE_MARG>(c, s);
  return walk_pair16_occupancy_mode<MODE_LD>(c, s);
}

cudaError_t walk_pair16_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                               cudaStream_t st, int* block_out) {
  *block_out = 32;
  if (p.mode == MODE_L1) return walk_pair16_launch_mode<MODE_L1>(p, scratch_tab, scratch_init, grid, st);
  if (p.mode == MODE_MARG) return walk_pair16_launch_mode<MODE_MARG>(p, scratch_tab, scratch_init, grid, st);
  return walk_pair16_launch_mode<MODE_LD>(p, scratch_tab, scratch_init, grid, st);
}

bool walk_u8_supported(int mode, int c, int s, int lpu) {
  int NW = 0, K = 4, PR = 1;
  if (mode == MODE_L1) { NW = walk_u8_words_mode<MODE_L1>(c); if (NW) K = walk_u8_unroll_mode<MODE_L1>(c, lpu); PR = walk_u8_paired_rows_mode<MODE_L1>(); }
  else if (mode == MODE_MARG) { NW = walk_u8_words_mode<MODE_MARG>(c); if (NW) K = walk_u8_unroll_mode<MODE_MARG>(c, lpu); PR = walk_u8_paired_rows_mode<MODE_MARG>(); }
  else if (mode == MODE_LD) { NW = walk_u8_words_mode<MODE_LD>(c); if (NW) K = walk_u8_unroll_mode<MODE_LD>(c, lpu); PR = walk_u8_paired_rows_mode<MODE_LD>(); }
  if (NW == 0 || s < K + PR || s > 31) return false;   // K unrolled digits + the paired last rows
  if (lpu > walk_u8_lanes_per_unit(mode, c)) return false;
  const int RW = 2 * (((NW + 1) / 2 + 3) & ~3);         // record words incl. lane-pair slice padding
  return 2 * s * RW <= 16384;
}

void walk_u8_table_sizes(int mode, int c, int k, int s, int lpu, int64_t* tab_words, int64_t* init_ints) {
  if (mode == MODE_L1) walk_u8_table_sizes_mode<MODE_L1>(c, k, s, lpu, tab_words, init_ints);
  else if (mode == MODE_MARG) walk_u8_table_sizes_mode<MODE_MARG>(c, k, s, lpu, tab_words, init_ints);
  else walk_u8_table_sizes_mode<MODE_LD>(c, k, s, lpu, tab_words, init_ints);
}

int walk_u8_words(int mode, int c) {
  if (mode == MODE_L1) return walk_u8_words_mode<MODE_L1>(c);
  if (mode == MODE_MARG) return walk_u8_words_mode<MODE_MARG>(c);
  return walk_u8_words_mode<MODE_LD>(c);
}

// largest lanes-per-unit an instance offers for c columns (1 or 2)
int walk_u8_lanes_per_unit(int mode, int c) {
  if (mode == MODE_L1) return walk_u8_lanes_per_unit_mode<MODE_L1>(c);
  if (mode == MODE_MARG) return walk_u8_lanes_per_unit_mode<MODE_MARG>(c);
  return walk_u8_lanes_per_unit_mode<MODE_LD>(c);
}

int walk_u8_units_per_lane(int mode, int c, int lpu) {
  if (mode == MODE_L1) return walk_u8_units_per_lane_mode<MODE_L1>(c, lpu);
  if (mode == MODE_MARG) return walk_u8_units_per_lane_mode<MODE_MARG>(c, lpu);
  return walk_u8_units_per_lane_mode<MODE_LD>(c, lpu);
}

int walk_u8_occupancy(int mode, int c, int s, int lpu, int* block_out) {
  *block_out = 32;
  if (mode == MODE_L1) return walk_u8_occupancy_mode<MODE_L1>(c, s, lpu);
  if (mode == MODE_MARG) return walk_u8_occupancy_mode<MODE_MARG>(c, s, lpu);
  return walk_u8_occupancy_mode<MODE_LD>(c, s, lpu);
}

cudaError_t walk_u8_launch(const WalkParams& p, int32_t* scratch_tab, int32_t* scratch_init, int grid,
                           cudaStream_t st, int* block_out) {
  *block_out = 32;
  if (p.mode == MODE_L1) return walk_u8_launch_mode<MODE_L1>(p, scratch_tab, scratch_init, grid, st);
  if (p.mode == MODE_MARG) return walk_u8_launch_mode<MODE_MARG>(p, scratch_tab, scratch_init, grid, st);
  return walk_u8_launch_mode<MODE_LD>(p, scratch_tab, scratch_init, grid, st);
}

}  // namespace lnorm
