// Binary walk kernels, mode l1 (see walk_bin_impl.cuh).
#define LN_BIN_MODE 0
#include "walk_bin_impl.cuh"
