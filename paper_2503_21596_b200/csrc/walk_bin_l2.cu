// Binary walk kernels, mode l2 (see walk_bin_impl.cuh).
#define LN_BIN_MODE 2
#include "walk_bin_impl.cuh"
