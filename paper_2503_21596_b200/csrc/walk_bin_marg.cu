// Binary walk kernels, mode marg (see walk_bin_impl.cuh).
#define LN_BIN_MODE 1
#include "walk_bin_impl.cuh"
