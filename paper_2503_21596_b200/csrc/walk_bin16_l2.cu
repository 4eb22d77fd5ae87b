// Packed 16-bit binary walk kernels, mode l2 (see walk_bin16_impl.cuh).
#define LN_BIN_MODE 2
#include "walk_bin16_impl.cuh"
