// Packed 16-bit binary walk kernels, mode l1 (see walk_bin16_impl.cuh).
#define LN_BIN_MODE 0
#include "walk_bin16_impl.cuh"
