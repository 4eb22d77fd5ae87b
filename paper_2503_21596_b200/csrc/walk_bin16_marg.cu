// Packed 16-bit binary walk kernels, mode marg (see walk_bin16_impl.cuh).
#define LN_BIN_MODE 1
#include "walk_bin16_impl.cuh"
