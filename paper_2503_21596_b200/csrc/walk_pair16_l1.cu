// Strategy-paired packed binary walk kernels, mode l1 (see walk_pair16_impl.cuh).
#define LN_BIN_MODE 0
#include "walk_pair16_impl.cuh"
