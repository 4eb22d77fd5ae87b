// Strategy-paired packed binary walk kernels, mode l2 (see walk_pair16_impl.cuh).
#define LN_BIN_MODE 2
#include "walk_pair16_impl.cuh"
