// Strategy-paired packed binary walk kernels, mode marg (see walk_pair16_impl.cuh).
#define LN_BIN_MODE 1
#include "walk_pair16_impl.cuh"
