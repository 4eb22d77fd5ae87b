// Byte-packed binary walk kernels, mode marg (see walk_u8_impl.cuh).
#define LN_BIN_MODE 1
#include "walk_u8_impl.cuh"
