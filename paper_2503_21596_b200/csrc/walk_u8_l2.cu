// Byte-packed binary walk kernels, mode l2 (see walk_u8_impl.cuh).
#define LN_BIN_MODE 2
#include "walk_u8_impl.cuh"
