// Byte-packed binary walk kernels, mode l1 (see walk_u8_impl.cuh).
#define LN_BIN_MODE 0
#include "walk_u8_impl.cuh"
