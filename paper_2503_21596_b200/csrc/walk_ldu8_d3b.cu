// Byte-packed d-ary walk kernels, d = 3, 7-12 packed words (see walk_ldu8_impl.cuh).
#define LN_LDU8_D 3
#define LN_LDU8_PART 1
#include "walk_ldu8_impl.cuh"
