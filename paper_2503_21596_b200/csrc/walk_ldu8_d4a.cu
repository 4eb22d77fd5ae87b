// Byte-packed d-ary walk kernels, d = 4, 1-6 packed words (see walk_ldu8_impl.cuh).
#define LN_LDU8_D 4
#define LN_LDU8_PART 0
#include "walk_ldu8_impl.cuh"
