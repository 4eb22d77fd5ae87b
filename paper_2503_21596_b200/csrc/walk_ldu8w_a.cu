// Byte-packed L_3 walk with 3-5 paired rows in the all-H form, 1-6 packed words (walk_ldu8w_impl.cuh).
#define LN_LDU8W_D 3
#define LN_LDU8W_PART 0
#include "walk_ldu8w_impl.cuh"
