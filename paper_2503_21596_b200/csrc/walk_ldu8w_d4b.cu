// Byte-packed L_4 walk with 3-4 paired rows in the all-H form, 7-12 packed words (walk_ldu8w_impl.cuh).
#define LN_LDU8W_D 4
#define LN_LDU8W_PART 1
#include "walk_ldu8w_impl.cuh"
