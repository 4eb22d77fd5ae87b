// Reflected Gray codes (binary and d-ary), host + device.
//
// PAPER.md:177-181 Eq. (8)   G_{i,j} = floor((j + 2^i) / 2^(i+1)) mod 2  (binary reflected, BRGC)
// PAPER.md:216-221 Eq. (9)   changed digit of word j: the i with j / 2^i odd  (= ctz(j))
// PAPER.md:286-291 Eqs. (13)-(15)  S = (0..d-1, d-1..0), I = floor(j / d^i) mod 2d, G = S[I]
// PAPER.md:301-305 Eq. (17)  changed digit = min{ i : floor(j / d^i) mod d != 0 }
//
// Digit i is least significant first (Tables 1 and 3 list i bottom-up).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define LN_HD __host__ __device__ __forceinline__
#else
#define LN_HD inline
#endif

namespace lnorm {

// Eq. (8): digit i of BRGC word j, with shifts only.
LN_HD uint32_t brgc_digit(uint32_t i, uint64_t j) {
  return (uint32_t)(((j + (1ull << i)) >> (i + 1)) & 1ull);
}

// Eq. (9): digit that changes between words j-1 and j (j >= 1).
LN_HD uint32_t brgc_change(uint64_t j) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)(__ffsll((long long)j) - 1);
#else
  return (uint32_t)__builtin_ctzll(j);
#endif
}

// Eqs. (13)-(15): digit i of word j of the d-ary reflected Gray code.
LN_HD uint32_t dary_digit(uint32_t d, uint32_t i, uint64_t j) {
  uint64_t q = j;
  for (uint32_t k = 0; k < i; ++k) q /= d;
  uint32_t I = (uint32_t)(q % (2ull * d));
  return I < d ? I : 2u * d - 1u - I;           // S = (0,1,..,d-1,d-1,..,1,0)
}

// Eq. (17): digit that changes between words j-1 and j (j >= 1).
LN_HD uint32_t dary_change(uint32_t d, uint64_t j) {
  uint32_t i = 0;
  while (j % d == 0) { j /= d; ++i; }
  return i;
}

// Old and new value of the changed digit between words j-1 and j.
LN_HD void dary_change_values(uint32_t d, uint64_t j, uint32_t* i, uint32_t* from, uint32_t* to) {
  uint32_t ci = dary_change(d, j);
  *i = ci;
  *from = dary_digit(d, ci, j - 1);
  *to = dary_digit(d, ci, j);
}

// Block-start step of a d-ary walk whose lowest digit is unrolled: word w = t*d
// (t >= 1, 32-bit).  The changed digit is 1 + (number of trailing zero base-d digits
// of t) (Eq. 17) and, with tt = t / d^ip, the old/new values are S[(tt-1) mod 2d] and
// S[tt mod 2d] (Eqs. 13-15: floor((w-1)/d^i) = tt - 1 because w = tt d^i).
template <int D>
LN_HD void dary_block_start(uint32_t t, uint32_t* i, uint32_t* from, uint32_t* to) {
  uint32_t tt = t, ip = 0;
  while (tt % D == 0) { tt /= D; ++ip; }
  const uint32_t a = (tt - 1) % (2 * D), b = tt % (2 * D);
  *i = 1 + ip;
  *from = a < D ? a : 2 * D - 1 - a;
  *to = b < D ? b : 2 * D - 1 - b;
}

// Lexicographic key of a suffix word: digit i of the Gray word <-> row n-1-i,
// so with the suffix's first row most significant the key is sum_i G_i d^i.
// For d = 2 this is the Gray word itself: j ^ (j >> 1).
LN_HD uint64_t brgc_word(uint64_t j) { return j ^ (j >> 1); }

}  // namespace lnorm
