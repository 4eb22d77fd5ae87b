/*
 * lnorm_oracle.c -- naive CPU oracle for the L_1, L_marg and L_d norms of
 * arXiv 2503.21596.  TEST INFRASTRUCTURE ONLY: nothing in the
 * product path (paper_2503_21596_b200/, include/) may include, link or call
 * this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.
 *
 * What it computes is the plain definition of each norm, enumerated with a
 * plain counter -- no Gray codes, no incremental updates, no symmetry
 * reduction beyond the optional "fix row 0" flag, no relabelling canonical
 * forms.  Every strategy's value is recomputed from scratch in int64
 * (the paper's "naive" n*m-per-strategy cost).
 *
 *   L_1    (Eq. 1):
 *     max over a in {+1,-1}^n of  sum_y | sum_x M_xy a_x |
 *   L_marg (Eq. 2):
 *     max over a with a_0 = +1 of sum_x M_x0 a_x + sum_{y>=1} | sum_x M_xy a_x |
 *   L_d, d >= 2 (Eqs. 6-7):
 *     max over a in {0..d-1}^n of sum_{g=0}^{d-1} sum_y | sum_{x: a_x = g} M_xy |
 *
 * Enumeration order / tie rule (reading R2): the counter runs
 * 0,1,2,... with row 0 the MOST significant digit; for +-1 strategies digit 1
 * means a_x = -1 (so +1 ranks before -1).  The oracle keeps the FIRST strict
 * maximum, i.e. the lexicographically smallest optimal strategy.
 *
 * Parity status: every entry point below is pinned by tests/test_oracle.py
 * (paper worked examples, closed forms, brute-force second opinions written
 * independently in tests/brute.py, invariances and norm-chain identities).
 *
 * Threading: OpenMP parallel-for over contiguous counter blocks; per-thread
 * (best, first index) merged in block order so the result is independent of
 * the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_MAX_ROWS 64
#define ORACLE_MAX_COLS 4096

static int64_t iabs64(int64_t v) { return v < 0 ? -v : v; }

/* Value of one +-1 strategy a (entries +1/-1), Eq. (1) or Eq. (2). */
static int64_t value_pm(const int32_t* M, int n, int m, const int8_t* a, int marg) {
  int64_t v = 0;
  for (int y = 0; y < m; ++y) {
    int64_t s = 0;
    for (int x = 0; x < n; ++x) s += (int64_t)a[x] * (int64_t)M[(int64_t)x * m + y];
    if (marg && y == 0) v += s;          /* Eq. (2): first column enters signed */
    else v += iabs64(s);
  }
  return v;
}

/* Value of one labelling a (entries 0..d-1), Eqs. (6)-(7). */
static int64_t value_ld(const int32_t* M, int n, int m, int d, const int8_t* a) {
  int64_t v = 0;
  for (int g = 0; g < d; ++g) {
    for (int y = 0; y < m; ++y) {
      int64_t s = 0;                      /* (m_g)_y = sum_{x: a_x = g} M_xy */
      for (int x = 0; x < n; ++x)
        if (a[x] == g) s += (int64_t)M[(int64_t)x * m + y];
      v += iabs64(s);
    }
  }
  return v;
}

/* Decode counter c into strategy digits, row 0 most significant.
 * first_row: rows < first_row are left untouched (caller-fixed). */
static void decode(uint64_t c, int n, int base, int first_row, int8_t* dig) {
  for (int x = n - 1; x >= first_row; --x) {
    dig[x] = (int8_t)(c % (uint64_t)base);
    c /= (uint64_t)base;
  }
}

static void digits_to_pm(const int8_t* dig, int n, int8_t* a) {
  for (int x = 0; x < n; ++x) a[x] = dig[x] ? (int8_t)-1 : (int8_t)1;
}

/*
 * Core enumerator.  mode: 0 = L_1, 1 = L_marg, 2 = L_d.
 * The first `nfixed` rows are fixed to `fixed[0..nfixed-1]` (digit values:
 * 0/1 for +-1 strategies meaning +1/-1, labels for L_d); the remaining
 * n - nfixed rows are enumerated over the counter range [c_begin, c_end)
 * (c_end = base^(n-nfixed) for the full space).
 * Returns 0 on success, -1 on bad arguments.  *best / best_dig receive the
 * first strict maximum in counter order (the whole row vector, digits).
 */
static int enumerate(const int32_t* M, int n, int m, int mode, int d,
                     int nfixed, const int8_t* fixed,
                     uint64_t c_begin, uint64_t c_end,
                     int64_t* best, int8_t* best_dig, int nthreads) {
  if (!M || n < 1 || m < 1 || n > ORACLE_MAX_ROWS || m > ORACLE_MAX_COLS) return -1;
  if (nfixed < 0 || nfixed > n || (nfixed > 0 && !fixed)) return -1;
  if (c_end <= c_begin) return -1;
  const int base = (mode == 2) ? d : 2;
  const int marg = (mode == 1);
#ifdef _OPENMP
  int T = nthreads > 0 ? nthreads : omp_get_max_threads();
#else
  int T = 1; (void)nthreads;
#endif
  uint64_t total = c_end - c_begin;
  if ((uint64_t)T > total) T = (int)total;
  int64_t* tbest = (int64_t*)malloc(sizeof(int64_t) * T);
  uint64_t* targ = (uint64_t*)malloc(sizeof(uint64_t) * T);
  int* tset = (int*)calloc(T, sizeof(int));
  if (!tbest || !targ || !tset) { free(tbest); free(targ); free(tset); return -1; }
#ifdef _OPENMP
#pragma omp parallel num_threads(T)
#endif
  {
#ifdef _OPENMP
    const int t = omp_get_thread_num();
#else
    const int t = 0;
#endif
    /* contiguous block t of the counter range */
    const uint64_t lo = c_begin + total / T * t + ((uint64_t)t < total % T ? (uint64_t)t : total % T);
    const uint64_t hi = lo + total / T + ((uint64_t)t < total % T ? 1 : 0);
    int8_t dig[ORACLE_MAX_ROWS], a[ORACLE_MAX_ROWS];
    for (int x = 0; x < nfixed; ++x) dig[x] = fixed[x];
    int64_t b = 0; uint64_t ba = 0; int have = 0;
    for (uint64_t c = lo; c < hi; ++c) {
      decode(c, n, base, nfixed, dig);
      int64_t v;
      if (mode == 2) v = value_ld(M, n, m, d, dig);
      else { digits_to_pm(dig, n, a); v = value_pm(M, n, m, a, marg); }
      if (!have || v > b) { b = v; ba = c; have = 1; }   /* first strict maximum */
    }
    tbest[t] = b; targ[t] = ba; tset[t] = have;
  }
  int64_t B = 0; uint64_t A = 0; int have = 0;
  for (int t = 0; t < T; ++t)                 /* merge in block order */
    if (tset[t] && (!have || tbest[t] > B)) { B = tbest[t]; A = targ[t]; have = 1; }
  free(tbest); free(targ); free(tset);
  if (!have) return -1;
  *best = B;
  if (best_dig) {
    for (int x = 0; x < nfixed; ++x) best_dig[x] = fixed[x];
    decode(A, n, base, nfixed, best_dig);
  }
  return 0;
}

static uint64_t ipow_sat(int base, int e) {
  uint64_t r = 1;
  for (int i = 0; i < e; ++i) {
    if (r > UINT64_MAX / (uint64_t)base) return 0;   /* overflow -> 0 = unsupported */
    r *= (uint64_t)base;
  }
  return r;
}

/* ------------------------------------------------------------------ API -- */

/* Value of one +-1 strategy (entries must be +1/-1); marg selects Eq. (2). */
int64_t oracle_value_pm(const int32_t* M, int n, int m, const int8_t* a, int marg) {
  return value_pm(M, n, m, a, marg);
}

/* Value of one labelling (entries 0..d-1), Eq. (6). */
int64_t oracle_value_ld(const int32_t* M, int n, int m, int d, const int8_t* a) {
  return value_ld(M, n, m, d, a);
}

/*
 * L_1 (Eq. 1).  fix_first = 0: all 2^n strategies; 1: a_0 = +1 only
 * (the +-a symmetry of PAPER.md:147).  argmax: int8[n] of +-1, may be NULL.
 */
int oracle_l1(const int32_t* M, int n, int m, int fix_first, int nthreads,
              int64_t* value, int8_t* argmax) {
  int8_t dig[ORACLE_MAX_ROWS], fx = 0;
  if (n > 63) return -1;
  int nf = fix_first ? 1 : 0;
  uint64_t cnt = ipow_sat(2, n - nf);
  if (!cnt) return -1;
  int rc = enumerate(M, n, m, 0, 2, nf, &fx, 0, cnt, value, dig, nthreads);
  if (rc == 0 && argmax) digits_to_pm(dig, n, argmax);
  return rc;
}

/* L_marg (Eq. 2): a_0 = +1 by definition; rows 1..n-1 enumerated. */
int oracle_marg(const int32_t* M, int n, int m, int nthreads, int64_t* value, int8_t* argmax) {
  int8_t dig[ORACLE_MAX_ROWS], fx = 0;
  if (n > 64) return -1;
  uint64_t cnt = ipow_sat(2, n - 1);
  if (!cnt) return -1;
  int rc = enumerate(M, n, m, 1, 2, 1, &fx, 0, cnt, value, dig, nthreads);
  if (rc == 0 && argmax) digits_to_pm(dig, n, argmax);
  return rc;
}

/*
 * L_d, d >= 2 (Eq. 6).  fix_first = 0: all d^n labellings; 1: a_0 = 0
 * (the relabelling symmetry of PAPER.md:284).  argmax: int8[n] labels.
 */
int oracle_ld(const int32_t* M, int n, int m, int d, int fix_first, int nthreads,
              int64_t* value, int8_t* argmax) {
  int8_t dig[ORACLE_MAX_ROWS], fx = 0;
  if (d < 2 || d > 127) return -1;
  int nf = fix_first ? 1 : 0;
  uint64_t cnt = ipow_sat(d, n - nf);
  if (!cnt) return -1;
  int rc = enumerate(M, n, m, 2, d, nf, &fx, 0, cnt, value, dig, nthreads);
  if (rc == 0 && argmax) memcpy(argmax, dig, (size_t)n);
  return rc;
}

/*
 * Restricted maximum: rows 0..nfixed-1 fixed to `fixed` (digits: 0/1 = +1/-1
 * for mode 0/1, labels for mode 2), the rest enumerated in full.  This is the
 * plain definition of "the best strategy that starts with this prefix" and is
 * what sampled-parity tests compare the GPU's per-prefix maxima against.
 * mode: 0 = L_1, 1 = L_marg (fixed[0] must be 0, i.e. a_0 = +1), 2 = L_d.
 * argmax_digits may be NULL.
 */
int oracle_prefix_max(const int32_t* M, int n, int m, int mode, int d,
                      int nfixed, const int8_t* fixed, int nthreads,
                      int64_t* value, int8_t* argmax_digits) {
  int base = (mode == 2) ? d : 2;
  if (mode < 0 || mode > 2 || nfixed < 1 || nfixed > n) return -1;
  if (mode == 1 && fixed[0] != 0) return -1;
  if (nfixed == n) {
    int8_t a[ORACLE_MAX_ROWS];
    if (mode == 2) *value = value_ld(M, n, m, d, fixed);
    else { digits_to_pm(fixed, n, a); *value = value_pm(M, n, m, a, mode == 1); }
    if (argmax_digits) memcpy(argmax_digits, fixed, (size_t)n);
    return 0;
  }
  uint64_t cnt = ipow_sat(base, n - nfixed);
  if (!cnt) return -1;
  return enumerate(M, n, m, mode, d, nfixed, fixed, 0, cnt, value, argmax_digits, nthreads);
}

/*
 * Bounded sample for CPU timing (bench.py cpu_baseline): enumerate counter
 * values [c_begin, c_end) of the a_0-fixed space (mode 0/1: 2^(n-1) counter,
 * mode 2: d^(n-1)), from scratch.  Returns the sample's max.
 */
int oracle_sample(const int32_t* M, int n, int m, int mode, int d,
                  uint64_t c_begin, uint64_t c_end, int nthreads, int64_t* value) {
  int8_t fx = 0, dig[ORACLE_MAX_ROWS];
  return enumerate(M, n, m, mode, mode == 2 ? d : 2, 1, &fx, c_begin, c_end, value, dig, nthreads);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
