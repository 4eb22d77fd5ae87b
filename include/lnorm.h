/*
 * lnorm.h -- C ABI of the B200-native exhaustive Gray-code search for the
 * L_1, L_marg and L_d norms of an integer matrix (arXiv 2503.21596).
 *
 * Citations are to /root/reference/PAPER.md lines ("P:n") as recorded in
 * DESIGN.md (the reference tree is not shipped).
 *
 *   L_1(M)    = max_{a in {+-1}^n}          sum_y | sum_x M_xy a_x |              P:58-61, Eq. (1)
 *   L_marg(M) = max_{a_0 = +1, a_x = +-1}   sum_x M_x0 a_x + sum_{y>=1} |sum_x M_xy a_x|   P:64-68, Eq. (2)
 *   L_d(M)    = max_{a in {0..d-1}^n}       sum_{g} sum_y | sum_{x: a_x = g} M_xy |  P:95-107, Eqs. (6)-(7)
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  M       caller-owned, read-only, row-major contiguous n*m int32 (host memory
 *          unless the name says _device).  Nothing is retained after return.
 *          Marginal layout (Eq. 2): column 0 is summed signed, row 0 is the
 *          strategy entry fixed to +1; M[0][0] is the constant term.
 *  d       d = 1 selects L_1 (L_1 is NOT L_d at d = 1); d >= 2 selects L_d.
 *          Supported: 1 <= d <= 8 (L_d for d > n equals L_n; handled exactly).
 *  with_marginals  0 or 1; 1 is legal only with d = 1 (selects L_marg).
 *  value   caller-allocated int64: the exact norm (may be negative for L_marg).
 *  argmax  caller-allocated int8[n] (may be NULL), in the input's row order:
 *          d = 1: entries +1/-1 with entry 0 = +1; d >= 2: labels 0..d-1 in
 *          restricted-growth form (entry 0 = 0, new labels appear in order).
 *          Canonical choice (R2): the lexicographically smallest
 *          optimal strategy (row 0 most significant, +1 before -1, labels in
 *          numeric order).  Exception (R6): for L_1/L_marg with
 *          n > m the search runs on M^T and argmax is x_i = sgn((M y*)_i)
 *          (sgn 0 = +1, then x_0 normalised to +1), which attains the value
 *          but need not be lexicographically smallest.
 *  Errors  every function returns an lnorm_status; on error the outputs are
 *          untouched.  LNORM_EINVAL: null pointer, n < 1, m < 1, d out of
 *          range, bad flag combination.  LNORM_EOVERFLOW: sum |M_ij| > 2^31-1
 *          (the int32 column sums and values could overflow; P:259 integer
 *          exactness).  LNORM_ETOOLARGE: the search space does not fit the
 *          64-bit word index (P:261 / P:336-340: more than 63 enumerated rows
 *          after orientation for d = 1, or d^(n-1) >= 2^63 for d >= 2), or the
 *          problem exceeds the kernels' column limit (m > 1024 after
 *          orientation).  LNORM_ENODEV / ECUDA / ENCCL / ENOMEM: runtime.
 *          LNORM_EINTERNAL: the always-on self-check of the argmax recovery
 *          failed (the re-walk of the winning unit did not reproduce the
 *          reduced maximum exactly: no strategy of the unit attains the key's
 *          value, or one exceeds it); value and argmax are then untouched.
 *  Threads re-entrant per device (an internal per-device context is guarded by
 *          a mutex); all calls synchronise before returning.
 *  Streams entry points taking `cuda_stream` (a cudaStream_t; NULL = the
 *          library's internal non-blocking stream) enqueue ALL their device
 *          work -- copies, kernels, the NCCL all-reduce -- on that stream, in
 *          stream order after whatever the caller enqueued before the call,
 *          and synchronise it before returning.  The other entry points use the
 *          internal stream.
 *
 * Every step of the search runs in the library's sm_100a kernels; there is no
 * CPU fallback (no device => LNORM_ENODEV).
 */
#ifndef LNORM_H
#define LNORM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LNORM_OK = 0,
  LNORM_EINVAL = 1,
  LNORM_EOVERFLOW = 2,
  LNORM_ETOOLARGE = 3,
  LNORM_ENODEV = 4,
  LNORM_ECUDA = 5,
  LNORM_ENCCL = 6,
  LNORM_ENOMEM = 7,
  LNORM_EINTERNAL = 8
} lnorm_status;

/* Human-readable name of a status code (static storage). */
const char* lnorm_status_string(int status);

/* ABI version: (major << 16) | minor. */
int32_t lnorm_version(void);

/*
 * Exact norm of M on the current CUDA device (per-worker maxima of the
 * Gray-code walk compared at the end).  Host buffers; the H2D copy of M, the
 * walk, the reduction and the argmax recovery all happen inside this call.
 */
int lnorm_compute(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                  int64_t* value, int8_t* argmax);

/*
 * Same as lnorm_compute but M is a DEVICE pointer on the current device
 * (row-major n*m int32, caller-owned, read-only) and the work is enqueued on
 * `cuda_stream` (see "Streams"), so a producer kernel enqueued earlier on the
 * same stream is complete before M is read.  Used to time the search with its
 * input already resident in HBM.  The exactness guards (sum |M|, per-column
 * window sums) are computed on the device by a one-block kernel; its ~0.5 KB
 * result is copied back on the same stream and synchronised, because the plan
 * (kernel family, prefix/suffix split) depends on them -- the only host round
 * trip before the walk.  Synchronises before return.
 */
int lnorm_compute_device(const int32_t* M_device, int32_t n, int32_t m, int32_t d,
                         int32_t with_marginals, void* cuda_stream,
                         int64_t* value, int8_t* argmax);

/*
 * One process, several GPUs (single-node, NVLink/NVSwitch): the unit range is
 * split across devices by Algorithm 1, every device walks its
 * slice, one ncclAllReduce(max) on an 8-byte key combines them and every
 * device recovers the same argmax.  device_ids: NULL = 0..num_devices-1.
 * Communicators are created and destroyed inside the call.
 */
int lnorm_compute_multi(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                        int32_t num_devices, const int32_t* device_ids,
                        int64_t* value, int8_t* argmax);

/*
 * One rank per GPU (torchrun): rank `rank` of `world` walks its
 * Algorithm-1 slice of the unit list, the 8-byte reduction key is
 * all-reduced with ncclMax on `cuda_stream` (no host round trip), and every
 * rank recovers and returns the same value and argmax (bit-identical).
 * nccl_comm: a caller-owned ncclComm_t of exactly `world` ranks whose rank
 * `rank` lives on the CURRENT CUDA device -- e.g. the communicator of a
 * torch.distributed NCCL process group, or one made by lnorm_comm_create.  The
 * library never destroys it.  nccl_comm == NULL is allowed only with world == 1
 * (no collective).  With a non-NULL comm the all-reduce runs even at world == 1.
 * M: host matrix (replicated on every rank); _device: M resident on the rank's
 * device (as lnorm_compute_device).  Errors after the slice walk started still
 * take part in the collective, so a failing rank never leaves its peers hanging.
 */
int lnorm_compute_rank(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                       void* nccl_comm, int32_t rank, int32_t world, void* cuda_stream,
                       int64_t* value, int8_t* argmax);
int lnorm_compute_rank_device(const int32_t* M_device, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                              void* nccl_comm, int32_t rank, int32_t world, void* cuda_stream,
                              int64_t* value, int8_t* argmax);

/*
 * A library-made NCCL communicator for callers without one.
 * lnorm_comm_unique_id writes a 128-byte ncclUniqueId (rank 0 calls it and
 * broadcasts the bytes, e.g. through torch.distributed); every rank then calls
 * lnorm_comm_create with its rank, the world size and its CUDA device
 * (ncclCommInitRank; a real communicator for every world >= 1 when `id` is
 * given; id == NULL is allowed only with world == 1 and yields a handle without
 * a communicator).  lnorm_comm_nccl returns the ncclComm_t (or NULL) to pass to
 * lnorm_compute_rank; the handle owns it until lnorm_comm_destroy.
 */
typedef struct lnorm_comm lnorm_comm;
int lnorm_comm_unique_id(uint8_t id_out[128]);
int lnorm_comm_create(const uint8_t id[128], int32_t rank, int32_t world, int32_t device,
                      lnorm_comm** comm_out);
int lnorm_comm_nccl(lnorm_comm* comm, void** nccl_comm_out);
int lnorm_comm_destroy(lnorm_comm* comm);

/*
 * Checkpoint / resume for long searches: the unit list is walked in
 * chunks of chunk_units (<= 0: one chunk) and after every chunk the state
 * (units done, best 8-byte key) is written atomically to `path` with a
 * fingerprint of the matrix and plan.  A later call with the same matrix and
 * path resumes from the saved state.  max_chunks (<= 0: unlimited) bounds the
 * chunks walked by this call.  *done = 1 when the search finished: value and
 * argmax are then final (bit-identical to lnorm_compute); otherwise value holds
 * the best value found so far (INT64_MIN if none) and argmax is untouched.
 * units_done (may be NULL) receives the number of units walked so far.
 */
int lnorm_compute_checkpointed(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                               const char* path, int64_t chunk_units, int32_t max_chunks, int64_t* value,
                               int8_t* argmax, int32_t* done, int64_t* units_done);

/*
 * Batched search (the inner oracle of see-saw / branch-and-bound
 * loops): `batch` matrices of the same shape, contiguous
 * (batch x n x m int32, host).  values: int64[batch]; argmax: int8[batch][n]
 * (may be NULL), same conventions as lnorm_compute.  One walk launch covers the
 * whole batch (units of all matrices in one grid, per-matrix keys, batched
 * recovery and finalisation): the strategy-paired packed kernel when every
 * matrix is within its guard (sum |M| <= 16383, d <= 2) and the shape has a
 * long enough suffix, else the generic warp-per-unit kernel (any d, any shape).
 * Any batch size (launches are chunked internally).
 */
int lnorm_compute_batch(const int32_t* M, int32_t batch, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                        int64_t* values, int8_t* argmax);

/*
 * Exact norm with the paper's norm-preserving reductions applied first
 * (App. A/B): zero rows/columns removed,
 * proportional rows (L_1, L_marg: any sign; L_d: positive factor only) and
 * proportional columns merged, sign-uniform columns merged for L_d, row 0 and
 * column 0 of L_marg exempt (both zero => L_1 of the rest).  The reduction runs
 * in single-block kernels; the reduced matrix is searched as by lnorm_compute
 * and the argmax is expanded back (merged row x'' = sgn(c) * its partner for
 * L_1 / L_marg, same label for L_d; removed zero rows get +1 / label 0).  The
 * value equals lnorm_compute's; the returned argmax attains it but need not be
 * the lexicographically smallest optimum.  reduced_shape (may be NULL)
 * receives {n', m'}.
 */
int lnorm_compute_reduced(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                          int64_t* value, int8_t* argmax, int32_t* reduced_shape);

/*
 * Test hook for the multi-GPU decomposition on ONE device: plans for `slices`
 * ranks, walks the Algorithm-1 slice of every virtual rank one after the other
 * into the same 8-byte key (what ncclAllReduce(max) combines across GPUs) and
 * recovers the argmax.  Results must be bit-identical to lnorm_compute.
 */
int lnorm_compute_sliced(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                         int32_t slices, int64_t* value, int8_t* argmax);

/*
 * Test hook for sampled parity at sizes the oracle cannot finish: for each of
 * `count` prefixes (int8[count][nfixed], row-major; digits 0/1 meaning +1/-1
 * for d = 1, labels 0..d-1 for d >= 2; for L_marg digit 0 of every prefix
 * must be 0) return in out[i] the maximum value over all strategies whose
 * rows 0..nfixed-1 equal prefix i and whose remaining rows are free.  No
 * orientation is applied.  Runs the same walk kernels as lnorm_compute: the
 * byte-packed kernel when the prefixes come in aligned groups of its lane group
 * (P = 4 consecutive prefixes equal on rows 0..nfixed-3 and running through the
 * four values of the last two rows, row nfixed-1 least significant), else a
 * per-unit kernel.  lnorm_last_stats then reports the kernel variant and walk time.
 * Requires 1 <= nfixed <= n.
 */
int lnorm_prefix_maxima(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                        int32_t nfixed, const int8_t* prefixes, int64_t count, int64_t* out);

/*
 * SURVEY 8(b)'s sampled-parity hook in unit coordinates: the per-unit maxima of
 * `count` units of the split with `prefix_digits` = k prefix rows beyond row 0
 * (unit prefix = rows 0..k).  units[i] indexes the lexicographically ordered
 * unit list lnorm_compute walks: for +-1 strategies and L_2 the digits of rows
 * 1..k are the bits of units[i] (row k least significant, bit 1 = -1 / label 1),
 * row 0 fixed; for d >= 3 units[i] is the index of the restricted-growth prefix
 * (length k+1, at most min(d, n) labels) in lexicographic order.  unit_max[i]
 * receives the maximum over all completions of unit i (no orientation: the
 * rows are the caller's).  Same kernels as lnorm_prefix_maxima.  EINVAL if a
 * unit index is out of range or k >= n.
 */
int lnorm_unit_maxima(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                      int32_t prefix_digits, const uint64_t* units, int64_t count, int32_t* unit_max);

/*
 * Test hook: the device walk of ONE unit, step by step.  Rows 0..nfixed-1 are
 * fixed to `prefix` (digits as above); the remaining s = n - nfixed rows are
 * walked in reflected Gray order (binary for d = 1 and d = 2, d-ary
 * otherwise; suffix digit i <-> row n-1-i) starting from all-zero digits.
 * values[w] receives the value after step w (w = 0 .. base^s - 1) and, if
 * digits is non-NULL, digits[w*n + x] the strategy digit of row x at step w.
 * base^s must be <= max_steps.
 */
int lnorm_walk_trace(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals,
                     int32_t nfixed, const int8_t* prefix, int64_t max_steps,
                     int64_t* values, int8_t* digits);

/*
 * Host-side reflected Gray-code helpers -- the same __host__ __device__ code the
 * kernels use.  lnorm_gray_digit: digit i of word j of the d-ary reflected
 * Gray code (d = 2: Eq. 8; d >= 2: Eqs. 13-15).
 * lnorm_gray_change: for j >= 1 the digit that differs between words j-1 and
 * j (Eq. 9 / Eq. 17) and its old/new values.
 */
int32_t lnorm_gray_digit(int32_t d, int32_t i, uint64_t j);
int lnorm_gray_change(int32_t d, uint64_t j, int32_t* digit, int32_t* from, int32_t* to);

/*
 * Algorithm 1: inclusive word range [j_min, j_max] of worker t out
 * of T over C words; an empty range has j_max = j_min - 1.
 */
int lnorm_partition(uint64_t C, int64_t T, int64_t t, int64_t* j_min, int64_t* j_max);

/*
 * The 8-byte reduction key every walk kernel, the grid-wide atomicMax and the
 * multi-rank ncclAllReduce(max) combine (the same __host__ __device__ code as
 * the kernels): high word = value with its sign bit flipped (unsigned order =
 * signed order, negative L_marg values included), low word = 0xFFFFFFFF - unit,
 * so the max over keys is the maximal value and, among equal values, the
 * SMALLEST unit -- the one holding the lexicographically smallest optimum
 * ("thread-wise maximal values are compared"; R2).
 * lnorm_key_decode inverts it.  Host-only, no device needed.
 */
uint64_t lnorm_reduction_key(int32_t value, uint32_t unit);
int lnorm_key_decode(uint64_t key, int32_t* value, uint32_t* unit);

/*
 * Host-only planning (no device needed): the orientation, unit split and
 * kernel family lnorm_compute would use for this input on `world` ranks.
 * variant: 0 int32 binary walk, 1 int32 d-ary walk, 2 generic warp-per-unit,
 * 3 packed-16 binary walk, 4 packed-16 d-ary walk, 5 strategy-paired packed-16
 * binary walk, 6 last-row-paired packed-16 d-ary walk, 7 byte-packed binary walk
 * (L_1, L_marg, L_2), 8 byte-packed d-ary walk (L_3, L_4).  The planner takes the
 * first exact family in the order 7/8 > 5/6 > 3/4 > 0/1 > 2; the environment
 * variable LNORM_KERNEL=auto|u8|pair16|packed|int32|generic starts that order at
 * the named family (tests, A/B timing).  units = 2^k for +-1
 * strategies and L_2, else the number of restricted-growth prefixes of
 * length k+1 with at most d labels.  Returns the same validation errors as
 * lnorm_compute.
 */
typedef struct {
  int32_t rows, cols, transposed, d_walked, prefix_digits, suffix_digits, variant, packed_ok;
  int64_t units;
  double steps;                /* strategies walked in total */
  int32_t lanes_per_unit;      /* byte-packed binary walk: 1, or 2 (lane pairs, > 128 columns) */
  int32_t words;               /* byte-packed binary walk: packed words per unit of the instance
                                  (columns / 4 rounded up to the instance; padding = 4 words - c) */
} lnorm_plan_info;
int lnorm_plan(const int32_t* M, int32_t n, int32_t m, int32_t d, int32_t with_marginals, int32_t world,
               lnorm_plan_info* out);

/*
 * SURVEY.md §8(f4) experiment -- the tcgen05 kind::i8 (integer tensor-core) formulation of
 * the L_1 search (Eq. 1), measured against the byte walk and NOT used by
 * lnorm_compute.  Strategies (row 0 fixed to +1) are numbered
 * (t, i, l): rows 1, 2 carry the two bits of i in [0, 4), rows 3..n-8 the bits of the
 * reflected Gray word t ^ (t >> 1), rows n-7..n-1 the bits of l in [0, 128)
 * (set bit = -1).  Tile t = all (i, l) = 512 strategies, whose column sums one tcgen05.mma
 * (M = 128, N = 4 * ceil4(m), K = 32, int8 x int8 -> int32 in TMEM) forms; the kernel covers
 * tiles [tile_begin, tile_begin + tile_count) of the 2^(n-10) tiles (tile_count = 0: all of
 * them, i.e. the exact L_1 of M with rows as given, no orientation).
 * M: host, row-major n x m int32, caller-owned.  Limits: 10 <= n <= 43, 1 <= m <= 64,
 * |M_xy| <= 127 on rows 1, 2 and the last 7 rows, sum over rows 0 and 3..n-8 of |M_xy| <= 508
 * per column (four int8 pieces), sum |M| < 2^21 (key layout): else LNORM_EINVAL /
 * ETOOLARGE / EOVERFLOW.
 * Outputs: value = the maximum over the covered strategies; argmax (int8[n], may be NULL)
 * = one strategy attaining it (not necessarily the lexicographically smallest);
 * strategies (may be NULL) = strategies covered; kernel_ms (may be NULL) = CUDA-event time
 * of the kernel.  Synchronises before return.
 */
int lnorm_imma_l1(const int32_t* M, int32_t n, int32_t m, uint64_t tile_begin, uint64_t tile_count,
                  int64_t* value, int8_t* argmax, uint64_t* strategies, double* kernel_ms);

/* Statistics of the last successful compute call on the calling thread. */
typedef struct {
  int32_t rows, cols;          /* enumerated rows / columns after orientation */
  int32_t transposed;          /* 1 if M^T was searched */
  int32_t prefix_digits;       /* k: rows 1..k form the unit prefix */
  int32_t suffix_digits;       /* s: rows k+1..r-1 are walked per unit */
  int32_t d;                   /* 1 (+-1 strategies) or the label count */
  int64_t units;               /* units in this call (this rank's slice for _rank) */
  int64_t units_total;         /* units over all ranks */
  double  steps;               /* Gray steps (strategies) walked by this call */
  double  column_updates;      /* algorithmic column updates (c per step, 2c for d >= 3) */
  double  walk_ms;             /* CUDA-event time of the walk kernel(s) */
  double  total_ms;            /* CUDA-event time from first H2D to last D2H */
  int32_t launches;            /* kernels launched by the call */
  int32_t variant;             /* kernel variant id */
  int32_t block_threads, grid_blocks;
  int32_t paired_rows;         /* packed kernels: last rows evaluated for all labels per walked word (0: none) */
  int32_t packed_units;        /* L_3 / L_4 byte walk: 2 if two units per lane share 16-bit packed sums, else 0 */
} lnorm_stats;
int lnorm_last_stats(lnorm_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* LNORM_H */
