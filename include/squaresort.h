/*
 * squaresort.h -- C ABI of the B200-native SquareSort library (libsquaresort.so).
 *
 * SquareSort (arXiv 2407.14801) views n keys as an m x m column-major matrix,
 * m = ceil(sqrt(n)), sorts every column, samples
 * m-1 random pivots, computes the bucket positions
 * (P:283), moves every key into its bucket with SkewTranspose
 * (Alg 2/3) and sorts every bucket.  This library runs
 * each recursion level as batched sm_100a kernels on one B200.
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n; "L#" = a reading
 * of the paper listed in DESIGN.md section 3.
 *
 * Conventions (all entry points):
 *  - Data pointers of the sq_sort_* / sq_skew_transpose calls are caller-owned
 *    CUDA DEVICE memory (cudaMalloc or a torch CUDA tensor's data_ptr()),
 *    naturally aligned (4 B for u32, 8 B for u64); 16-byte alignment is not
 *    required.  The library never frees them or keeps them after return.
 *    The *_host variants take caller-owned HOST memory (pinned memory gives
 *    full copy bandwidth) and copy it to and from the device themselves.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *    enqueued on it; the call also blocks the host on it once per recursion
 *    level (a device->host read of the bucket sizes that plans the next
 *    level), and the result is complete when the call returns.
 *  - Scratch: up to 2n keys (+ 2n values when the multi-CTA merge base case
 *    runs, sq_set_big_bucket_mode 1) plus O(n / 32) metadata (the paper's O(n)
 *    extra space), allocated stream-ordered from a memory pool the
 *    library owns (one per device; the device's default pool is not touched)
 *    and freed into that pool before return.  The pool keeps freed scratch
 *    reserved so a repeated sort does not re-map it; sq_trim_memory() returns
 *    it to the system.
 *  - Repeated small sorts (n <= 2^22 by default, env SQ_GRAPH_MAX_N; default
 *    knobs): the second call with the same device, key/value pointers, n and
 *    seed captures the level's launches into a CUDA graph over scratch the
 *    library keeps for it (about 3n keys + metadata, at most 4 levels per key
 *    type), and later such calls replay it -- the result is the same sort of
 *    the buffer's current contents, with ~40 fewer host API calls.
 *    sq_trim_memory() drops those graphs and their scratch.
 *  - Errors are return codes only (sq_status); nothing is printed, no
 *    exception crosses the ABI.  sq_last_error_message() gives detail for the
 *    calling thread's last non-OK return.
 *  - n = 0 and n = 1 return SQ_OK without touching memory.
 *  - Limits: n <= 2^30 for u32 keys and pairs, n <= 2^28 for u64 keys (the
 *    pivot sample of m-1 keys is sorted on chip by one CTA).
 *  - The sorted keys do not depend on `seed` (the sorted order is unique);
 *    pairs are sorted stably (equal keys keep their input order, L16), so
 *    their output does not depend on `seed` either.  Only internal pivots do.
 *  - Concurrent calls on different streams with disjoint buffers are allowed.
 */
#ifndef SQUARESORT_H
#define SQUARESORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SQ_OK = 0,
  SQ_ERR_INVALID_ARGUMENT = 1,   /* NULL with n > 0, aliasing, size limits, bad params   */
  SQ_ERR_OUT_OF_MEMORY = 2,      /* scratch allocation failed                             */
  SQ_ERR_CUDA = 3,               /* a CUDA runtime call or kernel failed                  */
  SQ_ERR_PRECONDITION = 4,       /* SQ_FLAG_VALIDATE found unsorted columns / pivots      */
  SQ_ERR_UNSUPPORTED_DEVICE = 5  /* the current device is not sm_100 (B200)               */
} sq_status;

/* ------------------------------------------------------------------------- */
/* Sorting (Alg 1).  In place from the caller's view: keys[0..n)  */
/* (and vals) hold the ascending result on return.                           */
/* ------------------------------------------------------------------------- */

/* Sort n 32-bit unsigned keys ascending (unsigned order; L15). */
int sq_sort_u32(uint32_t *keys, size_t n, uint64_t seed, void *stream);

/* Sort n 64-bit unsigned keys ascending. */
int sq_sort_u64(uint64_t *keys, size_t n, uint64_t seed, void *stream);

/* Sort n (key, value) pairs by key, stably; vals[i] travels with keys[i].
 * keys and vals must not overlap. */
int sq_sort_pairs_u32_u32(uint32_t *keys, uint32_t *vals, size_t n, uint64_t seed, void *stream);

/* Sort n (u64 key, u32 value) pairs by key, stably (the paper's external-sort
 * workload is 64-bit integers); n <= 2^28.  keys and vals must not
 * overlap.  On chip the sorts order (key << 32 | position) 128-bit composites. */
int sq_sort_pairs_u64_u32(uint64_t *keys, uint32_t *vals, size_t n, uint64_t seed, void *stream);

/* Signed and IEEE-754 keys (the paper's workloads are signed
 * integers): an order-preserving bit map onto unsigned keys of the
 * same width (signed: flip the sign bit; float/double: flip all bits of a
 * negative value, the sign bit of a non-negative one), the unsigned sort, and the
 * inverse map, all on the device and in place.  Floats sort by IEEE 754-2008
 * totalOrder: -NaN < -inf < ... < -0.0 < +0.0 < ... < +inf < +NaN, NaN payloads
 * ordered by their bits (reading L25).  Limits and errors as the
 * unsigned calls of the same width. */
int sq_sort_i32(int32_t *keys, size_t n, uint64_t seed, void *stream);
int sq_sort_i64(int64_t *keys, size_t n, uint64_t seed, void *stream);
int sq_sort_f32(float *keys, size_t n, uint64_t seed, void *stream);
int sq_sort_f64(double *keys, size_t n, uint64_t seed, void *stream);

/* Same operations on HOST buffers: copy in, sort on the device, copy out,
 * synchronize.  The end-to-end path the bench's `e2e` figure measures. */
int sq_sort_u32_host(uint32_t *keys, size_t n, uint64_t seed, void *stream);
int sq_sort_u64_host(uint64_t *keys, size_t n, uint64_t seed, void *stream);
int sq_sort_pairs_u64_u32_host(uint64_t *keys, uint32_t *vals, size_t n, uint64_t seed, void *stream);
int sq_sort_pairs_u32_u32_host(uint32_t *keys, uint32_t *vals, size_t n, uint64_t seed,
                               void *stream);

/* A batch of `count` independent sorts of n HOST keys each: item i reads
 * in[i] and writes the ascending result to out[i] (in[i] == out[i] sorts in
 * place; several items may share one input buffer).  The items are
 * pipelined: the host->device copy of item i+1 and the device->host copy of
 * item i-1 run on two library-owned copy streams while item i sorts on
 * `stream`, so with pinned buffers the batch costs about
 * max(copy in, sort, copy out) per item instead of their sum.  Up to three
 * device buffers of n keys are allocated for the call.  Each item is the same
 * operation as sq_sort_u32_host / sq_sort_u64_host (same seed).
 * Requirements: in, out and every in[i], out[i] non-NULL when count > 0;
 * out[i] must not overlap in[j] for any j > i (a later item's input).
 * Outputs may be reused: copies out run in item order, so where out[i] and
 * out[j] (i < j) overlap, item j's result is what remains.
 * Returns on completion (all items copied out) or at the first error; on
 * error the contents of out[] are unspecified. */
int sq_sort_u32_host_batch(const uint32_t *const *in, uint32_t *const *out, size_t n,
                           size_t count, uint64_t seed, void *stream);
int sq_sort_u64_host_batch(const uint64_t *const *in, uint64_t *const *out, size_t n,
                           size_t count, uint64_t seed, void *stream);

/* ------------------------------------------------------------------------- */
/* SkewTranspose exactly as Alg 2/3 define it.        */
/* ------------------------------------------------------------------------- */
#define SQ_FLAG_VALIDATE 1u /* check columns sorted and pivots non-decreasing first */

typedef struct {
  /* Device pointer: the k-1 finite pivots p_1 <= ... <= p_{k-1},
   * non-decreasing.  Bucket j (0-based) takes the keys x with
   * bucket(x) = #{p < x} + [x is a pivot] = j (Alg 3 with strict '<' and the
   * equal-pivot rule, L2/L4).  The last bucket is unbounded; +infinity is
   * implicit and is never a stored value (L3).  May be NULL when k = 1. */
  const uint32_t *pivots;
  uint32_t k;               /* number of buckets, >= 1 */
  uint64_t n;               /* keys present; 0 means rows*cols.  Column c is
                               src[c*rows, min((c+1)*rows, n)). */
  const uint32_t *buc_in;   /* device, k entries: initial write cursors (0-based
                               offsets into dst), or NULL: the bucket starts are
                               computed (analysis convention P:461, L1):
                               buc[0] = 0, buc[j] = #{x : bucket(x) < j}. */
  uint32_t *buc_out;        /* device, k entries, required: final cursors
                               buc_in[j] + size_j -- the "shifted by one
                               position" state of Alg 1. */
  uint32_t naive_threshold; /* Alg 2 leaf threshold (default 4), >= 2.
                               Alg 2 and Alg 3 give identical results for any
                               threshold, so it never changes the output. */
  uint32_t flags;           /* SQ_FLAG_VALIDATE or 0 */
} sq_skew_params;

/* dst[buc[j] + r] = the r-th key of bucket j in column-major order of src
 * (stable: column order, then position in the column).  src holds
 * `cols` sorted columns of `rows` keys (the last ones ragged or empty when
 * n < rows*cols).  src and dst are device buffers of at least n keys and must
 * not overlap.  Errors: SQ_ERR_INVALID_ARGUMENT for NULL src/dst/buc_out with
 * n > 0, NULL pivots with k > 1, k = 0, threshold < 2, rows*cols overflow,
 * n > rows*cols, n >= 2^32, or overlapping src/dst; SQ_ERR_PRECONDITION
 * (with SQ_FLAG_VALIDATE) for an unsorted column or decreasing pivots (without
 * the flag these are the caller's preconditions, as in Alg 2's input
 * specification P:406, and violating them is undefined behaviour);
 * SQ_ERR_INVALID_ARGUMENT also when a caller-given cursor range
 * [buc_in[j], buc_in[j] + size_j) does not fit in dst[0, n). */
int sq_skew_transpose(const uint32_t *src, uint32_t *dst, size_t rows, size_t cols,
                      const sq_skew_params *params, void *stream);

/* The same for 64-bit keys (the paper's external-sort workload): the
 * pivots are u64; cursors, sizes and every rule as above.  The call blocks the
 * host once, at its end (twice with SQ_FLAG_VALIDATE); the cursors are scanned
 * and checked on the device. */
typedef struct {
  const uint64_t *pivots;   /* device, k-1 non-decreasing u64 pivots (NULL when k = 1) */
  uint32_t k;
  uint64_t n;
  const uint32_t *buc_in;
  uint32_t *buc_out;
  uint32_t naive_threshold;
  uint32_t flags;
} sq_skew_params_u64;
int sq_skew_transpose_u64(const uint64_t *src, uint64_t *dst, size_t rows, size_t cols,
                          const sq_skew_params_u64 *params, void *stream);

/* ------------------------------------------------------------------------- */
/* The sampler's counter-based RNG, on the host, for callers    */
/* that run a SquareSort level across several GPUs (paper_2407_14801_b200.dist):*/
/* every rank derives the same sample positions of the global level.         */
/* ------------------------------------------------------------------------- */
/* Root node key of a sort with this seed (mix(seed)). */
uint64_t sq_root_key(uint64_t seed);
/* out[r*count + i] = floor(draw(node, r, i) * n / 2^64): position i of sampling
 * round r of a level of n keys at `node` (the positions the
 * single-GPU sampler draws).  out is HOST memory of rounds*count entries.
 * SQ_ERR_INVALID_ARGUMENT for NULL out or n = 0 with work to do.  No GPU use. */
int sq_draw_positions(uint64_t node, uint32_t rounds, uint32_t count, uint64_t n, uint64_t *out);

/* ------------------------------------------------------------------------- */
/* Introspection and test hooks.                                             */
/* ------------------------------------------------------------------------- */
const char *sq_status_string(int status);
const char *sq_last_error_message(void);

typedef struct {
  uint32_t levels;          /* SquareSort levels run (recursion into oversize segments) */
  uint32_t kernel_launches; /* kernels this library launched in the last call          */
  uint32_t host_syncs;      /* device->host planning reads                             */
  uint32_t top_round;       /* accepted sampling round of the top level (0-based)      */
  uint32_t top_degenerate;  /* 1 if the top level hit the resample cap          */
  uint32_t top_m;           /* m of the top level (0 if the input fit on chip)         */
  uint64_t oversize_keys;   /* keys in buckets that needed another level               */
} sq_stats;

/* Release the scratch the library's pool on the current device keeps reserved
 * between calls (cudaMemPoolTrimTo 0), and the cached graphs of small levels
 * with their scratch (graphs being replayed by another thread stay).  Safe to
 * call at any time; memory of calls still in flight on other streams stays
 * mapped until they finish. */
int sq_trim_memory(void);

/* Statistics of the calling thread's last sort / transpose call. */
void sq_get_stats(sq_stats *out);

/* Tuning/test knob: the largest segment sorted on chip by one CTA (a power of
 * two between 64 and the key type's maximum, 32768 for u32 and 16384 for
 * 64-bit sorts).  Lowering it forces more SquareSort levels on small inputs.
 * 0 restores the default.  Process-wide; returns SQ_ERR_INVALID_ARGUMENT for
 * other values. */
int sq_set_max_tile(uint32_t max_tile);

/* Tuning/test knob: how buckets larger than one CTA's tile (16384 32-bit or
 * 8192 64-bit keys by default) are sorted.  0: another SquareSort level
 * (P:291-293); 1 (default): the multi-CTA base case -- chunks sorted on chip,
 * then merge passes through HBM, up to 16 chunks (larger buckets recurse);
 * 2: thread-block clusters of 4/8/16 CTAs merging through distributed shared
 * memory; 3: for 32-bit keys with the counting-sort base case, thread-block
 * clusters of 2/4/8 counting-sort tiles that split the bucket into value ranges
 * through distributed shared memory (buckets up to 8 x 16128 keys; other key
 * types run mode 1); 4: keys-only sorts split an inner bucket b (keys in
 * [P[b-1], P[b]), readings L2/L4) into up to 16 value ranges, each sorted on chip
 * by one CTA that reads the whole bucket and keeps its range (no merge passes;
 * pairs and the outer buckets run mode 1).  Process-wide;
 * SQ_ERR_INVALID_ARGUMENT for other values. */
int sq_set_big_bucket_mode(int mode);

/* Tuning/test knob: the on-chip base case of keys-only 32-bit sorts (the GPU's
 * simple_sort).  1 (default): counting sort on a monotone bin of the
 * key followed by a sorting-network fix-up inside the bins;
 * 0: merge sort (Batcher network, warp bitonic merges, merge-path passes).
 * Both give the same (unique) result.  Process-wide; SQ_ERR_INVALID_ARGUMENT
 * for other values. */
int sq_set_base_case(int which);

/* Per-kernel device timing: when enabled, every kernel the library launches is
 * bracketed by CUDA events on its stream and the elapsed times accumulate per
 * kernel role (colsort, bucketsort, smallsort, sample, count, transpose, ...).
 * sq_profile_read writes {"role": [launches, total_ms], ...} (JSON) into buf
 * and clears the totals; SQ_ERR_INVALID_ARGUMENT if buf is too small. */
int sq_profile(int enable);
int sq_profile_read(char *buf, size_t cap);

/* One SquareSort level of u32 keys as the sorts run it, stopped after the
 * SkewTranspose (for intermediate-state parity tests): src (device, n keys,
 * unchanged) is copied; pivots are sampled at node key mix(seed) from the level
 * input (reading L9: before the column sort, P:279 draws from D), the
 * m = ceil(sqrt(n)) columns are sorted, min-exclusion is applied, and
 * the keys are moved into their buckets; dst (device, n keys) receives the
 * paper's SkewTranspose result (bucket-contiguous, column order within a
 * bucket).  pivots_out (device, m-1 entries), bucend_out (device, m entries:
 * the final cursors) and info_out (device, 2 entries: accepted round,
 * degenerate flag) may not be NULL.  Requires 5 <= n <= 2^30. */
int sq_debug_level_u32(const uint32_t *src, uint32_t *dst, size_t n, uint64_t seed,
                       uint32_t *pivots_out, uint32_t *bucend_out, uint32_t *info_out,
                       void *stream);

/* The same for u64 keys (the pivots are u64; n in [5, 2^28]). */
int sq_debug_level_u64(const uint64_t *src, uint64_t *dst, size_t n, uint64_t seed,
                       uint64_t *pivots_out, uint32_t *bucend_out, uint32_t *info_out,
                       void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SQUARESORT_H */
