/*
 * oracle/squaresort_oracle.c -- the CPU oracle for SquareSort (arXiv 2407.14801).
 *
 * TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded C11 written directly
 * from the paper's Algorithms 1-3.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load this library.  It
 * shares no source, header, table or helper with the CUDA path
 * (paper_2407_14801_b200/csrc), and neither side includes or links the other.
 *
 * Citations: "P:n" is /root/reference/PAPER.md line n, "S:n" is SPEC.md line n.
 * Readings of the paper where it is silent or garbled are the numbered
 * "L#" entries of DESIGN.md section 3 (taken from SURVEY.md 8(c)).
 *
 * Indexing is 0-based everywhere (S:172 allows a uniform offset): the paper's
 * col[i] = 1 + min((i-1)m, n) becomes col[i] = min(i*m, n), and so on.
 *
 * Items are 64-bit unsigned keys (u32 keys are widened; the order is the same)
 * with an optional 32-bit payload that moves with its key (pairs, reading L16).
 *
 * Pin status: every function below is pinned by a
 * `-m "not gpu"` test in tests/test_oracle.py, except the pivot sampler's
 * choice of pivots, which the paper leaves to "uniformly at random":
 * the concrete pivots are fixed by the RNG specification, so the
 * sampler is pinned only by its invariants and by the closed-form acceptance
 * rate, i.e. "parity unpinned" for the exact pivot values.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint32_t cutoff;            /* base case n <= cutoff (default 16); >= 4 (L5)      */
  uint32_t naive_threshold;   /* Alg 2 leaf: l < T or k < T (default 4); >= 2 (L6)   */
  uint32_t resample_cap;      /* sampling rounds before degenerate mode (default 32)  */
  uint32_t sample_from_input; /* 0: sample from D after the column sort;
                                 1: from the level input A (L9, the GPU's source)           */
} sqo_params;

typedef struct {
  uint64_t nodes;       /* SquareSort calls with n > cutoff                               */
  uint64_t rounds;      /* sampling rounds summed over those calls                        */
  uint64_t degenerate;  /* calls whose sampler hit the cap                         */
  uint64_t max_depth;   /* deepest recursion level reached (root = 0)                     */
  uint64_t single_value_buckets; /* buckets copied without recursion             */
} sqo_stats;

/* ------------------------------------------------------------------------ */
/* RNG (reading L10).  The paper names no generator.            */
/* mix = SplitMix64 output function applied to (z + golden ratio increment).  */
/* ------------------------------------------------------------------------ */
uint64_t sqo_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
uint64_t sqo_root_key(uint64_t seed) { return sqo_mix(seed); }
/* phase 0 = column child, phase 1 = bucket child. */
uint64_t sqo_child_key(uint64_t key, uint32_t phase, uint64_t idx) {
  return sqo_mix(key ^ sqo_mix(2u * idx + phase));
}
uint64_t sqo_draw(uint64_t key, uint32_t round, uint32_t i) {
  return sqo_mix(key ^ sqo_mix(((uint64_t)round << 32) | (uint64_t)i));
}
/* Uniform position in [0, len): floor(draw * len / 2^64) (a 128-bit product). */
uint64_t sqo_index(uint64_t draw, uint64_t len) {
  return (uint64_t)(((unsigned __int128)draw * (unsigned __int128)len) >> 64);
}

/* ------------------------------------------------------------------------ */
/* Column layout (Alg 1 line "calculate span of each column").   */
/* ------------------------------------------------------------------------ */
/* m = ceil(sqrt(n)) with an exact integer correction (L11). */
uint64_t sqo_ceil_sqrt(uint64_t n) {
  uint64_t r = (uint64_t)sqrt((double)n);
  while (r > 0 && r * r >= n) r--;   /* now r*r < n (or r = 0) */
  while (r * r < n) r++;             /* smallest r with r*r >= n */
  return r;
}

/* col[i] = min(i*m, n), colEnd[i] = min((i+1)*m, n) for i = 0..m-1. */
uint64_t sqo_column_layout(uint64_t n, uint64_t *col, uint64_t *colEnd) {
  uint64_t m = sqo_ceil_sqrt(n);
  for (uint64_t i = 0; i < m; i++) {
    uint64_t a = i * m, b = (i + 1) * m;
    if (col) col[i] = a < n ? a : n;
    if (colEnd) colEnd[i] = b < n ? b : n;
  }
  return m;
}

/* ------------------------------------------------------------------------ */
/* simple_sort (Alg 1): insertion sort for small arrays. */
/* Copies A into D and sorts D; stable (a later equal key never passes an   */
/* earlier one), so pairs keep their input order on ties (L16).             */
/* ------------------------------------------------------------------------ */
void sqo_simple_sort(const uint64_t *A, const uint32_t *Av, uint64_t *D, uint32_t *Dv,
                     uint64_t n) {
  for (uint64_t i = 0; i < n; i++) {
    uint64_t x = A[i];
    uint32_t xv = Av ? Av[i] : 0;
    uint64_t j = i;
    while (j > 0 && D[j - 1] > x) {
      D[j] = D[j - 1];
      if (Dv) Dv[j] = Dv[j - 1];
      j--;
    }
    D[j] = x;
    if (Dv) Dv[j] = xv;
  }
}

/* Ordinary top-down MergeSort of the pivot candidates. */
static void merge_sort_rec(uint64_t *a, uint64_t *tmp, uint64_t n) {
  if (n < 2) return;
  uint64_t h = n / 2;
  merge_sort_rec(a, tmp, h);
  merge_sort_rec(a + h, tmp, n - h);
  uint64_t i = 0, j = h, o = 0;
  while (i < h && j < n) tmp[o++] = (a[j] < a[i]) ? a[j++] : a[i++];
  while (i < h) tmp[o++] = a[i++];
  while (j < n) tmp[o++] = a[j++];
  memcpy(a, tmp, n * sizeof(uint64_t));
}
void sqo_merge_sort(uint64_t *a, uint64_t n) {
  uint64_t *tmp = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
  merge_sort_rec(a, tmp, n);
  free(tmp);
}

/* ------------------------------------------------------------------------ */
/* Pivot sampling (readings L7, L8, L9, L10).     */
/*                                                                          */
/* Round r = 0..cap-1: draw m-1 positions t_i uniformly with repetition,    */
/* take src[t_i], MergeSort them, and accept iff they are strictly          */
/* increasing (distinct values, L7) and the smallest exceeds min(D), where  */
/* min(D) is the least head of the sorted columns.  A failed    */
/* round re-samples the whole set.  After `cap` failures    */
/* the pivots are degenerate: round cap-1's sorted sample is kept.   */
/* Returns the accepted round, or cap-1 with *degenerate = 1.               */
/* ------------------------------------------------------------------------ */
uint32_t sqo_sample_pivots(uint64_t node, const uint64_t *src, const uint64_t *D,
                           uint64_t n, uint32_t cap, uint64_t *pivots,
                           uint32_t *degenerate) {
  uint64_t m = sqo_ceil_sqrt(n);
  uint64_t np = m - 1;
  /* min(D) from the column heads. */
  uint64_t minD = UINT64_MAX;
  for (uint64_t i = 0; i < m; i++) {
    uint64_t c = i * m;
    if (c < n && D[c] < minD) minD = D[c];
  }
  *degenerate = 0;
  for (uint32_t r = 0; r < cap; r++) {
    for (uint64_t i = 0; i < np; i++)
      pivots[i] = src[sqo_index(sqo_draw(node, r, (uint32_t)i), n)];
    sqo_merge_sort(pivots, np);
    int ok = (np == 0) || (pivots[0] > minD);
    for (uint64_t i = 1; ok && i < np; i++)
      if (!(pivots[i - 1] < pivots[i])) ok = 0;
    if (ok) return r;
  }
  *degenerate = 1;
  return cap - 1;
}

/* ------------------------------------------------------------------------ */
/* Bucket membership (Alg 3; readings L2, L3, L4).   */
/* Bucket i (0-based, i = 0..m-1) accepts x iff x < P[i], or x <= P[i] when */
/* i >= 1 and P[i-1] = P[i] (the single-value-bucket rule); the last */
/* bucket i = np has the +infinity pivot and accepts everything (L3: the    */
/* sentinel is out of band, never a stored value).                          */
/* ------------------------------------------------------------------------ */
static int accepts(const uint64_t *P, uint64_t np, uint64_t i, uint64_t x) {
  if (i >= np) return 1;
  if (x < P[i]) return 1;
  if (i >= 1 && P[i - 1] == P[i] && x <= P[i]) return 1;
  return 0;
}

/* Bucket positions (analysis convention P:461; L1).
 * For each sorted column, a simultaneous scan of the column and the pivots
 * counts the bucket sizes; an exclusive prefix sum of the counts
 * gives buc[j] = first slot of bucket j (0-based; buc[0] = 0). */
void sqo_initial_bucket_cursors(const uint64_t *D, uint64_t ncols, const uint64_t *col,
                                const uint64_t *colEnd, const uint64_t *P, uint64_t k,
                                uint64_t base, uint64_t *buc) {
  uint64_t np = k - 1;
  for (uint64_t j = 0; j < k; j++) buc[j] = 0;
  for (uint64_t c = 0; c < ncols; c++) {
    uint64_t i = 0;
    for (uint64_t t = col[c]; t < colEnd[c]; t++) {
      while (!accepts(P, np, i, D[t])) i++;
      buc[i]++;
    }
  }
  uint64_t s = base;
  for (uint64_t j = 0; j < k; j++) {
    uint64_t c = buc[j];
    buc[j] = s;
    s += c;
  }
}

/* Alg 3, NaiveSkewTranspose.  Pivots are indexed
 * globally: this call handles buckets poff .. poff+k-1 of the np+1 buckets, so
 * the equal-pivot rule can look one pivot to the left of the slice (L4). */
void sqo_naive_skew_transpose(const uint64_t *A, const uint32_t *Av, uint64_t *D, uint32_t *Dv,
                              uint64_t l, uint64_t *col, const uint64_t *colEnd,
                              uint64_t k, uint64_t poff, const uint64_t *P, uint64_t np,
                              uint64_t *buc) {
  for (uint64_t i = 0; i < k; i++) {
    for (uint64_t j = 0; j < l; j++) {
      while (col[j] < colEnd[j] && accepts(P, np, poff + i, A[col[j]])) {
        D[buc[i]] = A[col[j]];
        if (Dv) Dv[buc[i]] = Av[col[j]];
        buc[i] = buc[i] + 1;
        col[j] = col[j] + 1;
      }
    }
  }
}

/* Alg 2, SkewTranspose.  Cursor arrays are shared by
 * reference between the four calls, made in exactly the paper's order. */
void sqo_skew_transpose(const uint64_t *A, const uint32_t *Av, uint64_t *D, uint32_t *Dv,
                        uint64_t l, uint64_t *col, const uint64_t *colEnd, uint64_t k,
                        uint64_t poff, const uint64_t *P, uint64_t np, uint64_t *buc,
                        uint32_t T) {
  if (l < T || k < T) {
    sqo_naive_skew_transpose(A, Av, D, Dv, l, col, colEnd, k, poff, P, np, buc);
    return; /* L14 */
  }
  uint64_t l2 = l / 2, k2 = k / 2;
  sqo_skew_transpose(A, Av, D, Dv, l2, col, colEnd, k2, poff, P, np, buc, T);
  sqo_skew_transpose(A, Av, D, Dv, l - l2, col + l2, colEnd + l2, k2, poff, P, np, buc, T);
  sqo_skew_transpose(A, Av, D, Dv, l2, col, colEnd, k - k2, poff + k2, P, np, buc + k2, T);
  sqo_skew_transpose(A, Av, D, Dv, l - l2, col + l2, colEnd + l2, k - k2, poff + k2, P, np,
                     buc + k2, T);
}

/* ------------------------------------------------------------------------ */
/* Alg 1, SquareSort(A, D, n).                       */
/* Sorts A into D; A is scratch afterwards.                         */
/* ------------------------------------------------------------------------ */
static void square_sort_rec(uint64_t *A, uint32_t *Av, uint64_t *D, uint32_t *Dv, uint64_t n,
                            uint64_t node, const sqo_params *p, sqo_stats *st,
                            uint64_t depth) {
  if (st && depth > st->max_depth) st->max_depth = depth;
  if (n <= p->cutoff) {
    sqo_simple_sort(A, Av, D, Dv, n);
    return; /* L14 */
  }
  uint64_t m = sqo_ceil_sqrt(n);
  uint64_t *col = (uint64_t *)malloc(m * sizeof(uint64_t));
  uint64_t *colEnd = (uint64_t *)malloc(m * sizeof(uint64_t));
  uint64_t *pivots = (uint64_t *)malloc(m * sizeof(uint64_t)); /* m-1 used; +inf implicit */
  uint64_t *buc = (uint64_t *)malloc(m * sizeof(uint64_t));
  uint64_t *bucStart = (uint64_t *)malloc(m * sizeof(uint64_t));
  sqo_column_layout(n, col, colEnd);

  /* L9: the GPU samples the level input before its columns are sorted; the
   * oracle keeps a copy of that input so it can sample the same values. */
  uint64_t *A0 = NULL;
  if (p->sample_from_input) {
    A0 = (uint64_t *)malloc(n * sizeof(uint64_t));
    memcpy(A0, A, n * sizeof(uint64_t));
  }

  /* Sort each column of A into D. */
  for (uint64_t i = 0; i < m; i++) {
    uint64_t len = colEnd[i] - col[i];
    if (len == 0) continue;
    square_sort_rec(A + col[i], Av ? Av + col[i] : NULL, D + col[i], Dv ? Dv + col[i] : NULL,
                    len, sqo_child_key(node, 0, i), p, st, depth + 1);
  }

  /* Select pivots. */
  uint32_t degenerate = 0;
  uint32_t round = sqo_sample_pivots(node, p->sample_from_input ? A0 : D, D, n,
                                     p->resample_cap, pivots, &degenerate);
  if (st) {
    st->nodes++;
    st->rounds += (uint64_t)round + 1;
    st->degenerate += degenerate;
  }

  /* Bucket positions (P:283 with the analysis convention of P:461, L1). */
  sqo_initial_bucket_cursors(D, m, col, colEnd, pivots, m, 0, buc);
  memcpy(bucStart, buc, m * sizeof(uint64_t));

  /* SkewTranspose D into A. */
  sqo_skew_transpose(D, Dv, A, Av, m, col, colEnd, m, 0, pivots, m - 1, buc,
                     p->naive_threshold);

  /* buc is now "shifted by one position": bucket j is
   * [bucStart[j], buc[j]) = [buc[j-1], buc[j]) (L12: half-open). */
  for (uint64_t j = 0; j < m; j++) {
    uint64_t s = bucStart[j], e = buc[j];
    uint64_t len = e - s;
    if (len == 0) continue;
    if (j >= 1 && j < m - 1 && pivots[j - 1] == pivots[j]) {
      /* Single-value bucket: copy, no recursion (L4). */
      memcpy(D + s, A + s, len * sizeof(uint64_t));
      if (Dv) memcpy(Dv + s, Av + s, len * sizeof(uint32_t));
      if (st) st->single_value_buckets++;
      continue;
    }
    square_sort_rec(A + s, Av ? Av + s : NULL, D + s, Dv ? Dv + s : NULL, len,
                    sqo_child_key(node, 1, j), p, st, depth + 1);
  }
  free(A0);
  free(col);
  free(colEnd);
  free(pivots);
  free(buc);
  free(bucStart);
}

/* Public entry: SquareSort of A (n items, optional payload Av) into D. */
int sqo_square_sort(uint64_t *A, uint32_t *Av, uint64_t *D, uint32_t *Dv, uint64_t n,
                    uint64_t seed, const sqo_params *p, sqo_stats *st) {
  if (p->cutoff < 4 || p->naive_threshold < 2 || p->resample_cap < 1) return 1; /* L5, L6 */
  if (st) memset(st, 0, sizeof(*st));
  square_sort_rec(A, Av, D, Dv, n, sqo_root_key(seed), p, st, 0);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* One SquareSort level, stopped after the SkewTranspose (for the GPU's     */
/* intermediate-state parity): columns of A sorted (by SquareSort with p),  */
/* pivots sampled at `node`, cursors computed, D transposed into A.         */
/* Outputs: A = post-transpose array, pivots[0..m-2], bucEnd[0..m-1] (the   */
/* "shifted" cursors), returns the round, *degenerate set.           */
/* Requires n > 4 so that m >= 3.  D is scratch of n items.                 */
/* ------------------------------------------------------------------------ */
uint32_t sqo_level(uint64_t *A, uint32_t *Av, uint64_t *D, uint32_t *Dv, uint64_t n,
                   uint64_t node, const sqo_params *p, uint64_t *pivots, uint64_t *bucEnd,
                   uint32_t *degenerate) {
  uint64_t m = sqo_ceil_sqrt(n);
  uint64_t *col = (uint64_t *)malloc(m * sizeof(uint64_t));
  uint64_t *colEnd = (uint64_t *)malloc(m * sizeof(uint64_t));
  sqo_column_layout(n, col, colEnd);
  uint64_t *A0 = NULL;
  if (p->sample_from_input) {
    A0 = (uint64_t *)malloc(n * sizeof(uint64_t));
    memcpy(A0, A, n * sizeof(uint64_t));
  }
  for (uint64_t i = 0; i < m; i++) {
    uint64_t len = colEnd[i] - col[i];
    if (len == 0) continue;
    square_sort_rec(A + col[i], Av ? Av + col[i] : NULL, D + col[i], Dv ? Dv + col[i] : NULL,
                    len, sqo_child_key(node, 0, i), p, NULL, 1);
  }
  uint32_t round = sqo_sample_pivots(node, p->sample_from_input ? A0 : D, D, n,
                                     p->resample_cap, pivots, degenerate);
  sqo_initial_bucket_cursors(D, m, col, colEnd, pivots, m, 0, bucEnd);
  sqo_skew_transpose(D, Dv, A, Av, m, col, colEnd, m, 0, pivots, m - 1, bucEnd,
                     p->naive_threshold);
  free(A0);
  free(col);
  free(colEnd);
  return round;
}

/* ------------------------------------------------------------------------ */
/* Standalone SkewTranspose with the ABI's parameters:        */
/* `cols` sorted columns of `rows` items (column c = src[c*rows,            */
/* min((c+1)*rows, n))), k buckets given by k-1 pivots, initial cursors     */
/* buc_in (NULL: computed by the merge-scan count), final        */
/* cursors in buc_out, leaf threshold T.                            */
/* ------------------------------------------------------------------------ */
void sqo_skew_transpose_matrix(const uint64_t *src, const uint32_t *srcv, uint64_t *dst,
                               uint32_t *dstv, uint64_t rows, uint64_t cols, uint64_t n,
                               const uint64_t *P, uint64_t k, const uint64_t *buc_in,
                               uint64_t *buc_out, uint32_t T) {
  uint64_t *col = (uint64_t *)malloc((cols ? cols : 1) * sizeof(uint64_t));
  uint64_t *colEnd = (uint64_t *)malloc((cols ? cols : 1) * sizeof(uint64_t));
  for (uint64_t c = 0; c < cols; c++) {
    uint64_t a = c * rows, b = (c + 1) * rows;
    col[c] = a < n ? a : n;
    colEnd[c] = b < n ? b : n;
  }
  if (buc_in)
    memcpy(buc_out, buc_in, k * sizeof(uint64_t));
  else
    sqo_initial_bucket_cursors(src, cols, col, colEnd, P, k, 0, buc_out);
  sqo_skew_transpose(src, srcv, dst, dstv, cols, col, colEnd, k, 0, P, k - 1, buc_out, T);
  free(col);
  free(colEnd);
}
