// level.cuh -- kernels of one data-parallel SquareSort level (Alg 1).
//
// A level takes a batch of segments, each viewed as an m x m column-major
// matrix (m = ceil(sqrt(len))), and runs
//   column sort (blocksort.cuh) -> column-head minimum -> pivot sampling ->
//   bucket count -> bucket scan (host) -> SkewTranspose -> bucket sorts.
// Every kernel below handles all segments of the batch in one grid.
#pragma once
#include "blocksort.cuh"

namespace sq {

constexpr int kTB = 32;          // buckets per SkewTranspose tile (one warp lane per bucket)
constexpr uint32_t kCap = 32;    // resample cap

// Per-segment metadata of a level (host-built).  A segment is a matrix of
// `ncols` columns of `rows` items (column c = [off + c*rows, off + min((c+1)*rows, len)),
// P:271 / S:41) with k buckets defined by k-1 pivots.  SquareSort uses
// ncols = rows = k = m; the standalone SkewTranspose call may use any shape.
struct LevelSeg {
  uint32_t off, len;
  uint32_t rows, ncols, k, nbt;  // nbt = ceil(k / kTB) bucket tiles
  uint32_t piv_base;             // pivots arena: k-1 entries
  uint32_t buck_base;            // bucket arrays (counts, starts): k entries
  uint64_t segmat_base;          // (nbt+1) tile-boundary positions per column (sort path: tile-major)
  uint64_t cand_base;            // sampler candidates: (R+1) slots of k-1 entries
  uint64_t node;                 // RNG node key
};

struct TaskDesc {  // (segment, a, b): column range [a, b) or tile index a or sampler slot a
  uint32_t seg, a, b;
};

// ------------------------------------------------------------------------------
// min(D) from the heads of the sorted columns.  One CTA per segment.
template <typename K>
__global__ void k_colmin(const LevelSeg* __restrict__ segs, const K* __restrict__ data,
                         K* __restrict__ segmin) {
  const LevelSeg s = segs[blockIdx.x];
  K v = KeyTraits<K>::kMax;
  for (uint32_t c = threadIdx.x; c < s.ncols; c += blockDim.x) {
    uint64_t a = uint64_t(c) * s.rows;
    if (a < s.len) v = min(v, data[s.off + a]);
  }
  __shared__ K red[32];
  for (int o = 16; o; o >>= 1) {
    K w = __shfl_xor_sync(0xffffffffu, v, o);
    v = min(v, w);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : KeyTraits<K>::kMax;
    for (int o = 16; o; o >>= 1) {
      K w = __shfl_xor_sync(0xffffffffu, v, o);
      v = min(v, w);
    }
    if (threadIdx.x == 0) segmin[blockIdx.x] = v;
  }
}

// ------------------------------------------------------------------------------
// Bucket count: for each sorted column, a simultaneous scan
// of the column and the pivots gives the position of every bucket boundary;
// bucket sizes accumulate per CTA in shared memory and go to the CTA's row of a
// (column range, bucket) count matrix (zeroed by the caller), and the positions
// of the tile boundaries (every kTB-th bucket) are stored for the SkewTranspose.
// CTA = (segment, column range).
// Boundary j (1..k-1): x lies before it iff x < P[j-1], or x == P[j-1] when
// P[j-1] == P[j-2] (single-value bucket rule, L4).
template <typename K, int NT, int STAGE, int KSMEM>
__global__ void __launch_bounds__(NT)
k_count(const LevelSeg* __restrict__ segs, const TaskDesc* __restrict__ tasks, const K* __restrict__ data,
        const K* __restrict__ piv, uint32_t* __restrict__ segmat, uint32_t* __restrict__ gcnt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K* col = reinterpret_cast<K*>(smem_raw);                                   // STAGE keys
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw + STAGE * sizeof(K));  // KSMEM counters
  const TaskDesc tk = tasks[blockIdx.x];
  const LevelSeg sg = segs[tk.seg];
  const uint32_t k = sg.k;
  const bool smem_cnt = k <= (uint32_t)KSMEM;
  const bool staged = sg.rows <= (uint32_t)STAGE;
  const K* P = piv + sg.piv_base;
  if (smem_cnt)
    for (uint32_t b = threadIdx.x; b < k; b += NT) cnt[b] = 0;
  const uint32_t chunk = (k + NT - 1) / NT;
  const uint32_t b0 = threadIdx.x * chunk;
  const uint32_t b1 = min(b0 + chunk, k);
  for (uint32_t c = tk.a; c < tk.b; c++) {
    const uint64_t a = uint64_t(c) * sg.rows;
    const uint32_t L = (uint32_t)(a < sg.len ? min((uint64_t)sg.rows, (uint64_t)(sg.len - a)) : 0);
    const K* g = data + sg.off + a;
    __syncthreads();
    if (staged)
      for (uint32_t i = threadIdx.x; i < L; i += NT) col[i] = g[i];
    __syncthreads();
    const K* cs = staged ? col : g;
    uint32_t* row = segmat + sg.segmat_base + uint64_t(c) * (sg.nbt + 1);
    if (b0 < b1) {
      uint32_t pos = 0;
      if (b0 > 0) {  // binary search for boundary b0
        const K pj = P[b0 - 1];
        const bool dup = b0 >= 2 && P[b0 - 2] == pj;
        uint32_t lo = 0, hi = L;
        while (lo < hi) {
          uint32_t mid = (lo + hi) >> 1;
          if (before_boundary(cs[mid], pj, dup)) lo = mid + 1; else hi = mid;
        }
        pos = lo;
      }
      for (uint32_t b = b0; b < b1; b++) {
        if (b % kTB == 0) row[b / kTB] = pos;
        uint32_t nxt = L;
        if (b + 1 < k) {  // walk to boundary b+1
          const K pj = P[b];
          const bool dup = b >= 1 && P[b - 1] == pj;
          nxt = pos;
          while (nxt < L && before_boundary(cs[nxt], pj, dup)) nxt++;
        }
        const uint32_t n_b = nxt - pos;
        if (smem_cnt) cnt[b] += n_b;
        else if (n_b) atomicAdd(&gcnt[uint64_t(blockIdx.x) * k + b], n_b);
        pos = nxt;
      }
    }
    if (threadIdx.x == 0) row[sg.nbt] = L;
  }
  if (smem_cnt) {  // this task's row of the (task, bucket) count matrix
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < k; b += NT) gcnt[uint64_t(blockIdx.x) * k + b] = cnt[b];
  }
}

// ------------------------------------------------------------------------------
// SkewTranspose (Alg 2/3): the stable partition of the column-major
// level array by bucket -- within a bucket, items keep column order and the
// order inside each column (the four-call order of Alg 2 guarantees this,
// S:153).  Work is split by bucket tile (kTB buckets), which balances by
// construction even for presorted inputs.  A tile's CTA streams all
// columns in order: for a group of G columns it reads the tile's run of each
// column (contiguous, sorted), and in pieces of S keys computes every key's
// bucket, its rank among the piece's keys of that bucket (column order), and
// writes each bucket's piece contiguously at the bucket's cursor.
template <typename K, bool PAIRS, int NT, int S, int G>
struct TransposeCfg {
  static constexpr int NW = NT / 32;
  static constexpr int VS = S / NT;  // keys per thread in blocked passes
  static constexpr size_t al(size_t x) { return (x + 15) & ~size_t(15); }
  static constexpr size_t off_stage = 0;
  static constexpr size_t off_out = al(off_stage + S * sizeof(K));
  static constexpr size_t off_vstage = al(off_out + S * sizeof(K));
  static constexpr size_t off_vout = al(off_vstage + (PAIRS ? S * 4 : 0));
  static constexpr size_t off_hd = al(off_vout + (PAIRS ? S * 4 : 0));
  static constexpr size_t off_tb = al(off_hd + S * 4);
  static constexpr size_t off_frag = al(off_tb + S);
  static constexpr size_t off_table = al(off_frag + S);  // G x kTB u16
  static constexpr size_t off_run = al(off_table + G * kTB * 2);
  static constexpr size_t off_rsrc = al(off_run + (G + 1) * 4);
  static constexpr size_t off_wsum = al(off_rsrc + G * 4);  // NW x 32 u32
  static constexpr size_t off_misc = al(off_wsum + NW * 32 * 4);
  static constexpr size_t off_bval = al(off_misc + (64 + 5 * kTB + 8) * 4);
  static constexpr size_t SMEM = al(off_bval + kTB * sizeof(K));
};

// Block-wide exclusive max-scan helper: returns max over all earlier threads' v.
template <int NW>
__device__ __forceinline__ uint32_t block_excl_max(uint32_t v, uint32_t* misc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = max(x, y);
  }
  __syncthreads();
  if (lane == 31) misc[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s2 = lane < NW ? misc[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s2, o);
      if (lane >= o) s2 = max(s2, y);
    }
    if (lane < NW) misc[lane] = s2;
  }
  __syncthreads();
  uint32_t c = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) c = 0;
  if (w > 0) c = max(c, misc[w - 1]);
  return c;
}

// Block-wide exclusive sum-scan; *total receives the sum over the block.
template <int NW>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* misc, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) misc[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t s2 = lane < NW ? misc[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s2, o);
      if (lane >= o) s2 += y;
    }
    if (lane < NW) misc[lane] = s2;
  }
  __syncthreads();
  *total = misc[NW - 1];
  return x - v + (w > 0 ? misc[w - 1] : 0);
}

template <typename K, bool PAIRS, int NT, int S, int G>
__global__ void __launch_bounds__(NT)
k_transpose(const LevelSeg* __restrict__ segs, const TaskDesc* __restrict__ tiles, const K* __restrict__ src,
            K* __restrict__ dst, const uint32_t* __restrict__ vsrc, uint32_t* __restrict__ vdst,
            const K* __restrict__ piv, const uint32_t* __restrict__ segmat, const uint32_t* __restrict__ bstart,
            const uint32_t* __restrict__ bad, const TaskDesc* __restrict__ cranges,
            const uint32_t* __restrict__ cpre) {
  // CTA (tile, column range r): columns cranges[r] of bucket tile tiles[.]; the
  // cursor of bucket j starts at bstart[j] + cpre[r][j] (the keys of bucket j in
  // the column ranges before r)
  using C = TransposeCfg<K, PAIRS, NT, S, G>;
  if (bad && (*bad & 4u)) return;  // caller cursors out of range: nothing is written
  static_assert(G <= 256, "fragment index is a byte");
  static_assert(S % NT == 0 && NT % 32 == 0 && NT >= G, "shape");
  static_assert(S <= 65535, "u16 table");
  extern __shared__ __align__(128) unsigned char sm[];
  K* stage = reinterpret_cast<K*>(sm + C::off_stage);
  K* outb = reinterpret_cast<K*>(sm + C::off_out);
  uint32_t* vstage = reinterpret_cast<uint32_t*>(sm + C::off_vstage);
  uint32_t* vout = reinterpret_cast<uint32_t*>(sm + C::off_vout);
  uint32_t* hd = reinterpret_cast<uint32_t*>(sm + C::off_hd);
  uint8_t* tbk = reinterpret_cast<uint8_t*>(sm + C::off_tb);
  uint8_t* frag = reinterpret_cast<uint8_t*>(sm + C::off_frag);
  uint16_t* table = reinterpret_cast<uint16_t*>(sm + C::off_table);
  uint32_t* runStart = reinterpret_cast<uint32_t*>(sm + C::off_run);
  uint32_t* runSrc = reinterpret_cast<uint32_t*>(sm + C::off_rsrc);
  uint32_t* wsum = reinterpret_cast<uint32_t*>(sm + C::off_wsum);
  uint32_t* misc = reinterpret_cast<uint32_t*>(sm + C::off_misc);  // [0..31] scan scratch, [33..34] ra rb
  uint32_t* cursor = misc + 64;
  uint32_t* ptot = cursor + kTB;
  uint32_t* poff = ptot + kTB;
  uint32_t* bdupv = poff + kTB;
  K* bval = reinterpret_cast<K*>(sm + C::off_bval);

  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t nr = gridDim.y, r = blockIdx.y;
  const TaskDesc tk = tiles[blockIdx.x];
  const TaskDesc cr = cranges[r];
  const LevelSeg sg = segs[tk.seg];
  const uint32_t bt = tk.a;
  const uint32_t b0 = bt * kTB;
  const uint32_t nb = min((uint32_t)kTB, sg.k - b0);
  const uint32_t nint = nb - 1;  // internal boundaries b0+1 .. b0+nb-1
  const K* P = piv + sg.piv_base;
  (void)nr;
  if (t < (int)nb) cursor[t] = bstart[sg.buck_base + b0 + t] + cpre[uint64_t(r) * sg.k + b0 + t];
  if (t < (int)nint) {
    const uint32_t j = b0 + 1 + t;
    bval[t] = P[j - 1];
    bdupv[t] = (j >= 2 && P[j - 2] == P[j - 1]) ? 1u : 0u;
  }
  __syncthreads();
  const int i0 = t * C::VS;

  for (uint32_t g0 = cr.a; g0 < cr.b; g0 += G) {
    const uint32_t ng = min((uint32_t)G, cr.b - g0);
    // ---- this tile's run in each column g0 .. g0+ng-1; exclusive scan of the lengths
    uint32_t len = 0;
    if (t < (int)ng) {
      const uint32_t c = g0 + t;
      const uint32_t* row = segmat + sg.segmat_base + uint64_t(c) * (sg.nbt + 1);
      const uint32_t a = row[bt], e = row[bt + 1];
      len = e - a;
      runSrc[t] = sg.off + c * sg.rows + a;
    }
    uint32_t Kg;
    const uint32_t excl = block_excl_sum<C::NW>(len, misc, &Kg);
    if (t < (int)ng) runStart[t] = excl;
    if (t == 0) runStart[ng] = Kg;
    __syncthreads();

    for (uint32_t p = 0; p < Kg; p += S) {
      const uint32_t Pn = min((uint32_t)S, Kg - p);
      // ---- run fragments overlapping [p, p+Pn)
      if (t == 0) {
        uint32_t lo = 0, hi = ng;  // ra = last r with runStart[r] <= p
        while (hi - lo > 1) {
          uint32_t mid = (lo + hi) >> 1;
          if (runStart[mid] <= p) lo = mid; else hi = mid;
        }
        uint32_t rb = lo;
        while (rb < ng && runStart[rb] < p + Pn) rb++;
        misc[33] = lo;
        misc[34] = rb;
      }
      __syncthreads();
      const uint32_t ra = misc[33], rb = misc[34];
      const uint32_t nf = rb - ra;
      for (uint32_t i = t; i < nf * kTB; i += NT) table[i] = 0;
      // ---- load: one warp per run fragment (coalesced reads of the sorted run)
      for (uint32_t r = ra + w; r < rb; r += C::NW) {
        const uint32_t lo = max(runStart[r], p), hi = min(runStart[r + 1], p + Pn);
        const uint32_t sbase = runSrc[r] - runStart[r];
        for (uint32_t q = lo + lane; q < hi; q += 32) {
          stage[q - p] = src[sbase + q];
          if (PAIRS) vstage[q - p] = vsrc[sbase + q];
          frag[q - p] = (uint8_t)(r - ra);
        }
      }
      __syncthreads();
      // ---- bucket of each key within the tile (binary search over its boundaries)
      for (int q = 0; q < C::VS; q++) {
        const int i = i0 + q;
        if (i < (int)Pn) {
          const K xk = stage[i];
          uint32_t lo = 0, hi = nint;
          while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            if (before_boundary(xk, bval[mid], bdupv[mid] != 0)) hi = mid; else lo = mid + 1;
          }
          tbk[i] = (uint8_t)lo;
        }
      }
      __syncthreads();
      // ---- group heads: groups are maximal runs of equal (fragment, bucket); within a
      // fragment buckets never decrease, so each (fragment, bucket) is one group.
      uint32_t runmax = 0;
      for (int q = 0; q < C::VS; q++) {
        const int i = i0 + q;
        if (i < (int)Pn && (i == 0 || frag[i] != frag[i - 1] || tbk[i] != tbk[i - 1])) runmax = i;
        hd[i] = runmax;
      }
      const uint32_t carry = block_excl_max<C::NW>(runmax, misc);
      for (int q = 0; q < C::VS; q++) hd[i0 + q] = max(hd[i0 + q], carry);
      __syncthreads();
      // ---- (fragment, bucket) sizes: the last key of each group writes the group length
      for (int q = 0; q < C::VS; q++) {
        const int i = i0 + q;
        if (i < (int)Pn && (i == (int)Pn - 1 || hd[i + 1] != hd[i]))
          table[frag[i] * kTB + tbk[i]] = (uint16_t)(i - hd[i] + 1);
      }
      __syncthreads();
      // ---- exclusive scan of the table down the fragments, per bucket (lane = bucket)
      const uint32_t per = (nf + C::NW - 1) / C::NW;
      const uint32_t f0 = min(nf, w * per), f1 = min(nf, f0 + per);
      {
        uint32_t sum = 0;
        for (uint32_t f = f0; f < f1; f++) sum += table[f * kTB + lane];
        wsum[w * 32 + lane] = sum;
      }
      __syncthreads();
      {
        uint32_t run = 0, total = 0;
        for (int ww = 0; ww < C::NW; ww++) {
          const uint32_t v = wsum[ww * 32 + lane];
          if (ww < w) run += v;
          total += v;
        }
        for (uint32_t f = f0; f < f1; f++) {
          const uint32_t v = table[f * kTB + lane];
          table[f * kTB + lane] = (uint16_t)run;
          run += v;
        }
        if (w == 0) {
          ptot[lane] = total;
          uint32_t v = lane < (int)nb ? total : 0, xs = v;
          for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
            if (lane >= o) xs += y;
          }
          poff[lane] = xs - v;
        }
      }
      __syncthreads();
      // ---- scatter into the piece's bucket-major buffer (stable: column order, then row)
      for (int q = 0; q < C::VS; q++) {
        const int i = i0 + q;
        if (i < (int)Pn) {
          const uint32_t b = tbk[i];
          const uint32_t o = poff[b] + table[frag[i] * kTB + b] + (i - hd[i]);
          outb[o] = stage[i];
          if (PAIRS) vout[o] = vstage[i];
        }
      }
      __syncthreads();
      // ---- flush: one warp per bucket, contiguous at the bucket's cursor
      for (uint32_t b = w; b < nb; b += C::NW) {
        const uint32_t cnt = ptot[b], o0 = poff[b], d0 = cursor[b];
        for (uint32_t q = lane; q < cnt; q += 32) {
          dst[d0 + q] = outb[o0 + q];
          if (PAIRS) vdst[d0 + q] = vout[o0 + q];
        }
      }
      __syncthreads();
      if (t < (int)nb) cursor[t] += ptot[t];
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------------------
// Copy whole ranges (single-value buckets; trivially sorted segments).
template <typename K>
__global__ void k_copy_ranges(const SegDesc* __restrict__ r, const K* __restrict__ src, K* __restrict__ dst,
                              const uint32_t* __restrict__ vsrc, uint32_t* __restrict__ vdst) {
  const SegDesc d = r[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < d.len; i += blockDim.x) {
    dst[d.off + i] = src[d.off + i];
    if (vsrc) vdst[d.off + i] = vsrc[d.off + i];
  }
}

// Precondition check for the standalone SkewTranspose (SQ_FLAG_VALIDATE):
// columns sorted and pivots non-decreasing.
template <typename K>
__global__ void k_validate(const K* __restrict__ src, uint64_t rows, uint64_t n, const K* __restrict__ piv,
                           uint32_t np, uint32_t* __restrict__ bad) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    if (i % rows != 0 && src[i - 1] > src[i]) atomicOr(bad, 1u);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x + 1; i < np; i += stride)
    if (piv[i - 1] > piv[i]) atomicOr(bad, 2u);
}

// Column-range prefix of the (range, bucket) count matrix, in place (exclusive,
// per bucket), and each bucket's total.  Thread per bucket.
static __global__ void k_skew_range_prefix(uint32_t* __restrict__ cnt, uint32_t nr, uint32_t k,
                                           uint32_t* __restrict__ tot) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    uint32_t run = 0;
    for (uint32_t r = 0; r < nr; r++) {
      const uint32_t c = cnt[uint64_t(r) * k + j];
      cnt[uint64_t(r) * k + j] = run;
      run += c;
    }
    tot[j] = run;
  }
}

// Standalone SkewTranspose cursors, on the device (no host round trip): with
// buc_in == NULL the bucket starts are the exclusive prefix of the counts
// (analysis convention); otherwise the caller's cursors are checked
// (every range [buc_in[j], buc_in[j] + size_j) inside [0, n); bad[0] |= 4 if
// not).  One CTA of 1024 threads.
static __global__ void __launch_bounds__(1024)
k_skew_cursors(const uint32_t* __restrict__ cnt, uint32_t k, uint64_t n, const uint32_t* __restrict__ buc_in,
               uint32_t* __restrict__ start, uint32_t* __restrict__ bad) {
  __shared__ uint32_t misc[64];
  if (buc_in) {
    for (uint32_t j = threadIdx.x; j < k; j += 1024) {
      const uint64_t b = buc_in[j];
      if (b + cnt[j] > n) atomicOr(bad, 4u);
      start[j] = uint32_t(b);
    }
    return;
  }
  const uint32_t per = (k + 1023) / 1024, j0 = min(k, threadIdx.x * per), j1 = min(k, j0 + per);
  uint32_t sum = 0;
  for (uint32_t j = j0; j < j1; j++) sum += cnt[j];
  uint32_t tot;
  uint32_t o = block_excl_sum<32>(sum, misc, &tot);
  for (uint32_t j = j0; j < j1; j++) {
    start[j] = o;
    o += cnt[j];
  }
}

// buc_out[j] = start[j] + size_j (the final cursors)
static __global__ void k_skew_finish(const uint32_t* __restrict__ start, const uint32_t* __restrict__ cnt, uint32_t k,
                                     uint32_t* __restrict__ buc_out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    buc_out[j] = start[j] + cnt[j];
}

}  // namespace sq
