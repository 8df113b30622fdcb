// level2.cuh -- the fused, host-sync-light SquareSort level used by the sorts.
//
// Differences from the paper's sequential structure, none of
// which changes the sorted result:
//  * pivots are sampled from the level input before its columns are sorted
//    (reading L9: same distribution of pivot sets), all 32 rounds in parallel,
//    so the column sort can emit the bucket-tile boundaries of every column in
//    its epilogue (no separate bucket-count pass);
//  * min-exclusion is checked after the column sort (it needs min(D));
//    in the rare case it rejects the tentative round, the tile boundaries are
//    recomputed from the sorted columns;
//  * SkewTranspose writes each bucket tile "piece-major": pieces of S keys, each
//    the stable bucket-major partition of S consecutive keys of the tile's
//    column-major stream.  A bucket is the concatenation, in piece order, of its
//    sub-chunk in every piece of its tile -- exactly the paper's bucket in the
//    paper's order (column order, then row), only not yet contiguous; the bucket
//    sort gathers the sub-chunks on chip and writes the sorted bucket to its
//    final position, so no bucket sizes are needed before the transpose.
#pragma once
#include <cooperative_groups.h>
#include <type_traits>
#include "level.cuh"
#include "binsort.cuh"

namespace sq {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
template <typename K>
__device__ __forceinline__ void cp_async_elem(K* sdst, const K* gsrc) {
  if constexpr (sizeof(K) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_addr(sdst)), "l"(gsrc));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr(sdst)), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Per-tile bookkeeping of the piece-major transpose.
struct TileInfo {
  uint32_t seg, bt;      // segment and bucket tile
  uint32_t out;          // absolute output offset of the tile's region
  uint32_t size;         // keys in the tile
  uint32_t piece_base;   // first entry in the piece tables
  uint32_t npieces;      // pieces written (set by the piece plan)
  uint32_t dense;        // piece count, then (k_piece_dense) first position in the dense piece list
};

// Per-bucket record for the bucket phase.
struct BucketRec {
  uint32_t tile;    // tile index (TileInfo)
  uint32_t lane;    // bucket index within the tile (0..31)
  uint32_t out;     // absolute final offset of the sorted bucket
  uint32_t size;
  uint64_t node;    // RNG node key of the bucket (child(node, 1, b)), for deeper levels
  uint32_t chunk;   // merge-sort base case: keys per sorted chunk (= size otherwise)
  uint32_t passes;  // merge passes after the chunk sorts (0: sorted by one CTA)
};

// Bucket-sort work items: bucket index * 16 + chunk index.
__host__ __device__ __forceinline__ uint32_t item_bucket(uint32_t e) { return e >> 4; }
__host__ __device__ __forceinline__ uint32_t item_chunk(uint32_t e) { return e & 15u; }

// Merge-pass work item: pair j of runs, output tile t of the merged pair.
struct MTile {
  uint32_t bucket;
  uint16_t pair, tile;
};
constexpr int kMaxPasses = 4;  // 16 chunks

constexpr int kPP = kTB + 1;  // prefix entries per piece

// The counting-sort base case (binsort.cuh) serves 32-bit sort keys with 16 or 32
// keys per thread and 64-bit sort keys (u64 keys, u32-key pair composites) with 16;
// everything else (fewer keys per thread, u64-key pair composites) uses the merge
// sort (blocksort.cuh).
template <typename K, int V, bool PAIRS>
__host__ __device__ constexpr bool bin_ok() {
  using SK = sortkey_t<K, PAIRS>;
  return sizeof(SK) == 4 ? (V == 16 || V == 32) : (sizeof(SK) == 8 && V == 16);
}
template <typename K, int NT, int V, bool PAIRS>
using BinSortOf = BinSort<sortkey_t<K, PAIRS>, NT, V>;
// shared memory of the counting sort's counters (0 when the merge sort runs)
template <typename K, int NT, int V, bool PAIRS, bool BIN>
__host__ __device__ constexpr size_t bin_smem() {
  if constexpr (BIN && bin_ok<K, V, PAIRS>()) return BinSortOf<K, NT, V, PAIRS>::CNT_BYTES;
  else return 0;
}
// Physical slot of tile position i in the sort kernels' shared-memory tile: the
// counting sort's swizzled rows, else the merge sort's padded layout.
template <typename K, int NT, int V, bool PAIRS, bool BIN>
__device__ __forceinline__ uint32_t tpos(uint32_t i) {
  if constexpr (BIN && bin_ok<K, V, PAIRS>()) return BinSortOf<K, NT, V, PAIRS>::pad(i);
  else return BlockSort<sortkey_t<K, PAIRS>, NT, V>::pad(i);
}
// Sort the tile in shared memory with the selected base case.
template <typename K, int NT, int V, bool PAIRS, bool BIN, typename SK>
__device__ __forceinline__ void tile_sort(SK* s, uint32_t* cnt, uint32_t len) {
  if constexpr (BIN && bin_ok<K, V, PAIRS>()) BinSortOf<K, NT, V, PAIRS>::sort_smem(s, cnt, len);
  else BlockSort<SK, NT, V>::sort_smem(s, len);
}

// ------------------------------------------------------------------------------
// All kCap sampling rounds of every segment in parallel (CTA = (segment, round)),
// drawn from the level input A before the column sort (L9).  Stores the sorted
// candidates, whether they are strictly increasing, and their smallest value.
// BIN: the candidates are sorted by the counting sort (binsort.cuh) where it serves
// the key type and shape, else by the merge sort.
// Candidate gather for large samples: one round's m-1 random reads issued by a single
// CTA are bound by that SM's outstanding misses (~40 us for 16383 reads), so they are
// spread over CTAs of kSampleChunk candidates each; k_sample_all then reads the
// round's candidates back contiguously.  Grid: (segment, round, chunk), chunk-minor.
constexpr uint32_t kSampleChunk = 1024;
template <typename K>
__global__ void __launch_bounds__(256)
k_sample_gather(const LevelSeg* __restrict__ segs, const K* __restrict__ data, K* __restrict__ cand,
                uint32_t nchunk) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const uint32_t sr = blockIdx.x / nchunk, chunk = blockIdx.x % nchunk;
  const uint32_t seg = sr / kCap, r = sr % kCap;
  const LevelSeg sg = segs[seg];
  const uint32_t np = sg.k - 1;
  const K* lvl = data + sg.off;
  K* out = cand + sg.cand_base + uint64_t(r) * np;
  constexpr int J = kSampleChunk / 256;
  K x[J];
#pragma unroll
  for (int j = 0; j < J; j++) {
    const uint32_t i = chunk * kSampleChunk + threadIdx.x + uint32_t(j) * 256;
    x[j] = i < np ? __ldg(&lvl[draw_index(draw(sg.node, r, i), sg.len)]) : K(0);
  }
#pragma unroll
  for (int j = 0; j < J; j++) {
    const uint32_t i = chunk * kSampleChunk + threadIdx.x + uint32_t(j) * 256;
    if (i < np) out[i] = x[j];
  }
}

// `gathered`: the round's candidates were already written to `cand` by k_sample_gather.
template <typename K, int NT, int V, bool BIN = false>
__global__ void __launch_bounds__(NT)
k_sample_all(const LevelSeg* __restrict__ segs, const K* __restrict__ data, K* __restrict__ cand,
             uint8_t* __restrict__ flags, K* __restrict__ p0s, bool gathered) {
  using BS = BlockSort<K, NT, V>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K* s = reinterpret_cast<K*>(smem_raw);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES);
  auto TP = [](uint32_t i) { return tpos<K, NT, V, false, BIN>(i); };
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // the selection may launch now
  const uint32_t seg = blockIdx.x / kCap, r = blockIdx.x % kCap;
  const LevelSeg sg = segs[seg];
  const uint32_t np = sg.k - 1;
  const K* lvl = data + sg.off;
  if (gathered) {  // (programmatic dependent of k_sample_gather)
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const K* in = cand + sg.cand_base + uint64_t(r) * np;
    K x[V];
#pragma unroll
    for (int j = 0; j < V; j++) {
      const uint32_t i = threadIdx.x + uint32_t(j) * NT;
      x[j] = i < np ? in[i] : KeyTraits<K>::kMax;
    }
#pragma unroll
    for (int j = 0; j < V; j++) s[TP(threadIdx.x + uint32_t(j) * NT)] = x[j];
  } else {  // every random read of the thread in flight at once (they are DRAM-latency bound)
    K x[V];
#pragma unroll
    for (int j = 0; j < V; j++) {
      const uint32_t i = threadIdx.x + uint32_t(j) * NT;
      x[j] = i < np ? __ldg(&lvl[draw_index(draw(sg.node, r, i), sg.len)]) : KeyTraits<K>::kMax;
    }
#pragma unroll
    for (int j = 0; j < V; j++) s[TP(threadIdx.x + uint32_t(j) * NT)] = x[j];
  }
  __syncthreads();
  tile_sort<K, NT, V, false, BIN>(s, cnt, np);
  int viol = 0;
  for (int i = threadIdx.x + 1; i < (int)np; i += NT)
    if (!(s[TP(i - 1)] < s[TP(i)])) viol = 1;
  const bool distinct = !__syncthreads_or(viol);
  K* out = cand + sg.cand_base + uint64_t(r) * np;
  for (int i = threadIdx.x; i < (int)np; i += NT) out[i] = s[TP(i)];
  if (threadIdx.x == 0) {
    flags[uint64_t(seg) * kCap + r] = distinct ? 1 : 2;
    p0s[uint64_t(seg) * kCap + r] = np ? s[TP(0)] : KeyTraits<K>::kMax;
  }
}

// Round selection.  mode 0 (before the column sort): the
// first strictly increasing round -- tentative.  mode 1 (after): the first round
// that is strictly increasing AND whose smallest pivot exceeds min(D); none ->
// degenerate (round cap-1).  When the final round differs from the tentative
// one, the pivots are replaced and fix[seg] / fix[nseg] are raised so the tile
// boundaries get recomputed.  info = round | degenerate << 31.
template <typename K>
__global__ void k_select_round(const LevelSeg* __restrict__ segs, uint32_t nseg, const K* __restrict__ cand,
                               const uint8_t* __restrict__ flags, const K* __restrict__ p0s,
                               const K* __restrict__ segmin, K* __restrict__ piv, uint32_t* __restrict__ info,
                               uint32_t* __restrict__ fix, int mode) {
  // launched as a programmatic dependent: let the column sort start, then wait for
  // the sampler (and, in mode 1, for the column sort)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uint32_t seg = blockIdx.x;
  const LevelSeg sg = segs[seg];
  __shared__ uint32_t sel, change;
  static_assert(kCap <= 32, "one lane per round");
  if (threadIdx.x < 32) {  // lane q tests round q; the first accepted round wins
    const uint32_t q = threadIdx.x;
    const bool ok = q < kCap && flags[uint64_t(seg) * kCap + q] == 1 &&
                    (mode == 0 || sg.k == 1 || p0s[uint64_t(seg) * kCap + q] > segmin[seg]);
    const uint32_t acc = __ballot_sync(0xffffffffu, ok);
    const uint32_t r = acc ? uint32_t(__ffs(acc) - 1) : kCap;
    if (q == 0) {
      const uint32_t inf = r < kCap ? r : ((kCap - 1) | 0x80000000u);
      change = mode == 0 || info[seg] != inf;
      if (mode == 1 && change) {
        fix[seg] = 1;
        fix[nseg] = 1;
      }
      info[seg] = inf;
      sel = r < kCap ? r : kCap - 1;
    }
  }
  __syncthreads();
  if (!change) return;
  const uint32_t np = sg.k - 1;
  const K* in = cand + sg.cand_base + uint64_t(sel) * np;
  // (on the column sort's critical path: 1024 threads, several loads in flight each)
#pragma unroll 8
  for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) piv[sg.piv_base + i] = in[i];
}

// ------------------------------------------------------------------------------
// Column sort with the fused epilogue: each CTA sorts one column on chip (the
// m T(m) term) and, from the sorted column in shared memory, writes the
// position of every bucket-tile boundary (every kTB-th bucket, with the
// equal-pivot rule) and folds the column head into min(D).
struct ColDesc {
  uint32_t off, len, seg, col;
};

// resident CTAs per SM the counting-sort kernels are compiled for (64 registers)
template <typename K, int NT, int V, bool PAIRS, bool BIN>
__host__ __device__ constexpr int bin_min_blocks() {
  // (64-bit sort keys: no register cap; their tiles' shared memory allows ~1 CTA per SM)
  return (BIN && bin_ok<K, V, PAIRS>() && sizeof(sortkey_t<K, PAIRS>) == 4) ? (NT >= 1024 ? 1 : 1024 / NT) : 1;
}

template <typename K, int NT, int V, bool PAIRS, bool BIN>
__global__ void __launch_bounds__(NT, (bin_min_blocks<K, NT, V, PAIRS, BIN>()))
k_colsort(const ColDesc* __restrict__ cols, const LevelSeg* __restrict__ segs, K* __restrict__ keys,
          uint32_t* __restrict__ vals, const K* __restrict__ piv, uint32_t* __restrict__ segmat,
          K* __restrict__ segmin) {
  using SK = sortkey_t<K, PAIRS>;
  using BS = BlockSort<SK, NT, V, 32>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SK* s = reinterpret_cast<SK*>(smem_raw);
  uint32_t* vs = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES);
  auto TP = [](uint32_t i) { return tpos<K, NT, V, PAIRS, BIN>(i); };
  const ColDesc d = cols[blockIdx.x];
  const LevelSeg sg = segs[d.seg];
  constexpr int VW = 16 / sizeof(K), NV = BS::TILE / (NT * VW);  // 16-byte vectors per thread
  constexpr bool VEC = !PAIRS && NV >= 1 && NV * NT * VW == BS::TILE;
  const bool vec_ok = VEC && d.len == BS::TILE && (reinterpret_cast<uintptr_t>(keys + d.off) & 15) == 0;
  bool sorted = false;
  // the counting sort's counters follow the tile (and, for pairs, the values)
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES + (PAIRS ? size_t(BS::TILE) * 4 : 0));
  if constexpr (BIN && bin_ok<K, V, PAIRS>() && !PAIRS) {
    if (vec_ok) {  // full, aligned column: straight from 16-byte loads into the sort's registers
      static_assert(NV * VW == V, "vector loads fill the thread's keys");
      K r[V];
      const uint4* g = reinterpret_cast<const uint4*>(keys + d.off);
#pragma unroll
      for (int q = 0; q < NV; q++) {
        const uint4 x = g[threadIdx.x + q * NT];
        if constexpr (sizeof(K) == 4) {
          r[4 * q] = x.x;
          r[4 * q + 1] = x.y;
          r[4 * q + 2] = x.z;
          r[4 * q + 3] = x.w;
        } else {
          r[2 * q] = (uint64_t(x.y) << 32) | x.x;
          r[2 * q + 1] = (uint64_t(x.w) << 32) | x.z;
        }
      }
      BinSortOf<K, NT, V, PAIRS>::sort_regs(r, s, cnt, d.len,
                                            [&](int j) { return (threadIdx.x + (j / VW) * NT) * VW + (j % VW); });
      sorted = true;
    }
  }
  if (!sorted) {
    if (vec_ok) {
      // full, aligned column: every vector load in flight before the first store
      const uint4* g = reinterpret_cast<const uint4*>(keys + d.off);
      uint4 v[NV > 0 ? NV : 1];
#pragma unroll
      for (int q = 0; q < NV; q++) v[q] = g[threadIdx.x + q * NT];
#pragma unroll
      for (int q = 0; q < NV; q++) {
        const uint32_t i0 = (threadIdx.x + q * NT) * VW;
        const K* e = reinterpret_cast<const K*>(&v[q]);
#pragma unroll
        for (int j = 0; j < VW; j++) s[TP(i0 + j)] = SK(e[j]);
      }
    } else {
      for (int i = threadIdx.x; i < BS::TILE; i += NT) {
        SK x = KeyTraits<SK>::kMax;
        if (i < (int)d.len) {
          if constexpr (PAIRS) {
            x = (SK(keys[d.off + i]) << 32) | SK(uint32_t(i));
            vs[i] = vals[d.off + i];
          } else {
            x = keys[d.off + i];
          }
        }
        s[TP(i)] = x;
      }
    }
    __syncthreads();
    tile_sort<K, NT, V, PAIRS, BIN>(s, cnt, d.len);
  }
  // (programmatic dependent launch) the sampler must be done reading the unsorted
  // input, and the pivots must be selected, before this CTA writes or reads them
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  auto key_at = [&](int i) -> K {
    if constexpr (PAIRS) return K(s[TP(i)] >> 32);
    else return s[TP(i)];
  };
  bool stored = false;
  if constexpr (BIN && bin_ok<K, V, PAIRS>() && !PAIRS) {
    if (vec_ok) {  // 16-byte chunks of the swizzled tile
      uint4* g = reinterpret_cast<uint4*>(keys + d.off);
      for (uint32_t c = threadIdx.x; c < uint32_t(BS::TILE) / VW; c += NT)
        g[c] = BinSortOf<K, NT, V, PAIRS>::chunk(s, c);
      stored = true;
    }
  }
  if (!stored)
  for (int i = threadIdx.x; i < (int)d.len; i += NT) {
    const SK x = s[TP(i)];
    if constexpr (PAIRS) {
      keys[d.off + i] = K(x >> 32);
      vals[d.off + i] = vs[uint32_t(x)];
    } else {
      keys[d.off + i] = x;
    }
  }
  // epilogue: tile boundaries of this column
  const K* P = piv + sg.piv_base;
  uint32_t* row = segmat + sg.segmat_base + d.col;  // tile-major: entry (bt, c) at bt * ncols + c
  for (uint32_t bt = threadIdx.x; bt <= sg.nbt; bt += NT) {
    uint32_t pos;
    const uint32_t j = bt * kTB;  // boundary index (bucket j starts here)
    if (bt == 0) pos = 0;
    else if (j >= sg.k) pos = d.len;
    else {
      const K pj = P[j - 1];
      const bool dup = j >= 2 && P[j - 2] == pj;
      uint32_t lo = 0, hi = d.len;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (before_boundary(key_at(mid), pj, dup)) lo = mid + 1; else hi = mid;
      }
      pos = lo;
    }
    row[uint64_t(bt) * sg.ncols] = pos;
  }
  if (threadIdx.x == 0 && d.len) {
    if constexpr (sizeof(K) == 4) atomicMin((unsigned int*)&segmin[d.seg], (unsigned int)key_at(0));
    else atomicMin((unsigned long long*)&segmin[d.seg], (unsigned long long)key_at(0));
  }
}

// Tile boundaries from sorted columns in global memory: used when the columns
// were sorted by a recursive level (too long for one CTA) and to repair the
// rare min-exclusion rejection (only segments with fix[seg] set, if `only_fix`).
template <typename K>
__global__ void k_segmat(const LevelSeg* __restrict__ segs, const TaskDesc* __restrict__ tasks,
                         const K* __restrict__ data, const K* __restrict__ piv, uint32_t* __restrict__ segmat,
                         const uint32_t* __restrict__ fix, int only_fix) {
  const TaskDesc tk = tasks[blockIdx.x];
  if (only_fix && !fix[tk.seg]) return;
  const LevelSeg sg = segs[tk.seg];
  const K* P = piv + sg.piv_base;
  for (uint32_t c = tk.a; c < tk.b; c++) {
    const uint64_t a = uint64_t(c) * sg.rows;
    const uint32_t L = (uint32_t)(a < sg.len ? min((uint64_t)sg.rows, (uint64_t)(sg.len - a)) : 0);
    const K* col = data + sg.off + a;
    uint32_t* row = segmat + sg.segmat_base + c;  // tile-major
    for (uint32_t bt = threadIdx.x; bt <= sg.nbt; bt += blockDim.x) {
      const uint32_t j = bt * kTB;
      uint32_t pos;
      if (bt == 0) pos = 0;
      else if (j >= sg.k) pos = L;
      else {
        const K pj = P[j - 1];
        const bool dup = j >= 2 && P[j - 2] == pj;
        uint32_t lo = 0, hi = L;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (before_boundary(col[mid], pj, dup)) lo = mid + 1; else hi = mid;
        }
        pos = lo;
      }
      row[uint64_t(bt) * sg.ncols] = pos;
    }
  }
}

// Keys per bucket tile (sum of the tile's run in every column), and the tile's piece
// count: the piece plan's windows (plan_fw columns each) cut into pieces of at most
// S keys -- counted here so that k_piece_dense can give every tile its place in the
// dense piece list before the plan runs.  CTA per tile.
__host__ __device__ __forceinline__ uint32_t plan_fw(uint32_t size, uint32_t ncols, uint32_t S, uint32_t FWMAX);
template <int S, int FW>
__global__ void k_tile_sizes(const LevelSeg* __restrict__ segs, TileInfo* __restrict__ tiles,
                             const uint32_t* __restrict__ segmat) {
  constexpr int PL = (FW + 31) / 32;
  TileInfo ti = tiles[blockIdx.x];
  const LevelSeg sg = segs[ti.seg];
  const uint32_t* rows = segmat + sg.segmat_base + uint64_t(ti.bt) * sg.ncols;  // tile-major
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t sum = 0;
  for (uint32_t c = threadIdx.x; c < sg.ncols; c += blockDim.x) sum += rows[c + sg.ncols] - rows[c];
  __shared__ uint32_t red[32];
  __shared__ uint32_t tsize;
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[w] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    sum = threadIdx.x < nw ? red[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (threadIdx.x == 0) tsize = sum;
  }
  __syncthreads();
  const uint32_t size = tsize;
  const uint32_t fw = plan_fw(size, sg.ncols, S, FW), nwin = (sg.ncols + fw - 1) / fw;
  uint32_t cnt = 0;
  for (uint32_t win = w; win < nwin; win += nw) {  // warp per window, as in the plan
    uint32_t ws = 0;
#pragma unroll
    for (int q = 0; q < PL; q++) {
      const uint32_t j = lane * PL + q, c = win * fw + j;
      if (j < fw && c < sg.ncols) ws += rows[c + sg.ncols] - rows[c];
    }
    for (int o = 16; o; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
    cnt += (ws + S - 1) / S;
  }
  __syncthreads();
  if (lane == 0) red[w] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t c = 0;
    for (int q = 0; q < nw; q++) c += red[q];
    tiles[blockIdx.x].size = size;
    tiles[blockIdx.x].dense = c;
  }
}

// Dense piece list: exclusive scan of the tiles' piece counts in tile order (one
// CTA); the total is the transpose's piece count.
static __global__ void k_piece_dense(TileInfo* __restrict__ tiles, uint32_t ntiles, uint32_t* __restrict__ pcount) {
  __shared__ uint32_t misc[64];
  uint32_t carry = 0;
  for (uint32_t c0 = 0; c0 < ntiles; c0 += blockDim.x) {
    const uint32_t i = c0 + threadIdx.x;
    const uint32_t v = i < ntiles ? tiles[i].dense : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_sum<32>(v, misc, &tot);
    if (i < ntiles) tiles[i].dense = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) pcount[0] = carry;
}

// Per segment: tile output offsets (exclusive scan of sizes) and piece-table
// bases (capacity ceil(size/S) + ceil(ncols/G) pieces per tile).  Also resets
// the per-segment bucket bookkeeping.  One CTA per segment (tiles contiguous).
// Piece-plan window of a bucket tile: columns per window chosen so that a window
// holds ~31/32 of a piece on average (runs average size/ncols keys), at most FWMAX.
__host__ __device__ __forceinline__ uint32_t plan_fw(uint32_t size, uint32_t ncols, uint32_t S, uint32_t FWMAX) {
  if (!size) return FWMAX;
  const uint64_t fw = (uint64_t(S) * 31 / 32) * ncols / size;
  // at least 32 columns: a huge tile (low-cardinality input) gets windows of many
  // pieces rather than one window per column, so its plan is not a serial walk
  return (uint32_t)max((uint64_t)min(32u, FWMAX), min((uint64_t)FWMAX, fw));
}

static __global__ void k_tile_scan(const LevelSeg* __restrict__ segs, const uint32_t* __restrict__ tile_base,
                            TileInfo* __restrict__ tiles, uint32_t S, uint32_t G,
                            const uint32_t* __restrict__ piece_seg_base, uint32_t* __restrict__ pcount) {
  const LevelSeg sg = segs[blockIdx.x];
  const uint32_t t0 = tile_base[blockIdx.x], nt = sg.nbt;
  __shared__ uint32_t carry_out, carry_piece;
  if (threadIdx.x == 0) {
    carry_out = sg.off;
    carry_piece = piece_seg_base[blockIdx.x];
  }
  __syncthreads();
  for (uint32_t c0 = 0; c0 < nt; c0 += blockDim.x) {
    const uint32_t i = c0 + threadIdx.x;
    uint32_t sz = 0, cp = 0;
    if (i < nt) {
      sz = tiles[t0 + i].size;
      const uint32_t fw = plan_fw(sz, sg.ncols, S, G);
      cp = (sz + S - 1) / S + (sg.ncols + fw - 1) / fw;
    }
    // block scan of (sz, cp)
    __shared__ uint32_t ws[32], wc[32];
    uint32_t xs = sz, xc = cp;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t ys = __shfl_up_sync(0xffffffffu, xs, o), yc = __shfl_up_sync(0xffffffffu, xc, o);
      if (lane >= o) { xs += ys; xc += yc; }
    }
    if (lane == 31) { ws[w] = xs; wc[w] = xc; }
    __syncthreads();
    if (w == 0) {
      const int nw = blockDim.x >> 5;
      uint32_t a = lane < nw ? ws[lane] : 0, b = lane < nw ? wc[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
        if (lane >= o) { a += ya; b += yb; }
      }
      if (lane < nw) { ws[lane] = a; wc[lane] = b; }
    }
    __syncthreads();
    const uint32_t es = xs - sz + (w ? ws[w - 1] : 0), ec = xc - cp + (w ? wc[w - 1] : 0);
    if (i < nt) {
      tiles[t0 + i].out = carry_out + es;
      tiles[t0 + i].piece_base = carry_piece + ec;
      tiles[t0 + i].npieces = 0;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_out += es + sz;
      carry_piece += ec + cp;
    }
    __syncthreads();
  }
  // one-segment levels (pcount given; 256 threads): the dense piece list too, so that
  // k_piece_dense is not a launch of its own
  if (pcount) {
    __shared__ uint32_t misc[64];
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < nt; c0 += blockDim.x) {
      const uint32_t i = c0 + threadIdx.x;
      const uint32_t v = i < nt ? tiles[t0 + i].dense : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_sum<8>(v, misc, &tot);
      if (i < nt) tiles[t0 + i].dense = carry + ex;
      carry += tot;
    }
    if (threadIdx.x == 0) pcount[0] = carry;
  }
}

// ------------------------------------------------------------------------------
// TMA helpers (cp.async.bulk: SASS UBLKCP) and an mbarrier.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  // try_wait with a suspend-time hint: a waiting warp sleeps in hardware until the
  // phase completes (or the hint expires) instead of spinning on issue slots
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// shared -> global bulk copy (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(smem_addr(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }


template <typename K> struct Thr;
template <> struct Thr<uint32_t> {
  uint64_t t;
  __device__ __forceinline__ static Thr make(uint32_t p, bool dup, bool inf) {
    return Thr{inf ? ~0ull : uint64_t(p) + (dup ? 1u : 0u)};
  }
  __device__ __forceinline__ bool passed(uint32_t x) const { return uint64_t(x) >= t; }
};
template <> struct Thr<uint64_t> {
  uint64_t p, dup;  // dup = 2: never passed (sentinel)
  __device__ __forceinline__ static Thr make(uint64_t p, bool dup, bool inf) { return Thr{p, inf ? 2ull : (dup ? 1ull : 0ull)}; }
  __device__ __forceinline__ bool passed(uint64_t x) const { return dup != 2 && (x > p || (x == p && dup == 0)); }
};

// ------------------------------------------------------------------------------
// Piece plan: the piece boundaries of every bucket tile depend only on the run
// lengths (segmat), so a light pre-pass (one CTA per tile) computes them with the
// same window rule as k_transpose_ms (up to S keys from up to F runs), and the
// transpose then processes pieces as independent work items (no serial chain per
// tile, no wave tail).
// Self-contained piece descriptor (the transpose needs no other metadata load):
// fragment f (f < nf) is the run of bucket tile `bt` in column col+f, whose key
// run is [segmat[row0 + f], segmat[row0 + f + rstride]) within its column (segmat is
// tile-major: entry (bt, c) at bt * ncols + c), keys src0 + f*rows + that (+ off for f = 0).
struct __align__(16) PieceDesc {
  uint32_t pn, out, nf, off;         // keys, output offset, runs, offset into the first run
  uint32_t src0, rows, row0, rstride;  // first column's start; column length; segmat index of (bt, col); ncols
  uint32_t nb, thr0, slot, bt;       // buckets in the tile, pivot index of its first boundary, piece table slot, tile
  uint32_t bbase;                    // index of the tile's first bucket in the level's bucket arrays
};

// Piece plan, parallel form: every bucket tile's stream is cut into windows of FW
// consecutive columns; a window of T keys gives ceil(T / S) pieces (one for the
// usual T <= S), cut at stream positions that are multiples of S.  CTA per tile;
// warps work on windows independently (no serial chain over the tile).
// The pieces are listed in tile order: the transpose takes list positions in
// order, so the two pieces that share a column's boundary sectors (tiles bt and
// bt+1 of one window) run close together in time and the shared sectors are read
// from DRAM once (an arbitrary tile order doubled the transpose's DRAM reads).
template <int NT, int S, int FW>
__global__ void __launch_bounds__(NT)
k_piece_plan2(const LevelSeg* __restrict__ segs, TileInfo* __restrict__ tiles, const uint32_t* __restrict__ segmat,
              PieceDesc* __restrict__ pieces, uint32_t* __restrict__ pout) {
  constexpr int NW = NT / 32, PL = (FW + 31) / 32;  // columns per lane within a window
  constexpr uint32_t MAXW = 1024;                    // windows per chunk
  static_assert(FW <= 128, "window");
  __shared__ uint32_t wtot[MAXW], wpc[MAXW], woff[MAXW], wpb[MAXW];
  __shared__ uint32_t misc[64];
  __shared__ uint32_t carry_o, carry_p;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t me = blockIdx.x;
  const TileInfo ti = tiles[me];
  const uint32_t base = ti.dense;  // the tile's first position in the dense piece list
  const LevelSeg sg = segs[ti.seg];
  const uint32_t bt = ti.bt, rstride = sg.ncols;  // tile-major segmat: (bt+1, c) is ncols after (bt, c)
  const uint32_t* rows = segmat + sg.segmat_base + uint64_t(bt) * sg.ncols;
  const uint32_t fw = plan_fw(ti.size, sg.ncols, S, FW);  // columns per window (<= FW)
  const uint32_t nwin = (sg.ncols + fw - 1) / fw;
  const uint32_t nb = min((uint32_t)kTB, sg.k - bt * kTB);
  auto run_len = [&](uint32_t c) -> uint32_t {
    if (c >= sg.ncols) return 0u;
    return rows[c + rstride] - rows[c];
  };
  if (t == 0) {
    carry_o = 0;
    carry_p = 0;
  }
  __syncthreads();
  for (uint32_t w0 = 0; w0 < nwin; w0 += MAXW) {
    const uint32_t nw = min(MAXW, nwin - w0);
    for (uint32_t wi = w; wi < nw; wi += NW) {  // window totals
      const uint32_t win = w0 + wi;
      uint32_t sum = 0;
#pragma unroll
      for (int q = 0; q < PL; q++) {
        const uint32_t j = lane * PL + q;
        if (j < fw) sum += run_len(win * fw + j);
      }
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) {
        wtot[wi] = sum;
        wpc[wi] = (sum + S - 1) / S;
      }
    }
    __syncthreads();
    {  // exclusive scans over the windows of the chunk: stream offsets and piece indices
      uint32_t co = carry_o, cp = carry_p;
      for (uint32_t c0 = 0; c0 < nw; c0 += NT) {
        const uint32_t i = c0 + t;
        const uint32_t a = i < nw ? wtot[i] : 0u, b = i < nw ? wpc[i] : 0u;
        uint32_t ta, tb;
        const uint32_t ea = block_excl_sum<NW>(a, misc, &ta);
        const uint32_t eb = block_excl_sum<NW>(b, misc + 32, &tb);
        if (i < nw) {
          woff[i] = co + ea;
          wpb[i] = cp + eb;
        }
        co += ta;
        cp += tb;
      }
      __syncthreads();
      if (t == 0) {
        carry_o = co;
        carry_p = cp;
      }
      __syncthreads();
    }
    for (uint32_t wi = w; wi < nw; wi += NW) {  // emit the pieces of each window
      const uint32_t win = w0 + wi;
      const uint32_t T = wtot[wi], npc = wpc[wi];
      if (!npc) continue;
      const uint32_t c0 = win * fw, ncw = min(fw, sg.ncols - c0);
      // run lengths of the window's columns, lane-major (lane holds PL columns)
      uint32_t lens[PL], incl[PL], acc = 0;
#pragma unroll
      for (int q = 0; q < PL; q++) {
        lens[q] = (lane * PL + q < ncw) ? run_len(c0 + lane * PL + q) : 0u;
        acc += lens[q];
        incl[q] = acc;
      }
      uint32_t x = acc;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t lane_ex = x - acc;  // keys before this lane's first column
      for (uint32_t p = 0; p < npc; p++) {
        const uint32_t sp = p * S, ep = min(sp + S, T);  // stream range [sp, ep) of the window
        // first column holding stream position sp; last column with keys before ep
        uint32_t cfirst = 0xffffffffu, clast = 0, offs = 0;
#pragma unroll
        for (int q = 0; q < PL; q++) {
          const uint32_t j = lane * PL + q;
          const uint32_t ex = lane_ex + incl[q] - lens[q], in = lane_ex + incl[q];
          if (j < ncw && in > sp && ex <= sp && lens[q]) {
            cfirst = j;
            offs = sp - ex;
          }
          if (j < ncw && ex < ep) clast = j;
        }
        const uint32_t cf = __reduce_min_sync(0xffffffffu, cfirst);
        const uint32_t cl = __reduce_max_sync(0xffffffffu, clast);
        const uint32_t of = __shfl_sync(0xffffffffu, offs, cf / PL);
        if (lane == 0) {
          const uint32_t j = wpb[wi] + p;  // piece index within the tile
          const uint32_t pe = ti.piece_base + j, oc = ti.out + woff[wi] + sp;
          const uint32_t col = c0 + cf;
          pieces[base + j] = PieceDesc{ep - sp, oc, cl - cf + 1, of, sg.off + col * sg.rows, sg.rows,
                                       (uint32_t)(sg.segmat_base + uint64_t(bt) * sg.ncols + col), rstride, nb,
                                       sg.piv_base + bt * kTB, pe, bt, sg.buck_base + bt * kTB};
          pout[pe] = oc;
        }
      }
    }
    __syncthreads();
  }
  SQ_CHECK(t != 0 || me + 1 >= gridDim.x || carry_p == tiles[me + 1].dense - base);
  if (t == 0) tiles[me].npieces = carry_p;
}

// ------------------------------------------------------------------------------
// Bucket planning, per segment (one CTA): bucket sizes from the piece tables,
// final offsets (exclusive scan, P:283 / P:461), RNG node keys, and the work
// lists: single-value buckets (copy), on-chip classes, oversize.
struct Unit {
  uint32_t tile, j0, j1, out, size;  // buckets j0..j1 (lanes) of a tile, their output start and total
};
constexpr uint32_t kUnitFlag = 0x80000000u;

struct PlanOut {
  uint32_t* list;       // [ncls + 2][cap_per_list] work items (bucket * 16 + chunk)
  uint32_t* count;      // [ncls + 2] atomic counters; ncls = copy list, ncls+1 = oversize
  uint32_t cap_per_list;
  uint32_t ncls;
  uint32_t cls_tile[20];  // class tile sizes (ascending)
  uint32_t max_tile;      // largest bucket sorted by one CTA
  // merge-sort base case for max_tile < size <= msort_max: chunks of <= max_tile keys,
  // sorted by one CTA each, then up to kMaxPasses merge passes with tiles of mtile keys
  uint32_t msort_max;
  uint32_t mtile;
  MTile* mlist;           // [kMaxPasses][mcap]
  uint32_t* mcount;       // [kMaxPasses]
  uint32_t mcap;
  // units: consecutive buckets of one tile, each of at most max_tile keys, packed
  // into work items of at most max_tile keys (their keys are value-ordered ranges,
  // so sorting the concatenation sorts every bucket); items are kUnitFlag | index
  Unit* units;
  uint32_t* nunits;
  uint32_t unit_max;  // largest unit (and bucket packed into units): the biggest one-CTA class
  // value split (mode 4): inner buckets of max_tile < size <= split_max keys go to
  // list split_list as ceil(size / split_part) value-range items (k_bucketsplit)
  uint32_t split_max;
  uint32_t split_part;
  uint32_t split_list;
};

// Bucket plan, one warp per bucket tile: lane j takes bucket j of the tile; its final offset is the tile's
// offset plus the sizes of the tile's earlier buckets (a warp scan -- the tile
// offsets are already the segment's prefix, P:283 / P:461); then the records and
// work lists (single-value, size classes, merge chunks and tiles, oversize), and lane 0 packs the small buckets into units.
template <typename K>
__global__ void k_tile_bucket_plan(const LevelSeg* __restrict__ segs, const TileInfo* __restrict__ tiles,
                                   uint32_t ntiles, const uint32_t* __restrict__ bsize, const K* __restrict__ piv,
                                   BucketRec* __restrict__ recs, PlanOut po) {
  const uint32_t ti_idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (ti_idx >= ntiles) return;  // warp-uniform
  const TileInfo ti = tiles[ti_idx];
  const LevelSeg sg = segs[ti.seg];
  const uint32_t nb = min((uint32_t)kTB, sg.k - ti.bt * kTB);
  const uint32_t b = ti.bt * kTB + lane, gi = sg.buck_base + b;
  const uint32_t size = lane < nb ? bsize[gi] : 0u;
  uint32_t x = size;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const uint32_t out = ti.out + x - size;
  if (lane < nb) {
    const K* P = piv + sg.piv_base;
    BucketRec rc;
    rc.tile = ti_idx;
    rc.lane = lane;
    rc.out = out;
    rc.size = size;
    rc.node = child_key(sg.node, 1, b);
    rc.chunk = size;
    rc.passes = 0;
    const bool single = b >= 1 && b + 1 < sg.k && P[b - 1] == P[b];
    const bool vsplit = !single && b >= 1 && b + 1 < sg.k && size > po.max_tile && size <= po.split_max;
    uint32_t q = 1;  // chunks
    const uint32_t chunk_len = po.max_tile;
    if (vsplit) {
      rc.chunk = (size + po.split_part - 1) / po.split_part;  // value ranges
      const uint32_t slot = atomicAdd(&po.count[po.split_list], rc.chunk);
      for (uint32_t k = 0; k < rc.chunk; k++) po.list[uint64_t(po.split_list) * po.cap_per_list + slot + k] = gi * 16 + k;
    } else if (size && !single && size > po.max_tile && size <= po.msort_max) {
      q = (size + chunk_len - 1) / chunk_len;
      rc.chunk = chunk_len;  // full chunks; the last one takes the remainder
      uint32_t np = 0;
      while ((1u << np) < q) np++;
      rc.passes = np;
      for (uint32_t p = 0; p < np; p++) {  // merge tiles of every pass
        const uint32_t R = rc.chunk << p;
        uint32_t ntile = 0;
        for (uint32_t j = 0; 2 * j * R < size; j++)
          ntile += (min(size, (2 * j + 2) * R) - 2 * j * R + po.mtile - 1) / po.mtile;
        uint32_t slot = atomicAdd(&po.mcount[p], ntile);
        for (uint32_t j = 0; 2 * j * R < size; j++) {
          const uint32_t plen = min(size, (2 * j + 2) * R) - 2 * j * R;
          for (uint32_t t = 0; t * po.mtile < plen; t++)
            po.mlist[uint64_t(p) * po.mcap + slot++] = MTile{gi, (uint16_t)j, (uint16_t)t};
        }
      }
    }
    recs[gi] = rc;
    if (size && !vsplit && !(po.units && size <= po.unit_max)) {  // else packed into a unit below
      if (single || size > po.msort_max) {
        const int cls = single ? po.ncls : po.ncls + 1;
        const uint32_t slot = atomicAdd(&po.count[cls], 1u);
        po.list[uint64_t(cls) * po.cap_per_list + slot] = gi * 16;
      } else {
        const uint32_t lbase = rc.passes ? po.ncls + 3 : 0;  // chunks of merge-sorted buckets: own lists
        for (uint32_t k = 0; k < q; k++) {
          const uint32_t len = min(rc.chunk, size - k * rc.chunk);
          uint32_t cls = 0;
          while (po.cls_tile[cls] < len) cls++;
          cls += lbase;
          const uint32_t slot = atomicAdd(&po.count[cls], 1u);
          po.list[uint64_t(cls) * po.cap_per_list + slot] = gi * 16 + k;
        }
      }
    }
  }
  if (!po.units) return;
  // units: greedy, in bucket order, at most unit_max keys each.  Every lane walks the
  // same (warp-uniform) packing; the lane of a unit's first bucket keeps the unit, and
  // the units are then published by their lanes in parallel (one atomic for the
  // tile's unit count, one per unit for its class list) instead of serially by lane 0
  // -- the plan is on the critical path of small levels.
  uint32_t j0 = 0, acc = 0, out0 = 0;
  uint32_t my_j1 = 0, my_acc = 0, my_out = 0;  // the unit starting at this lane's bucket
  auto flush = [&](uint32_t j1) {  // buckets j0..j1-1
    if (acc && lane == j0) {
      my_j1 = j1 - 1;
      my_acc = acc;
      my_out = out0;
    }
  };
  for (uint32_t j = 0; j < nb; j++) {
    const uint32_t sz = __shfl_sync(0xffffffffu, size, j), o = __shfl_sync(0xffffffffu, out, j);
    const bool small = sz <= po.unit_max;
    if (!small || acc + sz > po.unit_max) {
      flush(j);
      acc = 0;
    }
    if (small && sz) {
      if (!acc) {
        j0 = j;
        out0 = o;
      }
      acc += sz;
    }
  }
  flush(nb);
  const uint32_t has = __ballot_sync(0xffffffffu, my_acc != 0);
  if (!has) return;
  uint32_t ubase = 0;
  if (lane == 0) ubase = atomicAdd(po.nunits, (uint32_t)__popc(has));
  ubase = __shfl_sync(0xffffffffu, ubase, 0);
  if (my_acc) {
    const uint32_t u = ubase + __popc(has & ((1u << lane) - 1));
    po.units[u] = Unit{ti_idx, lane, my_j1, my_out, my_acc};
    int cls = 0;
    while (po.cls_tile[cls] < my_acc) cls++;
    const uint32_t slot = atomicAdd(&po.count[cls], 1u);
    po.list[uint64_t(cls) * po.cap_per_list + slot] = kUnitFlag | u;
  }
}

// Gather the bucket positions [lo, hi) (piece order = the paper's order) of a
// bucket: copy_chunk(global_offset, length, position - lo, lane) is called for
// every intersecting sub-chunk, one warp per sub-chunk.
template <int NT, typename F>
__device__ __forceinline__ void gather_bucket(const TileInfo& ti, uint32_t lane_j, const uint32_t* __restrict__ pout,
                                              const uint16_t* __restrict__ ppre, uint32_t* s_off, uint32_t* s_len,
                                              uint32_t* s_dst, uint32_t* misc, uint32_t lo, uint32_t hi,
                                              F&& copy_chunk, uint32_t lane_end = 0) {
  if (!lane_end) lane_end = lane_j + 1;  // buckets [lane_j, lane_end) of the tile
  constexpr int NW = NT / 32;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t base = 0;
  for (uint32_t c0 = 0; c0 < ti.npieces && base < hi; c0 += NT) {
    const uint32_t q = c0 + t;
    uint32_t o = 0, l = 0;
    if (q < ti.npieces) {
      const uint16_t* pr = ppre + uint64_t(ti.piece_base + q) * kPP;
      const uint32_t a = pr[lane_j], e = pr[lane_end];
      o = pout[ti.piece_base + q] + a;
      l = e - a;
    }
    uint32_t tot;
    const uint32_t ex = block_excl_sum<NW>(l, misc, &tot);
    if (q < ti.npieces) {
      // clip [base+ex, base+ex+l) to [lo, hi)
      const uint32_t p0 = base + ex, p1 = p0 + l;
      const uint32_t c0c = max(p0, lo), c1c = min(p1, hi);
      s_off[t] = o + (c0c - p0);
      s_len[t] = c1c > c0c ? c1c - c0c : 0;
      s_dst[t] = c0c - lo;
    }
    __syncthreads();
    const uint32_t nq = min((uint32_t)NT, ti.npieces - c0);
    for (uint32_t c = w; c < nq; c += NW)
      if (s_len[c]) copy_chunk(s_off[c], s_len[c], s_dst[c], lane);
    base += tot;
    __syncthreads();
  }
}

// Bucket sort with gather: CTA loops over its class list.  An item is a
// whole bucket or one chunk of a merge-sorted bucket; chunks of a bucket with an
// odd number of merge passes go to `dst_odd`, so the last pass ends in `dst`.
template <typename K, int NT, int V, bool PAIRS, bool BIN>
__global__ void __launch_bounds__(NT, (bin_min_blocks<K, NT, V, PAIRS, BIN>()))
k_bucketsort(const BucketRec* __restrict__ recs, const TileInfo* __restrict__ tiles, const uint32_t* __restrict__ list,
             const uint32_t* __restrict__ count, const K* __restrict__ src, K* __restrict__ dst,
             const uint32_t* __restrict__ vsrc, uint32_t* __restrict__ vdst, const uint32_t* __restrict__ pout,
             const uint16_t* __restrict__ ppre, K* __restrict__ dst_odd, uint32_t* __restrict__ vdst_odd,
             const Unit* __restrict__ units) {
  using SK = sortkey_t<K, PAIRS>;
  using BS = BlockSort<SK, NT, V>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SK* s = reinterpret_cast<SK*>(smem_raw);
  uint32_t* vs = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES + (PAIRS ? BS::TILE * 4 : 0));
  uint32_t* s_len = s_off + NT;
  uint32_t* s_dst = s_len + NT;
  uint32_t* misc = s_dst + NT;
  uint32_t* cnt = misc + 64;  // counting-sort counters (BIN)
  auto TP = [](uint32_t i) { return tpos<K, NT, V, PAIRS, BIN>(i); };
  const uint32_t total = *count;
  for (uint32_t it = blockIdx.x; it < total; it += gridDim.x) {
    const uint32_t e = list[it];
    uint32_t tile, lane0, lane1, lo, hi, outpos, passes;
    if (e & kUnitFlag) {  // packed run of whole buckets
      const Unit u = units[e & ~kUnitFlag];
      tile = u.tile;
      lane0 = u.j0;
      lane1 = u.j1 + 1;
      lo = 0;
      hi = u.size;
      outpos = u.out;
      passes = 0;
    } else {
      const BucketRec rc = recs[item_bucket(e)];
      tile = rc.tile;
      lane0 = rc.lane;
      lane1 = rc.lane + 1;
      lo = item_chunk(e) * rc.chunk;
      hi = min(rc.size, lo + rc.chunk);
      outpos = rc.out;
      passes = rc.passes;
    }
    const TileInfo ti = tiles[tile];
    const uint32_t len = hi - lo;
    K* out = (passes & 1) ? dst_odd : dst;
    uint32_t* vout = (passes & 1) ? vdst_odd : vdst;
    for (int i = threadIdx.x + len; i < BS::TILE; i += NT) s[TP(i)] = KeyTraits<SK>::kMax;
    gather_bucket<NT>(ti, lane0, pout, ppre, s_off, s_len, s_dst, misc, lo, hi,
                      [&](uint32_t o, uint32_t l, uint32_t d, int ln) {
                        SQ_CHECK(d + l <= uint32_t(BS::TILE) && o >= ti.out && o + l <= ti.out + ti.size);
                        for (uint32_t q = ln; q < l; q += 32) {
                          if constexpr (PAIRS) {
                            // key into the low half of the composite slot, fixed up below
                            cp_async_elem(reinterpret_cast<K*>(&s[TP(d + q)]), &src[o + q]);
                            cp_async_elem(&vs[d + q], &vsrc[o + q]);
                          } else {
                            cp_async_elem(&s[TP(d + q)], &src[o + q]);
                          }
                        }
                      },
                      lane1);
    cp_async_wait_all();
    __syncthreads();
    if constexpr (PAIRS) {  // composite = key << 32 | position (stable order)
      for (int i = threadIdx.x; i < (int)len; i += NT) {
        const K key = *reinterpret_cast<K*>(&s[TP(i)]);
        s[TP(i)] = (SK(key) << 32) | SK(uint32_t(i));
      }
      __syncthreads();
    }
    SQ_CHECK(len <= uint32_t(BS::TILE));
    tile_sort<K, NT, V, PAIRS, BIN>(s, cnt, len);
    for (int i = threadIdx.x; i < (int)len; i += NT) {
      const SK x = s[TP(i)];
      if constexpr (PAIRS) {
        out[outpos + lo + i] = K(x >> 32);
        vout[outpos + lo + i] = vs[uint32_t(x)];
      } else {
        out[outpos + lo + i] = x;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------
// Value-split sort of a bucket beyond one CTA (big-bucket mode 4, keys only).  An
// inner bucket b holds keys in [P[b-1], P[b]) (L2, L4: a single-value bucket b-1
// has taken x = P[b-1]), so the bucket is sorted by sorting q value ranges
// separately (P:291-293 applied to a split of the bucket's range instead of a
// second sample).  Item (bucket, j) owns [s_j, s_{j+1}), s_j = P[b-1] +
// floor(j (P[b] - P[b-1]) / q): its CTA reads the whole bucket (the q readers of a
// bucket run together, so the re-reads are L2 hits), keeps the keys of its range
// and counts the smaller ones (its output offset), sorts its keys on chip and
// writes them to their final place: every key crosses HBM twice and no merge pass
// runs.  A range with more keys than the tile is halved and re-read until it
// fits; a range of one value is written as copies of that value.
template <typename K>
__device__ __forceinline__ K split_point(K lo, K hi, uint32_t j, uint32_t q) {
  const K d = hi - lo;  // floor(j d / q) without overflow (j <= q <= 16)
  return lo + (d / q) * j + ((d % q) * j) / q;
}

template <typename K, int NT, int V, bool BIN>
__global__ void __launch_bounds__(NT, (bin_min_blocks<K, NT, V, false, BIN>()))
k_bucketsplit(const LevelSeg* __restrict__ segs, const K* __restrict__ piv, const BucketRec* __restrict__ recs,
              const TileInfo* __restrict__ tiles, const uint32_t* __restrict__ list,
              const uint32_t* __restrict__ count, const K* __restrict__ src, K* __restrict__ dst,
              const uint32_t* __restrict__ pout, const uint16_t* __restrict__ ppre) {
  using BS = BlockSort<K, NT, V>;
  constexpr int NW = NT / 32;
  constexpr uint32_t TILE = BS::TILE;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K* s = reinterpret_cast<K*>(smem_raw);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES);
  uint32_t* s_len = s_off + NT;
  uint32_t* s_dst = s_len + NT;
  uint32_t* misc = s_dst + NT;
  uint32_t* cnt = misc + 64;  // counting-sort counters (BIN)
  __shared__ uint32_t s_fill;
  auto TP = [](uint32_t i) { return tpos<K, NT, V, false, BIN>(i); };
  const uint32_t total = *count;
  for (uint32_t it = blockIdx.x; it < total; it += gridDim.x) {
    const uint32_t e = list[it];
    const BucketRec rc = recs[item_bucket(e)];
    const TileInfo ti = tiles[rc.tile];
    const LevelSeg sg = segs[ti.seg];
    const K* P = piv + sg.piv_base;
    const uint32_t b = ti.bt * kTB + rc.lane, q = rc.chunk, j = item_chunk(e);
    const K plo = P[b - 1], phi = P[b];
    K a = split_point(plo, phi, j, q), c = split_point(plo, phi, j + 1, q);
    K stk_a[8 * sizeof(K)], stk_c[8 * sizeof(K)];  // halves still to do (thread-uniform)
    int sp = 0;
    while (true) {
      if (a < c) {
        if (threadIdx.x == 0) s_fill = 0;
        __syncthreads();
        uint32_t below = 0;
        gather_bucket<NT>(ti, rc.lane, pout, ppre, s_off, s_len, s_dst, misc, 0u, rc.size,
                          [&](uint32_t o, uint32_t l, uint32_t, int ln) {
                            for (uint32_t q0 = 0; q0 < l; q0 += 128) {  // 4 loads in flight per lane
                              K x[4];
#pragma unroll
                              for (int u = 0; u < 4; u++) {
                                const uint32_t qq = q0 + u * 32 + ln;
                                x[u] = qq < l ? src[o + qq] : c;
                              }
#pragma unroll
                              for (int u = 0; u < 4; u++) {
                                below += x[u] < a;
                                const bool in = x[u] >= a && x[u] < c;
                                const uint32_t m = __ballot_sync(0xffffffffu, in);
                                if (!m) continue;
                                uint32_t base = 0;
                                if (ln == 0) base = atomicAdd(&s_fill, __popc(m));
                                base = __shfl_sync(0xffffffffu, base, 0);
                                const uint32_t pos = base + __popc(m & ((1u << ln) - 1u));
                                if (in && pos < TILE) s[TP(pos)] = x[u];
                              }
                            }
                          });
        uint32_t off;
        block_excl_sum<NW>(below, misc, &off);  // (its barriers also publish s_fill and the tile)
        const uint32_t len = s_fill;
        K* out = dst + rc.out + off;
        if (len <= TILE) {
          for (uint32_t i = threadIdx.x + len; i < TILE; i += NT) s[TP(i)] = KeyTraits<K>::kMax;
          __syncthreads();
          tile_sort<K, NT, V, false, BIN>(s, cnt, len);
          for (uint32_t i = threadIdx.x; i < len; i += NT) out[i] = s[TP(i)];
        } else if (c - a == 1) {
          for (uint32_t i = threadIdx.x; i < len; i += NT) out[i] = a;
        } else {  // too many keys: the lower half now, the upper half later
          const K mid = a + (c - a) / 2;
          stk_a[sp] = mid;
          stk_c[sp] = c;
          sp++;
          c = mid;
          __syncthreads();
          continue;
        }
        __syncthreads();
      }
      if (!sp) break;
      sp--;
      a = stk_a[sp];
      c = stk_c[sp];
    }
  }
}

// ------------------------------------------------------------------------------
// Merge pass of the multi-CTA base case: an item is output tile t of the merge of
// runs 2j and 2j+1 (length R = chunk << pass) of one bucket.  The tile's input
// ranges come from two merge-path splits in global memory (32-ary warp search);
// they are staged in shared memory, merged (each thread VM outputs, ties from the
// earlier run: stable) and written back coalesced.  Buffers alternate so that the
// bucket's last pass writes its final place.
template <typename K>
struct GSeq {  // sorted run in global memory
  const K* p;
  uint32_t len;
  template <int PER>
  __device__ __forceinline__ K at(uint32_t i) const { return p[i]; }
};

// Merge-path split of every merge item of a pass, one thread per item (a binary
// search in global memory; all items in flight at once instead of one latency-bound
// search per CTA inside the merge kernel).  splits[it] = A keys before output tile it.
template <typename K>
__global__ void k_merge_split(const BucketRec* __restrict__ recs, const MTile* __restrict__ items,
                              const uint32_t* __restrict__ count, uint32_t pass, uint32_t TM,
                              const K* __restrict__ bufX, const K* __restrict__ bufU, uint32_t* __restrict__ splits) {
  const uint32_t total = *count;
  for (uint32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < total; it += gridDim.x * blockDim.x) {
    const MTile mt = items[it];
    const BucketRec rc = recs[mt.bucket];
    const uint32_t R = rc.chunk << pass;
    const bool src_is_U = ((rc.passes - pass) & 1) != 0;
    const K* src = src_is_U ? bufU : bufX;
    const uint32_t a0 = 2 * mt.pair * R;
    const uint32_t b0 = min(rc.size, a0 + R), b1 = min(rc.size, a0 + 2 * R);
    const K* A = src + rc.out + a0;
    const K* B = src + rc.out + b0;
    const uint32_t la = b0 - a0, lb = b1 - b0;
    const uint32_t d = mt.tile * TM;
    uint32_t lo = d > lb ? d - lb : 0, hi = min(d, la);
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (A[mid] <= B[d - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    splits[it] = lo;
  }
}

template <typename K, bool PAIRS, int NT, int VM>
__global__ void __launch_bounds__(NT, PAIRS ? 1 : (sizeof(K) == 8 ? 512 : 1024) / NT)  // 64 (u32) / 128 (u64) registers
k_merge_pass(const BucketRec* __restrict__ recs, const MTile* __restrict__ items, const uint32_t* __restrict__ count,
             uint32_t pass, K* __restrict__ bufX, K* __restrict__ bufU, uint32_t* __restrict__ vX,
             uint32_t* __restrict__ vU, const uint32_t* __restrict__ splits) {
  using SK = sortkey_t<K, PAIRS>;
  constexpr int TM = NT * VM;
  using BS = BlockSort<K, NT, VM>;  // padding helper only
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K* sk = reinterpret_cast<K*>(smem_raw);                        // TM (+pad) keys: A part then B part
  uint32_t* sv = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES);  // TM vals (pairs)
  __shared__ uint32_t split[2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t total = *count;
  for (uint32_t it = blockIdx.x; it < total; it += gridDim.x) {
    const MTile mt = items[it];
    const BucketRec rc = recs[mt.bucket];
    const uint32_t R = rc.chunk << pass;
    const bool src_is_U = ((rc.passes - pass) & 1) != 0;
    const K* src = src_is_U ? bufU : bufX;
    K* dst = src_is_U ? bufX : bufU;
    const uint32_t* vsrc = src_is_U ? vU : vX;
    uint32_t* vdst = src_is_U ? vX : vU;
    const uint32_t a0 = 2 * mt.pair * R;
    const uint32_t b0 = min(rc.size, a0 + R), b1 = min(rc.size, a0 + 2 * R);
    GSeq<K> A{src + rc.out + a0, b0 - a0}, B{src + rc.out + b0, b1 - b0};
    const uint32_t d0 = mt.tile * TM, d1 = min(d0 + TM, A.len + B.len);
    // the next item is the next output tile of the same pair, unless this is the last
    bool last = it + 1 >= total;
    if (!last) {
      const MTile nx = items[it + 1];
      last = nx.bucket != mt.bucket || nx.pair != mt.pair;
    }
    const uint32_t sa0 = splits[it], sa1 = last ? A.len : splits[it + 1];
    (void)split;
    (void)w;
    (void)lane;
    const uint32_t na = sa1 - sa0, nb = (d1 - sa1) - (d0 - sa0), sb0 = d0 - sa0;
    const uint32_t m = na + nb, dd = threadIdx.x * VM;
    K r[VM];
    uint32_t ri[VM];
    if (!PAIRS && m == (uint32_t)TM) {  // uniform across the CTA
      // keys only, full tile: A ascending at [0, na), B DESCENDING at [na, m)
      // (bitonic), so the merge needs no bounds checks (as in BlockSort; ties between
      // a phantom and a real key carry equal values, so keys-only output is
      // unaffected).  Partial tiles (the last of a pair) take the checked merge.
      for (uint32_t i = threadIdx.x; i < m; i += NT) {  // all loads in flight at once
        const bool fa = i < na;
        const uint32_t gi = fa ? a0 + sa0 + i : b0 + sb0 + (i - na);
        cp_async_elem(&sk[BS::pad(fa ? i : na + m - 1 - i)], &src[rc.out + gi]);
      }
      cp_async_wait_all();
      __syncthreads();
      if (dd < m) {
        uint32_t lo = dd > nb ? dd - nb : 0, hi = min(dd, na);
        while (lo < hi) {  // smallest i with A[i] > B[dd-1-i]; B[k] lives at m-1-k
          const uint32_t mid = (lo + hi) >> 1;
          const bool le = sk[BS::pad(mid)] <= sk[BS::pad(m - dd + mid)];
          lo = le ? mid + 1 : lo;
          hi = le ? hi : mid;
        }
        const uint32_t pa = lo, pb = m - 1 - (dd - lo);
        K a = sk[BS::pad(pa)];
        K b = nb ? sk[BS::pad(pb)] : KeyTraits<K>::kMax;
        uint32_t na_ = pa + 1, nb_ = pb - 1;
#pragma unroll
        for (int k = 0; k < VM; k++) {
          const bool takeA = a <= b;
          r[k] = takeA ? a : b;
          const uint32_t idx = takeA ? na_ : nb_;
          na_ += takeA ? 1u : 0u;
          nb_ -= takeA ? 0u : 1u;
          const K v = sk[BS::pad(idx)];
          a = takeA ? v : a;
          b = takeA ? b : v;
        }
      }
    } else {
      for (uint32_t i = threadIdx.x; i < m; i += NT) {  // all loads in flight at once
        const bool fa = i < na;
        const uint32_t gi = fa ? a0 + sa0 + i : b0 + sb0 + (i - na);
        cp_async_elem(&sk[BS::pad(i)], &src[rc.out + gi]);
        if (PAIRS) cp_async_elem(&sv[i], &vsrc[rc.out + gi]);
      }
      cp_async_wait_all();
      __syncthreads();
      // merge stage[0,na) with stage[na,na+nb): thread t -> outputs [t*VM, t*VM+VM)
      if (dd < m) {
        uint32_t lo = dd > nb ? dd - nb : 0, hi = min(dd, na);
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          const bool le = sk[BS::pad(mid)] <= sk[BS::pad(na + dd - 1 - mid)];
          lo = le ? mid + 1 : lo;
          hi = le ? hi : mid;
        }
        uint32_t ja = lo, jb = na + dd - lo;
        K a = ja < na ? sk[BS::pad(ja)] : KeyTraits<K>::kMax;
        K b = jb < m ? sk[BS::pad(jb)] : KeyTraits<K>::kMax;
#pragma unroll
        for (int k = 0; k < VM; k++) {
          // ties and exhausted runs: take A unless A is exhausted (stability for pairs)
          const bool takeA = ja < na && (jb >= m || a <= b);
          r[k] = takeA ? a : b;
          ri[k] = takeA ? ja : jb;
          const uint32_t jn = (takeA ? ja : jb) + 1;
          const uint32_t end = takeA ? na : m;
          K v = sk[BS::pad(jn)];
          v = jn < end ? v : KeyTraits<K>::kMax;
          a = takeA ? v : a;
          b = takeA ? b : v;
          ja = takeA ? jn : ja;
          jb = takeA ? jb : jn;
        }
      }
    }
    uint32_t rv[VM];
    if (PAIRS) {
#pragma unroll
      for (int k = 0; k < VM; k++) rv[k] = dd + k < m ? sv[ri[k]] : 0u;
    }
    (void)ri;
    __syncthreads();
    if (dd + VM <= m) {
      K* sb = sk + BS::pad(dd);
#pragma unroll
      for (int k = 0; k < VM; k++) {
        sb[BS::poff(k)] = r[k];
        if (PAIRS) sv[dd + k] = rv[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < VM; k++)
        if (dd + k < m) {
          sk[BS::pad(dd + k)] = r[k];
          if (PAIRS) sv[dd + k] = rv[k];
        }
    }
    __syncthreads();
    SQ_CHECK(a0 + d0 + m <= rc.size && m <= uint32_t(TM));
    for (uint32_t i = threadIdx.x; i < m; i += NT) {
      dst[rc.out + a0 + d0 + i] = sk[BS::pad(i)];
      if (PAIRS) vdst[rc.out + a0 + d0 + i] = sv[i];
    }
    __syncthreads();
  }
}

// Gather-copy (single-value buckets, oversize buckets, debug): the bucket's
// keys in the paper's order, contiguous at rc.out in dst.  CTA loops over a list.
template <typename K, int NT>
__global__ void __launch_bounds__(NT)
k_bucket_gather(const BucketRec* __restrict__ recs, const TileInfo* __restrict__ tiles,
                const uint32_t* __restrict__ list, const uint32_t* __restrict__ count, uint32_t all_k,
                const K* __restrict__ src, K* __restrict__ dst, const uint32_t* __restrict__ vsrc,
                uint32_t* __restrict__ vdst, const uint32_t* __restrict__ pout, const uint16_t* __restrict__ ppre) {
  __shared__ uint32_t s_off[NT], s_len[NT], s_dst[NT], misc[64];
  const uint32_t total = list ? *count : all_k;
  for (uint32_t it = blockIdx.x; it < total; it += gridDim.x) {
    const BucketRec rc = recs[list ? item_bucket(list[it]) : it];
    const TileInfo ti = tiles[rc.tile];
    gather_bucket<NT>(ti, rc.lane, pout, ppre, s_off, s_len, s_dst, misc, 0u, rc.size,
                      [&](uint32_t o, uint32_t l, uint32_t d, int ln) {
                        SQ_CHECK(d + l <= rc.size && o >= ti.out && o + l <= ti.out + ti.size);
                        for (uint32_t q = ln; q < l; q += 32) {
                          dst[rc.out + d + q] = src[o + q];
                          if (vsrc) vdst[rc.out + d + q] = vsrc[o + q];
                        }
                      });
  }
}

// Work units of the copy and oversize lists: a bucket is copied in units of
// kGatherKeys keys (its key range [q*kGatherKeys, ...)), so one huge bucket (a
// single-value bucket of a low-cardinality input holds up to n/2 keys) is copied
// by many CTAs instead of one.  One CTA scans the items' unit counts;
// units[u] = (list position, part).
constexpr uint32_t kGatherKeys = 65536;

static __global__ void __launch_bounds__(1024)
k_gather_units(const BucketRec* __restrict__ recs, const uint32_t* __restrict__ list,
               const uint32_t* __restrict__ count, uint32_t nlists, uint32_t list_stride, uint2* __restrict__ units,
               uint32_t* __restrict__ nunits, const uint32_t* __restrict__ rb_count, uint32_t rb_n,
               const uint32_t* __restrict__ rb_info, uint32_t* __restrict__ rb_out) {
  // the level's read-back (one launch fewer on a small level's critical path): the
  // class counts, then the round word, into pinned memory
  for (uint32_t i = threadIdx.x; i < rb_n; i += blockDim.x) rb_out[i] = rb_count[i];
  if (threadIdx.x == 0) rb_out[rb_n] = rb_info[0];
  // units of the lists [0, nlists) (list l at list + l * list_stride, count[l] items):
  // unit = (item | l << 31, part)
  __shared__ uint32_t misc[64];
  uint32_t carry = 0;
  for (uint32_t l = 0; l < nlists; l++) {
    const uint32_t total = count[l];
    const uint32_t* li = list + uint64_t(l) * list_stride;
    for (uint32_t c0 = 0; c0 < total; c0 += 1024) {
      const uint32_t it = c0 + threadIdx.x;
      uint32_t parts = 0;
      if (it < total) parts = max(1u, (recs[item_bucket(li[it])].size + kGatherKeys - 1) / kGatherKeys);
      uint32_t tot;
      const uint32_t ex = block_excl_sum<32>(parts, misc, &tot);
      for (uint32_t q = 0; q < parts; q++) units[carry + ex + q] = make_uint2(it | (l << 31), q);
      carry += tot;
    }
  }
  if (threadIdx.x == 0) *nunits = carry;
}

// Copy of the listed buckets, contiguous at rc.out in dst (keys in the paper's
// order), one unit (a key range of one bucket) per CTA iteration.
template <typename K, int NT>
__global__ void __launch_bounds__(NT)
k_bucket_gather_units(const BucketRec* __restrict__ recs, const TileInfo* __restrict__ tiles,
                      const uint32_t* __restrict__ list, uint32_t list_stride, const uint2* __restrict__ units,
                      const uint32_t* __restrict__ nunits, const K* __restrict__ src, K* __restrict__ dst,
                      const uint32_t* __restrict__ vsrc, uint32_t* __restrict__ vdst,
                      const uint32_t* __restrict__ pout, const uint16_t* __restrict__ ppre) {
  __shared__ uint32_t s_off[NT], s_len[NT], s_dst[NT], misc[64];
  const uint32_t total = *nunits;
  for (uint32_t u = blockIdx.x; u < total; u += gridDim.x) {
    const uint2 un = units[u];
    const BucketRec rc = recs[item_bucket(list[uint64_t(un.x >> 31) * list_stride + (un.x & 0x7fffffffu)])];
    const TileInfo ti = tiles[rc.tile];
    const uint32_t lo = un.y * kGatherKeys, hi = min(rc.size, lo + kGatherKeys);
    K* out = dst + rc.out + lo;
    uint32_t* vout = vdst ? vdst + rc.out + lo : nullptr;
    gather_bucket<NT>(ti, rc.lane, pout, ppre, s_off, s_len, s_dst, misc, lo, hi,
                      [&](uint32_t o, uint32_t l, uint32_t d, int ln) {
                        SQ_CHECK(lo + d + l <= rc.size && o >= ti.out && o + l <= ti.out + ti.size);
                        uint32_t q = ln;
                        for (; q + 96 < l; q += 128) {  // four independent loads in flight per lane
                          const K x0 = src[o + q], x1 = src[o + q + 32], x2 = src[o + q + 64], x3 = src[o + q + 96];
                          out[d + q] = x0;
                          out[d + q + 32] = x1;
                          out[d + q + 64] = x2;
                          out[d + q + 96] = x3;
                        }
                        for (; q < l; q += 32) out[d + q] = src[o + q];
                        if (vsrc)
                          for (uint32_t v = ln; v < l; v += 32) vout[d + v] = vsrc[o + v];
                      });
  }
}

// ------------------------------------------------------------------------------
// Cluster bucket sort (the GPU's simple_sort for buckets larger than one CTA
// holds, P:259-261 / P:852): a cluster of CL CTAs (CL = 4, 8, 16) sorts one
// bucket of up to CL*TILE keys.  CTA r gathers bucket positions
// [r*chunk, (r+1)*chunk) and sorts them on chip; then log2(CL) rounds of
// pairwise merge-path merges read the partner runs through distributed shared
// memory (each CTA produces its `chunk` positions of the merged group), the
// last round writing the sorted bucket straight to HBM.  No extra HBM pass.
template <typename SK>
struct DistSeq {  // a sorted sequence spread over consecutive CTAs, `chunk` keys each
  SK* const* parts;  // shared-memory pointers of the cluster's CTAs (mapped)
  uint32_t first;    // first CTA
  uint32_t chunk;
  uint32_t len;
  template <int PER>
  __device__ __forceinline__ SK at(uint32_t i) const {
    const uint32_t c = i / chunk, off = i - c * chunk;
    return parts[first + c][off + off / PER];
  }
};

// Merge-path split of diagonal d between two distributed sorted sequences,
// found by one warp with 32-ary search: smallest a in [max(0,d-|B|), min(d,|A|)]
// with A[a] > B[d-1-a] (ties taken from A first).  Result broadcast to the warp.
template <typename SK, int PER>
__device__ __forceinline__ uint32_t warp_merge_split(const DistSeq<SK>& A, const DistSeq<SK>& B, uint32_t d) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = d > B.len ? d - B.len : 0, hi = min(d, A.len);
  // invariant: the answer lies in [lo, hi]; pred(a) = A[a] > B[d-1-a] is monotone
  while (hi > lo) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t p = lo + lane * step;
    bool gt = true;  // probes at or beyond hi count as true
    if (p < hi) gt = A.template at<PER>(p) > B.template at<PER>(d - 1 - p);
    const uint32_t m = __ballot_sync(0xffffffffu, gt);
    const uint32_t first = m ? (uint32_t)(__ffs(m) - 1) : 32u;  // first probe with pred true
    if (first == 0) {
      hi = lo;
    } else {
      const uint32_t lo_old = lo;
      lo = lo_old + (first - 1) * step + 1;                       // pred(probe first-1) is false
      hi = (uint32_t)min((uint64_t)hi, (uint64_t)lo_old + (uint64_t)first * step);  // pred(probe first) true
    }
  }
  return lo;
}

template <typename K, int NT, int V, int CL, bool PAIRS>
__global__ void __launch_bounds__(NT)
k_clustersort(const BucketRec* __restrict__ recs, const TileInfo* __restrict__ tiles,
              const uint32_t* __restrict__ list, const uint32_t* __restrict__ count, const K* __restrict__ src,
              K* __restrict__ dst, const uint32_t* __restrict__ vsrc, uint32_t* __restrict__ vdst,
              const uint32_t* __restrict__ pout, const uint16_t* __restrict__ ppre) {
  namespace cg = cooperative_groups;
  using SK = sortkey_t<K, PAIRS>;
  using BS = BlockSort<SK, NT, V>;
  constexpr int PER = BS::PER;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SK* bufA = reinterpret_cast<SK*>(smem_raw);                     // my part of the current sequence
  SK* bufB = reinterpret_cast<SK*>(smem_raw + BS::SMEM_BYTES);   // staged merge inputs
  uint32_t* vs = reinterpret_cast<uint32_t*>(smem_raw + 2 * BS::SMEM_BYTES);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(smem_raw + 2 * BS::SMEM_BYTES + (PAIRS ? BS::TILE * 4 : 0));
  uint32_t* s_len = s_off + NT;
  uint32_t* s_dst = s_len + NT;
  uint32_t* misc = s_dst + NT;
  __shared__ SK* partsA[CL];
  __shared__ uint32_t* partsV[CL];
  __shared__ uint32_t split[2];
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t rank = cluster.block_rank();
  if (threadIdx.x < CL) {
    partsA[threadIdx.x] = cluster.map_shared_rank(bufA, threadIdx.x);
    partsV[threadIdx.x] = cluster.map_shared_rank(vs, threadIdx.x);
  }
  __syncthreads();
  const uint32_t total = *count;
  const uint32_t ncl = gridDim.x / CL, cid = blockIdx.x / CL;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t it = cid; it < total; it += ncl) {
    const BucketRec rc = recs[item_bucket(list[it])];
    const TileInfo ti = tiles[rc.tile];
    const uint32_t L = rc.size;
    const uint32_t chunk = (L + CL - 1) / CL;
    const uint32_t lo = min(L, rank * chunk), hi = min(L, lo + chunk);
    const uint32_t mylen = hi - lo;
    // ---- gather this CTA's chunk and sort it on chip
    for (int i = threadIdx.x + mylen; i < BS::TILE; i += NT) bufA[BS::pad(i)] = KeyTraits<SK>::kMax;
    gather_bucket<NT>(ti, rc.lane, pout, ppre, s_off, s_len, s_dst, misc, lo, hi,
                      [&](uint32_t o, uint32_t l, uint32_t d, int ln) {
                        for (uint32_t q = ln; q < l; q += 32) {
                          if constexpr (PAIRS) {
                            bufA[BS::pad(d + q)] = (SK(src[o + q]) << 32) | SK(lo + d + q);
                            vs[d + q] = vsrc[o + q];
                          } else {
                            cp_async_elem(&bufA[BS::pad(d + q)], &src[o + q]);
                          }
                        }
                      });
    cp_async_wait_all();
    __syncthreads();
    BS::sort_smem(bufA);
    // ---- merge rounds: groups of 2h CTAs merge the sequences held by [g, g+h) and [g+h, g+2h)
    for (uint32_t h = 1; h < CL; h *= 2) {
      const bool last = 2 * h == CL;
      const uint32_t g = rank & ~(2 * h - 1);
      const uint32_t la = (uint32_t)min((uint64_t)h * chunk, (uint64_t)(L > g * chunk ? L - g * chunk : 0));
      const uint32_t lb = (uint32_t)min((uint64_t)h * chunk, (uint64_t)(L > (g + h) * chunk ? L - (g + h) * chunk : 0));
      DistSeq<SK> A{partsA, g, chunk, la};
      DistSeq<SK> B{partsA, g + h, chunk, lb};
      const uint32_t mbeg = min((rank - g) * chunk, la + lb);
      const uint32_t mend = min(mbeg + chunk, la + lb);
      cluster.sync();  // previous round's parts are complete everywhere
      if (w < 2) {
        const uint32_t sp = warp_merge_split<SK, PER>(A, B, w == 0 ? mbeg : mend);
        if (lane == 0) split[w] = sp;
      }
      __syncthreads();
      const uint32_t a0 = split[0], a1 = split[1];
      const uint32_t b0 = mbeg - a0, b1 = mend - a1;
      const uint32_t na = a1 - a0, nbk = b1 - b0;
      // stage A[a0,a1) then B[b0,b1) into bufB (bulk DSMEM reads, coalesced)
      for (uint32_t i = threadIdx.x; i < na; i += NT) bufB[BS::pad(i)] = A.template at<PER>(a0 + i);
      for (uint32_t i = threadIdx.x; i < nbk; i += NT) bufB[BS::pad(na + i)] = B.template at<PER>(b0 + i);
      cluster.sync();  // all partners finished reading my bufA
      // local merge of bufB[0,na) and bufB[na,na+nbk): thread t produces outputs [t*V, t*V+V)
      const uint32_t mlen = na + nbk;
      const uint32_t d0 = threadIdx.x * V;
      SK r[V];
      if (d0 < mlen) {
        uint32_t lo2 = d0 > nbk ? d0 - nbk : 0, hi2 = min(d0, na);
        while (lo2 < hi2) {
          const uint32_t mid = (lo2 + hi2) >> 1;
          if (bufB[BS::pad(mid)] <= bufB[BS::pad(na + d0 - 1 - mid)]) lo2 = mid + 1; else hi2 = mid;
        }
        uint32_t ia = lo2, ib = d0 - lo2;
        SK a = ia < na ? bufB[BS::pad(ia)] : KeyTraits<SK>::kMax;
        SK b = ib < nbk ? bufB[BS::pad(na + ib)] : KeyTraits<SK>::kMax;
#pragma unroll
        for (int k = 0; k < V; k++) {
          const bool takeA = ib >= nbk || (ia < na && a <= b);
          r[k] = takeA ? a : b;
          if (takeA) {
            ia++;
            a = ia < na ? bufB[BS::pad(ia)] : KeyTraits<SK>::kMax;
          } else {
            ib++;
            b = ib < nbk ? bufB[BS::pad(na + ib)] : KeyTraits<SK>::kMax;
          }
        }
      }
      if (!last) {
#pragma unroll
        for (int k = 0; k < V; k++)
          if (d0 + k < mlen) bufA[BS::pad(d0 + k)] = r[k];
      } else {
#pragma unroll
        for (int k = 0; k < V; k++) {
          const uint32_t pos = mbeg + d0 + k;
          if (d0 + k < mlen) {
            if constexpr (PAIRS) {
              const uint32_t src_pos = uint32_t(r[k]);  // position in the bucket's gathered order
              dst[rc.out + pos] = K(r[k] >> 32);
              vdst[rc.out + pos] = partsV[src_pos / chunk][src_pos % chunk];
            } else {
              dst[rc.out + pos] = r[k];
            }
          }
        }
      }
    }
    cluster.sync();  // the next bucket may not overwrite shared memory others still read
  }
}

}  // namespace sq
