// binclust.cuh -- bucket sort of a bucket larger than one CTA's tile by a thread-block
// cluster of CL CTAs over distributed shared memory, each CTA with the counting
// sort's 16K-key tile (two CTAs per SM), so the bucket costs one read and one write
// of HBM like every other bucket (P:291-293 sorts each bucket; here the base case
// spans CL SMs instead of recursing or merge-sorting through HBM).
//
// Per bucket (CTA r of the cluster holds the bucket positions [r*h, (r+1)*h), h =
// ceil(size / CL), gathered in the paper's order like k_bucketsort):
//   1. min and max of the bucket (every CTA's, exchanged through DSMEM);
//   2. a coarse histogram of NC monotone bins of the key over [min, max] per CTA;
//      every CTA adds all CL histograms (DSMEM reads) and scans them;
//   3. CL - 1 cuts between coarse bins split the bucket into CL value ranges of
//      about size / CL keys (the cut before the coarse bin holding key d*h of the
//      sorted bucket); range d belongs to CTA d.  A range above one tile (a coarse
//      bin larger than the slack: skewed input) sends the bucket to the next level
//      instead (the level's oversize list);
//   4. every CTA writes its keys into its own tile grouped by range, publishes its
//      group sizes, and pulls (DSMEM reads, warp-contiguous) the group of its own
//      range from every CTA of the cluster into registers;
//   5. the counting sort (binsort.cuh) sorts those registers on chip, and the CTA
//      writes them at the range's place in the bucket's output.
// Range d's keys precede range d+1's (the coarse bin is monotone), so the CL sorted
// ranges are the sorted bucket.  Keys only: the result is unique, the order in
// which keys are gathered does not matter.
// Measured (cfg5, sq_set_big_bucket_mode 3; profiles/r02_experiments.md): correct,
// but 9-15 ns per key against 4-7 ns for the one-CTA classes plus merge passes of
// mode 1 (the default): the bucket phase takes 2.5 ms instead of 1.9.  Kept as an
// option and tested; not the default.
#pragma once
#include <cooperative_groups.h>
#include "level2.cuh"

namespace sq {

__host__ __device__ constexpr size_t bc_al(size_t x) { return (x + 15) & ~size_t(15); }

struct BinClusterCfg {
  static constexpr int NT = 512, V = 32, TILE = NT * V;  // the counting sort's 16K tile
  static constexpr int NC = 1024;                       // coarse bins
  static constexpr uint32_t SLACK = 256;                // keys per CTA kept free for uneven ranges
  using BN = BinSort<uint32_t, NT, V>;
  using BS = BlockSort<uint32_t, NT, V>;               // (the fallback's padded layout sizes the tile)
  static constexpr size_t off_s = 0;
  static constexpr size_t off_cnt = bc_al(BS::SMEM_BYTES);
  static constexpr size_t off_tab = off_cnt + bc_al(BN::CNT_BYTES);   // gather tables s_off, s_len, s_dst, misc
  static constexpr size_t off_ch = off_tab + (3 * NT + 64) * 4;    // coarse histogram (NC words)
  static constexpr size_t off_x = off_ch + NC * 4;                // exchange words
  static constexpr size_t SMEM = off_x + 64 * 4;
  // largest bucket a cluster of cl CTAs takes
  __host__ __device__ static constexpr uint32_t cap(int cl) { return uint32_t(cl) * (TILE - SLACK); }
};

// exchange words (x[]): 0 min, 1 max, 2..2+CL own group sizes by range, 20.. cuts
enum { kXMin = 0, kXMax = 1, kXGrp = 2, kXCut = 20, kXBase = 40, kXTot = 41, kXFail = 42 };

template <int CL>
__global__ void __launch_bounds__(BinClusterCfg::NT, 2)
k_binsort_cluster(const BucketRec* __restrict__ recs, const TileInfo* __restrict__ tiles,
                  const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                  const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, const uint32_t* __restrict__ pout,
                  const uint16_t* __restrict__ ppre, uint32_t* __restrict__ ovf_list,
                  uint32_t* __restrict__ ovf_count) {
  namespace cg = cooperative_groups;
  using C = BinClusterCfg;
  using BN = C::BN;
  constexpr int NT = C::NT, V = C::V, NC = C::NC, NW = NT / 32;
  static_assert(CL >= 2 && CL <= 16 && 2 + CL <= kXCut && kXCut + CL + 1 <= kXBase, "cluster size");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* s = reinterpret_cast<uint32_t*>(smem_raw + C::off_s);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw + C::off_cnt);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(smem_raw + C::off_tab);
  uint32_t* s_len = s_off + NT;
  uint32_t* s_dst = s_len + NT;
  uint32_t* misc = s_dst + NT;
  uint32_t* ch = reinterpret_cast<uint32_t*>(smem_raw + C::off_ch);
  uint32_t* x = reinterpret_cast<uint32_t*>(smem_raw + C::off_x);
  __shared__ uint32_t* rs[CL];  // every CTA's tile, coarse histogram and exchange words
  __shared__ uint32_t* rch[CL];
  __shared__ uint32_t* rx[CL];
  __shared__ uint32_t grp[CL][CL];  // grp[k][d]: CTA k's keys of range d
  __shared__ uint32_t s_ip[CL + 2], s_gb[CL];
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t rank = cluster.block_rank();
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t < CL) {
    rs[t] = cluster.map_shared_rank(s, t);
    rch[t] = cluster.map_shared_rank(ch, t);
    rx[t] = cluster.map_shared_rank(x, t);
  }
  __syncthreads();
  const uint32_t total = *count;
  const uint32_t ncl = gridDim.x / CL, cid = blockIdx.x / CL;
  const uint32_t b0 = uint32_t(t) * V;
  for (uint32_t it = cid; it < total; it += ncl) {
    const uint32_t e = list[it];
    const BucketRec rc = recs[item_bucket(e)];
    const TileInfo ti = tiles[rc.tile];
    const uint32_t S = rc.size;
    const uint32_t h = (S + CL - 1) / CL;
    const uint32_t lo = min(S, rank * h), hi = min(S, lo + h), mylen = hi - lo;
    for (int i = t; i < NC; i += NT) ch[i] = 0u;
    // ---- gather this CTA's share of the bucket
    gather_bucket<NT>(ti, rc.lane, pout, ppre, s_off, s_len, s_dst, misc, lo, hi,
                      [&](uint32_t o, uint32_t l, uint32_t d, int ln) {
                        SQ_CHECK(d + l <= uint32_t(C::TILE));
                        for (uint32_t q = ln; q < l; q += 32) cp_async_elem(&s[swz32(d + q)], &src[o + q]);
                      });
    cp_async_wait_all();
    __syncthreads();
    uint32_t r[V];
    BN::template ld_block<V>(s, b0, r);
    // ---- 1. min and max of the bucket
    uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
    for (int j = 0; j < V; j++)
      if (b0 + j < mylen) {
        mn = min(mn, r[j]);
        mx = max(mx, r[j]);
      }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
      misc[w] = mn;
      misc[32 + w] = mx;
    }
    __syncthreads();
    if (t == 0) {
      for (int q = 1; q < NW; q++) {
        mn = min(mn, misc[q]);
        mx = max(mx, misc[32 + q]);
      }
      x[kXMin] = mn;
      x[kXMax] = mx;
    }
    cluster.sync();  // #1: every CTA's min and max
    if (t == 0) {
      uint32_t gmn = 0xffffffffu, gmx = 0u;
      for (int k = 0; k < CL; k++) {
        gmn = min(gmn, rx[k][kXMin]);
        gmx = max(gmx, rx[k][kXMax]);
      }
      misc[0] = gmn;
      const uint32_t range = gmx - gmn;
      misc[1] = range < uint32_t(NC) ? 0u : (uint32_t)((uint64_t(NC) << 32) / (uint64_t(range) + 1));
    }
    __syncthreads();
    const uint32_t gmn = misc[0], fc = misc[1];
    auto cbin = [&](uint32_t v) -> uint32_t { return fc ? __umulhi(v - gmn, fc) : v - gmn; };
    // ---- 2. coarse histogram
#pragma unroll
    for (int j = 0; j < V; j++)
      if (b0 + j < mylen) atomicAdd(&ch[cbin(r[j])], 1u);
    cluster.sync();  // #2: every CTA's histogram
    // combined histogram: thread t owns coarse bins 2t, 2t+1; own counts too
    const uint32_t c0 = 2 * t, c1 = 2 * t + 1;
    uint32_t a0 = 0, a1 = 0;
#pragma unroll
    for (int k = 0; k < CL; k++) {
      const uint2 v2 = *reinterpret_cast<const uint2*>(rch[k] + c0);
      a0 += v2.x;
      a1 += v2.y;
    }
    const uint32_t o0 = ch[c0], o1 = ch[c1];
    uint32_t tot;
    const uint32_t p0 = block_excl_sum<NW>(a0 + a1, misc, &tot);  // combined prefix before bin c0
    const uint32_t q0 = block_excl_sum<NW>(o0 + o1, misc + 32, &tot);  // own prefix before bin c0
    // ---- 3. cuts: range d starts at the coarse bin holding key d*h of the bucket
    if (t <= CL) x[kXCut + t] = t == 0 ? 0u : uint32_t(NC);
    __syncthreads();
#pragma unroll
    for (int d = 1; d < CL; d++) {
      const uint32_t target = uint32_t(d) * h;
      if (target < S) {
        if (p0 <= target && target < p0 + a0) x[kXCut + d] = c0;
        else if (p0 + a0 <= target && target < p0 + a0 + a1) x[kXCut + d] = c1;
      }
    }
    // combined and own prefix at every bin boundary, for the range sizes below
    cnt[c0] = p0;
    cnt[c1] = p0 + a0;
    cnt[NC + c0] = q0;
    cnt[NC + c1] = q0 + o0;
    __syncthreads();
    auto cut = [&](int d) -> uint32_t { return x[kXCut + d]; };
    auto pref = [&](const uint32_t* P, uint32_t c, uint32_t end) { return c >= uint32_t(NC) ? end : P[c]; };
    bool fail = false;
    uint32_t obase = 0, mytot = 0;
#pragma unroll
    for (int d = 0; d < CL; d++) {
      const uint32_t td = pref(cnt, cut(d + 1), S) - pref(cnt, cut(d), S);
      fail = fail || td > uint32_t(C::TILE);
      if (d < int(rank)) obase += td;
      if (d == int(rank)) mytot = td;
    }
    if (fail) {  // skewed bucket: the next SquareSort level sorts it (it is gathered to X later)
      if (rank == 0 && t == 0) ovf_list[atomicAdd(ovf_count, 1u)] = e;
      cluster.sync();  // nobody still reads this item's histograms
      continue;
    }
    // ---- 4. own keys into the own tile ordered by coarse bin (a counting-sort scatter
    // on the own prefix), so the keys of range d are the contiguous group
    // [Pown(cut[d]), Pown(cut[d+1])); group sizes published
    if (t < CL) x[kXGrp + t] = pref(cnt + NC, cut(t + 1), mylen) - pref(cnt + NC, cut(t), mylen);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < V; j++)
      if (b0 + j < mylen) {
        const uint32_t slot = atomicAdd(&cnt[NC + cbin(r[j])], 1u);
        s[swz32(slot)] = r[j];
        if (j % 8 == 7) asm volatile("" ::: "memory");
      }
    __syncthreads();
    cluster.sync();  // #3: every CTA's groups and group sizes
    if (t < CL * CL) grp[t / CL][t % CL] = rx[t / CL][kXGrp + t % CL];
    __syncthreads();
    // pull range `rank` from every CTA: incoming key q (thread q % NT, slot q / NT);
    // CTA k's group starts at s_gb[k] in its tile and covers incoming [s_ip[k], s_ip[k+1])
    if (t == 0) {
      uint32_t acc = 0;
      for (int k = 0; k < CL; k++) {
        uint32_t b = 0;
        for (int d = 0; d < int(rank); d++) b += grp[k][d];
        s_gb[k] = b;
        s_ip[k] = acc;
        acc += grp[k][rank];
      }
      s_ip[CL] = acc;
      s_ip[CL + 1] = 0xffffffffu;  // sentinel
      SQ_CHECK(acc == mytot);
    }
    __syncthreads();
    uint32_t k = 0, ipk = 0, ipn = s_ip[1], gbk = s_gb[0];
    const uint32_t* from = rs[0];
#pragma unroll
    for (int j = 0; j < V; j++) {
      const uint32_t q = uint32_t(j) * NT + t;
      uint32_t v = 0xffffffffu;
      if (q < mytot) {
        while (q >= ipn) {  // the groups are thousands of keys: rarely more than one step
          k++;
          ipk = ipn;
          ipn = s_ip[k + 1];
          gbk = s_gb[k];
          from = rs[k];
        }
        v = from[swz32(gbk + (q - ipk))];
      }
      r[j] = v;
    }
    cluster.sync();  // #4: every CTA has pulled its range; tiles may be overwritten
    // ---- 5. sort the range on chip and write it at its place in the bucket
    if (mytot) {  // (uniform over the CTA)
      BN::sort_regs(r, s, cnt, mytot, [&](int j) { return uint32_t(j) * NT + t; });
      uint32_t* out = dst + rc.out + obase;
      for (uint32_t i = t; i < mytot; i += NT) out[i] = s[swz32(i)];
    }
    __syncthreads();
  }
}

}  // namespace sq
