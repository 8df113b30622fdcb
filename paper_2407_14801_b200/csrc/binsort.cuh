// binsort.cuh -- the B200 base case for 32- and 64-bit sort keys: one CTA sorts a
// tile held in shared memory by a counting sort on a monotone bin of the key, then
// fixes the order inside the (short) bins with two sorting-network passes.
//
// The paper's base case is any direct sort of a small array ("simple_sort",
// P:259-261; std::sort below 1000 items in the experiments).  On B200 the
// comparison merge sort of blocksort.cuh costs ~180 instructions per key and is
// bound by the integer ALU pipe; shared-memory atomics, random stores and random
// loads all issue at ~1.4 clk per warp instruction per SM (tools/ubench/ubench2,
// profiles/r02_ubench2.txt), so a counting sort is cheaper:
//   1. min and max of the tile; bin(x) = floor((x - min) * f / 2^w) with
//      f = floor(NB * 2^w / (max - min + 1)) spreads [min, max] over NB bins
//      (w = key bits; one multiply-high).  bin is monotone: bin(x) < bin(y)
//      implies x < y.  When max - min < NB the bin is x - min itself (exact).
//   2. histogram of the bins (shared-memory atomics), exclusive scan -> the start
//      of every bin, and the largest bin.
//   3. scatter: each key takes the next slot of its bin (atomic increment).  The
//      tile is now ordered by bin; only keys of one bin can be out of order.
//   4. if the bins are exact (single values): done.  Otherwise, when no bin holds
//      more than V/2 keys, pass 1 sorts every thread's block of V consecutive keys
//      in registers (Batcher's network), and pass 2 merges the upper half of block
//      t with the lower half of block t+1: a bin of at most V/2 keys lies inside
//      one block, where pass 1 sorts it, or straddles one block boundary and lies
//      inside the window pass 2 merges.  A larger bin (skewed input) falls back to
//      the merge sort of blocksort.cuh on the bin-ordered tile.
// Shapes: 32-bit keys with V = 32 use NB = TILE/2 bins (mean 2 keys, runs <= 16),
// with V = 16 NB = 2*TILE; 64-bit keys (u64 keys, or the stable pair composites
// key << 32 | position of L16) use V = 16 and NB = TILE (mean 1 key, runs <= 8).
// The tile lives in shared memory in an XOR-swizzled row layout (see pad()), so
// the fix-up passes move 16-byte vectors without bank conflicts.
// The result is the sorted tile.  The scatter is unstable, which does not matter:
// 32/64-bit keys are compared as whole values, and pair composites are unique.
#pragma once
#include "blocksort.cuh"

namespace sq {

template <typename K, int NT_, int V_>
struct BinSort {
  static_assert(sizeof(K) == 4 || sizeof(K) == 8, "32- or 64-bit sort keys");
  static constexpr int NT = NT_;
  static constexpr int V = V_;
  static constexpr int NW = NT / 32;
  static constexpr int TILE = NT * V;
  static_assert(sizeof(K) == 4 ? (V == 16 || V == 32) : V == 16, "fix-up networks: 16 or 32 keys per thread");
  static_assert(NT % 32 == 0, "whole warps");
  static constexpr int E = sizeof(K) == 8 ? 16 : (V == 32 ? 16 : 32);  // counters per thread in the scan
  static constexpr int NB = NT * E;
  static constexpr int RUNMAX = V / 2;
  static constexpr int EPC = 16 / sizeof(K);  // keys per 16-byte chunk
  // shared memory for the counters and the block reductions (bytes), besides the tile
  // (+16 bytes: the counters are aligned up to 16 bytes for vector access):
  // NB counters, then K-typed warp minima [0, 32), maxima [32, 64) and 4 misc slots
  static constexpr size_t RED_WORDS = (2 * 32 + 4) * sizeof(K) / 4;
  static constexpr size_t CNT_WORDS = NB + RED_WORDS;
  static constexpr size_t CNT_BYTES = CNT_WORDS * 4 + 16;
  // (pointer arithmetic on p, so the compiler keeps it in the shared window)
  __device__ __forceinline__ static uint32_t* align_cnt(uint32_t* p) {
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(p)) & 15u;
    return p + ((16u - mis) & 15u) / 4u;
  }

  // Tile layout: rows of 128 bytes; the 16-byte chunk c of the tile (keys
  // [EPC*c, EPC*c + EPC)) is stored at chunk slot c ^ ((c / 8) % 8) of its row.
  // Per-thread blocks of consecutive keys are then read and written with
  // conflict-free 16-byte accesses (8 threads of a phase hit 8 different slots),
  // warp-contiguous scalar accesses stay conflict-free, and the tile takes exactly
  // TILE keys.
  __device__ __forceinline__ static uint32_t pad(uint32_t i) {
    if constexpr (sizeof(K) == 4) return swz32(i);
    else return i ^ (((i >> 4) & 7) << 1);
  }
  __device__ __forceinline__ static uint4& chunk(K* s, uint32_t c) {
    return reinterpret_cast<uint4*>(s)[c ^ ((c >> 3) & 7)];
  }
  // keys [b, b + N) (b a multiple of EPC) to r[0..N) / from r[0..N)
  template <int N>
  __device__ __forceinline__ static void ld_block(const K* s, uint32_t b, K* r) {
#pragma unroll
    for (int q = 0; q < N / EPC; q++) {
      const uint4 v = chunk(const_cast<K*>(s), b / EPC + q);
      if constexpr (sizeof(K) == 4) {
        r[4 * q] = v.x;
        r[4 * q + 1] = v.y;
        r[4 * q + 2] = v.z;
        r[4 * q + 3] = v.w;
      } else {
        r[2 * q] = (uint64_t(v.y) << 32) | v.x;
        r[2 * q + 1] = (uint64_t(v.w) << 32) | v.z;
      }
    }
  }
  template <int N>
  __device__ __forceinline__ static void st_block(K* s, uint32_t b, const K* r) {
#pragma unroll
    for (int q = 0; q < N / EPC; q++) {
      if constexpr (sizeof(K) == 4)
        chunk(s, b / EPC + q) = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
      else
        chunk(s, b / EPC + q) = make_uint4(uint32_t(r[2 * q]), uint32_t(r[2 * q] >> 32), uint32_t(r[2 * q + 1]),
                                           uint32_t(r[2 * q + 1] >> 32));
    }
  }

  // the bin of x: exact (x - min) or floor((x - min) * f / 2^w)
  __device__ __forceinline__ static uint32_t bin_of(K x, K mn, K f, bool exact) {
    if constexpr (sizeof(K) == 4) return exact ? x - mn : __umulhi(x - mn, f);
    else return exact ? uint32_t(x - mn) : uint32_t(__umul64hi(x - mn, f));
  }
  __device__ __forceinline__ static K warp_min(K v) {
    if constexpr (sizeof(K) == 4) {
      return __reduce_min_sync(0xffffffffu, v);
    } else {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const K y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y < v ? y : v;
      }
      return v;
    }
  }
  __device__ __forceinline__ static K warp_max(K v) {
    if constexpr (sizeof(K) == 4) {
      return __reduce_max_sync(0xffffffffu, v);
    } else {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const K y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y > v ? y : v;
      }
      return v;
    }
  }

  template <bool SCATTER>
  __device__ __forceinline__ static void bin_op(K* s, uint32_t* cnt, K x, uint32_t b) {
    if constexpr (SCATTER) {
      const uint32_t d = atomicAdd(&cnt[b], 1u);
      SQ_CHECK(d < uint32_t(TILE) && b < uint32_t(NB));
      s[pad(d)] = x;
    } else {
      atomicAdd(&cnt[b], 1u);
    }
  }
  // Histogram (SCATTER = false) or scatter (true) of the thread's keys; the branch on
  // `exact` and `full` is uniform across the CTA.
  template <bool SCATTER, typename POS>
  __device__ __forceinline__ static void hist_or_scatter(K* s, uint32_t* cnt, const K (&r)[V], K mn, K f,
                                                         bool exact, bool full, uint32_t len, POS pos) {
    // groups of G keys: a scatter's returned slots stay live until the store, so the
    // compiler may not hoist all V atomics (register pressure, spills)
    constexpr int G = SCATTER ? 8 : V;
    if (full) {
      if (exact) {
#pragma unroll
        for (int j = 0; j < V; j++) {
          bin_op<SCATTER>(s, cnt, r[j], bin_of(r[j], mn, f, true));
          if (j % G == G - 1) asm volatile("" ::: "memory");
        }
      } else {
#pragma unroll
        for (int j = 0; j < V; j++) {
          bin_op<SCATTER>(s, cnt, r[j], bin_of(r[j], mn, f, false));
          if (j % G == G - 1) asm volatile("" ::: "memory");
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < V; j++)
        if (pos(j) < len) bin_op<SCATTER>(s, cnt, r[j], bin_of(r[j], mn, f, exact));
    }
  }

  // Sort the TILE keys at s[pad(0..TILE-1)]; positions >= len hold the key type's
  // maximum as padding (left in place).  cnt: CNT_WORDS words of shared memory; s
  // must have room for the padded layout of BlockSort<K, NT, V> (the skewed-input
  // fallback).  On return the sorted tile is in s and a __syncthreads() has been
  // executed.
  __device__ static void sort_smem(K* s, uint32_t* cnt, uint32_t len = TILE) {
    const uint32_t b0 = uint32_t(threadIdx.x) * V;
    K r[V];
    ld_block<V>(s, b0, r);
    sort_regs(r, s, cnt, len, [&](int j) { return b0 + j; });
  }

  // Same, with the tile's keys already in registers: r[j] holds the key at tile
  // position pos(j) (any arrangement; positions >= len are ignored).  s receives the
  // sorted tile (swizzled layout, positions >= len set to the maximum key).
  template <typename POS>
  __device__ static void sort_regs(K (&r)[V], K* s, uint32_t* cnt, uint32_t len, POS pos) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    cnt = align_cnt(cnt);
    K* red = reinterpret_cast<K*>(cnt + NB);  // [0, 32): warp minima, [32, 64): warp maxima, [64, 68): misc
    const uint32_t b0 = uint32_t(t) * V;
    bool full = true;
#pragma unroll
    for (int j = 0; j < V; j++) full = full && pos(j) < len;
    // ---- 1. min and max of the real keys; counters cleared
    K mn = KeyTraits<K>::kMax, mx = K(0);
    if (full) {
#pragma unroll
      for (int j = 0; j < V; j++) {
        mn = r[j] < mn ? r[j] : mn;
        mx = r[j] > mx ? r[j] : mx;
      }
    } else {
#pragma unroll
      for (int j = 0; j < V; j++)
        if (pos(j) < len) {
          mn = r[j] < mn ? r[j] : mn;
          mx = r[j] > mx ? r[j] : mx;
        }
    }
    // padding positions of the sorted tile (the scatter fills [0, len)); every thread
    // takes part, whichever of them hold keys past len
    if (len < uint32_t(TILE))
      for (uint32_t i = t; i < uint32_t(TILE) - len; i += NT) s[pad(len + i)] = KeyTraits<K>::kMax;
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (lane == 0) {
      red[w] = mn;
      red[32 + w] = mx;
    }
#pragma unroll
    for (int q = 0; q < E; q++) cnt[q * NT + t] = 0u;
    __syncthreads();
    if (t == 0) {  // tile minimum, bin factor, exactness
      mn = red[0];
      mx = red[32];
      for (int q = 1; q < NW; q++) {
        mn = red[q] < mn ? red[q] : mn;
        mx = red[32 + q] > mx ? red[32 + q] : mx;
      }
      const K range = mx - mn;
      red[64] = mn;
      // f = floor(NB * 2^w / (range + 1)) < 2^w when range >= NB
      if constexpr (sizeof(K) == 4)
        red[65] = range < K(NB) ? 0u : (uint32_t)((uint64_t(NB) << 32) / (uint64_t(range) + 1));
      else
        red[65] = range < K(NB) ? K(0) : K((u128(NB) << 64) / (u128(range) + 1));
    }
    __syncthreads();
    mn = red[64];
    K f = red[65];
    const bool exact = f == K(0);
    // ---- 2. histogram of the bins
    hist_or_scatter<false>(s, cnt, r, mn, f, exact, full, len, pos);
    __syncthreads();
    // ---- exclusive scan of the NB counters (thread t owns [t*E, t*E+E)) and the largest
    // bin.  16-byte chunks are read and written in a per-thread rotated order so the
    // 8 threads of a shared-memory phase hit 8 different bank groups.  The scan's
    // block reduction uses words [0, 64) of red's region; mn and f were read above,
    // and red[64], red[65] (K-typed) lie past those words.
    uint32_t* red32 = reinterpret_cast<uint32_t*>(red);
    constexpr int NQ = E / 4;
    const int rot = E == 16 ? ((t >> 1) & 3) : (t & 7);
    uint4* c4 = reinterpret_cast<uint4*>(cnt + t * E);
    uint4 v[NQ];
    uint32_t cs[NQ], sum = 0, big = 0;
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      v[q] = c4[(q + rot) % NQ];
      cs[q] = v[q].x + v[q].y + v[q].z + v[q].w;
      big = max(big, max(max(v[q].x, v[q].y), max(v[q].z, v[q].w)));
      sum += cs[q];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    big = __reduce_max_sync(0xffffffffu, big);
    if (lane == 31) red32[w] = incl;
    if (lane == 0) red32[32 + w] = big;
    __syncthreads();
    uint32_t tb = incl - sum;
#pragma unroll
    for (int q = 0; q < NW; q++) tb += q < w ? red32[q] : 0u;
    uint32_t gbig = 0;
#pragma unroll
    for (int q = 0; q < NW; q++) gbig = max(gbig, red32[32 + q]);
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      const int cq = (q + rot) % NQ;  // logical chunk of v[q]
      uint32_t pre = tb;
#pragma unroll
      for (int q2 = 0; q2 < NQ; q2++) pre += ((q2 + rot) % NQ < cq) ? cs[q2] : 0u;
      uint4 o;
      o.x = pre;
      o.y = pre + v[q].x;
      o.z = o.y + v[q].y;
      o.w = o.z + v[q].z;
      c4[cq] = o;
    }
    __syncthreads();
    // ---- 3. scatter: each key to the next free slot of its bin.  The bins are
    // recomputed (mn and f laundered through asm) rather than kept live across the
    // scan: V extra registers would spill.
    if constexpr (sizeof(K) == 4) {
      asm volatile("mov.b32 %0, %0;" : "+r"(mn));
      asm volatile("mov.b32 %0, %0;" : "+r"(f));
    } else {
      asm volatile("mov.b64 %0, %0;" : "+l"(mn));
      asm volatile("mov.b64 %0, %0;" : "+l"(f));
    }
    hist_or_scatter<true>(s, cnt, r, mn, f, exact, full, len, pos);
    __syncthreads();
    if (exact) return;  // every bin is one value
    if (gbig > RUNMAX) {  // a bin too long for the fix-up (skewed input): merge sort,
      // in the merge sort's padded layout (converted there and back through registers)
      using MS = BlockSort<K, NT, V>;
      ld_block<V>(s, b0, r);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < V; j++) s[MS::pad(b0 + j)] = r[j];
      __syncthreads();
      MS::sort_smem(s, len);
#pragma unroll
      for (int j = 0; j < V; j++) r[j] = s[MS::pad(b0 + j)];
      __syncthreads();
      st_block<V>(s, b0, r);
      __syncthreads();
      return;
    }
    // ---- 4a. fix-up pass 1: every thread sorts its block of V consecutive keys
    const bool live = (uint32_t(t) & ~31u) * V < len;  // warp-uniform: padding-only warps skip
    if (live) {
      ld_block<V>(s, b0, r);
      thread_sort<K, V>(r);
      st_block<V>(s, b0, r);
    }
    __syncthreads();
    // ---- 4b. fix-up pass 2: merge [b0 + V/2, b0 + V) with [b0 + V, b0 + 3V/2)
    constexpr int H = V / 2;
    if (t < NT - 1 && b0 + H < len) {
      ld_block<H>(s, b0 + H, r);
      {
        K u[H];
        ld_block<H>(s, b0 + V, u);
#pragma unroll
        for (int j = 0; j < H; j++) r[H + j] = u[H - 1 - j];  // descending: a bitonic sequence
      }
      const uint32_t one = (uint32_t)c_one, mone = (uint32_t)c_mone;
#pragma unroll
      for (int d = H; d >= 1; d >>= 1)
#pragma unroll
        for (int i = 0; i < V; i++)
          if ((i & d) == 0) {
            if (i & 1) cas_fma_k(r[i], r[i + d], one, mone);
            else cas(r[i], r[i + d]);
          }
      st_block<V>(s, b0 + H, r);
    }
    __syncthreads();
  }
};

}  // namespace sq
