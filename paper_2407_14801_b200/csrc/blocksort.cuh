// blocksort.cuh -- on-chip sort of one segment by one CTA (the GPU's simple_sort).
//
// The paper's base case sorts small arrays directly (Alg 1; the
// experiments use std::sort below 1000 items).  On B200 the base case is
// whatever one CTA can hold on chip: the segment is staged in shared memory,
// each thread sorts V keys in registers with Batcher's odd-even merge network,
// and log2(NT) merge-path passes (runs of V -> NT*V) merge through shared
// memory into registers.  Keys only need a correct sort (the result is
// unique); pairs sort 64-bit composites (key << 32 | position) so the result is
// the stable order (L16) and the payload is gathered once at the end.
#pragma once
#include <utility>
#include "common.cuh"

namespace sq {

template <typename K>
__device__ __forceinline__ void cas(K& a, K& b) {
  K lo = a < b ? a : b;
  K hi = a < b ? b : a;
  a = lo;
  b = hi;
}

// Batcher's odd-even merge sort network on V (a power of two) registers,
// generated at compile time and applied with a fold so every index is static
// (the registers never spill to local memory).
template <int V>
struct OddEvenNet {
  static constexpr int count() {
    int c = 0;
    for (int p = 1; p < V; p += p)
      for (int k = p; k > 0; k /= 2)
        for (int j = k % p; j < V - k; j += 2 * k)
          for (int i = 0; i < k; i++)
            if (i + j + k < V && (i + j) / (p + p) == (i + j + k) / (p + p)) c++;
    return c;
  }
  static constexpr int N = count();
  int a[N > 0 ? N : 1], b[N > 0 ? N : 1];
  constexpr OddEvenNet() : a{}, b{} {
    int c = 0;
    for (int p = 1; p < V; p += p)
      for (int k = p; k > 0; k /= 2)
        for (int j = k % p; j < V - k; j += 2 * k)
          for (int i = 0; i < k; i++)
            if (i + j + k < V && (i + j) / (p + p) == (i + j + k) / (p + p)) {
              a[c] = i + j;
              b[c] = i + j + k;
              c++;
            }
  }
};

// Compare-exchange that puts half of its work on the FMA pipe: min on the ALU pipe,
// max = a + b - min (exact modulo 2^32) as two integer multiply-adds.  The sorts are
// ALU-pipe bound (min/max/select/compare all issue there at half rate), the FMA pipe
// is nearly idle; alternating the two forms balances the pipes.
// The multiplier is read from constant memory so that ptxas cannot fold the
// multiply-adds into ALU adds.
static __constant__ int32_t c_one = 1, c_mone = -1, c_mtwo = -2;
__device__ __forceinline__ void cas_fma(uint32_t& a, uint32_t& b, uint32_t one, uint32_t mone) {
  const uint32_t lo = min(a, b);
  uint32_t sum, hi;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(sum) : "r"(a), "r"(one), "r"(b));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(lo), "r"(mone), "r"(sum));
  a = lo;
  b = hi;
}
template <typename K>
__device__ __forceinline__ void cas_fma_k(K& a, K& b, uint32_t one, uint32_t mone) {
  if constexpr (sizeof(K) == 4) cas_fma(a, b, one, mone);
  else cas(a, b);
}
template <typename K, int C>
__device__ __forceinline__ void cas_bal(K& a, K& b, uint32_t one, uint32_t mone) {
  if constexpr (sizeof(K) == 4 && (C & 1)) cas_fma(a, b, one, mone);
  else cas(a, b);
}

template <typename K, int V, int... I>
__device__ __forceinline__ void apply_net(K (&r)[V], std::integer_sequence<int, I...>) {
  constexpr OddEvenNet<V> net{};
  const uint32_t one = (uint32_t)c_one, mone = (uint32_t)c_mone;
  (cas_bal<K, I>(r[net.a[I]], r[net.b[I]], one, mone), ...);
}

template <typename K, int V>
__device__ __forceinline__ void thread_sort(K (&r)[V]) {
  if constexpr (V > 1) apply_net<K, V>(r, std::make_integer_sequence<int, OddEvenNet<V>::N>{});
}

// Warp-shuffle bitonic merge of sorted runs held by G/2-lane groups (each lane V
// ascending keys, lanes in run order) into runs held by G-lane groups.  The
// first half-cleaner compares element x of run A with element x of run B read
// backwards (partner lane = lane ^ (G-1), register V-1-i), leaving the lower
// half in A's lanes and the upper half in B's lanes, each a bitonic sequence in
// storage order; the cross-lane half-cleaners (lane ^ d/V) and the in-register
// ones then sort each half ascending.  No shared memory is touched.
// upper ? max(x, y) : min(x, y).  For 32-bit keys with F set, one min on the ALU
// pipe and three multiply-adds on the FMA pipe: m + u*(x + y - 2m), u = upper.
template <typename K>
__device__ __forceinline__ K dir_minmax(bool F, K x, K y, bool upper, uint32_t u, uint32_t one, uint32_t mtwo) {
  if (sizeof(K) == 4 && F) {
    const uint32_t m = min(uint32_t(x), uint32_t(y));
    uint32_t sum, d, o;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(sum) : "r"(uint32_t(x)), "r"(one), "r"(uint32_t(y)));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(m), "r"(mtwo), "r"(sum));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(o) : "r"(u), "r"(d), "r"(m));
    return K(o);
  } else {
    return upper ? (x < y ? y : x) : (x < y ? x : y);
  }
}

template <typename K, int V, int G>
__device__ __forceinline__ void warp_bitonic_merge(K (&r)[V]) {
  const int lane = threadIdx.x & 31;
  const bool upper = (lane & (G / 2)) != 0;
  const uint32_t one = (uint32_t)c_one, mtwo = (uint32_t)c_mtwo;
  {
    K p[V];
#pragma unroll
    for (int i = 0; i < V; i++) p[i] = shfl_xor_k(r[V - 1 - i], G - 1);
#pragma unroll
    for (int i = 0; i < V; i++) r[i] = dir_minmax<K>(false, r[i], p[i], upper, upper ? 1u : 0u, one, mtwo);
  }
#pragma unroll
  for (int d = G / 4; d >= 1; d >>= 1) {  // cross-lane half-cleaners (distance d*V keys)
    const bool hi = (lane & d) != 0;
    const uint32_t u = hi ? 1u : 0u;
#pragma unroll
    for (int i = 0; i < V; i++) {
      const K q = shfl_xor_k(r[i], d);
      r[i] = dir_minmax<K>(false, r[i], q, hi, u, one, mtwo);
    }
  }
#pragma unroll
  for (int d = V / 2; d >= 1; d >>= 1)  // in-register half-cleaners
#pragma unroll
    for (int i = 0; i < V; i++)
      if ((i & d) == 0) cas(r[i], r[i + d]);
}

template <typename K, int NT_, int V_, int WGM_ = 32>
struct BlockSort {
  static constexpr int NT = NT_;
  static constexpr int V = V_;
  static constexpr int TILE = NT * V;
  static constexpr int PER = 128 / sizeof(K);  // elements per 128-byte pad period
  static constexpr int PSH = sizeof(K) == 4 ? 5 : (sizeof(K) == 8 ? 4 : 3);
  static constexpr int SMEM_ELEMS = TILE + TILE / PER + 1;
  static constexpr size_t SMEM_BYTES = size_t(SMEM_ELEMS) * sizeof(K);

  // one pad element per 128 bytes keeps the blocked per-thread accesses conflict-free
  __device__ __forceinline__ static uint32_t pad(uint32_t i) { return i + (i >> PSH); }

  // Sort the TILE keys held in s[pad(0..TILE-1)] (padding slots hold KeyTraits::kMax).
  // On return s holds the sorted tile (padded layout); a __syncthreads() has
  // been executed so all threads may read it.
  // pad(q + j) for q a multiple of V and 0 <= j < V: the V keys of a thread block
  // never straddle a pad period unevenly, so the offsets are compile-time constants.
  __device__ __forceinline__ static constexpr uint32_t poff(int j) { return uint32_t(j + j / PER); }

  // Merge step of one thread: run A = s[a0, a0+la) ascending, run B = s[a0+la, bend)
  // DESCENDING (a bitonic pair); the thread produces the V merged keys at positions
  // [tv, tv+V) of the pair (tv >= a0) into r.  Reading one past the end of A lands on
  // B's largest key and one past the end of B on A's largest: neither is ever taken
  // too early, so the merge needs no bounds checks.
  __device__ __forceinline__ static void merge_bitonic(const K* s, uint32_t a0, uint32_t la, uint32_t bend,
                                                       uint32_t tv, K (&r)[V]) {
    const uint32_t lb = bend - a0 - la;
    const uint32_t diag = tv - a0;
    // merge path: smallest i with A[i] > B[diag-1-i]; B[k] lives at bend-1-k
    uint32_t lo = diag > lb ? diag - lb : 0;
    uint32_t hi = diag < la ? diag : la;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const K x = s[pad(a0 + mid)];
      const K y = s[pad(bend - diag + mid)];
      const bool le = x <= y;
      lo = le ? mid + 1 : lo;
      hi = le ? hi : mid;
    }
    const uint32_t pa = a0 + lo;                 // physical index of the next A key
    const uint32_t pb = bend - 1 - (diag - lo);  // physical index of the next B key (descending)
    // state: h = head of run L (initially A), o = head of the other run.  The taken
    // key is min(h, o), the untaken head max(h, o); the next key comes from the run
    // just taken from, so the new h is always the key just loaded.  (Ties may take
    // either run: equal keys carry equal values, and the pair composites of the
    // stable sorts are unique.)
    K h = s[pad(pa)];
    K o = lb ? s[pad(pb)] : KeyTraits<K>::kMax;
    bool L = true;                      // h belongs to A
    uint32_t na = pa + 1, nb = pb - 1;  // the index each run reads next
    const uint32_t one = (uint32_t)c_one, mone = (uint32_t)c_mone;
#pragma unroll
    for (int k = 0; k < V; k++) {
      const bool takeL = h <= o;
      r[k] = takeL ? h : o;
      K mx;
      if constexpr (sizeof(K) == 4) {  // max = h + o - min on the FMA pipe (the ALU pipe is the bound)
        uint32_t sum, m;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(sum) : "r"(uint32_t(h)), "r"(one), "r"(uint32_t(o)));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(m) : "r"(uint32_t(r[k])), "r"(mone), "r"(sum));
        mx = K(m);
      } else {
        mx = takeL ? o : h;
      }
      L = takeL ? L : !L;  // the run taken from
      const uint32_t idx = L ? na : nb;
      if (L) na = idx + 1;
      else nb = idx - 1;
      h = s[pad(idx)];
      o = mx;
    }
  }

  // lanes per run after the warp-shuffle merge levels (a merge pass costs about
  // as much per key as a warp level of 16-32 lanes; 32 measured best)
  static constexpr int WGMAX = WGM_;
  static constexpr int WG = (NT >= WGMAX && TILE >= WGMAX * V) ? WGMAX
                            : (NT >= 4 && TILE >= 4 * V) ? 4 : (NT >= 2 && TILE >= 2 * V) ? 2 : 1;

  // Keys at positions >= len are padding (kMax).  Sorted, every position >= len holds
  // kMax after every merge pass, so threads whose whole block lies there skip the
  // work (and warps entirely in the padding skip the register stages).
  __device__ static void sort_smem(K* s, uint32_t len = TILE) {
    const uint32_t t = threadIdx.x;
    K r[V];
    if ((t & ~31u) * V < len) {  // warp-uniform
      {
        const K* sb = s + pad(t * V);
#pragma unroll
        for (int j = 0; j < V; j++) r[j] = sb[poff(j)];
      }
      thread_sort<K, V>(r);
      // the first merge levels (runs of V -> 2V -> ... -> WG*V keys) stay in registers
      if constexpr (WG >= 2) warp_bitonic_merge<K, V, 2>(r);
      if constexpr (WG >= 4) warp_bitonic_merge<K, V, 4>(r);
      if constexpr (WG >= 8) warp_bitonic_merge<K, V, 8>(r);
      if constexpr (WG >= 16) warp_bitonic_merge<K, V, 16>(r);
      if constexpr (WG >= 32) warp_bitonic_merge<K, V, 32>(r);
    } else {
#pragma unroll
      for (int j = 0; j < V; j++) r[j] = KeyTraits<K>::kMax;
    }
    constexpr uint32_t WL = WG * V;
#pragma unroll 1
    for (uint32_t w = WL; w < (uint32_t)TILE; w *= 2) {  // w is a power of two
      // Runs of width w: run A = [a0, b0) ascending, run B = [b0, bend) stored
      // DESCENDING, so that each pair is a bitonic sequence.  Reading one past the
      // end of A lands on B's largest key and one past the end of B on A's largest:
      // neither is ever taken too early, so the merge needs no bounds checks.
      const uint32_t tv = t * V;
      const uint32_t a0 = tv & ~(2 * w - 1);
      const uint32_t b0 = min(a0 + w, (uint32_t)TILE), bend = min(a0 + 2 * w, (uint32_t)TILE);
      const uint32_t la = b0 - a0;
      {
        // this thread's V keys belong to run tv / w; odd runs are stored reversed: the
        // thread's block [tv, tv+V) of run [r0, r0+rlen) lands, reversed, on the block
        // starting at r0 + rlen - V - (tv - r0) (a multiple of V, as rlen is)
        const bool rev = (tv & w) != 0;
        const uint32_t r0 = tv & ~(w - 1);
        const uint32_t rlen = min(w, (uint32_t)TILE - r0);
        const uint32_t q = rev ? 2 * r0 + rlen - V - tv : tv;
        K* sb = s + pad(q);
        __syncthreads();  // previous readers of s are done
        if (w < 32 * V) {  // rev differs within a warp: per-key selects
#pragma unroll
          for (int j = 0; j < V; j++) sb[poff(j)] = rev ? r[V - 1 - j] : r[j];
        } else if (rev) {  // warp-uniform: no selects
#pragma unroll
          for (int j = 0; j < V; j++) sb[poff(j)] = r[V - 1 - j];
        } else {
#pragma unroll
          for (int j = 0; j < V; j++) sb[poff(j)] = r[j];
        }
        __syncthreads();
      }
      if (tv >= len) continue;  // r[] stays all kMax
      merge_bitonic(s, a0, la, bend, tv, r);
    }
    __syncthreads();
    {
      K* sb = s + pad(t * V);
#pragma unroll
      for (int j = 0; j < V; j++) sb[poff(j)] = r[j];
    }
    __syncthreads();
  }
};

// ------------------------------------------------------------------------
// Segment descriptors for batched sorts.
struct SegDesc {
  uint32_t off;  // first element
  uint32_t len;  // number of elements (<= the class's TILE)
};

// Keys-only batched sort: CTA b sorts segment segs[b] from src into dst (same
// offsets; src may equal dst).
template <typename K, int NT, int V>
__global__ void __launch_bounds__(NT)
k_blocksort(const SegDesc* __restrict__ segs, const K* __restrict__ src, K* __restrict__ dst) {
  using BS = BlockSort<K, NT, V>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K* s = reinterpret_cast<K*>(smem_raw);
  const SegDesc d = segs[blockIdx.x];
  const K* in = src + d.off;
  for (int i = threadIdx.x; i < BS::TILE; i += NT) s[BS::pad(i)] = i < (int)d.len ? in[i] : KeyTraits<K>::kMax;
  __syncthreads();
  BS::sort_smem(s, d.len);
  K* out = dst + d.off;
  for (int i = threadIdx.x; i < (int)d.len; i += NT) out[i] = s[BS::pad(i)];
}

// Pairs batched sort (u32 or u64 keys, u32 payload), stable: composites key<<32 | pos.
template <typename K, int NT, int V>
__global__ void __launch_bounds__(NT)
k_blocksort_pairs(const SegDesc* __restrict__ segs, const K* __restrict__ ksrc,
                  const uint32_t* __restrict__ vsrc, K* __restrict__ kdst,
                  uint32_t* __restrict__ vdst) {
  using SK = sortkey_t<K, true>;
  using BS = BlockSort<SK, NT, V>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SK* s = reinterpret_cast<SK*>(smem_raw);
  uint32_t* vs = reinterpret_cast<uint32_t*>(smem_raw + BS::SMEM_BYTES);
  const SegDesc d = segs[blockIdx.x];
  for (int i = threadIdx.x; i < BS::TILE; i += NT) {
    SK c = KeyTraits<SK>::kMax;
    if (i < (int)d.len) {
      c = (SK(ksrc[d.off + i]) << 32) | SK(uint32_t(i));
      vs[i] = vsrc[d.off + i];
    }
    s[BS::pad(i)] = c;
  }
  __syncthreads();
  BS::sort_smem(s, d.len);
  for (int i = threadIdx.x; i < (int)d.len; i += NT) {
    const SK c = s[BS::pad(i)];
    kdst[d.off + i] = K(c >> 32);
    vdst[d.off + i] = vs[uint32_t(c)];
  }
}

}  // namespace sq
