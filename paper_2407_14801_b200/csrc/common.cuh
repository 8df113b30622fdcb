// common.cuh -- shared device/host helpers of the B200 SquareSort library.
//
// Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
// "L#" = a reading listed in DESIGN.md section 3.  Nothing here is shared with
// the CPU oracle (oracle/): the RNG below is a second, independent
// implementation of the specification in DESIGN.md section 4.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace sq {

// Device-side consistency checks for debug builds (-DSQ_DEBUG_CHECKS, e.g.
// SQ_NVCC_EXTRA=-DSQ_DEBUG_CHECKS python -m paper_2407_14801_b200.build --force):
// an index outside the range its producer promised traps the kernel.  This is
// the memory check of this pool (compute-sanitizer is closed).
#ifdef SQ_DEBUG_CHECKS
#define SQ_CHECK(cond)                                                                        \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("SQ_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                              \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define SQ_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// ---------------------------------------------------------------- RNG (L10)
// mix = SplitMix64's output function applied to z + golden-ratio increment.
__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t root_key(uint64_t seed) { return mix(seed); }
// phase 0 = column child, 1 = bucket child
__host__ __device__ __forceinline__ uint64_t child_key(uint64_t key, uint32_t phase, uint64_t idx) {
  return mix(key ^ mix(2ull * idx + phase));
}
__host__ __device__ __forceinline__ uint64_t draw(uint64_t key, uint32_t round, uint32_t i) {
  return mix(key ^ mix((uint64_t(round) << 32) | uint64_t(i)));
}
// floor(d * len / 2^64): a uniform position in [0, len).
__device__ __forceinline__ uint64_t draw_index(uint64_t d, uint64_t len) { return __umul64hi(d, len); }
inline uint64_t draw_index_host(uint64_t d, uint64_t len) { return (uint64_t)(((unsigned __int128)d * len) >> 64); }

// ---------------------------------------------------------------- m = ceil(sqrt(n))
__host__ __device__ inline uint64_t ceil_sqrt(uint64_t n) {
  uint64_t r = (uint64_t)sqrt((double)n);
  while (r > 0 && r * r >= n) r--;
  while (r * r < n) r++;
  return r;
}

// ---------------------------------------------------------------- key traits
template <typename K> struct KeyTraits;
template <> struct KeyTraits<uint32_t> {
  static constexpr uint32_t kMax = 0xffffffffu;
};
template <> struct KeyTraits<uint64_t> {
  static constexpr uint64_t kMax = 0xffffffffffffffffull;
};
typedef unsigned __int128 u128;
template <> struct KeyTraits<u128> {
  static constexpr u128 kMax = ~u128(0);
};

// The on-chip sort key: the key itself, or for pairs the stable composite
// (key << 32 | position in the tile), L16: 64-bit for u32 keys, 128-bit for u64 keys.
template <typename K, bool PAIRS> struct SortKey { using type = K; };
template <> struct SortKey<uint32_t, true> { using type = uint64_t; };
template <> struct SortKey<uint64_t, true> { using type = u128; };
template <typename K, bool PAIRS> using sortkey_t = typename SortKey<K, PAIRS>::type;

// __shfl_xor_sync for 4-, 8- and 16-byte keys
template <typename K>
__device__ __forceinline__ K shfl_xor_k(K v, int m) {
  if constexpr (sizeof(K) == 16) {
    const uint64_t lo = __shfl_xor_sync(0xffffffffu, uint64_t(v), m);
    const uint64_t hi = __shfl_xor_sync(0xffffffffu, uint64_t(v >> 64), m);
    return (K(hi) << 64) | K(lo);
  } else {
    return __shfl_xor_sync(0xffffffffu, v, m);
  }
}

// ---------------------------------------------------------------- bucket membership
// Boundary j (1 <= j <= k-1) separates bucket j-1 from bucket j.  A key x lies
// before boundary j iff bucket(x) < j, where bucket(x) = #{P < x} + [x in P]
// (closed form of Alg 3 with strict '<' and the equal-pivot rule, L2/L4):
//   x < P[j-1], or x == P[j-1] when P[j-1] repeats P[j-2] (a single-value bucket).
template <typename K>
__host__ __device__ __forceinline__ bool before_boundary(K x, K pj, bool dup) {
  return x < pj || (dup && x == pj);
}

// ---------------------------------------------------------------- smem padding
// One pad word per 32 words keeps blocked per-thread accesses conflict-free.
__host__ __device__ __forceinline__ uint32_t pad32(uint32_t i) { return i + (i >> 5); }

// XOR-swizzled rows of 32 words: the 16-byte chunk c (words [4c, 4c+4)) sits at
// chunk slot c ^ ((c / 8) % 8) of its 128-byte row (the counting sort's tile layout).
__host__ __device__ __forceinline__ uint32_t swz32(uint32_t i) { return i ^ (((i >> 5) & 7) << 2); }

__host__ __device__ constexpr uint32_t ilog2c(uint32_t x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }

}  // namespace sq
