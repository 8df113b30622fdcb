/*
 * sqinputs/gen.c -- seeded synthetic input generators.
 *
 * Serves both the CPU oracle (tests) and the GPU path (tests, bench) with the
 * same inputs.  Holds none of SquareSort's arithmetic: it only produces keys.
 * Stream: SplitMix64 seeded with the config seed, x_i = the i-th output
 * (state_i = seed + (i+1)*0x9e3779b97f4a7c15, then the output function).
 */
#include <stdint.h>

static inline uint64_t out_fn(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline uint64_t x_at(uint64_t seed, uint64_t i) {
  return out_fn(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
}
static inline uint64_t scale(uint64_t x, uint64_t n) {
  return (uint64_t)(((unsigned __int128)x * n) >> 64);
}

void sqg_stream(uint64_t seed, uint64_t start, uint64_t n, uint64_t *out) {
  for (uint64_t i = 0; i < n; i++) out[i] = x_at(seed, start + i);
}
/* key_i = x_i >> 32: i.i.d. uniform over [0, 2^32). */
void sqg_uniform_u32(uint64_t seed, uint64_t n, uint32_t *out) {
  for (uint64_t i = 0; i < n; i++) out[i] = (uint32_t)(x_at(seed, i) >> 32);
}
/* key_i = floor(x_i * card / 2^64): i.i.d. uniform over [0, card). */
void sqg_uniform_mod_u64(uint64_t seed, uint64_t n, uint64_t card, uint64_t *out) {
  for (uint64_t i = 0; i < n; i++) out[i] = scale(x_at(seed, i), card);
}
/* nswaps random transpositions (i, j), drawn from the stream from `start`. */
void sqg_swaps_u32(uint32_t *a, uint64_t n, uint64_t seed, uint64_t start, uint64_t nswaps) {
  for (uint64_t s = 0; s < nswaps; s++) {
    uint64_t i = scale(x_at(seed, start + 2 * s), n);
    uint64_t j = scale(x_at(seed, start + 2 * s + 1), n);
    uint32_t t = a[i];
    a[i] = a[j];
    a[j] = t;
  }
}
/* Fisher-Yates permutation of 0..n-1: for i = n-1..1, j = floor(x*(i+1)/2^64). */
void sqg_permutation_u32(uint64_t seed, uint64_t n, uint32_t *out) {
  for (uint64_t i = 0; i < n; i++) out[i] = (uint32_t)i;
  uint64_t t = 0;
  for (uint64_t i = n; i-- > 1;) {
    uint64_t j = scale(x_at(seed, t++), i + 1);
    uint32_t v = out[i];
    out[i] = out[j];
    out[j] = v;
  }
}
