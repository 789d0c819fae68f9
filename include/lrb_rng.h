/*
 * lrb_rng.h — counter-based uniform[-1,1) generator shared bit-for-bit by the
 * host (oracle, harness) and the device (fill kernels).
 *
 * The reference seeds every operand from a sequential mt19937_64 +
 * normal_distribution stream (reference: proj/include/lrbatch/common.hpp:78-91,
 * used by LowRankBatch::random, low_rank.hpp:135-145). A sequential stream
 * cannot be regenerated per shard/chunk on a GPU, and BASELINE.json asks for
 * i.i.d. uniform[-1,1) entries per config seed, so the synthetic inputs here
 * are keyed by (seed, role, item, element) instead:
 *
 *   key   = lrb_mix64(seed * GOLDEN + role * ROLE_MUL + ROLE_ADD)
 *   u     = lrb_mix64(key + ((item << 32) | elem) * GOLDEN)     (SplitMix64 step)
 *   value = (u >> 11) * 2^-52 - 1                               (exact in binary64)
 *
 * `elem` is the column-major element index `row + col * rows` inside the item
 * (independent of the leading dimension), so a matrix's values do not depend
 * on how items are packed, padded, sharded or chunked.
 */
#ifndef LRB_RNG_H
#define LRB_RNG_H

#include <stdint.h>

#if defined(__CUDACC__)
#define LRB_HD __host__ __device__ __forceinline__
#else
#define LRB_HD static inline
#endif

#define LRB_RNG_GOLDEN 0x9E3779B97F4A7C15ull
#define LRB_RNG_ROLE_MUL 0xD1B54A32D192ED03ull
#define LRB_RNG_ROLE_ADD 0x632BE59BD9B4E019ull

/* operand roles */
#define LRB_ROLE_A 0u
#define LRB_ROLE_B 1u
#define LRB_ROLE_C 2u
#define LRB_ROLE_SHAPE_B 3u /* cfg4: per-item block size draw */
#define LRB_ROLE_SHAPE_R 4u /* cfg4: per-item rank draw */

LRB_HD uint64_t lrb_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

LRB_HD uint64_t lrb_stream_key(uint64_t seed, uint32_t role) {
  return lrb_mix64(seed * LRB_RNG_GOLDEN + (uint64_t)role * LRB_RNG_ROLE_MUL + LRB_RNG_ROLE_ADD);
}

LRB_HD uint64_t lrb_bits(uint64_t key, uint64_t item, uint64_t elem) {
  return lrb_mix64(key + ((item << 32) | (elem & 0xFFFFFFFFull)) * LRB_RNG_GOLDEN);
}

LRB_HD double lrb_uniform(uint64_t key, uint64_t item, uint64_t elem) {
  /* 53-bit mantissa draw scaled to [0,2) then shifted: exact, in [-1, 1). */
  return (double)(lrb_bits(key, item, elem) >> 11) * (1.0 / 4503599627370496.0) - 1.0;
}

/* uniform integer in [0, n) from the high 32 bits (Lemire multiply-shift) */
LRB_HD uint32_t lrb_below(uint64_t key, uint64_t item, uint32_t n) {
  return (uint32_t)(((lrb_bits(key, item, 0) >> 32) * (uint64_t)n) >> 32);
}

#endif /* LRB_RNG_H */
