// Counter-based randomness on device, bit-exact with chainscan/noise.py.
//
//   mix      = splitmix64 finaliser (noise.py:50-57)
//   hash     = mix(mix(mix(mix(seed+G) ^ (a+G)) ^ (b+G)) ^ (c+G)) (noise.py:60-67)
//   unit     = ((h >> 11) + 0.5) * 2^-53                       (noise.py:70-72)
//   probe    = +1 if bit 63 of hash(seed, 0xA5B35705+it, t, (k<<32)+d) (noise.py:159-171)
//
// All uint64 arithmetic wraps exactly like numpy's uint64, so the hash, the
// uniforms and the Rademacher probes are bit-identical to the reference.  The
// first two rounds depend only on (seed, a) and are hoisted by callers.
#pragma once
#include "cs_common.cuh"

namespace cs {

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kProbeNs = 0xA5B35705ull;

CS_HD uint64_t mix64(uint64_t h) {
  h ^= h >> 30;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 27;
  h *= 0x94D049BB133111EBull;
  h ^= h >> 31;
  return h;
}

// first two rounds: (seed, a) -> h2
CS_HD uint64_t hash_prefix(uint64_t seed, uint64_t a) { return mix64(mix64(seed + kGold) ^ (a + kGold)); }
CS_HD uint64_t hash_t(uint64_t h2, uint64_t t) { return mix64(h2 ^ (t + kGold)); }
CS_HD uint64_t hash_c(uint64_t h3, uint64_t c) { return mix64(h3 ^ (c + kGold)); }

CS_HD double bits_to_unit(uint64_t h) {
  return ((double)(h >> 11) + 0.5) * 1.1102230246251565404e-16;  // 2^-53
}

// probe prefix for one solver iteration (Hutchinson, deer.py:129)
CS_HD uint64_t probe_prefix(uint64_t seed, int64_t iteration) {
  return hash_prefix(seed, kProbeNs + (uint64_t)iteration);
}
// +-1 for (t, sample, d) given the iteration prefix
CS_HD double probe_sign(uint64_t h3, int sample, int d) {
  uint64_t h = hash_c(h3, ((uint64_t)sample << 32) + (uint64_t)d);
  return (h >> 63) ? 1.0 : -1.0;
}

// the same sign from the hash's top bit alone: the final xorshift leaves bit 63
// alone and bit 63 of the last product is bit 31 of its high word, so only that
// word is formed (bit-identical to probe_sign; fewer integer ops per probe)
CS_HD double probe_sign_fast(uint64_t h3, int sample, int d) {
  uint64_t h = h3 ^ ((((uint64_t)sample << 32) + (uint64_t)d) + kGold);
  h ^= h >> 30;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 27;
  constexpr uint64_t M = 0x94D049BB133111EBull;
  const uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
#ifdef __CUDA_ARCH__
  const uint32_t top = __umulhi(lo, (uint32_t)M) + lo * (uint32_t)(M >> 32) + hi * (uint32_t)M;
#else
  const uint32_t top = (uint32_t)(((uint64_t)lo * (uint32_t)M) >> 32) + lo * (uint32_t)(M >> 32) + hi * (uint32_t)M;
#endif
  return (top >> 31) ? 1.0 : -1.0;
}

}  // namespace cs
