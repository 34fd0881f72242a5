// The compression point of the gradient channel (steps a6 / a8): 32 -> 16 bits.
//
//   TRUNC16 (reading A5): q = bits(x) >> 16.
//   SR16    (reading A26, the "mathematically correct probabilistic rounding" of
//            PAPER.md:819-821): q = (bits(x) + r) >> 16 with r uniform
//            on [0, 2^16), which rounds |x| up with probability (bits & 0xFFFF) / 2^16;
//            +-Inf / NaN are truncated.
//
// r is drawn by a counter-based generator (reading A27): r = mix32(idx ^ key) >> 16
// with idx the element's position in its layer bucket [dW ; db] and key a mix32
// chain of (seed, step, layer, stage, rank) — stage 0 = the sender's rounding of
// its gradient, stage 1 = the owner's rounding of the mean.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace dflow {

struct Round16 {
  uint32_t key;        // stream key of this compression point
  int32_t stochastic;  // 0: truncation (TRUNC16), 1: probabilistic rounding (SR16)
};

__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

inline uint32_t round16_key(uint32_t seed, uint32_t step, uint32_t layer, uint32_t stage, uint32_t rank) {
  uint32_t k = mix32(stage * 256u + rank);
  k = mix32(layer ^ k);
  k = mix32(step ^ k);
  return mix32(seed ^ k);
}

// bits u of one fp32 value at bucket position idx -> its 16-bit code (low half of the result)
__device__ __forceinline__ uint32_t round16(uint32_t u, uint64_t idx, Round16 r) {
  if (r.stochastic && (u & 0x7F800000u) != 0x7F800000u) u += mix32(static_cast<uint32_t>(idx) ^ r.key) >> 16;
  return u >> 16;
}

}  // namespace dflow
