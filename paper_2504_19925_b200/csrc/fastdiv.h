// Integer division by a per-expert reciprocal (the dispatch's replica index, reading A8).
// Host-compilable on its own so tests/test_udiv.py can check it exhaustively.
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#define MOE_HD
#else
#define MOE_HD __host__ __device__
#endif

namespace moe {

// n / d for 0 <= n < 2^31, 1 <= d < 2^31, with rd = floor((2^32 - 1) / d): the estimate
// umulhi(n, rd) is exact or one short, fixed by one compare.
MOE_HD inline uint32_t udiv_fast(uint32_t n, uint32_t d, uint32_t rd) {
#ifdef __CUDA_ARCH__
  uint32_t qt = __umulhi(n, rd);
#else
  uint32_t qt = (uint32_t)(((uint64_t)n * rd) >> 32);
#endif
  if (n - qt * d >= d) ++qt;
  return qt;
}

}  // namespace moe
