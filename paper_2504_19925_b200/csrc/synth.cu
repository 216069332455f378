// Harness tooling (include/moe_synth.h): seeded synthetic slot grads and initial master
// weights on the device.  Not on the hot path; never inside a timed region.
// Same counter hash as synth/hashgen.py, implemented independently: values are built from
// hash bits (sign | exponent | mantissa), so no floating-point rounding is involved.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"
#include "moe_synth.h"

namespace {

constexpr uint64_t kGradTag = 0x4752414453ull;      // "GRADS"
constexpr uint64_t kMasterTag = 0x4D4153544552ull;  // "MASTER"

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_synth_grads(uint16_t *dst, uint64_t mix, int32_t t, int32_t slot_base, int32_t S,
                              int64_t P) {
  const int64_t n = (int64_t)S * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = i / P, idx = i - s * P;
    const uint64_t key = mix ^ ((uint64_t)t << 48) ^ ((uint64_t)(slot_base + s) << 32) ^ (uint64_t)idx;
    const uint64_t h = splitmix64(key);
    const uint32_t sign = (uint32_t)(h >> 63) & 1u;
    const uint32_t expo = 112u + (uint32_t)(((h >> 32) & 0xFFFFull) % 12ull);
    const uint32_t mant = (uint32_t)(h >> 8) & 0x7Fu;
    dst[i] = (uint16_t)((sign << 15) | (expo << 7) | mant);
  }
}

__global__ void k_synth_master(uint32_t *dst, uint64_t mix, int32_t E, int64_t lo, int64_t n) {
  const int64_t tot = (int64_t)E * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / n, idx = lo + (i - e * n);
    const uint64_t key = mix ^ ((uint64_t)e << 32) ^ (uint64_t)idx;
    const uint64_t h = splitmix64(key);
    const uint32_t sign = (uint32_t)(h >> 63) & 1u;
    const uint32_t expo = 119u + (uint32_t)(((h >> 32) & 0xFFFFull) % 5ull);
    const uint32_t mant = (uint32_t)(h >> 9) & 0x7FFFFFu;
    dst[i] = (sign << 31) | (expo << 23) | mant;
  }
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

extern "C" int moe_synth_grads(void *dst, uint64_t seed, int32_t t, int32_t slot_base, int32_t S,
                               int64_t P, void *stream) {
  if (!dst || t < 0 || t >= (1 << 16) || slot_base < 0 || S < 0 || slot_base + S > (1 << 16) || P < 0 ||
      P > ((int64_t)1 << 32))
    return moe::fail(MOE_ERR_INVALID, "moe_synth_grads: bad arguments");
  if ((int64_t)S * P == 0) return MOE_OK;
  k_synth_grads<<<grid_for((int64_t)S * P), 256, 0, (cudaStream_t)stream>>>(
      (uint16_t *)dst, splitmix64(seed ^ kGradTag), t, slot_base, S, P);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MOE_OK : moe::fail(MOE_ERR_CUDA, "moe_synth_grads: %s", cudaGetErrorString(e));
}

extern "C" int moe_synth_master(float *dst, uint64_t seed, int32_t E, int64_t lo, int64_t n, void *stream) {
  if (!dst || E < 0 || E > (1 << 16) || lo < 0 || n < 0 || lo + n > ((int64_t)1 << 32))
    return moe::fail(MOE_ERR_INVALID, "moe_synth_master: bad arguments");
  if ((int64_t)E * n == 0) return MOE_OK;
  k_synth_master<<<grid_for((int64_t)E * n), 256, 0, (cudaStream_t)stream>>>(
      (uint32_t *)dst, splitmix64(seed ^ kMasterTag), E, lo, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MOE_OK : moe::fail(MOE_ERR_CUDA, "moe_synth_master: %s", cudaGetErrorString(e));
}
