// datagen.cuh — counter-based synthetic data (DESIGN.md "Input recipe",
// SURVEY §8(c)-A29), implemented from the written spec:
//   h = splitmix64(splitmix64(splitmix64(seed) ^ job) ^ (tensor_id << 40 | idx >> 1))
//   u = b * 2^-24, b = h >> 40 (idx even) or (h >> 16) & 0xFFFFFF (idx odd)
//   v = fp32((2u - 1) * scale);  value = bf16_rne(v)
//   tensor_id = kind << 20 | layer << 16 | (iteration & 0xFFFF)
#pragma once
#include <stdint.h>

namespace salus {

enum : uint32_t { GEN_W = 0, GEN_X = 1, GEN_T = 2 };

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// per-(job, tensor) key; the element index is or-ed into the low 40 bits
__host__ __device__ __forceinline__ uint64_t gen_key(uint64_t seed, uint32_t job_id, uint32_t kind,
                                                     uint32_t layer, uint32_t iter) {
  uint64_t s = splitmix64(splitmix64(seed) ^ (uint64_t)job_id);
  uint64_t tid = ((uint64_t)kind << 20) | ((uint64_t)layer << 16) | (uint64_t)(iter & 0xFFFFu);
  return s ^ (tid << 40);
}

__device__ __forceinline__ float bf16_rne_f32(float v) {
  uint32_t b = __float_as_uint(v);
  b = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
  return __uint_as_float(b);
}

__device__ __forceinline__ float gen_from_bits(uint32_t bits, float scale) {
  float u = __fmul_rn((float)bits, 5.9604644775390625e-08f);   // 2^-24, exact
  float v = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale);
  return bf16_rne_f32(v);
}

// value of element idx; `key` from gen_key (xor with idx/2 == or, idx < 2^41)
__device__ __forceinline__ float gen_value(uint64_t key, uint64_t idx, float scale) {
  const uint64_t h = splitmix64(key ^ (idx >> 1));
  return gen_from_bits((idx & 1) ? (uint32_t)(h >> 16) & 0xFFFFFFu : (uint32_t)(h >> 40), scale);
}

// N consecutive elements base .. base+N-1 (N even): one hash per element pair
// when base is even (the usual case: even row lengths)
template <int N>
__device__ __forceinline__ void gen_run(uint64_t key, uint64_t base, float scale, float (&v)[N]) {
  if ((base & 1) == 0) {
#pragma unroll
    for (int p = 0; p < N / 2; p++) {
      const uint64_t h = splitmix64(key ^ ((base >> 1) + p));
      v[2 * p] = gen_from_bits((uint32_t)(h >> 40), scale);
      v[2 * p + 1] = gen_from_bits((uint32_t)(h >> 16) & 0xFFFFFFu, scale);
    }
  } else {
#pragma unroll
    for (int x = 0; x < N; x++) v[x] = gen_value(key, base + x, scale);
  }
}

// fp32(1/sqrt(d)) computed in double then rounded, as the oracle does
__host__ __device__ __forceinline__ float gen_wscale(uint32_t d_in) {
  return (float)(1.0 / sqrt((double)d_in));
}

}  // namespace salus
