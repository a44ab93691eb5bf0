// fdp_rng.cuh -- counter-based Gaussian noise for the DP epilogue.
//
// KEYED: the reference's construction (/root/reference/pkg/src/dpflows/rng.py:24-85):
//   base  = absorb(seed, layer_id, step)                        rng.py:42-47 (host side)
//   h     = mix64((base + GAMMA) ^ flat_index)                   rng.py:77 (vector tail)
//   w1,w2 = mix64(h ^ SALT_A), mix64(h ^ SALT_B)                 rng.py:51-52
//   u1    = ((w1 >> 11) + 1) * 2^-53  in (0, 1]                  rng.py:53
//   u2    = (w2 >> 11) * 2^-53        in [0, 1)                  rng.py:54
//   n     = sqrt(-2 ln u1) * cos(2 pi u2)                        rng.py:55
// The host passes base_g = base + GAMMA (mod 2^64).
// PHILOX: Philox4x32-10 keyed by base, counter = flat_index (statistical mode).
#pragma once
#include <cstdint>

namespace fdp {

constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;
constexpr uint64_t kSaltA = 0xD1B54A32D192ED03ull;
constexpr uint64_t kSaltB = 0x8BB84B93962EACC9ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

// Reference-keyed draw, final transform in fp32 (|err| vs the fp64 draw ~1e-6).
__device__ __forceinline__ float keyed_normal_f32(uint64_t base_g, uint64_t idx) {
  const uint64_t h = mix64(base_g ^ idx);
  const uint64_t w1 = mix64(h ^ kSaltA) >> 11;
  const uint64_t w2 = mix64(h ^ kSaltB) >> 11;
  // One rounding of the exact 53-bit integer, then an exact power-of-two scale.
  const float u1 = __ull2float_rn(w1 + 1) * 0x1p-53f;
  const float u2 = __ull2float_rn(w2) * 0x1p-53f;
  return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

// Reference-keyed draw in fp64 (libdevice log/cos are within ~1 ulp of libm).
static __device__ __noinline__ double keyed_normal_f64(uint64_t base_g, uint64_t idx) {
  const uint64_t h = mix64(base_g ^ idx);
  const uint64_t w1 = mix64(h ^ kSaltA) >> 11;
  const uint64_t w2 = mix64(h ^ kSaltB) >> 11;
  const double u1 = static_cast<double>(w1 + 1) * 0x1p-53;
  const double u2 = static_cast<double>(w2) * 0x1p-53;
  const double two_pi = 6.283185307179586;  // 2.0 * math.pi as a double (rng.py:33)
  return sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
}

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Philox noise: flat indices are grouped in aligned blocks of 4; block g uses
// one Philox4x32-10 call (counter = g) whose 4 words feed two Box-Muller pairs
// (cos and sin branches). u1 = (w + 1) 2^-32 in (0, 1], angle = 2 pi w 2^-32 - pi.
// The transform uses the SFU approximations (MUFU lg2 / rsqrt / sin / cos,
// ~2^-21 relative): this mode is checked statistically, and every path (fused
// epilogues, fdp_noise) uses this one function, so draws agree bit for bit.
__device__ __forceinline__ float4 philox_normal4(uint64_t base, uint64_t block) {
  uint32_t c[4] = {static_cast<uint32_t>(block), static_cast<uint32_t>(block >> 32), 0x44504E5Au, 0u};
  philox4x32_10(c, static_cast<uint32_t>(base), static_cast<uint32_t>(base >> 32));
  constexpr float kM2Ln2 = -1.3862943611198906f;  // -2 ln 2: -2 ln u = -2 ln2 * log2 u
  const float t0 = fmaxf(kM2Ln2 * __log2f((__uint2float_rn(c[0]) + 1.0f) * 0x1p-32f), 1e-30f);
  const float t1 = fmaxf(kM2Ln2 * __log2f((__uint2float_rn(c[2]) + 1.0f) * 0x1p-32f), 1e-30f);
  const float r0 = t0 * rsqrtf(t0), r1 = t1 * rsqrtf(t1);
  constexpr float kPi = 3.14159265358979f;
  float s0, c0, s1, c1;
  __sincosf(fmaf(__uint2float_rn(c[1]), 0x1p-31f * kPi, -kPi), &s0, &c0);
  __sincosf(fmaf(__uint2float_rn(c[3]), 0x1p-31f * kPi, -kPi), &s1, &c1);
  return make_float4(r0 * c0, r0 * s0, r1 * c1, r1 * s1);
}

__device__ __forceinline__ float philox_normal(uint64_t base, uint64_t idx) {
  const float4 v = philox_normal4(base, idx >> 2);
  switch (idx & 3) {
    case 0: return v.x;
    case 1: return v.y;
    case 2: return v.z;
    default: return v.w;
  }
}

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

// absorb(seed, layer_id, step) of rng.py:42-47 (device side, for device step counters)
__host__ __device__ __forceinline__ uint64_t absorb3(uint64_t seed, uint64_t layer, uint64_t step) {
  uint64_t h = mix64(seed);
  h = mix64((h + kGamma) ^ layer);
  return mix64((h + kGamma) ^ step);
}

// impl: 0 keyed f32, 1 keyed f64, 2 philox. `base_g` = absorb(...) + GAMMA,
// `base` = absorb(...) (philox key).
__device__ __forceinline__ float noise_draw(int impl, uint64_t base_g, uint64_t base, uint64_t idx) {
  if (impl == 2) return philox_normal(base, idx);
  if (impl == 1) return static_cast<float>(keyed_normal_f64(base_g, idx));
  return keyed_normal_f32(base_g, idx);
}

// Draws for the 4 consecutive flat indices idx4*4 .. idx4*4+3.
__device__ __forceinline__ float4 noise_draw4(int impl, uint64_t base_g, uint64_t base, uint64_t idx4) {
  if (impl == 2) return philox_normal4(base, idx4);
  const uint64_t i0 = idx4 << 2;
  if (impl == 1)
    return make_float4(static_cast<float>(keyed_normal_f64(base_g, i0)), static_cast<float>(keyed_normal_f64(base_g, i0 + 1)),
                       static_cast<float>(keyed_normal_f64(base_g, i0 + 2)), static_cast<float>(keyed_normal_f64(base_g, i0 + 3)));
  return make_float4(keyed_normal_f32(base_g, i0), keyed_normal_f32(base_g, i0 + 1), keyed_normal_f32(base_g, i0 + 2),
                     keyed_normal_f32(base_g, i0 + 3));
}

}  // namespace fdp
