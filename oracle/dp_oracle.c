/* dp_oracle.c -- C restatement of the reference's keyed RNG and DP backward.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ (ctypes) as a second, independent
 * checker next to oracle/dp_oracle.py; never linked into the product.
 *
 *   keyed RNG   rng.py:35-85   (splitmix64 absorb, salted words, Box-Muller; libm)
 *   clip        dpcore.py:41-47
 *   finalize    dpcore.py:60-73
 *   backward    oracle.py:16-65 (per-sample G, norms, clip, sum, finalize), float64
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define GAMMA 0x9E3779B97F4A7C15ull
#define MIX1 0xBF58476D1CE4E5B9ull
#define MIX2 0x94D049BB133111EBull
#define SALT_A 0xD1B54A32D192ED03ull
#define SALT_B 0x8BB84B93962EACC9ull

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}

uint64_t oracle_absorb3(uint64_t seed, uint64_t layer, uint64_t step) {
  uint64_t h = mix64(seed);
  h = mix64((h + GAMMA) ^ layer);
  return mix64((h + GAMMA) ^ step);
}

static double draw(uint64_t base_g, uint64_t idx) {
  uint64_t h = mix64(base_g ^ idx);
  uint64_t w1 = mix64(h ^ SALT_A) >> 11, w2 = mix64(h ^ SALT_B) >> 11;
  double u1 = (double)(w1 + 1) * 0x1p-53;
  double u2 = (double)w2 * 0x1p-53;
  return sqrt(-2.0 * log(u1)) * cos((2.0 * 3.141592653589793) * u2);
}

void oracle_keyed_normal(uint64_t seed, uint64_t layer, uint64_t step, const uint64_t* idx, int64_t n, double* out) {
  uint64_t bg = oracle_absorb3(seed, layer, step) + GAMMA;
  for (int64_t i = 0; i < n; ++i) out[i] = draw(bg, idx[i]);
}

static double clip_factor(double ns, double c) {
  if (ns == 0.0) return 1.0;
  double f = c / sqrt(ns);
  return f < 1.0 ? f : 1.0;
}

/* x (B,T,P), dy (B,T,D) row-major float64 -> grad (D,P), norms (B). */
int oracle_dp_backward(const double* x, const double* dy, int64_t B, int64_t T, int64_t P, int64_t D,
                       double clip_c, double sigma, int mean, uint64_t seed, uint64_t layer, uint64_t step,
                       double* grad, double* norms) {
  double* g = (double*)malloc(sizeof(double) * (size_t)(D * P));
  if (!g) return 1;
  for (int64_t i = 0; i < D * P; ++i) grad[i] = 0.0;
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t i = 0; i < D * P; ++i) g[i] = 0.0;
    for (int64_t t = 0; t < T; ++t) {
      const double* yr = dy + (b * T + t) * D;
      const double* xr = x + (b * T + t) * P;
      for (int64_t d = 0; d < D; ++d) {
        const double yv = yr[d];
        double* gr = g + d * P;
        for (int64_t p = 0; p < P; ++p) gr[p] += yv * xr[p];
      }
    }
    double ns = 0.0;
    for (int64_t i = 0; i < D * P; ++i) ns += g[i] * g[i];
    norms[b] = ns;
    const double f = clip_factor(ns, clip_c);
    for (int64_t i = 0; i < D * P; ++i) grad[i] += f * g[i];
  }
  free(g);
  const uint64_t bg = oracle_absorb3(seed, layer, step) + GAMMA;
  for (int64_t i = 0; i < D * P; ++i) {
    double v = mean ? grad[i] / (double)B : grad[i];
    if (sigma != 0.0) v += sigma * clip_c * draw(bg, (uint64_t)i);
    grad[i] = v;
  }
  return 0;
}
