// fdp_optim.cu -- DP optimizer steps on the finalized gradient.
//
// dp_sgd_step  (dpcore.py:132-136):  theta <- theta - eta * g
// dp_adam_step (dpcore.py:139-156):  m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;
//                                    theta <- theta - (eta / (sqrt(v) + eps)) * m
//                                    (no bias correction, post-update v)
// In place, fp32 or fp64 state, one pass over HBM (HBM-bound: 16 B/elem read +
// 12 B written for fp32 Adam). Optionally the step adds the layer's DP noise
// sigma*C*N(seed, layer, step, offset + i) to g first: the reduce-scatter form
// of data parallelism, where each rank owns a shard of the clipped sum and adds
// the noise of exactly that shard before its optimizer step (noise once).
#include "fdp_internal.h"
#include "fdp_rng.cuh"

namespace fdp {

namespace {

struct NoiseArgs {
  int on;
  int impl;
  float scale;
  uint64_t base, base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long offset;  // flat index of element 0 in the layer's [0, D*P)
};

template <typename T>
__device__ __forceinline__ T noise_at(const NoiseArgs& a, uint64_t base, uint64_t base_g, long long i) {
  const uint64_t idx = static_cast<uint64_t>(a.offset + i);
  if (a.impl == 1) return static_cast<T>(static_cast<double>(a.scale) * keyed_normal_f64(base_g, idx));
  return static_cast<T>(a.scale * noise_draw(a.impl, base_g, base, idx));
}

template <typename T>
__global__ void __launch_bounds__(256) k_adam(T* __restrict__ theta, T* __restrict__ m, T* __restrict__ v,
                                              const T* __restrict__ g, long long n, T eta, T b1, T b2, T eps,
                                              NoiseArgs na) {
  uint64_t base = na.base, base_g = na.base_g;
  if (na.on && na.step_ptr) {
    base = absorb3(na.seed_u, na.layer_u, static_cast<uint64_t>(*na.step_ptr));
    base_g = base + kGamma;
  }
  const T one = static_cast<T>(1);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    T gi = g[i];
    if (na.on) gi += noise_at<T>(na, base, base_g, i);
    const T mi = b1 * m[i] + (one - b1) * gi;
    const T vi = b2 * v[i] + (one - b2) * (gi * gi);
    const T eta_hat = eta / (sqrt(vi) + eps);
    theta[i] = theta[i] - eta_hat * mi;
    m[i] = mi;
    v[i] = vi;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_sgd(T* __restrict__ theta, const T* __restrict__ g, long long n, T eta,
                                             NoiseArgs na) {
  uint64_t base = na.base, base_g = na.base_g;
  if (na.on && na.step_ptr) {
    base = absorb3(na.seed_u, na.layer_u, static_cast<uint64_t>(*na.step_ptr));
    base_g = base + kGamma;
  }
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    T gi = g[i];
    if (na.on) gi += noise_at<T>(na, base, base_g, i);
    theta[i] = theta[i] - eta * gi;
  }
}

int blocks_for(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t optim_step(int adam, int f64, void* theta, void* m, void* v, const void* g, long long n, double eta,
                       double b1, double b2, double eps, const OptimNoise& nz, cudaStream_t s) {
  NoiseArgs na{nz.on, nz.impl, nz.scale, nz.base, nz.base_g, nz.step_ptr, nz.seed_u, nz.layer_u, nz.offset};
  if (n <= 0) return cudaSuccess;
  if (adam) {
    if (f64)
      k_adam<double><<<blocks_for(n), 256, 0, s>>>(static_cast<double*>(theta), static_cast<double*>(m),
                                                   static_cast<double*>(v), static_cast<const double*>(g), n, eta, b1,
                                                   b2, eps, na);
    else
      k_adam<float><<<blocks_for(n), 256, 0, s>>>(static_cast<float*>(theta), static_cast<float*>(m),
                                                  static_cast<float*>(v), static_cast<const float*>(g), n,
                                                  static_cast<float>(eta), static_cast<float>(b1),
                                                  static_cast<float>(b2), static_cast<float>(eps), na);
  } else {
    if (f64)
      k_sgd<double><<<blocks_for(n), 256, 0, s>>>(static_cast<double*>(theta), static_cast<const double*>(g), n, eta,
                                                  na);
    else
      k_sgd<float><<<blocks_for(n), 256, 0, s>>>(static_cast<float*>(theta), static_cast<const float*>(g), n,
                                                 static_cast<float>(eta), na);
  }
  return cudaGetLastError();
}

}  // namespace fdp
