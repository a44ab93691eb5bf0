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
  const float* gscale;  // deferred clip (fdp_dw_deferred): g = *gscale * grad, rounded, before the noise
};

template <typename T>
__device__ __forceinline__ T noise_at(const NoiseArgs& a, uint64_t base, uint64_t base_g, long long i) {
  const uint64_t idx = static_cast<uint64_t>(a.offset + i);
  if (a.impl == 1) return static_cast<T>(static_cast<double>(a.scale) * keyed_normal_f64(base_g, idx));
  return static_cast<T>(a.scale * noise_draw(a.impl, base_g, base, idx));
}

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }  // never contracted
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(256) k_adam(T* __restrict__ theta, T* __restrict__ m, T* __restrict__ v,
                                              const T* __restrict__ g, long long n, T eta, T b1, T b2, T eps,
                                              NoiseArgs na) {
  const T* gs = reinterpret_cast<const T*>(na.gscale);  // fp32 state only (checked by the C-ABI)
  uint64_t base = na.base, base_g = na.base_g;
  if (na.on && na.step_ptr) {
    base = absorb3(na.seed_u, na.layer_u, static_cast<uint64_t>(*na.step_ptr));
    base_g = base + kGamma;
  }
  const T one = static_cast<T>(1);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    T gi = g[i];
    if (gs) gi = mul_rn(gi, *gs);
    if (na.on) gi += noise_at<T>(na, base, base_g, i);
    const T mi = b1 * m[i] + (one - b1) * gi;
    const T vi = b2 * v[i] + (one - b2) * (gi * gi);
    const T eta_hat = eta / (sqrt(vi) + eps);
    theta[i] = theta[i] - eta_hat * mi;
    m[i] = mi;
    v[i] = vi;
  }
}

// fp32 Adam without noise (all-reduce DP-Adam, the non-DP baseline): float4 streams,
// two quads in flight per thread, evict-first loads; the same per-element arithmetic
// as k_adam<float> (bitwise: identical operation order). Element i4 covers [4 i4, 4 i4 + 4).
__device__ __forceinline__ void adam_quad(float4& t, float4& mm, float4& vv, const float4 gg, float eta, float b1,
                                          float b2, float eps) {
  const float c1 = 1.0f - b1, c2 = 1.0f - b2;
#define FDP_ADAM1(c)                                      \
  {                                                       \
    const float mi = b1 * mm.c + c1 * gg.c;               \
    const float vi = b2 * vv.c + c2 * (gg.c * gg.c);      \
    const float eta_hat = eta / (sqrtf(vi) + eps);        \
    t.c = t.c - eta_hat * mi;                             \
    mm.c = mi;                                            \
    vv.c = vi;                                            \
  }
  FDP_ADAM1(x) FDP_ADAM1(y) FDP_ADAM1(z) FDP_ADAM1(w)
#undef FDP_ADAM1
}

// kNoise: add the shard's Philox noise first, one quad draw per float4 (the noise
// index offset is a multiple of 4, so quad i4 of this segment is Philox block
// offset / 4 + i4 -- the same draws as the scalar kernel's per-element calls)
// The noisy variant is held to 3 resident blocks per SM (<= 85 registers; unbounded it
// took 78 and the occupancy that went with them): 134 M parameters 685-777 -> 603 us,
// the Philox draws then cost nothing over the plain step (6.23 TB/s, tools/hbm_timing.py,
// profiles/r2_adam_occupancy_ab.jsonl)
#ifndef FDP_ADAM_NOISE_MINB
#define FDP_ADAM_NOISE_MINB 3
#endif
template <bool kNoise>
__global__ void __launch_bounds__(256, kNoise ? FDP_ADAM_NOISE_MINB : 1) k_adam_f32x4(float4* __restrict__ theta, float4* __restrict__ m,
                                                    float4* __restrict__ v, const float4* __restrict__ g,
                                                    long long n4, float eta, float b1, float b2, float eps,
                                                    NoiseArgs na) {
  uint64_t base = na.base;
  if (kNoise && na.step_ptr) base = absorb3(na.seed_u, na.layer_u, static_cast<uint64_t>(*na.step_ptr));
  const uint64_t q0 = static_cast<uint64_t>(na.offset) >> 2;
  const float f = na.gscale ? *na.gscale : 1.0f;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4; i += 2 * stride) {
    const long long j = i + stride;
    const bool two = j < n4;
    float4 g0 = __ldcs(g + i), m0 = __ldcs(m + i), v0 = __ldcs(v + i), t0 = __ldcs(theta + i);
    float4 g1 = g0, m1 = m0, v1 = v0, t1 = t0;
    if (two) {
      g1 = __ldcs(g + j);
      m1 = __ldcs(m + j);
      v1 = __ldcs(v + j);
      t1 = __ldcs(theta + j);
    }
    if (na.gscale) {  // __fmul_rn: the same rounding as the finalize pass (fdp_simt.cu k_single_finalize)
      g0.x = __fmul_rn(g0.x, f);
      g0.y = __fmul_rn(g0.y, f);
      g0.z = __fmul_rn(g0.z, f);
      g0.w = __fmul_rn(g0.w, f);
      g1.x = __fmul_rn(g1.x, f);
      g1.y = __fmul_rn(g1.y, f);
      g1.z = __fmul_rn(g1.z, f);
      g1.w = __fmul_rn(g1.w, f);
    }
    if constexpr (kNoise) {
      const float4 z0 = philox_normal4(base, q0 + static_cast<uint64_t>(i));
      g0.x += na.scale * z0.x;
      g0.y += na.scale * z0.y;
      g0.z += na.scale * z0.z;
      g0.w += na.scale * z0.w;
      if (two) {
        const float4 z1 = philox_normal4(base, q0 + static_cast<uint64_t>(j));
        g1.x += na.scale * z1.x;
        g1.y += na.scale * z1.y;
        g1.z += na.scale * z1.z;
        g1.w += na.scale * z1.w;
      }
    }
    adam_quad(t0, m0, v0, g0, eta, b1, b2, eps);
    __stcs(theta + i, t0);
    __stcs(m + i, m0);
    __stcs(v + i, v0);
    if (two) {
      adam_quad(t1, m1, v1, g1, eta, b1, b2, eps);
      __stcs(theta + j, t1);
      __stcs(m + j, m1);
      __stcs(v + j, v1);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_sgd(T* __restrict__ theta, const T* __restrict__ g, long long n, T eta,
                                             NoiseArgs na) {
  const T* gs = reinterpret_cast<const T*>(na.gscale);  // fp32 state only (checked by the C-ABI)
  uint64_t base = na.base, base_g = na.base_g;
  if (na.on && na.step_ptr) {
    base = absorb3(na.seed_u, na.layer_u, static_cast<uint64_t>(*na.step_ptr));
    base_g = base + kGamma;
  }
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    T gi = g[i];
    if (gs) gi = mul_rn(gi, *gs);
    if (na.on) gi += noise_at<T>(na, base, base_g, i);
    theta[i] = theta[i] - eta * gi;
  }
}

// ---- multi-segment fp32 Adam (fdp_adam_step_multi): every parameter segment of an
// optimizer step in ONE launch. Segment table in device memory (AdamSeg, prefix q0 over
// quads); a block walks one contiguous chunk of quads, so a thread's consecutive quads
// stay in one segment and the segment lookup / noise key are recomputed only on change.
// Per element the arithmetic is k_adam_f32x4's: grad * scale (__fmul_rn), + sigma*C*z
// (Philox, one draw per quad of the segment's index space), then adam_quad.
constexpr int kMultiChunk = 256 * 8;  // quads per block

__device__ __forceinline__ int seg_of(const AdamSeg* segs, int n_seg, long long q) {
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].q0 <= q) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// kAdam false: the plain DP-SGD step theta -= eta * g (k_sgd's arithmetic; m / v unused)
template <bool kAdam>
__global__ void __launch_bounds__(256, FDP_ADAM_NOISE_MINB) k_adam_multi(const AdamSeg* __restrict__ segs, int n_seg,
                                                                         long long total_q, float eta, float b1,
                                                                         float b2, float eps) {
  const long long c0 = static_cast<long long>(blockIdx.x) * kMultiChunk;
  int cur = -1;
  AdamSeg S{};
  uint64_t base = 0;
  float f = 1.0f;
  for (long long q = c0 + threadIdx.x; q < c0 + kMultiChunk && q < total_q; q += blockDim.x) {
    if (cur < 0 || q < S.q0 || q >= S.q0 + ((S.n + 3) >> 2)) {
      cur = seg_of(segs, n_seg, q);
      S = segs[cur];
      base = S.base;
      if (S.noise_on && S.step_ptr) base = absorb3(S.seed_u, S.layer_u, static_cast<uint64_t>(*S.step_ptr));
      f = S.gscale ? *S.gscale : 1.0f;
    }
    const long long lq = q - S.q0;
    const long long e0 = lq << 2;
    float4* th4 = reinterpret_cast<float4*>(S.theta);
    float4* m4 = reinterpret_cast<float4*>(S.m);
    float4* v4 = reinterpret_cast<float4*>(S.v);
    const float4* g4 = reinterpret_cast<const float4*>(S.g);
    const bool full = e0 + 4 <= S.n;
    float4 gg, mm = make_float4(0.f, 0.f, 0.f, 0.f), vv = mm, tt;
    if (full) {
      gg = __ldcs(g4 + lq);
      if constexpr (kAdam) {
        mm = __ldcs(m4 + lq);
        vv = __ldcs(v4 + lq);
      }
      tt = __ldcs(th4 + lq);
    } else {  // the segment's last partial quad (elements past n are never stored)
      const long long r = S.n - e0;
      gg = make_float4(S.g[e0], r > 1 ? S.g[e0 + 1] : 0.f, r > 2 ? S.g[e0 + 2] : 0.f, 0.f);
      if constexpr (kAdam) {
        mm = make_float4(S.m[e0], r > 1 ? S.m[e0 + 1] : 0.f, r > 2 ? S.m[e0 + 2] : 0.f, 0.f);
        vv = make_float4(S.v[e0], r > 1 ? S.v[e0 + 1] : 0.f, r > 2 ? S.v[e0 + 2] : 0.f, 0.f);
      }
      tt = make_float4(S.theta[e0], r > 1 ? S.theta[e0 + 1] : 0.f, r > 2 ? S.theta[e0 + 2] : 0.f, 0.f);
    }
    if (S.gscale) {
      gg.x = __fmul_rn(gg.x, f);
      gg.y = __fmul_rn(gg.y, f);
      gg.z = __fmul_rn(gg.z, f);
      gg.w = __fmul_rn(gg.w, f);
    }
    if (S.noise_on) {
      const float4 z = philox_normal4(base, S.noise_q0 + static_cast<uint64_t>(lq));
      gg.x += S.scale * z.x;
      gg.y += S.scale * z.y;
      gg.z += S.scale * z.z;
      gg.w += S.scale * z.w;
    }
    if constexpr (kAdam) {
      adam_quad(tt, mm, vv, gg, eta, b1, b2, eps);
    } else {
      tt.x = tt.x - eta * gg.x;
      tt.y = tt.y - eta * gg.y;
      tt.z = tt.z - eta * gg.z;
      tt.w = tt.w - eta * gg.w;
    }
    if (full) {
      __stcs(th4 + lq, tt);
      if constexpr (kAdam) {
        __stcs(m4 + lq, mm);
        __stcs(v4 + lq, vv);
      }
    } else {
      const long long r = S.n - e0;
      S.theta[e0] = tt.x;
      if (r > 1) S.theta[e0 + 1] = tt.y;
      if (r > 2) S.theta[e0 + 2] = tt.z;
      if constexpr (kAdam) {
        S.m[e0] = mm.x;
        S.v[e0] = vv.x;
        if (r > 1) { S.m[e0 + 1] = mm.y; S.v[e0 + 1] = vv.y; }
        if (r > 2) { S.m[e0 + 2] = mm.z; S.v[e0 + 2] = vv.z; }
      }
    }
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
  NoiseArgs na{nz.on, nz.impl, nz.scale, nz.base, nz.base_g, nz.step_ptr, nz.seed_u, nz.layer_u, nz.offset,
               nz.grad_scale};
  if (n <= 0) return cudaSuccess;
  if (adam) {
    if (f64)
      k_adam<double><<<blocks_for(n), 256, 0, s>>>(static_cast<double*>(theta), static_cast<double*>(m),
                                                   static_cast<double*>(v), static_cast<const double*>(g), n, eta, b1,
                                                   b2, eps, na);
    else if ((!na.on || (na.impl == 2 && (na.offset & 3) == 0)) &&
             ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(m) |
               reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(g)) & 15u) == 0) {
      // quads over the aligned body (Philox noise: one draw per quad), the scalar kernel for the tail
      const long long n4 = n >> 2;
      if (n4 > 0) {
        long long blocks = (n4 + 511) / 512;
        if (blocks > 148LL * 8) blocks = 148LL * 8;
        auto k = na.on ? k_adam_f32x4<true> : k_adam_f32x4<false>;
        k<<<static_cast<int>(blocks), 256, 0, s>>>(
            static_cast<float4*>(theta), static_cast<float4*>(m), static_cast<float4*>(v),
            static_cast<const float4*>(g), n4, static_cast<float>(eta), static_cast<float>(b1),
            static_cast<float>(b2), static_cast<float>(eps), na);
      }
      const long long done = n4 << 2;
      if (done < n) {
        NoiseArgs tail = na;
        tail.offset += done;
        k_adam<float><<<1, 256, 0, s>>>(static_cast<float*>(theta) + done, static_cast<float*>(m) + done,
                                        static_cast<float*>(v) + done, static_cast<const float*>(g) + done, n - done,
                                        static_cast<float>(eta), static_cast<float>(b1), static_cast<float>(b2),
                                        static_cast<float>(eps), tail);
      }
    } else {
      k_adam<float><<<blocks_for(n), 256, 0, s>>>(static_cast<float*>(theta), static_cast<float*>(m),
                                                  static_cast<float*>(v), static_cast<const float*>(g), n,
                                                  static_cast<float>(eta), static_cast<float>(b1),
                                                  static_cast<float>(b2), static_cast<float>(eps), na);
    }
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

cudaError_t adam_multi(const AdamSeg* dev_segs, int n_seg, long long total_q, double eta, double b1, double b2,
                       double eps, cudaStream_t s, bool adam) {
  if (n_seg <= 0 || total_q <= 0) return cudaSuccess;
  const long long blocks = (total_q + kMultiChunk - 1) / kMultiChunk;
  auto k = adam ? k_adam_multi<true> : k_adam_multi<false>;
  k<<<static_cast<unsigned>(blocks), 256, 0, s>>>(dev_segs, n_seg, total_q, static_cast<float>(eta),
                                                  static_cast<float>(b1), static_cast<float>(b2),
                                                  static_cast<float>(eps));
  return cudaGetLastError();
}

}  // namespace fdp
