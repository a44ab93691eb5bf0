// fdp_simt.cu -- CUDA-core kernels: the generic path for any shape / fp32 inputs,
// the explicit (Opacus-style) baseline stages, the norm->clip-factor reduction and
// standalone keyed noise.
//
// The generic DP path is the two-pass structure of backward_implicit
// (workflows.py:246-324): pass 1 reduces per-sample norm^2 partials per 32x32
// tile without storing G, pass 2 recomputes the tiles and sums c_b * G_b. It is
// exact fp32 FMA arithmetic, so fp32 inputs meet the 1e-5 bar.
#include <cstdlib>

#include "fdp_internal.h"
#include "fdp_ptx.cuh"
#include "fdp_rng.cuh"
#include <cuda_bf16.h>

namespace fdp {

namespace {

constexpr int kTS = 32;  // tile extent (d, p, and t chunk)

__device__ __forceinline__ float load_in(const void* base, long long idx, int in_f32) {
  if (in_f32) return static_cast<const float*>(base)[idx];
  return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
}

// Accumulate the 2x2 micro-tile of G_b[d0 + 2ty + {0,1}, p0 + 2tx + {0,1}] over all t.
__device__ __forceinline__ void sample_tile(const SimtParams& p, int b, int d0, int p0, float (&g)[2][2],
                                            float (*sy)[kTS + 1], float (*sx)[kTS + 1]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  g[0][0] = g[0][1] = g[1][0] = g[1][1] = 0.0f;
  const long long ybase = static_cast<long long>(b) * p.T * p.D;
  const long long xbase = static_cast<long long>(b) * p.T * p.P;
  for (int t0 = 0; t0 < p.T; t0 += kTS) {
    for (int e = threadIdx.x; e < kTS * kTS; e += blockDim.x) {
      const int tt = e / kTS, cc = e % kTS;
      const int t = t0 + tt;
      const int dd = d0 + cc, pp = p0 + cc;
      sy[tt][cc] = (t < p.T && dd < p.D) ? load_in(p.dy, ybase + static_cast<long long>(t) * p.D + dd, p.in_f32) : 0.0f;
      sx[tt][cc] = (t < p.T && pp < p.P) ? load_in(p.x, xbase + static_cast<long long>(t) * p.P + pp, p.in_f32) : 0.0f;
    }
    __syncthreads();
#pragma unroll 8
    for (int tt = 0; tt < kTS; ++tt) {
      const float y0 = sy[tt][2 * ty], y1 = sy[tt][2 * ty + 1];
      const float x0 = sx[tt][2 * tx], x1 = sx[tt][2 * tx + 1];
      g[0][0] = fmaf(y0, x0, g[0][0]);
      g[0][1] = fmaf(y0, x1, g[0][1]);
      g[1][0] = fmaf(y1, x0, g[1][0]);
      g[1][1] = fmaf(y1, x1, g[1][1]);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_partial_norms(const SimtParams p) {
  __shared__ float sy[kTS][kTS + 1];
  __shared__ float sx[kTS][kTS + 1];
  __shared__ float red[8];
  const int pt = blockIdx.x, dt = blockIdx.y, b = blockIdx.z;
  float g[2][2];
  sample_tile(p, b, dt * kTS, pt * kTS, g, sy, sx);
  float s = g[0][0] * g[0][0] + g[0][1] * g[0][1] + g[1][0] * g[1][0] + g[1][1] * g[1][1];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int w = 0; w < 8; ++w) t += red[w];
    p.ws_part[static_cast<long long>(b) * p.n_tiles + dt * p.n_pt + pt] = t;
  }
}

// One warp per sample: fixed-order double sum of the partials -> norm^2, clip factor.
__global__ void k_reduce_norms(const float* part, int B, int n_tiles, double clip_c, double clip_c2,
                               float inv_batch, float* norms_out, float* factors) {
  pdl_launch_dependents();  // the reweight may start its prologue / mainloop now
  pdl_wait();               // the norm partials are complete (no-op without PDL)
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  double s = 0.0;
  for (int i = lane; i < n_tiles; i += 32) s += static_cast<double>(part[static_cast<long long>(b) * n_tiles + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const double cf = (s <= clip_c2) ? 1.0 : clip_c / sqrt(s);  // dpcore.py:41-47
    if (norms_out) norms_out[b] = static_cast<float>(s);
    if (factors) factors[b] = static_cast<float>(cf) * inv_batch;
  }
}

__device__ __forceinline__ float draw(const SimtParams& p, long long flat) {
  uint64_t kb = p.key_base, kbg = p.key_base_g;
  if (p.step_ptr) {
    kb = absorb3(p.seed_u, p.layer_u, static_cast<uint64_t>(*p.step_ptr));
    kbg = kb + kGamma;
  }
  return noise_draw(p.noise_impl, kbg, kb, static_cast<uint64_t>(flat));
}

__global__ void __launch_bounds__(256) k_weighted_sum(const SimtParams p) {
  __shared__ float sy[kTS][kTS + 1];
  __shared__ float sx[kTS][kTS + 1];
  const int pt = blockIdx.x, dt = blockIdx.y;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  for (int b = 0; b < p.B; ++b) {
    float g[2][2];
    sample_tile(p, b, dt * kTS, pt * kTS, g, sy, sx);
    const float f = p.with_clip ? p.ws_factor[b] : 1.0f;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j] = fmaf(f, g[i][j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int d = dt * kTS + 2 * ty + i;
    if (d >= p.D) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int pp = pt * kTS + 2 * tx + j;
      if (pp >= p.P) continue;
      const long long flat = static_cast<long long>(d) * p.P + pp;
      float v = acc[i][j];
      if (p.with_clip && p.add_noise && flat >= p.noise_lo && flat < p.noise_hi) v += p.noise_scale * draw(p, flat);
      if (p.accumulate) v += p.grad_w[flat];
      p.grad_w[flat] = v;
    }
  }
}

__global__ void __launch_bounds__(256) k_store_g(const SimtParams p, float* gout) {
  __shared__ float sy[kTS][kTS + 1];
  __shared__ float sx[kTS][kTS + 1];
  const int pt = blockIdx.x, dt = blockIdx.y, b = blockIdx.z;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float g[2][2];
  sample_tile(p, b, dt * kTS, pt * kTS, g, sy, sx);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int d = dt * kTS + 2 * ty + i;
    if (d >= p.D) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int pp = pt * kTS + 2 * tx + j;
      if (pp < p.P) gout[(static_cast<long long>(b) * p.D + d) * p.P + pp] = g[i][j];
    }
  }
}

// Explicit stage 2 (workflows.py:197-210): per-sample squared norm partials.
__global__ void __launch_bounds__(256) k_explicit_norms(const float* g, long long DP, int nchunks, float* part) {
  __shared__ float red[8];
  const int chunk = blockIdx.x, b = blockIdx.y;
  const long long per = (DP + nchunks - 1) / nchunks;
  const long long lo = chunk * per, hi = (lo + per < DP) ? lo + per : DP;
  const float* gb = g + static_cast<long long>(b) * DP;
  float s = 0.0f;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) s = fmaf(gb[i], gb[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[static_cast<long long>(b) * nchunks + chunk] = t;
  }
}

// Explicit stage 3 (workflows.py:212-225): G' = c_b * G, written to a second buffer.
__global__ void k_explicit_clip(const float* __restrict__ g, float* __restrict__ gp, const float* factors, int B,
                                long long DP) {
  const long long n = static_cast<long long>(B) * DP;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    gp[i] = factors[i / DP] * g[i];
}

// Explicit stage 4 (workflows.py:227-237): sum over samples, finalize with noise.
__global__ void k_explicit_sum(const float* __restrict__ gp, int B, long long DP, const SimtParams p) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < DP;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float s = 0.0f;
    for (int b = 0; b < B; ++b) s += gp[static_cast<long long>(b) * DP + i];
    float v = s * p.inv_batch;
    if (p.add_noise && i >= p.noise_lo && i < p.noise_hi) v += p.noise_scale * draw(p, i);
    if (p.accumulate) v += p.grad_w[i];
    p.grad_w[i] = v;
  }
}

__global__ void k_noise_fill(float* out, long long lo, long long hi, float scale, int impl, uint64_t base,
                             uint64_t base_g) {
  for (long long i = lo + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < hi;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (impl == 1)
      out[i - lo] = static_cast<float>(static_cast<double>(scale) * keyed_normal_f64(base_g, static_cast<uint64_t>(i)));
    else
      out[i - lo] = scale * noise_draw(impl, base_g, base, static_cast<uint64_t>(i));
  }
}

__global__ void k_noise_fill64(double* out, long long lo, long long hi, double scale, int impl, uint64_t base,
                               uint64_t base_g) {
  for (long long i = lo + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < hi;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (impl == 1)
      out[i - lo] = scale * keyed_normal_f64(base_g, static_cast<uint64_t>(i));
    else
      out[i - lo] = scale * static_cast<double>(noise_draw(impl, base_g, base, static_cast<uint64_t>(i)));
  }
}

// kMode: 0 = any noise impl (per-element range checks), 1 = Philox with the whole
// range noised, 2 = no noise. The Philox / no-noise variants are lean enough
// to keep 48 warps per SM streaming, which the elementwise pass needs to reach
// HBM bandwidth with the Philox arithmetic interleaved.
template <int kMode, int kUV = 2, int kMinB = 6>
__global__ void __launch_bounds__(256, kMode == 0 ? 1 : kMinB)
    k_single_finalize(float* __restrict__ g, long long n, const float* __restrict__ part, int n_parts, double clip_c,
                      double clip_c2, float inv_batch, float* norms_out, int add_noise, int impl, float scale,
                      uint64_t base, uint64_t base_g, const long long* step_ptr, uint64_t seed_u, uint64_t layer_u,
                      long long lo, long long hi) {
  pdl_wait();  // PDL launch behind the single-sample GEMM: G and its partials are complete
  float4* g4 = reinterpret_cast<float4*>(g);
  const long long n4 = n >> 2;  // n = D * P, P % 8 == 0
  constexpr int kU = kMode == 0 ? 4 : kUV;  // float4 per thread per iteration: loads in flight
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  float4 v[kU];
  auto load = [&]() {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long i = i0 + u * stride;
      if (i < n4) v[u] = __ldcs(g4 + i);
    }
  };
  load();  // the first loads are in flight while warp 0 forms the clip factor
  __shared__ float s_f;
  if (threadIdx.x < 32) {  // every block sums the partials in the same fixed order
    double t = 0.0;
    for (int i = threadIdx.x; i < n_parts; i += 32) t += static_cast<double>(part[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      const double cf = (t <= clip_c2) ? 1.0 : clip_c / sqrt(t);  // dpcore.py:41-47
      s_f = static_cast<float>(cf) * inv_batch;
      if (blockIdx.x == 0 && norms_out) norms_out[0] = static_cast<float>(t);
    }
  }
  __syncthreads();
  const float f = s_f;
  if (step_ptr) {
    base = absorb3(seed_u, layer_u, static_cast<uint64_t>(*step_ptr));
    base_g = base + kGamma;
  }
  for (; i0 < n4; i0 += stride * kU, load()) {
    float4 z[kU];
    if constexpr (kMode == 1) {  // the draws do not depend on the loads in flight: compute them first
#pragma unroll
      for (int u = 0; u < kU; ++u) z[u] = philox_normal4(base, static_cast<uint64_t>(i0 + u * stride));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long i = i0 + u * stride;
      if (i >= n4) continue;
      // explicit roundings (c * G, then one fma with the noise): the same bits as the
      // finalize a stream-K GEMM carries for a deferred chain (fdp_stream.cu fin_chunk)
      v[u].x = __fmul_rn(v[u].x, f);
      v[u].y = __fmul_rn(v[u].y, f);
      v[u].z = __fmul_rn(v[u].z, f);
      v[u].w = __fmul_rn(v[u].w, f);
      if constexpr (kMode == 1) {
        v[u].x = __fmaf_rn(scale, z[u].x, v[u].x);
        v[u].y = __fmaf_rn(scale, z[u].y, v[u].y);
        v[u].z = __fmaf_rn(scale, z[u].z, v[u].z);
        v[u].w = __fmaf_rn(scale, z[u].w, v[u].w);
      } else if constexpr (kMode == 0) {
        const long long e = i << 2;
        if (add_noise && e + 3 >= lo && e < hi) {
          const float4 z = impl == 2 ? philox_normal4(base, static_cast<uint64_t>(i))
                                     : noise_draw4(impl, base_g, base, static_cast<uint64_t>(i));
          if (e + 0 >= lo && e + 0 < hi) v[u].x = __fmaf_rn(scale, z.x, v[u].x);
          if (e + 1 >= lo && e + 1 < hi) v[u].y = __fmaf_rn(scale, z.y, v[u].y);
          if (e + 2 >= lo && e + 2 < hi) v[u].z = __fmaf_rn(scale, z.z, v[u].z);
          if (e + 3 >= lo && e + 3 < hi) v[u].w = __fmaf_rn(scale, z.w, v[u].w);
        }
      }
      __stcs(g4 + i, v[u]);
    }
  }
}

// FDP_PDL=0 turns the programmatic dependent launches off (A/B)
bool pdl_enabled() {
  const char* v = std::getenv("FDP_PDL");
  return !v || std::atoi(v) != 0;
}

int grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

cudaError_t single_sample_finalize(float* grad_w, long long n, const float* part, int n_parts, double clip_c,
                                   double clip_c2, float inv_batch, float* norms_out, int add_noise, int impl,
                                   float noise_scale, uint64_t base, uint64_t base_g, const long long* step_ptr,
                                   uint64_t seed_u, uint64_t layer_u, long long lo, long long hi, cudaStream_t s) {
  // Philox over the whole tensor (the common case) or no noise: the lean variants
  const int mode = !add_noise || hi <= lo ? 2 : (impl == 2 && lo <= 0 && hi >= n) ? 1 : 0;
  const int threads = 256;
  // plain launch: as a programmatic dependent of the GEMM (its blocks resident early, waiting)
  // it measured 1-2 % slower on the up / down projections, neutral on square ones
  // (profiles/r2_pdl_ab.jsonl); the kernel's griddepcontrol.wait is then a no-op
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (mode == 0) {
    cfg.gridDim = dim3(grid_for(n / 16, threads));
    return cudaLaunchKernelEx(&cfg, k_single_finalize<0>, grad_w, n, part, n_parts, clip_c, clip_c2, inv_batch,
                              norms_out, add_noise, impl, noise_scale, base, base_g, step_ptr, seed_u, layer_u, lo, hi);
  } else {
    long long blocks = (n / 8 + threads - 1) / threads;
    const long long cap = 148LL * 6 * 4;  // 6 resident blocks per SM, a few rounds each
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    // measured (tools/ab_layer.py): 4 float4 per thread at 4 blocks/SM, or 8 blocks/SM, are slower;
    // the pass sits at HBM speed without noise and the Philox draws add ~20 %
    auto k = mode == 1 ? k_single_finalize<1> : k_single_finalize<2>;
    cfg.gridDim = dim3(static_cast<unsigned>(blocks));
    return cudaLaunchKernelEx(&cfg, k, grad_w, n, part, n_parts, clip_c, clip_c2, inv_batch, norms_out, add_noise,
                              impl, noise_scale, base, base_g, step_ptr, seed_u, layer_u, lo, hi);
  }
}

// spill combine: out = (accumulate ? out : 0) + sum_b fac[b] * G[b] (+ noise), b in order
// (fixed fp32 order), float4 streams; kMode as in k_single_finalize.
template <int kMode>
__global__ void __launch_bounds__(256) k_spill_combine(float* __restrict__ out, const float* __restrict__ G, int B,
                                                       long long n, const float* __restrict__ fac, int accumulate,
                                                       int impl, float scale, uint64_t base, uint64_t base_g,
                                                       const long long* step_ptr, uint64_t seed_u, uint64_t layer_u,
                                                       long long lo, long long hi) {
  __shared__ float s_fac[64];
  for (int b = threadIdx.x; b < B && b < 64; b += blockDim.x) s_fac[b] = fac[b];
  __syncthreads();
  if (kMode != 2 && step_ptr) {
    base = absorb3(seed_u, layer_u, static_cast<uint64_t>(*step_ptr));
    base_g = base + kGamma;
  }
  float4* o4 = reinterpret_cast<float4*>(out);
  const float4* g4 = reinterpret_cast<const float4*>(G);
  const long long n4 = n >> 2;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 a = accumulate ? o4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int b = 0; b < B; ++b) {
      const float f = b < 64 ? s_fac[b] : fac[b];
      const float4 g = __ldcs(g4 + static_cast<long long>(b) * n4 + i);
      a.x = __fmaf_rn(f, g.x, a.x);
      a.y = __fmaf_rn(f, g.y, a.y);
      a.z = __fmaf_rn(f, g.z, a.z);
      a.w = __fmaf_rn(f, g.w, a.w);
    }
    if constexpr (kMode == 1) {
      const float4 z = philox_normal4(base, static_cast<uint64_t>(i));
      a.x = __fmaf_rn(scale, z.x, a.x);
      a.y = __fmaf_rn(scale, z.y, a.y);
      a.z = __fmaf_rn(scale, z.z, a.z);
      a.w = __fmaf_rn(scale, z.w, a.w);
    } else if constexpr (kMode == 0) {
      const long long e = i << 2;
      if (e + 3 >= lo && e < hi) {
        const float4 z = impl == 2 ? philox_normal4(base, static_cast<uint64_t>(i))
                                   : noise_draw4(impl, base_g, base, static_cast<uint64_t>(i));
        if (e + 0 >= lo && e + 0 < hi) a.x = __fmaf_rn(scale, z.x, a.x);
        if (e + 1 >= lo && e + 1 < hi) a.y = __fmaf_rn(scale, z.y, a.y);
        if (e + 2 >= lo && e + 2 < hi) a.z = __fmaf_rn(scale, z.z, a.z);
        if (e + 3 >= lo && e + 3 < hi) a.w = __fmaf_rn(scale, z.w, a.w);
      }
    }
    __stcs(o4 + i, a);
  }
}

cudaError_t spill_combine(float* out, const float* G, int B, long long n, const float* fac, int accumulate,
                          int add_noise, int impl, float scale, uint64_t base, uint64_t base_g,
                          const long long* step_ptr, uint64_t seed_u, uint64_t layer_u, long long lo, long long hi,
                          cudaStream_t s) {
  const int mode = !add_noise || hi <= lo ? 2 : (impl == 2 && lo <= 0 && hi >= n) ? 1 : 0;
  long long blocks = (n / 4 + 255) / 256;
  if (blocks > 148LL * 8) blocks = 148LL * 8;
  if (blocks < 1) blocks = 1;
  auto k = mode == 1 ? k_spill_combine<1> : mode == 0 ? k_spill_combine<0> : k_spill_combine<2>;
  k<<<static_cast<int>(blocks), 256, 0, s>>>(out, G, B, n, fac, accumulate, impl, scale, base, base_g, step_ptr, seed_u,
                                             layer_u, lo, hi);
  return cudaGetLastError();
}

// Deferred clip (fdp_dw_deferred): the finalize's clip factor without its pass over
// grad_w. One warp sums the partials in k_single_finalize's fixed order and writes
// scale_out[0] = float(c) * inv_batch (the same float the pass multiplies by) and
// ||G||^2; part == nullptr writes scale 1 (the call finalised grad_w in place).
__global__ void k_single_factor(const float* __restrict__ part, int n_parts, double clip_c, double clip_c2,
                                float inv_batch, float* norms_out, float* scale_out) {
  pdl_wait();  // PDL launch behind the single-sample GEMM
  if (!part) {
    if (threadIdx.x == 0) scale_out[0] = 1.0f;
    return;
  }
  double t = 0.0;
  for (int i = threadIdx.x; i < n_parts; i += 32) t += static_cast<double>(part[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) {
    const double cf = (t <= clip_c2) ? 1.0 : clip_c / sqrt(t);  // dpcore.py:41-47
    scale_out[0] = static_cast<float>(cf) * inv_batch;
    if (norms_out) norms_out[0] = static_cast<float>(t);
  }
}

cudaError_t single_sample_factor(const FinJob& j, float* scale_out, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_single_factor, static_cast<const float*>(j.part), j.n_parts, j.clip_c, j.clip_c2,
                            j.inv_batch, j.norms_out, scale_out);
}

cudaError_t single_sample_finalize(const FinJob& j, cudaStream_t s) {
  return single_sample_finalize(j.g, j.n, j.part, j.n_parts, j.clip_c, j.clip_c2, j.inv_batch, j.norms_out,
                                j.add_noise, j.impl, j.scale, j.base, j.base_g, j.step_ptr, j.seed_u, j.layer_u, j.lo,
                                j.hi, s);
}

cudaError_t simt_partial_norms(const SimtParams& p, cudaStream_t s) {
  k_partial_norms<<<dim3(p.n_pt, p.n_dt, p.B), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t reduce_norms_to_factors(const float* part, int B, int n_tiles, double clip_c, double clip_c2,
                                    float inv_batch, float* norms_out, float* factors, cudaStream_t s, bool pdl) {
  const int warps_per_block = 4;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((B + warps_per_block - 1) / warps_per_block);
  cfg.blockDim = dim3(32 * warps_per_block);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_reduce_norms, part, B, n_tiles, clip_c, clip_c2, inv_batch, norms_out, factors);
}

cudaError_t simt_weighted_sum(const SimtParams& p, cudaStream_t s) {
  k_weighted_sum<<<dim3(p.n_pt, p.n_dt), 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t explicit_store_g_simt(const SimtParams& p, float* g, cudaStream_t s) {
  k_store_g<<<dim3(p.n_pt, p.n_dt, p.B), 256, 0, s>>>(p, g);
  return cudaGetLastError();
}

cudaError_t explicit_norms(const float* g, int B, long long DP, float* part, int nchunks, cudaStream_t s) {
  k_explicit_norms<<<dim3(nchunks, B), 256, 0, s>>>(g, DP, nchunks, part);
  return cudaGetLastError();
}

cudaError_t explicit_clip(const float* g, float* gp, const float* factors, int B, long long DP, cudaStream_t s) {
  k_explicit_clip<<<grid_for(static_cast<long long>(B) * DP, 256), 256, 0, s>>>(g, gp, factors, B, DP);
  return cudaGetLastError();
}

cudaError_t explicit_sum_finalize(const float* gp, int B, long long DP, int /*P*/, const SimtParams& p,
                                  cudaStream_t s) {
  k_explicit_sum<<<grid_for(DP, 256), 256, 0, s>>>(gp, B, DP, p);
  return cudaGetLastError();
}

cudaError_t noise_fill(float* out, long long lo, long long hi, double scale, int impl, uint64_t base,
                       uint64_t base_g, cudaStream_t s) {
  if (hi <= lo) return cudaSuccess;
  k_noise_fill<<<grid_for(hi - lo, 256), 256, 0, s>>>(out, lo, hi, static_cast<float>(scale), impl, base, base_g);
  return cudaGetLastError();
}

cudaError_t noise_fill64(double* out, long long lo, long long hi, double scale, int impl, uint64_t base,
                         uint64_t base_g, cudaStream_t s) {
  if (hi <= lo) return cudaSuccess;
  k_noise_fill64<<<grid_for(hi - lo, 256), 256, 0, s>>>(out, lo, hi, scale, impl, base, base_g);
  return cudaGetLastError();
}

}  // namespace fdp
