// fdp_params.cu -- DP gradients of the non-linear parameter groups of a model
// (SURVEY 8f rank 3): bias / RMSNorm / LayerNorm vectors and embedding tables,
// each clipped per sample as its own per-layer group and finalized with the
// reference's arithmetic (clip factor dpcore.py:41-47, sum or mean + sigma*C*N
// dpcore.py:60-73, keyed noise rng.py:69-85 on the group's own index space).
// The reference clips linear weights only; these are the textbook
// per-sample gradients, pinned to oracle/dp_oracle.py's restatements.
//
// Vector groups (length L = D, or 2 D for LayerNorm's [gamma, beta]): per-sample
// g_b = sum_t dY (bias, beta), sum_t dY * xhat (gamma). Aligned rows: one CTA per
// (sample, 32-byte column slice) sums all T rows (k_vec_cols) with the slice's norm^2
// partial, then the clip / sum / noise pass (k_vec_finalize, PDL dependent). Unaligned
// rows: three deterministic passes -- row-chunk partial sums, a fixed-order sum of the
// chunks with per-block norm^2 partials, the same finalize. All HBM-bound on reading dY
// (and xhat) once.
//
// Embedding (V x d table, tokens (B, T)): the per-sample gradient is a scatter of
// dY rows onto the rows of the sample's tokens, so ||G_b||^2 is the token-
// equality Gram sum_{t,s: tok_t = tok_s} <dY_t, dY_s>. Each sample's (token,
// position) keys are sorted once in shared memory; the norm pass sums dY rows per
// run of equal tokens (never materialising G_b); a streaming pass writes every
// row's noise, and the add pass walks all samples' sorted runs per vocabulary row
// in fixed order onto the touched rows -- deterministic, no atomics.
#include <algorithm>
#include <cstdlib>

#include "../../include/fdp.h"
#include "fdp_internal.h"
#include "fdp_ptx.cuh"
#include "fdp_rng.cuh"
#include <cuda_bf16.h>

namespace fdp {
namespace {

constexpr int kVCols = 256;  // columns per block
constexpr int kVRows = 32;   // T rows per partial-sum block

__device__ __forceinline__ void nk_resolve(NoiseKey& nk) {  // device step counter (graph replays)
  if (nk.step_ptr) {
    nk.base = absorb3(nk.seed_u, nk.layer_u, static_cast<uint64_t>(*nk.step_ptr));
    nk.base_g = nk.base + kGamma;
  }
}
__device__ __forceinline__ float nk_draw(const NoiseKey& nk, uint64_t i) {
  return noise_draw(nk.impl, nk.base_g, nk.base, i);
}

template <typename T>
__device__ __forceinline__ float ld(const T* p, long long i) {
  if constexpr (sizeof(T) == 4) return __ldg(reinterpret_cast<const float*>(p) + i);
  else return __bfloat162float(p[i]);
}

// pass 1: gpart[b][tc][l] = sum over rows [tc*kVRows, ...) of the group's per-row term.
// VW consecutive columns per thread (16-byte loads when D % VW == 0, else VW = 1),
// all kVRows rows' loads issued before the sums: the pass is latency-bound on a
// few tens of MB, so bytes in flight per SM decide its speed.
template <typename T, int kKind, int VW>
__global__ void __launch_bounds__(kVCols) k_vec_rows(const T* __restrict__ dy, const T* __restrict__ xh, int T_, int D,
                                                     int n_tc, float* __restrict__ gpart) {
  if (threadIdx.x == 0) pdl_launch_dependents();  // the reduce may queue up behind this pass
  const int b = blockIdx.z, tc = blockIdx.y;
  const int d = (blockIdx.x * kVCols + threadIdx.x) * VW;
  if (d >= D) return;
  const int t0 = tc * kVRows, t1 = min(T_, t0 + kVRows);
  float s[VW], sx[VW];
#pragma unroll
  for (int j = 0; j < VW; ++j) s[j] = sx[j] = 0.0f;
  const long long base = static_cast<long long>(b) * T_ * D + d;
#pragma unroll 8
  for (int t = t0; t < t1; ++t) {
    const long long i = base + static_cast<long long>(t) * D;
    float y[VW], x[VW];
    if constexpr (VW == 1) {
      y[0] = ld(dy, i);
      if constexpr (kKind != FDP_VEC_BIAS) x[0] = ld(xh, i);
    } else if constexpr (sizeof(T) == 4) {  // VW = 4 floats
      const float4 a = __ldcs(reinterpret_cast<const float4*>(dy + i));
      y[0] = a.x; y[1] = a.y; y[2] = a.z; y[3] = a.w;
      if constexpr (kKind != FDP_VEC_BIAS) {
        const float4 c = __ldcs(reinterpret_cast<const float4*>(xh + i));
        x[0] = c.x; x[1] = c.y; x[2] = c.z; x[3] = c.w;
      }
    } else {  // VW = 8 bf16
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(dy + i));
      const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(pa[j]);
        y[2 * j] = f.x;
        y[2 * j + 1] = f.y;
      }
      if constexpr (kKind != FDP_VEC_BIAS) {
        const uint4 c = __ldcs(reinterpret_cast<const uint4*>(xh + i));
        const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(pc[j]);
          x[2 * j] = f.x;
          x[2 * j + 1] = f.y;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      if constexpr (kKind != FDP_VEC_RMSNORM) s[j] += y[j];
      if constexpr (kKind != FDP_VEC_BIAS) sx[j] = fmaf(y[j], x[j], sx[j]);
    }
  }
  const long long L = kKind == FDP_VEC_LAYERNORM ? 2LL * D : D;
  float* o = gpart + (static_cast<long long>(b) * n_tc + tc) * L;
#pragma unroll
  for (int j = 0; j < VW; ++j) {
    if constexpr (kKind == FDP_VEC_BIAS) o[d + j] = s[j];
    if constexpr (kKind == FDP_VEC_RMSNORM) o[d + j] = sx[j];
    if constexpr (kKind == FDP_VEC_LAYERNORM) {
      o[d + j] = sx[j];
      o[D + d + j] = s[j];
    }
  }
}

// pass 2: g[b][l] = sum_tc gpart[b][tc][l] (fixed order), part[b][chunk] = sum over the block of g^2
__global__ void __launch_bounds__(kVCols) k_vec_reduce(const float* __restrict__ gpart, int n_tc, int L,
                                                       float* __restrict__ g, float* __restrict__ part, int n_chunks) {
  if (threadIdx.x == 0) pdl_launch_dependents();
  pdl_wait();  // PDL launch: the row partials are complete
  const int b = blockIdx.y, chunk = blockIdx.x;
  const int l = chunk * kVCols + threadIdx.x;
  float s = 0.0f;
  if (l < L) {
    const float* p = gpart + static_cast<long long>(b) * n_tc * L + l;
    for (int tc = 0; tc < n_tc; ++tc) s += p[static_cast<long long>(tc) * L];
    g[static_cast<long long>(b) * L + l] = s;
  }
  __shared__ float red[kVCols / 32];
  float sq = s * s;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int w = 0; w < kVCols / 32; ++w) t += red[w];
    part[static_cast<long long>(b) * n_chunks + chunk] = t;
  }
}

// pass 3: out[l] (+)= sum_b c_b g[b][l] / batch + sigma C N(l) on [lo, hi)
__global__ void __launch_bounds__(256) k_vec_finalize(const float* __restrict__ g, const float* __restrict__ part,
                                                      int B, long long L, int n_chunks, double clip_c, double clip_c2,
                                                      float inv_batch, float* out, float* norms_out, int accumulate,
                                                      NoiseKey nk) {
  extern __shared__ float fac[];  // [B] clip factor x mean scale
  pdl_wait();  // PDL launch: g and the norm partials are complete
  // one warp per sample: lane-strided fp64 partial sums, then a fixed butterfly
  for (int b = threadIdx.x >> 5; b < B; b += blockDim.x >> 5) {
    double s = 0.0;
    for (int c = threadIdx.x & 31; c < n_chunks; c += 32)
      s += static_cast<double>(part[static_cast<long long>(b) * n_chunks + c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) {
      const double cf = (s <= clip_c2) ? 1.0 : clip_c / sqrt(s);  // dpcore.py:41-47
      fac[b] = static_cast<float>(cf) * inv_batch;
      if (blockIdx.x == 0 && norms_out) norms_out[b] = static_cast<float>(s);
    }
  }
  __syncthreads();
  nk_resolve(nk);
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < L;
       l += static_cast<long long>(gridDim.x) * blockDim.x) {
    float v = 0.0f;
    for (int b = 0; b < B; ++b) v = fmaf(fac[b], g[static_cast<long long>(b) * L + l], v);
    if (nk.add_noise && l >= nk.lo && l < nk.hi) v += nk.scale * nk_draw(nk, static_cast<uint64_t>(l));
    if (accumulate) v += out[l];
    out[l] = v;
  }
}

// ---- two-launch vector group: every CTA owns a column slice (kTPR x 16 bytes) of one
// sample over ALL T rows, so the per-sample sum needs no cross-CTA pass. 256 threads =
// 256/kTPR row lanes x kTPR 16-byte loads per row; each row lane sums its rows
// (t = lane, lane + 256/kTPR, ...), a fixed butterfly over the row lanes of a warp and a
// fixed-order sum over the 8 warps give g[b][slice] and the slice's norm^2 partial
// part[b][cb]; k_vec_finalize (PDL dependent) then clips, sums and adds noise. One HBM
// read of dY (and xhat), two launches instead of three and no row-chunk partials.
template <typename T, int kKind, int kTPR>
__global__ void __launch_bounds__(256) k_vec_cols(const T* __restrict__ dy, const T* __restrict__ xh, int T_, int D,
                                                  int n_cb, float* __restrict__ g, float* __restrict__ part) {
  constexpr int VW = 16 / sizeof(T);  // columns per thread
  constexpr int CW = kTPR * VW;       // columns per CTA (kTPR x 16 bytes)
  constexpr int kLanes = 256 / kTPR;  // row lanes
  constexpr int kH = kKind == FDP_VEC_LAYERNORM ? 2 : 1;
  __shared__ float red[8][kH][CW];
  __shared__ float wsq[kH * CW];
  if (threadIdx.x == 0) pdl_launch_dependents();
  const int half = threadIdx.x % kTPR, row = threadIdx.x / kTPR, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cb = blockIdx.x, b = blockIdx.y;
  const int d = cb * CW + half * VW;
  const long long L = static_cast<long long>(kH) * D;
  float s[VW], sx[VW];
#pragma unroll
  for (int j = 0; j < VW; ++j) s[j] = sx[j] = 0.0f;
  if (d < D) {
    const T* py = dy + static_cast<long long>(b) * T_ * D + d;
    const T* px = xh + static_cast<long long>(b) * T_ * D + d;
#pragma unroll 8
    for (int t = row; t < T_; t += kLanes) {
      const long long i = static_cast<long long>(t) * D;
      float y[VW], x[VW];
      if constexpr (sizeof(T) == 4) {
        const float4 a = __ldcs(reinterpret_cast<const float4*>(py + i));
        y[0] = a.x; y[1] = a.y; y[2] = a.z; y[3] = a.w;
        if constexpr (kKind != FDP_VEC_BIAS) {
          const float4 c = __ldcs(reinterpret_cast<const float4*>(px + i));
          x[0] = c.x; x[1] = c.y; x[2] = c.z; x[3] = c.w;
        }
      } else {
        const uint4 a = __ldcs(reinterpret_cast<const uint4*>(py + i));
        const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(pa[j]);
          y[2 * j] = f.x;
          y[2 * j + 1] = f.y;
        }
        if constexpr (kKind != FDP_VEC_BIAS) {
          const uint4 c = __ldcs(reinterpret_cast<const uint4*>(px + i));
          const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(pc[j]);
            x[2 * j] = f.x;
            x[2 * j + 1] = f.y;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        if constexpr (kKind != FDP_VEC_RMSNORM) s[j] += y[j];
        if constexpr (kKind != FDP_VEC_BIAS) sx[j] = fmaf(y[j], x[j], sx[j]);
      }
    }
  }
  // sum the row lanes of the warp (lanes equal mod kTPR), fixed butterfly
#pragma unroll
  for (int o = kTPR; o < 32; o <<= 1) {
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
      sx[j] += __shfl_xor_sync(0xffffffffu, sx[j], o);
    }
  }
  if (lane < kTPR) {
#pragma unroll
    for (int j = 0; j < VW; ++j) {  // half 0 = the xhat term (gamma / RMSNorm weight) or the bias sum
      red[warp][0][half * VW + j] = kKind == FDP_VEC_BIAS ? s[j] : sx[j];
      if constexpr (kH == 2) red[warp][1][half * VW + j] = s[j];
    }
  }
  __syncthreads();
  if (threadIdx.x < kH * CW) {
    const int h = threadIdx.x / CW, c = threadIdx.x % CW;
    float v = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][h][c];
    const bool in = cb * CW + c < D;
    if (in) g[static_cast<long long>(b) * L + static_cast<long long>(h) * D + cb * CW + c] = v;
    wsq[threadIdx.x] = in ? v * v : 0.0f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
#pragma unroll
    for (int c = 0; c < kH * CW; ++c) t += wsq[c];
    part[static_cast<long long>(b) * n_cb + cb] = t;
  }
}

// ---- embedding
constexpr uint64_t kNoKey = ~0ull;
constexpr int kESeg = 64;     // sorted positions per norm block
constexpr int kEVRows = 32;   // vocabulary rows per output block
constexpr int kECols = 1024;  // columns per output block (4 per thread)

__global__ void __launch_bounds__(1024) k_emb_sort(const long long* __restrict__ tok, int T_, long long V, int n2,
                                                   uint64_t* __restrict__ keys) {
  extern __shared__ uint64_t sk[];  // [n2]
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    uint64_t k = kNoKey;
    if (i < T_) {
      const long long v = tok[static_cast<long long>(b) * T_ + i];
      if (v >= 0 && v < V) k = (static_cast<uint64_t>(v) << 32) | static_cast<uint32_t>(i);
    }
    sk[i] = k;
  }
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {  // bitonic sort, ascending
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a = sk[lo], c = sk[hi];
        if ((a > c) == up) {
          sk[lo] = c;
          sk[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < T_; i += blockDim.x) keys[static_cast<long long>(b) * T_ + i] = sk[i];
}

// norm^2 partial of sample b over the runs of equal tokens that START in sorted
// positions [sc*kESeg, (sc+1)*kESeg), columns [dc*kVCols, ...). The block's keys
// (plus the tail of its last run) are staged in shared memory first, so the dY
// row loads of the run sums are independent and pipeline.
constexpr int kEStage = 4 * kESeg;  // staged keys: own positions + the spill of the last run
template <typename T>
__global__ void __launch_bounds__(kVCols) k_emb_norms(const uint64_t* __restrict__ keys, const T* __restrict__ dy,
                                                      int T_, int D, int n_sc, int n_dc, float* __restrict__ part) {
  const int dc = blockIdx.x, sc = blockIdx.y, b = blockIdx.z;
  const int col = dc * kVCols + threadIdx.x;
  const uint64_t* K = keys + static_cast<long long>(b) * T_;
  __shared__ uint64_t sk[kEStage + 1];
  __shared__ int s_range[2];
  __shared__ float red[kVCols / 32];
  const int k0 = sc * kESeg, k1 = min(T_, k0 + kESeg);
  if (threadIdx.x == 0) {
    int k = k0;
    if (k > 0) {  // skip the continuation of a run owned by the previous block
      const uint64_t prev = K[k - 1] >> 32;
      while (k < k1 && K[k] != kNoKey && (K[k] >> 32) == prev) ++k;
    }
    int e = k1;  // finish the last run this block starts
    if (e > k && e < T_ && K[e - 1] != kNoKey) {
      const uint64_t last = K[e - 1] >> 32;
      while (e < T_ && K[e] != kNoKey && (K[e] >> 32) == last) ++e;
    }
    while (e > k && K[e - 1] == kNoKey) --e;  // invalid tokens sort last: never summed
    s_range[0] = k;
    s_range[1] = e;
  }
  __syncthreads();
  const int kb = s_range[0], ke = s_range[1];
  float sq = 0.0f;
  const long long rbase = static_cast<long long>(b) * T_ * D + col;
  for (int c0 = kb; c0 < ke; c0 += kEStage) {  // usually one stage
    const int c1 = min(ke, c0 + kEStage);
    for (int i = threadIdx.x; i <= c1 - c0; i += blockDim.x)
      sk[i] = (c0 + i < ke) ? K[c0 + i] : kNoKey;  // sk[c1 - c0]: sentinel closing the last run
    __syncthreads();
    // sk[c1 - c0] is the next key (or kNoKey at the end): a token change closes a run
    const int n = c1 - c0;
    float acc = 0.0f;
    if (col < D) {
#pragma unroll 8
      for (int k = 0; k < n; ++k) {
        acc += ld(dy, rbase + static_cast<long long>(sk[k] & 0xffffffffull) * D);
        if ((sk[k + 1] >> 32) != (sk[k] >> 32)) {
          sq = fmaf(acc, acc, sq);
          acc = 0.0f;
        }
      }
    }
    const bool open = c1 < ke && (sk[n] >> 32) == (sk[n - 1] >> 32);
    if (open && col < D) {  // a run longer than the stage: finish it from global memory
      const uint64_t tk = sk[n - 1] >> 32;
      for (int k = c1; k < ke && (K[k] >> 32) == tk; ++k)
        acc += ld(dy, rbase + static_cast<long long>(K[k] & 0xffffffffull) * D);
      sq = fmaf(acc, acc, sq);
    }
    __syncthreads();
    if (c1 < ke) {  // resume after the run that crossed the boundary
      int k = c1;
      const uint64_t tk = K[c1 - 1] >> 32;
      while (k < ke && (K[k] >> 32) == tk) ++k;
      c0 = k - kEStage;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int w = 0; w < kVCols / 32; ++w) t += red[w];
    part[(static_cast<long long>(b) * n_sc + sc) * n_dc + dc] = t;
  }
}

// The table's base: out = (accumulate ? out : 0) + sigma C N(flat index) on [lo, hi),
// a streaming pass over every row (untouched rows get their noise only). kMode 1:
// Philox over the whole table (one draw call per float4), 0: any generator with
// per-element range checks, 2: no noise (zero fill; nothing to do when accumulating).
template <int kMode>
__global__ void __launch_bounds__(256, 6) k_emb_fill(float* __restrict__ out, long long n, int accumulate,
                                                     NoiseKey nk) {
  nk_resolve(nk);
  const long long n4 = n >> 2;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  float4* o4 = reinterpret_cast<float4*>(out);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (kMode == 1) {
      z = philox_normal4(nk.base, static_cast<uint64_t>(i));
    } else if constexpr (kMode == 0) {
      const long long e = i << 2;
      if (e + 3 >= nk.lo && e < nk.hi) {
        const float4 q = noise_draw4(nk.impl, nk.base_g, nk.base, static_cast<uint64_t>(i));
        z.x = (e + 0 >= nk.lo && e + 0 < nk.hi) ? q.x : 0.f;
        z.y = (e + 1 >= nk.lo && e + 1 < nk.hi) ? q.y : 0.f;
        z.z = (e + 2 >= nk.lo && e + 2 < nk.hi) ? q.z : 0.f;
        z.w = (e + 3 >= nk.lo && e + 3 < nk.hi) ? q.w : 0.f;
      }
    }
    float4 v = make_float4(nk.scale * z.x, nk.scale * z.y, nk.scale * z.z, nk.scale * z.w);
    if (kMode == 2) v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (accumulate) {
      const float4 p = __ldcs(o4 + i);
      v.x += p.x;
      v.y += p.y;
      v.z += p.z;
      v.w += p.w;
    }
    __stcs(o4 + i, v);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {  // tail of a table whose size is not a multiple of 4
    const long long e = (n4 << 2) + threadIdx.x;
    float v = (kMode != 2 && e >= nk.lo && e < nk.hi) ? nk.scale * nk_draw(nk, static_cast<uint64_t>(e)) : 0.f;
    if (accumulate) v += out[e];
    out[e] = v;
  }
}

// out[v][c] += sum_b c_b sum_{t: tok_bt = v} dY[b,t,c] for the rows some sample
// touches (after k_emb_fill). One pre-pass per block finds each sample's sorted
// range of every row of the block's kEVRows vocabulary rows (one barrier); the
// row loop then runs barrier-free over the touched rows, samples in fixed order.
template <typename T>
__global__ void __launch_bounds__(256) k_emb_add(const uint64_t* __restrict__ keys, const T* __restrict__ dy,
                                                 const float* __restrict__ factors, int B, int T_, long long V, int D,
                                                 float* out) {
  extern __shared__ int sm[];  // bound[B][kEVRows + 1]; fac[B]; touched[kEVRows]
  int* bound = sm;
  float* fac = reinterpret_cast<float*>(sm + B * (kEVRows + 1));
  int* touched = reinterpret_cast<int*>(fac + B);
  const long long v0 = static_cast<long long>(blockIdx.x) * kEVRows;
  const int nrows = static_cast<int>(min(static_cast<long long>(kEVRows), V - v0));
  for (int r = threadIdx.x; r < kEVRows; r += blockDim.x) touched[r] = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const uint64_t* K = keys + static_cast<long long>(b) * T_;
    const uint64_t want = static_cast<uint64_t>(v0) << 32;
    int lo = 0, hi = T_;  // first sorted position with token >= v0
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (K[mid] < want) lo = mid + 1;
      else hi = mid;
    }
    int* bd = bound + b * (kEVRows + 1);
    int e = lo;
    for (int r = 0; r < nrows; ++r) {  // bd[r] .. bd[r+1]: the sample's positions of row v0 + r
      bd[r] = e;
      while (e < T_ && K[e] != kNoKey && static_cast<long long>(K[e] >> 32) == v0 + r) ++e;
      if (e > bd[r]) touched[r] = 1;
    }
    bd[nrows] = e;
    fac[b] = factors[b];
  }
  __syncthreads();
  const bool vec = (D & 3) == 0;
  for (int c0 = blockIdx.y * kECols + 4 * threadIdx.x; c0 < D && c0 < (blockIdx.y + 1) * kECols; c0 += 4 * 256) {
    for (int r = 0; r < nrows; ++r) {
      if (!touched[r]) continue;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int b = 0; b < B; ++b) {
        const int* bd = bound + b * (kEVRows + 1);
        const uint64_t* K = keys + static_cast<long long>(b) * T_;
        for (int k = bd[r]; k < bd[r + 1]; ++k) {
          const long long row = (static_cast<long long>(b) * T_ + static_cast<long long>(K[k] & 0xffffffffull)) * D;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (c0 + j < D) acc[j] = fmaf(fac[b], ld(dy, row + c0 + j), acc[j]);
        }
      }
      const long long f0 = (v0 + r) * D + c0;
      if (vec) {
        float4* po = reinterpret_cast<float4*>(out + f0);
        float4 o = *po;
        o.x += acc[0];
        o.y += acc[1];
        o.z += acc[2];
        o.w += acc[3];
        *po = o;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c0 + j < D) out[f0 + j] += acc[j];
      }
    }
  }
}

size_t emb_out_smem(int B) { return sizeof(int) * (static_cast<size_t>(B) * (kEVRows + 2) + kEVRows + 4); }
long long n_tchunks(int T_) { return (T_ + kVRows - 1) / kVRows; }
int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace

size_t vec_dp_work_bytes(int kind, int B, int T_, int D) {
  // three-pass layout [gpart | g | part(L/256)]; the column-slice schedule's [g | part(<= D/8)]
  // fits inside it (gpart alone holds at least B L floats)
  const long long L = kind == FDP_VEC_LAYERNORM ? 2LL * D : D;
  const long long n_chunks = (L + kVCols - 1) / kVCols;
  return sizeof(float) * static_cast<size_t>(B * n_tchunks(T_) * L + B * L + B * n_chunks);
}

cudaError_t vec_dp(int kind, const void* dy, const void* xhat, int in_f32, int B, int T_, int D, float* work,
                   double clip_c, float inv_batch, float* out, float* norms_out, int accumulate, const NoiseKey& nk,
                   cudaStream_t s) {
  const long long L = kind == FDP_VEC_LAYERNORM ? 2LL * D : D;
  // 16-byte loads when every row start stays aligned (D a multiple of the vector width)
  const bool aligned = (reinterpret_cast<uintptr_t>(dy) % 16 == 0) && (reinterpret_cast<uintptr_t>(xhat) % 16 == 0);
  const int vw = !aligned ? 1 : in_f32 ? ((D % 4 == 0) ? 4 : 1) : ((D % 8 == 0) ? 8 : 1);
  // column-slice schedule whenever the rows take 16-byte loads (FDP_VEC_COLS=0: three passes)
  const char* cv = std::getenv("FDP_VEC_COLS");
  const bool cols = vw > 1 && !(cv && std::atoi(cv) == 0);
  float *g, *part;
  int n_chunks;
  cudaError_t e;
  if (cols) {
    // widest slice (longer contiguous row segments) that still gives two CTAs per SM
    int tpr = 8;
    while (tpr > 2 && static_cast<long long>((D + tpr * vw - 1) / (tpr * vw)) * B < 2 * 148) tpr >>= 1;
    const int cw = tpr * vw;
    n_chunks = (D + cw - 1) / cw;
    g = work;                                   // [B][L]
    part = g + static_cast<long long>(B) * L;   // [B][n_chunks]
    const dim3 grid(n_chunks, B);
#define FDP_VEC_C(TY, K, P) \
  k_vec_cols<TY, K, P><<<grid, 256, 0, s>>>(static_cast<const TY*>(dy), static_cast<const TY*>(xhat), T_, D, n_chunks, g, part)
#define FDP_VEC_CP(TY, K)                       \
  do {                                          \
    if (tpr == 8) FDP_VEC_C(TY, K, 8);          \
    else if (tpr == 4) FDP_VEC_C(TY, K, 4);     \
    else FDP_VEC_C(TY, K, 2);                   \
  } while (0)
#define FDP_VEC_CK(TY)                                               \
  do {                                                               \
    if (kind == FDP_VEC_BIAS) FDP_VEC_CP(TY, FDP_VEC_BIAS);           \
    else if (kind == FDP_VEC_RMSNORM) FDP_VEC_CP(TY, FDP_VEC_RMSNORM); \
    else FDP_VEC_CP(TY, FDP_VEC_LAYERNORM);                           \
  } while (0)
    if (in_f32) FDP_VEC_CK(float);
    else FDP_VEC_CK(__nv_bfloat16);
#undef FDP_VEC_CK
#undef FDP_VEC_CP
#undef FDP_VEC_C
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // the reduce and the finalize are programmatic dependents of the pass before them: their
  // launch latency hides under it (FDP_PDL=0 turns it off)
  const char* pv = std::getenv("FDP_PDL");
  const bool pdl = !pv || std::atoi(pv) != 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t c2{};
  c2.stream = s;
  c2.attrs = attr;
  c2.numAttrs = pdl ? 1 : 0;
  if (!cols) {
    const int n_tc = static_cast<int>(n_tchunks(T_));
    n_chunks = static_cast<int>((L + kVCols - 1) / kVCols);
    float* gpart = work;                                    // [B][n_tc][L]
    g = gpart + static_cast<long long>(B) * n_tc * L;       // [B][L]
    part = g + static_cast<long long>(B) * L;               // [B][n_chunks]
    const dim3 g1((D / vw + kVCols - 1) / kVCols, n_tc, B);
#define FDP_VEC_ROWS(TY, K, V) \
  k_vec_rows<TY, K, V><<<g1, kVCols, 0, s>>>(static_cast<const TY*>(dy), static_cast<const TY*>(xhat), T_, D, n_tc, gpart)
#define FDP_VEC_KINDS(TY, V)                                        \
  do {                                                              \
    if (kind == FDP_VEC_BIAS) FDP_VEC_ROWS(TY, FDP_VEC_BIAS, V);    \
    else if (kind == FDP_VEC_RMSNORM) FDP_VEC_ROWS(TY, FDP_VEC_RMSNORM, V); \
    else FDP_VEC_ROWS(TY, FDP_VEC_LAYERNORM, V);                    \
  } while (0)
    if (in_f32) {
      if (vw == 4) FDP_VEC_KINDS(float, 4);
      else FDP_VEC_KINDS(float, 1);
    } else {
      if (vw == 8) FDP_VEC_KINDS(__nv_bfloat16, 8);
      else FDP_VEC_KINDS(__nv_bfloat16, 1);
    }
#undef FDP_VEC_KINDS
#undef FDP_VEC_ROWS
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    c2.gridDim = dim3(n_chunks, B);
    c2.blockDim = dim3(kVCols);
    if ((e = cudaLaunchKernelEx(&c2, k_vec_reduce, static_cast<const float*>(gpart), n_tc, static_cast<int>(L), g, part,
                                n_chunks)) != cudaSuccess)
      return e;
  }
  const long long blocks = (L + 255) / 256 < 148 ? (L + 255) / 256 : 148;
  // factor table rounded up to whole 16-byte words: the unrolled sample loop may read fac[] in vectors
  cudaLaunchConfig_t c3 = c2;
  c3.gridDim = dim3(static_cast<unsigned>(blocks));
  c3.blockDim = dim3(256);
  c3.dynamicSmemBytes = static_cast<size_t>((B + 3) / 4) * 16;
  return cudaLaunchKernelEx(&c3, k_vec_finalize, static_cast<const float*>(g), static_cast<const float*>(part), B, L,
                            n_chunks, clip_c, clip_c * clip_c, inv_batch, out, norms_out, accumulate, nk);
}

size_t emb_dp_work_bytes(int B, int T_, int D) {
  const long long n_sc = (T_ + kESeg - 1) / kESeg, n_dc = (D + kVCols - 1) / kVCols;
  return sizeof(uint64_t) * static_cast<size_t>(B) * T_ + sizeof(float) * static_cast<size_t>(B * n_sc * n_dc + B);
}

int emb_max_tokens() { return 16384; }
int emb_max_batch() { return 1024; }

cudaError_t emb_dp(const long long* tokens, const void* dy, int in_f32, int B, int T_, long long V, int D, void* work,
                   double clip_c, float inv_batch, float* out, float* norms_out, int accumulate, const NoiseKey& nk,
                   cudaStream_t s) {
  uint64_t* keys = static_cast<uint64_t*>(work);  // [B][T]
  const int n_sc = (T_ + kESeg - 1) / kESeg, n_dc = (D + kVCols - 1) / kVCols;
  float* part = reinterpret_cast<float*>(keys + static_cast<long long>(B) * T_);  // [B][n_sc][n_dc]
  float* fac = part + static_cast<long long>(B) * n_sc * n_dc;                     // [B]
  const int n2 = pow2_at_least(T_);
  const size_t sort_smem = sizeof(uint64_t) * n2;
  // function attributes are per device: track them per device ordinal
  static bool attr_done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 63;
  if (!attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_emb_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(uint64_t) * emb_max_tokens()));
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  k_emb_sort<<<B, 1024, sort_smem, s>>>(tokens, T_, V, n2, keys);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (in_f32)
    k_emb_norms<float><<<dim3(n_dc, n_sc, B), kVCols, 0, s>>>(keys, static_cast<const float*>(dy), T_, D, n_sc, n_dc,
                                                             part);
  else
    k_emb_norms<__nv_bfloat16><<<dim3(n_dc, n_sc, B), kVCols, 0, s>>>(
        keys, static_cast<const __nv_bfloat16*>(dy), T_, D, n_sc, n_dc, part);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = reduce_norms_to_factors(part, B, n_sc * n_dc, clip_c, clip_c * clip_c, inv_batch, norms_out, fac, s)) !=
      cudaSuccess)
    return e;
  // base pass over the whole table: the noise (or zeros / the old values)
  const long long n = V * static_cast<long long>(D);
  const int fmode = !nk.add_noise || nk.hi <= nk.lo ? 2 : (nk.impl == 2 && nk.lo <= 0 && nk.hi >= n) ? 1 : 0;
  if (!(fmode == 2 && accumulate)) {
    long long blocks = (n / 4 + 255) / 256;
    if (blocks > 148LL * 6 * 4) blocks = 148LL * 6 * 4;
    if (blocks < 1) blocks = 1;
    auto kf = fmode == 1 ? k_emb_fill<1> : fmode == 0 ? k_emb_fill<0> : k_emb_fill<2>;
    kf<<<static_cast<int>(blocks), 256, 0, s>>>(out, n, accumulate, nk);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // the clipped sums onto the touched rows
  const dim3 g3(static_cast<unsigned>((V + kEVRows - 1) / kEVRows), (D + kECols - 1) / kECols);
  const size_t smem = emb_out_smem(B);
  static bool out_attr[64] = {};
  if (!out_attr[dev]) {
    if ((e = cudaFuncSetAttribute(k_emb_add<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(emb_out_smem(emb_max_batch())))) != cudaSuccess ||
        (e = cudaFuncSetAttribute(k_emb_add<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(emb_out_smem(emb_max_batch())))) != cudaSuccess)
      return e;
    out_attr[dev] = true;
  }
  if (in_f32)
    k_emb_add<float><<<g3, 256, smem, s>>>(keys, static_cast<const float*>(dy), fac, B, T_, V, D, out);
  else
    k_emb_add<__nv_bfloat16><<<g3, 256, smem, s>>>(keys, static_cast<const __nv_bfloat16*>(dy), fac, B, T_, V, D,
                                                   out);
  return cudaGetLastError();
}

}  // namespace fdp
