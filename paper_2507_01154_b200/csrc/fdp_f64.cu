// fdp_f64.cu -- the fp64 parity path: the reference computes in float64
// throughout (workflows.py, numpy); with in_dtype = FDP_DTYPE_F64 the drop-in
// boundary takes float64 X / dY and returns float64 grad_w / norms_sq, computed
// with fp64 FMA on the CUDA cores and the reference's keyed noise transformed in
// fp64 (rng.py:69-85), so the reference's own acceptance streams can be checked
// at its 1e-12 bar through the C ABI. Throughput is not the point of this path.
//
// Two passes like backward_implicit (workflows.py:246-324): pass 1 reduces
// per-sample ||G_b||^2 partials per 32x32 tile of G without storing it, a fixed-
// order reduce forms the clip factors (dpcore.py:41-47), pass 2 recomputes the
// tiles and sums c_b G_b, then finalize (mean, noise; dpcore.py:60-73).
#include "fdp_internal.h"
#include "fdp_rng.cuh"

namespace fdp {

namespace {

constexpr int kTS = 32;

__device__ __forceinline__ void tile64(const F64Params& p, int b, int d0, int p0, double (&g)[2][2],
                                       double (*sy)[kTS + 1], double (*sx)[kTS + 1]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  g[0][0] = g[0][1] = g[1][0] = g[1][1] = 0.0;
  const long long ybase = static_cast<long long>(b) * p.T * p.D;
  const long long xbase = static_cast<long long>(b) * p.T * p.P;
  for (int t0 = 0; t0 < p.T; t0 += kTS) {
    for (int e = threadIdx.x; e < kTS * kTS; e += blockDim.x) {
      const int tt = e / kTS, cc = e % kTS;
      const int t = t0 + tt, dd = d0 + cc, pp = p0 + cc;
      sy[tt][cc] = (t < p.T && dd < p.D) ? p.dy[ybase + static_cast<long long>(t) * p.D + dd] : 0.0;
      sx[tt][cc] = (t < p.T && pp < p.P) ? p.x[xbase + static_cast<long long>(t) * p.P + pp] : 0.0;
    }
    __syncthreads();
    for (int tt = 0; tt < kTS; ++tt) {
      const double y0 = sy[tt][2 * ty], y1 = sy[tt][2 * ty + 1];
      const double x0 = sx[tt][2 * tx], x1 = sx[tt][2 * tx + 1];
      g[0][0] = fma(y0, x0, g[0][0]);
      g[0][1] = fma(y0, x1, g[0][1]);
      g[1][0] = fma(y1, x0, g[1][0]);
      g[1][1] = fma(y1, x1, g[1][1]);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k64_partial_norms(const F64Params p) {
  __shared__ double sy[kTS][kTS + 1];
  __shared__ double sx[kTS][kTS + 1];
  __shared__ double red[8];
  const int pt = blockIdx.x, dt = blockIdx.y, b = blockIdx.z;
  double g[2][2];
  tile64(p, b, dt * kTS, pt * kTS, g, sy, sx);
  double s = g[0][0] * g[0][0] + g[0][1] * g[0][1] + g[1][0] * g[1][0] + g[1][1] * g[1][1];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    p.part[static_cast<long long>(b) * p.n_tiles + dt * p.n_pt + pt] = t;
  }
}

__global__ void k64_factors(const F64Params p) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= p.B) return;
  double s = 0.0;
  for (int i = 0; i < p.n_tiles; ++i) s += p.part[static_cast<long long>(b) * p.n_tiles + i];
  p.norms_out[b] = s;
  p.factor[b] = p.with_clip ? ((s <= p.clip_c * p.clip_c) ? 1.0 : p.clip_c / sqrt(s)) : 1.0;
}

__global__ void __launch_bounds__(256) k64_weighted_sum(const F64Params p) {
  __shared__ double sy[kTS][kTS + 1];
  __shared__ double sx[kTS][kTS + 1];
  const int pt = blockIdx.x, dt = blockIdx.y;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int b = 0; b < p.B; ++b) {
    double g[2][2];
    tile64(p, b, dt * kTS, pt * kTS, g, sy, sx);
    const double f = p.with_clip ? p.factor[b] : 1.0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j] = fma(f, g[i][j], acc[i][j]);
  }
  uint64_t base = p.key_base, base_g = p.key_base_g;
  if (p.step_ptr) {
    base = absorb3(p.seed_u, p.layer_u, static_cast<uint64_t>(*p.step_ptr));
    base_g = base + kGamma;
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
      // finalize (dpcore.py:60-73): sum or sum / B, then sigma*C*draw (noise not divided)
      double v = acc[i][j] * p.inv_batch;
      if (p.with_clip && p.add_noise && flat >= p.noise_lo && flat < p.noise_hi) {
        const double z = p.noise_impl == 2 ? static_cast<double>(philox_normal(base, static_cast<uint64_t>(flat)))
                                           : keyed_normal_f64(base_g, static_cast<uint64_t>(flat));
        v += p.noise_scale * z;
      }
      if (p.accumulate) v += p.grad_w[flat];
      p.grad_w[flat] = v;
    }
  }
}

}  // namespace

cudaError_t f64_backward(const F64Params& p, cudaStream_t s) {
  if (p.with_clip) {
    k64_partial_norms<<<dim3(p.n_pt, p.n_dt, p.B), 256, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k64_factors<<<(p.B + 127) / 128, 128, 0, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  k64_weighted_sum<<<dim3(p.n_pt, p.n_dt), 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace fdp
