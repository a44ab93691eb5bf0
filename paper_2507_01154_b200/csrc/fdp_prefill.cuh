// Noise pre-fill of grad_w rows, run by the two spare warps of warpgroup 0 while
// the MMA and the epilogue work on the same tile (fdp_tc.cu, fdp_group.cu).
//
// grad_w[d, p] = (accumulate ? grad_w[d, p] : 0) + scale * N(key, d*P + p) for
// d in [d_lo, min(d_hi, D)), p in [p0, min(p0 + BN, P)), restricted to the flat
// noise range [lo, hi) (rank partition). Reference: dpcore.py:60-73 (finalize),
// rng.py:35-85 (draws).
//
// Only 64 threads do this, so the loop is latency-bound on the dependent
// Philox / Box-Muller chain: each thread keeps kIlp independent draws in flight
// (the noise implementation is a template parameter so the unrolled body has no
// runtime branch to serialise it).
#pragma once
#include "fdp_rng.cuh"

namespace fdp {

template <int BN, int IMPL>
__device__ __forceinline__ void prefill_rows_impl(float* __restrict__ grad_w, int D, int P, int d_lo, int d_hi, int p0,
                                                  bool accumulate, bool draw, uint64_t kbg, uint64_t kb, float scale,
                                                  long long lo, long long hi, int ntid) {
  constexpr int kQ = BN / 4;  // float4 per tile row
#ifndef FDP_PREFILL_ILP
#define FDP_PREFILL_ILP 4
#endif
  constexpr int kIlp = FDP_PREFILL_ILP;
  const int q_all = (d_hi - d_lo) * kQ;
  for (int base = ntid; base < q_all; base += 64 * kIlp) {
    long long flat[kIlp];
    bool ok[kIlp];
#pragma unroll
    for (int u = 0; u < kIlp; ++u) {
      const int e4 = base + u * 64;
      const int dd = d_lo + e4 / kQ, pp = p0 + (e4 % kQ) * 4;
      ok[u] = e4 < q_all && dd < D && pp < P;  // P % 8 == 0: a float4 never straddles a row
      flat[u] = static_cast<long long>(dd) * P + pp;
    }
    // flat grows with e4, so the batch overlaps [lo, hi) iff its ends do
    const bool any = draw && flat[kIlp - 1] + 3 >= lo && flat[0] < hi;
    float4 n[kIlp];
    if (any) {
#pragma unroll
      for (int u = 0; u < kIlp; ++u) n[u] = noise_draw4(IMPL, kbg, kb, static_cast<uint64_t>(flat[u] >> 2));
    }
#pragma unroll
    for (int u = 0; u < kIlp; ++u) {
      if (!ok[u]) continue;
      float4* dst = reinterpret_cast<float4*>(grad_w + flat[u]);
      float4 v = accumulate ? __ldcg(dst) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (any) {
        const long long f = flat[u];
        if (f + 0 >= lo && f + 0 < hi) v.x += scale * n[u].x;
        if (f + 1 >= lo && f + 1 < hi) v.y += scale * n[u].y;
        if (f + 2 >= lo && f + 2 < hi) v.z += scale * n[u].z;
        if (f + 3 >= lo && f + 3 < hi) v.w += scale * n[u].w;
      }
      __stcg(dst, v);
    }
  }
}

template <int BN>
__device__ __forceinline__ void prefill_rows(float* grad_w, int D, int P, int d_lo, int d_hi, int p0, bool accumulate,
                                             bool draw, int impl, uint64_t kbg, uint64_t kb, float scale, long long lo,
                                             long long hi, int ntid) {
  if (!draw || impl == 2)
    prefill_rows_impl<BN, 2>(grad_w, D, P, d_lo, d_hi, p0, accumulate, draw, kbg, kb, scale, lo, hi, ntid);
  else if (impl == 1)
    prefill_rows_impl<BN, 1>(grad_w, D, P, d_lo, d_hi, p0, accumulate, draw, kbg, kb, scale, lo, hi, ntid);
  else
    prefill_rows_impl<BN, 0>(grad_w, D, P, d_lo, d_hi, p0, accumulate, draw, kbg, kb, scale, lo, hi, ntid);
}

}  // namespace fdp
