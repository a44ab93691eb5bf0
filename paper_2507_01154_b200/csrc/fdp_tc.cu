// fdp_tc.cu -- persistent tcgen05 kernel for the per-layer DP weight gradient.
//
// One CTA owns one 128 x BN output tile (d rows x p columns) of grad_w (D,P).
// For every sample b it assigned it computes the per-sample gradient tile
//   G_b[d,p] = sum_t dY[b,t,d] * X[b,t,p]                 (workflows.py:384, tensor.py:64-73)
// on the 5th-gen tensor cores: TMA stages dY/X tiles (both MN-major, 128B
// swizzle) into shared memory, one elected thread issues tcgen05.mma into a
// TMEM accumulator (NBUF = 512/BN buffers, so the MMA of sample b+1.. runs
// while the epilogue of sample b waits on the norm all-reduce).
//
// MODE_FUSED is Algorithm 1 in one launch:
//   intra-block reduce   sum of G_b^2 over the tile (warp shuffle + smem)  workflows.py:387
//   inter-block reduce   partial -> ws_part[b][tile], release-add counter  workflows.py:389
//   block-wise sync      spin (acquire) until all tiles of sample b arrive workflows.py:394-395
//   clip                 c_b = min(1, C/||G_b||), 1 if ||G_b|| == 0         workflows.py:59-65
//   aggregate            acc += c_b * G_b (fp32 registers)                  workflows.py:402-407
//   finalize             mean scaling + keyed noise, store grad_w           workflows.py:103-115
// Per-sample gradients never reach HBM; the only per-sample values that do are
// the B x n_tiles norm partials. The partials are summed in a fixed order by
// every CTA, so the clip factors (and the result) are deterministic.
//
// The other modes reuse the same pipeline: NORMS (norm partials only),
// REWEIGHT (clip factors precomputed), STORE_G (explicit baseline stage 1),
// NONDP (plain dW GEMM accumulated in TMEM over all samples).
#include "fdp_internal.h"
#include "fdp_ptx.cuh"
#include "fdp_rng.cuh"

namespace fdp {

template <int BN>
struct TcCfg {
  static constexpr int kABytes = kBM * kBK * 2;          // 16 KB: two 64-wide d atoms x 64 t rows
  static constexpr int kBBytes = BN * kBK * 2;           // BN/64 atoms x 8 KB
  static constexpr int kStageBytes = kABytes + kBBytes;  // 32 KB (BN=128) / 48 KB (BN=256)
  static constexpr int kStages = BN == 128 ? 6 : 4;
  static constexpr int kNBuf = 512 / BN;                 // TMEM accumulator buffers
  static constexpr int kCPT = BN / 2;                    // accumulator columns per epilogue thread
  static constexpr int kBarBytes = 1024;
  static constexpr size_t kSmem = 1024 /*align slack*/ + size_t(kStages) * kStageBytes + kBarBytes;
  static constexpr uint32_t kIdesc = make_idesc_bf16_mn(kBM, BN);
};

#define FDP_TRACE(slot)                                                           \
  do {                                                                            \
    if (p.trace && etid == 0 && (slot) < 128) p.trace[blockIdx.x * 128 + (slot)] = globaltimer_ns(); \
  } while (0)

template <int BN>
__global__ void __launch_bounds__(kTcThreads, 1)
    dpdw_tc_kernel(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_x,
                   const TcParams p) {
  using C = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kNBuf;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + C::kNBuf);
  float* red = reinterpret_cast<float*>(tmem_holder + 4);  // [kEpiWarps]
  float* bcast = red + kEpiWarps;                           // [1] (ordered by named barriers)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned* err = p.ws_ctrl + 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kNBuf; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
    prefetch_tmap(&tm_dy);
    prefetch_tmap(&tm_x);
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // Register budget: the TMA/MMA warpgroup needs few registers, the epilogue
  // warpgroups hold BN/2 fp32 accumulators per thread.
#if FDP_SETMAXNREG
  if (warp < kEpiWarp0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
  }
#endif

  // ---- work assignment
  const bool fused = p.mode == MODE_FUSED;
  const bool per_sample = p.mode != MODE_NONDP;
  int first_tile, tile_stride, b0, b_step, group;
  if (fused) {
    first_tile = blockIdx.x % p.n_tiles;
    group = blockIdx.x / p.n_tiles;
    tile_stride = p.n_tiles;  // exactly one tile per CTA
    b0 = group;
    b_step = p.groups;
  } else {
    first_tile = blockIdx.x;
    tile_stride = gridDim.x;
    group = 0;
    b0 = 0;
    b_step = 1;
  }
  const int unit_step = per_sample ? b_step : p.B;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int tile = first_tile; tile < p.n_tiles; tile += tile_stride) {
        const int d0 = (tile / p.n_pt) * kBM;
        const int p0 = (tile % p.n_pt) * BN;
        for (int ub = b0; ub < p.B; ub += unit_step) {
          const int b_end = per_sample ? ub + 1 : p.B;
          for (int b = ub; b < b_end; ++b) {
            for (int kb = 0; kb < p.n_kb; ++kb) {
              mbar_wait(&empty[stage], phase ^ 1, err, p.budget_ns, 0x101);
              uint8_t* sa = smem + stage * C::kStageBytes;
              uint8_t* sb = sa + C::kABytes;
              mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
              tma_load_3d(sa, &tm_dy, &full[stage], d0, kb * kBK, b);
              tma_load_3d(sa + 8192, &tm_dy, &full[stage], d0 + 64, kb * kBK, b);
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_3d(sb + j * 8192, &tm_x, &full[stage], p0 + 64 * j, kb * kBK, b);
              if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, buf = 0, tphase = 0;
      for (int tile = first_tile; tile < p.n_tiles; tile += tile_stride) {
        for (int ub = b0; ub < p.B; ub += unit_step) {
          const int b_end = per_sample ? ub + 1 : p.B;
          mbar_wait(&tempty[buf], tphase ^ 1, err, p.budget_ns, 0x102);
          tc_fence_after();
          const uint32_t dtm = tmem_base + buf * BN;
          uint32_t accum = 0;
          for (int b = ub; b < b_end; ++b) {
            for (int kb = 0; kb < p.n_kb; ++kb) {
              mbar_wait(&full[stage], phase, err, p.budget_ns, 0x103);
              tc_fence_after();
              const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
              const uint32_t b_base = a_base + C::kABytes;
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                const uint64_t ad = make_sdesc_sw128(a_base + k * 2048, 8192, 1024);
                const uint64_t bd = make_sdesc_sw128(b_base + k * 2048, 8192, 1024);
                tc_mma_f16(dtm, ad, bd, C::kIdesc, accum);
                accum = 1;
              }
              tc_commit(&empty[stage]);
              if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            }
          }
          tc_commit(&tfull[buf]);
          if (++buf == C::kNBuf) { buf = 0; tphase ^= 1; }
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ======================= epilogue (8 warps) =======================
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int half = ew >> 2;            // column half
    const int etid = ew * 32 + lane;     // 0..255
    const int row = q * 32 + lane;       // tile-local d
    const int col0 = half * C::kCPT;     // tile-local first p
    uint32_t buf = 0, tphase = 0;

    const bool dp_sum = p.mode == MODE_FUSED || p.mode == MODE_REWEIGHT;
    uint64_t kb = p.key_base, kbg = p.key_base_g;
    if (p.step_ptr) {
      kb = absorb3(p.seed_u, p.layer_u, static_cast<uint64_t>(*p.step_ptr));
      kbg = kb + kGamma;
    }
    const bool reduce_scatter = fused && p.groups > 1;
    // noise is pre-written into grad_w in chunks while the MMA of the next
    // sample runs (single-group tiles); with sample groups it is drawn in the
    // reduce-scatter phase, split across the group's CTAs.
    const bool pre_noise = dp_sum && p.add_noise;
    const bool rmw_store = pre_noise || p.accumulate;
    const int n_units = per_sample ? (p.B - b0 + b_step - 1) / b_step : 1;
    // rows of the tile this CTA finalizes (its reduce-scatter slice with sample groups)
    const int own_r0 = reduce_scatter ? group * kBM / p.groups : 0;
    const int own_r1 = reduce_scatter ? (group + 1) * kBM / p.groups : kBM;

    for (int tile = first_tile; tile < p.n_tiles; tile += tile_stride) {
      const int d0 = (tile / p.n_pt) * kBM;
      const int p0 = (tile % p.n_pt) * BN;
      const int d = d0 + row;
      float acc[C::kCPT];
#pragma unroll
      for (int i = 0; i < C::kCPT; ++i) acc[i] = 0.0f;

      int unit = 0;
      FDP_TRACE(0);
      for (int ub = b0; ub < p.B; ub += unit_step, ++unit) {
        if (pre_noise) {
          // chunk `unit` of this CTA's noise, drawn while the MMA of sample `ub`
          // runs: grad_w = (accumulate ? grad_w : 0) + sigma*C*n(flat), 4 at a time
          // (P % 8 == 0: a float4 never straddles a row or the tile edge).
          const int q_all = (own_r1 - own_r0) * (BN / 4);
          const int q_lo = static_cast<int>((static_cast<long long>(unit) * q_all) / n_units);
          const int q_hi = static_cast<int>((static_cast<long long>(unit + 1) * q_all) / n_units);
          for (int e4 = q_lo + etid; e4 < q_hi; e4 += 32 * kEpiWarps) {
            const int dd = d0 + own_r0 + e4 / (BN / 4);
            const int pp = p0 + (e4 % (BN / 4)) * 4;
            if (dd < p.D && pp < p.P) {
              const long long flat = static_cast<long long>(dd) * p.P + pp;
              float4* dst = reinterpret_cast<float4*>(p.grad_w + flat);
              float4 v = p.accumulate ? __ldcg(dst) : make_float4(0.f, 0.f, 0.f, 0.f);
              if (flat + 3 >= p.noise_lo && flat < p.noise_hi) {
                const float4 n = noise_draw4(p.noise_impl, kbg, kb, static_cast<uint64_t>(flat >> 2));
                const float s = p.noise_scale;
                if (flat + 0 >= p.noise_lo && flat + 0 < p.noise_hi) v.x += s * n.x;
                if (flat + 1 >= p.noise_lo && flat + 1 < p.noise_hi) v.y += s * n.y;
                if (flat + 2 >= p.noise_lo && flat + 2 < p.noise_hi) v.z += s * n.z;
                if (flat + 3 >= p.noise_lo && flat + 3 < p.noise_hi) v.w += s * n.w;
              }
              __stcg(dst, v);
            }
          }
        }
        FDP_TRACE(8 + 4 * unit);
        mbar_wait(&tfull[buf], tphase, err, p.budget_ns, 0x104);
        tc_fence_after();
        FDP_TRACE(9 + 4 * unit);
        const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * BN + col0;

        if (p.mode == MODE_NONDP || p.mode == MODE_STORE_G) {
#pragma unroll
          for (int c = 0; c < C::kCPT / 32; ++c) {
            float v[32];
            tmem_ld32(tb + c * 32, v);
            tmem_wait_ld();
            if (p.mode == MODE_NONDP) {
#pragma unroll
              for (int i = 0; i < 32; ++i) acc[c * 32 + i] = v[i];
            } else if (d < p.D) {
              float* dst = p.g_out + (static_cast<long long>(ub) * p.D + d) * p.P + p0 + col0 + c * 32;
              if (p0 + col0 + c * 32 + 32 <= p.P) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) __stcs(reinterpret_cast<float4*>(dst + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (p0 + col0 + c * 32 + i < p.P) dst[i] = v[i];
              }
            }
          }
        } else {
          float f;
          if (p.mode == MODE_REWEIGHT) {
            f = p.factors_in[ub];
          } else {
            // ---- pass 1: intra-block reduce of ||G_b||^2 over this tile
            float part = 0.0f;
#pragma unroll
            for (int c = 0; c < C::kCPT / 32; ++c) {
              float v[32];
              tmem_ld32(tb + c * 32, v);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) part = fmaf(v[i], v[i], part);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (lane == 0) red[ew] = part;
            named_bar_sync(1, 32 * kEpiWarps);
            const int tiles_b = p.n_tiles;
            if (etid == 0) {
              float s = 0.0f;
#pragma unroll
              for (int w = 0; w < kEpiWarps; ++w) s += red[w];
              if (fused && p.skip_barrier && tile == p.n_tiles - 1) {
                // fault injection: publish late so the premature clip is observable
                const uint64_t t0 = globaltimer_ns();
                while (globaltimer_ns() - t0 < 200000ull) __nanosleep(1000);
              }
              p.ws_part[static_cast<long long>(ub) * tiles_b + tile] = s;
              if (fused) red_release_add_u32(&p.ws_cnt[ub], 1u);
            }
            if (p.mode == MODE_NORMS) {
              named_bar_sync(1, 32 * kEpiWarps);  // red[] reuse guard
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[buf]);
              if (++buf == C::kNBuf) { buf = 0; tphase ^= 1; }
              continue;
            }
            // ---- inter-block all-reduce: wait for every tile of sample b
            if (ew == 0) {
              if (lane == 0) {
                if (!p.skip_barrier) {
                  const uint64_t t0 = globaltimer_ns();
                  while (ld_acquire_u32(&p.ws_cnt[ub]) < static_cast<unsigned>(tiles_b)) {
                    if (globaltimer_ns() - t0 > p.budget_ns) watchdog_trap(err, 0x105);
                    __nanosleep(32);
                  }
                } else if (ld_acquire_u32(&p.ws_cnt[ub]) < static_cast<unsigned>(tiles_b)) {
                  atomicOr(err, 0x200u);  // ordering fault: clip reads an incomplete all-reduce
                }
              }
              __syncwarp();
              double s = 0.0;
              for (int i = lane; i < tiles_b; i += 32)
                s += static_cast<double>(__ldcg(p.ws_part + static_cast<long long>(ub) * tiles_b + i));
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
              if (lane == 0) {
                // clip_factor (dpcore.py:41-47): zero norm and ||g|| <= C pass through unscaled
                const double cf = (s <= p.clip_c2) ? 1.0 : p.clip_c / sqrt(s);
                *bcast = static_cast<float>(cf) * p.inv_batch;
                if (tile == 0) p.norms_out[ub] = static_cast<float>(s);
              }
            }
            named_bar_sync(1, 32 * kEpiWarps);
            f = *bcast;
            FDP_TRACE(10 + 4 * unit);
          }
          // ---- pass 2: clip and aggregate on chip
#pragma unroll
          for (int c = 0; c < C::kCPT / 32; ++c) {
            float v[32];
            tmem_ld32(tb + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[c * 32 + i] = fmaf(f, v[i], acc[c * 32 + i]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (++buf == C::kNBuf) { buf = 0; tphase ^= 1; }
      }

      FDP_TRACE(1);
      if (p.mode == MODE_NORMS || p.mode == MODE_STORE_G) continue;

      if (reduce_scatter) {
        // ---- reduce-scatter of the clipped sums across the tile's sample groups:
        // every group parks its partial tile (row-major) in L2, then group g sums
        // rows [g*BM/S, (g+1)*BM/S) of all S partials in a fixed order
        // (deterministic), adds noise and writes them.
        const long long tile_elems = static_cast<long long>(kBM) * BN;
        float* slots = p.ws_acc + static_cast<long long>(tile) * p.groups * tile_elems;
        {
          float* mine = slots + group * tile_elems + static_cast<long long>(row) * BN + col0;
#pragma unroll
          for (int i = 0; i < C::kCPT; i += 4)
            __stcg(reinterpret_cast<float4*>(mine + i), make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]));
        }
        __threadfence();
        named_bar_sync(1, 32 * kEpiWarps);
        if (etid == 0) {
          red_release_add_u32(&p.ws_tile_cnt[tile], 1u);
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_u32(&p.ws_tile_cnt[tile]) < static_cast<unsigned>(p.groups)) {
            if (globaltimer_ns() - t0 > p.budget_ns) watchdog_trap(err, 0x106);
            __nanosleep(64);
          }
        }
        named_bar_sync(1, 32 * kEpiWarps);
        const int n4 = (own_r1 - own_r0) * BN / 4;
        constexpr int kU = 4;  // float4 groups in flight per thread
        for (int base4 = etid; base4 < n4; base4 += kU * 32 * kEpiWarps) {
          float4 s[kU], o[kU];
          long long off[kU], flat[kU];
          bool ok[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int e4 = base4 + u * 32 * kEpiWarps;
            const int r = own_r0 + (e4 * 4) / BN, c = (e4 * 4) % BN;
            ok[u] = e4 < n4 && d0 + r < p.D && p0 + c < p.P;  // P % 8 == 0: all-in or all-out
            off[u] = static_cast<long long>(r) * BN + c;
            flat[u] = static_cast<long long>(d0 + r) * p.P + p0 + c;
            s[u] = ok[u] ? __ldcg(reinterpret_cast<const float4*>(slots + off[u])) : make_float4(0.f, 0.f, 0.f, 0.f);
            o[u] = (ok[u] && rmw_store) ? __ldcg(reinterpret_cast<const float4*>(p.grad_w + flat[u]))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          for (int g = 1; g < p.groups; ++g) {
            float4 t4[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u)
              t4[u] = ok[u] ? __ldcg(reinterpret_cast<const float4*>(slots + g * tile_elems + off[u]))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              s[u].x += t4[u].x; s[u].y += t4[u].y; s[u].z += t4[u].z; s[u].w += t4[u].w;
            }
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            if (!ok[u]) continue;
            // noise (and the accumulated gradient) already sit in grad_w when rmw_store
            s[u].x += o[u].x; s[u].y += o[u].y; s[u].z += o[u].z; s[u].w += o[u].w;
            *reinterpret_cast<float4*>(p.grad_w + flat[u]) = s[u];
          }
        }
        FDP_TRACE(2);
        continue;
      }

      // ---- finalize: mean is folded into the clip factor; the noise (if any) is
      // already in grad_w from the pre_noise chunks.
      if (pre_noise) {
        __threadfence_block();
        named_bar_sync(1, 32 * kEpiWarps);
      }
      if (d < p.D) {
        float* dst = p.grad_w + static_cast<long long>(d) * p.P + p0 + col0;
        if (p0 + col0 + C::kCPT <= p.P) {
#pragma unroll
          for (int i = 0; i < C::kCPT; i += 4) {
            float4 v = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
            if (rmw_store) {
              const float4 old = __ldcg(reinterpret_cast<const float4*>(dst + i));
              v.x += old.x; v.y += old.y; v.z += old.z; v.w += old.w;
            }
            *reinterpret_cast<float4*>(dst + i) = v;
          }
        } else {
#pragma unroll
          for (int i = 0; i < C::kCPT; ++i) {
            if (p0 + col0 + i < p.P) {
              float v = acc[i];
              if (rmw_store) v += __ldcg(dst + i);
              dst[i] = v;
            }
          }
        }
      }
      FDP_TRACE(2);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem_base);

  if (fused && threadIdx.x == 0) {
    // last CTA out re-arms the workspace counters for the next call
    __threadfence();
    const unsigned old = atomicAdd(&p.ws_ctrl[0], 1u);
    if (old == gridDim.x - 1) {
      __threadfence();
      for (int b = 0; b < p.B; ++b) p.ws_cnt[b] = 0u;
      for (int t = 0; t < p.n_tiles; ++t) p.ws_tile_cnt[t] = 0u;
      p.ws_ctrl[0] = 0u;
      __threadfence();
    }
  }
}

template <int BN>
static cudaError_t launch_tc_impl(const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const TcParams& p, int grid,
                                  bool cooperative, cudaStream_t stream) {
  using C = TcCfg<BN>;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(dpdw_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (cooperative) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, dpdw_tc_kernel<BN>, tm_dy, tm_x, p);
}

cudaError_t launch_tc(int bn, const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const TcParams& p, int grid,
                      bool cooperative, cudaStream_t stream) {
  if (bn == 256) return launch_tc_impl<256>(tm_dy, tm_x, p, grid, cooperative, stream);
  return launch_tc_impl<128>(tm_dy, tm_x, p, grid, cooperative, stream);
}

size_t tc_smem_bytes(int bn) { return bn == 256 ? TcCfg<256>::kSmem : TcCfg<128>::kSmem; }

int tc_max_coresident(int bn) {
  // cached per device and tile width (the occupancy query is not free)
  static int cache[64][2];
  static bool have[64][2];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  const int k = bn == 256 ? 1 : 0;
  if (have[dev][k]) return cache[dev][k];
  int n = 0;
  cudaError_t e;
  if (bn == 256) {
    cudaFuncSetAttribute(dpdw_tc_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(TcCfg<256>::kSmem));
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dpdw_tc_kernel<256>, kTcThreads, TcCfg<256>::kSmem);
  } else {
    cudaFuncSetAttribute(dpdw_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(TcCfg<128>::kSmem));
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dpdw_tc_kernel<128>, kTcThreads, TcCfg<128>::kSmem);
  }
  if (e != cudaSuccess) return 0;
  cache[dev][k] = n;
  have[dev][k] = true;
  return n;
}

}  // namespace fdp
