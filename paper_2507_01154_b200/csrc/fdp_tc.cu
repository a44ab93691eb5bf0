// fdp_tc.cu -- persistent tcgen05 kernel for the per-layer DP weight gradient.
//
// A work tile is CG x 128 d-rows x BN p-columns of grad_w (D,P); CG = 2 pairs two
// SMs (a cluster) on one 256-row UMMA (cta_group::2): each CTA stages its own 128
// dY rows and half of the X columns, so per-SM operand traffic drops by a third
// (BN=128) or half (BN=256) versus a single-CTA tile. Each CTA owns the
// 128 x BN accumulator of its rows in its TMEM.
//
// For every sample b the tile computes the per-sample gradient
//   G_b[d,p] = sum_t dY[b,t,d] * X[b,t,p]                 (workflows.py:384, tensor.py:64-73)
// TMA stages dY/X (both MN-major, 128B swizzle) into shared memory, one elected
// thread issues tcgen05.mma into one of NBUF = 512/BN TMEM buffers, so the MMA of
// samples b+1.. runs while the epilogue of sample b waits on the norm all-reduce.
//
// MODE_FUSED is Algorithm 1 in one launch:
//   intra-block reduce   sum of G_b^2 over the CTA tile (warp shuffle + smem) workflows.py:387
//   inter-block reduce   partial -> ws_part[b][tile], release-add counter     workflows.py:389
//   block-wise sync      spin (acquire) until all tiles of sample b arrive    workflows.py:394-395
//   clip                 c_b = min(1, C/||G_b||), 1 if ||G_b|| == 0            workflows.py:59-65
//   aggregate            acc += c_b * G_b (fp32 registers)                     workflows.py:402-407
//   finalize             mean scaling + keyed noise, store grad_w              workflows.py:103-115
// Per-sample gradients never reach HBM; the only per-sample values that do are
// the B x n_tiles norm partials. Every CTA sums the partials in a fixed order,
// so clip factors and results are deterministic.
//
// The other modes reuse the pipeline: NORMS (norm partials only), REWEIGHT
// (clip factors precomputed: the second phase of the two-phase path), STORE_G
// (explicit baseline stage 1), NONDP (plain dW GEMM accumulated in TMEM).
#include <cstdio>
#include <cstdlib>

#include "fdp_internal.h"
#include "fdp_ptx.cuh"
#include "fdp_prefill.cuh"
#include "fdp_rng.cuh"

namespace fdp {

template <int BN, int CG>
struct TcCfg {
  static constexpr int kBCols = BN / CG;                  // X columns staged per CTA
  static constexpr int kABytes = kBM * kBK * 2;           // 16 KB: two 64-wide d atoms x 64 t rows
  static constexpr int kBBytes = kBCols * kBK * 2;        // kBCols/64 atoms x 8 KB
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kNBuf = 512 / BN;                  // TMEM accumulator buffers
  static constexpr int kCPT = BN / 2;                     // accumulator columns per epilogue thread
  static constexpr int kBarBytes = 1024;
  // epilogue staging: two buffers x two 128-row x 32-column fp32 boxes (TMA store /
  // reduce-add of a persistent tile while the next tile's MMAs run); MODE_STORE_G
  // reuses it as per-warp 32x33 transpose buffers
  static constexpr int kStgBytes = 4 * kBM * 128;
  static_assert(kStgBytes >= kEpiWarps * 32 * 33 * 4, "transpose buffers must fit the staging area");
  static constexpr int kStages = (232448 - 1024 - kBarBytes - kStgBytes) / kStageBytes;
  static constexpr size_t kSmem = 1024 /*align slack*/ + size_t(kStages) * kStageBytes + kStgBytes + kBarBytes;
  static constexpr uint32_t kIdesc = make_idesc_bf16_mn(kBM * CG, BN);
};

#define FDP_TRACE(slot)                                                                          \
  do {                                                                                           \
    if (p.trace && etid == 0 && (slot) < 128) p.trace[blockIdx.x * 128 + (slot)] = globaltimer_ns(); \
  } while (0)

template <int BN, int CG>
__global__ void __launch_bounds__(kTcThreads, 1)
    dpdw_tc_kernel(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_x,
                   const __grid_constant__ EpiMaps em, const TcParams p) {
  using C = TcCfg<BN, CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + C::kStages * C::kStageBytes;  // 1024-aligned staging boxes (kStgBytes)
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + C::kStgBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kNBuf;
  uint64_t* rs_bar = tempty + C::kNBuf;  // reduce-scatter slice loads (one phase per launch)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(rs_bar + 1);
  float* red = reinterpret_cast<float*>(tmem_holder + 4);  // [kEpiWarps]
  float* bcast = red + kEpiWarps;                           // [1] (ordered by named barriers)
  float* stage_buf = reinterpret_cast<float*>(stg);  // MODE_STORE_G transpose buffers

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned* err = p.ws_ctrl + 1;
  const int rank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kNBuf; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CG);
    }
    mbar_init(rs_bar, 1);
    fence_mbar_init();
    fence_proxy_async_smem();
    prefetch_tmap(&tm_dy);
    prefetch_tmap(&tm_x);
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair<512>(tmem_holder);
    else tmem_alloc<512>(tmem_holder);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // ---- work assignment (a "work tile" is processed by the CG CTAs of a cluster)
  const bool fused = p.mode == MODE_FUSED;
  const bool per_sample = p.mode != MODE_NONDP;
  const int cid = blockIdx.x / CG, n_clusters = gridDim.x / CG;
  int first_wt, wt_stride, b0, b_step, group;
  if (fused) {
    first_wt = cid % p.n_wtiles;
    group = cid / p.n_wtiles;
    wt_stride = p.n_wtiles;  // exactly one work tile per cluster
    b0 = group;
    b_step = p.groups;
  } else {
    first_wt = cid;
    wt_stride = n_clusters;
    group = 0;
    b0 = 0;
    b_step = 1;
  }
  const int unit_step = per_sample ? b_step : p.B;

  if (warp == 0) {
    // ======================= TMA producer (every CTA loads its own operands) =======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int wt = first_wt; wt < p.n_wtiles; wt += wt_stride) {
        const int d0 = ((wt / p.n_pt) * CG + rank) * kBM;
        const int p0 = (wt % p.n_pt) * BN + rank * C::kBCols;
        for (int ub = b0; ub < p.B; ub += unit_step) {
          const int b_end = per_sample ? ub + 1 : p.B;
          for (int b = ub; b < b_end; ++b) {
            for (int kb = 0; kb < p.n_kb; ++kb) {
              mbar_wait(&empty[stage], phase ^ 1, err, p.budget_ns, 0x101);
              uint8_t* sa = smem + stage * C::kStageBytes;
              uint8_t* sb = sa + C::kABytes;
              if constexpr (CG == 2) {
                if (leader) mbar_arrive_expect_tx(&full[stage], C::kStageBytes * CG);
                tma_load_3d_pair(sa, &tm_dy, &full[stage], d0, kb * kBK, b);
                tma_load_3d_pair(sa + 8192, &tm_dy, &full[stage], d0 + 64, kb * kBK, b);
#pragma unroll
                for (int j = 0; j < C::kBCols / 64; ++j)
                  tma_load_3d_pair(sb + j * 8192, &tm_x, &full[stage], p0 + 64 * j, kb * kBK, b);
              } else {
                mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                tma_load_3d(sa, &tm_dy, &full[stage], d0, kb * kBK, b);
                tma_load_3d(sa + 8192, &tm_dy, &full[stage], d0 + 64, kb * kBK, b);
#pragma unroll
                for (int j = 0; j < C::kBCols / 64; ++j)
                  tma_load_3d(sb + j * 8192, &tm_x, &full[stage], p0 + 64 * j, kb * kBK, b);
              }
              if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA only) =======================
    if (lane == 0 && leader) {
      uint32_t stage = 0, phase = 0, buf = 0, tphase = 0;
      for (int wt = first_wt; wt < p.n_wtiles; wt += wt_stride) {
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
                if constexpr (CG == 2) tc_mma_f16_pair(dtm, ad, bd, C::kIdesc, accum);
                else tc_mma_f16(dtm, ad, bd, C::kIdesc, accum);
                accum = 1;
              }
              if constexpr (CG == 2) tc_commit_pair(&empty[stage]);
              else tc_commit(&empty[stage]);
              if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            }
          }
          if constexpr (CG == 2) tc_commit_pair(&tfull[buf]);
          else tc_commit(&tfull[buf]);
          if (++buf == C::kNBuf) { buf = 0; tphase ^= 1; }
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ======================= noise warps (warpgroup 0's spare warps) =======================
    // Pre-fill this CTA's rows of grad_w with (accumulate ? grad_w : 0) + sigma*C*noise
    // (rng.py keyed draws or Philox, 4 consecutive columns per thread) while the MMA
    // and the epilogue run; the epilogue waits on named barrier 2 before its final
    // (reduce-add) store. No accumulator registers live here.
    // (the persistent reweight pass draws Philox noise in its epilogue instead)
    const bool reduce_scatter = fused && p.groups > 1;
    const bool atomic_groups = reduce_scatter && !p.deterministic;
    const bool draw_noise = (fused || (p.mode == MODE_REWEIGHT && !p.epi_noise)) && p.add_noise;
    const bool pre_noise = draw_noise || atomic_groups;
    if (pre_noise) {
      uint64_t kb = p.key_base, kbg = p.key_base_g;
      if (p.step_ptr) {
        kb = absorb3(p.seed_u, p.layer_u, static_cast<uint64_t>(*p.step_ptr));
        kbg = kb + kGamma;
      }
      const int own_r0 = reduce_scatter ? group * kBM / p.groups : 0;
      const int own_r1 = reduce_scatter ? (group + 1) * kBM / p.groups : kBM;
      const int ntid = (warp - 2) * 32 + lane;
      for (int wt = first_wt; wt < p.n_wtiles; wt += wt_stride) {
        const int d0 = ((wt / p.n_pt) * CG + rank) * kBM;
        const int p0 = (wt % p.n_pt) * BN;
        prefill_rows<BN>(p.grad_w, p.D, p.P, d0 + own_r0, d0 + own_r1, p0, p.accumulate != 0, draw_noise,
                         p.noise_impl, kbg, kb, p.noise_scale, p.noise_lo, p.noise_hi, ntid);
        __threadfence();
        if (atomic_groups) {  // count this group's pre-fill right away (see the epilogue's reduce-add)
          named_bar_sync(3, 64);
          if (ntid == 0) red_release_add_u32(&p.ws_tile_cnt[wt * CG + rank], 1u);
        }
        // bar.sync (not arrive): the noise warps must not run a whole tile ahead
        // of the epilogue in persistent modes, or barrier generations would mix
        named_bar_sync(2, 32 * (2 + kEpiWarps));
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ======================= epilogue (8 warps per CTA) =======================
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int half = ew >> 2;            // column half
    const int etid = ew * 32 + lane;     // 0..255
    const int row = q * 32 + lane;       // tile-local d
    const int col0 = half * C::kCPT;     // tile-local first p
    float* tbuf = stage_buf + ew * (32 * 33);  // this warp's 32x33 transpose buffer (MODE_STORE_G)
    uint32_t rbuf = 0, rph = 0;          // next TMEM buffer to wait for (buffers complete in order)

    auto wait_ready = [&]() -> uint32_t {
      mbar_wait(&tfull[rbuf], rph, err, p.budget_ns, 0x104);
      tc_fence_after();
      const uint32_t b = rbuf;
      if (++rbuf == C::kNBuf) { rbuf = 0; rph ^= 1; }
      return b;
    };
    auto release = [&](uint32_t b) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_leader(&tempty[b]);
        else mbar_arrive(&tempty[b]);
      }
    };
    auto taddr = [&](uint32_t b) { return tmem_base + (static_cast<uint32_t>(q * 32) << 16) + b * BN + col0; };

    const bool reduce_scatter = fused && p.groups > 1;
    // grad_w rows are pre-filled by the noise warps (old value if accumulating,
    // + noise) when noise is drawn, and always when sample groups combine their
    // tiles with TMA reduce-add (every group then adds onto initialised rows).
    const bool atomic_groups = reduce_scatter && !p.deterministic;
    const bool pre_noise = ((fused || (p.mode == MODE_REWEIGHT && !p.epi_noise)) && p.add_noise) || atomic_groups;
    const bool rmw_store = pre_noise || p.accumulate;
    // MODE_REWEIGHT with p.epi_noise (Philox; host default, FDP_EPI_NOISE=0 turns it off):
    // the epilogue starts each tile's accumulator at sigma*C*N(key, d*P + p), so
    // the tile leaves with a plain TMA store and no grad_w pre-fill.
    const bool epi_noise = p.mode == MODE_REWEIGHT && p.add_noise && p.epi_noise;
    uint64_t nkb = p.key_base;
    if (epi_noise && p.step_ptr) nkb = absorb3(p.seed_u, p.layer_u, static_cast<uint64_t>(*p.step_ptr));
    // launch tag of the tagged norm-partial slots (bumped by the last CTA at exit)
    unsigned tag = __ldcg(p.ws_ctrl + 2) + 1u;
    if (tag == 0u) tag = 1u;
    const int n_units = per_sample ? (p.B - b0 + b_step - 1) / b_step : 1;
    const int own_r0 = reduce_scatter ? group * kBM / p.groups : 0;
    const int own_r1 = reduce_scatter ? (group + 1) * kBM / p.groups : kBM;

    for (int wt = first_wt; wt < p.n_wtiles; wt += wt_stride) {
      const int tile = wt * CG + rank;  // CTA-level tile id (norm partials, reduce-scatter slots)
      const int d0 = ((wt / p.n_pt) * CG + rank) * kBM;
      const int p0 = (wt % p.n_pt) * BN;
      float acc[C::kCPT];
#pragma unroll
      for (int i = 0; i < C::kCPT; ++i) acc[i] = 0.0f;
      // Philox noise of this thread's 128 columns is the accumulator's initial value
      // (drawn while the tile's first MMAs run; the rank's slice only)
      if (epi_noise) {
        const long long frow = static_cast<long long>(d0 + row) * p.P;
        const bool row_ok = d0 + row < p.D;
#pragma unroll
        for (int q4 = 0; q4 < C::kCPT / 4; ++q4) {
          const int col = p0 + col0 + 4 * q4;
          const long long f = frow + col;
          if (row_ok && col < p.P && f + 3 >= p.noise_lo && f < p.noise_hi) {  // P % 8 == 0: quads stay in a row
            const float4 n = philox_normal4(nkb, static_cast<uint64_t>(f >> 2));
            acc[4 * q4 + 0] = (f + 0 >= p.noise_lo && f + 0 < p.noise_hi) ? p.noise_scale * n.x : 0.0f;
            acc[4 * q4 + 1] = (f + 1 >= p.noise_lo && f + 1 < p.noise_hi) ? p.noise_scale * n.y : 0.0f;
            acc[4 * q4 + 2] = (f + 2 >= p.noise_lo && f + 2 < p.noise_hi) ? p.noise_scale * n.z : 0.0f;
            acc[4 * q4 + 3] = (f + 3 >= p.noise_lo && f + 3 < p.noise_hi) ? p.noise_scale * n.w : 0.0f;
          }
        }
      }

      // Coalesced write of this warp's 32 rows x kCPT accumulator columns via a
      // 32x33 smem transpose: every store instruction covers 128 contiguous bytes
      // of one row. `dst` is the (row 0, col 0) element of the tile in a row-major
      // matrix with leading dimension `ld`; rows/cols beyond (nrow, ncol) are masked.
      auto store_tile = [&](float* dst, long long ld, int nrow, int ncol, bool add_old, const float* vals) {
#pragma unroll
        for (int c = 0; c < C::kCPT / 32; ++c) {
#pragma unroll
          for (int i = 0; i < 32; ++i) tbuf[lane * 33 + i] = vals[c * 32 + i];
          __syncwarp();
          const int cc = col0 + c * 32 + lane;
#pragma unroll 4
          for (int r = 0; r < 32; ++r) {
            const int rr = q * 32 + r;
            if (rr < nrow && cc < ncol) {
              float* g = dst + static_cast<long long>(rr) * ld + cc;
              float v = tbuf[r * 33 + lane];
              if (add_old) v += __ldcg(g);
              __stcg(g, v);
            }
          }
          __syncwarp();
        }
      };
      int trace_u = -1;
      // pass 1 + publish: intra-block reduce of ||G_b||^2 (workflows.py:387-389)
      auto publish = [&](int ub, uint32_t b) {
        float part = 0.0f;
        const uint32_t tb = taddr(b);
#pragma unroll
        for (int c = 0; c < C::kCPT / 16; ++c) {
          float v[16];
          tmem_ld16(tb + c * 16, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) part = fmaf(v[i], v[i], part);
        }
        if (trace_u >= 0) FDP_TRACE(64 + 4 * trace_u);  // pass-1 TMEM reads + FMAs done
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) red[ew] = part;
        named_bar_sync(1, 32 * kEpiWarps);
        if (trace_u >= 0) FDP_TRACE(65 + 4 * trace_u);  // block reduce done
        if (etid == 0) {
          float s = 0.0f;
#pragma unroll
          for (int w = 0; w < kEpiWarps; ++w) s += red[w];
          if (fused && p.skip_barrier && tile == p.n_tiles - 1) {
            // fault injection: publish late so the premature clip is observable
            const uint64_t t0 = globaltimer_ns();
            while (globaltimer_ns() - t0 < 200000ull) __nanosleep(1000);
          }
          if (fused) {
            // one 8-byte store carries the partial and this launch's tag: the
            // readers need no separate counter or fence (single-copy atomic)
            publish_u64(p.ws_tagged + static_cast<long long>(ub) * p.n_tiles + tile,
                        (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(s), p.pub_mode);
          } else {
            p.ws_part[static_cast<long long>(ub) * p.n_tiles + tile] = s;
          }
        }
      };
      // inter-block all-reduce of sample ub, then the clip factor (workflows.py:394-403)
      auto wait_factor = [&](int ub) -> float {
        if (ew == 0) {
          // lane l owns partial slots l, l+32, ...; spin on each until it carries this
          // launch's tag, then sum in a fixed order (fp64) -> identical on every CTA
          const unsigned long long* slots = p.ws_tagged + static_cast<long long>(ub) * p.n_tiles;
          constexpr int kMaxPer = 5;  // fused grids have n_tiles <= 160 CTA tiles
          unsigned long long v[kMaxPer];
#pragma unroll
          for (int k = 0; k < kMaxPer; ++k) {  // all loads in flight at once: one L2 round trip
            const int i = lane + 32 * k;
            v[k] = i < p.n_tiles ? poll_u64(slots + i, p.poll_mode) : (static_cast<unsigned long long>(tag) << 32);
          }
          bool stale = false;
          if (!p.skip_barrier) {
          const uint64_t t0 = globaltimer_ns();
          while (true) {  // re-poll every stale slot at once: one L2 round trip per iteration
            bool all = true;
#pragma unroll
            for (int k = 0; k < kMaxPer; ++k) all &= static_cast<unsigned>(v[k] >> 32) == tag;
            if (all) break;
            if (globaltimer_ns() - t0 > p.budget_ns) watchdog_trap(err, 0x105);
            if (p.poll_ns) __nanosleep(p.poll_ns);
#pragma unroll
            for (int k = 0; k < kMaxPer; ++k)
              if (static_cast<unsigned>(v[k] >> 32) != tag) v[k] = poll_u64(slots + lane + 32 * k, p.poll_mode);
          }
          if (trace_u >= 0) FDP_TRACE(67 + 4 * trace_u);  // every partial of the sample seen
          } else {
#pragma unroll
            for (int k = 0; k < kMaxPer; ++k) stale |= static_cast<unsigned>(v[k] >> 32) != tag;
          }
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < kMaxPer; ++k)
            if (lane + 32 * k < p.n_tiles) s += static_cast<double>(__uint_as_float(static_cast<unsigned>(v[k])));
          if (__any_sync(0xffffffffu, stale) && lane == 0)
            atomicOr(err, 0x200u);  // ordering fault: clip reads an incomplete all-reduce
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) {
            // clip_factor (dpcore.py:41-47): zero norm and ||g|| <= C pass through unscaled
            *bcast = clip_factor_f(s, p.clip_c, p.clip_c2) * p.inv_batch;
            if (tile == 0) p.norms_out[ub] = static_cast<float>(s);
          }
        }
        named_bar_sync(1, 32 * kEpiWarps);
        return *bcast;
      };
      // pass 2: clip and aggregate on chip (workflows.py:402-407)
      auto accumulate_scaled = [&](uint32_t b, float f) {
        const uint32_t tb = taddr(b);
#pragma unroll
        for (int c = 0; c < C::kCPT / 16; ++c) {
          float v[16];
          tmem_ld16(tb + c * 16, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c * 16 + i] = fmaf(f, v[i], acc[c * 16 + i]);
        }
      };

      FDP_TRACE(0);
      if (p.mode == MODE_FUSED) {
        // per sample: publish the norm partial, draw a noise chunk while the
        // block-wise all-reduce is in flight, clip + accumulate, free the TMEM
        // buffer (the MMA of the next samples proceeds meanwhile)
        for (int u = 0; u < n_units; ++u) {
          const int ub = b0 + u * b_step;
          const uint32_t b = wait_ready();
          FDP_TRACE(9 + 4 * u);
          trace_u = u < 16 ? u : -1;
          publish(ub, b);
          FDP_TRACE(8 + 4 * u);
          const float f = wait_factor(ub);
          FDP_TRACE(10 + 4 * u);
          accumulate_scaled(b, f);
          if (trace_u >= 0) FDP_TRACE(66 + 4 * trace_u);  // pass 2 done
          trace_u = -1;
          release(b);
        }
      } else if (p.mode == MODE_REWEIGHT) {
        float f_next = b0 < p.B ? __ldg(p.factors_in + b0) : 0.0f;  // one unit ahead (L2 latency off the path)
        for (int ub = b0; ub < p.B; ub += b_step) {
          const float f = f_next;
          if (ub + b_step < p.B) f_next = __ldg(p.factors_in + ub + b_step);
          const uint32_t b = wait_ready();
          accumulate_scaled(b, f);
          release(b);
        }
      } else if (p.mode == MODE_NORMS) {
        for (int ub = b0; ub < p.B; ub += b_step) {
          const uint32_t b = wait_ready();
          publish(ub, b);
          named_bar_sync(1, 32 * kEpiWarps);  // red[] reuse guard
          release(b);
        }
        continue;
      } else if (p.mode == MODE_STORE_G) {
        for (int ub = b0; ub < p.B; ub += b_step) {
          const uint32_t b = wait_ready();
          const uint32_t tb = taddr(b);
#pragma unroll
          for (int c = 0; c < C::kCPT / 32; ++c) {
            float v[32];
            tmem_ld32(tb + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[c * 32 + i] = v[i];
          }
          release(b);
          store_tile(p.g_out + (static_cast<long long>(ub) * p.D + d0) * p.P + p0, p.P, p.D - d0, p.P - p0, false,
                     acc);
        }
        continue;
      } else {  // MODE_NONDP: one accumulation unit per tile
        const uint32_t b = wait_ready();
        const uint32_t tb = taddr(b);
#pragma unroll
        for (int c = 0; c < C::kCPT / 32; ++c) {
          float v[32];
          tmem_ld32(tb + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[c * 32 + i] = v[i];
        }
        release(b);
      }
      FDP_TRACE(1);
      // grad_w rows pre-filled by the noise warps (generic stores, fenced) before
      // any store / TMA reduce-add of this tile
      if (pre_noise) named_bar_sync(2, 32 * (2 + kEpiWarps));

      if (fused) {
        // ---- epilogue I/O through TMA. The accumulator tile goes to shared memory
        // (free now: every stage has been consumed) in 32-column boxes with the
        // 128B swizzle, then bulk tensor stores move it. When grad_w already holds
        // the noise (or the accumulated gradient) the store is a TMA reduce-add.
        uint8_t* stg0 = smem;  // box kb at stg0 + kb * 16 KB: 128 rows x 128 B
#pragma unroll
        for (int c = 0; c < C::kCPT / 32; ++c) {
          uint8_t* box = stg0 + (col0 / 32 + c) * (kBM * 128) + row * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(box + ((j ^ (row & 7)) << 4)) =
                make_float4(acc[c * 32 + 4 * j], acc[c * 32 + 4 * j + 1], acc[c * 32 + 4 * j + 2],
                            acc[c * 32 + 4 * j + 3]);
        }
        fence_proxy_async_smem();
        if (rmw_store) __threadfence_block();  // noise chunks (generic) before the TMA reduce
        named_bar_sync(1, 32 * kEpiWarps);
        if (reduce_scatter && !p.deterministic) {
          // every group reduce-adds its whole clipped tile onto grad_w once all
          // groups have initialised (pre-filled) their row slices (the noise warps
          // count each pre-fill as soon as it is visible)
          if (etid == 0) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_u32(&p.ws_tile_cnt[tile]) < static_cast<unsigned>(p.groups)) {
              if (globaltimer_ns() - t0 > p.budget_ns) watchdog_trap(err, 0x106);
              __nanosleep(64);
            }
            fence_proxy_async_global();
            for (int kbx = 0; kbx < BN / 32; ++kbx)
              tma_reduce_add_2d(&em.gw, stg0 + kbx * (kBM * 128), p0 + kbx * 32, d0);
            bulk_commit();
            bulk_wait_all();
          }
          FDP_TRACE(2);
          continue;
        }
        if (!reduce_scatter) {
          if (etid == 0) {
            fence_proxy_async_global();
            for (int kbx = 0; kbx < BN / 32; ++kbx) {
              if (rmw_store) tma_reduce_add_2d(&em.gw, stg0 + kbx * (kBM * 128), p0 + kbx * 32, d0);
              else tma_store_2d(&em.gw, stg0 + kbx * (kBM * 128), p0 + kbx * 32, d0);
            }
            bulk_commit();
            bulk_wait_all();
          }
          FDP_TRACE(2);
          continue;
        }
        // ---- reduce-scatter across the tile's sample groups (deterministic order):
        // park the partial tile in L2, then group g sums rows [g*BM/S, (g+1)*BM/S)
        // of all S partials and adds them onto its (pre-noised) rows of grad_w.
        const int rows_own = own_r1 - own_r0;
        const int slot0 = tile * p.groups;
        if (etid == 0) {
          for (int kbx = 0; kbx < BN / 32; ++kbx) tma_store_3d(&em.slot, stg0 + kbx * (kBM * 128), kbx * 32, 0, slot0 + group);
          bulk_commit();
          bulk_wait_all();
          fence_proxy_async_global();
          red_release_add_u32(&p.ws_tile_cnt[tile], 1u);
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_u32(&p.ws_tile_cnt[tile]) < static_cast<unsigned>(p.groups)) {
            if (globaltimer_ns() - t0 > p.budget_ns) watchdog_trap(err, 0x106);
            __nanosleep(64);
          }
          fence_proxy_async_global();
          mbar_arrive_expect_tx(rs_bar, static_cast<uint32_t>(p.groups * (BN / 32) * rows_own * 128));
          for (int g = 0; g < p.groups; ++g)
            for (int kbx = 0; kbx < BN / 32; ++kbx)
              tma_load_3d(stg0 + (g * (BN / 32) + kbx) * (rows_own * 128), &em.slice, rs_bar, kbx * 32, own_r0,
                          slot0 + g);
        }
        mbar_wait(rs_bar, 0, err, p.budget_ns, 0x107);
        const int n4 = rows_own * (BN / 4);  // float4 chunks of the slice
        const int box_bytes = rows_own * 128;
        for (int e4 = etid; e4 < n4; e4 += 32 * kEpiWarps) {
          const int kbx = e4 / (rows_own * 8);
          const int rem = e4 % (rows_own * 8);
          const int r = rem >> 3, j = rem & 7;
          const int off = kbx * box_bytes + r * 128 + ((j ^ (r & 7)) << 4);
          float4 s = *reinterpret_cast<const float4*>(stg0 + off);
          for (int g = 1; g < p.groups; ++g) {
            const float4 t4 = *reinterpret_cast<const float4*>(stg0 + g * (BN / 32) * box_bytes + off);
            s.x += t4.x; s.y += t4.y; s.z += t4.z; s.w += t4.w;
          }
          *reinterpret_cast<float4*>(stg0 + off) = s;
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 32 * kEpiWarps);
        if (etid == 0) {
          fence_proxy_async_global();
          for (int kbx = 0; kbx < BN / 32; ++kbx) {
            if (rmw_store) tma_reduce_add_2d(&em.gw_slice, stg0 + kbx * box_bytes, p0 + kbx * 32, d0 + own_r0);
            else tma_store_2d(&em.gw_slice, stg0 + kbx * box_bytes, p0 + kbx * 32, d0 + own_r0);
          }
          bulk_commit();
          bulk_wait_all();
        }
        FDP_TRACE(2);
        continue;
      }

      // ---- finalize (persistent modes: REWEIGHT, NONDP): mean is folded into the
      // clip factor; the noise (if any) is already in grad_w. The tile leaves through
      // TMA in 32-column boxes, double-buffered, so the next tile's MMAs (already
      // running into the free TMEM buffer) never wait on the stores; rows / columns
      // beyond (D, P) are clipped by the tensor map.
#pragma unroll
      for (int c = 0; c < C::kCPT / 32; ++c) {
        uint8_t* sbuf = stg + (c & 1) * (2 * kBM * 128);
        if (etid == 0) bulk_wait_read_le1();  // the boxes issued two rounds ago have left this buffer
        named_bar_sync(1, 32 * kEpiWarps);
        uint8_t* box = sbuf + half * (kBM * 128) + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(box + ((j ^ (row & 7)) << 4)) =
              make_float4(acc[c * 32 + 4 * j], acc[c * 32 + 4 * j + 1], acc[c * 32 + 4 * j + 2],
                          acc[c * 32 + 4 * j + 3]);
        fence_proxy_async_smem();
        named_bar_sync(1, 32 * kEpiWarps);
        if (etid == 0) {
          fence_proxy_async_global();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = p0 + h * C::kCPT + c * 32;
            if (rmw_store) tma_reduce_add_2d(&em.gw, sbuf + h * (kBM * 128), col, d0);
            else tma_store_2d(&em.gw, sbuf + h * (kBM * 128), col, d0);
          }
          bulk_commit();
        }
      }
      FDP_TRACE(2);
    }
  }

  if (warp >= kEpiWarp0 && threadIdx.x == 32 * kEpiWarp0) bulk_wait_all();  // staging reads + stores complete
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // the leader's MMAs wrote the peer's TMEM / read its smem
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (CG == 2) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }

  if (fused && threadIdx.x == 0) {
    // last CTA out re-arms the workspace counters for the next call
    __threadfence();
    const unsigned old = atomicAdd(&p.ws_ctrl[0], 1u);
    if (old == gridDim.x - 1) {
      __threadfence();
      for (int t = 0; t < p.n_tiles; ++t) p.ws_tile_cnt[t] = 0u;
      unsigned tag = p.ws_ctrl[2] + 1u;
      if (tag == 0u) tag = 1u;
      p.ws_ctrl[2] = tag;  // the next fused launch on this workspace uses tag + 1
      p.ws_ctrl[0] = 0u;
      __threadfence();
    }
  }
}

template <int BN, int CG>
static cudaError_t set_attr_once() {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(dpdw_tc_kernel<BN, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(TcCfg<BN, CG>::kSmem));
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}

template <int BN, int CG>
static cudaError_t launch_tc_impl(const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const EpiMaps& em,
                                  const TcParams& p, int grid, bool cooperative, cudaStream_t stream) {
  using C = TcCfg<BN, CG>;
  cudaError_t e = set_attr_once<BN, CG>();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  // FDP_NO_COOP=1: plain launch (profilers that cannot replay cooperative cluster
  // launches); the grid never exceeds the co-resident capacity either way
  if (cooperative && !std::getenv("FDP_NO_COOP")) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, dpdw_tc_kernel<BN, CG>, tm_dy, tm_x, em, p);
  if (e != cudaSuccess && cooperative && CG == 2 && std::getenv("FDP_ALLOW_NONCOOP")) {
    // A rejected cooperative launch is an error: the fused kernel's grid barrier
    // needs co-residency (see fdp_group.cu). FDP_ALLOW_NONCOOP=1 opts into a
    // plain cluster launch (grid <= co-resident capacity, watchdog-guarded).
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, dpdw_tc_kernel<BN, CG>, tm_dy, tm_x, em, p);
  }
  return e;
}

cudaError_t launch_tc(int bn, int cg, const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const EpiMaps& em,
                      const TcParams& p, int grid, bool cooperative, cudaStream_t stream) {
  if (cg == 2) {
    if (bn == 256) return launch_tc_impl<256, 2>(tm_dy, tm_x, em, p, grid, cooperative, stream);
    return launch_tc_impl<128, 2>(tm_dy, tm_x, em, p, grid, cooperative, stream);
  }
  if (bn == 256) return launch_tc_impl<256, 1>(tm_dy, tm_x, em, p, grid, cooperative, stream);
  return launch_tc_impl<128, 1>(tm_dy, tm_x, em, p, grid, cooperative, stream);
}

template <int BN, int CG>
static int coresident_impl(int sms) {
  if (set_attr_once<BN, CG>() != cudaSuccess) return 0;
  if (CG == 1) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, dpdw_tc_kernel<BN, CG>, kTcThreads,
                                                      TcCfg<BN, CG>::kSmem) != cudaSuccess)
      return 0;
    return n * sms;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * sms);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = TcCfg<BN, CG>::kSmem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, dpdw_tc_kernel<BN, CG>, &cfg) != cudaSuccess) return 0;
  return clusters * CG;
}

int tc_max_coresident_ctas(int bn, int cg) {
  static int cache[64][4];
  static bool have[64][4];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  const int k = (bn == 256 ? 1 : 0) + (cg == 2 ? 2 : 0);
  if (have[dev][k]) return cache[dev][k];
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  int n;
  if (cg == 2) n = bn == 256 ? coresident_impl<256, 2>(sms) : coresident_impl<128, 2>(sms);
  else n = bn == 256 ? coresident_impl<256, 1>(sms) : coresident_impl<128, 1>(sms);
  (void)cudaGetLastError();
  cache[dev][k] = n;
  have[dev][k] = true;
  return n;
}

}  // namespace fdp
