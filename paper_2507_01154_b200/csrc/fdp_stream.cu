// fdp_stream.cu -- stream-K persistent tcgen05 kernel for the second phase of the
// two-phase DP backward (reweight: grad_w = sum_b c_b dY_b^T X_b + noise, with the
// clip factors c_b from the norm phase) and for the non-DP dW GEMM.
//
// Work is a list of (work tile, sample) units on the K co-resident clusters: whole
// tiles in wave order while full waves last, then the units of the last partial
// wave split evenly (stream-K), so every cluster carries the same work whatever
// the tile count (a 4096x4096 layer has 256 pair tiles on 74 clusters: 3 waves +
// 34 tiles x B samples shared by all). A cluster's work is a list of segments
// (tile, samples [bb, be)); a tile split across
// clusters is combined with TMA reduce-adds onto rows initialised once by the
// noise warps of the cluster holding the tile's first samples (old value when
// accumulating, + sigma*C*noise), signalled through a per-CTA-tile counter.
// A tile held whole by one cluster leaves with a plain TMA store (or a reduce-add
// when accumulating); its Philox noise can start the accumulator instead.
//
// Reference: the recompute / reweight half of workflows.py:246-324 (implicit) and
// the non-DP sum workflows.py:121-150; finalize and noise dpcore.py:60-73.
#include <cstdio>
#include <cstdlib>

#include "fdp_internal.h"
#include "fdp_prefill.cuh"
#include "fdp_ptx.cuh"
#include "fdp_rng.cuh"

namespace fdp {

template <int BN, int CG>
struct SCfg {
  static constexpr int kBCols = BN / CG;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = kBCols * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStgBytes = 4 * kBM * 128;  // 2 buffers x two 128-row x 32-column fp32 boxes
  static constexpr int kBarBytes = 1024;
  static constexpr int kStages = (232448 - 1024 - kBarBytes - kStgBytes) / kStageBytes;
  static constexpr int kNBuf = 512 / BN;
  static constexpr int kCPT = BN / 2;
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes + kStgBytes + kBarBytes;
  static constexpr uint32_t kIdesc = make_idesc_bf16_mn(kBM * CG, BN);
};

// Segment walk of one cluster: the first floor(n_wtiles / K) waves hand out whole
// tiles in wave order (tile w*K + c), so the clusters of a wave work on
// neighbouring tiles whose operand rows share L2; the units of the remaining
// R = n_wtiles mod K tiles (tile-major, R*B of them) are split evenly, cluster c
// taking [R B c / K, R B (c+1) / K). The tail range is walked from its END, and
// its last segment -- the tile the cluster opens (samples from 0) -- goes before
// the waves: a split tile's opening segment is finished (its rows initialised)
// long before the clusters continuing it reach their stores, which come last.
struct SegWalk {
  int cid, K, B, waves, w;
  int phase;  // 0: the tail's opening segment (if any), 1: the waves, 2: the rest of the tail
  long long u, hi, tail0;
  __device__ __forceinline__ SegWalk(int cid_, int K_, int B_, int n_wtiles)
      : cid(cid_), K(K_), B(B_), w(0), phase(0) {
    waves = n_wtiles / K_;
    tail0 = static_cast<long long>(waves) * K_;
    const long long tail_units = (static_cast<long long>(n_wtiles) - tail0) * B_;
    u = tail_units * cid_ / K_;
    hi = tail_units * (cid_ + 1) / K_;
  }
  // the last segment of the remaining tail range [u, hi)
  __device__ __forceinline__ void tail_seg(int& wt, int& bb, int& be) {
    const long long t0 = ((hi - 1) / B) * B;  // first unit of the tile holding the range's last unit
    const long long s0 = t0 > u ? t0 : u;
    wt = static_cast<int>(tail0 + (hi - 1) / B);
    bb = static_cast<int>(s0 - t0);
    be = static_cast<int>(hi - t0);
    hi = s0;
  }
  __device__ __forceinline__ bool next(int& wt, int& bb, int& be) {
    if (phase == 0) {  // the tile this cluster opens goes first: its rows are published early
      phase = 1;
      if (u < hi && ((hi - 1) / B) * B >= u) {
        tail_seg(wt, bb, be);
        return true;
      }
    }
    if (w < waves) {
      wt = w * K + cid;
      bb = 0;
      be = B;
      ++w;
      return true;
    }
    if (u >= hi) return false;
    tail_seg(wt, bb, be);
    return true;
  }
};

// Carried deferred finalize (FinJob): this CTA's contiguous slice of the float4
// index space, handed out in warp-sized chunks of 32 x kFinU float4 through a
// shared-memory counter to whichever worker warp is idle (the noise warps all
// the time, the epilogue warps while they wait for a TMEM buffer). Streaming
// loads / stores (evict-first) keep the GEMM operands in L2. No per-warp state
// lives across the epilogue's tile work (the job is read from the kernel
// parameters, the clip factor and the noise key from shared memory), so the
// accumulator registers are untouched.
constexpr int kFinU = 4;
constexpr int kFinPf = 24;  // chunks prefetched ahead into L2 (48 KB per CTA in flight)
struct FinShared {
  unsigned ctr;       // next chunk
  unsigned ready;     // factor + key published
  float f;            // clip factor x mean scale
  unsigned pad;
  uint64_t base, base_g;
};

// fixed-order fp64 sum of the partials (the same factor in every CTA); the key of a
// device step counter is absorbed once. Every warp may call it: identical results.
__device__ __forceinline__ void fin_setup(const FinJob& j, FinShared* fs, int lane) {
  double t = 0.0;
  for (int i = lane; i < j.n_parts; i += 32) t += static_cast<double>(j.part[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) {
    const double cf = (t <= j.clip_c2) ? 1.0 : j.clip_c / sqrt(t);  // dpcore.py:41-47
    uint64_t base = j.base, base_g = j.base_g;
    if (j.add_noise && j.step_ptr) {
      base = absorb3(j.seed_u, j.layer_u, static_cast<uint64_t>(*j.step_ptr));
      base_g = base + kGamma;
    }
    fs->f = static_cast<float>(cf) * j.inv_batch;
    fs->base = base;
    fs->base_g = base_g;
    __threadfence_block();
    atomicExch(&fs->ready, 1u);
    if (blockIdx.x == 0 && threadIdx.x == 64 && j.norms_out) j.norms_out[0] = static_cast<float>(t);
  }
  __syncwarp();
}

// one chunk for the calling warp; false when this CTA's slice is exhausted
__device__ __forceinline__ bool fin_chunk(const FinJob& j, FinShared* fs, int lane) {
  unsigned k = 0;
  if (lane == 0) k = atomicAdd(&fs->ctr, 1u);
  k = __shfl_sync(0xffffffffu, k, 0);
  const long long n4 = j.n >> 2;
  const long long lo = n4 * blockIdx.x / gridDim.x, hi = n4 * (blockIdx.x + 1) / gridDim.x;
  const long long s0 = lo + static_cast<long long>(k) * (32 * kFinU);
  if (s0 >= hi) return false;
  if (lane == 0) {  // keep DRAM busy ahead of the workers: the chunk kFinPf claims from now into L2
    const long long pf = s0 + static_cast<long long>(kFinPf) * (32 * kFinU);
    if (pf < hi) {
      const long long e = pf + 32 * kFinU < hi ? pf + 32 * kFinU : hi;
      prefetch_l2_bulk_evict_first(reinterpret_cast<const float4*>(j.g) + pf, static_cast<uint32_t>((e - pf) * 16));
    }
  }
  if (!*reinterpret_cast<volatile unsigned*>(&fs->ready)) fin_setup(j, fs, lane);
  const float f = fs->f;
  const uint64_t base = fs->base, base_g = fs->base_g;
  const int mode = (!j.add_noise || j.hi <= j.lo) ? 2 : (j.impl == 2 && j.lo <= 0 && j.hi >= j.n) ? 1 : 0;
  float4* g4 = reinterpret_cast<float4*>(j.g);
  float4 v[kFinU];
#pragma unroll
  for (int u = 0; u < kFinU; ++u) {
    const long long i = s0 + u * 32 + lane;
    if (i < hi) v[u] = __ldcs(g4 + i);
  }
#pragma unroll
  for (int u = 0; u < kFinU; ++u) {
    const long long i = s0 + u * 32 + lane;
    if (i >= hi) continue;
    // explicit roundings (c * G, then one fma with the noise): bitwise the standalone pass
    float4 r = make_float4(__fmul_rn(v[u].x, f), __fmul_rn(v[u].y, f), __fmul_rn(v[u].z, f),
                           __fmul_rn(v[u].w, f));
    if (mode == 1) {
      const float4 z = philox_normal4(base, static_cast<uint64_t>(i));
      r.x = __fmaf_rn(j.scale, z.x, r.x);
      r.y = __fmaf_rn(j.scale, z.y, r.y);
      r.z = __fmaf_rn(j.scale, z.z, r.z);
      r.w = __fmaf_rn(j.scale, z.w, r.w);
    } else if (mode == 0) {
      const long long e = i << 2;
      if (e + 3 >= j.lo && e < j.hi) {
        const float4 z = j.impl == 2 ? philox_normal4(base, static_cast<uint64_t>(i))
                                     : noise_draw4(j.impl, base_g, base, static_cast<uint64_t>(i));
        if (e + 0 >= j.lo && e + 0 < j.hi) r.x = __fmaf_rn(j.scale, z.x, r.x);
        if (e + 1 >= j.lo && e + 1 < j.hi) r.y = __fmaf_rn(j.scale, z.y, r.y);
        if (e + 2 >= j.lo && e + 2 < j.hi) r.z = __fmaf_rn(j.scale, z.z, r.z);
        if (e + 3 >= j.lo && e + 3 < j.hi) r.w = __fmaf_rn(j.scale, z.w, r.w);
      }
    }
    __stcs(g4 + i, r);
  }
  return true;
}

// Tile raster: work tile wt -> (row block r, column tile c). swz <= 1: row-major (a
// wave of K consecutive tiles spans ~K/n_pt row blocks and EVERY column tile, so the
// whole X operand streams through L2 once per wave). swz = G > 1: grouped raster --
// G row blocks walked column by column, so a wave covers a compact G x (K/G) block
// of tiles and its operand rows / columns are re-read from L2 instead of DRAM.
__device__ __forceinline__ void tile_rc(int wt, int n_rows, int n_pt, int swz, int& r, int& c) {
  if (swz <= 1) {
    r = wt / n_pt;
    c = wt - r * n_pt;
    return;
  }
  const int per_group = swz * n_pt;
  const int grp = wt / per_group;
  const int first = grp * swz;
  const int rows_in = n_rows - first < swz ? n_rows - first : swz;
  const int local = wt - grp * per_group;
  c = local / rows_in;
  r = first + (local - c * rows_in);
}

// MC = 2: a 4-CTA cluster holds two CTA pairs working on vertically adjacent pair
// tiles (same X columns, consecutive dY row blocks) in lockstep; each X box is
// loaded once and multicast to the CTA of both pairs that needs it, so L2 serves
// 3/4 of the operand bytes of two independent pairs. A stage is refilled only
// after BOTH pairs' MMAs released it (every commit arrives in all four CTAs).
// wait-time accounting of one role's thread (FDP_STREAM_TRACE; timing experiments only)
struct WaitClock {
  unsigned long long* slot;
  unsigned long long acc = 0;
  __device__ __forceinline__ explicit WaitClock(unsigned long long* s) : slot(s) {}
  __device__ __forceinline__ uint64_t start() const { return slot ? globaltimer_ns() : 0; }
  __device__ __forceinline__ void stop(uint64_t t0) {
    if (slot) acc += globaltimer_ns() - t0;
  }
  __device__ __forceinline__ void flush() const {
    if (slot) *slot = acc;
  }
};

template <int BN, int CG, int MC, bool FIN>
__global__ void __launch_bounds__(kTcThreads, 1)
    dpdw_stream_kernel(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_x,
                       const __grid_constant__ CUtensorMap tm_gw, const StreamParams p) {
  using C = SCfg<BN, CG>;
  constexpr int CL = CG * MC;  // CTAs per cluster
  // a PDL-launched successor (the single-sample finalize / clip factor) may queue up now;
  // it waits for this grid's completion before it reads anything
  if (threadIdx.x == 0) pdl_launch_dependents();
  static_assert(MC == 1 || (CG == 2 && C::kBCols / 64 == MC), "multicast: one X box per pair");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + C::kStages * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + C::kStgBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kNBuf;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + C::kNBuf);
  float* red = reinterpret_cast<float*>(tmem_holder + 4);  // [kEpiWarps] tile sum-of-squares partials
  FinShared* fin_sh = reinterpret_cast<FinShared*>(
      (reinterpret_cast<uintptr_t>(red + kEpiWarps) + 15) & ~uintptr_t(15));  // carried finalize state
  // carried finalize: a separate instantiation, so the plain kernels keep their register allocation
  const bool fin_on = FIN && p.fin.g != nullptr;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned* err = p.ctrl + 1;
  const int crank = CL > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int rank = crank % CG;  // CTA within its pair
  const int pi = crank / CG;    // pair within the cluster
  const bool leader = rank == 0;
  const int cid = blockIdx.x / CL, n_clusters = gridDim.x / CL;
  const bool per_unit = p.reweight != 0;  // one TMEM accumulation per sample (scaled by c_b) vs per segment
  // work tiles: MC pair tiles stacked along D (rows past D load zeros and are never stored)
  const int n_wt_real = MC == 1 ? p.n_wtiles : ((p.n_wtiles / p.n_pt + MC - 1) / MC) * p.n_pt;
  // spill: virtual work tiles (sample-major) of one unit each: wt' = b * n_wt_real + wt
  const bool spill = MC == 1 && p.spill != 0;
  const int n_wt = spill ? n_wt_real * p.B : n_wt_real;
  const int walk_B = spill ? 1 : p.B;
  const uint16_t pair_mask = static_cast<uint16_t>(((1u << CG) - 1u) << (CG * pi));
#ifdef FDP_STREAM_TRACE_ON  // timing experiments (build with -DFDP_STREAM_TRACE_ON, run with FDP_STREAM_TRACE=1)
  unsigned long long* trace = p.trace ? p.trace + blockIdx.x * 8 : nullptr;
#else
  constexpr unsigned long long* trace = nullptr;
#endif
  const uint64_t t_start = trace ? globaltimer_ns() : 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // MC == 2: the commits of both pairs
    }
    for (int s = 0; s < C::kNBuf; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CG);
    }
    fin_sh->ctr = 0u;
    fin_sh->ready = 0u;
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
  if constexpr (CL > 1) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // Philox noise drawn into the accumulator of a tile's first segment (the whole tile,
  // or the split tile's first samples) by the 256 epilogue threads, instead of a
  // pre-fill by the two noise warps that every later segment of the tile waits for
  const bool epi_noise = p.add_noise && p.epi_noise && p.noise_impl == 2;
  // epi_init: the noise, if any, is drawn by the epilogue. A split tile then needs no
  // pre-fill: when accumulating every segment reduce-adds; otherwise the tile's
  // opening segment (samples from 0) stores plainly and publishes the rows through
  // the tile counter, and the continuing segments reduce-add after it.
  const bool epi_init = !p.add_noise || epi_noise;
  // does tile (split or whole) get its rows initialised by a noise-warp pre-fill?
  auto tile_prefilled = [&](bool whole) {
    return whole ? (p.add_noise && !epi_noise) : (!epi_init && (!p.accumulate || p.add_noise));
  };

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      WaitClock wc(trace ? trace + 0 : nullptr);
      SegWalk w(cid, n_clusters, walk_B, n_wt);
      int wt, bb, be;
      while (w.next(wt, bb, be)) {
        const int sb = spill ? wt / n_wt_real : 0;  // spill: the unit's sample
        if (spill) {
          wt -= sb * n_wt_real;
          bb = sb;
          be = sb + 1;
        }
        int tr, tc;
        tile_rc(wt, n_wt_real / p.n_pt, p.n_pt, p.swizzle, tr, tc);
        const int d0 = (tr * CL + crank) * kBM;
        const int p0 = tc * BN + rank * C::kBCols;
        for (int b = bb; b < be; ++b) {
          for (int kb = 0; kb < p.n_kb; ++kb) {
            const uint64_t tw = wc.start();
            mbar_wait(&empty[stage], phase ^ 1, err, p.budget_ns, 0x501);
            wc.stop(tw);
            uint8_t* sa = smem + stage * C::kStageBytes;
            uint8_t* sb = sa + C::kABytes;
            if constexpr (MC == 2) {  // own dY rows; X box `pi` multicast to this rank's CTA of both pairs
              if (leader) mbar_arrive_expect_tx(&full[stage], C::kStageBytes * CG);
              tma_load_3d_pair(sa, &tm_dy, &full[stage], d0, kb * kBK, b);
              tma_load_3d_pair(sa + 8192, &tm_dy, &full[stage], d0 + 64, kb * kBK, b);
              tma_load_3d_pair_mc(sb + pi * 8192, &tm_x, &full[stage], p0 + 64 * pi, kb * kBK, b,
                                  static_cast<uint16_t>((1u << rank) | (1u << (CG + rank))));
            } else if constexpr (CG == 2) {
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
      wc.flush();
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA) =======================
    if (lane == 0 && leader) {
      uint32_t stage = 0, phase = 0, buf = 0, tphase = 0;
      WaitClock wt_e(trace ? trace + 1 : nullptr), wt_f(trace ? trace + 2 : nullptr);
      SegWalk w(cid, n_clusters, walk_B, n_wt);
      int wt, bb, be;
      while (w.next(wt, bb, be)) {
        for (int ub = bb; ub < be; ub += per_unit ? 1 : (be - bb)) {
          const int ue = per_unit ? ub + 1 : be;
          const uint64_t t0 = wt_e.start();
          mbar_wait(&tempty[buf], tphase ^ 1, err, p.budget_ns, 0x502);
          wt_e.stop(t0);
          tc_fence_after();
          const uint32_t dtm = tmem_base + buf * BN;
          uint32_t accum = 0;
          for (int b = ub; b < ue; ++b) {
            for (int kb = 0; kb < p.n_kb; ++kb) {
              const uint64_t t1 = wt_f.start();
              mbar_wait(&full[stage], phase, err, p.budget_ns, 0x503);
              wt_f.stop(t1);
              tc_fence_after();
              const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
              const uint32_t b_base = a_base + C::kABytes;
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k) {
                const uint64_t ad = make_sdesc_sw128(a_base + k * 2048, 8192, 1024);
                const uint64_t bd = make_sdesc_sw128(b_base + k * 2048, 8192, 1024);
                if (p.dbg & 2) continue;
                if constexpr (CG == 2) tc_mma_f16_pair(dtm, ad, bd, C::kIdesc, accum);
                else tc_mma_f16(dtm, ad, bd, C::kIdesc, accum);
                accum = 1;
              }
              if constexpr (MC == 2) tc_commit_pair_mask(&empty[stage], 0xF);
              else if constexpr (CG == 2) tc_commit_pair(&empty[stage]);
              else tc_commit(&empty[stage]);
              if (++stage == C::kStages) { stage = 0; phase ^= 1; }
            }
          }
          if constexpr (MC == 2) tc_commit_pair_mask(&tfull[buf], pair_mask);
          else if constexpr (CG == 2) tc_commit_pair(&tfull[buf]);
          else tc_commit(&tfull[buf]);
          if (++buf == C::kNBuf) { buf = 0; tphase ^= 1; }
        }
      }
      wt_e.flush();
      wt_f.flush();
    }
  } else if (warp == 2 || warp == 3) {
    // ======================= noise warps: initialise the rows of tiles this cluster opens =======================
    // Runs ahead of the epilogue (rows of different tiles are disjoint); each
    // initialisation is published through the CTA tile's counter.
    const int ntid = (warp - 2) * 32 + lane;
    uint64_t kb = p.key_base, kbg = p.key_base_g;
    if (p.step_ptr) {
      kb = absorb3(p.seed_u, p.layer_u, static_cast<uint64_t>(*p.step_ptr));
      kbg = kb + kGamma;
    }
    SegWalk w(cid, n_clusters, walk_B, n_wt);
    int wt, bb, be;
    while (w.next(wt, bb, be)) {
      const bool whole = bb == 0 && be == walk_B;
      if (spill || bb != 0 || !tile_prefilled(whole)) continue;  // spill units are whole, stored unscaled
      int tr, tc;
      tile_rc(wt, n_wt_real / p.n_pt, p.n_pt, p.swizzle, tr, tc);
      const int d0 = (tr * CL + crank) * kBM;
      const int p0 = tc * BN;
      prefill_rows<BN>(p.grad_w, p.D, p.P, d0, d0 + kBM, p0, p.accumulate != 0, p.add_noise && !epi_noise, p.noise_impl,
                       kbg, kb, p.noise_scale, p.noise_lo, p.noise_hi, ntid);
      __threadfence();
      named_bar_sync(3, 64);
      if (ntid == 0) red_release_add_u32(&p.tile_cnt[wt * CL + crank], 1u);
    }
    if (fin_on) {  // the carried finalize of the previous layer, for as long as work is left
      if (warp == 2) {
        if (lane == 0) {  // the first kFinPf chunks of this CTA's slice into L2
          const long long n4 = p.fin.n >> 2;
          const long long lo = n4 * blockIdx.x / gridDim.x, hi = n4 * (blockIdx.x + 1) / gridDim.x;
          const long long e = lo + static_cast<long long>(kFinPf) * 32 * kFinU < hi
                                  ? lo + static_cast<long long>(kFinPf) * 32 * kFinU : hi;
          for (long long a = lo; a < e; a += 32 * kFinU) {
            const long long b = a + 32 * kFinU < e ? a + 32 * kFinU : e;
            prefetch_l2_bulk_evict_first(reinterpret_cast<const float4*>(p.fin.g) + a, static_cast<uint32_t>((b - a) * 16));
          }
        }
        fin_setup(p.fin, fin_sh, lane);  // CTA 0's also writes the layer's ||G||^2
      }
      while (fin_chunk(p.fin, fin_sh, lane)) {
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ======================= epilogue =======================
    // PDL launch: the clip factors come from the grid before us (the factor reduce);
    // producer and MMA warps (inputs only) run ahead while it finishes
    if (p.pdl) pdl_wait();
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3, half = ew >> 2, etid = ew * 32 + lane;
    const int row = q * 32 + lane, col0 = half * C::kCPT;
    uint64_t nkb = p.key_base;
    if (epi_noise && p.step_ptr) nkb = absorb3(p.seed_u, p.layer_u, static_cast<uint64_t>(*p.step_ptr));
    uint32_t rbuf = 0, rph = 0;
    WaitClock wc_t(trace && etid == 0 ? trace + 3 : nullptr), wc_c(trace && etid == 0 ? trace + 4 : nullptr),
        wc_s(trace && etid == 0 ? trace + 5 : nullptr);
    bool fin_left = fin_on && p.fin_epi;
    SegWalk w(cid, n_clusters, walk_B, n_wt);
    int wt, bb, be;
    while (w.next(wt, bb, be)) {
      if (fin_left) {  // idle until this segment's first accumulator is complete: stream the carried finalize
        const uint32_t a = smem_u32(&tfull[rbuf]);
        while (!__any_sync(0xffffffffu, mbar_try_wait(a, rph))) {  // warp-uniform exit
          if (!fin_chunk(p.fin, fin_sh, lane)) {
            fin_left = false;
            break;
          }
        }
      }
      const bool whole = bb == 0 && be == walk_B;
      const int tile = wt * CL + crank;  // spill: (b * n_wtiles + wt) * CL + crank, the unit's partial slot
      const int sb = spill ? wt / n_wt_real : 0;
      if (spill) wt -= sb * n_wt_real;
      int tr, tc;
      tile_rc(wt, n_wt_real / p.n_pt, p.n_pt, p.swizzle, tr, tc);
      const int d0 = (tr * CL + crank) * kBM;
      const int p0 = tc * BN;
      float acc[C::kCPT];
#pragma unroll
      for (int i = 0; i < C::kCPT; ++i) acc[i] = 0.0f;
      if (epi_noise) {
        // the tile's Philox noise starts the accumulators (rank slice only), split over the
        // tile's segments by column quads in proportion to their samples: every quad is
        // drawn once, and the drawing is spread like the units (a split tile's first
        // cluster no longer draws the whole tile while the others wait)
        const int q_lo = (C::kCPT / 4) * bb / walk_B, q_hi = (C::kCPT / 4) * be / walk_B;
        const long long frow = static_cast<long long>(d0 + row) * p.P;
        const bool row_ok = d0 + row < p.D;
#pragma unroll
        for (int q4 = 0; q4 < C::kCPT / 4; ++q4) {
          const int col = p0 + col0 + 4 * q4;
          const long long f = frow + col;
          if (q4 >= q_lo && q4 < q_hi && row_ok && col < p.P && f + 3 >= p.noise_lo &&
              f < p.noise_hi) {  // P % 8 == 0: quads stay in a row
            const float4 n = philox_normal4(nkb, static_cast<uint64_t>(f >> 2));
            acc[4 * q4 + 0] = (f + 0 >= p.noise_lo && f + 0 < p.noise_hi) ? p.noise_scale * n.x : 0.0f;
            acc[4 * q4 + 1] = (f + 1 >= p.noise_lo && f + 1 < p.noise_hi) ? p.noise_scale * n.y : 0.0f;
            acc[4 * q4 + 2] = (f + 2 >= p.noise_lo && f + 2 < p.noise_hi) ? p.noise_scale * n.z : 0.0f;
            acc[4 * q4 + 3] = (f + 3 >= p.noise_lo && f + 3 < p.noise_hi) ? p.noise_scale * n.w : 0.0f;
          }
        }
      }
      // the next unit's clip factor is loaded one unit ahead: its L2 latency overlaps
      // this unit's TMEM readout instead of sitting between the buffer wait and the FMAs
      float f_next = per_unit ? __ldg(p.factors_in + bb) : 1.0f;
      for (int ub = bb; ub < be; ub += per_unit ? 1 : (be - bb)) {
        const float f = f_next;
        if (per_unit && ub + 1 < be) f_next = __ldg(p.factors_in + ub + 1);
        const uint64_t tw = wc_t.start();
        mbar_wait(&tfull[rbuf], rph, err, p.budget_ns, 0x504);
        wc_t.stop(tw);
        tc_fence_after();
        const uint32_t buf = rbuf;
        if (++rbuf == C::kNBuf) { rbuf = 0; rph ^= 1; }
        const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * BN + col0;
        if (p.dbg & 1) {
        } else if constexpr (C::kCPT <= 64) {  // 128-column tiles: registers allow 32 columns per TMEM round trip
#pragma unroll
          for (int c = 0; c < C::kCPT / 32; ++c) {
            float v[32];
            tmem_ld32(tb + c * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[c * 32 + i] = fmaf(f, v[i], acc[c * 32 + i]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < C::kCPT / 16; ++c) {
            float v[16];
            tmem_ld16(tb + c * 16, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[c * 16 + i] = fmaf(f, v[i], acc[c * 16 + i]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_leader(&tempty[buf]);
          else mbar_arrive(&tempty[buf]);
        }
      }
      if (p.norm_part) {  // single-sample path: this CTA tile's ||G||^2 partial (tiles are whole)
        float sq = 0.0f;
#pragma unroll
        for (int i = 0; i < C::kCPT; ++i) sq = fmaf(acc[i], acc[i], sq);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) red[ew] = sq;
        named_bar_sync(1, 32 * kEpiWarps);
        if (etid == 0) {
          float t = 0.0f;
#pragma unroll
          for (int k = 0; k < kEpiWarps; ++k) t += red[k];
          p.norm_part[tile] = t;
        }
      }
      // ---- finalize: reduce-add onto initialised rows (split tiles, accumulation,
      // pre-filled noise) or plain store; 32-column boxes, double-buffered
      const bool split_init = epi_init && !whole && !p.accumulate && !spill;  // opening store / continuations
      const bool opening = split_init && bb == 0;
      const bool rmw = !opening && (!whole || p.accumulate || (p.add_noise && !epi_noise));
      if ((tile_prefilled(whole) || (split_init && bb != 0)) && etid == 0) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_u32(&p.tile_cnt[tile]) < 1u) {
          if (globaltimer_ns() - t0 > p.budget_ns) watchdog_trap(err, 0x505);
          __nanosleep(64);
        }
        if (trace) wc_c.acc += globaltimer_ns() - t0;
      }
      const uint64_t ts = wc_s.start();
#pragma unroll
      for (int c = 0; c < C::kCPT / 32; ++c) {
        uint8_t* sbuf = stg + (c & 1) * (2 * kBM * 128);
        if (etid == 0) bulk_wait_read_le1();
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
            if (spill) tma_store_3d(&tm_gw, sbuf + h * (kBM * 128), col, d0, sb);  // G[b], unscaled
            else if (rmw) tma_reduce_add_2d(&tm_gw, sbuf + h * (kBM * 128), col, d0);
            else tma_store_2d(&tm_gw, sbuf + h * (kBM * 128), col, d0);
          }
          bulk_commit();
        }
      }
      if (opening && etid == 0) {  // the rows are initialised once this segment's stores have landed
        bulk_wait_all();
        fence_proxy_async_global();
        __threadfence();
        red_release_add_u32(&p.tile_cnt[tile], 1u);
      }
      wc_s.stop(ts);
    }
    while (fin_left && fin_chunk(p.fin, fin_sh, lane)) {
    }
    if (etid == 0) bulk_wait_all();
    wc_t.flush();
    wc_c.flush();
    wc_s.flush();
    if (trace && etid == 0) trace[6] = globaltimer_ns() - t_start;  // the epilogue's last store drained
  }

  tc_fence_before();
  if constexpr (CL > 1) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (CG == 2) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
  if (trace && threadIdx.x == 0) trace[7] = globaltimer_ns() - t_start;
  if (threadIdx.x == 0) {  // last CTA out re-arms the tile counters
    __threadfence();
    const unsigned old = atomicAdd(&p.ctrl[0], 1u);
    if (old == gridDim.x - 1) {
      __threadfence();
      if (!spill)  // spill units are whole tiles: their counters are never touched
        for (int t = 0; t < n_wt * CL; ++t) p.tile_cnt[t] = 0u;
      p.ctrl[0] = 0u;
      __threadfence();
    }
  }
}

template <int BN, int CG, int MC, bool FIN>
static cudaError_t launch_stream_impl(const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const CUtensorMap& tm_gw,
                                      const StreamParams& p, int grid, cudaStream_t stream) {
  using C = SCfg<BN, CG>;
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(dpdw_stream_kernel<BN, CG, MC, FIN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(C::kSmem));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) done[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CG * MC > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG * MC;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (p.pdl) {  // programmatic dependent of the factor reduce: CTAs start as SMs free up
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  // Split tiles wait on the cluster that initialises them, which is resident:
  // the grid never exceeds the co-resident capacity (host planner).
  return cudaLaunchKernelEx(&cfg, dpdw_stream_kernel<BN, CG, MC, FIN>, tm_dy, tm_x, tm_gw, p);
}

template <bool FIN>
static cudaError_t launch_stream_fin(int bn, int cg, const CUtensorMap& tm_dy, const CUtensorMap& tm_x,
                                     const CUtensorMap& tm_gw, const StreamParams& p, int grid, cudaStream_t stream) {
  if (cg == 2) {
    if (bn == 256) {
      if (p.mc == 2) return launch_stream_impl<256, 2, 2, FIN>(tm_dy, tm_x, tm_gw, p, grid, stream);
      return launch_stream_impl<256, 2, 1, FIN>(tm_dy, tm_x, tm_gw, p, grid, stream);
    }
    return launch_stream_impl<128, 2, 1, FIN>(tm_dy, tm_x, tm_gw, p, grid, stream);
  }
  if (bn == 256) return launch_stream_impl<256, 1, 1, FIN>(tm_dy, tm_x, tm_gw, p, grid, stream);
  return launch_stream_impl<128, 1, 1, FIN>(tm_dy, tm_x, tm_gw, p, grid, stream);
}

cudaError_t launch_stream(int bn, int cg, const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const CUtensorMap& tm_gw,
                          const StreamParams& p, int grid, cudaStream_t stream) {
  if (p.fin.g) return launch_stream_fin<true>(bn, cg, tm_dy, tm_x, tm_gw, p, grid, stream);
  return launch_stream_fin<false>(bn, cg, tm_dy, tm_x, tm_gw, p, grid, stream);
}

// Co-resident 4-CTA clusters of the multicast variant (0 if it cannot launch).
int stream_mc_max_clusters() {
  static int cache[64];
  static bool have[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  if (have[dev]) return cache[dev];
  using C = SCfg<256, 2>;
  int n = 0;
  if (cudaFuncSetAttribute(dpdw_stream_kernel<256, 2, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(C::kSmem)) == cudaSuccess) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4 * sms);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 4;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, dpdw_stream_kernel<256, 2, 2, false>, &cfg) != cudaSuccess) n = 0;
  }
  (void)cudaGetLastError();
  cache[dev] = n;
  have[dev] = true;
  return n;
}

}  // namespace fdp
