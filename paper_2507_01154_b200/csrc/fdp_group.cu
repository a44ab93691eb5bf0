// fdp_group.cu -- the fused DP weight-gradient backward of a LIST of layers in one
// persistent cooperative launch.
//
// Same per-layer algorithm as dpdw_tc_kernel's MODE_FUSED (Algorithm 1,
// PAPER.md:109-137; workflows.py:340-421), but the TMA producer, the MMA issuer,
// the noise warps and the epilogue all walk the layer list in the same order,
// so the pipelines never drain between layers: layer l+1's operand loads and
// first MMAs run while layer l's epilogue finishes its last norm all-reduce and
// its TMA stores. Every layer keeps its own tagged norm-partial slots and tile
// counters; a CTA whose cluster id is beyond a layer's work simply skips it.
// Layer descriptors (with their TMA maps) are a __grid_constant__ parameter
// block, so the launch is CUDA-graph capturable with no host->device copy.
//
// Layer packing: layer l occupies the cluster range [c_off, c_off + n_wtiles *
// groups) (mod the cluster count); the host planner packs small layers next to
// each other (e.g. GPT-2's c_attn on 54 clusters and attn_proj on the other 18),
// so every cluster carries the same number of sample units per step. Norm
// all-reduces only couple the clusters of one layer.
//
// The noise warps run ahead of the epilogue across layers (the layers' grad_w
// rows are disjoint); a shared-memory counter tells the epilogue which layers'
// pre-fills are complete.
#include <cstdio>
#include <cstdlib>

#include "fdp_internal.h"
#include "fdp_ptx.cuh"
#include "fdp_prefill.cuh"
#include "fdp_rng.cuh"

namespace fdp {

// NSTG: store-staging buffers (2 = double-buffered 32-column box pairs; 1 = one
// buffer, whose 32 KB become a sixth operand stage at BN 256, CG 2: FDP_GROUP_STG1)
template <int BN, int CG, int NSTG = 2>
struct GCfg {
  static constexpr int kBCols = BN / CG;
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = kBCols * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStgBytes = NSTG * 2 * kBM * 128;  // NSTG buffers x two 32-column fp32 boxes (column halves)
  static constexpr int kStages = (232448 - 2048 - kStgBytes) / kStageBytes;
  static constexpr int kNBuf = 512 / BN;
  static constexpr int kCPT = BN / 2;
  static constexpr int kBarBytes = 1024;
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes + kStgBytes + kBarBytes;
  static constexpr uint32_t kIdesc = make_idesc_bf16_mn(kBM * CG, BN);
};

#define GTRACE(slot)                                                                                 \
  do {                                                                                               \
    if (gp.trace && etid == 0 && (slot) < 256) gp.trace[blockIdx.x * 256 + (slot)] = globaltimer_ns(); \
  } while (0)

template <int BN, int CG, int NSTG>
__global__ void __launch_bounds__(kTcThreads, 1) dpdw_group_kernel(const __grid_constant__ GroupParams gp) {
  using C = GCfg<BN, CG, NSTG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + C::kStages * C::kStageBytes;  // 1024-aligned: two 16 KB swizzled boxes
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + C::kStgBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + C::kNBuf;
  uint64_t* pair_bar = tempty + C::kNBuf;  // CG == 2: the follower's norm partial has landed (leader)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(pair_bar + 1);
  float* red = reinterpret_cast<float*>(tmem_holder + 4);
  float* bcast = red + kEpiWarps;
  volatile unsigned* pf_done = reinterpret_cast<volatile unsigned*>(bcast + 1);  // layers pre-filled so far
  volatile int* ep_layer = reinterpret_cast<volatile int*>(bcast + 2);          // layer the epilogue is on
  float* pair_sx = bcast + 4;  // [2] (leader) the follower CTA's tile partial, by unit parity

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned* err = gp.ctrl + 1;
  const int rank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;
  const bool leader = rank == 0;
  const int cid = blockIdx.x / CG;
  const int n_clusters = static_cast<int>(gridDim.x) / CG;
  // this cluster's index within layer L's cluster range (>= L.n_wtiles * L.groups: idle)
  auto lcid = [&](const GLayer& L) {
    const int c = cid - L.c_off;
    return c < 0 ? c + n_clusters : c;
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kNBuf; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CG);
    }
    mbar_init(pair_bar, 1);
    *pf_done = 0u;
    *ep_layer = 0;
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair<512>(tmem_holder);
    else tmem_alloc<512>(tmem_holder);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  unsigned tag = __ldcg(gp.ctrl + 2) + 1u;
  if (tag == 0u) tag = 1u;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int l = 0; l < gp.n_layers; ++l) {
        const GLayer& L = gp.L[l];
        const int lc = lcid(L);
        if (lc >= L.n_wtiles * L.groups) continue;
        const int wt = lc % L.n_wtiles, group = lc / L.n_wtiles;
        const int d0 = ((wt / L.n_pt) * CG + rank) * kBM;
        const int p0 = (wt % L.n_pt) * BN + rank * C::kBCols;
        for (int b = group; b < L.B; b += L.groups) {
          for (int kb = 0; kb < L.n_kb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1, err, gp.budget_ns, 0x401);
            uint8_t* sa = smem + stage * C::kStageBytes;
            uint8_t* sb = sa + C::kABytes;
            if constexpr (CG == 2) {
              if (leader) mbar_arrive_expect_tx(&full[stage], C::kStageBytes * CG);
              tma_load_3d_pair(sa, &L.tm_dy, &full[stage], d0, kb * kBK, b);
              tma_load_3d_pair(sa + 8192, &L.tm_dy, &full[stage], d0 + 64, kb * kBK, b);
#pragma unroll
              for (int j = 0; j < C::kBCols / 64; ++j)
                tma_load_3d_pair(sb + j * 8192, &L.tm_x, &full[stage], p0 + 64 * j, kb * kBK, b);
            } else {
              mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
              tma_load_3d(sa, &L.tm_dy, &full[stage], d0, kb * kBK, b);
              tma_load_3d(sa + 8192, &L.tm_dy, &full[stage], d0 + 64, kb * kBK, b);
#pragma unroll
              for (int j = 0; j < C::kBCols / 64; ++j)
                tma_load_3d(sb + j * 8192, &L.tm_x, &full[stage], p0 + 64 * j, kb * kBK, b);
            }
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA) =======================
    if (lane == 0 && leader) {
      uint32_t stage = 0, phase = 0, buf = 0, tphase = 0;
      // FDP_FLAG_TRACE: where the MMA issuer waits (ns): on a TMEM buffer (epilogue
      // behind) and on operand stages (TMA behind); slots 248-251 of the CTA's row
      const bool tr = gp.trace != nullptr;
      uint64_t w_tmem = 0, w_full = 0, t_first = 0, units = 0;
      for (int l = 0; l < gp.n_layers; ++l) {
        const GLayer& L = gp.L[l];
        const int lc = lcid(L);
        if (lc >= L.n_wtiles * L.groups) continue;
        const int group = lc / L.n_wtiles;
        for (int b = group; b < L.B; b += L.groups) {
          uint64_t t0 = tr ? globaltimer_ns() : 0;
          if (tr && !t_first) t_first = t0;
          mbar_wait(&tempty[buf], tphase ^ 1, err, gp.budget_ns, 0x402);
          if (tr) w_tmem += globaltimer_ns() - t0;
          ++units;
          tc_fence_after();
          const uint32_t dtm = tmem_base + buf * BN;
          for (int kb = 0; kb < L.n_kb; ++kb) {
            if (tr) t0 = globaltimer_ns();
            mbar_wait(&full[stage], phase, err, gp.budget_ns, 0x403);
            if (tr) w_full += globaltimer_ns() - t0;
            tc_fence_after();
            const uint32_t a_base = smem_u32(smem + stage * C::kStageBytes);
            const uint32_t b_base = a_base + C::kABytes;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t ad = make_sdesc_sw128(a_base + k * 2048, 8192, 1024);
              const uint64_t bd = make_sdesc_sw128(b_base + k * 2048, 8192, 1024);
              if constexpr (CG == 2) tc_mma_f16_pair(dtm, ad, bd, C::kIdesc, (kb | k) != 0);
              else tc_mma_f16(dtm, ad, bd, C::kIdesc, (kb | k) != 0);
            }
            if constexpr (CG == 2) tc_commit_pair(&empty[stage]);
            else tc_commit(&empty[stage]);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
          if constexpr (CG == 2) tc_commit_pair(&tfull[buf]);
          else tc_commit(&tfull[buf]);
          if (++buf == C::kNBuf) { buf = 0; tphase ^= 1; }
        }
      }
      if (tr) {
        unsigned long long* row = gp.trace + blockIdx.x * 256;
        row[248] = w_tmem;
        row[249] = w_full;
        row[250] = globaltimer_ns() - t_first;  // first unit's wait .. last MMA issued
        row[251] = units;
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ======================= noise warps: pre-fill this CTA's grad_w rows =======================
    // (accumulate ? old : 0) + sigma*C*noise, or zeros when only sample groups need
    // initialised rows for their reduce-adds. Runs ahead across layers.
    // Bounded run-ahead: a pre-filled row must still be in L2 when the epilogue's
    // reduce-add of the same row arrives. Unbounded, the two noise warps finish
    // every layer's pre-fill early in the launch and the rows are evicted and
    // re-read (grad_w crosses DRAM three times: 1.245x the algorithmic bytes on
    // the 48-layer GPT-2 step); started with the layer's own epilogue, a row lives
    // in L2 for about one layer's sample units.
    const int ntid = (warp - 2) * 32 + lane;
    for (int l = 0; l < gp.n_layers; ++l) {
      const GLayer& L = gp.L[l];
      const int lc = lcid(L);
      const bool draw = L.add_noise != 0 && gp.dbg_noise != 1;
      if (lc < L.n_wtiles * L.groups && (L.add_noise != 0 || L.groups > 1)) {
        if (gp.pf_ahead >= 0) {
          const uint64_t t0 = globaltimer_ns();
          while (*ep_layer < l - gp.pf_ahead) {
            if (globaltimer_ns() - t0 > gp.budget_ns) watchdog_trap(err, 0x408);
            __nanosleep(256);
          }
        }
        uint64_t kb = L.key_base, kbg = L.key_base_g;
        if (L.step_ptr) {
          kb = absorb3(L.seed_u, L.layer_u, static_cast<uint64_t>(*L.step_ptr));
          kbg = kb + kGamma;
        }
        const int wt = lc % L.n_wtiles, group = lc / L.n_wtiles;
        const int d0 = ((wt / L.n_pt) * CG + rank) * kBM;
        const int p0 = (wt % L.n_pt) * BN;
        const int r0 = group * kBM / L.groups, r1 = (group + 1) * kBM / L.groups;
        prefill_rows<BN>(L.grad_w, L.D, L.P, d0 + r0, d0 + r1, p0, L.accumulate != 0, draw, L.noise_impl, kbg, kb,
                         gp.dbg_noise == 2 ? 0.0f : L.noise_scale, L.noise_lo, L.noise_hi, ntid);
        __threadfence();
        named_bar_sync(3, 64);
        // this group's rows are globally visible: count them right away, so the
        // groups' reduce-adds never wait on another group's epilogue
        if (L.groups > 1 && ntid == 0) red_release_add_u32(&L.tile_cnt[(lc % L.n_wtiles) * CG + rank], 1u);
        if (gp.trace && ntid == 0 && l < 16) gp.trace[blockIdx.x * 256 + 8 * l + 6] = globaltimer_ns();
      }
      if (ntid == 0) *pf_done = static_cast<unsigned>(l + 1);
    }
  } else if (warp >= kEpiWarp0) {
    // ======================= epilogue =======================
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3, half = ew >> 2, etid = ew * 32 + lane;
    const int row = q * 32 + lane, col0 = half * C::kCPT;
    uint32_t rbuf = 0, rph = 0;
    // FDP_PAIR_DSMEM=1 (gp.pair_dsmem): CTA pairs (CG == 2) combine their two tile
    // partials on chip: the follower CTA writes its partial into the leader's shared
    // memory (DSMEM) and release-arrives on the leader's barrier; the leader adds the
    // two in a fixed order and publishes ONE tagged slot per pair tile, so the
    // block-wise all-reduce polls n_wtiles slots per sample instead of n_tiles
    // (north_star (2): warp shuffles -> named barrier -> cluster DSMEM -> grid-level
    // all-reduce in L2). Off by default: the leader's publish now waits for the
    // follower's, an extra on-chip hop on every sample's critical path -- measured
    // 1432 vs 1275 us on the 48-layer GPT-2 step (profiles/r2_pair_dsmem_ab.jsonl);
    // each CTA publishing its own 8-byte slot and every poller summing both is cheaper.
    uint32_t pair_phase = 0;
    const uint32_t pair_bar_leader = CG == 2 ? dsmem_map(pair_bar, 0) : 0u;
    const uint32_t pair_sx_leader = CG == 2 ? dsmem_map(pair_sx, 0) : 0u;
    // pass 1 of sample b's unit in TMEM buffer `buf`: intra-block reduce of
    // ||G_b||^2 over this CTA tile, published as one tagged 8-byte atomic
    auto pass1_publish = [&](const GLayer& Lx, int bx, int tilex, uint32_t bufx) {
      const uint32_t tbx = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + bufx * BN + col0;
      float part = 0.0f;
      if (gp.dbg_tmem != 1) {
#pragma unroll
        for (int c = 0; c < C::kCPT / 16; ++c) {
          float v[16];
          tmem_ld16(tbx + c * 16, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) part = fmaf(v[i], v[i], part);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) red[ew] = part;
      named_bar_sync(1, 32 * kEpiWarps);
      if (etid == 0) {
        float sx = 0.0f;
#pragma unroll
        for (int w = 0; w < kEpiWarps; ++w) sx += red[w];
        if (CG == 2 && gp.pair_dsmem) {
          const uint32_t par = pair_phase & 1u;
          if (rank != 0) {
            dsmem_st_f32(pair_sx_leader + 4u * par, sx);
            mbar_arrive_remote_release(pair_bar_leader);
          } else {
            const uint32_t a = smem_u32(pair_bar);
            const uint64_t t0 = globaltimer_ns();
            while (!mbar_try_wait_cluster(a, par)) {
              if (globaltimer_ns() - t0 > gp.budget_ns) watchdog_trap(err, 0x409);
            }
            const float sp = reinterpret_cast<volatile float*>(pair_sx)[par];
            publish_u64(Lx.tagged + static_cast<long long>(bx) * Lx.n_tiles + tilex / 2,
                        (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(sx + sp), gp.pub_mode);
          }
          ++pair_phase;
        } else {
          publish_u64(Lx.tagged + static_cast<long long>(bx) * Lx.n_tiles + tilex,
                      (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(sx), gp.pub_mode);
        }
      }
    };
    for (int l = 0; l < gp.n_layers; ++l) {
      const GLayer& L = gp.L[l];
      const int lc = lcid(L);
      if (etid == 0) *ep_layer = l;  // releases the noise warps' pre-fill of layers <= l + pf_ahead
      if (lc >= L.n_wtiles * L.groups) continue;
      const int wt = lc % L.n_wtiles, group = lc / L.n_wtiles;
      const int tile = wt * CG + rank;
      const int d0 = ((wt / L.n_pt) * CG + rank) * kBM;
      const int p0 = (wt % L.n_pt) * BN;
      const bool prefill = L.add_noise != 0 || L.groups > 1;
      const bool rmw = prefill || L.accumulate;
      float acc[C::kCPT];
#pragma unroll
      for (int i = 0; i < C::kCPT; ++i) acc[i] = 0.0f;

      bool first = true;
      for (int b = group; b < L.B; b += L.groups) {
        mbar_wait(&tfull[rbuf], rph, err, gp.budget_ns, 0x404);
        tc_fence_after();
        const uint32_t buf = rbuf;
        if (++rbuf == C::kNBuf) { rbuf = 0; rph ^= 1; }
        pass1_publish(L, b, tile, buf);
        if (first && l < 16) GTRACE(8 * l);  // layer l: first sample published
        first = false;
        const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * BN + col0;
        // block-wise all-reduce: fixed-order fp64 sum of the tagged partials
        if (ew == 0) {
          const unsigned long long* slots = L.tagged + static_cast<long long>(b) * L.n_tiles;
          const int n_slots = gp.pair_dsmem ? L.n_tiles / CG : L.n_tiles;  // per pair tile (DSMEM) or CTA tile
          constexpr int kMaxPer = 5;
          unsigned long long v[kMaxPer];
#pragma unroll
          for (int k = 0; k < kMaxPer; ++k) {
            const int i = lane + 32 * k;
            v[k] = i < n_slots ? poll_u64(slots + i, gp.poll_mode) : (static_cast<unsigned long long>(tag) << 32);
          }
          const uint64_t t0 = globaltimer_ns();
          while (true) {  // re-poll every stale slot at once: one L2 round trip per iteration
            bool all = true;
#pragma unroll
            for (int k = 0; k < kMaxPer; ++k) all &= static_cast<unsigned>(v[k] >> 32) == tag;
            if (all || gp.nosync) break;
            if (globaltimer_ns() - t0 > gp.budget_ns) watchdog_trap(err, 0x405);
            if (gp.poll_ns) __nanosleep(gp.poll_ns);
#pragma unroll
            for (int k = 0; k < kMaxPer; ++k)
              if (static_cast<unsigned>(v[k] >> 32) != tag) v[k] = poll_u64(slots + lane + 32 * k, gp.poll_mode);
          }
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < kMaxPer; ++k)
            if (lane + 32 * k < n_slots) s += static_cast<double>(__uint_as_float(static_cast<unsigned>(v[k])));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) {
            *bcast = clip_factor_f(s, L.clip_c, L.clip_c2) * L.inv_batch;  // dpcore.py:41-47
            if (tile == 0) L.norms_out[b] = static_cast<float>(s);
          }
        }
        named_bar_sync(1, 32 * kEpiWarps);
        const float f = *bcast;
        if (gp.dbg_tmem != 2) {
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

      if (l < 16) GTRACE(8 * l + 1);  // layer l: last clip factor applied
      // ---- finalize: wait for the noise warps' pre-fill (and, with sample groups,
      // for every group's pre-fill), then TMA store / reduce-add in 32-column boxes
      if (prefill && etid == 0) {  // this CTA's pre-fill of layer l is complete and visible
        const uint64_t t0 = globaltimer_ns();
        while (*pf_done < static_cast<unsigned>(l + 1)) {
          if (globaltimer_ns() - t0 > gp.budget_ns) watchdog_trap(err, 0x407);
          __nanosleep(32);
        }
        __threadfence();
      }
      if (l < 16) GTRACE(8 * l + 2);
      if (L.groups > 1) {
        if (etid == 0) {  // every group's rows are pre-filled (counted by the noise warps)
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_u32(&L.tile_cnt[tile]) < static_cast<unsigned>(L.groups)) {
            if (globaltimer_ns() - t0 > gp.budget_ns) watchdog_trap(err, 0x406);
            __nanosleep(64);
          }
        }
      }
      if (l < 16) GTRACE(8 * l + 3);
#pragma unroll
      for (int c = 0; c < C::kCPT / 32; ++c) {
        uint8_t* sbuf = stg + (NSTG == 2 ? (c & 1) : 0) * (2 * kBM * 128);
        if (etid == 0) {  // the boxes issued NSTG rounds ago have left this buffer
          if constexpr (NSTG == 2) bulk_wait_read_le1();
          else bulk_wait_read_all();
        }
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
            if (rmw) tma_reduce_add_2d(&L.gw, sbuf + h * (kBM * 128), col, d0);
            else tma_store_2d(&L.gw, sbuf + h * (kBM * 128), col, d0);
          }
          bulk_commit();
        }
        if (l < 16 && c == 0) GTRACE(8 * l + 4);
      }
      if (l < 16) GTRACE(8 * l + 5);  // layer l: stores issued
    }
    if (etid == 0) bulk_wait_all();
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (CG == 2) tmem_dealloc_pair<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned old = atomicAdd(&gp.ctrl[0], 1u);
    if (old == gridDim.x - 1) {
      __threadfence();
      for (int l = 0; l < gp.n_layers; ++l)
        for (int t = 0; t < gp.L[l].n_tiles; ++t) gp.L[l].tile_cnt[t] = 0u;
      unsigned nt = gp.ctrl[2] + 1u;
      if (nt == 0u) nt = 1u;
      gp.ctrl[2] = nt;
      gp.ctrl[0] = 0u;
      __threadfence();
    }
  }
}

template <int BN, int CG, int NSTG = 2>
static cudaError_t launch_group_impl(const GroupParams& gp, int grid, cudaStream_t stream) {
  using C = GCfg<BN, CG, NSTG>;
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(dpdw_group_kernel<BN, CG, NSTG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem));
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
  if (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CG;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (!std::getenv("FDP_NO_COOP")) {  // see fdp_tc.cu
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dpdw_group_kernel<BN, CG, NSTG>, gp);
  // The in-kernel norm all-reduce spin-waits on other CTAs: it needs the
  // co-residency guarantee of the cooperative launch, especially while a
  // collective runs concurrently on other SMs. A rejected cooperative launch is
  // an error (no silent plain-launch retry); FDP_ALLOW_NONCOOP=1 opts into the
  // plain cluster launch (grid <= co-resident capacity; the in-kernel watchdog
  // turns a broken assumption into an error) for profilers that cannot replay
  // cooperative launches.
  if (e != cudaSuccess && CG == 2 && std::getenv("FDP_ALLOW_NONCOOP")) {
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, dpdw_group_kernel<BN, CG, NSTG>, gp);
  }
  return e;
}

// ---- pre-drawn noise (small batches). At B <= 4 the two noise warps' draws bound
// the group launch (48 GPT-2 layers, B = 1: 0.652 ms with noise, 0.370 with a zero
// pre-fill). This grid-wide pass writes every noised layer's sigma C N(d P + p) into
// grad_w with all SMs' warps first; the group launch then reduce-adds onto it
// (accumulate, no draws). Bit for bit the pre-fill path: round(sigma C N) + acc in
// one fp32 add either way. Quads of 4 flat indices (P % 8 == 0); outside [lo, hi)
// (rank partition) the rows are written as zeros.
__global__ void __launch_bounds__(256) k_group_noise(const GroupParams gp) {
  __shared__ long long start[kMaxGroupLayers + 1];
  __shared__ uint64_t kb_s[kMaxGroupLayers], kbg_s[kMaxGroupLayers];
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int l = 0; l < gp.n_layers; ++l) {
      const GLayer& L = gp.L[l];
      start[l] = s;
      if (L.add_noise) s += static_cast<long long>(L.D) * L.P / 4;
      uint64_t kb = L.key_base;
      if (L.step_ptr) kb = absorb3(L.seed_u, L.layer_u, static_cast<uint64_t>(*L.step_ptr));
      kb_s[l] = kb;
      kbg_s[l] = L.step_ptr ? kb + kGamma : L.key_base_g;
    }
    start[gp.n_layers] = s;
  }
  __syncthreads();
  const long long total = start[gp.n_layers];
  int l = 0;
  for (long long q = blockIdx.x * 256LL + threadIdx.x; q < total; q += static_cast<long long>(gridDim.x) * 256) {
    while (q >= start[l + 1]) ++l;  // q only grows: the layer index only moves forward
    const GLayer& L = gp.L[l];
    const long long f = (q - start[l]) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (gp.dbg_noise != 1 && f + 3 >= L.noise_lo && f < L.noise_hi) {
      const float4 n = noise_draw4(L.noise_impl, kbg_s[l], kb_s[l], static_cast<uint64_t>(f >> 2));
      const float sc = gp.dbg_noise == 2 ? 0.0f : L.noise_scale;
      if (f + 0 >= L.noise_lo && f + 0 < L.noise_hi) v.x = __fmul_rn(sc, n.x);
      if (f + 1 >= L.noise_lo && f + 1 < L.noise_hi) v.y = __fmul_rn(sc, n.y);
      if (f + 2 >= L.noise_lo && f + 2 < L.noise_hi) v.z = __fmul_rn(sc, n.z);
      if (f + 3 >= L.noise_lo && f + 3 < L.noise_hi) v.w = __fmul_rn(sc, n.w);
    }
    __stcg(reinterpret_cast<float4*>(L.grad_w + f), v);
  }
}

cudaError_t launch_group_noise(const GroupParams& gp, cudaStream_t stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_group_noise<<<sms * 8, 256, 0, stream>>>(gp);
  return cudaGetLastError();
}

cudaError_t launch_group(int bn, int cg, const GroupParams& gp, int grid, cudaStream_t stream) {
  if (cg == 2) {
    if (bn == 256) {
      const char* v = std::getenv("FDP_GROUP_STG1");  // read per call (A/B tooling)
      const bool stg1 = v && std::atoi(v) != 0;
      return stg1 ? launch_group_impl<256, 2, 1>(gp, grid, stream) : launch_group_impl<256, 2>(gp, grid, stream);
    }
    return launch_group_impl<128, 2>(gp, grid, stream);
  }
  if (bn == 256) return launch_group_impl<256, 1>(gp, grid, stream);
  return launch_group_impl<128, 1>(gp, grid, stream);
}

}  // namespace fdp
