// fdp_ghost.cu -- ghost-norm kernel: per-sample ||G_b||_F^2 without forming G_b.
//
// First phase of the TWO_PHASE path for layers whose per-sample gradient tiles
// do not fit the co-resident grid (Llama shapes). Using
//   ||dY_b^T X_b||_F^2 = < X_b X_b^T , dY_b dY_b^T >_F
// each work item (b, i, j), i <= j, computes the 128x128 Gram tiles
//   Gx = X_b[i] X_b[j]^T  (K = P)   and   Gy = dY_b[i] dY_b[j]^T  (K = D)
// on tcgen05 (both operands K-major: rows of X / dY are contiguous in p / d),
// keeps both in TMEM (2 x 128 columns, double-buffered), and reduces
// w_ij * sum(Gx .* Gy) (w = 1 on the diagonal, 2 off it) to one partial per
// (sample, tile pair). The partials are summed in a fixed order by
// k_reduce_norms, which also forms the clip factors (dpcore.py:41-47).
// Cost ~ T^2 (P + D) flops per sample versus 2 T P D for recomputing G_b, so
// the layer is never differentiated twice (the reference's implicit workflow
// recomputes: workflows.py:302-321).
#include "fdp_internal.h"
#include "fdp_ptx.cuh"

namespace fdp {

namespace {

constexpr int kGT = 128;                       // Gram tile rows (t) = cols (s)
constexpr int kGTileBytes = kGT * kBK * 2;     // 16 KB: 128 rows x 64 bf16 (one SW128 K-major atom column)
constexpr int kGStageBytes = 2 * kGTileBytes;  // A + B
constexpr int kGStages = 6;
constexpr int kGNBuf = 2;                      // (Gx, Gy) accumulator pairs
constexpr size_t kGSmem = 1024 + size_t(kGStages) * kGStageBytes + 1024;
// kind::f16, bf16 x bf16 -> fp32, A and B K-major, M = N = 128
constexpr uint32_t kGIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(128 >> 3) << 17) |
                             (static_cast<uint32_t>(128 >> 4) << 24);

// K-major SWIZZLE_128B canonical layout: 8-row core groups of 128 B rows,
// SBO = 1024 B between 8-row groups; LBO unused (one 64-element atom in K).
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) { return make_sdesc_sw128(saddr, 16, 1024); }

// Work item wi = ((b * n_pairs + pair) * split + s): sample b, Gram tile pair
// (i, j), K slice s of the split operand. The dot <Gx, Gy> is linear in each
// Gram, so a slice of the larger operand's K range paired with the full Gram of
// the smaller one gives a partial that sums to the sample's norm^2 (the smaller
// Gram is recomputed per slice: cheap when P and D differ a lot, e.g. an LM head).
// Mixed schedule (p.n_full > 0): work units 0 .. n_full - 1 are whole items (every
// full wave of the launch), the remaining items are split `split` ways so the last
// wave is filled instead of running a few whole items on mostly idle SMs; a whole
// item writes slot 0 of its `split` partial slots and zeroes the others.
struct GItem {
  int b, i, j, pair, s;
  int kx0, nx, ky0, ny;  // k-block ranges of the X and dY operands
  bool whole;            // mixed schedule: an unsplit item (zeroes its other partial slots)
};

__device__ __forceinline__ void decode_item(int wi, int n_pairs, int nT, int& b, int& i, int& j) {
  b = wi / n_pairs;
  int r = wi % n_pairs;
  // row-major upper triangle: row i has nT - i entries
  i = 0;
  while (r >= nT - i) {
    r -= nT - i;
    ++i;
  }
  j = i + r;
}

__device__ __forceinline__ GItem decode_split(int wi, const GhostParams& p, int nkx, int nky) {
  GItem it;
  int wp;
  it.whole = p.n_full > 0 && wi < p.n_full;
  if (it.whole) {
    it.s = 0;
    wp = wi;
  } else {
    const int j = wi - p.n_full;  // n_full = 0: the uniform schedule
    it.s = j % p.split;
    wp = p.n_full + j / p.split;
  }
  decode_item(wp, p.n_pairs, p.nT, it.b, it.i, it.j);
  it.pair = wp % p.n_pairs;
  it.kx0 = 0;
  it.nx = nkx;
  it.ky0 = 0;
  it.ny = nky;
  if (it.whole) return it;
  if (p.split_x) {
    it.kx0 = it.s * nkx / p.split;
    it.nx = (it.s + 1) * nkx / p.split - it.kx0;
  } else {
    it.ky0 = it.s * nky / p.split;
    it.ny = (it.s + 1) * nky / p.split - it.ky0;
  }
  return it;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    ghost_norm_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_dy,
                      const GhostParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGStages * kGStageBytes);
  uint64_t* empty = full + kGStages;
  uint64_t* tfull = empty + kGStages;
  uint64_t* tempty = tfull + kGNBuf;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + kGNBuf);
  float* red = reinterpret_cast<float*>(tmem_holder + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned* err = p.err;
  if (threadIdx.x == 0) pdl_launch_dependents();  // the factor reduce / reweight may queue up behind us
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kGNBuf; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
    prefetch_tmap(&tm_x);
    prefetch_tmap(&tm_dy);
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int nkx = (p.P + kBK - 1) / kBK, nky = (p.D + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int wi = blockIdx.x; wi < p.n_items; wi += gridDim.x) {
        const GItem it = decode_split(wi, p, nkx, nky);
        const int i = it.i, j = it.j, b = it.b;
        // diagonal tiles (A == B) carry two k-blocks per stage: twice the bytes in flight
        for (int k = 0; k < it.nx + it.ny;) {
          const bool isx = k < it.nx;
          const CUtensorMap* m = isx ? &tm_x : &tm_dy;
          const int end = isx ? it.nx : it.nx + it.ny;
          const int cnt = (i == j && k + 1 < end) ? 2 : 1;
          const int kk = (isx ? it.kx0 + k : it.ky0 + k - it.nx) * kBK;
          mbar_wait(&empty[stage], phase ^ 1, err, p.budget_ns, 0x301);
          uint8_t* sa = smem + stage * kGStageBytes;
          mbar_arrive_expect_tx(&full[stage], (i == j ? cnt : 2) * kGTileBytes);
          tma_load_3d(sa, m, &full[stage], kk, i * kGT, b);
          if (i != j) tma_load_3d(sa + kGTileBytes, m, &full[stage], kk, j * kGT, b);
          else if (cnt == 2) tma_load_3d(sa + kGTileBytes, m, &full[stage], kk + kBK, i * kGT, b);
          k += cnt;
          if (++stage == kGStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, buf = 0, tphase = 0;
      for (int wi = blockIdx.x; wi < p.n_items; wi += gridDim.x) {
        const GItem it = decode_split(wi, p, nkx, nky);
        const int i = it.i, j = it.j;
        mbar_wait(&tempty[buf], tphase ^ 1, err, p.budget_ns, 0x302);
        tc_fence_after();
        for (int k = 0; k < it.nx + it.ny;) {
          const bool isx = k < it.nx;
          const int end = isx ? it.nx : it.nx + it.ny;
          const int cnt = (i == j && k + 1 < end) ? 2 : 1;
          const uint32_t dtm = tmem_base + buf * 256 + (isx ? 0 : 128);
          mbar_wait(&full[stage], phase, err, p.budget_ns, 0x303);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + stage * kGStageBytes);
          for (int h = 0; h < cnt; ++h) {
            const uint32_t a = base + h * kGTileBytes;
            const uint32_t bb = (i == j) ? a : a + kGTileBytes;
#pragma unroll
            for (int kq = 0; kq < kBK / 16; ++kq)
              tc_mma_f16(dtm, kdesc(a + kq * 32), kdesc(bb + kq * 32), kGIdesc,
                         (k == 0 || k == it.nx) && h == 0 && kq == 0 ? 0u : 1u);
          }
          tc_commit(&empty[stage]);
          k += cnt;
          if (++stage == kGStages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[buf]);
        if (++buf == kGNBuf) { buf = 0; tphase ^= 1; }
      }
    }
  } else if (warp >= kEpiWarp0) {
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3, half = ew >> 2, etid = ew * 32 + lane;
    uint32_t buf = 0, tphase = 0;
    for (int wi = blockIdx.x; wi < p.n_items; wi += gridDim.x) {
      const GItem it = decode_split(wi, p, nkx, nky);
      const int i = it.i, j = it.j, b = it.b;
      mbar_wait(&tfull[buf], tphase, err, p.budget_ns, 0x304);
      tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * 256 + half * 64;
      float part = 0.0f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float gx[32], gy[32];
        tmem_ld32(tb + c * 32, gx);
        tmem_ld32(tb + 128 + c * 32, gy);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) part = fmaf(gx[e], gy[e], part);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if (++buf == kGNBuf) { buf = 0; tphase ^= 1; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) red[ew] = part;
      named_bar_sync(1, 32 * kEpiWarps);
      if (etid == 0) {
        float s = 0.0f;
#pragma unroll
        for (int w = 0; w < kEpiWarps; ++w) s += red[w];
        float* slot = p.part + (static_cast<long long>(b) * p.n_pairs + it.pair) * p.split;
        slot[it.s] = (i == j ? 1.0f : 2.0f) * s;
        if (it.whole)
          for (int k = 1; k < p.split; ++k) slot[k] = 0.0f;
      }
      named_bar_sync(1, 32 * kEpiWarps);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem_base);
}

// ---------------------------------------------------------------- CTA-pair variant
// Work item (b, i, j), i <= j over 256-row blocks of t: a 2-CTA cluster computes
// the 256x256 Gram tiles with tcgen05.mma.cta_group::2 (M = 256: CTA r owns rows
// i*256 + r*128 .. +128 of the tile; N = 256: each CTA stages 128 of the j-block
// rows), Gx into TMEM columns [0, 256) and Gy into [256, 512). The epilogue pulls
// Gx into registers as soon as it is complete (so the next item's Gx MMAs can
// start while Gy is still accumulating), then reduces Gx .* Gy against Gy. Per
// SM this halves the operand bytes per flop of the 128x128 single-CTA kernel,
// which is bound by shared-memory fill. Partials: [B][n_pairs][2] (one per CTA).
constexpr int kPT = 256;                               // Gram tile rows per pair
constexpr int kPHalf = 128;                            // rows staged per CTA
constexpr int kPTileBytes = kPHalf * kBK * 2;          // 16 KB
constexpr int kPStageBytes = 2 * kPTileBytes;          // A + B halves
constexpr int kPStages = 6;
constexpr size_t kPSmem = 1024 + size_t(kPStages) * kPStageBytes + 1024;
// kind::f16, bf16 x bf16 -> fp32, A and B K-major, M = 256 (pair), N = 256
constexpr uint32_t kPIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kPT >> 3) << 17) |
                             (static_cast<uint32_t>(kPT >> 4) << 24);

__global__ void __launch_bounds__(kTcThreads, 1)
    ghost_norm_pair_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_dy,
                           const __grid_constant__ CUtensorMap tm_dy1, const __grid_constant__ CUtensorMap tm_dy2,
                           const GhostParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kPStages * kPStageBytes);
  uint64_t* empty = full + kPStages;
  uint64_t* tfull = empty + kPStages;  // [0] Gx done, [1] Gy done
  uint64_t* tempty = tfull + 2;        // [0] Gx read, [1] Gy read
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  float* red = reinterpret_cast<float*>(tmem_holder + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned* err = p.err;
  const int rank = static_cast<int>(cluster_ctarank());
  const bool leader = rank == 0;
  const int cid = blockIdx.x / 2, n_clusters = gridDim.x / 2;
  // layers sharing X (n_dy > 1, split == 1): one Gx per item, then one Gy per layer
  const int n_dy = p.n_dy > 1 ? p.n_dy : 1;
  if (threadIdx.x == 0) pdl_launch_dependents();  // the factor reduce / reweight may queue up behind us
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * 2);
    }
    fence_mbar_init();
    fence_proxy_async_smem();
    prefetch_tmap(&tm_x);
    prefetch_tmap(&tm_dy);
    if (n_dy > 1) prefetch_tmap(&tm_dy1);
    if (n_dy > 2) prefetch_tmap(&tm_dy2);
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_holder);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int nkx = (p.P + kBK - 1) / kBK, nky = (p.D + kBK - 1) / kBK;
  // k-block range of layer l's dY operand for an item (layer 0 carries the K split)
  auto y_range = [&](const GItem& it, int l, int& ky0, int& ny) {
    ky0 = l == 0 ? it.ky0 : 0;
    ny = l == 0 ? it.ny : ((l == 1 ? p.D1 : p.D2) + kBK - 1) / kBK;
  };

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (int wi = cid; wi < p.n_items; wi += n_clusters) {
        const GItem it = decode_split(wi, p, nkx, nky);
        const int i = it.i, j = it.j, b = it.b;
        const int ra = i * kPT + rank * kPHalf, rb = j * kPT + rank * kPHalf;
        auto load = [&](const CUtensorMap* m, int kk) {
          mbar_wait(&empty[stage], phase ^ 1, err, p.budget_ns, 0x311);
          uint8_t* sa = smem + stage * kPStageBytes;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * (i == j ? kPTileBytes : kPStageBytes));
          tma_load_3d_pair(sa, m, &full[stage], kk, ra, b);
          if (i != j) tma_load_3d_pair(sa + kPTileBytes, m, &full[stage], kk, rb, b);
          if (++stage == kPStages) { stage = 0; phase ^= 1; }
        };
        for (int k = 0; k < it.nx; ++k) load(&tm_x, (it.kx0 + k) * kBK);
        for (int l = 0; l < n_dy; ++l) {
          const CUtensorMap* m = l == 0 ? &tm_dy : (l == 1 ? &tm_dy1 : &tm_dy2);
          int ky0, ny;
          y_range(it, l, ky0, ny);
          for (int k = 0; k < ny; ++k) load(m, (ky0 + k) * kBK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      uint32_t stage = 0, phase = 0, ph0 = 0, ph1 = 0;
      for (int wi = cid; wi < p.n_items; wi += n_clusters) {
        const GItem it = decode_split(wi, p, nkx, nky);
        const int i = it.i, j = it.j;
        // n k-blocks into the accumulator at column offset col (the previous use has been read out)
        auto gram = [&](int n, uint32_t col, uint64_t* free_bar, uint32_t free_ph, uint64_t* done_bar) {
          mbar_wait(free_bar, free_ph ^ 1, err, p.budget_ns, 0x312);
          tc_fence_after();
          for (int k = 0; k < n; ++k) {
            mbar_wait(&full[stage], phase, err, p.budget_ns, 0x313);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + stage * kPStageBytes);
            const uint32_t bb = (i == j) ? a : a + kPTileBytes;
#pragma unroll
            for (int kq = 0; kq < kBK / 16; ++kq)
              tc_mma_f16_pair(tmem_base + col, kdesc(a + kq * 32), kdesc(bb + kq * 32), kPIdesc,
                              k == 0 && kq == 0 ? 0u : 1u);
            tc_commit_pair(&empty[stage]);
            if (++stage == kPStages) { stage = 0; phase ^= 1; }
          }
          tc_commit_pair(done_bar);
        };
        gram(it.nx, 0u, &tempty[0], ph0, &tfull[0]);
        ph0 ^= 1;
        for (int l = 0; l < n_dy; ++l) {
          int ky0, ny;
          y_range(it, l, ky0, ny);
          gram(ny, static_cast<uint32_t>(kPT), &tempty[1], ph1, &tfull[1]);
          ph1 ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3, half = ew >> 2, etid = ew * 32 + lane;
    uint32_t ph0 = 0, ph1 = 0;
    for (int wi = cid; wi < p.n_items; wi += n_clusters) {
      const GItem it = decode_split(wi, p, nkx, nky);
      const int i = it.i, j = it.j, b = it.b;
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + half * 128;
      float gx[128];
      mbar_wait(&tfull[0], ph0, err, p.budget_ns, 0x314);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float v[16];
        tmem_ld16(tb + c * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) gx[c * 16 + e] = v[e];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[0]);
      ph0 ^= 1;
      for (int l = 0; l < n_dy; ++l) {
        mbar_wait(&tfull[1], ph1, err, p.budget_ns, 0x315);
        tc_fence_after();
        float part = 0.0f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float v[16];
          tmem_ld16(tb + kPT + c * 16, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) part = fmaf(gx[c * 16 + e], v[e], part);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty[1]);
        ph1 ^= 1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) red[ew] = part;
        named_bar_sync(1, 32 * kEpiWarps);
        if (etid == 0) {
          float s = 0.0f;
#pragma unroll
          for (int w = 0; w < kEpiWarps; ++w) s += red[w];
          float* out = l == 0 ? p.part : (l == 1 ? p.part1 : p.part2);
          float* slot = out + (static_cast<long long>(b) * p.n_pairs + it.pair) * p.split * 2;
          slot[it.s * 2 + rank] = (i == j ? 1.0f : 2.0f) * s;
          if (it.whole)
            for (int k = 1; k < p.split; ++k) slot[k * 2 + rank] = 0.0f;
        }
        named_bar_sync(1, 32 * kEpiWarps);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair<512>(tmem_base);
}

}  // namespace

cudaError_t launch_ghost_pair(const CUtensorMap& tm_x, const CUtensorMap& tm_dy, const GhostParams& p, int grid,
                              cudaStream_t stream, const CUtensorMap* tm_dy1, const CUtensorMap* tm_dy2) {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(ghost_norm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kPSmem));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) done[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = kPSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ghost_norm_pair_kernel, tm_x, tm_dy, tm_dy1 ? *tm_dy1 : tm_dy,
                            tm_dy2 ? *tm_dy2 : tm_dy, p);
}

cudaError_t launch_ghost(const CUtensorMap& tm_x, const CUtensorMap& tm_dy, const GhostParams& p, int grid,
                         cudaStream_t stream) {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !done[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(ghost_norm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGSmem));
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) done[dev] = true;
  }
  ghost_norm_kernel<<<grid, kTcThreads, kGSmem, stream>>>(tm_x, tm_dy, p);
  return cudaGetLastError();
}

}  // namespace fdp
