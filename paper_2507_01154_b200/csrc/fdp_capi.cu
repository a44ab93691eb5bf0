// fdp_capi.cu -- the C ABI (include/fdp.h): validation, planning, workspace
// layout, TMA descriptors and dispatch of the four workflow kinds
// (workflows.py:427-440).
#include "../../include/fdp.h"
#include "fdp_internal.h"
#include "fdp_rng.cuh"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <map>
#include <vector>

// Host-side state of a deferred-finalize chain (include/fdp.h, fdp_dw_chained):
// at most one pending single-sample finalize, and two device slots (ping-pong)
// for the norm partials of the pending layer, so the call carrying the pending
// job can write its own partials meanwhile.
struct fdp_chain {
  bool pending = false;
  fdp::FinJob job{};
  float* part[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};
  int slot = 0;  // slot the next pending job's partials go to
  int dev = -1;
  long long carried = 0, flushed = 0;  // statistics: jobs carried by a GEMM / run standalone
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(FDP_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// ---- reference key construction (rng.py:35-47), host side
using fdp::kGamma;
uint64_t absorb3(int64_t seed, int64_t layer, int64_t step) {
  return fdp::absorb3(static_cast<uint64_t>(seed), static_cast<uint64_t>(layer), static_cast<uint64_t>(step));
}

struct DevInfo {
  int dev = -1;
  int sms = 0;
  int major = 0, minor = 0;
};

int get_dev(DevInfo& di) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  static std::mutex mu;
  static DevInfo cache[64];
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && cache[dev].dev == dev) {
    di = cache[dev];
    return FDP_OK;
  }
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  di.dev = dev;
  di.sms = prop.multiProcessorCount;
  di.major = prop.major;
  di.minor = prop.minor;
  if (dev >= 0 && dev < 64) cache[dev] = di;
  return FDP_OK;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// bf16 (inner, T, B) tensor, box (64, box_rows, 1), 128B swizzle.
int make_tmap(CUtensorMap* m, const void* ptr, int64_t inner, int64_t T, int64_t B, int box_rows = fdp::kBK) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(FDP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(T), static_cast<cuuint64_t>(B)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner * 2), static_cast<cuuint64_t>(inner * T * 2)};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FDP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return FDP_OK;
}

// fp32 2-D/3-D maps for the fused epilogue's TMA stores (128B swizzle, 32-column boxes)
int make_tmap_f32(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                  const cuuint32_t* box) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(FDP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FDP_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", static_cast<int>(r));
  return FDP_OK;
}

int validate(const fdp_desc* d, int32_t kind) {
  if (!d) return fail(FDP_ERR_USAGE, "null descriptor");
  if (kind < FDP_KIND_NON_DP || kind > FDP_KIND_FLASHDP) return fail(FDP_ERR_USAGE, "unknown workflow kind %d", kind);
  if (d->B < 1 || d->T < 1 || d->P < 1 || d->D < 1)
    return fail(FDP_ERR_SHAPE, "all extents must be >= 1, got B=%lld T=%lld P=%lld D=%lld", (long long)d->B,
                (long long)d->T, (long long)d->P, (long long)d->D);
  if (d->B > (1ll << 30) || d->T > (1ll << 30) || d->P > (1ll << 30) || d->D > (1ll << 30))
    return fail(FDP_ERR_SHAPE, "extent too large");
  if (d->in_dtype != FDP_DTYPE_BF16 && d->in_dtype != FDP_DTYPE_F32 && d->in_dtype != FDP_DTYPE_F64)
    return fail(FDP_ERR_USAGE, "in_dtype must be bf16 (0), f32 (1) or f64 (2), got %d", d->in_dtype);
  if (kind != FDP_KIND_NON_DP) {
    if (!(d->clip_c > 0.0) || !std::isfinite(d->clip_c))
      return fail(FDP_ERR_USAGE, "clip_c must be positive, got %g", d->clip_c);
    if (!(d->sigma >= 0.0) || !std::isfinite(d->sigma))
      return fail(FDP_ERR_USAGE, "sigma must be >= 0, got %g", d->sigma);
    if (d->reduction != FDP_REDUCE_SUM && d->reduction != FDP_REDUCE_MEAN)
      return fail(FDP_ERR_USAGE, "reduction must be sum (0) or mean (1), got %d", d->reduction);
  }
  if (d->world < 1 || d->rank < 0 || d->rank >= d->world)
    return fail(FDP_ERR_USAGE, "rank %d out of range for world %d", d->rank, d->world);
  if (d->mean_batch < 0) return fail(FDP_ERR_USAGE, "mean_batch must be >= 0");
  if (d->noise_impl < FDP_NOISE_KEYED_F32 || d->noise_impl > FDP_NOISE_PHILOX)
    return fail(FDP_ERR_USAGE, "unknown noise_impl %d", d->noise_impl);
  if (d->path < FDP_PATH_AUTO || d->path > FDP_PATH_SIMT) return fail(FDP_ERR_USAGE, "unknown path %d", d->path);
  if (d->norm_phase < FDP_NORMS_AUTO || d->norm_phase > FDP_NORMS_SPILL)
    return fail(FDP_ERR_USAGE, "unknown norm_phase %d", d->norm_phase);
  if (d->norm_phase == FDP_NORMS_SINGLE && (d->B != 1 || d->accumulate))
    return fail(FDP_ERR_USAGE, "norm_phase single needs B == 1 and accumulate == 0");
  return FDP_OK;
}

struct Plan {
  int stream_mc = 1;     // stream-K kernel cluster layout: 2 = two pairs per 4-CTA cluster (X multicast)
  int stream_tiles = 0;  // per-CTA tile slots of the stream kernel
  int path = FDP_PATH_SIMT;
  int norm_phase = FDP_NORMS_RECOMPUTE;
  int bn = 128;
  int cg = 1;
  int n_dt = 0, n_pt = 0, n_tiles = 0, n_wtiles = 0;
  int groups = 1;
  int grid = 0;
  int launches = 0;
  bool tc = false;
  // workspace layout (byte offsets)
  size_t off_ctrl = 0, off_cnt = 0, off_tile_cnt = 0, off_part = 0, off_tag = 0, off_factor = 0, off_acc = 0,
         off_g = 0, off_gp = 0, total = 0;
  int part_tiles = 0;  // partial norms per sample
  int expl_chunks = 0;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

bool tc_shape_ok(const fdp_desc* d) {
  return d->in_dtype == FDP_DTYPE_BF16 && d->P % 8 == 0 && d->D % 8 == 0 && d->T <= (1ll << 30);
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

// SMs a per-layer call leaves free (FDP_RESERVE_SMS, default 0): under data
// parallelism (ddp.DataParallelStep sets it to its NCCL CTA budget) every grid is
// capped so the collective's CTAs stay resident next to ours and the grids that
// rely on co-residency (split tiles waiting on the cluster that initialises them,
// the fused per-sample all-reduce) never wait on a CTA that cannot be scheduled.
int reserved_sms() {
  const int r = env_int("FDP_RESERVE_SMS", 0);
  return r > 0 ? r : 0;
}

// Ghost norms cost ~T^2 (P + D) (1 + 1/nT) flops per sample, recomputing the
// per-sample gradient 2 T P D: take the cheaper one unless the caller forces it.
bool single_ok(const fdp_desc* d) { return d->B == 1 && !d->accumulate; }

int choose_norm_phase(const fdp_desc* d) {
  if (d->norm_phase != FDP_NORMS_AUTO) return d->norm_phase;
  if (single_ok(d)) return FDP_NORMS_SINGLE;
  // FDP_NORM_PHASE=spill: opt into the per-sample-spill phase for every auto two-phase layer
  if (const char* v = std::getenv("FDP_NORM_PHASE"))
    if (std::strcmp(v, "spill") == 0 && d->B <= 64) return FDP_NORMS_SPILL;
  const double nT = static_cast<double>((d->T + 127) / 128);
  const double ghost = static_cast<double>(d->T) * d->T * (d->P + d->D) * (1.0 + 1.0 / nT);
  const double recompute = 2.0 * d->T * d->P * d->D;
  return ghost < recompute ? FDP_NORMS_GHOST : FDP_NORMS_RECOMPUTE;
}

// Ghost-norm kernel variant: 256-row Gram tiles on CTA pairs (half the operand
// bytes per flop) or 128-row tiles on single CTAs (finer work items). Both take
// the same time per wave of work items at the rates measured on B200 (the
// single-CTA tile is bound by shared-memory fill at ~half the pair's per-SM
// rate, so a pair wave costs ~1.2 single waves), so the cheaper schedule wins.
struct GhostShape {
  bool pair;
  int nT, n_pairs, parts;  // parts: norm partials per sample
  int split, split_x;      // K slices of the larger operand per tile pair
  int n_full;              // > 0: mixed schedule (whole items for the full waves, the last wave split)
  long long units;         // work units of the launch
};
GhostShape ghost_shape(const fdp_desc* d, int sms) {
  const long long nT2 = (d->T + 255) / 256, np2 = nT2 * (nT2 + 1) / 2;
  const long long nT1 = (d->T + 127) / 128, np1 = nT1 * (nT1 + 1) / 2;
  const int eff = std::max(2, sms - reserved_sms());  // the SMs the ghost launch gets
  const long long clusters = eff / 2 > 0 ? eff / 2 : 1;
  const long long ctas = eff > 0 ? eff : 1;
  const long long nkx = (d->P + 63) / 64, nky = (d->D + 63) / 64;
  const long long big = std::max(nkx, nky), small = std::min(nkx, nky);
  const int forced = env_int("FDP_GHOST_PAIR", -1);
  const int forced_split = env_int("FDP_GHOST_SPLIT", 0);
  // Modelled time in single-CTA k-block units: waves x per-item k-blocks; a pair
  // k-block (256x256 tile on 2 SMs) takes ~1.1-1.2x a single-CTA one (128x128 on
  // 1 SM). Slicing the larger operand's K range S ways multiplies the items by S
  // and recomputes the smaller Gram per slice (tools/ghost_split_sweep.py: LM head
  // 768 -> 50304 at B=8 974 -> 924 us per layer, Llama 4096 -> 32000 at B=1 665 -> 610).
  // Mixed schedule: when the items leave a partial last wave, the full waves run whole
  // items and only the last wave's items are split (FDP_GHOST_MIXED=0 turns it off).
  const bool mixed_ok = forced_split == 0 && env_int("FDP_GHOST_MIXED", 1) != 0;
  double best = 1e300;
  GhostShape g{};
  for (int pair = 1; pair >= 0; --pair) {
    if (forced >= 0 && forced != pair) continue;
    const long long items = d->B * (pair ? np2 : np1), slots = pair ? clusters : ctas;
    const double f = pair ? 1.1 : 1.0;
    for (long long S = 1; S <= 16 && S <= big; ++S) {
      if (forced_split > 0 && S != forced_split) continue;
      const long long waves = (items * S + slots - 1) / slots;
      const double t = static_cast<double>(waves) * static_cast<double>(small + (big + S - 1) / S) * f;
      if (t < best * 0.98) {
        best = t;
        g.pair = pair != 0;
        g.split = static_cast<int>(S);
        g.n_full = 0;
      }
    }
    const long long fw = items / slots, tail = items - fw * slots;
    if (mixed_ok && fw >= 1 && tail > 0) {
      const long long S = std::min<long long>({16, big, slots / tail});
      if (S >= 2) {
        const double t = (static_cast<double>(fw) * static_cast<double>(small + big) +
                          static_cast<double>(small + (big + S - 1) / S)) * f;
        if (t < best * 0.98) {
          best = t;
          g.pair = pair != 0;
          g.split = static_cast<int>(S);
          g.n_full = static_cast<int>(fw * slots);
        }
      }
    }
  }
  if (g.split == 0) {  // forced split larger than the K range: no slicing
    g.pair = forced != 0;
    g.split = 1;
  }
  g.split_x = nkx >= nky ? 1 : 0;
  g.nT = static_cast<int>(g.pair ? nT2 : nT1);
  g.n_pairs = static_cast<int>(g.pair ? np2 : np1);
  g.parts = (g.pair ? 2 : 1) * g.n_pairs * g.split;
  const long long items = d->B * static_cast<long long>(g.n_pairs);
  g.units = g.n_full > 0 ? g.n_full + (items - g.n_full) * g.split : items * g.split;
  return g;
}

int make_plan(const fdp_desc* d, int32_t kind, const DevInfo& di, Plan& pl) {
  const bool tc_dev = di.major == 10;  // sm_100 family
  const bool tc_ok = tc_dev && tc_shape_ok(d);
  const int want = d->path;
  pl = Plan();
  const int forced_bn = env_int("FDP_FORCE_BN", 0);
  const int forced_cg = env_int("FDP_FORCE_CG", 0);

  // Work tile = cg x 128 d-rows x bn p-cols; returns the number of work tiles.
  auto tiles_for = [&](int bn, int cg, int& ndt2, int& npt) {
    const long long ndt = (d->D + fdp::kBM - 1) / fdp::kBM;
    ndt2 = static_cast<int>((ndt + cg - 1) / cg);
    npt = static_cast<int>((d->P + bn - 1) / bn);
    return static_cast<long long>(ndt2) * npt;
  };
  // Preference order among equally good fills: CTA pairs (half the operand
  // traffic per SM) and the 64-register accumulator width first.
  const int cands[4][2] = {{128, 2}, {256, 2}, {256, 1}, {128, 1}};
  auto allowed = [&](int bn, int cg) {
    return (!forced_bn || bn == forced_bn) && (!forced_cg || cg == forced_cg);
  };
  const int pcands[4][2] = {{256, 2}, {256, 1}, {128, 2}, {128, 1}};  // persistent: widest tile first
  auto persistent_choice = [&]() {
    for (auto& cd : pcands)
      if (allowed(cd[0], cd[1]) && fdp::tc_max_coresident_ctas(cd[0], cd[1]) > 0) {
        pl.bn = cd[0];
        pl.cg = cd[1];
        return;
      }
    pl.bn = 128;
    pl.cg = 1;
  };

  if (kind == FDP_KIND_FLASHDP) {
    if ((want == FDP_PATH_FUSED || want == FDP_PATH_TWO_PHASE) && !tc_ok)
      return fail(FDP_ERR_USAGE,
                  "path %d needs bf16 inputs, P %% 8 == 0, D %% 8 == 0 and an sm_100 device (got dtype=%d P=%lld "
                  "D=%lld cc=%d.%d)",
                  want, d->in_dtype, (long long)d->P, (long long)d->D, di.major, di.minor);
    if (want == FDP_PATH_SIMT || !tc_ok) {
      pl.path = FDP_PATH_SIMT;
    } else {
      // Choose the tile shape with the smallest modelled time: per-CTA samples x
      // one sample's MMA time at the measured per-SM rate of that shape, plus the
      // cross-group reduction when samples are split over CTAs. Per-SM rates
      // (TFLOP/s, B200, fused loop; tools/trace_fused.py): operand traffic per
      // flop halves from a 128x128 single-CTA tile to a 256x256 CTA-pair tile.
      auto sm_rate = [](int bn, int cg) {
        if (bn == 256) return cg == 2 ? 9.6e12 : 7.4e12;
        return cg == 2 ? 6.4e12 : 6.3e12;
      };
      double best = 1e300;
      int best_bn = 0, best_cg = 1, best_groups = 1;
      for (auto& cd : cands) {
        const int bn = cd[0], cg = cd[1];
        if (!allowed(bn, cg)) continue;
        int ndt2, npt;
        const long long nwt = tiles_for(bn, cg, ndt2, npt);
        long long cap = fdp::tc_max_coresident_ctas(bn, cg);
        if (cap > 0) cap = std::max<long long>(0, cap - ((reserved_sms() + cg - 1) / cg) * cg);
        const long long need = nwt * cg;
        if (cap <= 0 || need > cap) continue;
        long long g = cap / need;
        if (g > d->B) g = d->B;
        if (g > 8) g = 8;
        while (g & (g - 1)) --g;  // 1, 2, 4 or 8: slices of 128 rows stay whole 8-row swizzle atoms
        const double units = static_cast<double>((d->B + g - 1) / g);
        const double unit_flops = 2.0 * fdp::kBM * bn * static_cast<double>(d->T);
        // a sample unit: its MMA or the two TMEM passes over its accumulator (norm, clip;
        // ~160 GB/s per SM), whichever is longer, plus one block-wise all-reduce round
        // (calibrated on B200: 1024^2 / 2048^2 at B=64, T=128; 2048^2 at B=32, T=256;
        // GPT-2 c_fc at B=8, T=1024 -- tools/nondp_cmp.py)
        const double read_t = 2.0 * fdp::kBM * bn * 4.0 / 160e9;
        const double unit_t = std::max(unit_flops / sm_rate(bn, cg), read_t) + 1.2e-6;
        const double est = units * unit_t + (g > 1 ? 4e-6 : 0.0) + 8e-6;
        if (est < best * 0.97) {
          best = est;
          best_bn = bn;
          best_cg = cg;
          best_groups = static_cast<int>(g);
        }
      }
      // two-phase estimate: norm phase + one reweighted pass at the persistent rate
      const double dw_flops = 2.0 * d->B * d->T * static_cast<double>(d->P) * d->D;
      const double nT = static_cast<double>((d->T + 127) / 128);
      const double ghost_flops = d->B * static_cast<double>(d->T) * d->T * (d->P + d->D) * (1.0 + 1.0 / nT);
      const double norm_flops = (single_ok(d) && d->norm_phase != FDP_NORMS_GHOST &&
                                 d->norm_phase != FDP_NORMS_RECOMPUTE)
                                    ? 0.0
                                    : std::min(ghost_flops, dw_flops);
      const double two_phase_est = (norm_flops / 0.55e15) + dw_flops / 1.1e15 + 25e-6;
      if (best_bn && want == FDP_PATH_AUTO && two_phase_est < best) best_bn = 0;
      if (best_bn && want != FDP_PATH_TWO_PHASE) {
        pl.path = FDP_PATH_FUSED;
        pl.bn = best_bn;
        pl.cg = best_cg;
        pl.groups = best_groups;
      } else {
        pl.path = FDP_PATH_TWO_PHASE;
        persistent_choice();
        pl.norm_phase = choose_norm_phase(d);
      }
    }
  } else if (kind == FDP_KIND_IMPLICIT_DP) {
    pl.path = (tc_ok && want != FDP_PATH_SIMT) ? FDP_PATH_TWO_PHASE : FDP_PATH_SIMT;
    persistent_choice();
    pl.norm_phase = FDP_NORMS_RECOMPUTE;
  } else {  // NON_DP / EXPLICIT_DP: tensor-core GEMM stage when possible
    pl.path = (tc_ok && want != FDP_PATH_SIMT) ? FDP_PATH_FUSED : FDP_PATH_SIMT;
    persistent_choice();
  }
  pl.tc = pl.path != FDP_PATH_SIMT;

  if (pl.tc) {
    pl.n_wtiles = static_cast<int>(tiles_for(pl.bn, pl.cg, pl.n_dt, pl.n_pt));
    pl.n_tiles = pl.n_wtiles * pl.cg;
  } else {
    pl.cg = 1;
    pl.n_dt = static_cast<int>((d->D + 31) / 32);
    pl.n_pt = static_cast<int>((d->P + 31) / 32);
    pl.n_tiles = pl.n_dt * pl.n_pt;
    pl.n_wtiles = pl.n_tiles;
  }

  // grid + launch count
  if (kind == FDP_KIND_FLASHDP && pl.path == FDP_PATH_FUSED) {
    pl.grid = pl.n_tiles * pl.groups;
    pl.launches = 1;
  } else if (pl.tc) {
    const int cap = fdp::tc_max_coresident_ctas(pl.bn, pl.cg);
    const int max_clusters = std::max(1, ((cap > 0 ? cap : di.sms) - reserved_sms()) / pl.cg);
    pl.grid = (pl.n_wtiles < max_clusters ? pl.n_wtiles : max_clusters) * pl.cg;
    if (kind == FDP_KIND_NON_DP) pl.launches = 1;
    else if (kind == FDP_KIND_EXPLICIT_DP) pl.launches = 5;  // G, norms, reduce, clip, sum
    else if (pl.path == FDP_PATH_TWO_PHASE && pl.norm_phase == FDP_NORMS_SINGLE) pl.launches = 2;  // GEMM, finalize
    else if (pl.path == FDP_PATH_TWO_PHASE && pl.norm_phase == FDP_NORMS_SPILL) pl.launches = 3;  // GEMMs, factors, combine
    else pl.launches = 3;                                     // norms, reduce, reweight
  } else {
    pl.grid = pl.n_tiles;
    if (kind == FDP_KIND_NON_DP) pl.launches = 1;
    else if (kind == FDP_KIND_EXPLICIT_DP) pl.launches = 5;
    else pl.launches = 3;
  }

  // stream-K kernel layout (two-phase reweight, B = 1 GEMM, non-DP): two CTA pairs per
  // 4-CTA cluster with the X operand multicast when the 256x256 pair tile is used
  // (X boxes multicast to the pair below): measured 2.5-3 % faster on down projections
  // (13824 -> 5120 at B = 2 / 4), 1.5-3 % slower on square / up projections
  // (tools/ab_layer.py, profiles/r1_stream_mc_ab.jsonl), so chosen for P >= 2 D only
  // round 2: on the same down projections a grouped tile raster on 2-CTA clusters beats the
  // multicast layout (13824 -> 5120, T=2048: B=1 358 -> 332 us, B=2 612 -> 572 us, A/B in
  // profiles/r2_stream_swizzle_ab.jsonl; the 4-CTA layout only fits 33 clusters = 132 SMs), so
  // multicast is opt-in (FDP_STREAM_MC=1) and the raster is grouped by 8 row blocks there
  const int mc_env = env_int("FDP_STREAM_MC", -1);
  const bool mc_want = mc_env >= 0 ? mc_env != 0 : false;
  const bool spill = pl.path == FDP_PATH_TWO_PHASE && pl.norm_phase == FDP_NORMS_SPILL;
  pl.stream_mc = (pl.tc && pl.bn == 256 && pl.cg == 2 && mc_want && !spill && fdp::stream_mc_max_clusters() > 0)
                     ? 2 : 1;
  pl.stream_tiles = pl.tc ? fdp::stream_wtiles(pl.n_wtiles, pl.n_pt, pl.stream_mc) * pl.cg * pl.stream_mc
                          : pl.n_tiles;
  const long long n_slots = std::max<long long>(pl.n_tiles, pl.stream_tiles);

  // workspace layout
  const long long B = d->B;
  pl.part_tiles = static_cast<int>(n_slots);
  if (pl.path == FDP_PATH_TWO_PHASE && pl.norm_phase == FDP_NORMS_GHOST) pl.part_tiles = ghost_shape(d, di.sms).parts;
  if (kind == FDP_KIND_EXPLICIT_DP && d->in_dtype != FDP_DTYPE_F64) {
    pl.expl_chunks = 64;
    pl.part_tiles = pl.expl_chunks;
  }
  size_t off = 0;
  pl.off_ctrl = off;
  off += 256;
  pl.off_cnt = off;
  off = align_up(off + 4 * B, 256);
  pl.off_tile_cnt = off;
  off = align_up(off + 4ull * n_slots, 256);
  const size_t esz = d->in_dtype == FDP_DTYPE_F64 ? 8 : 4;  // fp64 parity path keeps partials / factors in fp64
  pl.off_part = off;
  off = align_up(off + esz * B * pl.part_tiles, 256);
  pl.off_tag = off;
  off = align_up(off + 8ull * B * pl.n_tiles, 256);
  pl.off_factor = off;
  off = align_up(off + esz * B, 256);
  pl.off_acc = off;
  if (kind == FDP_KIND_FLASHDP && pl.path == FDP_PATH_FUSED && pl.groups > 1 && (d->flags & FDP_FLAG_DETERMINISTIC))
    off = align_up(off + 4ull * pl.groups * pl.n_tiles * fdp::kBM * pl.bn, 256);
  pl.off_g = off;
  pl.off_gp = off;
  if (spill) {  // the per-sample gradients G[b] (B, D, P) fp32
    off = align_up(off + 4ull * B * d->D * d->P, 256);
    pl.off_gp = off;
  }
  if (kind == FDP_KIND_EXPLICIT_DP && d->in_dtype != FDP_DTYPE_F64) {
    const size_t gbytes = 4ull * B * d->D * d->P;
    pl.off_gp = align_up(off + gbytes, 256);
    off = align_up(pl.off_gp + gbytes, 256);
  }
  if (d->flags & FDP_FLAG_TRACE) off = align_up(off, 256) + 1024ull * (pl.grid > 0 ? pl.grid : 1);
  pl.total = off;
  return FDP_OK;
}

struct Common {
  uint64_t key_base, key_base_g;
  long long noise_lo, noise_hi;
  float noise_scale;
  float inv_batch;
  int add_noise;
};

Common common_of(const fdp_desc* d) {
  Common c;
  c.key_base = absorb3(d->seed, d->layer_id, d->step);
  c.key_base_g = c.key_base + kGamma;
  const long long n = d->D * d->P;
  c.noise_lo = n * d->rank / d->world;
  c.noise_hi = n * (d->rank + 1) / d->world;
  c.noise_scale = static_cast<float>(d->sigma * d->clip_c);
  c.add_noise = (d->add_noise && d->sigma > 0.0) ? 1 : 0;
  const long long mb = d->mean_batch > 0 ? d->mean_batch : d->B;
  c.inv_batch = d->reduction == FDP_REDUCE_MEAN ? static_cast<float>(1.0 / static_cast<double>(mb)) : 1.0f;
  return c;
}

template <typename T>
T* ws_at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

fdp::SimtParams simt_params(const fdp_desc* d, const Plan& pl, const Common& c, const void* x, const void* dy,
                            float* grad_w, float* norms, void* ws) {
  fdp::SimtParams s{};
  s.B = static_cast<int>(d->B);
  s.T = static_cast<int>(d->T);
  s.P = static_cast<int>(d->P);
  s.D = static_cast<int>(d->D);
  s.in_f32 = d->in_dtype == FDP_DTYPE_F32;
  s.x = x;
  s.dy = dy;
  s.n_dt = static_cast<int>((d->D + 31) / 32);
  s.n_pt = static_cast<int>((d->P + 31) / 32);
  s.n_tiles = s.n_dt * s.n_pt;
  s.clip_c = d->clip_c;
  s.clip_c2 = d->clip_c * d->clip_c;
  s.inv_batch = c.inv_batch;
  s.accumulate = d->accumulate;
  s.add_noise = c.add_noise;
  s.noise_impl = d->noise_impl;
  s.noise_scale = c.noise_scale;
  s.key_base = c.key_base;
  s.key_base_g = c.key_base_g;
  s.step_ptr = reinterpret_cast<const long long*>(d->device_step);
  s.seed_u = static_cast<uint64_t>(d->seed);
  s.layer_u = static_cast<uint64_t>(d->layer_id);
  s.noise_lo = c.noise_lo;
  s.noise_hi = c.noise_hi;
  s.grad_w = grad_w;
  s.norms_out = norms;
  s.ws_part = ws_at<float>(ws, pl.off_part);
  s.ws_factor = ws_at<float>(ws, pl.off_factor);
  s.with_clip = 1;
  return s;
}

fdp::StreamParams stream_params(const fdp_desc* d, const Plan& pl, const Common& c, float* grad_w, void* ws,
                                bool reweight) {
  fdp::StreamParams p{};
  p.B = static_cast<int>(d->B);
  p.P = static_cast<int>(d->P);
  p.D = static_cast<int>(d->D);
  p.n_pt = pl.n_pt;
  p.n_wtiles = pl.n_wtiles;
  p.n_kb = static_cast<int>((d->T + fdp::kBK - 1) / fdp::kBK);
  p.reweight = reweight ? 1 : 0;
  p.accumulate = d->accumulate;
  p.add_noise = reweight ? c.add_noise : 0;
  // epilogue-drawn Philox noise for tiles held whole (accumulator initial value, plain
  // TMA store) instead of a noise-warp pre-fill + TMA reduce-add: 5120x13824 at B=2
  // 496 -> 433 us; at B=4 / 8 1.6-2 % faster, neutral on 4096^2 (tools/ab_layer.py)
  p.epi_noise = (d->noise_impl == FDP_NOISE_PHILOX && env_int("FDP_EPI_NOISE", 1)) ? 1 : 0;
  p.noise_impl = d->noise_impl;
  p.noise_scale = c.noise_scale;
  p.key_base = c.key_base;
  p.key_base_g = c.key_base_g;
  p.step_ptr = reinterpret_cast<const long long*>(d->device_step);
  p.seed_u = static_cast<uint64_t>(d->seed);
  p.layer_u = static_cast<uint64_t>(d->layer_id);
  p.noise_lo = c.noise_lo;
  p.noise_hi = c.noise_hi;
  p.grad_w = grad_w;
  p.factors_in = ws_at<float>(ws, pl.off_factor);
  p.tile_cnt = ws_at<unsigned>(ws, pl.off_tile_cnt);
  p.ctrl = ws_at<unsigned>(ws, pl.off_ctrl);
  p.budget_ns = (d->flags & FDP_FLAG_TIMEOUT_SHORT) ? 200000000ull : 4000000000ull;
  p.mc = pl.stream_mc;
  p.fin_epi = env_int("FDP_FIN_EPI", 1);
  p.swizzle = env_int("FDP_STREAM_SWIZZLE", d->P >= 2 * d->D ? 8 : 0);
  p.dbg = env_int("FDP_DEBUG_STREAM", 0);
  if (env_int("FDP_STREAM_TRACE", 0)) {  // timing experiments: per-CTA wait totals (synchronous report)
    static unsigned long long* buf[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!buf[dev & 63] && cudaMalloc(&buf[dev & 63], 1024 * 8 * sizeof(unsigned long long)) != cudaSuccess)
      buf[dev & 63] = nullptr;
    p.trace = buf[dev & 63];
  }
  return p;
}

// FDP_STREAM_TRACE: mean / max over CTAs of each wait total, one JSON line on stderr
void stream_trace_report(const fdp::StreamParams& q, const char* what, int grid, cudaStream_t s) {
  if (!q.trace || grid > 1024) return;
  std::vector<unsigned long long> h(static_cast<size_t>(grid) * 8);
  cudaStreamSynchronize(s);
  cudaMemcpy(h.data(), q.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  static const char* names[8] = {"prod_wait_empty", "mma_wait_tempty", "mma_wait_full", "epi_wait_tfull",
                                 "epi_wait_prefill", "epi_store", "epi_end", "cta_end"};
  std::fprintf(stderr, "{\"stream_trace\": \"%s\", \"grid\": %d", what, grid);
  for (int k = 0; k < 8; ++k) {
    double sum = 0.0, mx = 0.0;
    for (int b = 0; b < grid; ++b) {
      const double v = static_cast<double>(h[static_cast<size_t>(b) * 8 + k]) * 1e-3;
      sum += v;
      mx = v > mx ? v : mx;
    }
    std::fprintf(stderr, ", \"%s_us\": [%.2f, %.2f]", names[k], sum / grid, mx);
  }
  if (env_int("FDP_STREAM_TRACE", 0) > 1) {  // every CTA's row
    std::fprintf(stderr, ", \"ctas\": [");
    for (int b = 0; b < grid; ++b) {
      std::fprintf(stderr, "%s[", b ? ", " : "");
      for (int k = 0; k < 8; ++k)
        std::fprintf(stderr, "%s%.1f", k ? ", " : "", static_cast<double>(h[static_cast<size_t>(b) * 8 + k]) * 1e-3);
      std::fprintf(stderr, "]");
    }
    std::fprintf(stderr, "]");
  }
  std::fprintf(stderr, "}\n");
  cudaMemset(q.trace, 0, h.size() * sizeof(unsigned long long));
}

// Grid of the stream-K kernel: every co-resident cluster, capped by the unit count.
int stream_grid(const fdp_desc* d, const Plan& pl, const DevInfo& di) {
  const long long units =
      static_cast<long long>(fdp::stream_wtiles(pl.n_wtiles, pl.n_pt, pl.stream_mc)) * d->B;
  if (pl.stream_mc == 2) {
    const long long clusters = std::max(1, fdp::stream_mc_max_clusters() - (reserved_sms() + 3) / 4);
    return static_cast<int>((units < clusters ? units : clusters) * 4);
  }
  const int cap = fdp::tc_max_coresident_ctas(pl.bn, pl.cg);
  const long long clusters = std::max(1, ((cap > 0 ? cap : di.sms) - reserved_sms()) / pl.cg);
  return static_cast<int>((units < clusters ? units : clusters) * pl.cg);
}

fdp::TcParams tc_params(const fdp_desc* d, const Plan& pl, const Common& c, float* grad_w, float* norms, void* ws,
                        int mode) {
  fdp::TcParams p{};
  p.B = static_cast<int>(d->B);
  p.T = static_cast<int>(d->T);
  p.P = static_cast<int>(d->P);
  p.D = static_cast<int>(d->D);
  p.n_dt2 = pl.n_dt;
  p.n_pt = pl.n_pt;
  p.n_wtiles = pl.n_wtiles;
  p.n_tiles = pl.n_tiles;
  p.groups = mode == fdp::MODE_FUSED ? pl.groups : 1;
  p.mode = mode;
  p.n_kb = static_cast<int>((d->T + fdp::kBK - 1) / fdp::kBK);
  p.clip_c = d->clip_c;
  p.clip_c2 = d->clip_c * d->clip_c;
  p.inv_batch = c.inv_batch;
  p.accumulate = d->accumulate;
  p.add_noise = c.add_noise;
  p.noise_impl = d->noise_impl;
  p.noise_scale = c.noise_scale;
  p.key_base = c.key_base;
  p.key_base_g = c.key_base_g;
  p.step_ptr = reinterpret_cast<const long long*>(d->device_step);
  p.seed_u = static_cast<uint64_t>(d->seed);
  p.layer_u = static_cast<uint64_t>(d->layer_id);
  p.noise_lo = c.noise_lo;
  p.noise_hi = c.noise_hi;
  p.grad_w = grad_w;
  p.norms_out = norms;
  p.g_out = nullptr;
  p.factors_in = ws_at<float>(ws, pl.off_factor);
  p.ws_part = ws_at<float>(ws, pl.off_part);
  p.ws_cnt = ws_at<unsigned>(ws, pl.off_cnt);
  p.ws_tagged = ws_at<unsigned long long>(ws, pl.off_tag);
  p.ws_tile_cnt = ws_at<unsigned>(ws, pl.off_tile_cnt);
  p.ws_ctrl = ws_at<unsigned>(ws, pl.off_ctrl);
  p.ws_acc = ws_at<float>(ws, pl.off_acc);
  p.skip_barrier = (d->flags & FDP_FLAG_SKIP_BARRIER) ? 1 : 0;
  p.deterministic = (d->flags & FDP_FLAG_DETERMINISTIC) ? 1 : 0;
  p.poll_ns = env_int("FDP_POLL_NS", 0);
  // epilogue-drawn noise for the reweight pass (see stream_params)
  p.epi_noise = (d->noise_impl == FDP_NOISE_PHILOX && env_int("FDP_EPI_NOISE", 1)) ? 1 : 0;
  p.pub_mode = env_int("FDP_PUB_MODE", 1);
  p.poll_mode = env_int("FDP_POLL_MODE", 0);
  p.budget_ns = (d->flags & FDP_FLAG_TIMEOUT_SHORT) ? 200000000ull : 4000000000ull;
  p.trace = (d->flags & FDP_FLAG_TRACE) ? ws_at<unsigned long long>(ws, pl.total - 1024ull * pl.grid) : nullptr;
  return p;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- workspace counters (include/fdp.h "Workspace"). Every kernel that uses the
// in-kernel counters (tile arrival / row-initialisation flags, exit counter) zeroes
// them again when it exits, but only in ITS layout: the counter range of a call
// lies at a shape-dependent place, so the first call with a new layout on a
// workspace could find stale non-zero words there (norm partials, factors, another
// layout's flags). The counters of every layout therefore live in one prefix
// [0, prefix) of the workspace, and the prefix is zeroed on the stream before a
// call whose layout differs from the previous call's on that workspace (and
// always while a stream is being captured, so every CUDA graph carries its own
// reset). Word 2 of the control block, the launch-tag generation of the tagged
// norm partials, is never reset: tags keep increasing per workspace, so a stale
// tagged partial can never pass for a fresh one.
uint64_t sig_mix(uint64_t h, uint64_t v) {
  h ^= v + kGamma + (h << 6) + (h >> 2);
  return fdp::mix64(h);
}

std::mutex g_ws_mu;
std::map<uintptr_t, uint64_t> g_ws_sig;

int ws_prepare(void* ws, uint64_t sig, size_t prefix, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamIsCapturing");
  bool need = true;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    const uintptr_t key = reinterpret_cast<uintptr_t>(ws);
    auto it = g_ws_sig.find(key);
    if (st == cudaStreamCaptureStatusNone && it != g_ws_sig.end() && it->second == sig) need = false;
    if (g_ws_sig.size() > 4096) g_ws_sig.clear();
    g_ws_sig[key] = sig;
  }
  if (!need) return FDP_OK;
  // exit counter + error word, then the counter arrays after the 256-byte control block
  if ((e = cudaMemsetAsync(ws, 0, 8, s)) != cudaSuccess) return cuda_fail(e, "workspace counter reset");
  if (prefix > 256 && (e = cudaMemsetAsync(static_cast<char*>(ws) + 256, 0, prefix - 256, s)) != cudaSuccess)
    return cuda_fail(e, "workspace counter reset");
  return FDP_OK;
}

uint64_t plan_sig(int32_t kind, const fdp_desc* d, const Plan& pl) {
  uint64_t h = 0x5eed;
  const long long v[] = {kind, pl.path, pl.norm_phase, pl.bn, pl.cg, pl.n_tiles, pl.n_wtiles, pl.stream_tiles,
                         pl.stream_mc, pl.groups, static_cast<long long>(pl.off_tile_cnt),
                         static_cast<long long>(pl.off_part), static_cast<long long>(pl.off_tag),
                         static_cast<long long>(pl.off_acc), d->B};
  for (long long x : v) h = sig_mix(h, static_cast<uint64_t>(x));
  return h;
}

int chain_flush(fdp_chain* c, cudaStream_t s) {
  if (!c || !c->pending) return FDP_OK;
  c->pending = false;
  ++c->flushed;
  cudaError_t e = fdp::single_sample_finalize(c->job, s);
  if (e != cudaSuccess) return cuda_fail(e, "deferred single-sample finalize");
  return FDP_OK;
}

// device slot for `n` partials of the next pending job (grown outside graph capture only)
float* chain_slot(fdp_chain* c, size_t n, cudaStream_t s) {
  const int k = c->slot;
  if (c->cap[k] >= n && c->part[k]) return c->part[k];
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess || st != cudaStreamCaptureStatusNone) return nullptr;
  if (c->part[k]) {
    cudaStreamSynchronize(s);
    cudaFree(c->part[k]);
    c->part[k] = nullptr;
    c->cap[k] = 0;
  }
  const size_t want = n < 4096 ? 4096 : n;
  if (cudaMalloc(reinterpret_cast<void**>(&c->part[k]), want * sizeof(float)) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  c->cap[k] = want;
  return c->part[k];
}

// pre_parts > 0: the two-phase ghost norm partials of this layer (pre_parts per sample)
// are already in the workspace (fdp_backward_shared_x); the norm phase is skipped.
// scale_out (fdp_dw_deferred): on the single-sample path without noise, leave the
// unclipped G in grad_w and write its clip factor x 1/mean_batch to scale_out[0]
// instead of running the elementwise pass (*deferred = true); the caller applies it.
int run(int32_t kind, const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms, void* ws,
        size_t ws_bytes, cudaStream_t s, fdp_chain* chain = nullptr, int pre_parts = 0, float* scale_out = nullptr,
        bool* deferred = nullptr) {
  int rc = validate(d, kind);
  if (rc) return rc;
  if (!x || !dy || !grad_w) return fail(FDP_ERR_USAGE, "null tensor pointer");
  if (kind != FDP_KIND_NON_DP && !norms) return fail(FDP_ERR_USAGE, "norms_sq must not be null for DP workflows");
  DevInfo di;
  if ((rc = get_dev(di))) return rc;
  Plan pl;
  if ((rc = make_plan(d, kind, di, pl))) return rc;
  if (!ws || ws_bytes < pl.total)
    return fail(FDP_ERR_CAPACITY, "workspace of %zu bytes is smaller than the %zu bytes this call needs", ws_bytes,
                pl.total);
  if (pl.tc && !(aligned16(x) && aligned16(dy)))
    return fail(FDP_ERR_USAGE, "x and dy must be 16-byte aligned for the tensor-core path");
  const Common c = common_of(d);
  cudaError_t e;

  // Deferred-finalize chain: a pending job is carried by this call's first stream-K
  // launch (single-sample GEMM, two-phase reweight, non-DP), else run standalone
  // first; it must not touch this call's buffers.
  const bool stream_k = env_int("FDP_STREAMK", 1) != 0;
  const bool has_stream_launch =
      pl.tc && d->in_dtype != FDP_DTYPE_F64 &&
      ((kind == FDP_KIND_NON_DP && stream_k) ||
       ((kind == FDP_KIND_FLASHDP || kind == FDP_KIND_IMPLICIT_DP) && pl.path == FDP_PATH_TWO_PHASE &&
        (pl.norm_phase == FDP_NORMS_SINGLE || stream_k)));
  fdp::FinJob carry{};
  if (chain && chain->pending) {
    const void* g = chain->job.g;
    const bool alias = g == grad_w || g == x || g == dy || g == norms;
    if (has_stream_launch && !alias && env_int("FDP_NO_CARRY", 0) == 0) {
      carry = chain->job;
      chain->pending = false;
      ++chain->carried;
    } else if ((rc = chain_flush(chain, s))) {
      return rc;
    }
  }

  if (d->in_dtype == FDP_DTYPE_F64) {  // fp64 parity path: every workflow kind computes the same quantity
    fdp::F64Params q{};
    q.B = static_cast<int>(d->B);
    q.T = static_cast<int>(d->T);
    q.P = static_cast<int>(d->P);
    q.D = static_cast<int>(d->D);
    q.n_dt = static_cast<int>((d->D + 31) / 32);
    q.n_pt = static_cast<int>((d->P + 31) / 32);
    q.n_tiles = q.n_dt * q.n_pt;
    q.x = static_cast<const double*>(x);
    q.dy = static_cast<const double*>(dy);
    q.grad_w = reinterpret_cast<double*>(grad_w);
    q.norms_out = reinterpret_cast<double*>(norms);
    q.part = ws_at<double>(ws, pl.off_part);
    q.factor = ws_at<double>(ws, pl.off_factor);
    q.with_clip = kind != FDP_KIND_NON_DP;
    q.clip_c = d->clip_c;
    const long long mb = d->mean_batch > 0 ? d->mean_batch : d->B;
    q.inv_batch = (q.with_clip && d->reduction == FDP_REDUCE_MEAN) ? 1.0 / static_cast<double>(mb) : 1.0;
    q.add_noise = c.add_noise;
    q.noise_impl = d->noise_impl;
    q.noise_scale = d->sigma * d->clip_c;
    q.key_base = c.key_base;
    q.key_base_g = c.key_base_g;
    q.step_ptr = reinterpret_cast<const long long*>(d->device_step);
    q.seed_u = static_cast<uint64_t>(d->seed);
    q.layer_u = static_cast<uint64_t>(d->layer_id);
    q.noise_lo = c.noise_lo;
    q.noise_hi = c.noise_hi;
    q.accumulate = d->accumulate;
    if ((e = fdp::f64_backward(q, s)) != cudaSuccess) return cuda_fail(e, "fp64 backward");
    return FDP_OK;
  }

  if (!pl.tc) {
    fdp::SimtParams sp = simt_params(d, pl, c, x, dy, grad_w, norms, ws);
    if (kind == FDP_KIND_NON_DP) {
      sp.with_clip = 0;
      if ((e = fdp::simt_weighted_sum(sp, s)) != cudaSuccess) return cuda_fail(e, "simt nondp");
      return FDP_OK;
    }
    if (kind == FDP_KIND_EXPLICIT_DP) {
      const long long DP = d->D * d->P;
      float* g = ws_at<float>(ws, pl.off_g);
      float* gp = ws_at<float>(ws, pl.off_gp);
      float* part = ws_at<float>(ws, pl.off_part);
      float* fac = ws_at<float>(ws, pl.off_factor);
      if ((e = fdp::explicit_store_g_simt(sp, g, s)) != cudaSuccess) return cuda_fail(e, "explicit G");
      if ((e = fdp::explicit_norms(g, sp.B, DP, part, pl.expl_chunks, s)) != cudaSuccess)
        return cuda_fail(e, "explicit norms");
      if ((e = fdp::reduce_norms_to_factors(part, sp.B, pl.expl_chunks, d->clip_c, sp.clip_c2, 1.0f, norms, fac, s)) !=
          cudaSuccess)
        return cuda_fail(e, "explicit reduce");
      if ((e = fdp::explicit_clip(g, gp, fac, sp.B, DP, s)) != cudaSuccess) return cuda_fail(e, "explicit clip");
      if ((e = fdp::explicit_sum_finalize(gp, sp.B, DP, sp.P, sp, s)) != cudaSuccess)
        return cuda_fail(e, "explicit sum");
      return FDP_OK;
    }
    // FLASHDP (generic) and IMPLICIT: norm pass, factor reduce, weighted pass
    if ((e = fdp::simt_partial_norms(sp, s)) != cudaSuccess) return cuda_fail(e, "simt norms");
    if ((e = fdp::reduce_norms_to_factors(sp.ws_part, sp.B, sp.n_tiles, d->clip_c, sp.clip_c2, c.inv_batch, norms,
                                          sp.ws_factor, s)) != cudaSuccess)
      return cuda_fail(e, "simt reduce");
    if ((e = fdp::simt_weighted_sum(sp, s)) != cudaSuccess) return cuda_fail(e, "simt weighted sum");
    return FDP_OK;
  }

  // ---- tensor-core paths
  if ((rc = ws_prepare(ws, plan_sig(kind, d, pl), pl.off_part, s))) return rc;
  CUtensorMap tm_dy, tm_x;
  if ((rc = make_tmap(&tm_dy, dy, d->D, d->T, d->B))) return rc;
  if ((rc = make_tmap(&tm_x, x, d->P, d->T, d->B))) return rc;
  fdp::EpiMaps em;
  em.gw = em.gw_slice = em.slot = em.slice = tm_dy;  // placeholders (unused by the modes that skip them)
  if (kind != FDP_KIND_EXPLICIT_DP) {
    // grad_w store / reduce-add map: the TMA epilogue of the fused, reweight and non-DP modes
    if ((reinterpret_cast<uintptr_t>(grad_w) & 15u) != 0)
      return fail(FDP_ERR_USAGE, "grad_w must be 16-byte aligned for the tensor-core path");
    const cuuint64_t gdims[2] = {static_cast<cuuint64_t>(d->P), static_cast<cuuint64_t>(d->D)};
    const cuuint64_t gstr[1] = {static_cast<cuuint64_t>(d->P * 4)};
    const cuuint32_t gbox[2] = {32, static_cast<cuuint32_t>(fdp::kBM)};
    if ((rc = make_tmap_f32(&em.gw, grad_w, 2, gdims, gstr, gbox))) return rc;
  }
  if (kind == FDP_KIND_FLASHDP && pl.path == FDP_PATH_FUSED) {
    const cuuint64_t gdims[2] = {static_cast<cuuint64_t>(d->P), static_cast<cuuint64_t>(d->D)};
    const cuuint64_t gstr[1] = {static_cast<cuuint64_t>(d->P * 4)};
    if (pl.groups > 1 && (d->flags & FDP_FLAG_DETERMINISTIC)) {
      const cuuint32_t rows_own = static_cast<cuuint32_t>(fdp::kBM / pl.groups);
      const cuuint32_t sbox[2] = {32, rows_own};
      if ((rc = make_tmap_f32(&em.gw_slice, grad_w, 2, gdims, gstr, sbox))) return rc;
      const cuuint64_t sdims[3] = {static_cast<cuuint64_t>(pl.bn), static_cast<cuuint64_t>(fdp::kBM),
                                   static_cast<cuuint64_t>(pl.n_tiles) * pl.groups};
      const cuuint64_t sstr[2] = {static_cast<cuuint64_t>(pl.bn * 4), static_cast<cuuint64_t>(pl.bn * 4 * fdp::kBM)};
      const cuuint32_t box_full[3] = {32, static_cast<cuuint32_t>(fdp::kBM), 1};
      const cuuint32_t box_sl[3] = {32, rows_own, 1};
      float* slots = ws_at<float>(ws, pl.off_acc);
      if ((rc = make_tmap_f32(&em.slot, slots, 3, sdims, sstr, box_full))) return rc;
      if ((rc = make_tmap_f32(&em.slice, slots, 3, sdims, sstr, box_sl))) return rc;
    }
    if ((reinterpret_cast<uintptr_t>(grad_w) & 15u) != 0)
      return fail(FDP_ERR_USAGE, "grad_w must be 16-byte aligned for the fused tensor-core path");
  }

  const bool use_stream = env_int("FDP_STREAMK", 1) != 0;
  if (kind == FDP_KIND_NON_DP) {
    if (use_stream) {
      fdp::StreamParams q = stream_params(d, pl, c, grad_w, ws, false);
      q.fin = carry;
      if ((e = fdp::launch_stream(pl.bn, pl.cg, tm_dy, tm_x, em.gw, q, stream_grid(d, pl, di), s)) != cudaSuccess)
        return cuda_fail(e, "stream-K nondp launch");
      stream_trace_report(q, "nondp", stream_grid(d, pl, di), s);
      return FDP_OK;
    }
    fdp::TcParams p = tc_params(d, pl, c, grad_w, nullptr, ws, fdp::MODE_NONDP);
    if ((e = fdp::launch_tc(pl.bn, pl.cg, tm_dy, tm_x, em, p, pl.grid, false, s)) != cudaSuccess)
      return cuda_fail(e, "tc nondp launch");
    return FDP_OK;
  }
  if (kind == FDP_KIND_EXPLICIT_DP) {
    const long long DP = d->D * d->P;
    float* g = ws_at<float>(ws, pl.off_g);
    float* gp = ws_at<float>(ws, pl.off_gp);
    float* part = ws_at<float>(ws, pl.off_part);
    float* fac = ws_at<float>(ws, pl.off_factor);
    fdp::TcParams p = tc_params(d, pl, c, grad_w, norms, ws, fdp::MODE_STORE_G);
    p.g_out = g;
    if ((e = fdp::launch_tc(pl.bn, pl.cg, tm_dy, tm_x, em, p, pl.grid, false, s)) != cudaSuccess)
      return cuda_fail(e, "tc explicit G launch");
    fdp::SimtParams sp = simt_params(d, pl, c, x, dy, grad_w, norms, ws);
    if ((e = fdp::explicit_norms(g, sp.B, DP, part, pl.expl_chunks, s)) != cudaSuccess)
      return cuda_fail(e, "explicit norms");
    if ((e = fdp::reduce_norms_to_factors(part, sp.B, pl.expl_chunks, d->clip_c, sp.clip_c2, 1.0f, norms, fac, s)) !=
        cudaSuccess)
      return cuda_fail(e, "explicit reduce");
    if ((e = fdp::explicit_clip(g, gp, fac, sp.B, DP, s)) != cudaSuccess) return cuda_fail(e, "explicit clip");
    if ((e = fdp::explicit_sum_finalize(gp, sp.B, DP, sp.P, sp, s)) != cudaSuccess)
      return cuda_fail(e, "explicit sum");
    return FDP_OK;
  }
  if (pl.path == FDP_PATH_FUSED) {
    fdp::TcParams p = tc_params(d, pl, c, grad_w, norms, ws, fdp::MODE_FUSED);
    if ((e = fdp::launch_tc(pl.bn, pl.cg, tm_dy, tm_x, em, p, pl.grid, true, s)) != cudaSuccess)
      return cuda_fail(e, "tc fused launch");
    return FDP_OK;
  }
  // TWO_PHASE, B == 1: the sample's gradient is the GEMM itself; its norm comes from
  // the GEMM epilogue and one elementwise pass applies the clip factor and the noise
  if (pl.norm_phase == FDP_NORMS_SINGLE) {
    fdp::StreamParams q = stream_params(d, pl, c, grad_w, ws, false);
    q.fin = carry;
    // with a chain, the partials go to a chain slot and this layer's finalize becomes
    // the chain's pending job (carried by the next call's GEMM, or fdp_chain_flush)
    float* slot = chain ? chain_slot(chain, static_cast<size_t>(pl.stream_tiles), s) : nullptr;
    q.norm_part = slot ? slot : ws_at<float>(ws, pl.off_part);
    if ((e = fdp::launch_stream(pl.bn, pl.cg, tm_dy, tm_x, em.gw, q, stream_grid(d, pl, di), s)) != cudaSuccess)
      return cuda_fail(e, "stream-K single-sample GEMM launch");
    fdp::FinJob j{};
    j.g = grad_w;
    j.n = d->D * d->P;
    j.part = q.norm_part;
    j.n_parts = pl.stream_tiles;
    j.clip_c = d->clip_c;
    j.clip_c2 = d->clip_c * d->clip_c;
    j.inv_batch = c.inv_batch;
    j.norms_out = norms;
    j.add_noise = c.add_noise;
    j.impl = d->noise_impl;
    j.scale = c.noise_scale;
    j.base = c.key_base;
    j.base_g = c.key_base_g;
    j.step_ptr = reinterpret_cast<const long long*>(d->device_step);
    j.seed_u = static_cast<uint64_t>(d->seed);
    j.layer_u = static_cast<uint64_t>(d->layer_id);
    j.lo = c.noise_lo;
    j.hi = c.noise_hi;
    if (slot) {
      chain->job = j;
      chain->pending = true;
      chain->slot ^= 1;
      return FDP_OK;
    }
    if (scale_out && !c.add_noise) {  // deferred clip: the consumer forms scale * G
      if ((e = fdp::single_sample_factor(j, scale_out, s)) != cudaSuccess)
        return cuda_fail(e, "single-sample clip factor");
      if (deferred) *deferred = true;
      return FDP_OK;
    }
    if ((e = fdp::single_sample_finalize(j, s)) != cudaSuccess) return cuda_fail(e, "single-sample finalize");
    return FDP_OK;
  }
  // TWO_PHASE, spill (opt-in): per-sample GEMMs to G[b] with their norms, factors, one combine pass
  if (pl.norm_phase == FDP_NORMS_SPILL) {
    float* G = ws_at<float>(ws, pl.off_g);
    CUtensorMap tm_g;
    const cuuint64_t gdims[3] = {static_cast<cuuint64_t>(d->P), static_cast<cuuint64_t>(d->D),
                                 static_cast<cuuint64_t>(d->B)};
    const cuuint64_t gstr[2] = {static_cast<cuuint64_t>(d->P * 4), static_cast<cuuint64_t>(d->P * d->D * 4)};
    const cuuint32_t gbox[3] = {32, static_cast<cuuint32_t>(fdp::kBM), 1};
    if ((rc = make_tmap_f32(&tm_g, G, 3, gdims, gstr, gbox))) return rc;
    fdp::StreamParams q = stream_params(d, pl, c, G, ws, false);
    q.spill = 1;
    q.accumulate = 0;
    q.add_noise = 0;
    q.epi_noise = 0;
    q.norm_part = ws_at<float>(ws, pl.off_part);
    q.fin = carry;
    if ((e = fdp::launch_stream(pl.bn, pl.cg, tm_dy, tm_x, tm_g, q, stream_grid(d, pl, di), s)) != cudaSuccess)
      return cuda_fail(e, "stream-K per-sample (spill) GEMM launch");
    float* fac = ws_at<float>(ws, pl.off_factor);
    if ((e = fdp::reduce_norms_to_factors(q.norm_part, static_cast<int>(d->B), pl.stream_tiles, d->clip_c,
                                          d->clip_c * d->clip_c, c.inv_batch, norms, fac, s)) != cudaSuccess)
      return cuda_fail(e, "factor reduce");
    if ((e = fdp::spill_combine(grad_w, G, static_cast<int>(d->B), d->D * d->P, fac, d->accumulate, c.add_noise,
                                d->noise_impl, c.noise_scale, c.key_base, c.key_base_g,
                                reinterpret_cast<const long long*>(d->device_step), static_cast<uint64_t>(d->seed),
                                static_cast<uint64_t>(d->layer_id), c.noise_lo, c.noise_hi, s)) != cudaSuccess)
      return cuda_fail(e, "spill combine");
    return FDP_OK;
  }
  // TWO_PHASE: norm phase (ghost Gram norms or recompute), factors, one reweighted pass
  {
    fdp::TcParams p = tc_params(d, pl, c, grad_w, norms, ws, fdp::MODE_NORMS);
    bool pdl = false;
    if (pl.norm_phase == FDP_NORMS_GHOST && pre_parts > 0) {
      // shared X: the partials come from the Gram launch (first layer) -- or wait on the
      // previous layer's reweight, which the PDL reduce does by itself (it waits for the
      // grid before it to complete)
      pdl = use_stream && env_int("FDP_PDL", 1) != 0;
      if ((e = fdp::reduce_norms_to_factors(p.ws_part, p.B, pre_parts, d->clip_c, p.clip_c2, c.inv_batch, norms,
                                            ws_at<float>(ws, pl.off_factor), s, pdl)) != cudaSuccess)
        return cuda_fail(e, "factor reduce");
    } else if (pl.norm_phase == FDP_NORMS_GHOST) {
      CUtensorMap gx, gy;
      if ((rc = make_tmap(&gx, x, d->P, d->T, d->B, 128))) return rc;
      if ((rc = make_tmap(&gy, dy, d->D, d->T, d->B, 128))) return rc;
      const GhostShape gs = ghost_shape(d, di.sms);
      fdp::GhostParams g{};
      g.B = p.B;
      g.T = p.T;
      g.P = p.P;
      g.D = p.D;
      g.nT = gs.nT;
      g.n_pairs = gs.n_pairs;
      g.split = gs.split;
      g.split_x = gs.split_x;
      g.n_full = gs.n_full;
      g.n_items = static_cast<int>(gs.units);
      g.part = p.ws_part;
      g.err = p.ws_ctrl + 1;
      g.budget_ns = p.budget_ns;
      if (gs.pair) {
        const int clusters = std::max(1, (di.sms - reserved_sms()) / 2);
        const int grid = 2 * (g.n_items < clusters ? g.n_items : clusters);
        if ((e = fdp::launch_ghost_pair(gx, gy, g, grid, s)) != cudaSuccess) return cuda_fail(e, "ghost-norm launch");
      } else {
        const int slots = std::max(1, di.sms - reserved_sms());
        const int grid = g.n_items < slots ? g.n_items : slots;
        if ((e = fdp::launch_ghost(gx, gy, g, grid, s)) != cudaSuccess) return cuda_fail(e, "ghost-norm launch");
      }
      // programmatic dependent launches (FDP_PDL, default on): the reduce and the reweight
      // are queued while the ghost kernel drains; only the reweight's epilogue waits
      pdl = use_stream && env_int("FDP_PDL", 1) != 0;
      if ((e = fdp::reduce_norms_to_factors(p.ws_part, p.B, gs.parts, d->clip_c, p.clip_c2, c.inv_batch, norms,
                                            ws_at<float>(ws, pl.off_factor), s, pdl)) != cudaSuccess)
        return cuda_fail(e, "factor reduce");
    } else {
      if ((e = fdp::launch_tc(pl.bn, pl.cg, tm_dy, tm_x, em, p, pl.grid, false, s)) != cudaSuccess)
        return cuda_fail(e, "tc norm-phase launch");
      if ((e = fdp::reduce_norms_to_factors(p.ws_part, p.B, pl.n_tiles, d->clip_c, p.clip_c2, c.inv_batch, norms,
                                            ws_at<float>(ws, pl.off_factor), s)) != cudaSuccess)
        return cuda_fail(e, "factor reduce");
    }
    if (use_stream) {  // stream-K over (tile, sample) units: no partial last wave
      fdp::StreamParams q = stream_params(d, pl, c, grad_w, ws, true);
      q.fin = carry;
      q.pdl = pdl ? 1 : 0;
      if ((e = fdp::launch_stream(pl.bn, pl.cg, tm_dy, tm_x, em.gw, q, stream_grid(d, pl, di), s)) != cudaSuccess)
        return cuda_fail(e, "stream-K reweight launch");
      stream_trace_report(q, "reweight", stream_grid(d, pl, di), s);
    } else {
      fdp::TcParams q = tc_params(d, pl, c, grad_w, norms, ws, fdp::MODE_REWEIGHT);
      if ((e = fdp::launch_tc(pl.bn, pl.cg, tm_dy, tm_x, em, q, pl.grid, false, s)) != cudaSuccess)
        return cuda_fail(e, "tc reweight launch");
    }
  }
  return FDP_OK;
}


// ---- multi-layer fused launch
struct GroupPlan {
  int bn = 0, cg = 1, grid = 0;
  std::vector<int> groups, c_off, n_dt2, n_pt, n_wtiles;
  std::vector<size_t> off_tagged, off_tile_cnt;
  size_t prefix = 0;  // end of the counter prefix (ws_prepare)
  size_t total = 0;
};

int plan_group_uncached(int32_t n, const fdp_desc* descs, const DevInfo& di, int max_ctas, GroupPlan& gpl);

// The packing search costs milliseconds; a training loop calls the same layer
// list every step, so plans are cached by (device, layer extents, flags, env).
int plan_group(int32_t n, const fdp_desc* descs, const DevInfo& di, int max_ctas, GroupPlan& gpl) {
  static std::mutex mu;
  static std::map<std::vector<long long>, GroupPlan> cache;
  std::vector<long long> key;
  key.reserve(4 * n + 8);
  key.push_back(di.dev);
  key.push_back(n);
  key.push_back(env_int("FDP_FORCE_BN", 0));
  key.push_back(env_int("FDP_FORCE_CG", 0));
  key.push_back(env_int("FDP_NO_PACK", 0));
  key.push_back(max_ctas);
  if (n > 0 && n <= fdp::kMaxGroupLayers) {
    key.push_back(descs[0].flags & FDP_FLAG_TRACE);
    for (int l = 0; l < n; ++l) {
      key.push_back(descs[l].B);
      key.push_back(descs[l].T);
      key.push_back(descs[l].P);
      key.push_back(descs[l].D);
    }
  }
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      // extents match a validated plan; the per-call descriptor fields are still checked
      for (int l = 0; l < n; ++l) {
        int rc = validate(&descs[l], FDP_KIND_FLASHDP);
        if (rc) return rc;
      }
      gpl = it->second;
      return FDP_OK;
    }
  }
  int rc = plan_group_uncached(n, descs, di, max_ctas, gpl);
  if (rc == FDP_OK) {
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 256) cache.clear();
    cache[key] = gpl;
  }
  return rc;
}

int plan_group_uncached(int32_t n, const fdp_desc* descs, const DevInfo& di, int max_ctas, GroupPlan& gpl) {
  if (n < 1 || n > fdp::kMaxGroupLayers)
    return fail(FDP_ERR_USAGE, "fdp_backward_group takes 1..%d layers, got %d", fdp::kMaxGroupLayers, n);
  if (di.major != 10) return fail(FDP_ERR_USAGE, "fdp_backward_group needs an sm_100 device");
  for (int l = 0; l < n; ++l) {
    int rc = validate(&descs[l], FDP_KIND_FLASHDP);
    if (rc) return rc;
    if (!tc_shape_ok(&descs[l]))
      return fail(FDP_ERR_USAGE, "layer %d is not tensor-core eligible (bf16, P %% 8 == 0, D %% 8 == 0)", l);
  }
  const int cands[4][2] = {{256, 2}, {128, 2}, {256, 1}, {128, 1}};
  const int forced_bn = env_int("FDP_FORCE_BN", 0), forced_cg = env_int("FDP_FORCE_CG", 0);
  const bool no_pack = env_int("FDP_NO_PACK", 0) != 0;
  // cost of splitting a tile's samples over g > 1 clusters (the groups' reduce-add combine),
  // and of a cluster holding ONE sample of a B > 1 layer: nothing to run while its norm
  // barrier resolves (with two or more, the next sample's MMAs overlap the wait)
  const double g_pen = 1e-9 * env_int("FDP_GROUP_GPEN_NS", 3000);
  const double x_pen = 1e-9 * env_int("FDP_GROUP_XPEN_NS", 5000);
  double best = 1e300;
  for (auto& cd : cands) {
    const int bn = cd[0], cg = cd[1];
    if ((forced_bn && bn != forced_bn) || (forced_cg && cg != forced_cg)) continue;
    long long cap = fdp::tc_max_coresident_ctas(bn, cg);
    if (max_ctas > 0 && cap > max_ctas) cap = max_ctas;  // SMs left free (e.g. for a concurrent NCCL kernel)
    if (cap < cg) continue;
    const int K = static_cast<int>(cap / cg);  // co-resident clusters
    const double rate = bn == 256 ? (cg == 2 ? 9.6e12 : 7.4e12) : (cg == 2 ? 6.4e12 : 6.3e12);
    // Pack layers onto cluster ranges: every cluster walks the layers in order,
    // so a layer's finish time on a cluster is (that cluster's load) + (its units'
    // time). For each layer pick the sample-group count g and the cyclic range
    // start that minimise the layer's finish time (ties: least idle time inside
    // the range, then fewer groups), e.g. GPT-2's c_attn (27 tiles x 2 groups)
    // and attn_proj (9 tiles x 2 groups) side by side on 54 + 18 clusters.
    std::vector<double> load(K, 0.0);
    bool ok = true;
    GroupPlan cand;
    cand.bn = bn;
    cand.cg = cg;
    for (int l = 0; l < n && ok; ++l) {
      const fdp_desc* d = &descs[l];
      const long long ndt = (d->D + fdp::kBM - 1) / fdp::kBM;
      const int ndt2 = static_cast<int>((ndt + cg - 1) / cg);
      const int npt = static_cast<int>((d->P + bn - 1) / bn);
      const int nwt = ndt2 * npt;
      if (nwt > K) { ok = false; break; }
      const double unit = std::max(2.0 * fdp::kBM * bn * static_cast<double>(d->T) / rate, 2.5e-6);
      double bfin = 1e300, bidle = 1e300;
      int bg = 0, boff = 0;
      const int gmax = static_cast<int>(std::min<long long>(std::min<long long>(d->B, 8), K / nwt));
      for (int g = 1; g <= gmax; ++g) {
        if (no_pack && (g & (g - 1))) continue;
        const int nc = nwt * g;
        const long long per = (d->B + g - 1) / g;
        const double t = static_cast<double>(per) * unit + (g > 1 ? g_pen : 0.0) + (per == 1 && d->B > 1 ? x_pen : 0.0);
        for (int off = 0; off < (no_pack ? 1 : K); ++off) {
          double m = 0.0, sum = 0.0;
          for (int i = 0; i < nc; ++i) {
            const double v = load[(off + i) % K];
            m = std::max(m, v);
            sum += v;
          }
          const double fin = m + t, idle = m * nc - sum;
          if (fin < bfin * (1 - 1e-9) || (fin <= bfin * (1 + 1e-9) && idle < bidle * (1 - 1e-9) - 1e-12)) {
            bfin = fin;
            bidle = idle;
            bg = g;
            boff = off;
          }
        }
      }
      if (no_pack && !bg) { ok = false; break; }
      for (int i = 0; i < nwt * bg; ++i) load[(boff + i) % K] = bfin;
      cand.groups.push_back(bg);
      cand.c_off.push_back(boff);
      cand.n_dt2.push_back(ndt2);
      cand.n_pt.push_back(npt);
      cand.n_wtiles.push_back(nwt);
      cand.grid = std::max(cand.grid, (boff + nwt * bg > K ? K : boff + nwt * bg) * cg);
    }
    if (!ok) continue;
    const double est = *std::max_element(load.begin(), load.end());
    if (est < best * 0.97) {
      best = est;
      gpl = cand;
    }
  }
  if (!gpl.bn) return fail(FDP_ERR_USAGE, "a layer does not fit the co-resident fused grid; use fdp_backward per layer");
  size_t off = 256;  // control words, then every layer's tile counters (the reset prefix), then the partials
  for (int l = 0; l < n; ++l) {
    gpl.off_tile_cnt.push_back(off);
    off += 4ull * gpl.n_wtiles[l] * gpl.cg;
  }
  off = align_up(off, 256);
  gpl.prefix = off;
  for (int l = 0; l < n; ++l) {
    gpl.off_tagged.push_back(off);
    off = align_up(off + 8ull * descs[l].B * gpl.n_wtiles[l] * gpl.cg, 256);
  }
  if (descs[0].flags & FDP_FLAG_TRACE) off += 2048ull * gpl.grid;  // [grid][256] u64
  gpl.total = off;
  return FDP_OK;
}

}  // namespace

extern "C" {

int fdp_abi_version(void) { return FDP_ABI_VERSION; }

const char* fdp_last_error(void) { return g_last_error.c_str(); }

int fdp_device_info(int32_t* sms, int32_t* cc_major, int32_t* cc_minor) {
  DevInfo di;
  int rc = get_dev(di);
  if (rc) return rc;
  if (sms) *sms = di.sms;
  if (cc_major) *cc_major = di.major;
  if (cc_minor) *cc_minor = di.minor;
  return FDP_OK;
}

int fdp_plan(const fdp_desc* d, int32_t kind, fdp_plan_info* out) {
  int rc = validate(d, kind);
  if (rc) return rc;
  if (!out) return fail(FDP_ERR_USAGE, "null plan output");
  DevInfo di;
  if ((rc = get_dev(di))) return rc;
  Plan pl;
  if ((rc = make_plan(d, kind, di, pl))) return rc;
  out->path = pl.path;
  out->norm_phase = pl.path == FDP_PATH_TWO_PHASE ? pl.norm_phase : 0;
  out->tile_d = pl.tc ? fdp::kBM * pl.cg : 32;
  out->tile_p = pl.tc ? pl.bn : 32;
  out->tile_t = pl.tc ? fdp::kBK : 32;
  out->n_d = pl.n_dt;
  out->n_p = pl.n_pt;
  out->groups = pl.groups;
  out->grid = pl.grid;
  out->launches = pl.launches;
  out->sms = di.sms;
  out->workspace_bytes = static_cast<int64_t>(pl.total);
  return FDP_OK;
}

int fdp_workspace_bytes(const fdp_desc* d, int32_t kind, size_t* bytes) {
  fdp_plan_info info;
  int rc = fdp_plan(d, kind, &info);
  if (rc) return rc;
  if (!bytes) return fail(FDP_ERR_USAGE, "null output");
  *bytes = static_cast<size_t>(info.workspace_bytes);
  return FDP_OK;
}

int fdp_workspace_init(void* ws, size_t ws_bytes, void* stream) {
  if (!ws && ws_bytes) return fail(FDP_ERR_USAGE, "null workspace");
  if (!ws_bytes) return FDP_OK;
  cudaError_t e = cudaMemsetAsync(ws, 0, ws_bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  return FDP_OK;
}

int fdp_backward(int32_t kind, const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms_sq,
                 void* ws, size_t ws_bytes, void* stream) {
  return run(kind, d, x, dy, grad_w, norms_sq, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int fdp_dw(const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms_sq, void* ws,
           size_t ws_bytes, void* stream) {
  return run(FDP_KIND_FLASHDP, d, x, dy, grad_w, norms_sq, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int fdp_dw_deferred(const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms_sq,
                    float* grad_scale, void* ws, size_t ws_bytes, void* stream) {
  if (!grad_scale) return fail(FDP_ERR_USAGE, "grad_scale must not be null");
  if (reinterpret_cast<uintptr_t>(grad_scale) & 3u) return fail(FDP_ERR_USAGE, "grad_scale must be 4-byte aligned");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  bool deferred = false;
  int rc = run(FDP_KIND_FLASHDP, d, x, dy, grad_w, norms_sq, ws, ws_bytes, s, nullptr, 0, grad_scale, &deferred);
  if (rc || deferred) return rc;
  fdp::FinJob none{};  // finalised in place: the consumer's scale is 1
  cudaError_t e = fdp::single_sample_factor(none, grad_scale, s);
  if (e != cudaSuccess) return cuda_fail(e, "grad_scale fill");
  return FDP_OK;
}

int fdp_backward_shared_x(int32_t n, const fdp_desc* descs, const void* x, const void* const* dy,
                          float* const* grad_w, float* const* norms_sq, void* const* ws, const size_t* ws_bytes,
                          void* stream) {
  if (n < 1 || n > 3) return fail(FDP_ERR_USAGE, "fdp_backward_shared_x takes 1..3 layers, got %d", n);
  if (!descs || !x || !dy || !grad_w || !norms_sq || !ws || !ws_bytes) return fail(FDP_ERR_USAGE, "null argument");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  for (int l = 0; l < n; ++l)
    if ((rc = validate(&descs[l], FDP_KIND_FLASHDP))) return rc;
  DevInfo di;
  if ((rc = get_dev(di))) return rc;
  // the shared X Gram applies when every layer runs the two-phase path with ghost norms on
  // the same (B, T, P) bf16 input; otherwise each layer runs on its own (same results)
  bool shared = n > 1 && env_int("FDP_SHARED_X", 1) != 0;
  Plan pls[3];
  const fdp_desc* d0 = &descs[0];
  for (int l = 0; l < n; ++l) {
    const fdp_desc* d = &descs[l];
    if ((rc = make_plan(d, FDP_KIND_FLASHDP, di, pls[l]))) return rc;
    if (d->B != d0->B || d->T != d0->T || d->P != d0->P || d->in_dtype != FDP_DTYPE_BF16 ||
        pls[l].path != FDP_PATH_TWO_PHASE || pls[l].norm_phase != FDP_NORMS_GHOST || !dy[l] || !aligned16(dy[l]))
      shared = false;
  }
  const long long nT2 = (d0->T + 255) / 256, np2 = nT2 * (nT2 + 1) / 2;
  const int parts = static_cast<int>(2 * np2);  // CTA-pair Gram tiles, no K split
  if (shared) {
    for (int l = 0; l < n; ++l) {
      const size_t need = static_cast<size_t>(d0->B) * parts * sizeof(float);
      if (!ws[l] || ws_bytes[l] < pls[l].total || pls[l].off_factor - pls[l].off_part < need || !aligned16(x))
        shared = false;
    }
  }
  if (shared) {
    CUtensorMap gx, gy[3];
    if ((rc = make_tmap(&gx, x, d0->P, d0->T, d0->B, 128))) return rc;
    for (int l = 0; l < n; ++l)
      if ((rc = make_tmap(&gy[l], dy[l], descs[l].D, descs[l].T, descs[l].B, 128))) return rc;
    fdp::GhostParams g{};
    g.B = static_cast<int>(d0->B);
    g.T = static_cast<int>(d0->T);
    g.P = static_cast<int>(d0->P);
    g.D = static_cast<int>(descs[0].D);
    g.nT = static_cast<int>(nT2);
    g.n_pairs = static_cast<int>(np2);
    g.split = 1;
    g.split_x = 1;
    g.n_items = g.n_pairs * g.B;
    g.part = ws_at<float>(ws[0], pls[0].off_part);
    g.err = ws_at<unsigned>(ws[0], pls[0].off_ctrl) + 1;
    g.budget_ns = (d0->flags & FDP_FLAG_TIMEOUT_SHORT) ? 200000000ull : 4000000000ull;
    g.n_dy = n;
    g.D1 = n > 1 ? static_cast<int>(descs[1].D) : 0;
    g.D2 = n > 2 ? static_cast<int>(descs[2].D) : 0;
    g.part1 = n > 1 ? ws_at<float>(ws[1], pls[1].off_part) : nullptr;
    g.part2 = n > 2 ? ws_at<float>(ws[2], pls[2].off_part) : nullptr;
    const int clusters = std::max(1, (di.sms - reserved_sms()) / 2);
    const int grid = 2 * (g.n_items < clusters ? g.n_items : clusters);
    cudaError_t e = fdp::launch_ghost_pair(gx, gy[0], g, grid, s, n > 1 ? &gy[1] : nullptr, n > 2 ? &gy[2] : nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "shared-X ghost-norm launch");
  }
  for (int l = 0; l < n; ++l)
    if ((rc = run(FDP_KIND_FLASHDP, &descs[l], x, dy[l], grad_w[l], norms_sq[l], ws[l], ws_bytes[l], s, nullptr,
                  shared ? parts : 0)))
      return rc;
  return FDP_OK;
}

int fdp_chain_create(fdp_chain** out) {
  if (!out) return fail(FDP_ERR_USAGE, "null output");
  *out = new (std::nothrow) fdp_chain();
  if (!*out) return fail(FDP_ERR_CAPACITY, "out of host memory");
  return FDP_OK;
}

int fdp_chain_destroy(fdp_chain* c) {
  if (!c) return FDP_OK;
  if (c->pending) return fail(FDP_ERR_USAGE, "fdp_chain_destroy: a finalize is still pending (fdp_chain_flush first)");
  for (int k = 0; k < 2; ++k)
    if (c->part[k]) cudaFree(c->part[k]);
  delete c;
  return FDP_OK;
}

int fdp_chain_flush(fdp_chain* c, void* stream) {
  if (!c) return fail(FDP_ERR_USAGE, "null chain");
  return chain_flush(c, static_cast<cudaStream_t>(stream));
}

int fdp_chain_stats(const fdp_chain* c, int64_t* carried, int64_t* flushed, int32_t* pending) {
  if (!c) return fail(FDP_ERR_USAGE, "null chain");
  if (carried) *carried = c->carried;
  if (flushed) *flushed = c->flushed;
  if (pending) *pending = c->pending ? 1 : 0;
  return FDP_OK;
}

int fdp_backward_chained(int32_t kind, const fdp_desc* d, const void* x, const void* dy, float* grad_w,
                         float* norms_sq, void* ws, size_t ws_bytes, fdp_chain* chain, void* stream) {
  if (!chain) return fail(FDP_ERR_USAGE, "null chain");
  return run(kind, d, x, dy, grad_w, norms_sq, ws, ws_bytes, static_cast<cudaStream_t>(stream), chain);
}

int fdp_dw_chained(const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms_sq, void* ws,
                   size_t ws_bytes, fdp_chain* chain, void* stream) {
  return fdp_backward_chained(FDP_KIND_FLASHDP, d, x, dy, grad_w, norms_sq, ws, ws_bytes, chain, stream);
}

int fdp_group_workspace_bytes_ex(int32_t n, const fdp_desc* descs, int32_t max_ctas, size_t* bytes) {
  if (!descs || !bytes) return fail(FDP_ERR_USAGE, "null argument");
  if (max_ctas < 0) return fail(FDP_ERR_USAGE, "max_ctas must be >= 0, got %d", max_ctas);
  DevInfo di;
  int rc = get_dev(di);
  if (rc) return rc;
  GroupPlan gpl;
  if ((rc = plan_group(n, descs, di, max_ctas, gpl))) return rc;
  *bytes = gpl.total;
  return FDP_OK;
}

int fdp_group_workspace_bytes(int32_t n, const fdp_desc* descs, size_t* bytes) {
  return fdp_group_workspace_bytes_ex(n, descs, 0, bytes);
}

int fdp_backward_group(int32_t n, const fdp_desc* descs, const void* const* x, const void* const* dy,
                       float* const* grad_w, float* const* norms_sq, void* ws, size_t ws_bytes, void* stream) {
  return fdp_backward_group_ex(n, descs, x, dy, grad_w, norms_sq, ws, ws_bytes, 0, stream);
}

int fdp_backward_group_ex(int32_t n, const fdp_desc* descs, const void* const* x, const void* const* dy,
                          float* const* grad_w, float* const* norms_sq, void* ws, size_t ws_bytes, int32_t max_ctas,
                          void* stream) {
  if (!descs || !x || !dy || !grad_w || !norms_sq) return fail(FDP_ERR_USAGE, "null argument");
  if (max_ctas < 0) return fail(FDP_ERR_USAGE, "max_ctas must be >= 0, got %d", max_ctas);
  DevInfo di;
  int rc = get_dev(di);
  if (rc) return rc;
  GroupPlan gpl;
  if ((rc = plan_group(n, descs, di, max_ctas, gpl))) return rc;
  if (!ws || ws_bytes < gpl.total)
    return fail(FDP_ERR_CAPACITY, "workspace of %zu bytes is smaller than the %zu bytes this call needs", ws_bytes,
                gpl.total);
  {
    uint64_t h = sig_mix(0x9409, static_cast<uint64_t>(n));
    h = sig_mix(h, static_cast<uint64_t>(gpl.bn * 4 + gpl.cg));
    for (int l = 0; l < n; ++l) {
      h = sig_mix(h, gpl.off_tile_cnt[l]);
      h = sig_mix(h, gpl.off_tagged[l]);
      h = sig_mix(h, static_cast<uint64_t>(gpl.n_wtiles[l]));
    }
    if ((rc = ws_prepare(ws, h, gpl.prefix, static_cast<cudaStream_t>(stream)))) return rc;
  }
  static thread_local fdp::GroupParams gp;  // ~28 KB: keep it off the stack
  std::memset(&gp, 0, sizeof(gp));
  for (int l = 0; l < n; ++l) {
    const fdp_desc* d = &descs[l];
    if (!x[l] || !dy[l] || !grad_w[l] || !norms_sq[l]) return fail(FDP_ERR_USAGE, "null tensor pointer (layer %d)", l);
    if (!(aligned16(x[l]) && aligned16(dy[l]) && aligned16(grad_w[l])))
      return fail(FDP_ERR_USAGE, "layer %d: x, dy and grad_w must be 16-byte aligned", l);
    fdp::GLayer& L = gp.L[l];
    if ((rc = make_tmap(&L.tm_dy, dy[l], d->D, d->T, d->B))) return rc;
    if ((rc = make_tmap(&L.tm_x, x[l], d->P, d->T, d->B))) return rc;
    const cuuint64_t gdims[2] = {static_cast<cuuint64_t>(d->P), static_cast<cuuint64_t>(d->D)};
    const cuuint64_t gstr[1] = {static_cast<cuuint64_t>(d->P * 4)};
    const cuuint32_t gbox[2] = {32, static_cast<cuuint32_t>(fdp::kBM)};
    if ((rc = make_tmap_f32(&L.gw, grad_w[l], 2, gdims, gstr, gbox))) return rc;
    const Common c = common_of(d);
    L.grad_w = grad_w[l];
    L.norms_out = norms_sq[l];
    L.tagged = ws_at<unsigned long long>(ws, gpl.off_tagged[l]);
    L.tile_cnt = ws_at<unsigned>(ws, gpl.off_tile_cnt[l]);
    L.key_base = c.key_base;
    L.key_base_g = c.key_base_g;
    L.step_ptr = reinterpret_cast<const long long*>(d->device_step);
    L.seed_u = static_cast<uint64_t>(d->seed);
    L.layer_u = static_cast<uint64_t>(d->layer_id);
    L.noise_lo = c.noise_lo;
    L.noise_hi = c.noise_hi;
    L.clip_c = d->clip_c;
    L.clip_c2 = d->clip_c * d->clip_c;
    L.inv_batch = c.inv_batch;
    L.noise_scale = c.noise_scale;
    L.B = static_cast<int>(d->B);
    L.T = static_cast<int>(d->T);
    L.P = static_cast<int>(d->P);
    L.D = static_cast<int>(d->D);
    L.n_dt2 = gpl.n_dt2[l];
    L.n_pt = gpl.n_pt[l];
    L.n_wtiles = gpl.n_wtiles[l];
    L.n_tiles = gpl.n_wtiles[l] * gpl.cg;
    L.groups = gpl.groups[l];
    L.c_off = gpl.c_off[l];
    L.n_kb = static_cast<int>((d->T + fdp::kBK - 1) / fdp::kBK);
    L.accumulate = d->accumulate;
    L.add_noise = c.add_noise;
    L.noise_impl = d->noise_impl;
  }
  gp.ctrl = ws_at<unsigned>(ws, 0);
  gp.budget_ns = (descs[0].flags & FDP_FLAG_TIMEOUT_SHORT) ? 200000000ull : 4000000000ull;
  gp.trace = (descs[0].flags & FDP_FLAG_TRACE) ? ws_at<unsigned long long>(ws, gpl.total - 2048ull * gpl.grid) : nullptr;
  gp.n_layers = n;
  gp.nosync = env_int("FDP_DEBUG_NOSYNC", 0);
  gp.dbg_tmem = env_int("FDP_DEBUG_GROUP_TMEM", 0);
  gp.dbg_noise = env_int("FDP_DEBUG_NOISE", 0);
  gp.poll_ns = env_int("FDP_POLL_NS", 0);
  gp.pub_mode = env_int("FDP_PUB_MODE", 1);
  gp.poll_mode = env_int("FDP_POLL_MODE", 0);
  gp.pf_ahead = env_int("FDP_PF_AHEAD", 0);
  gp.pair_dsmem = env_int("FDP_PAIR_DSMEM", 0);
  // small batches: a noised, non-accumulating layer whose tiles hold all its samples
  // (one sample group: reduce-add straight onto the rows, no pre-fill copy) gets its
  // noise drawn by the whole GPU first (fdp_group.cu k_group_noise); the group launch
  // then reduce-adds onto it. FDP_GROUP_PRENOISE_MAXB (default 2; 0 = off) bounds B:
  // from B = 3 the MMAs hide the noise warps' draws and the pass only adds a DRAM
  // round trip of grad_w (48 GPT-2 layers: B = 3 0.81 -> 0.99 ms).
  {
    const int maxb = env_int("FDP_GROUP_PRENOISE_MAXB", 2);
    bool pre[fdp::kMaxGroupLayers], any = false;
    for (int l = 0; l < n; ++l) {
      const fdp::GLayer& L = gp.L[l];
      pre[l] = maxb > 0 && L.add_noise && !L.accumulate && L.groups == 1 && L.B <= maxb;
      any |= pre[l];
    }
    if (any) {
      static thread_local fdp::GroupParams gn;  // the pass's view: only the pre-drawn layers noised
      gn = gp;
      for (int l = 0; l < n; ++l)
        if (!pre[l]) gn.L[l].add_noise = 0;
      cudaError_t e = fdp::launch_group_noise(gn, static_cast<cudaStream_t>(stream));
      if (e != cudaSuccess) return cuda_fail(e, "group noise launch");
      for (int l = 0; l < n; ++l)
        if (pre[l]) {
          gp.L[l].add_noise = 0;
          gp.L[l].accumulate = 1;
        }
    }
  }
  cudaError_t e = fdp::launch_group(gpl.bn, gpl.cg, gp, gpl.grid, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "group launch");
  return FDP_OK;
}

int fdp_noise(const fdp_desc* d, float* out, int64_t lo, int64_t hi, double scale, void* stream) {
  if (!d) return fail(FDP_ERR_USAGE, "null descriptor");
  if (lo < 0 || hi < lo) return fail(FDP_ERR_USAGE, "bad index range [%lld, %lld)", (long long)lo, (long long)hi);
  if (hi > lo && !out) return fail(FDP_ERR_USAGE, "null output");
  if (d->noise_impl < FDP_NOISE_KEYED_F32 || d->noise_impl > FDP_NOISE_PHILOX)
    return fail(FDP_ERR_USAGE, "unknown noise_impl %d", d->noise_impl);
  const uint64_t base = absorb3(d->seed, d->layer_id, d->step);
  cudaError_t e = fdp::noise_fill(out, lo, hi, scale, d->noise_impl, base, base + kGamma,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "noise_fill");
  return FDP_OK;
}

int fdp_noise_f64(const fdp_desc* d, double* out, int64_t lo, int64_t hi, double scale, void* stream) {
  if (!d) return fail(FDP_ERR_USAGE, "null descriptor");
  if (lo < 0 || hi < lo) return fail(FDP_ERR_USAGE, "bad index range [%lld, %lld)", (long long)lo, (long long)hi);
  if (hi > lo && !out) return fail(FDP_ERR_USAGE, "null output");
  if (d->noise_impl < FDP_NOISE_KEYED_F32 || d->noise_impl > FDP_NOISE_PHILOX)
    return fail(FDP_ERR_USAGE, "unknown noise_impl %d", d->noise_impl);
  const uint64_t base = absorb3(d->seed, d->layer_id, d->step);
  cudaError_t e = fdp::noise_fill64(out, lo, hi, scale, d->noise_impl, base, base + kGamma,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "noise_fill64");
  return FDP_OK;
}

// ---- non-linear parameter groups (fdp_params.cu)
namespace {
fdp::NoiseKey group_noise(const fdp_desc* d, long long L) {
  const Common c = common_of(d);
  fdp::NoiseKey nk{};
  nk.add_noise = c.add_noise;
  nk.impl = d->noise_impl;
  nk.scale = c.noise_scale;
  nk.base = c.key_base;
  nk.base_g = c.key_base_g;
  nk.step_ptr = reinterpret_cast<const long long*>(d->device_step);
  nk.seed_u = static_cast<uint64_t>(d->seed);
  nk.layer_u = static_cast<uint64_t>(d->layer_id);
  nk.lo = L * d->rank / d->world;  // the rank's slice of the group's own index space
  nk.hi = L * (d->rank + 1) / d->world;
  return nk;
}

int group_validate(const fdp_desc* d) {
  int rc = validate(d, FDP_KIND_FLASHDP);
  if (rc) return rc;
  if (d->in_dtype != FDP_DTYPE_BF16 && d->in_dtype != FDP_DTYPE_F32)
    return fail(FDP_ERR_USAGE, "parameter-group gradients take bf16 (0) or f32 (1) inputs, got dtype %d", d->in_dtype);
  if (d->B > (1 << 24) || d->T > (1 << 30) || d->D > (1 << 28)) return fail(FDP_ERR_SHAPE, "extent too large");
  return FDP_OK;
}

int check_ws(void* ws, size_t ws_bytes, size_t need) {
  if (!ws || ws_bytes < need)
    return fail(FDP_ERR_CAPACITY, "workspace of %zu bytes is smaller than the %zu bytes this call needs", ws_bytes,
                need);
  return FDP_OK;
}
}  // namespace

int fdp_vec_workspace_bytes(const fdp_desc* d, int32_t kind, size_t* bytes) {
  int rc = group_validate(d);
  if (rc) return rc;
  if (kind < FDP_VEC_BIAS || kind > FDP_VEC_LAYERNORM) return fail(FDP_ERR_USAGE, "unknown vector group kind %d", kind);
  if (!bytes) return fail(FDP_ERR_USAGE, "null output");
  *bytes = fdp::vec_dp_work_bytes(kind, static_cast<int>(d->B), static_cast<int>(d->T), static_cast<int>(d->D));
  return FDP_OK;
}

int fdp_vec_dw(const fdp_desc* d, int32_t kind, const void* dy, const void* xhat, float* grad, float* norms_sq,
               void* ws, size_t ws_bytes, void* stream) {
  size_t need = 0;
  int rc = fdp_vec_workspace_bytes(d, kind, &need);
  if (rc) return rc;
  if (!dy || !grad || (kind != FDP_VEC_BIAS && !xhat)) return fail(FDP_ERR_USAGE, "null tensor pointer");
  if ((rc = check_ws(ws, ws_bytes, need))) return rc;
  const Common c = common_of(d);
  const long long L = kind == FDP_VEC_LAYERNORM ? 2 * d->D : d->D;
  cudaError_t e = fdp::vec_dp(kind, dy, xhat, d->in_dtype == FDP_DTYPE_F32, static_cast<int>(d->B),
                              static_cast<int>(d->T), static_cast<int>(d->D), static_cast<float*>(ws), d->clip_c,
                              c.inv_batch, grad, norms_sq, d->accumulate ? 1 : 0, group_noise(d, L),
                              static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "vector-group dp");
  return FDP_OK;
}

int fdp_bias_workspace_bytes(const fdp_desc* d, size_t* bytes) {
  return fdp_vec_workspace_bytes(d, FDP_VEC_BIAS, bytes);
}

int fdp_bias_dw(const fdp_desc* d, const void* dy, float* grad_b, float* norms_sq, void* ws, size_t ws_bytes,
                void* stream) {
  return fdp_vec_dw(d, FDP_VEC_BIAS, dy, nullptr, grad_b, norms_sq, ws, ws_bytes, stream);
}

int fdp_embedding_workspace_bytes(const fdp_desc* d, size_t* bytes) {
  int rc = group_validate(d);
  if (rc) return rc;
  if (!bytes) return fail(FDP_ERR_USAGE, "null output");
  if (d->T > fdp::emb_max_tokens())
    return fail(FDP_ERR_SHAPE, "embedding gradients take T <= %d positions per sample, got %lld", fdp::emb_max_tokens(),
                (long long)d->T);
  if (d->P >= (1ll << 31)) return fail(FDP_ERR_SHAPE, "vocabulary too large");
  if (d->B > fdp::emb_max_batch())
    return fail(FDP_ERR_SHAPE, "embedding gradients take B <= %d samples per call, got %lld", fdp::emb_max_batch(),
                (long long)d->B);
  *bytes = fdp::emb_dp_work_bytes(static_cast<int>(d->B), static_cast<int>(d->T), static_cast<int>(d->D));
  return FDP_OK;
}

int fdp_embedding_dw(const fdp_desc* d, const int64_t* tokens, const void* dy, float* grad, float* norms_sq, void* ws,
                     size_t ws_bytes, void* stream) {
  size_t need = 0;
  int rc = fdp_embedding_workspace_bytes(d, &need);
  if (rc) return rc;
  if (!tokens || !dy || !grad) return fail(FDP_ERR_USAGE, "null tensor pointer");
  if (reinterpret_cast<uintptr_t>(grad) % 16 != 0) return fail(FDP_ERR_USAGE, "grad must be 16-byte aligned");
  if ((rc = check_ws(ws, ws_bytes, need))) return rc;
  const Common c = common_of(d);
  cudaError_t e = fdp::emb_dp(reinterpret_cast<const long long*>(tokens), dy, d->in_dtype == FDP_DTYPE_F32,
                              static_cast<int>(d->B), static_cast<int>(d->T), d->P, static_cast<int>(d->D), ws,
                              d->clip_c, c.inv_batch, grad, norms_sq, d->accumulate ? 1 : 0,
                              group_noise(d, d->P * d->D), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "embedding dp");
  return FDP_OK;
}

static int optim_common(int adam, int32_t dtype, void* theta, void* m, void* v, const void* grad, int64_t n,
                        double eta, double b1, double b2, double eps, const fdp_desc* noise, int64_t noise_offset,
                        void* stream, const float* grad_scale = nullptr) {
  if (grad_scale && dtype != FDP_DTYPE_F32) return fail(FDP_ERR_USAGE, "grad_scale needs fp32 state");
  if (grad_scale && (reinterpret_cast<uintptr_t>(grad_scale) & 3u))
    return fail(FDP_ERR_USAGE, "grad_scale must be 4-byte aligned");
  if (dtype != FDP_DTYPE_F32 && dtype != FDP_DTYPE_F64)
    return fail(FDP_ERR_USAGE, "optimizer state must be fp32 (1) or fp64 (2), got dtype %d", dtype);
  if (n < 0) return fail(FDP_ERR_SHAPE, "negative element count %lld", (long long)n);
  if (n > 0 && (!theta || !grad || (adam && (!m || !v)))) return fail(FDP_ERR_USAGE, "null tensor pointer");
  if (!(eta == eta) || !std::isfinite(eta)) return fail(FDP_ERR_USAGE, "eta must be finite");
  if (adam && !(b1 >= 0.0 && b1 < 1.0 && b2 >= 0.0 && b2 < 1.0))
    return fail(FDP_ERR_USAGE, "beta1 and beta2 must lie in [0, 1), got %g, %g", b1, b2);
  fdp::OptimNoise nz{};
  if (noise) {
    int rc = validate(noise, FDP_KIND_FLASHDP);
    if (rc) return rc;
    if (noise_offset < 0) return fail(FDP_ERR_USAGE, "noise_offset must be >= 0");
    const Common c = common_of(noise);
    nz.on = c.add_noise;
    nz.impl = noise->noise_impl;
    nz.scale = c.noise_scale;
    nz.base = c.key_base;
    nz.base_g = c.key_base_g;
    nz.step_ptr = reinterpret_cast<const long long*>(noise->device_step);
    nz.seed_u = static_cast<uint64_t>(noise->seed);
    nz.layer_u = static_cast<uint64_t>(noise->layer_id);
    nz.offset = noise_offset;
  }
  nz.grad_scale = grad_scale;
  cudaError_t e = fdp::optim_step(adam, dtype == FDP_DTYPE_F64, theta, m, v, grad, n, eta, b1, b2, eps, nz,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, adam ? "adam step" : "sgd step");
  return FDP_OK;
}

int fdp_sgd_step(int32_t dtype, void* theta, const void* grad, int64_t n, double eta, const fdp_desc* noise,
                 int64_t noise_offset, void* stream) {
  return optim_common(0, dtype, theta, nullptr, nullptr, grad, n, eta, 0.0, 0.0, 0.0, noise, noise_offset, stream);
}

int fdp_adam_step(int32_t dtype, void* theta, void* m, void* v, const void* grad, int64_t n, double eta,
                  double beta1, double beta2, double eps, const fdp_desc* noise, int64_t noise_offset, void* stream) {
  return optim_common(1, dtype, theta, m, v, grad, n, eta, beta1, beta2, eps, noise, noise_offset, stream);
}

int fdp_sgd_step_scaled(int32_t dtype, void* theta, const void* grad, const float* grad_scale, int64_t n, double eta,
                        const fdp_desc* noise, int64_t noise_offset, void* stream) {
  if (!grad_scale) return fail(FDP_ERR_USAGE, "grad_scale must not be null");
  return optim_common(0, dtype, theta, nullptr, nullptr, grad, n, eta, 0.0, 0.0, 0.0, noise, noise_offset, stream,
                      grad_scale);
}

int fdp_adam_step_scaled(int32_t dtype, void* theta, void* m, void* v, const void* grad, const float* grad_scale,
                         int64_t n, double eta, double beta1, double beta2, double eps, const fdp_desc* noise,
                         int64_t noise_offset, void* stream) {
  if (!grad_scale) return fail(FDP_ERR_USAGE, "grad_scale must not be null");
  return optim_common(1, dtype, theta, m, v, grad, n, eta, beta1, beta2, eps, noise, noise_offset, stream,
                      grad_scale);
}

int fdp_adam_multi_table_bytes(int32_t n_seg, size_t* bytes) {
  if (n_seg < 0 || !bytes) return fail(FDP_ERR_USAGE, "bad arguments");
  *bytes = static_cast<size_t>(n_seg) * sizeof(fdp::AdamSeg);
  return FDP_OK;
}

int fdp_adam_multi_prepare(int32_t n_seg, const fdp_adam_segment* segs, void* table, size_t table_bytes,
                           int64_t* total_quads, void* stream) {
  if (n_seg < 0 || (n_seg > 0 && (!segs || !table)) || !total_quads) return fail(FDP_ERR_USAGE, "bad arguments");
  if (table_bytes < static_cast<size_t>(n_seg) * sizeof(fdp::AdamSeg))
    return fail(FDP_ERR_CAPACITY, "segment table of %zu bytes is smaller than the %zu bytes needed", table_bytes,
                static_cast<size_t>(n_seg) * sizeof(fdp::AdamSeg));
  std::vector<fdp::AdamSeg> host(static_cast<size_t>(n_seg));
  long long q = 0;
  for (int i = 0; i < n_seg; ++i) {
    const fdp_adam_segment& a = segs[i];
    if (a.n < 0) return fail(FDP_ERR_SHAPE, "segment %d: negative element count", i);
    if (a.n > 0 && (!a.theta || !a.grad)) return fail(FDP_ERR_USAGE, "segment %d: null pointer", i);
    if (a.n > 0 && (!a.m != !a.v)) return fail(FDP_ERR_USAGE, "segment %d: m and v both set or both NULL", i);
    if (((reinterpret_cast<uintptr_t>(a.theta) | reinterpret_cast<uintptr_t>(a.m) |
          reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.grad)) & 15u) != 0)
      return fail(FDP_ERR_USAGE, "segment %d: theta / m / v / grad must be 16-byte aligned", i);
    if (a.grad_scale && (reinterpret_cast<uintptr_t>(a.grad_scale) & 3u))
      return fail(FDP_ERR_USAGE, "segment %d: grad_scale must be 4-byte aligned", i);
    fdp::AdamSeg& h = host[static_cast<size_t>(i)];
    h = fdp::AdamSeg{};
    h.theta = a.theta;
    h.m = a.m;
    h.v = a.v;
    h.g = a.grad;
    h.gscale = a.grad_scale;
    h.n = a.n;
    h.q0 = q;
    if (a.noise) {
      int rc = validate(a.noise, FDP_KIND_FLASHDP);
      if (rc) return rc;
      if (a.noise->noise_impl != FDP_NOISE_PHILOX || (a.noise_offset & 3) != 0 || a.noise_offset < 0)
        return fail(FDP_ERR_USAGE, "segment %d: multi-segment noise is Philox with a 4-aligned offset", i);
      const Common c = common_of(a.noise);
      h.noise_on = c.add_noise;
      h.scale = c.noise_scale;
      h.base = c.key_base;
      h.step_ptr = reinterpret_cast<const long long*>(a.noise->device_step);
      h.seed_u = static_cast<uint64_t>(a.noise->seed);
      h.layer_u = static_cast<uint64_t>(a.noise->layer_id);
      h.noise_q0 = a.noise_offset >> 2;
    }
    q += (a.n + 3) / 4;
  }
  *total_quads = q;
  if (n_seg == 0) return FDP_OK;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(table, host.data(), host.size() * sizeof(fdp::AdamSeg), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the host array goes out of scope
  if (e != cudaSuccess) return cuda_fail(e, "segment table upload");
  return FDP_OK;
}

int fdp_adam_step_multi(int32_t n_seg, const void* table, int64_t total_quads, double eta, double beta1,
                        double beta2, double eps, void* stream) {
  if (n_seg < 0 || (n_seg > 0 && !table) || total_quads < 0) return fail(FDP_ERR_USAGE, "bad arguments");
  if (!(eta == eta) || !std::isfinite(eta)) return fail(FDP_ERR_USAGE, "eta must be finite");
  if (!(beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0))
    return fail(FDP_ERR_USAGE, "beta1 and beta2 must lie in [0, 1), got %g, %g", beta1, beta2);
  cudaError_t e = fdp::adam_multi(static_cast<const fdp::AdamSeg*>(table), n_seg, total_quads, eta, beta1, beta2, eps,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "multi-segment adam step");
  return FDP_OK;
}

int fdp_sgd_step_multi(int32_t n_seg, const void* table, int64_t total_quads, double eta, void* stream) {
  if (n_seg < 0 || (n_seg > 0 && !table) || total_quads < 0) return fail(FDP_ERR_USAGE, "bad arguments");
  if (!(eta == eta) || !std::isfinite(eta)) return fail(FDP_ERR_USAGE, "eta must be finite");
  cudaError_t e = fdp::adam_multi(static_cast<const fdp::AdamSeg*>(table), n_seg, total_quads, eta, 0.0, 0.0, 0.0,
                                  static_cast<cudaStream_t>(stream), false);
  if (e != cudaSuccess) return cuda_fail(e, "multi-segment sgd step");
  return FDP_OK;
}

int fdp_noise_partition(int64_t n, int32_t rank, int32_t world, int64_t* lo, int64_t* hi) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world) return fail(FDP_ERR_USAGE, "bad partition arguments");
  if (lo) *lo = n * rank / world;
  if (hi) *hi = n * (rank + 1) / world;
  return FDP_OK;
}

}  // extern "C"
