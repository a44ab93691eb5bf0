// fdp_internal.h -- shared declarations between the C-ABI layer and the kernels.
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda.h>
#include <cuda_runtime.h>

namespace fdp {

constexpr int kBM = 128;  // d rows per output tile (UMMA M, one TMEM lane per row)
constexpr int kBK = 64;   // t extent of one pipeline stage (4 x UMMA K=16)
constexpr int kEpiWarps = 8;
constexpr int kEpiWarp0 = 4;  // warpgroup 0: warp 0 TMA producer, warp 1 MMA issuer, 2 spare
constexpr int kTcThreads = 32 * kEpiWarp0 + 32 * kEpiWarps;  // warpgroups 1-2: epilogue

enum TcMode : int {
  MODE_FUSED = 0,     // per-sample G tile -> norm all-reduce + grid barrier -> clip -> sum -> noise
  MODE_NORMS = 1,     // per-sample G tile -> partial norm^2 only (recompute norm phase)
  MODE_REWEIGHT = 2,  // per-sample G tile scaled by a precomputed factor -> sum -> noise
  MODE_STORE_G = 3,   // per-sample G tile stored to HBM (explicit / Opacus-style stage 1)
  MODE_NONDP = 4      // plain sum_b dY_b^T X_b (non-DP baseline)
};

struct TcParams {
  int B, T, P, D;
  int n_dt2;     // work-tile rows: ceil(ceil(D/128) / CG)   (a work tile is CG x 128 d-rows x BN p-cols)
  int n_pt;      // work-tile columns: ceil(P / BN)
  int n_wtiles;  // n_dt2 * n_pt
  int n_tiles;   // CTA-level tiles = n_wtiles * CG (one norm partial per CTA tile and sample)
  int groups;  // sample groups per output tile (FUSED)
  int mode;
  int n_kb;
  double clip_c;
  double clip_c2;
  float inv_batch;
  int accumulate;
  int add_noise;
  int noise_impl;
  float noise_scale;
  uint64_t key_base;    // absorb(seed, layer_id, step)
  uint64_t key_base_g;  // key_base + GAMMA
  const long long* step_ptr;  // device step counter (nullptr: use key_base)
  uint64_t seed_u, layer_u;
  long long noise_lo, noise_hi;
  float* grad_w;
  float* norms_out;
  float* g_out;
  const float* factors_in;
  float* ws_part;          // [B][n_tiles] (NORMS mode)
  unsigned long long* ws_tagged;  // [B][n_tiles] {float partial, uint32 launch tag} (FUSED mode)
  unsigned* ws_cnt;        // [B]
  unsigned* ws_tile_cnt;   // [n_tiles]
  unsigned* ws_ctrl;       // [0] exit counter, [1] error word
  float* ws_acc;           // [n_tiles][groups][kBM*BN]
  int skip_barrier;
  int deterministic;
  int epi_noise;  // MODE_REWEIGHT: draw Philox noise in the epilogue (no grad_w pre-fill)
  // publish the tagged norm partial with an L2 atomic exchange (1, default: reaches L2 at once;
  // 0 = st.relaxed, 2 = st.release) and poll with ld.relaxed (0) / volatile (1) / acquire (2)
  int pub_mode, poll_mode;
  int poll_ns;  // back-off between polls of the norm partials (FDP_POLL_NS, default 0: spin)
  unsigned long long budget_ns;
  unsigned long long* trace;  // [grid][128] phase timestamps or nullptr
};

// Launch the tcgen05 kernel: BN = 128 or 256 output columns per CTA, CG = 1 or
// 2 CTAs per MMA (cta_group::2 pairs two SMs on a 256-row tile). cooperative=true
// for MODE_FUSED (all CTAs must be co-resident for the in-kernel barriers).
// TMA maps of the fused epilogue: grad_w (D,P) fp32 with 32x128 and 32xrows_own
// boxes, and the reduce-scatter slots [n_tiles*groups][128][BN] (full / slice boxes).
struct EpiMaps {
  CUtensorMap gw, gw_slice, slot, slice;
};
cudaError_t launch_tc(int bn, int cg, const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const EpiMaps& em,
                      const TcParams& p, int grid, bool cooperative, cudaStream_t stream);
// Upper bound on co-resident CTAs of the (bn, cg) kernel on this device (0: cannot run).
int tc_max_coresident_ctas(int bn, int cg);

// Deferred finalize of a single-sample layer (B == 1): grad_w <- c * G + sigma*C*noise
// with c from the layer's norm partials (dpcore.py:41-47, 60-73). Run standalone
// (single_sample_finalize) or carried by the NEXT stream-K launch, whose idle noise
// and epilogue warps stream it while the tensor cores run that launch's GEMM.
struct FinJob {
  float* g;               // (D, P) fp32 gradient holding the unclipped G (nullptr: no job)
  long long n;            // D * P (P % 8 == 0)
  const float* part;      // per-tile sums of squares of G
  int n_parts;
  double clip_c, clip_c2;
  float inv_batch;
  float* norms_out;       // (1,) ||G||^2 or nullptr
  int add_noise, impl;
  float scale;
  uint64_t base, base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long lo, hi;       // the rank's noise slice of [0, n)
};

// ---- stream-K persistent kernel (fdp_stream.cu): two-phase reweight pass and non-DP dW
struct StreamParams {
  int B, P, D, n_pt, n_wtiles, n_kb;
  int reweight;     // 1: acc += factors_in[b] * G_b per sample; 0: plain sum over samples (non-DP)
  int accumulate, add_noise, epi_noise, noise_impl;
  float noise_scale;
  uint64_t key_base, key_base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long noise_lo, noise_hi;
  float* grad_w;
  const float* factors_in;  // [B] clip factor x mean scale
  unsigned* tile_cnt;       // [n_wtiles * CG] row-initialisation flags (left zeroed)
  float* norm_part;         // B == 1 single-sample path: sum of squares of each CTA tile ([n_wtiles * CG]) or null
  unsigned* ctrl;           // [0] exit counter, [1] error word
  unsigned long long budget_ns;
  int mc;                   // 2: 4-CTA clusters (two pairs, X boxes multicast; bn 256, cg 2), else 1
  FinJob fin;               // carried deferred finalize of the previous single-sample layer (fin.g == nullptr: none)
  int fin_epi;              // epilogue warps also stream the carried finalize while idle (FDP_FIN_EPI)
  // spill norm phase: every (tile, sample) unit is its own whole tile, stored unscaled to
  // the per-sample buffer G[b] (tm_gw is then a 3-D (P, D, B) map) with its sum of
  // squares in norm_part[(b * n_wtiles + wt) * CG * MC + crank]; p.B is the real batch
  int spill;
  int swizzle;  // tile raster: 0/1 row-major, G > 1 grouped by G row blocks (FDP_STREAM_SWIZZLE)
  int dbg;      // timing experiments only (FDP_DEBUG_STREAM): 1 skip the TMEM readout, 2 skip the MMAs
  unsigned long long* trace;  // FDP_STREAM_TRACE: per-CTA wait-time totals [gridDim.x][8] (ns), or null
  int pdl;  // launched as a programmatic dependent of the factor reduce (epilogue waits on it)
};
// Work tiles of the stream kernel (MC pair tiles stacked along D) and its per-CTA tile slots.
inline int stream_wtiles(int n_wtiles, int n_pt, int mc) {
  return mc == 2 ? ((n_wtiles / n_pt + 1) / 2) * n_pt : n_wtiles;
}
int stream_mc_max_clusters();
// grid <= co-resident CTAs (split tiles wait on the cluster that initialises them)
cudaError_t launch_stream(int bn, int cg, const CUtensorMap& tm_dy, const CUtensorMap& tm_x, const CUtensorMap& tm_gw,
                          const StreamParams& p, int grid, cudaStream_t stream);

// ---- multi-layer fused launch (fdp_group.cu)
struct GLayer {
  CUtensorMap tm_dy, tm_x, gw;  // operand maps (box 64x64 bf16) and the grad_w store map (32x128 fp32)
  float* grad_w;
  float* norms_out;
  unsigned long long* tagged;   // [B][n_tiles] tagged norm partials
  unsigned* tile_cnt;           // [n_tiles] sample-group arrivals
  uint64_t key_base, key_base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long noise_lo, noise_hi;
  double clip_c, clip_c2;
  float inv_batch, noise_scale;
  int B, T, P, D, n_dt2, n_pt, n_wtiles, n_tiles, groups, n_kb;
  int accumulate, add_noise, noise_impl;
  int c_off;  // first cluster of this layer's range (layers are packed onto cluster ranges, fdp_capi.cu)
};
constexpr int kMaxGroupLayers = 48;  // keeps the parameter block under 32 KB
struct GroupParams {
  GLayer L[kMaxGroupLayers];
  unsigned* ctrl;  // [0] exit counter, [1] error word, [2] launch epoch
  unsigned long long budget_ns;
  unsigned long long* trace;  // [grid][256] per-layer phase timestamps (FDP_FLAG_TRACE) or nullptr
  int n_layers;
  int dbg_noise;  // debug (FDP_DEBUG_NOISE): 1 = no draws (zero pre-fill), 2 = draws scaled by 0
  int pub_mode, poll_mode, poll_ns;  // experiments (FDP_PUB_MODE, FDP_POLL_MODE, FDP_POLL_NS)
  int nosync;  // debug (FDP_DEBUG_NOSYNC): clip factors from whatever partials are present, no wait
  int dbg_tmem;  // timing experiments only (FDP_DEBUG_GROUP_TMEM): 1 skip the norm pass's TMEM loads, 2 the clip pass's
  // noise / row pre-fill run-ahead bound: the noise warps start layer l once the
  // epilogue has started layer l - pf_ahead (FDP_PF_AHEAD; < 0 = unbounded)
  int pf_ahead;
  int pair_dsmem;  // CTA-pair norm partials combined in DSMEM before publishing (FDP_PAIR_DSMEM; default off)
};
cudaError_t launch_group(int bn, int cg, const GroupParams& gp, int grid, cudaStream_t stream);
cudaError_t launch_group_noise(const GroupParams& gp, cudaStream_t stream);  // pre-drawn noise (fdp_group.cu)

// ---- ghost norms (TWO_PHASE first phase): ||G_b||^2 = <X_b X_b^T, dY_b dY_b^T>
struct GhostParams {
  int B, T, P, D;
  int nT;        // ceil(T / 128)
  int n_pairs;   // nT (nT + 1) / 2 upper-triangle Gram tile pairs per sample
  int n_items;   // B * n_pairs * split
  int split;     // K slices of the larger operand per tile pair (1 = none)
  int split_x;   // 1: slice X's K (P >= D), 0: slice dY's K
  int n_full;    // > 0: mixed schedule -- work units [0, n_full) are whole items, the rest split `split` ways
  float* part;   // [B][n_pairs][split] weighted partials (x2 for the CTA-pair kernel)
  unsigned* err;
  unsigned long long budget_ns;
  // CTA-pair kernel only: n_dy (2 or 3) layers sharing X -- one X Gram per item, one dY
  // Gram per layer (split must be 1); layer l in {1, 2} has D_l and its partials in part_l
  int n_dy;
  int D1, D2;
  float *part1, *part2;
};
cudaError_t launch_ghost(const CUtensorMap& tm_x, const CUtensorMap& tm_dy, const GhostParams& p, int grid,
                         cudaStream_t stream);
// CTA-pair variant: 256x256 Gram tiles (nT = ceil(T/256)), partials [B][n_pairs][2], grid = 2 x clusters.
cudaError_t launch_ghost_pair(const CUtensorMap& tm_x, const CUtensorMap& tm_dy, const GhostParams& p, int grid,
                              cudaStream_t stream, const CUtensorMap* tm_dy1 = nullptr,
                              const CUtensorMap* tm_dy2 = nullptr);

// ---- SIMT (CUDA-core) kernels: generic shapes, fp32 inputs, explicit baseline
struct SimtParams {
  int B, T, P, D;
  int in_f32;  // 1: fp32 inputs, 0: bf16
  const void* x;
  const void* dy;
  int n_dt, n_pt, n_tiles;  // 32x32 tiles
  double clip_c;
  double clip_c2;
  float inv_batch;
  int accumulate;
  int add_noise;
  int noise_impl;
  float noise_scale;
  uint64_t key_base, key_base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long noise_lo, noise_hi;
  float* grad_w;
  float* norms_out;
  float* ws_part;     // [B][n_tiles]
  float* ws_factor;   // [B]
  int with_clip;      // 0: non-DP sum
};
cudaError_t simt_partial_norms(const SimtParams& p, cudaStream_t s);
// pdl: launched as a programmatic dependent of the norm-phase kernel (starts while it drains)
cudaError_t reduce_norms_to_factors(const float* part, int B, int n_tiles, double clip_c, double clip_c2,
                                    float inv_batch, float* norms_out, float* factors, cudaStream_t s,
                                    bool pdl = false);
cudaError_t simt_weighted_sum(const SimtParams& p, cudaStream_t s);

// explicit (Opacus-style) stages over a materialised G (B,D,P)
cudaError_t explicit_store_g_simt(const SimtParams& p, float* g, cudaStream_t s);
cudaError_t explicit_norms(const float* g, int B, long long DP, float* part, int nchunks, cudaStream_t s);
cudaError_t explicit_clip(const float* g, float* gp, const float* factors, int B, long long DP, cudaStream_t s);
cudaError_t explicit_sum_finalize(const float* gp, int B, long long DP, int P, const SimtParams& p,
                                  cudaStream_t s);

// B == 1 second pass: ||G||^2 from the per-tile partials (fixed order), then
// grad_w = grad_w * min(1, C/||G||) * inv_batch (+ sigma*C*noise on [lo, hi)).
cudaError_t single_sample_finalize(const FinJob& j, cudaStream_t s);
// deferred clip: scale_out[0] = c * inv_batch and norms_out[0] = ||G||^2 from j's
// partials, grad_w untouched (j.part == nullptr: scale_out[0] = 1)
cudaError_t single_sample_factor(const FinJob& j, float* scale_out, cudaStream_t s);
// spill combine: out = (accumulate ? out : 0) + sum_b fac[b] * G[b] + scale * noise (rank slice)
cudaError_t spill_combine(float* out, const float* G, int B, long long n, const float* fac, int accumulate,
                          int add_noise, int impl, float scale, uint64_t base, uint64_t base_g,
                          const long long* step_ptr, uint64_t seed_u, uint64_t layer_u, long long lo, long long hi,
                          cudaStream_t s);
cudaError_t single_sample_finalize(float* grad_w, long long n, const float* part, int n_parts, double clip_c,
                                   double clip_c2, float inv_batch, float* norms_out, int add_noise, int impl,
                                   float noise_scale, uint64_t base, uint64_t base_g, const long long* step_ptr,
                                   uint64_t seed_u, uint64_t layer_u, long long lo, long long hi, cudaStream_t s);

// ---- fp64 parity path (fdp_f64.cu): in_dtype FDP_DTYPE_F64, fp64 in / out
struct F64Params {
  int B, T, P, D, n_dt, n_pt, n_tiles;
  const double* x;
  const double* dy;
  double* grad_w;
  double* norms_out;
  double* part;    // [B][n_tiles]
  double* factor;  // [B]
  int with_clip, add_noise, noise_impl, accumulate;
  double clip_c, inv_batch, noise_scale;
  uint64_t key_base, key_base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long noise_lo, noise_hi;
};
cudaError_t f64_backward(const F64Params& p, cudaStream_t s);

// Noise of one parameter group: scale * N(key, i) for flat i in [lo, hi); the key
// comes from step_ptr (device counter) when set.
struct NoiseKey {
  int add_noise, impl;
  float scale;
  uint64_t base, base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long lo, hi;
};
// fdp_params.cu: bias / RMSNorm / LayerNorm vector groups (kind = FDP_VEC_*) and embedding tables
size_t vec_dp_work_bytes(int kind, int B, int T, int D);
cudaError_t vec_dp(int kind, const void* dy, const void* xhat, int in_f32, int B, int T, int D, float* work,
                   double clip_c, float inv_batch, float* out, float* norms_out, int accumulate, const NoiseKey& nk,
                   cudaStream_t s);
size_t emb_dp_work_bytes(int B, int T, int D);
int emb_max_tokens();
int emb_max_batch();
cudaError_t emb_dp(const long long* tokens, const void* dy, int in_f32, int B, int T, long long V, int D, void* work,
                   double clip_c, float inv_batch, float* out, float* norms_out, int accumulate, const NoiseKey& nk,
                   cudaStream_t s);

// ---- optimizer steps (fdp_optim.cu)
struct OptimNoise {
  int on, impl;
  float scale;
  uint64_t base, base_g;
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
  long long offset;
  const float* grad_scale;  // nullptr or a device scalar: g = grad_scale[0] * grad before the noise (fp32 only)
};
// one segment of a multi-segment fp32 Adam step (device table entry)
struct AdamSeg {
  float *theta, *m, *v;
  const float* g;
  const float* gscale;   // nullptr or a device scalar multiplied into g first
  long long n;           // elements
  long long q0;          // first quad of this segment in the launch's quad space
  long long noise_q0;    // Philox block of the segment's element 0 (noise offset / 4)
  int noise_on;
  float scale;           // sigma * C
  uint64_t base;         // Philox key (absorb(seed, layer, step)) when step_ptr is null
  const long long* step_ptr;
  uint64_t seed_u, layer_u;
};
cudaError_t adam_multi(const AdamSeg* dev_segs, int n_seg, long long total_q, double eta, double b1, double b2,
                       double eps, cudaStream_t s, bool adam = true);
cudaError_t optim_step(int adam, int f64, void* theta, void* m, void* v, const void* g, long long n, double eta,
                       double b1, double b2, double eps, const OptimNoise& nz, cudaStream_t s);

cudaError_t noise_fill(float* out, long long lo, long long hi, double scale, int impl, uint64_t base,
                       uint64_t base_g, cudaStream_t s);
cudaError_t noise_fill64(double* out, long long lo, long long hi, double scale, int impl, uint64_t base,
                         uint64_t base_g, cudaStream_t s);

}  // namespace fdp
