/*
 * fdp.h -- C ABI of the B200-native FlashDP per-layer DP weight-gradient backward.
 *
 * This is the drop-in boundary for the reference's hot path
 *   dpflows.workflows.run_backward / backward_flashdp
 *   (/root/reference/pkg/src/dpflows/workflows.py:340-440)
 * The reference binds nothing native (it is numpy); the Python mirror in
 * paper_2507_01154_b200/_lib.py binds these symbols with ctypes, exactly as a
 * maintainer would bind them from dpflows.
 *
 * Conventions (all entry points):
 *   - Layer convention Y = X W^T: X is (B,T,P), dY is (B,T,D), row-major,
 *     grad_w is (D,P) fp32 row-major (= nn.Linear.weight layout),
 *     norms_sq is (B,) fp32 (workflows.py:1-5, 40-44).
 *   - All pointers are DEVICE pointers owned by the caller. Nothing is
 *     allocated and nothing synchronises the host on the hot path.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - Work is stream-ordered. Two calls that may overlap (different streams)
 *     need distinct workspaces: the workspace holds the in-kernel norm
 *     all-reduce counters (the analogue of memmodel.py:261-285).
 *   - A workspace must be zero-filled once before first use
 *     (fdp_workspace_init). Only its counter prefix has to stay zero between
 *     calls (tile arrival / row-initialisation flags, exit counter): every call
 *     leaves the counters of ITS layout zeroed, and a call whose layout differs
 *     from the previous call's on the same workspace (a different shape, kind or
 *     layer list) first zeroes the prefix on the stream (cudaMemsetAsync; always
 *     done while the stream is being captured). Norm partials, clip factors and
 *     explicit-path buffers are scratch: rewritten before they are read.
 *   - Return codes mirror the reference exception types (errors.py):
 *     FDP_ERR_SHAPE    -> ShapeError   (workflows.py:47-52)
 *     FDP_ERR_USAGE    -> UsageError   (dpcore.py:32-38, workflows.py:330-337)
 *     FDP_ERR_CAPACITY -> CapacityError (workspace too small; errors.py:12-22)
 *     FDP_ERR_CUDA     -> RuntimeError (launch/device failure)
 *   fdp_last_error() returns the message of the last failing call on the
 *   calling host thread.
 */
#ifndef FDP_H_
#define FDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FDP_ABI_VERSION 1

#if defined(__GNUC__)
#define FDP_API __attribute__((visibility("default")))
#else
#define FDP_API
#endif

enum fdp_status {
  FDP_OK = 0,
  FDP_ERR_SHAPE = 1,
  FDP_ERR_USAGE = 2,
  FDP_ERR_CAPACITY = 3,
  FDP_ERR_CUDA = 4
};

/* Input element type of X and dY. bf16 / f32: fp32 accumulation and fp32
 * grad_w / norms_sq. F64 (the reference's own precision): the fp64 parity path --
 * X, dY are double and grad_w / norms_sq point to DOUBLE arrays (cast through
 * the float* parameters), fp64 FMA on the CUDA cores, keyed noise transformed in
 * fp64; every workflow kind computes the same quantity. Also the optimizer
 * steps' fp64 state. */
enum fdp_dtype { FDP_DTYPE_BF16 = 0, FDP_DTYPE_F32 = 1, FDP_DTYPE_F64 = 2 };

/* dpcore.REDUCTIONS (dpcore.py:20) */
enum fdp_reduction { FDP_REDUCE_SUM = 0, FDP_REDUCE_MEAN = 1 };

/* Noise generator.
 * KEYED_F32: the reference's keyed construction (rng.py:35-85: splitmix64
 *            absorb of (seed, layer_id, step, flat_index), two salted words,
 *            Box-Muller cosine branch) with the final transform in fp32.
 * KEYED_F64: same keys, transform in fp64 (matches the reference draw to
 *            ~1e-15; parity/debug mode).
 * PHILOX:    Philox4x32-10 keyed by absorb(seed, layer_id, step), counter =
 *            flat_index; Box-Muller. Statistically checked only. */
enum fdp_noise_impl { FDP_NOISE_KEYED_F32 = 0, FDP_NOISE_KEYED_F64 = 1, FDP_NOISE_PHILOX = 2 };

/* Workflow kinds (workflows.py:33-37, WorkflowKind). */
enum fdp_kind {
  FDP_KIND_NON_DP = 0,
  FDP_KIND_EXPLICIT_DP = 1,
  FDP_KIND_IMPLICIT_DP = 2,
  FDP_KIND_FLASHDP = 3
};

/* Execution path for FDP_KIND_FLASHDP.
 * FUSED:     one persistent tcgen05 launch: per-sample G tiles in TMEM, norm
 *            all-reduce across CTAs + grid barrier, in-register clip, batch sum,
 *            noise epilogue (Algorithm 1).
 * TWO_PHASE: norms from a first phase (ghost Gram norms or a norm-only tcgen05
 *            pass), then one reweighted tcgen05 pass (for layers whose
 *            per-sample gradient tiles exceed on-chip capacity).
 * SIMT:      generic CUDA-core path (any shape, fp32 inputs).
 * AUTO:      FUSED when it fits, else TWO_PHASE, SIMT for unaligned/fp32. */
enum fdp_path { FDP_PATH_AUTO = 0, FDP_PATH_FUSED = 1, FDP_PATH_TWO_PHASE = 2, FDP_PATH_SIMT = 3 };

/* Debug flags. SKIP_BARRIER removes the in-kernel norm barrier wait (the
 * analogue of backward_flashdp(skip_barrier=True), workflows.py:341,394) and
 * delays one CTA so the premature clip is observable. */
enum fdp_flags { FDP_FLAG_SKIP_BARRIER = 1, FDP_FLAG_TIMEOUT_SHORT = 2,
                 /* record per-CTA phase timestamps (%globaltimer, ns) of the fused kernel
                    in the workspace tail: grid x 128 uint64 after fdp_plan_info.workspace_bytes
                    minus grid*1024 bytes (see paper_2507_01154_b200/trace.py) */
                 FDP_FLAG_TRACE = 4,
                 /* sum the sample groups' clipped tiles in a fixed order (slot
                    reduce-scatter) instead of TMA reduce-add atomics: bitwise
                    reproducible across runs, slower for layers that need groups */
                 FDP_FLAG_DETERMINISTIC = 8 };

/* Norm phase of the TWO_PHASE path. SINGLE (B == 1, no accumulation): the only
 * sample's gradient IS the layer's GEMM, so it is computed once (stream-K
 * tcgen05, per-tile sums of squares in the epilogue) and one elementwise pass
 * applies the clip factor and the noise. */
/* SPILL (opt-in, never chosen by AUTO): every sample's gradient G_b is one GEMM
 * (K = T) written unscaled to the workspace (B * D * P fp32) with its norm from
 * the epilogue, then one elementwise pass forms sum_b c_b G_b + noise. It DOES
 * materialise per-sample gradients in HBM -- the thing FlashDP avoids -- trading
 * B * D * P * 8 bytes of traffic for the ghost phase's T^2 (P + D) flops; see
 * DESIGN.md for where that trade wins on B200. */
enum fdp_norm_phase { FDP_NORMS_AUTO = 0, FDP_NORMS_GHOST = 1, FDP_NORMS_RECOMPUTE = 2, FDP_NORMS_SINGLE = 3,
                      FDP_NORMS_SPILL = 4 };

typedef struct fdp_desc {
  int64_t B, T, P, D;       /* X (B,T,P), dY (B,T,D)                          */
  int32_t in_dtype;         /* fdp_dtype                                      */
  int32_t reduction;        /* fdp_reduction (DPConfig.reduction)             */
  double clip_c;            /* DPConfig.clip_c  (> 0)                         */
  double sigma;             /* DPConfig.sigma   (>= 0)                        */
  int64_t seed;             /* DPConfig.seed    (any sign; masked to 64 bits) */
  int64_t layer_id;         /* DPConfig.layer_id                              */
  int64_t step;             /* DPConfig.step                                  */
  int32_t rank, world;      /* noise partition: rank adds noise only on its
                               contiguous slice of [0, D*P) (world >= 1)     */
  int64_t mean_batch;       /* divisor for reduction=mean; 0 -> B (global B
                               under data parallelism)                       */
  int32_t accumulate;       /* 1: grad_w += result (micro-batch accumulation) */
  int32_t add_noise;        /* 0: skip noise (micro-steps; sigma still valid) */
  int32_t noise_impl;       /* fdp_noise_impl                                 */
  int32_t path;             /* fdp_path                                       */
  int32_t flags;            /* fdp_flags                                      */
  int32_t norm_phase;       /* fdp_norm_phase                                 */
  const int64_t* device_step; /* optional DEVICE pointer: when non-NULL the noise
                               key uses *device_step instead of `step`, so a
                               captured CUDA graph draws fresh noise per replay */
} fdp_desc;

/* Plan actually taken for a descriptor (analogue of tiling.BlockPlan,
 * tiling.py:31-44). Filled by fdp_plan(). */
typedef struct fdp_plan_info {
  int32_t path;             /* resolved fdp_path                              */
  int32_t norm_phase;       /* resolved fdp_norm_phase (TWO_PHASE only)       */
  int32_t tile_d, tile_p;   /* output tile extents (d, p)                     */
  int32_t tile_t;           /* t extent of one pipeline stage                 */
  int32_t n_d, n_p;         /* tile counts                                    */
  int32_t groups;           /* sample groups (CTAs sharing one output tile)   */
  int32_t grid;             /* CTAs of the main launch                        */
  int32_t launches;         /* kernel launches per call                       */
  int32_t sms;              /* SMs of the device                              */
  int64_t workspace_bytes;  /* bytes fdp_backward needs for this kind         */
} fdp_plan_info;

FDP_API int fdp_abi_version(void);
FDP_API const char* fdp_last_error(void);

/* Device properties relevant to planning (SM count, smem per block). */
FDP_API int fdp_device_info(int32_t* sms, int32_t* cc_major, int32_t* cc_minor);

FDP_API int fdp_plan(const fdp_desc* d, int32_t kind, fdp_plan_info* out);
FDP_API int fdp_workspace_bytes(const fdp_desc* d, int32_t kind, size_t* bytes);
FDP_API int fdp_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* run_backward(kind, x, dy, cfg, ...) (workflows.py:427-440).
 * norms_sq may be NULL for FDP_KIND_NON_DP (which ignores clip/noise). */
FDP_API int fdp_backward(int32_t kind, const fdp_desc* d, const void* x, const void* dy,
                 float* grad_w, float* norms_sq, void* ws, size_t ws_bytes, void* stream);

/* backward_flashdp(x, dy, cfg, plan, spec) (workflows.py:340-421). */
FDP_API int fdp_dw(const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms_sq,
           void* ws, size_t ws_bytes, void* stream);

/* fdp_dw with the clip factor handed to the consumer (deferred clip).
 * On the single-sample path (B == 1, accumulate == 0) without noise in this call
 * (add_noise == 0 or sigma == 0), grad_w receives the sample's UNCLIPPED gradient
 * G, norms_sq[0] its ||G||^2, and grad_scale[0] (a device float) the factor
 * min(1, C/||G||) / mean_batch (x 1 for reduction sum) -- the elementwise clip
 * pass over grad_w is not run. The DP gradient is grad_scale[0] * grad_w, formed
 * by whoever reads grad_w next: the optimizer step (fdp_adam_step_scaled /
 * fdp_sgd_step_scaled, rounding identical to the pass) or the data-parallel
 * collective (NCCL PreMulSum with grad_scale as the device scalar: every rank
 * scales its own contribution inside the reduction). On every other path the
 * call is fdp_dw and grad_scale[0] = 1. Replaces dpcore.clip_and_accumulate's
 * scaling step (dpcore.py:50-57, 60-73) in time only: same factor, same product. */
FDP_API int fdp_dw_deferred(const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms_sq,
                            float* grad_scale, void* ws, size_t ws_bytes, void* stream);

/* Deferred finalize chain. On the single-sample path (B == 1: the sample's
 * gradient is the layer's GEMM), the clip factor needs the norm of the whole
 * GEMM result, so the clip + noise pass over grad_w (an HBM-bound elementwise
 * pass, ~0.3-0.5 of the GEMM time at Llama shapes) cannot start before the GEMM
 * ends. A chained call leaves that pass PENDING in the chain instead; the next
 * chained call carries it inside its own stream-K GEMM, whose idle noise and
 * epilogue warps stream it while the tensor cores run (single-sample, two-phase
 * reweight or non-DP calls carry; any other call runs it standalone first), and
 * fdp_chain_flush runs the last one. Until then the pending layer's grad_w holds
 * the unclipped G and its norms_sq is unwritten. A chain is single-stream and
 * host-side state (one per backward stream); results are identical to
 * unchained calls. Reference semantics unchanged: workflows.py:340-421 /
 * dpcore.py:60-73, the pass is only moved in time.
 *   fdp_chain_create / fdp_chain_destroy: the chain object (destroy after a flush).
 *   fdp_dw_chained / fdp_backward_chained: fdp_dw / fdp_backward with a chain.
 *   fdp_chain_flush: run the pending finalize (if any) on `stream`.
 *   fdp_chain_stats: jobs carried by a later GEMM / run standalone, pending flag. */
typedef struct fdp_chain fdp_chain;
FDP_API int fdp_chain_create(fdp_chain** out);
FDP_API int fdp_chain_destroy(fdp_chain* chain);
FDP_API int fdp_chain_flush(fdp_chain* chain, void* stream);
FDP_API int fdp_chain_stats(const fdp_chain* chain, int64_t* carried, int64_t* flushed, int32_t* pending);
FDP_API int fdp_dw_chained(const fdp_desc* d, const void* x, const void* dy, float* grad_w, float* norms_sq,
                           void* ws, size_t ws_bytes, fdp_chain* chain, void* stream);
FDP_API int fdp_backward_chained(int32_t kind, const fdp_desc* d, const void* x, const void* dy, float* grad_w,
                                 float* norms_sq, void* ws, size_t ws_bytes, fdp_chain* chain, void* stream);

/* DP backward of n (1..3) layers that read the SAME input X (B, T, P) -- the q/k/v
 * projections of an attention block, gate/up of a SwiGLU MLP -- each with its own
 * dY_l (B, T, D_l), DPConfig, clip C_l and outputs. Per-layer clipping is unchanged
 * (||G_l||^2 = <X X^T, dY_l dY_l^T>); when every layer takes the two-phase path with
 * ghost norms, ONE Gram launch computes each X X^T tile once for all layers and the
 * dY Grams of each, then every layer runs its factor reduce and reweighted pass.
 * Otherwise the layers run one by one (fdp_backward; same results). Each layer has
 * its own workspace (fdp_workspace_bytes of its desc). Extends workflows.py:340-421
 * (per layer); the shared Gram is a scheduling of the ghost norms, not a new rule. */
FDP_API int fdp_backward_shared_x(int32_t n, const fdp_desc* descs, const void* x, const void* const* dy,
                                  float* const* grad_w, float* const* norms_sq, void* const* ws,
                                  const size_t* ws_bytes, void* stream);

/* The fused DP backward of n layers (n <= 48) in ONE persistent cooperative
 * launch: the training-step batching of Algorithm 1 (every layer keeps its own
 * DPConfig, noise key, per-sample norms and outputs; the producer/MMA/epilogue
 * pipelines never drain between layers). Every layer must be tensor-core
 * eligible (bf16, P % 8 == 0, D % 8 == 0) and fit the co-resident fused grid;
 * otherwise FDP_ERR_USAGE (call fdp_backward per layer instead). The arrays
 * hold one device pointer per layer; the workspace is shared by all layers. */
FDP_API int fdp_group_workspace_bytes(int32_t n, const fdp_desc* descs, size_t* bytes);
FDP_API int fdp_backward_group(int32_t n, const fdp_desc* descs, const void* const* x, const void* const* dy,
                               float* const* grad_w, float* const* norms_sq, void* ws, size_t ws_bytes,
                               void* stream);

/* Same as fdp_group_workspace_bytes / fdp_backward_group with the launch limited
 * to at most `max_ctas` CTAs (0 = all co-resident CTAs): the remaining SMs stay
 * free for a kernel running concurrently on another stream, e.g. the NCCL
 * all-reduce of the previous layer chunk under data parallelism. */
FDP_API int fdp_group_workspace_bytes_ex(int32_t n, const fdp_desc* descs, int32_t max_ctas, size_t* bytes);
FDP_API int fdp_backward_group_ex(int32_t n, const fdp_desc* descs, const void* const* x, const void* const* dy,
                                  float* const* grad_w, float* const* norms_sq, void* ws, size_t ws_bytes,
                                  int32_t max_ctas, void* stream);

/* dpcore.noise_for_indices for flat indices [lo, hi) scaled by `scale`
 * (rng.keyed_normal_array, rng.py:69-85): out[i-lo] = scale * N(seed, layer_id, step, i). */
FDP_API int fdp_noise(const fdp_desc* d, float* out, int64_t lo, int64_t hi, double scale, void* stream);
/* Same draws written as DOUBLE (the reference's own precision; with
 * FDP_NOISE_KEYED_F64 the draw matches rng.keyed_normal_array to ~1e-15):
 * dpcore.finalize_gradient / noise_for_indices on float64 gradients. */
FDP_API int fdp_noise_f64(const fdp_desc* d, double* out, int64_t lo, int64_t hi, double scale, void* stream);

/* Non-linear parameter groups (the reference clips linear
 * weights only). Each group is clipped per sample with its own norm at
 * the descriptor's clip_c (per-layer clipping), summed (or /mean_batch), and gets
 * sigma*C*N(seed, layer_id, step, i) on the rank's slice of its own index space
 * [0, L); accumulate adds onto `grad`. norms_sq (B,) may be NULL; `ws` needs the
 * matching *_workspace_bytes (no zeroing needed). in_dtype bf16 or fp32. */
enum fdp_vec_kind {
  FDP_VEC_BIAS = 0,      /* g_b = sum_t dY[b,t,:]                                L = D   */
  FDP_VEC_RMSNORM = 1,   /* g_b = sum_t dY[b,t,:] * xhat[b,t,:]  (gamma)         L = D   */
  FDP_VEC_LAYERNORM = 2  /* g_b = [sum_t dY * xhat (gamma), sum_t dY (beta)]    L = 2 D */
};
/* Vector groups: dY, xhat (B, T, D) row-major (xhat = the normalised input, unused
 * for FDP_VEC_BIAS); uses d->B, T, D (P ignored). */
FDP_API int fdp_vec_workspace_bytes(const fdp_desc* d, int32_t kind, size_t* bytes);
FDP_API int fdp_vec_dw(const fdp_desc* d, int32_t kind, const void* dy, const void* xhat, float* grad, float* norms_sq,
                       void* ws, size_t ws_bytes, void* stream);
/* fdp_vec_dw(kind = FDP_VEC_BIAS): the bias of a linear layer as its own group. */
FDP_API int fdp_bias_workspace_bytes(const fdp_desc* d, size_t* bytes);
FDP_API int fdp_bias_dw(const fdp_desc* d, const void* dy, float* grad_b, float* norms_sq, void* ws, size_t ws_bytes,
                        void* stream);
/* Embedding table (V, D) = (d->P, d->D): tokens (B, T) int64, dY (B, T, D); the
 * per-sample gradient scatters dY rows onto the sample's token rows, its norm is
 * the token-equality Gram; every row of `grad` is written (flat index v*D + c for
 * the noise). Token ids outside [0, V) contribute nothing. T <= 16384. */
FDP_API int fdp_embedding_workspace_bytes(const fdp_desc* d, size_t* bytes);
FDP_API int fdp_embedding_dw(const fdp_desc* d, const int64_t* tokens, const void* dy, float* grad, float* norms_sq,
                             void* ws, size_t ws_bytes, void* stream);

/* Optimizer steps on a finalized DP gradient, in place, fp32 or fp64 state
 * (dtype FDP_DTYPE_F32 / FDP_DTYPE_F64); reference dpcore.dp_sgd_step /
 * dp_adam_step (dpcore.py:131-156: Adam without bias correction, post-update v).
 * `noise` (optional, NULL = none): add sigma*clip_c*N(seed, layer_id, step,
 * noise_offset + i) to grad[i] first (noise_impl / device_step / add_noise of the
 * descriptor apply) -- the reduce-scatter form of data parallelism, where a
 * rank adds the noise of the shard it owns right before its optimizer step. */
FDP_API int fdp_sgd_step(int32_t dtype, void* theta, const void* grad, int64_t n, double eta, const fdp_desc* noise,
                         int64_t noise_offset, void* stream);
FDP_API int fdp_adam_step(int32_t dtype, void* theta, void* m, void* v, const void* grad, int64_t n, double eta,
                          double beta1, double beta2, double eps, const fdp_desc* noise, int64_t noise_offset,
                          void* stream);

/* The same steps on grad_scale[0] * grad (device scalar from fdp_dw_deferred;
 * fp32 state only): g = grad * grad_scale[0] rounded, then the noise, then the
 * update -- bitwise what fdp_dw's finalize followed by fdp_adam_step computes. */
FDP_API int fdp_sgd_step_scaled(int32_t dtype, void* theta, const void* grad, const float* grad_scale, int64_t n,
                                double eta, const fdp_desc* noise, int64_t noise_offset, void* stream);
FDP_API int fdp_adam_step_scaled(int32_t dtype, void* theta, void* m, void* v, const void* grad,
                                 const float* grad_scale, int64_t n, double eta, double beta1, double beta2,
                                 double eps, const fdp_desc* noise, int64_t noise_offset, void* stream);

/* Multi-segment fp32 Adam: every parameter segment of an optimizer step in ONE launch
 * (the bucketed DP-Adam of ddp.BucketedAdam; one kernel instead of one per parameter).
 * A segment is fdp_adam_step_scaled's arguments: theta / m / v / grad (n fp32 each,
 * 16-byte aligned), an optional device grad_scale, and optional noise (Philox only,
 * noise_offset a multiple of 4; the descriptor's add_noise / sigma / clip_c / seed /
 * layer_id / step / device_step apply -- with device_step the table is reusable
 * across steps and CUDA-graph capturable). fdp_adam_multi_prepare validates the
 * segments and writes the device table (blocking the host until it is written:
 * call it outside graph capture); fdp_adam_step_multi runs one step over it. */
typedef struct fdp_adam_segment {
  float* theta;
  float* m;                /* Adam moments (NULL for an SGD-only table) */
  float* v;
  const float* grad;
  const float* grad_scale; /* NULL or a device scalar: g = grad * grad_scale[0] first */
  int64_t n;
  const fdp_desc* noise;   /* NULL: no noise */
  int64_t noise_offset;
} fdp_adam_segment;
FDP_API int fdp_adam_multi_table_bytes(int32_t n_seg, size_t* bytes);
FDP_API int fdp_adam_multi_prepare(int32_t n_seg, const fdp_adam_segment* segs, void* table, size_t table_bytes,
                                   int64_t* total_quads, void* stream);
FDP_API int fdp_adam_step_multi(int32_t n_seg, const void* table, int64_t total_quads, double eta, double beta1,
                                double beta2, double eps, void* stream);
/* The DP-SGD step theta -= eta * g (g after grad_scale and noise, as fdp_sgd_step_scaled)
 * over the same kind of table; its segments may leave m / v NULL (dpcore.py:131-136). */
FDP_API int fdp_sgd_step_multi(int32_t n_seg, const void* table, int64_t total_quads, double eta, void* stream);

/* Noise slice [lo, hi) of [0, n) owned by `rank` of `world` (data-parallel
 * noise-once partition). Pure host arithmetic. */
FDP_API int fdp_noise_partition(int64_t n, int32_t rank, int32_t world, int64_t* lo, int64_t* hi);

#ifdef __cplusplus
}
#endif

#endif /* FDP_H_ */
