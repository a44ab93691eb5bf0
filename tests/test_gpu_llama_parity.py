"""GPU parity at the layer shapes behind the paper's headline configs (SURVEY 8a:
C3 Llama-2-7B and C4 Llama-13B at T=2048, C5 sweep extremes) and the bench's
whole 48-layer workload, against the fp64 CPU oracle on the same bf16 inputs.

Acceptance structure mirrored: reference pkg/tests/test_acceptance.py:38-81
(every workflow vs the oracle on random instances). Every two-phase variant the
planner can take at these shapes is forced at least once: ghost norms on CTA
pairs and on single CTAs, the ghost K-split of the larger operand, the recompute
norm phase, the stream-K reweight in both cluster layouts (FDP_STREAM_MC: 4-CTA
multicast for down projections, 2-CTA pairs otherwise) and the B=1 single-sample
path.

Inputs: X ~ N(0,1), dY_b ~ s_b N(0,1) with per-sample scales s_b so that, at the
chosen C, some samples pass through unclipped (c_b = 1) and the others clip
(c_b = C/||G_b||): ||G_b||^2 concentrates at s_b^2 T P D for iid inputs.

Tolerances (north_star, bf16 inputs with fp32 accumulation):
  * grad_w: max|got - want| / max|want| <= 1e-3 (normwise, as everywhere), AND
    the elementwise mixed bound max |got - want| / (|want| + rms(want)) <= 1e-3,
    which does not let small entries hide behind the largest one;
  * per-sample norms^2: elementwise relative error <= 1e-3 for every sample.
"""

import numpy as np
import pytest
import torch

import paper_2507_01154_b200 as fdp
from oracle import dp_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _inputs(B, T, P, D, seed, scales):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    s = torch.tensor(scales, dtype=torch.float32, device="cuda").view(B, 1, 1)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * s).to(torch.bfloat16)
    return x, dy


def _scales(B):
    return {1: [1.3], 2: [0.7, 1.4], 4: [0.5, 0.9, 1.3, 1.7]}.get(B, list(np.linspace(0.5, 1.7, B)))


def _oracle(x, dy, cfg):
    """fp64 oracle one sample at a time (bounded host memory at Llama sizes)."""
    xh = x.double().cpu().numpy()
    yh = dy.double().cpu().numpy()
    return O.dp_backward_streaming(xh, yh, O.Cfg(cfg.clip_c, cfg.sigma, cfg.reduction, cfg.seed, cfg.layer_id,
                                                 cfg.step), exact_noise=False)


def _check(res, want, wn, tol=TOL):
    got = res.grad_w.double().cpu().numpy()
    gn = res.per_sample_norms_sq.double().cpu().numpy()
    err = np.abs(got - want)
    normwise = float(err.max() / max(np.abs(want).max(), 1e-30))
    rms = float(np.sqrt(np.mean(want * want)))
    mixed = float(np.max(err / (np.abs(want) + rms)))
    nrel = float(np.max(np.abs(gn - wn) / wn))
    assert normwise < tol, ("normwise", normwise)
    assert mixed < tol, ("elementwise mixed", mixed)
    assert nrel < tol, ("norms elementwise", nrel)
    return normwise, mixed, nrel


def _run_case(B, T, P, D, *, seed=0, sigma=0.0, noise_impl="keyed_f32", expect_phase=None, **opts):
    x, dy = _inputs(B, T, P, D, seed, _scales(B))
    # C^2 = T P D: samples with s_b < 1 pass through, the others clip
    C = float(np.sqrt(T * P * D))
    cfg = fdp.DPConfig(C, sigma, "mean", seed=seed + 11, layer_id=7, step=3)
    plan = fdp.execution_plan((B, T, P), (B, T, D), path=opts.get("path", "auto"))
    if expect_phase is not None:
        assert (plan["path"], plan["norm_phase"]) == expect_phase, plan
    res = fdp.backward_flashdp(x, dy, cfg, noise_impl=noise_impl, **opts)
    torch.cuda.synchronize()
    want, wn = _oracle(x, dy, cfg)
    clipped = int(np.sum(wn > C * C))
    assert 0 < clipped < B or B == 1, (wn, C * C)  # a mix of clipped and unclipped samples
    return _check(res, want, wn)


# ---------------------------------------------------------------- C3 / C4 layer shapes, planner's own choice

LLAMA7 = [(4096, 4096), (4096, 11008), (11008, 4096)]
LLAMA13 = [(5120, 5120), (5120, 13824), (13824, 5120)]


@pytest.mark.parametrize("P,D", LLAMA7 + LLAMA13)
@pytest.mark.parametrize("B", [1, 2])
def test_llama_layers_auto_plan(B, P, D):
    """Every distinct projection shape of Llama-2-7B (q/k/v/o, gate/up, down) and
    Llama-13B at T=2048, B=1 (single-sample GEMM + clip/noise pass) and B=2
    (ghost norms + stream-K reweight), through the planner's own choice."""
    phase = ("two_phase", "single") if B == 1 else ("two_phase", "ghost")
    _run_case(B, 2048, P, D, seed=B, expect_phase=phase)


@pytest.mark.parametrize("P,D", [(4096, 4096), (5120, 13824), (13824, 5120)])
def test_llama_layers_b4(P, D):
    _run_case(4, 2048, P, D, seed=4, expect_phase=("two_phase", "ghost"))


# ---------------------------------------------------------------- forced variants at Llama shapes


@pytest.mark.parametrize("pair", ["0", "1"])
def test_llama_ghost_pair_and_single_cta(pair, monkeypatch):
    monkeypatch.setenv("FDP_GHOST_PAIR", pair)
    _run_case(2, 2048, 4096, 4096, seed=21, norm_phase="ghost")


@pytest.mark.parametrize("split", ["2", "4"])
@pytest.mark.parametrize("P,D", [(4096, 11008), (11008, 4096)])
def test_llama_ghost_k_split(split, P, D, monkeypatch):
    monkeypatch.setenv("FDP_GHOST_SPLIT", split)
    _run_case(2, 2048, P, D, seed=22, norm_phase="ghost")


@pytest.mark.parametrize("mc", ["0", "1"])
@pytest.mark.parametrize("P,D", [(4096, 4096), (13824, 5120)])
def test_llama_stream_cluster_layouts(mc, P, D, monkeypatch):
    """Reweight pass in both stream-K cluster layouts (2-CTA pairs; 4-CTA clusters
    with X boxes multicast to two pairs) on a square and a down projection."""
    monkeypatch.setenv("FDP_STREAM_MC", mc)
    _run_case(2, 2048, P, D, seed=23, norm_phase="ghost")


def test_llama_recompute_norm_phase():
    _run_case(2, 2048, 4096, 4096, seed=24, path="two_phase", norm_phase="recompute")


@pytest.mark.parametrize("mc", ["0", "1"])
def test_llama_single_sample_layouts(mc, monkeypatch):
    monkeypatch.setenv("FDP_STREAM_MC", mc)
    _run_case(1, 2048, 13824, 5120, seed=25, norm_phase="single")


@pytest.mark.parametrize("noise_impl", ["keyed_f32", "philox"])
def test_llama_layer_with_noise(noise_impl):
    """sigma > 0 at a Llama shape: keyed noise is deterministic and compared
    draw-for-draw; Philox is compared as out(sigma) - out(0) == sigma*C*N from
    fdp.noise_range (the same counter-based draws)."""
    B, T, P, D = 2, 2048, 4096, 4096
    x, dy = _inputs(B, T, P, D, 31, _scales(B))
    C = float(np.sqrt(T * P * D))
    sigma = 1e-3  # noise comparable to the clipped mean, so neither hides the other
    cfg = fdp.DPConfig(C, sigma, "mean", seed=5, layer_id=9, step=2)
    res = fdp.backward_flashdp(x, dy, cfg, noise_impl=noise_impl)
    if noise_impl == "keyed_f32":
        want, wn = _oracle(x, dy, cfg)
        _check(res, want, wn)
    else:
        cfg0 = fdp.DPConfig(C, 0.0, "mean", seed=5, layer_id=9, step=2)
        r0 = fdp.backward_flashdp(x, dy, cfg0, noise_impl=noise_impl)
        n = fdp.noise_range(cfg, 0, P * D, sigma * C, noise_impl="philox").view(D, P)
        d = (res.grad_w - r0.grad_w).double()
        assert float((d - n.double()).abs().max() / n.double().abs().max()) < 1e-4
        want, wn = _oracle(x, dy, cfg0)
        _check(r0, want, wn)


# ---------------------------------------------------------------- C5 sweep extremes


def test_c5_largest_layer_longest_sequence():
    """d = 8192 square at T = 4096, B = 1 (the sweep's largest layer and longest sequence)."""
    _run_case(1, 4096, 8192, 8192, seed=41, expect_phase=("two_phase", "single"))


def test_c5_largest_layer_b2():
    _run_case(2, 4096, 8192, 8192, seed=42, expect_phase=("two_phase", "ghost"))


@pytest.mark.parametrize("d", [1024, 2048])
def test_c5_short_sequences_large_batch(d):
    """B = 64, T = 128: the fused per-sample path (many samples per CTA)."""
    _run_case(64, 128, d, d, seed=43)


def test_c5_b64_t4096_fused_or_two_phase():
    _run_case(8, 4096, 1024, 1024, seed=44)


# ---------------------------------------------------------------- the bench workload, every layer


def test_bench_workload_every_layer_against_oracle():
    """All 48 layers of the bench step (GPT-2 small, B=8, T=1024) through the
    one-launch group kernel vs the fp64 oracle, sigma = 0 (the noise of the same
    launch is checked in test_gpu_parity.test_bench_workload_full_size_properties)."""
    shapes = [(768, 2304), (768, 768), (768, 3072), (3072, 768)]
    B, T = 8, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    layers = []
    for blk in range(12):
        for j, (P, D) in enumerate(shapes):
            x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
            s = torch.linspace(0.5, 1.5, B, device="cuda").view(B, 1, 1)
            dy = (torch.randn(B, T, D, device="cuda", generator=g) * s).to(torch.bfloat16)
            layers.append((x, dy, fdp.DPConfig(float(np.sqrt(T * P * D)), 0.0, "mean", seed=1, layer_id=4 * blk + j,
                                               step=3)))
    grp = fdp.PreparedGroup(layers, noise_impl="philox")
    grp()
    torch.cuda.synchronize()
    for i, (x, dy, cfg) in enumerate(layers):
        want, wn = _oracle(x, dy, cfg)

        class R:  # result view for _check
            grad_w = grp.grads[i]
            per_sample_norms_sq = grp.norms[i]

        _check(R, want, wn)


# ---------------------------------------------------------------- opt-in spill norm phase


@pytest.mark.parametrize("B,P,D", [(2, 4096, 4096), (4, 5120, 13824), (2, 13824, 5120)])
def test_llama_spill_norm_phase(B, P, D):
    """norm_phase="spill" (opt-in): per-sample GEMMs to G[b] + one combine pass."""
    _run_case(B, 2048, P, D, seed=60 + B, path="two_phase", norm_phase="spill")


@pytest.mark.parametrize("noise_impl,rank,world", [("keyed_f32", 0, 1), ("keyed_f32", 1, 3), ("keyed_f64", 0, 2)])
def test_spill_noise_partition_and_accumulate(noise_impl, rank, world):
    B, T, P, D = 3, 512, 1024, 768
    x, dy = _inputs(B, T, P, D, 70, [0.6, 1.0, 1.5])
    C = float(np.sqrt(T * P * D))
    cfg = fdp.DPConfig(C, 1e-3, "mean", seed=3, layer_id=4, step=1)
    base = torch.randn(D, P, device="cuda")
    got = base.clone()
    fdp.backward_flashdp(x, dy, cfg, path="two_phase", norm_phase="spill", noise_impl=noise_impl, rank=rank,
                         world=world, grad_out=got, accumulate=True)
    ref = base.clone()
    fdp.backward_flashdp(x, dy, cfg, path="two_phase", norm_phase="ghost", noise_impl=noise_impl, rank=rank,
                         world=world, grad_out=ref, accumulate=True)
    torch.cuda.synchronize()
    assert float((got - ref).abs().max() / ref.abs().max()) < 1e-5


@pytest.mark.parametrize("mixed", ["1", "0"])
@pytest.mark.parametrize("B,T,P,D,pair", [(8, 1024, 1024, 1024, "1"), (3, 2048, 4096, 4096, "1"),
                                          (8, 512, 2048, 1024, "0")])
def test_ghost_mixed_schedule(B, T, P, D, pair, mixed, monkeypatch):
    """Ghost norms with the mixed schedule (whole items for the full waves, the last
    wave's items K-split, their unused partial slots zeroed) vs the uniform one: both
    equal the oracle. Shapes whose items leave a partial last wave (80 pair items on
    74 clusters; B = 3 at T = 2048: 108; single-CTA items over 148)."""
    monkeypatch.setenv("FDP_GHOST_MIXED", mixed)
    monkeypatch.setenv("FDP_GHOST_PAIR", pair)
    _run_case(B, T, P, D, seed=70 + B, path="two_phase", norm_phase="ghost")
