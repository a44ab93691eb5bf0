"""Boundary hygiene on the GPU: workspace counters across
layout changes, float64 outputs of the prepared calls, output validation, and
the float64 dpcore drop-ins at the reference's 1e-12 tolerance."""

import os

import numpy as np
import pytest
import torch

import paper_2507_01154_b200 as fdp
from oracle import dp_oracle as O

pytestmark = pytest.mark.gpu
W = fdp.WorkflowKind


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _inputs(B, T, P, D, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * torch.linspace(0.5, 1.5, B, device="cuda").view(B, 1, 1)
          ).to(torch.bfloat16)
    return x, dy


def test_alternating_layouts_on_one_workspace():
    """fused, two-phase (ghost / single / recompute) and non-DP calls of different
    shapes alternate on ONE workspace (the pool's, keyed by device and stream);
    each result must equal the same call on a fresh zeroed workspace. A stale
    counter from another layout would let a wait pass early (wrong sums)."""
    cases = [((4, 256, 512, 768), "fused", "auto", W.FLASHDP), ((2, 512, 1024, 2048), "two_phase", "ghost", W.FLASHDP),
             ((8, 128, 256, 256), "fused", "auto", W.FLASHDP), ((1, 512, 2048, 1024), "two_phase", "single", W.FLASHDP),
             ((3, 256, 768, 512), "two_phase", "recompute", W.FLASHDP), ((4, 256, 1024, 512), "auto", "auto", W.NON_DP),
             ((16, 128, 512, 512), "fused", "auto", W.FLASHDP)]
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    for rnd in range(3):
        for i, ((B, T, P, D), path, phase, kind) in enumerate(cases):
            x, dy = _inputs(B, T, P, D, 100 * rnd + i)
            cfg = fdp.DPConfig(float(np.sqrt(T * P * D)), 0.0, "mean", seed=1, layer_id=i, step=rnd)
            kw = dict(path=path, norm_phase=phase) if kind == W.FLASHDP else {}
            shared = fdp.run_backward(kind, x, dy, cfg, workspace=ws, **kw)
            fresh = fdp.run_backward(kind, x, dy, cfg, workspace=torch.zeros_like(ws), **kw)
            torch.cuda.synchronize()
            assert torch.equal(shared.grad_w, fresh.grad_w) or _rel(shared.grad_w.cpu(), fresh.grad_w.cpu()) < 1e-6, \
                (rnd, i)
            if kind == W.FLASHDP:
                want, wn = O.dp_backward(x.double().cpu().numpy(), dy.double().cpu().numpy(),
                                         O.Cfg(cfg.clip_c, 0.0, "mean", 1, i, rnd), exact_noise=False)
                assert _rel(shared.grad_w.cpu(), want) < 1e-3, (rnd, i)


def test_alternating_group_lists_on_one_workspace():
    """Multi-layer launches with different layer lists share one workspace (as the
    chunked data-parallel backward does)."""
    shapes_a = [(768, 2304), (768, 768), (768, 3072), (3072, 768)]
    shapes_b = [(512, 512), (1024, 256), (256, 1024)]
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    for rnd in range(3):
        for shapes in (shapes_a, shapes_b, shapes_a[:2]):
            layers = []
            for j, (P, D) in enumerate(shapes):
                x, dy = _inputs(4, 256, P, D, 10 * rnd + j)
                layers.append((x, dy, fdp.DPConfig(float(np.sqrt(256 * P * D)), 0.0, "mean", layer_id=j)))
            g1 = fdp.PreparedGroup(layers, workspace=ws)
            g1()
            g2 = fdp.PreparedGroup(layers)
            g2()
            torch.cuda.synchronize()
            for a, b in zip(g1.grads, g2.grads):
                assert _rel(a.cpu(), b.cpu()) < 1e-6


def test_prepared_backward_float64_outputs():
    """fp64 inputs take the fp64 parity path: grad_w / norms are float64 (no
    out-of-bounds writes into float32 buffers) and match the oracle at 1e-12."""
    g = torch.Generator().manual_seed(3)
    x = torch.randn(3, 5, 6, generator=g, dtype=torch.float64).cuda()
    dy = torch.randn(3, 5, 4, generator=g, dtype=torch.float64).cuda()
    cfg = fdp.DPConfig(2.0, 0.0, "sum")
    call = fdp.PreparedBackward(W.FLASHDP, x, dy, cfg)
    assert call.grad_w.dtype == torch.float64 and call.norms_sq.dtype == torch.float64
    call()
    want, wn = O.dp_backward(x.cpu().numpy(), dy.cpu().numpy(), O.Cfg(2.0, 0.0, "sum", 0, 0, 0))
    assert np.max(np.abs(call.grad_w.cpu().numpy() - want)) < 1e-12
    assert np.max(np.abs(call.norms_sq.cpu().numpy() - wn)) < 1e-9


def test_caller_outputs_are_validated():
    x, dy = _inputs(2, 64, 128, 64, 0)
    cfg = fdp.DPConfig(1.0, 0.0)
    bad = [torch.empty(64, 128, dtype=torch.float64, device="cuda"), torch.empty(128, 64, device="cuda"),
           torch.empty(64, 256, device="cuda")[:, :128]]
    for g in bad:
        with pytest.raises(fdp.ShapeError):
            fdp.backward_flashdp(x, dy, cfg, grad_out=g)
        with pytest.raises(fdp.ShapeError):
            fdp.PreparedBackward(W.FLASHDP, x, dy, cfg, grad_w=g)
    with pytest.raises(fdp.ShapeError):
        fdp.backward_flashdp(x, dy, cfg, norms_out=torch.empty(3, device="cuda"))
    with pytest.raises(fdp.ShapeError):
        fdp.PreparedBackward(W.FLASHDP, x, dy, cfg, norms_sq=torch.empty(2, dtype=torch.float64, device="cuda"))


def test_dpcore_float64_dropins_against_reference_golden(golden_dir):
    """finalize_gradient / per_layer_process / accumulate_micro_batches on float64
    gradients default to the reference's fp64 keyed draw: 1e-12 vs dpflows."""
    g = np.load(os.path.join(golden_dir, "dpcore.npz"))
    for tag in ("sum_s0", "sum_s07", "mean_s13"):
        c, s, mean, seed, layer, step = g[f"cfg_{tag}"].tolist()
        cfg = fdp.DPConfig(c, s, "mean" if mean else "sum", int(seed), int(layer), int(step))
        gs = torch.tensor(g["g"], dtype=torch.float64, device="cuda")
        assert np.max(np.abs(fdp.finalize_gradient(gs, 3, cfg).cpu().numpy() - g[f"finalize_{tag}"])) < 1e-12
        ps = [torch.tensor(a, dtype=torch.float64, device="cuda") for a in g["per_sample"]]
        assert np.max(np.abs(fdp.per_layer_process(ps, cfg).cpu().numpy() - g[f"per_layer_{tag}"])) < 1e-12
        parts = [torch.tensor(a, dtype=torch.float64, device="cuda") for a in g["partials"]]
        got = fdp.accumulate_micro_batches(parts, 5, cfg).cpu().numpy()
        assert np.max(np.abs(got - g[f"micro_{tag}"])) < 1e-12
        # host float64 tensors work too (noise drawn on the device, result on the host)
        assert np.max(np.abs(fdp.finalize_gradient(gs.cpu(), 3, cfg).numpy() - g[f"finalize_{tag}"])) < 1e-12


def test_report_describes_the_executed_path():
    """BackwardResult.report is the ledger of what the device ran;
    reference_report keeps the reference simulator's ledger of the plan."""
    B, T, P, D = 4, 256, 512, 768
    x, dy = _inputs(B, T, P, D, 1)
    cfg = fdp.DPConfig(1.0, 1.0, "mean")
    inputs = B * T * (P + D) * 2
    fused = fdp.backward_flashdp(x, dy, cfg, path="fused")
    assert fused.report.kernel_launches == 1 and fused.report.redundant_flops == 0
    groups = fdp.execution_plan((B, T, P), (B, T, D), path="fused")["groups"]
    # inputs read once; sample groups reduce-add onto the pre-filled rows (one read per extra group)
    assert inputs <= fused.report.bytes_loaded < inputs + (groups + 1) * 4 * D * P
    assert fused.report.per_sample_grad_bytes_stored == 0 and fused.report.barriers == B
    ghost = fdp.backward_flashdp(x, dy, cfg, path="two_phase", norm_phase="ghost")
    assert ghost.report.bytes_loaded >= 2 * inputs and ghost.report.redundant_flops == B * T * T * (P + D)
    assert ghost.report.kernel_launches == 3
    x1, dy1 = _inputs(1, T, P, D, 2)
    single = fdp.backward_flashdp(x1, dy1, cfg, path="two_phase", norm_phase="single")
    assert single.report.kernel_launches == 2 and single.report.bytes_stored >= 2 * 4 * D * P
    expl = fdp.backward_explicit(x, dy, cfg)
    assert expl.report.per_sample_grad_bytes_stored == 2 * B * D * P * 4
    for r in (fused, ghost, single, expl):
        assert r.reference_report is not None and r.reference_report.kernel_launches >= 1


@pytest.mark.parametrize("n", [4096 * 1024 + 3, 17, 1 << 20])
def test_vectorized_adam_matches_the_scalar_formula(n):
    """fp32 Adam without noise takes the float4 kernel on aligned buffers (plus a
    scalar tail): same per-element arithmetic as dpcore.py:139-156 (no bias
    correction, post-update v), checked against a float64 evaluation."""
    from paper_2507_01154_b200.dpcore import OptimizerState, dp_adam_step_

    g = torch.Generator(device="cuda").manual_seed(n % 97)
    theta = torch.randn(n, device="cuda", generator=g)
    grad = torch.randn(n, device="cuda", generator=g)
    m = torch.randn(n, device="cuda", generator=g) * 0.1
    v = torch.rand(n, device="cuda", generator=g) * 0.01
    t64, m64, v64, g64 = theta.double(), m.double(), v.double(), grad.double()
    st = OptimizerState(theta=theta, m=m, v=v, eta=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8)
    dp_adam_step_(st, grad)
    # the kernel's constants are fp32 (1 - beta2 = 0.00099998713 in fp32): reference with the same constants
    f32 = lambda c: float(torch.tensor(c, dtype=torch.float32))  # noqa: E731
    b1, b2 = f32(0.9), f32(0.999)
    c1, c2 = f32(1.0 - b1), f32(1.0 - b2)
    m_ref = b1 * m64 + c1 * g64
    v_ref = b2 * v64 + c2 * g64 * g64
    t_ref = t64 - f32(1e-3) / (v_ref.sqrt() + f32(1e-8)) * m_ref
    torch.cuda.synchronize()
    assert torch.allclose(m.double(), m_ref, rtol=1e-6, atol=1e-7)
    assert torch.allclose(v.double(), v_ref, rtol=1e-6, atol=1e-9)
    assert torch.allclose(theta.double(), t_ref, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("offset,n", [(0, 1 << 20), (4096, 1000003), (3, 4099)])
def test_adam_with_shard_noise_vector_and_scalar_paths(offset, n):
    """ZeRO-1 owner-shard noise inside the fp32 Adam step: the quad-aligned float4
    kernel (offset % 4 == 0, Philox: one draw per quad) and the scalar kernel
    (other offsets) both add exactly sigma*C*N(seed, layer_id, step, offset + i)."""
    from paper_2507_01154_b200.dpcore import OptimizerState, dp_adam_step_

    g = torch.Generator(device="cuda").manual_seed(n % 89)
    theta = torch.randn(n, device="cuda", generator=g)
    grad = torch.randn(n, device="cuda", generator=g) * 1e-2
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    cfg = fdp.DPConfig(0.5, 0.8, "mean", seed=7, layer_id=3, step=11)
    noise = fdp.noise_range(cfg, offset, offset + n, cfg.sigma * cfg.clip_c, noise_impl="philox")
    g_eff = (grad + noise).double()
    t0 = theta.double()
    st = OptimizerState(theta=theta, m=m, v=v, eta=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8)
    dp_adam_step_(st, grad, noise=cfg, noise_offset=offset, noise_impl="philox", layer_numel=offset + n + 8)
    torch.cuda.synchronize()
    f32 = lambda c: float(torch.tensor(c, dtype=torch.float32))  # noqa: E731
    m_ref = f32(1.0 - f32(0.9)) * g_eff
    assert torch.allclose(m.double(), m_ref, rtol=1e-5, atol=1e-8)
    v_ref = f32(1.0 - f32(0.999)) * g_eff * g_eff
    t_ref = t0 - f32(1e-3) / (v_ref.sqrt() + f32(1e-8)) * m_ref
    assert torch.allclose(theta.double(), t_ref, rtol=1e-5, atol=1e-6)


def test_reserved_sms_caps_every_per_layer_grid(monkeypatch):
    """FDP_RESERVE_SMS (set by ddp.DataParallelStep under data parallelism): the
    per-layer grids leave that many SMs to NCCL, with unchanged results."""
    cases = [((2, 512, 2048, 2048), "two_phase", "ghost"), ((1, 512, 2048, 2048), "two_phase", "single"),
             ((4, 256, 512, 768), "fused", "auto")]
    for (B, T, P, D), path, phase in cases:
        x, dy = _inputs(B, T, P, D, 3)
        cfg = fdp.DPConfig(float(np.sqrt(T * P * D)), 0.0, "mean")
        ref = fdp.backward_flashdp(x, dy, cfg, path=path, norm_phase=phase).grad_w.clone()
        full = fdp.execution_plan((B, T, P), (B, T, D), path=path)["grid"]
        monkeypatch.setenv("FDP_RESERVE_SMS", "20")
        capped = fdp.execution_plan((B, T, P), (B, T, D), path=path)["grid"]
        got = fdp.backward_flashdp(x, dy, cfg, path=path, norm_phase=phase).grad_w
        monkeypatch.delenv("FDP_RESERVE_SMS")
        torch.cuda.synchronize()
        assert capped <= max(full, 148 - 20), (path, full, capped)
        assert _rel(got.cpu(), ref.cpu()) < 1e-5, path
