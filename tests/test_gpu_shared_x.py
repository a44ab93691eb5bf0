"""Layers that read the same input X (q/k/v, gate/up) through fdp_backward_shared_x:
one ghost Gram launch computes each X X^T tile once for all of them, per-layer
clipping is unchanged (||G_l||^2 = <X X^T, dY_l dY_l^T>, workflows.py:340-421 per
layer).

  * bitwise: with the per-layer ghost forced to the same CTA-pair kernel without a K
    split, every layer's grad_w and norms equal its own standalone call exactly;
  * oracle: each layer against the fp64 oracle on the same bf16 inputs (the Llama
    parity bars of tests/test_gpu_llama_parity.py), at a 7B attention block shape;
  * layers whose plan is not the ghost two-phase path run one by one (same results).
"""

import numpy as np
import pytest
import torch

import paper_2507_01154_b200 as fdp
from test_gpu_llama_parity import _check, _oracle

pytestmark = pytest.mark.gpu


def _layers(B, T, P, Ds, seed, Cs, sigma=0.0, noise_impl="philox", **opts):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    out = []
    for k, D in enumerate(Ds):
        s = torch.linspace(0.5, 1.5, B, device="cuda").view(B, 1, 1)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * s).to(torch.bfloat16)
        cfg = fdp.DPConfig(Cs[k], sigma, "mean", seed=seed + 5, layer_id=10 + k, step=2)
        out.append((dy, cfg))
    return x, out


def _prepared(x, layers, **opts):
    return [fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, **opts) for dy, cfg in layers]


@pytest.mark.parametrize("Ds", [(1024, 1024, 1024), (2048, 512), (768, 1536, 1024)])
@pytest.mark.parametrize("sigma", [0.0, 1.0])
def test_shared_x_bitwise_equals_per_layer(Ds, sigma, monkeypatch):
    monkeypatch.setenv("FDP_GHOST_PAIR", "1")
    monkeypatch.setenv("FDP_GHOST_SPLIT", "1")
    B, T, P = 2, 1024, 1024
    Cs = [float(np.sqrt(T * P * D)) for D in Ds]
    x, layers = _layers(B, T, P, Ds, 3, Cs, sigma)
    opts = dict(path="two_phase", norm_phase="ghost", noise_impl="philox")
    solo = _prepared(x, layers, **opts)
    for pb in solo:
        pb()
    shared_pbs = _prepared(x, layers, **opts)
    fdp.PreparedSharedX(shared_pbs)()
    torch.cuda.synchronize()
    for a, b in zip(solo, shared_pbs):
        assert torch.equal(a.norms_sq, b.norms_sq)
        assert torch.equal(a.grad_w, b.grad_w)


def test_shared_x_llama7b_attention_vs_oracle():
    """q, k, v of a Llama-2-7B block (4096 -> 4096 each) at B=2, T=2048 vs the oracle;
    per-layer C so that some samples clip and others pass through."""
    B, T, P = 2, 2048, 4096
    Ds = (4096, 4096, 4096)
    Cs = [float(np.sqrt(T * P * D)) for D in Ds]
    x, layers = _layers(B, T, P, Ds, 7, Cs)
    pbs = _prepared(x, layers, noise_impl="keyed_f32")
    assert all(fdp._lib.PATH_NAMES[pb.plan.path] == "two_phase" and
               fdp._lib.NORM_PHASE_NAMES[pb.plan.norm_phase] == "ghost" for pb in pbs)
    fdp.PreparedSharedX(pbs)()
    torch.cuda.synchronize()
    for pb, (dy, cfg) in zip(pbs, layers):
        want, wn = _oracle(x, dy, cfg)
        res = fdp.BackwardResult(pb.grad_w, None, pb.norms_sq)
        _check(res, want, wn)
        assert 0 < int(np.sum(wn > cfg.clip_c ** 2)) < B


def test_shared_x_gate_up_vs_oracle():
    """gate / up of a Llama-2-7B MLP (4096 -> 11008 each), B=2, T=2048."""
    B, T, P = 2, 2048, 4096
    Ds = (11008, 11008)
    Cs = [float(np.sqrt(T * P * D)) for D in Ds]
    x, layers = _layers(B, T, P, Ds, 8, Cs)
    pbs = _prepared(x, layers, noise_impl="keyed_f32")
    fdp.PreparedSharedX(pbs)()
    torch.cuda.synchronize()
    for pb, (dy, cfg) in zip(pbs, layers):
        want, wn = _oracle(x, dy, cfg)
        _check(fdp.BackwardResult(pb.grad_w, None, pb.norms_sq), want, wn)


def test_shared_x_falls_back_per_layer():
    """Small layers take the fused path: the call runs them one by one."""
    B, T, P = 4, 128, 256
    Ds = (256, 512)
    x, layers = _layers(B, T, P, Ds, 9, [1.0, 1.0])
    solo = _prepared(x, layers)
    for pb in solo:
        pb()
    pbs = _prepared(x, layers)
    fdp.PreparedSharedX(pbs)()
    torch.cuda.synchronize()
    for a, b in zip(solo, pbs):
        # the fused path combines sample groups with TMA reduce-adds (order not fixed)
        assert torch.allclose(a.norms_sq, b.norms_sq, rtol=1e-6, atol=0)
        assert torch.allclose(a.grad_w, b.grad_w, rtol=1e-5, atol=1e-6 * float(a.grad_w.abs().max()))


def test_shared_x_rejects_different_inputs():
    x1 = torch.zeros(2, 128, 256, dtype=torch.bfloat16, device="cuda")
    x2 = torch.zeros_like(x1)
    dy = torch.zeros(2, 128, 256, dtype=torch.bfloat16, device="cuda")
    cfg = fdp.DPConfig(1.0, 0.0)
    a = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x1, dy, cfg)
    b = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x2, dy, cfg)
    with pytest.raises(fdp.UsageError):
        fdp.PreparedSharedX([a, b])


def test_grouped_backward_shares_x_between_projections(monkeypatch):
    """Three DPLinear projections of one activation (an attention block's q/k/v, each
    4096 -> 4096, B=2, T=2048: over the co-resident grid, so per-layer two-phase
    kernels) inside GroupedDPBackward: the forward saves ONE bf16 copy of the input
    (_cast_shared) and the backward runs them through one fdp_backward_shared_x call;
    the gradients equal the per-layer path's (FDP_SHARED_X=0)."""
    from paper_2507_01154_b200.dplinear import DPLinear, GroupedDPBackward

    torch.manual_seed(0)
    d, B, T = 4096, 2, 2048
    layers = [DPLinear(d, d, bias=False, clip_c=50.0, sigma=0.0, layer_id=k, noise_impl="philox").cuda()
              for k in range(3)]
    h = torch.randn(B, T, d, device="cuda")  # fp32 activation (an RMSNorm's output): cast once for all three

    def step(shared):
        monkeypatch.setenv("FDP_SHARED_X", "1" if shared else "0")
        for m in layers:
            m.weight.grad = None
        with GroupedDPBackward() as gb:
            with torch.autocast("cuda", dtype=torch.bfloat16):
                ys = [m(h) for m in layers]
            sum((y.float() * (k + 1)).square().mean() for k, y in enumerate(ys)).backward()
        torch.cuda.synchronize()
        return [m.weight.grad.clone() for m in layers], gb.shared_x_calls

    g_shared, n_shared = step(True)
    g_solo, _ = step(False)
    assert n_shared == 1
    for a, b in zip(g_shared, g_solo):
        assert torch.allclose(a, b, rtol=1e-4, atol=1e-4 * float(b.abs().max()))
