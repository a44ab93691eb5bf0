"""Deferred-finalize chain (include/fdp.h fdp_dw_chained): a single-sample
layer's clip + noise pass carried by the next call's stream-K GEMM. Results must
be bitwise identical to unchained calls, for every noise generator and rank
partition, whatever kind of call carries the job (single-sample, two-phase
reweight, non-DP) or when it is flushed standalone (fused calls do not carry)."""

import numpy as np
import pytest
import torch

import paper_2507_01154_b200 as fdp
from oracle import dp_oracle as O

pytestmark = pytest.mark.gpu
W = fdp.WorkflowKind


def _inputs(B, T, P, D, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    return x, dy


SEQ = [  # (kind, B, T, P, D, path)
    (W.FLASHDP, 1, 512, 1024, 2048, "single"),      # single-sample: becomes pending
    (W.FLASHDP, 1, 512, 2048, 1024, "single"),      # single-sample: carries the previous one, becomes pending
    (W.FLASHDP, 2, 512, 1024, 1024, "two_phase"),   # ghost + reweight: carries
    (W.FLASHDP, 1, 256, 512, 1536, "single"),       # single: pending
    (W.FLASHDP, 4, 128, 256, 256, "fused"),         # fused: flushes the pending job standalone first
    (W.FLASHDP, 1, 256, 1536, 512, "single"),       # single: pending
    (W.NON_DP, 2, 256, 512, 512, "auto"),           # non-DP stream GEMM: carries
    (W.FLASHDP, 1, 384, 768, 768, "single"),        # single: pending until flush
]


@pytest.mark.parametrize("noise_impl,rank,world", [("philox", 0, 1), ("keyed_f32", 0, 1), ("philox", 1, 3),
                                                   ("keyed_f64", 2, 3)])
def test_chained_sequence_bitwise_equals_unchained(noise_impl, rank, world):
    data = [_inputs(B, T, P, D, 10 + i) for i, (_, B, T, P, D, _) in enumerate(SEQ)]
    cfgs = [fdp.DPConfig(float(0.5 * np.sqrt(T * P * D) * 1e-2), 0.7, "mean", seed=3, layer_id=i, step=2)
            for i, (_, B, T, P, D, _) in enumerate(SEQ)]

    def run(chain):
        outs = []
        for (kind, B, T, P, D, path), (x, dy), cfg in zip(SEQ, data, cfgs):
            kw = dict(noise_impl=noise_impl, rank=rank, world=world, chain=chain)
            if kind == W.FLASHDP and path == "single":
                r = fdp.backward_flashdp(x, dy, cfg, path="two_phase", norm_phase="single", **kw)
            elif kind == W.FLASHDP:
                r = fdp.backward_flashdp(x, dy, cfg, path=path, **kw)
            else:
                r = fdp.backward_nondp(x, dy, chain=chain)
            outs.append(r)
        if chain is not None:
            chain.flush()
        torch.cuda.synchronize()
        return [(r.grad_w.clone(), r.per_sample_norms_sq.clone()) for r in outs]

    ref = run(None)
    chain = fdp.DeferredChain()
    got = run(chain)
    st = chain.stats()
    assert st["carried"] == 3 and st["standalone"] == 2 and not st["pending"], st
    for i, ((g1, n1), (g2, n2)) in enumerate(zip(ref, got)):
        if SEQ[i][5] == "single":  # finalized by a carrying GEMM or standalone: the same bits
            assert torch.equal(g1, g2), i
            assert torch.equal(n1, n2), i
        else:  # split tiles combine by TMA reduce-add in arrival order: fp32-close, not bitwise
            assert torch.allclose(g1, g2, rtol=1e-5, atol=1e-5 * float(g1.abs().max())), i
            assert torch.allclose(n1, n2, rtol=1e-6), i


def test_chained_single_sample_against_oracle():
    """A chain of B = 1 layers against the fp64 oracle (clip active, keyed noise)."""
    chain = fdp.DeferredChain()
    outs = []
    shapes = [(512, 1024, 2048), (512, 2048, 1024), (256, 1024, 1024)]
    for i, (T, P, D) in enumerate(shapes):
        x, dy = _inputs(1, T, P, D, 40 + i)
        cfg = fdp.DPConfig(1e-2, 0.5, "sum", seed=1, layer_id=i, step=0)
        outs.append((x, dy, cfg, fdp.backward_flashdp(x, dy, cfg, noise_impl="keyed_f32", chain=chain,
                                                      path="two_phase", norm_phase="single")))
    chain.flush()
    torch.cuda.synchronize()
    for x, dy, cfg, r in outs:
        want, wn = O.dp_backward(x.double().cpu().numpy(), dy.double().cpu().numpy(),
                                 O.Cfg(cfg.clip_c, cfg.sigma, cfg.reduction, cfg.seed, cfg.layer_id, cfg.step),
                                 exact_noise=False)
        got = r.grad_w.double().cpu().numpy()
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-3
        assert abs(float(r.per_sample_norms_sq[0]) - wn[0]) / wn[0] < 1e-3


def test_chain_flushes_when_the_next_call_aliases_the_pending_gradient():
    x, dy = _inputs(1, 256, 512, 1024, 5)
    cfg = fdp.DPConfig(1e-2, 1.0, "mean", seed=9, layer_id=1)
    g = torch.zeros(1024, 512, device="cuda")
    kw = dict(noise_impl="philox", path="two_phase", norm_phase="single")
    ref = fdp.backward_flashdp(x, dy, cfg, **kw).grad_w.clone()
    chain = fdp.DeferredChain()
    fdp.backward_flashdp(x, dy, cfg, grad_out=g, chain=chain, **kw)
    # same grad_w again: the pending finalize must run first (accumulate: not single-sample)
    fdp.backward_flashdp(x, dy, cfg, grad_out=g, accumulate=True, chain=chain, noise_impl="philox")
    chain.flush()
    torch.cuda.synchronize()
    assert torch.allclose(g, 2 * ref, rtol=1e-5, atol=1e-6)
    st = chain.stats()
    assert st["standalone"] == 1 and st["carried"] == 0 and not st["pending"], st


def test_grouped_backward_uses_the_chain_for_per_layer_kernels():
    """GroupedDPBackward sends layers over the co-resident grid (4096 x 4096: per-layer
    two-phase kernels) through a chain: same gradients as without deferral."""
    from paper_2507_01154_b200.dplinear import DPLinear, GroupedDPBackward

    torch.manual_seed(0)
    layers = [DPLinear(4096, 4096, bias=False, clip_c=1e-2, sigma=0.5, layer_id=i, noise_impl="philox").cuda()
              for i in range(3)]
    x = torch.randn(1, 256, 4096, device="cuda")

    def grads(defer):
        for m in layers:
            m.weight.grad = None
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = layers[2](layers[1](layers[0](x))).float().pow(2).sum()
        with GroupedDPBackward(defer_finalize=defer) as gb:
            loss.backward()
        torch.cuda.synchronize()
        return [m.weight.grad.clone() for m in layers], gb

    a, _ = grads(False)
    b, gb = grads(True)
    for u, v in zip(a, b):
        assert torch.equal(u, v)
    st = gb.chain.stats()
    assert st["carried"] == 2 and st["standalone"] == 1 and not st["pending"], st
