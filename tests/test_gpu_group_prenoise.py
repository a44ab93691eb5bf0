"""The group launch's pre-drawn noise pass (fdp_capi.cu, fdp_group.cu k_group_noise):
at B <= 2 a noised, non-accumulating single-sample-group layer has its noise written
by a grid-wide pass before the launch, which then reduce-adds onto it. The result is
bit for bit the in-kernel pre-fill's (FDP_GROUP_PRENOISE_MAXB=0), for every noise
generator and a rank slice of the noise, and matches the oracle on keyed noise."""

import numpy as np
import pytest
import torch

import paper_2507_01154_b200 as fdp
from oracle import dp_oracle as O

pytestmark = pytest.mark.gpu


def _layers(B):
    shapes = [(B, 256, 768, 2304), (B, 256, 768, 768), (B, 256, 768, 3072), (B, 256, 3072, 768)]
    out = []
    for i, (b, T, P, D) in enumerate(shapes):
        g = torch.Generator().manual_seed(70 + i)
        x = torch.randn(b, T, P, generator=g).to(torch.bfloat16).cuda()
        dy = (torch.randn(b, T, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
        out.append((x, dy, fdp.DPConfig(0.4, 1.1, "mean", seed=5, layer_id=i, step=2)))
    return out


def _run(layers, monkeypatch, maxb, **kw):
    monkeypatch.setenv("FDP_GROUP_PRENOISE_MAXB", str(maxb))
    grp = fdp.PreparedGroup(layers, **kw)
    grp()
    torch.cuda.synchronize()
    return [g.clone() for g in grp.grads], [n.clone() for n in grp.norms]


@pytest.mark.parametrize("B", [1, 2])
@pytest.mark.parametrize("impl", ["philox", "keyed_f32", "keyed_f64"])
@pytest.mark.parametrize("rank,world", [(0, 1), (1, 3)])
def test_prenoise_bitwise_equals_prefill(B, impl, rank, world, monkeypatch):
    layers = _layers(B)
    a, na = _run(layers, monkeypatch, 2, noise_impl=impl, rank=rank, world=world)
    b, nb = _run(layers, monkeypatch, 0, noise_impl=impl, rank=rank, world=world)
    for i in range(len(layers)):
        assert torch.equal(a[i], b[i]), i
        assert torch.equal(na[i], nb[i]), i


def test_prenoise_against_oracle(monkeypatch):
    layers = _layers(1)
    g, n = _run(layers, monkeypatch, 2, noise_impl="keyed_f32")
    for i, (x, dy, cfg) in enumerate(layers):
        oc = O.Cfg(cfg.clip_c, cfg.sigma, cfg.reduction, cfg.seed, cfg.layer_id, cfg.step)
        want, wn = O.dp_backward(x.double().cpu().numpy(), dy.double().cpu().numpy(), oc, exact_noise=False)
        got = g[i].double().cpu().numpy()
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-3, i
