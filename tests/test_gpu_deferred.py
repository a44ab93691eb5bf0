"""Deferred clip (include/fdp.h fdp_dw_deferred, fdp_adam_step_scaled; ddp.GradBuckets
isolate / mark_ready(scale=)): a single-sample layer (B == 1) hands its gradient
over unclipped with its clip factor as a device scalar, and the consumer -- the
optimizer step, or the data-parallel collective -- forms the product. The result
must be the one the in-place clip pass gives (dpcore.py:41-47, 60-73): bitwise
for the optimizer path, and the same training step for the bucketed Llama."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2507_01154_b200 as fdp
from oracle import dp_oracle as O
from paper_2507_01154_b200.workflows import WorkflowKind, _run

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _layer(B, T, P, D, seed=0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(B, T, P, generator=g).to(torch.bfloat16).cuda()
    dy = (torch.randn(B, T, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
    return x, dy


@pytest.mark.parametrize("shape,clip_c", [((1, 256, 1024, 2048), 0.5), ((1, 512, 2048, 1024), 1e9),
                                          ((1, 2048, 4096, 4096), 1.0)])
def test_deferred_single_sample_equals_clip_pass(shape, clip_c):
    """grad_scale * G (torch fp32 multiply = the pass's __fmul_rn) is bitwise the
    finalised gradient; norms_sq identical; the factor is min(1, C/||G||)/B."""
    B, T, P, D = shape
    x, dy = _layer(*shape)
    cfg = fdp.DPConfig(clip_c, 1.0, "mean", seed=3, layer_id=5, step=2)
    # two-phase: the single-sample GEMM (small layers would take the fused path, which finalises in place)
    ref = _run(WorkflowKind.FLASHDP, x, dy, cfg, None, None, add_noise=False, noise_impl="philox", path="two_phase")
    assert ref.per_sample_norms_sq.shape == (1,)
    scale = torch.full((1,), -7.0, device="cuda")
    got = _run(WorkflowKind.FLASHDP, x, dy, cfg, None, None, add_noise=False, noise_impl="philox", path="two_phase",
               grad_scale_out=scale)
    torch.cuda.synchronize()
    assert torch.equal(got.per_sample_norms_sq, ref.per_sample_norms_sq)
    n2 = float(ref.per_sample_norms_sq[0])
    c = 1.0 if n2 <= clip_c ** 2 else clip_c / n2 ** 0.5
    assert abs(float(scale[0]) - c) <= 1e-6 * c
    assert torch.equal(got.grad_w * scale, ref.grad_w)
    if clip_c < 1e8:
        assert float(scale[0]) < 1.0  # the factor really was deferred (grad_w holds the unclipped G)
    # against the oracle on the same bf16 inputs (sigma = 0 twin)
    if T * P * D <= 512 * 2048 * 1024:
        g_o, n_o = O.dp_backward(x.float().cpu().double().numpy(), dy.float().cpu().double().numpy(),
                                 O.Cfg(clip_c, 0.0, "mean", 3, 5, 2), exact_noise=True)
        assert abs(n2 - float(n_o[0])) <= 1e-4 * float(n_o[0])
        d = (got.grad_w * scale).double().cpu().numpy() - g_o
        assert abs(d).max() <= 1e-3 * abs(g_o).max()


@pytest.mark.parametrize("case", ["batch2", "noise", "accumulate"])
def test_deferred_falls_back_with_scale_one(case):
    """Off the single-sample path (B > 1, noise in this call, accumulation) the call
    is fdp_dw and the scale is exactly 1."""
    B = 2 if case == "batch2" else 1
    x, dy = _layer(B, 256, 1024, 1024, seed=1)
    cfg = fdp.DPConfig(0.5, 1.0, "mean", seed=3, layer_id=5, step=2)
    kw = dict(add_noise=case == "noise", noise_impl="philox")
    base = torch.randn(1024, 1024, device="cuda") if case == "accumulate" else None
    g_ref = base.clone() if base is not None else None
    ref = _run(WorkflowKind.FLASHDP, x, dy, cfg, None, None, grad_out=g_ref, accumulate=base is not None, **kw)
    scale = torch.zeros(1, device="cuda")
    g_got = base.clone() if base is not None else None
    got = _run(WorkflowKind.FLASHDP, x, dy, cfg, None, None, grad_out=g_got, accumulate=base is not None,
               grad_scale_out=scale, **kw)
    torch.cuda.synchronize()
    assert float(scale[0]) == 1.0
    assert torch.allclose(got.grad_w, ref.grad_w, rtol=0, atol=1e-6 * float(ref.grad_w.abs().max()))


@pytest.mark.parametrize("n", [4096 * 33, 4099])
@pytest.mark.parametrize("noise", [False, True])
def test_adam_scaled_bitwise(n, noise):
    """fdp_adam_step_scaled(G, s) == fdp_adam_step(s * G) bit for bit (vector and
    scalar-tail kernels; Philox shard noise added after the scaling)."""
    from paper_2507_01154_b200.dpcore import OptimizerState, dp_adam_step_, dp_sgd_step_

    g = torch.Generator(device="cuda").manual_seed(2)
    G = torch.randn(n, device="cuda", generator=g)
    s = torch.tensor([0.0371], device="cuda")
    th, m = torch.randn(n, device="cuda", generator=g), torch.randn(n, device="cuda", generator=g) * 0.1
    v = torch.rand(n, device="cuda", generator=g)
    cfg = fdp.DPConfig(0.5, 1.0, "mean", seed=1, layer_id=3, step=4) if noise else None
    a = OptimizerState(theta=th.clone(), m=m.clone(), v=v.clone(), eta=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8)
    b = OptimizerState(theta=th.clone(), m=m.clone(), v=v.clone(), eta=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8)
    dp_adam_step_(a, G * s, noise=cfg, noise_offset=8, noise_impl="philox", layer_numel=n + 8)
    dp_adam_step_(b, G, noise=cfg, noise_offset=8, noise_impl="philox", layer_numel=n + 8, grad_scale=s)
    for t1, t2 in ((a.theta, b.theta), (a.m, b.m), (a.v, b.v)):
        assert torch.equal(t1, t2)
    t1, t2 = th.clone(), th.clone()
    dp_sgd_step_(t1, G * s, 0.1, noise=cfg, noise_offset=8, noise_impl="philox", layer_numel=n + 8)
    dp_sgd_step_(t2, G, 0.1, noise=cfg, noise_offset=8, noise_impl="philox", layer_numel=n + 8, grad_scale=s)
    assert torch.equal(t1, t2)


def test_scaled_step_rejects_bad_scale():
    from paper_2507_01154_b200.dpcore import OptimizerState, dp_adam_step_
    from paper_2507_01154_b200.errors import UsageError

    z = torch.zeros(16, device="cuda", dtype=torch.float64)
    st = OptimizerState(theta=z.clone(), m=z.clone(), v=z.clone(), eta=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8)
    with pytest.raises(UsageError):  # fp64 state
        dp_adam_step_(st, z, grad_scale=torch.ones(1, device="cuda"))
    f = torch.zeros(16, device="cuda")
    st = OptimizerState(theta=f.clone(), m=f.clone(), v=f.clone(), eta=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8)
    with pytest.raises(UsageError):  # not a one-element fp32 device tensor
        dp_adam_step_(st, f, grad_scale=torch.ones(2, device="cuda"))


# ---------------------------------------------------------------- bucketed Llama step with deferred clips


def _cfg():
    from paper_2507_01154_b200.llama import LlamaConfig

    return LlamaConfig(vocab=512, d=256, heads=4, layers=2, mlp=512, seq=128)


def _worker(rank, world, port, B, defer, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["FDP_NO_GROUP"] = "1"  # every DPLinear through the per-layer kernels,
    os.environ["FDP_SOLO_PATH"] = "two_phase"  # two-phase (B = 1: the single-sample GEMM, B = 2: ghost norms)
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01154_b200.ddp import DataParallelStep
    from paper_2507_01154_b200.llama import Llama

    cfg = _cfg()
    torch.manual_seed(0)
    with torch.device("cuda"):
        model = Llama(cfg, dp=True, clip_c=0.01, sigma=1.0, noise_impl="philox", nondp_linear="fp32grad")
    g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), generator=g).cuda()
    lo, hi = B * rank // world, B * (rank + 1) // world
    x, y = idx[lo:hi, :-1].contiguous(), idx[lo:hi, 1:].contiguous()
    step = DataParallelStep(model, dp=True, mode=mode, lr=1e-3, rank=rank, world=world, global_batch=B,
                            bucket_bytes=1 << 20, defer_clip=defer, isolate_min_numel=0)
    deferred = []
    for i in range(2):
        step(i, lambda: model.loss(x, y, reduction="sample_sum"))
        torch.cuda.synchronize()
        deferred.append(step.last_deferred)  # layers handed over unclipped with their factor this step
        if world == 1:  # the factors wait in the buckets' slots for the Adam step (< 1: really deferred)
            assert sum(1 for b in step.buckets.buckets if b.scale is not None and float(b.scale[0]) < 1) == \
                step.last_deferred
    torch.cuda.synchronize()
    out[(B, defer, world, rank, mode)] = ([p.detach().cpu().clone() for p in model.parameters()], deferred,
                                          len(step.buckets.buckets))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["allreduce", "reduce_scatter"])
def test_bucketed_llama_deferred_clip(mode):
    """Tiny Llama, every parameter DP, one sample per rank. World 1: the deferred
    clip (factor applied in the Adam step) gives the parameters of the in-place
    clip pass. World 2 over gloo (two processes on cuda:0): the factors applied in
    the collective (each rank scales its own contribution) give the parameters of
    the single-process run on both samples (B = 2: ghost norms, nothing deferred)."""
    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        for B, defer, world in ((1, False, 1), (1, True, 1), (2, False, 1), (2, None, 2)):
            mp.start_processes(_worker, args=(world, _free_port(), B, defer, mode, out), nprocs=world, join=True,
                               start_method="spawn")
        base, d0, nb0 = out[(1, False, 1, 0, mode)]
        got, d1, nb1 = out[(1, True, 1, 0, mode)]
        # every projection of both blocks and the (untied) LM head deferred, every step
        assert d0 == [0, 0] and min(d1) == 7 * 2 + 1
        assert nb1 > nb0  # isolated buckets
        for a, b in zip(got, base):
            assert torch.allclose(a, b, rtol=1e-6, atol=1e-7), float((a - b).abs().max())
        ref, dref, _ = out[(2, False, 1, 0, mode)]
        assert dref == [0, 0]
        for r in range(2):
            got2, d2, _ = out[(2, None, 2, r, mode)]
            assert min(d2) == 7 * 2 + 1
            for a, b in zip(got2, ref):
                assert torch.allclose(a, b, rtol=1e-4, atol=2e-6), (r, float((a - b).abs().max()))


def _nccl_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2507_01154_b200.ddp import GradBuckets

    res = {}
    # all-reduce only: NCCL runs a one-rank reduce-scatter as a plain copy (no PreMulSum
    # pre-op); the multi-rank reduce-scatter path is the gloo emulation's (test_ddp_gloo)
    for mode in ("allreduce",):
        w = torch.nn.Parameter(torch.zeros(64, 33, device="cuda"))
        bk = GradBuckets([w], mode=mode, flat_params=True, hooks=False, isolate=[w])
        bk.zero_grad()
        G = torch.randn(64, 33, device="cuda")
        w.grad.copy_(G)
        s = torch.tensor([0.3125], device="cuda")
        bk.mark_ready(w, scale=s)
        b = bk.buckets[0]
        assert not bk.premul  # the probe only runs at world > 1
        bk.premul = True  # world 1: force a real NCCL PreMulSum collective with the device scalar
        bk._collective(b)
        torch.cuda.synchronize()
        res[mode] = (bool(b.scale_applied), float((w.grad - G * s).abs().max()))
    out["nccl"] = res
    dist.destroy_process_group()


def test_nccl_premul_sum_collective_applies_scale():
    """The bucket all-reduce of a deferred-clip bucket on the real NCCL backend
    (one rank): PreMulSum with the device scalar leaves scale * G in the bucket."""
    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_nccl_worker, args=(1, _free_port(), out), nprocs=1, join=True, start_method="spawn")
        for mode, (applied, err) in out["nccl"].items():
            assert applied and err == 0.0, (mode, err)


def test_micro_batches_never_defer_and_match_full_batch(monkeypatch):
    """Two micro-batches of one sample each through GradBuckets + GroupedDPBackward
    (defer_clip on, isolated buckets): the first micro-batch writes its fresh
    bucket view (single-sample path, clip pass in place -- no collective after it,
    so nothing may be deferred), the second accumulates; the sum equals one
    backward over both samples (ghost norms), and no factor is left pending."""
    monkeypatch.setenv("FDP_NO_GROUP", "1")
    monkeypatch.setenv("FDP_SOLO_PATH", "two_phase")
    from paper_2507_01154_b200.ddp import GradBuckets
    from paper_2507_01154_b200.dplinear import DPLinear, GroupedDPBackward

    torch.manual_seed(0)
    lin = DPLinear(256, 384, bias=False, clip_c=0.05, sigma=0.0, noise_impl="philox", layer_id=3).cuda()
    g = torch.Generator().manual_seed(1)
    x = torch.randn(2, 128, 256, generator=g).cuda()
    w_ref = torch.randn(128, 384, generator=g).cuda()

    def loss_of(xs):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = lin(xs)
        return (y.float() * w_ref).sum()

    bk = GradBuckets([lin.weight], flat_params=False, isolate=[lin.weight])
    bk.set_deferred([lin.weight])
    outs = []
    for split in (False, True):
        bk.zero_grad()
        if split:
            for mb in range(2):
                bk.enabled = mb == 1
                lin.set_step(0, last_micro_batch=mb == 1, logical_batch=2)
                with GroupedDPBackward(buckets=bk, defer_clip=True) as grp:
                    loss_of(x[mb:mb + 1]).backward()
                assert grp.deferred_clips == 0
        else:
            bk.enabled = True
            lin.set_step(0, logical_batch=2)
            with GroupedDPBackward(buckets=bk, defer_clip=True) as grp:
                loss_of(x).backward()
            assert grp.deferred_clips == 0  # B = 2: ghost norms, nothing to defer
        bk.finish()
        assert all(b.scale is None for b in bk.buckets)
        torch.cuda.synchronize()
        outs.append(lin.weight.grad.detach().clone())
    full, split = outs
    assert float((split - full).abs().max()) <= 1e-3 * float(full.abs().max())


def test_adam_multi_segment_equals_per_segment_steps():
    """fdp_adam_step_multi over a table of segments (odd lengths, Philox noise at
    4-aligned offsets with a device step, a deferred factor) == one fdp_adam_step(_scaled)
    per segment, bit for bit."""
    import ctypes

    from paper_2507_01154_b200 import _lib
    from paper_2507_01154_b200.dpcore import OptimizerState, dp_adam_step_

    g = torch.Generator(device="cuda").manual_seed(7)
    sizes = [4096, 1001, 8, 3, 65536 + 5]
    noise = [True, False, True, True, False]
    dstep = torch.tensor([9], dtype=torch.int64, device="cuda")
    scale = torch.tensor([0.25], device="cuda")
    bufs = []
    for n in sizes:
        pad = -(-n // 4) * 4
        bufs.append([torch.randn(pad, device="cuda", generator=g) for _ in range(4)])  # theta, m, v, grad
    for b in bufs:
        b[2].abs_()  # v >= 0
    ref = [[t.clone() for t in b] for b in bufs]
    cfgs = [fdp.DPConfig(0.5, 1.0, "mean", seed=3, layer_id=10 + k, step=9) for k in range(len(sizes))]
    lib = _lib.load()
    segs, keep = [], []
    for k, (n, b) in enumerate(zip(sizes, bufs)):
        s = _lib.FdpAdamSegment(theta=b[0].data_ptr(), m=b[1].data_ptr(), v=b[2].data_ptr(), grad=b[3].data_ptr(),
                                grad_scale=scale.data_ptr() if k == 1 else None, n=n, noise=None, noise_offset=0)
        if noise[k]:
            d = _lib.make_desc(B=1, T=1, P=n + 8, D=1, clip_c=0.5, sigma=1.0, seed=3, layer_id=10 + k, step=0,
                               noise_impl="philox", device_step=dstep.data_ptr())
            keep.append(d)
            s.noise = ctypes.pointer(d)
            s.noise_offset = 8
        segs.append(s)
    arr = (_lib.FdpAdamSegment * len(segs))(*segs)
    nb = ctypes.c_size_t()
    _lib.check(lib.fdp_adam_multi_table_bytes(len(segs), ctypes.byref(nb)))
    table = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    tq = ctypes.c_int64()
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.fdp_adam_multi_prepare(len(segs), arr, table.data_ptr(), nb.value, ctypes.byref(tq), st))
    _lib.check(lib.fdp_adam_step_multi(len(segs), table.data_ptr(), tq.value, 1e-3, 0.9, 0.999, 1e-8, st))
    for k, (n, r) in enumerate(zip(sizes, ref)):
        stt = OptimizerState(theta=r[0][:n], m=r[1][:n], v=r[2][:n], eta=1e-3, beta1=0.9, beta2=0.999, eps_adam=1e-8)
        dp_adam_step_(stt, r[3][:n], noise=cfgs[k] if noise[k] else None, noise_offset=8, noise_impl="philox",
                      layer_numel=n + 8, grad_scale=scale if k == 1 else None)
    torch.cuda.synchronize()
    for k, (n, b, r) in enumerate(zip(sizes, bufs, ref)):
        # the per-segment path computes a noisy segment's last partial quad with its scalar
        # kernel (the noise FMA may round differently): bitwise up to the last whole quad
        whole = n if not noise[k] else n // 4 * 4
        for t1, t2 in zip(b[:3], r[:3]):
            assert torch.equal(t1[:whole], t2[:whole]), (k, float((t1[:whole] - t2[:whole]).abs().max()))
            assert torch.allclose(t1[whole:n], t2[whole:n], rtol=1e-6, atol=1e-6)
            assert torch.equal(t1[n:], t2[n:])  # padding never written
