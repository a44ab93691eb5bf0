"""World-size-2 data-parallel composition on CPU (gloo): per-rank contributions
(clipped sum over the rank's samples / global B + noise on the rank's index
slice, exactly what the kernel computes with rank/world/mean_batch) summed by
paper_2507_01154_b200.ddp.allreduce_grads_ equal the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dp_oracle as O
from paper_2507_01154_b200.ddp import allreduce_grads_, noise_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_contribution(x, dy, cfg, rank, world):
    """What rank `rank` of `world` produces for its batch slice (oracle arithmetic)."""
    B = x.shape[0]
    lo_b, hi_b = B * rank // world, B * (rank + 1) // world
    n = dy.shape[2] * x.shape[2]
    lo, hi = noise_partition(n, rank, world)
    g, _ = O.dp_backward(x[lo_b:hi_b], dy[lo_b:hi_b], cfg, exact_noise=True, mean_batch=B, noise_lo=lo,
                         noise_hi=hi)
    return g


def _worker(rank, world, port, x, dy, cfgs, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grads = [torch.tensor(_rank_contribution(x, dy, c, rank, world)) for c in cfgs]
    allreduce_grads_(grads, bucket_bytes=1024)  # several buckets
    if rank == 0:
        for i, g in enumerate(grads):
            out[i] = g.numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_allreduce_equals_single_process():
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (6, 5, 12))
    dy = rng.uniform(-1, 1, (6, 5, 7))
    cfgs = [O.Cfg(0.7, 1.3, "mean", 5, 2, 9), O.Cfg(1e9, 0.5, "sum", 1, 0, 0), O.Cfg(0.1, 0.0, "mean", 0, 0, 0)]
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), x, dy, cfgs, out), nprocs=world, join=True)
        for i, c in enumerate(cfgs):
            want, _ = O.dp_backward(x, dy, c, exact_noise=True)
            assert np.max(np.abs(out[i] - want)) <= 1e-12 * max(1.0, np.max(np.abs(want))), i


def test_partition_matches_kernel_partition():
    # same slices as fdp_noise_partition (tests/test_host_api.py checks the C side)
    for n in (1, 10, 65536, 999983):
        for world in (1, 2, 3, 8):
            sl = [noise_partition(n, r, world) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))


def _chunk_worker(rank, world, port, x, dy, cfgs, out):
    """ChunkedAllReduceBackward on CPU: each chunk's 'launch' writes the rank's
    oracle contribution into its slices of the flat buffer; the chunk buckets are
    all-reduced (gloo) as they complete."""
    from paper_2507_01154_b200.ddp import ChunkedAllReduceBackward

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    xt, dyt = torch.tensor(x), torch.tensor(dy)
    layers = [(xt, dyt, c) for c in cfgs]
    n_el = sum(dy.shape[2] * x.shape[2] for _ in cfgs)
    flat = torch.zeros(n_el, dtype=torch.float64)

    def make_group(chunk_layers, grads, cap):
        def run():
            for (_, _, c), g in zip(chunk_layers, grads):
                g.copy_(torch.tensor(_rank_contribution(x, dy, c, rank, world)))
        return run

    step = ChunkedAllReduceBackward(layers, flat, n_chunks=2, world=world, make_group=make_group)
    assert len(step.chunks) == 2
    step()
    if rank == 0:
        out["flat"] = flat.numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_chunked_allreduce_backward_two_ranks():
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (4, 3, 8))
    dy = rng.uniform(-1, 1, (4, 3, 6))
    cfgs = [O.Cfg(0.5, 1.0, "mean", 7, l, 3) for l in range(3)]
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_chunk_worker, args=(2, _free_port(), x, dy, cfgs, out), nprocs=2, join=True)
        want = np.concatenate([O.dp_backward(x, dy, c, exact_noise=True)[0].reshape(-1) for c in cfgs])
        assert np.max(np.abs(out["flat"] - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


def test_set_data_parallel_sets_every_module_and_validates():
    import pytest as _pytest

    from paper_2507_01154_b200 import DPEmbedding, DPLayerNorm, DPLinear, DPRMSNorm
    from paper_2507_01154_b200.ddp import set_data_parallel

    mods = [DPLinear(8, 8), DPLayerNorm(8), DPRMSNorm(8), DPEmbedding(10, 8)]
    set_data_parallel(mods, 1, 4)
    assert all((m.rank, m.world) == (1, 4) for m in mods)
    with _pytest.raises(ValueError):
        set_data_parallel(mods, 4, 4)


# ---------------------------------------------------------------- bucketed training step (GradBuckets)


def _bucket_model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.Tanh(), torch.nn.Linear(32, 24), torch.nn.Tanh(),
                               torch.nn.Linear(24, 8))


def _bucket_worker(rank, world, port, mode, out):
    from paper_2507_01154_b200.ddp import DataParallelStep, _torch_adam_

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    model = _bucket_model()
    g = torch.Generator().manual_seed(3)
    x, y = torch.randn(8, 16, generator=g), torch.randn(8, 8, generator=g)
    lo, hi = 8 * rank // world, 8 * (rank + 1) // world
    step = DataParallelStep(model, dp=False, mode=mode, lr=1e-2, rank=rank, world=world, global_batch=8,
                            adam_fn=_torch_adam_, bucket_bytes=600)  # several buckets
    seen = []
    model[0].weight.register_post_accumulate_grad_hook(lambda p: seen.append(len(step.buckets.issued)))
    for i in range(3):
        step(i, lambda: ((model(x[lo:hi]) - y[lo:hi]) ** 2).sum(1).sum() / 8)
    out[(mode, world, rank)] = ([p.detach().clone() for p in model.parameters()], list(step.buckets.issued),
                                len(step.buckets.buckets), seen)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def test_bucketed_step_two_ranks_equals_single_process():
    """DataParallelStep on a 5-layer model, world 2 over gloo, both bucket modes
    (all-reduce + replicated Adam; reduce-scatter + ZeRO-1 Adam + all-gather):
    the parameters after 3 steps equal the single-process run on the global
    batch; buckets are issued in the same order on both ranks, and the first
    buckets are issued while the backward is still running (before the first
    layer's gradient exists)."""
    for mode in ("allreduce", "reduce_scatter"):
        with mp.Manager() as mgr:
            out = mgr.dict()
            _bucket_worker(0, 1, _free_port(), mode, out)
            mp.spawn(_bucket_worker, args=(2, _free_port(), mode, out), nprocs=2, join=True)
            ref, _, nb, _ = out[(mode, 1, 0)]
            assert nb >= 3
            for r in range(2):
                got, issued, _, seen = out[(mode, 2, r)]
                for a, b in zip(got, ref):
                    assert torch.allclose(a, b, rtol=1e-5, atol=1e-6), mode
                assert issued == out[(mode, 2, 0)][1]
                assert all(s >= 1 for s in seen)  # overlap: earlier buckets already on the wire


def test_grad_buckets_layout_and_validation():
    from paper_2507_01154_b200.ddp import GradBuckets

    model = _bucket_model()
    bk = GradBuckets(model.parameters(), bucket_bytes=1200, mode="reduce_scatter", rank=1, world=3,
                     flat_params=True, hooks=False)
    ps = list(model.parameters())
    # reverse registration order, every grad / param a view of its bucket, shards padded to world
    assert bk.buckets[0].params[0] is ps[-1]
    for b in bk.buckets:
        assert b.flat.numel() == 3 * b.per >= b.n
        assert b.shard.data_ptr() == b.flat[b.per:].data_ptr()
        for p, o in zip(b.params, b.offsets):
            assert p.grad.data_ptr() == b.flat[o:].data_ptr() and p.data_ptr() == b.pflat[o:].data_ptr()
    with pytest.raises(ValueError):
        GradBuckets(model.parameters(), mode="ring")
    with pytest.raises(ValueError):
        GradBuckets([torch.nn.Parameter(torch.zeros(3, dtype=torch.float64))])


def test_nccl_options_cap_ctas(monkeypatch):
    from paper_2507_01154_b200.ddp import nccl_options

    monkeypatch.delenv("NCCL_MAX_CTAS", raising=False)
    opts = nccl_options(4)
    assert os.environ["NCCL_MAX_CTAS"] == "4"
    if opts is not None:
        assert opts.config.max_ctas == 4
    with pytest.raises(ValueError):
        nccl_options(0)


def _micro_worker(rank, world, port, out):
    """Two micro-batches per step: buckets disabled on the first (gradients accumulate
    into the bucket views, no collective), enabled on the last (one collective per
    bucket for the sum of both micro-batches)."""
    from paper_2507_01154_b200.ddp import BucketedAdam, GradBuckets, _torch_adam_

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    model = _bucket_model()
    g = torch.Generator().manual_seed(9)
    x, y = torch.randn(8, 16, generator=g), torch.randn(8, 8, generator=g)
    bk = GradBuckets(model.parameters(), bucket_bytes=600, rank=rank, world=world, flat_params=True)
    opt = BucketedAdam(bk, lr=1e-2, adam_fn=_torch_adam_)
    per = 8 // world
    for step in range(2):
        bk.zero_grad()
        for mb in range(2):  # micro-batches of this rank's samples
            bk.enabled = mb == 1
            lo = rank * per + mb * per // 2
            hi = lo + per // 2
            (((model(x[lo:hi]) - y[lo:hi]) ** 2).sum(1).sum() / 8).backward()
        bk.finish()
        opt.step(step)
    out[(world, rank)] = ([p.detach().clone() for p in model.parameters()], list(bk.issued))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def test_grad_buckets_micro_batches_reduce_once():
    with mp.Manager() as mgr:
        out = mgr.dict()
        _micro_worker(0, 1, _free_port(), out)
        mp.spawn(_micro_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        ref, issued1 = out[(1, 0)]
        assert len(issued1) == len(set(issued1))  # each bucket issued once per step
        for r in range(2):
            got, issued = out[(2, r)]
            assert issued == issued1
            for a, b in zip(got, ref):
                assert torch.allclose(a, b, rtol=1e-5, atol=1e-6)


# ---------------------------------------------------------------- deferred clip (scaled bucket)


def _scaled_worker(rank, world, port, mode, out):
    """One isolated weight is handed over UNscaled (grad / s_r) with its rank's
    factor s_r (GradBuckets.mark_ready(p, scale=)): the collective multiplies every
    rank's contribution by its own factor (gloo: in place first), at world 1 the
    Adam step does -- the parameters equal a run with the scaled gradients."""
    from paper_2507_01154_b200.ddp import BucketedAdam, GradBuckets, _torch_adam_

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    model = _bucket_model()
    w = model[2].weight
    g = torch.Generator().manual_seed(4)
    x, y = torch.randn(8, 16, generator=g), torch.randn(8, 8, generator=g)
    bk = GradBuckets(model.parameters(), bucket_bytes=600, mode=mode, rank=rank, world=world, flat_params=True,
                     hooks=False, isolate=[w])
    iso = [b for b in bk.buckets if any(p is w for p in b.params)]
    assert len(iso) == 1 and len(iso[0].params) == 1
    opt = BucketedAdam(bk, lr=1e-2, adam_fn=_torch_adam_)
    per = 8 // world
    for step in range(2):
        bk.zero_grad()
        assert bk.fresh(w)
        lo, hi = rank * per, (rank + 1) * per
        (((model(x[lo:hi]) - y[lo:hi]) ** 2).sum(1).sum() / 8).backward()
        s = torch.tensor([0.5 + 0.25 * rank + 0.125 * step])
        w.grad.div_(s)  # what the deferred kernel leaves: the gradient before its factor
        for p in reversed(list(model.parameters())):
            bk.mark_ready(p, scale=s if p is w else None)
            bk.note_written(p)
        assert not bk.fresh(w)
        bk.finish()
        opt.step(step)
    out[(mode, world, rank)] = [p.detach().clone() for p in model.parameters()]
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def test_grad_buckets_deferred_scale_two_ranks():
    for mode in ("allreduce", "reduce_scatter"):
        with mp.Manager() as mgr:
            out = mgr.dict()
            _micro_ref = _bucket_model()  # the plain run: scaled gradients never divided
            g = torch.Generator().manual_seed(4)
            x, y = torch.randn(8, 16, generator=g), torch.randn(8, 8, generator=g)
            from paper_2507_01154_b200.ddp import BucketedAdam, GradBuckets, _torch_adam_

            bk = GradBuckets(_micro_ref.parameters(), bucket_bytes=600, flat_params=True, hooks=False)
            opt = BucketedAdam(bk, lr=1e-2, adam_fn=_torch_adam_)
            for step in range(2):
                bk.zero_grad()
                (((_micro_ref(x) - y) ** 2).sum(1).sum() / 8).backward()
                bk.finish()
                opt.step(step)
            ref = [p.detach().clone() for p in _micro_ref.parameters()]
            _scaled_worker(0, 1, _free_port(), mode, out)
            mp.spawn(_scaled_worker, args=(2, _free_port(), mode, out), nprocs=2, join=True)
            for key in ((mode, 1, 0), (mode, 2, 0), (mode, 2, 1)):
                for a, b in zip(out[key], ref):
                    assert torch.allclose(a, b, rtol=1e-5, atol=1e-6), key


def test_grad_buckets_scale_needs_own_bucket():
    from paper_2507_01154_b200.ddp import GradBuckets

    model = _bucket_model()
    bk = GradBuckets(model.parameters(), bucket_bytes=1 << 20, flat_params=True, hooks=False)
    assert len(bk.buckets) == 1 and not bk.can_defer(model[2].weight)
    with pytest.raises(RuntimeError):
        bk.mark_ready(model[2].weight, scale=torch.ones(1))


def test_grad_buckets_materialize_scales_and_isolation_layout():
    from paper_2507_01154_b200.ddp import BucketedAdam, GradBuckets, _torch_adam_

    model = _bucket_model()
    w = model[2].weight
    bk = GradBuckets(model.parameters(), bucket_bytes=1 << 20, flat_params=True, hooks=False, isolate=[w])
    # the isolated weight sits alone between the buckets of its neighbours (reverse registration order)
    owners = [[q for q in b.params] for b in bk.buckets]
    assert [len(o) for o in owners] == [3, 1, 2] and owners[1][0] is w
    opt = BucketedAdam(bk, lr=1e-2, adam_fn=_torch_adam_)
    bk.zero_grad()
    w.grad.copy_(torch.ones_like(w))
    bk.mark_ready(w, scale=torch.tensor([0.25]))
    bk.materialize_scales()
    assert torch.all(w.grad == 0.25) and bk.buckets[1].scale_applied
    before = w.detach().clone()
    opt.step(0)  # the optimizer does not apply the factor a second time
    ref = before.clone()
    m, v = torch.zeros_like(ref), torch.zeros_like(ref)
    _torch_adam_(ref.view(-1), m.view(-1), v.view(-1), torch.full_like(ref, 0.25).view(-1), 1e-2, 0.9, 0.999, 1e-8,
                 None, 0, None, 0)
    assert torch.allclose(w.detach(), ref)


def _sgd_worker(rank, world, port, mode, out):
    from paper_2507_01154_b200.ddp import DataParallelStep, _torch_sgd_

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    model = _bucket_model()
    g = torch.Generator().manual_seed(3)
    x, y = torch.randn(8, 16, generator=g), torch.randn(8, 8, generator=g)
    lo, hi = 8 * rank // world, 8 * (rank + 1) // world
    step = DataParallelStep(model, dp=False, mode=mode, lr=1e-2, rank=rank, world=world, global_batch=8,
                            adam_fn=_torch_sgd_, bucket_bytes=600, optimizer="sgd")
    assert all(b.m is None for b in step.buckets.buckets)
    for i in range(3):
        step(i, lambda: ((model(x[lo:hi]) - y[lo:hi]) ** 2).sum(1).sum() / 8)
    out[(mode, world, rank)] = [p.detach().clone() for p in model.parameters()]
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def test_bucketed_sgd_step_two_ranks_equals_plain_sgd():
    """DataParallelStep(optimizer="sgd"): plain SGD on the bucket layout, world 2 over
    gloo in both bucket modes == three plain SGD steps on the global batch."""
    model = _bucket_model()
    g = torch.Generator().manual_seed(3)
    x, y = torch.randn(8, 16, generator=g), torch.randn(8, 8, generator=g)
    for _ in range(3):
        model.zero_grad()
        (((model(x) - y) ** 2).sum(1).sum() / 8).backward()
        with torch.no_grad():
            for p in model.parameters():
                p -= 1e-2 * p.grad
    ref = [p.detach().clone() for p in model.parameters()]
    for mode in ("allreduce", "reduce_scatter"):
        with mp.Manager() as mgr:
            out = mgr.dict()
            _sgd_worker(0, 1, _free_port(), mode, out)
            mp.spawn(_sgd_worker, args=(2, _free_port(), mode, out), nprocs=2, join=True)
            for key in ((mode, 1, 0), (mode, 2, 0), (mode, 2, 1)):
                for a, b in zip(out[key], ref):
                    assert torch.allclose(a, b, rtol=1e-5, atol=1e-6), key
