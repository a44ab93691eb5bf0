"""World-size-2 data-parallel composition on CPU (gloo): per-rank contributions
(clipped sum over the rank's samples / global B + noise on the rank's index
slice, exactly what the kernel computes with rank/world/mean_batch) summed by
paper_2507_01154_b200.ddp.allreduce_grads_ equal the single-process result."""

import os
import socket

import numpy as np
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
