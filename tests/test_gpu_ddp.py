"""Data-parallel composition on the GPU: two ranks (processes) sharing cuda:0,
gloo for the collective, each running the fused multi-layer DP backward on its
half of the batch through ChunkedAllReduceBackward (chunk launches capped below
the SM count, all-reduce of each chunk on a side stream). The summed result must
equal the single-GPU result with the noise added exactly once."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dp_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [(256, 768), (768, 256), (256, 512), (512, 512), (256, 256)]  # (P, D) per layer


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    g = torch.Generator().manual_seed(11)
    B, T = 4, 128
    return [((torch.randn(B, T, P, generator=g)).to(torch.bfloat16),
             (torch.randn(B, T, D, generator=g) * 0.05).to(torch.bfloat16)) for P, D in SHAPES]


def _cfg(i):
    import paper_2507_01154_b200 as fdp
    return fdp.DPConfig(0.5, 1.0, "mean", seed=21, layer_id=i, step=4)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01154_b200.ddp import ChunkedAllReduceBackward

    data = _inputs()
    B = data[0][0].shape[0]
    lo, hi = B * rank // world, B * (rank + 1) // world
    layers = [(x[lo:hi].contiguous().cuda(), dy[lo:hi].contiguous().cuda(), _cfg(i)) for i, (x, dy) in enumerate(data)]
    n = sum(P * D for P, D in SHAPES)
    flat = torch.zeros(n, device="cuda")
    step = ChunkedAllReduceBackward(layers, flat, n_chunks=2, comm_sms=24, noise_impl="keyed_f64", rank=rank,
                                    world=world, mean_batch=B)
    assert step.max_ctas > 0 and len(step.chunks) == 2
    step()
    torch.cuda.synchronize()
    if rank == 0:
        out["flat"] = flat.cpu().numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_gpu_chunked_allreduce_equals_single_gpu():
    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
        got = out["flat"]
    off = 0
    for i, (x, dy) in enumerate(_inputs()):
        c = _cfg(i)
        want, _ = O.dp_backward(x.double().numpy(), dy.double().numpy(),
                                O.Cfg(c.clip_c, c.sigma, c.reduction, c.seed, c.layer_id, c.step), exact_noise=True)
        g = got[off:off + want.size].reshape(want.shape)
        off += want.size
        assert np.max(np.abs(g - want)) / np.max(np.abs(want)) < 1e-3, i


def test_group_cta_cap_matches_uncapped():
    import paper_2507_01154_b200 as fdp

    data = _inputs()
    layers = [(x.cuda(), dy.cuda(), _cfg(i)) for i, (x, dy) in enumerate(data)]
    full = fdp.PreparedGroup(layers, noise_impl="keyed_f64")
    capped = fdp.PreparedGroup(layers, noise_impl="keyed_f64", max_ctas=40)
    full()
    capped()
    torch.cuda.synchronize()
    for a, b in zip(full.grads, capped.grads):
        assert torch.allclose(a, b, rtol=1e-5, atol=1e-6 * float(a.abs().max()))
