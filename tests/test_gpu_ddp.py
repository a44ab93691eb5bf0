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


def _zero1_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2507_01154_b200 as fdp
    from paper_2507_01154_b200.ddp import ShardedDPAdam

    data = _inputs()
    B = data[0][0].shape[0]
    lo, hi = B * rank // world, B * (rank + 1) // world
    grads = []
    for i, (x, dy) in enumerate(data):  # clipped sums of this rank's samples, no noise, / global B
        r = fdp.backward_flashdp(x[lo:hi].contiguous().cuda(), dy[lo:hi].contiguous().cuda(), _cfg(i),
                                 add_noise=False, mean_batch=B)
        grads.append(r.grad_w.reshape(-1))
    flat = torch.cat(grads)
    params = torch.linspace(-1, 1, flat.numel(), device="cuda")
    opt = ShardedDPAdam([(P * D, _cfg(i)) for i, (P, D) in enumerate(SHAPES)], params, eta=0.01,
                        noise_impl="keyed_f64", rank=rank, world=world)
    opt.step(flat, cfg_step=4)
    torch.cuda.synchronize()
    if rank == 0:
        out["params"] = params.cpu().numpy()
    dist.barrier()
    dist.destroy_process_group()


def test_zero1_sharded_adam_two_ranks_equals_single_gpu():
    """ZeRO-1 form of 8e: noise-free clipped sums reduce-scattered, each rank adds
    its shard's DP noise inside its Adam step, params all-gathered == one-process
    DP gradient (noise included) followed by Adam."""
    import paper_2507_01154_b200 as fdp

    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_zero1_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
        got = out["params"]
    grads = []
    for i, (x, dy) in enumerate(_inputs()):
        grads.append(fdp.backward_flashdp(x.cuda(), dy.cuda(), _cfg(i), noise_impl="keyed_f64").grad_w.reshape(-1))
    flat = torch.cat(grads)
    st = fdp.OptimizerState.fresh(torch.linspace(-1, 1, flat.numel(), device="cuda"), eta=0.01)
    st = fdp.dp_adam_step_(st, flat)
    want = st.theta.cpu().numpy()
    start = np.linspace(-1, 1, flat.numel())
    assert np.max(np.abs((got - start) - (want - start))) / np.max(np.abs(want - start)) < 1e-4


def _full_dp_worker(rank, world, port, out):
    """Every-parameter DP GPT-2 (tiny) on this rank's half of the batch, gloo all-reduce of all gradients."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01154_b200.ddp import allreduce_grads_, set_data_parallel
    from paper_2507_01154_b200.dplinear import GroupedDPBackward
    from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config

    torch.manual_seed(0)
    cfg = GPT2Config(vocab=512, seq=32, d=128, heads=4, layers=1, mlp=256)
    model = GPT2(cfg, dp="full", clip_c=0.3, sigma=0.5, noise_impl="keyed_f64", tied=False).cuda()
    g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, cfg.vocab, (4, cfg.seq + 1), generator=g).cuda()
    B = idx.shape[0]
    lo, hi = B * rank // world, B * (rank + 1) // world
    mods = model.dp_modules()
    set_data_parallel(mods, rank, world)
    for m in mods:
        m.set_step(3, logical_batch=B)
    x, y = idx[lo:hi, :-1].contiguous(), idx[lo:hi, 1:].contiguous()
    with GroupedDPBackward():
        # the loss is a per-token mean: rescale so this rank's share is the global mean's
        (model.loss(x, y) * ((hi - lo) / B)).backward()
    grads = [p.grad for p in model.parameters()]
    if world > 1:
        allreduce_grads_(grads)
    torch.cuda.synchronize()
    if rank == 0:
        out[f"w{world}"] = [t.detach().cpu().numpy() for t in grads]
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_full_dp_gpt2_equals_single_process():
    """SURVEY 8e for every parameter group: two ranks with rank-partitioned keyed
    noise and the global-batch mean, all-reduced, equal one process on the whole
    batch (noise added exactly once, per-sample clipping unchanged)."""
    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_full_dp_worker, args=(1, _free_port(), out), nprocs=1, join=True, start_method="spawn")
        mp.start_processes(_full_dp_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
        one, two = out["w1"], out["w2"]
    assert len(one) == len(two)
    for a, b in zip(one, two):
        assert np.max(np.abs(a - b)) <= 2e-2 * max(float(np.max(np.abs(a))), 1e-6)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rank_partitioned_noise_sums_to_single_gpu(world):
    """SURVEY 8e for W in {1, 2, 4, 8}: each rank runs its slice of the batch with
    noise on its slice of [0, D*P) only and the global-batch mean; the sum over
    ranks equals the one-process result, and the per-rank noise parts are disjoint
    and add up to the W = 1 noise (reference-keyed: exact draws)."""
    import paper_2507_01154_b200 as fdp

    g = torch.Generator().manual_seed(17)
    B, T, P, D = 8, 96, 256, 384
    x = torch.randn(B, T, P, generator=g).to(torch.bfloat16).cuda()
    dy = (torch.randn(B, T, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
    cfg = fdp.DPConfig(0.4, 1.0, "mean", seed=8, layer_id=2, step=6)
    cfg0 = fdp.DPConfig(0.4, 0.0, "mean", seed=8, layer_id=2, step=6)
    one = fdp.backward_flashdp(x, dy, cfg, noise_impl="keyed_f64").grad_w
    one0 = fdp.backward_flashdp(x, dy, cfg0, noise_impl="keyed_f64").grad_w
    total = torch.zeros_like(one)
    noise_parts = []
    for r in range(world):
        lo, hi = B * r // world, B * (r + 1) // world
        xs, ys = x[lo:hi].contiguous(), dy[lo:hi].contiguous()
        kw = dict(noise_impl="keyed_f64", rank=r, world=world, mean_batch=B)
        out = fdp.backward_flashdp(xs, ys, cfg, **kw).grad_w
        out0 = fdp.backward_flashdp(xs, ys, cfg0, **kw).grad_w
        total += out
        noise_parts.append((out - out0).reshape(-1))
    scale = float(one.abs().max())
    assert float((total - one).abs().max()) <= 1e-5 * scale
    full_noise = (one - one0).reshape(-1)
    n = P * D
    for r, part in enumerate(noise_parts):
        lo, hi = n * r // world, n * (r + 1) // world
        assert float(part[:lo].abs().max() if lo else 0.0) <= 1e-5 * scale  # nothing outside the slice
        assert float(part[hi:].abs().max() if hi < n else 0.0) <= 1e-5 * scale
        assert float((part[lo:hi] - full_noise[lo:hi]).abs().max()) <= 1e-5 * scale


# ---------------------------------------------------------------- bucketed Llama training step


def _tiny_llama_cfg():
    from paper_2507_01154_b200.llama import LlamaConfig

    return LlamaConfig(vocab=512, d=256, heads=4, layers=2, mlp=512, seq=128)


def _llama_step_worker(rank, world, port, mode, dp, out, opt_noise=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01154_b200.ddp import DataParallelStep
    from paper_2507_01154_b200.llama import Llama

    cfg = _tiny_llama_cfg()
    torch.manual_seed(0)
    with torch.device("cuda"):
        model = Llama(cfg, dp=dp, clip_c=0.5, sigma=1.0, noise_impl="philox", nondp_linear="fp32grad")
    B = 4
    g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), generator=g).cuda()
    lo, hi = B * rank // world, B * (rank + 1) // world
    x, y = idx[lo:hi, :-1].contiguous(), idx[lo:hi, 1:].contiguous()
    step = DataParallelStep(model, dp=dp, mode=mode, lr=1e-3, rank=rank, world=world, global_batch=B,
                            bucket_bytes=1 << 20, noise_in_optimizer=opt_noise)
    scale = 1.0 if dp else 1.0 / B
    grads = None
    for i in range(2):
        step(i, lambda: model.loss(x, y, reduction="sample_sum") * scale)
        if i == 0:  # the reduced gradients of step 0 (this rank's shard under reduce-scatter)
            torch.cuda.synchronize()
            bk = step.buckets
            grads = [(b.flat if mode == "allreduce" else b.shard).detach().cpu().clone() for b in bk.buckets]
            pers = [b.per for b in bk.buckets]
    step.finish()
    torch.cuda.synchronize()
    out[(mode, dp, world, rank, opt_noise)] = ([p.detach().cpu().clone() for p in model.parameters()],
                                    list(step.buckets.issued), len(step.buckets.buckets), step.last_flushes,
                                    grads, pers)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,opt_noise", [("allreduce", True), ("allreduce", False), ("reduce_scatter", True)])
@pytest.mark.parametrize("dp", [True, False])
def test_bucketed_llama_step_two_ranks_equals_single_process(mode, opt_noise, dp):
    """Two ranks (processes) sharing cuda:0 over gloo run the tiny-Llama training
    step through DataParallelStep: every parameter DP (DPLinear / DPRMSNorm /
    DPEmbedding, Philox noise), gradient buckets flushed from inside the backward
    (GroupedDPBackward(buckets=...)), then all-reduce + replicated DP-Adam or
    reduce-scatter + ZeRO-1 Adam with the noise added on the owner's shard
    (all-reduce: the noise either inside every replica's Adam step from the same
    keyed draws, or by the DP kernels on each rank's slice).
    After two steps the parameters equal the single-process run on the global
    batch (noise once per element either way). dp=False: the non-DP baseline
    (FP32GradLinear projections) through the same buckets and optimizer."""
    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_llama_step_worker, args=(1, _free_port(), mode, dp, out, opt_noise), nprocs=1,
                           join=True, start_method="spawn")
        mp.start_processes(_llama_step_worker, args=(2, _free_port(), mode, dp, out, opt_noise), nprocs=2,
                           join=True, start_method="spawn")
        ref, _, nb, flushes, ref_g, _ = out[(mode, dp, 1, 0, opt_noise)]
        assert nb >= 3
        if dp:
            assert flushes >= 2  # DP kernels ran bucket by bucket inside the backward
        for r in range(2):
            got, issued, _, _, g2, pers = out[(mode, dp, 2, r, opt_noise)]
            assert issued == out[(mode, dp, 2, 0, opt_noise)][1]
            # step-0 gradients: summed over the ranks == the single-process gradients
            for k, (a, full) in enumerate(zip(g2, ref_g)):
                b = full if mode == "allreduce" else torch.cat([full, torch.zeros(2 * pers[k])])[
                    r * pers[k]:(r + 1) * pers[k]]
                n = min(a.numel(), b.numel())
                assert torch.allclose(a[:n], b[:n], rtol=1e-4, atol=1e-6 * float(b.abs().max())), (mode, dp, k)
            if dp:  # parameters after two DP-Adam steps (noise keeps every gradient away from 0)
                for a, b in zip(got, ref):
                    assert torch.allclose(a, b, rtol=1e-4, atol=2e-6), (mode, dp, float((a - b).abs().max()))
