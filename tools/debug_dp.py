"""Debug: tiny-Llama DataParallelStep, world 1 vs 2 (two ranks on cuda:0, gloo)."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, prt, mode, dp, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(prt)
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01154_b200.ddp import DataParallelStep
    from paper_2507_01154_b200.llama import Llama, LlamaConfig

    cfg = LlamaConfig(vocab=512, d=256, heads=4, layers=2, mlp=512, seq=128)
    torch.manual_seed(0)
    with torch.device("cuda"):
        model = Llama(cfg, dp=dp, clip_c=0.5, sigma=float(os.environ.get("SIG", "1.0")), noise_impl="philox",
                      nondp_linear="fp32grad")
    B = 4
    g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), generator=g).cuda()
    lo, hi = B * rank // world, B * (rank + 1) // world
    x, y = idx[lo:hi, :-1].contiguous(), idx[lo:hi, 1:].contiguous()
    step = DataParallelStep(model, dp=dp, mode=mode, lr=1e-3, rank=rank, world=world, global_batch=B,
                            bucket_bytes=1 << 20)
    scale = 1.0 if dp else 1.0 / B
    losses, grads = [], []
    for i in range(2):
        losses.append(float(step(i, lambda: model.loss(x, y, reduction="sample_sum") * scale)))
        torch.cuda.synchronize()
        grads.append({n: p.grad.detach().cpu().clone() for n, p in model.named_parameters()})
    out[(world, rank)] = ({n: p.detach().cpu().clone() for n, p in model.named_parameters()}, losses, grads,
                          list(step.buckets.issued))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "allreduce"
    dp = (sys.argv[2] if len(sys.argv) > 2 else "1") == "1"
    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(worker, args=(1, port(), mode, dp, out), nprocs=1, join=True, start_method="spawn")
        mp.start_processes(worker, args=(2, port(), mode, dp, out), nprocs=2, join=True, start_method="spawn")
        p1, l1, g1, i1 = out[(1, 0)]
        p2, l2, g2, i2 = out[(2, 0)]
        print("mode", mode, "dp", dp, "losses w1", l1, "w2 r0", l2, "w2 r1", out[(2, 1)][1])
        print("issued", i1, i2)
        for s in range(2):
            for n in g1[s]:
                d = float((g1[s][n] - g2[s][n]).abs().max())
                ref = float(g1[s][n].abs().max())
                if d > 1e-5 * max(ref, 1e-3):
                    print("step", s, "grad", n, "maxdiff", d, "ref max", ref)
        for n in p1:
            d = float((p1[n] - p2[n]).abs().max())
            if d > 1e-5:
                print("param", n, "maxdiff", d)
