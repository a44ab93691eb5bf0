import os, socket, sys, warnings
warnings.filterwarnings("ignore")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist, torch.multiprocessing as mp
def port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p
def worker(rank, world, prt, out):
    warnings.filterwarnings("ignore")
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(prt)
    os.environ["FDP_DDP_TRACE"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_01154_b200.ddp import DataParallelStep
    from paper_2507_01154_b200.llama import Llama, LlamaConfig
    cfg = LlamaConfig(vocab=512, d=256, heads=4, layers=2, mlp=512, seq=128)
    B = 4; g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), generator=g).cuda()
    lo, hi = B * rank // world, B * (rank + 1) // world
    x, y = idx[lo:hi, :-1].contiguous(), idx[lo:hi, 1:].contiguous()
    res = {}
    for nocomm in ("1", "0"):
        os.environ["FDP_DDP_NOCOMM"] = nocomm
        torch.manual_seed(0)
        with torch.device("cuda"):
            model = Llama(cfg, dp=False, nondp_linear="fp32grad")
        step = DataParallelStep(model, dp=False, lr=1e-3, rank=rank, world=world, global_batch=B, bucket_bytes=1 << 20)
        step(0, lambda: model.loss(x, y, reduction="sample_sum") / B)
        torch.cuda.synchronize()
        res[nocomm] = ({n: p.grad.detach().cpu().clone() for n, p in model.named_parameters()}, step.buckets.trace,
                       [[[n for n, q in model.named_parameters() if q is p][0] for p in b.params] for b in step.buckets.buckets])
    out[rank] = res
    dist.destroy_process_group()
if __name__ == "__main__":
    with mp.get_context("spawn").Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(worker, args=(2, port(), out), nprocs=2, join=True, start_method="spawn")
        l0, l1 = out[0]["1"][0], out[1]["1"][0]
        c0 = out[0]["0"][0]
        print("buckets", out[0]["0"][2])
        print("trace", out[0]["0"][1])
        for n in l0:
            s = l0[n] + l1[n]
            d = float((c0[n] - s).abs().max()); r = float(s.abs().max())
            if d > 1e-4 * r:
                print(n, "diff", d, "ref", r, "eq local0?", float((c0[n] - l0[n]).abs().max()), "eq local1?", float((c0[n] - l1[n]).abs().max()), "eq 2*local0?", float((c0[n] - 2*l0[n]).abs().max()))
