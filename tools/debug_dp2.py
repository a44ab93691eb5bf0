"""world 1 vs the sum of world-2 LOCAL gradients (no collectives), tiny Llama on cuda:0."""
import os, socket, sys, warnings
warnings.filterwarnings("ignore")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.multiprocessing as mp
def port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p
def worker(rank, world, prt, dp, lin, out):
    warnings.filterwarnings("ignore")
    os.environ["FDP_DDP_NOCOMM"] = "1"
    torch.cuda.set_device(0)
    from paper_2507_01154_b200.ddp import DataParallelStep
    from paper_2507_01154_b200.llama import Llama, LlamaConfig
    cfg = LlamaConfig(vocab=512, d=256, heads=4, layers=2, mlp=512, seq=128)
    torch.manual_seed(0)
    with torch.device("cuda"):
        model = Llama(cfg, dp=dp, clip_c=0.5, sigma=0.0, noise_impl="philox", nondp_linear=lin)
    B = 4; g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), generator=g).cuda()
    lo, hi = B * rank // world, B * (rank + 1) // world
    x, y = idx[lo:hi, :-1].contiguous(), idx[lo:hi, 1:].contiguous()
    step = DataParallelStep(model, dp=dp, mode="allreduce", lr=1e-3, rank=rank, world=world, global_batch=B, bucket_bytes=1 << 20)
    step(0, lambda: model.loss(x, y, reduction="sample_sum") * (1.0 if dp else 1.0 / B))
    torch.cuda.synchronize()
    out[(world, rank)] = {n: p.grad.detach().cpu().clone() for n, p in model.named_parameters()}
if __name__ == "__main__":
    for dp, lin in ((False, "fp32grad"), (False, "torch"), (True, "torch")):
        with mp.get_context("spawn").Manager() as mgr:
            out = mgr.dict()
            for w in (1, 2):
                mp.start_processes(worker, args=(w, port(), dp, lin, out), nprocs=w, join=True, start_method="spawn")
            bad = []
            for n, g1 in out[(1, 0)].items():
                gs = out[(2, 0)][n] + out[(2, 1)][n]
                d = float((g1 - gs).abs().max()); r = float(g1.abs().max())
                if d > 1e-4 * max(r, 1e-6): bad.append((n, d, r))
            print("dp", dp, lin, "mismatches", bad[:8], flush=True)
