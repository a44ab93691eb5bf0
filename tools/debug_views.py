import os, sys, warnings
warnings.filterwarnings("ignore")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_01154_b200.ddp import DataParallelStep
from paper_2507_01154_b200.llama import Llama, LlamaConfig
cfg = LlamaConfig(vocab=512, d=256, heads=4, layers=2, mlp=512, seq=128)
for dp in (False, True):
    torch.manual_seed(0)
    with torch.device("cuda"):
        model = Llama(cfg, dp=dp, clip_c=0.5, sigma=0.0, noise_impl="philox", nondp_linear="fp32grad")
    idx = torch.randint(0, cfg.vocab, (2, cfg.seq + 1), device="cuda")
    x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
    step = DataParallelStep(model, dp=dp, lr=1e-3, global_batch=2, bucket_bytes=1 << 20)
    bk = step.buckets
    for it in range(2):
        step(it, lambda: model.loss(x, y, reduction="sample_sum") * (1.0 if dp else 0.5))
        torch.cuda.synchronize()
        for b in bk.buckets:
            for p, o in zip(b.params, b.offsets):
                view = b.flat[o:o + p.numel()]
                name = [n for n, q in model.named_parameters() if q is p][0]
                same = p.grad is not None and p.grad.data_ptr() == view.data_ptr()
                eq = p.grad is not None and torch.equal(p.grad.reshape(-1), view)
                if not (same and eq):
                    print("dp", dp, "step", it, name, "view?", same, "equal?", eq,
                          float(view.abs().max()), None if p.grad is None else float(p.grad.abs().max()))
print("done")
