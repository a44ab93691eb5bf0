import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_01154_b200.ddp import DataParallelStep, _torch_adam_
from paper_2507_01154_b200.llama import Llama, LlamaConfig
cfg = LlamaConfig.named("llama-7b", layers=2, seq=2048)
for lin in ["torch", "fp32grad"]:
    for fn in [None, _torch_adam_]:
        torch.manual_seed(0)
        with torch.device("cuda"):
            model = Llama(cfg, dp=False, nondp_linear=lin)
        g = torch.Generator(device="cuda").manual_seed(1)
        idx = torch.randint(0, cfg.vocab, (1, cfg.seq + 1), device="cuda", generator=g)
        x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
        step = DataParallelStep(model, dp=False, lr=1e-5, global_batch=1, adam_fn=fn)
        ls = []
        for i in range(4):
            ls.append(float(step(i, lambda: model.loss(x, y, reduction="sample_sum"))))
        gn = [float(p.grad.norm()) for p in list(model.parameters())[:3]]
        print(lin, "kernel" if fn is None else "torch", ls, gn, flush=True)
        del model, step
        torch.cuda.empty_cache()
