"""torch.profiler breakdown of the GPT-2 training step (DP vs non-DP): top CUDA kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2507_01154_b200.dplinear import GroupedDPBackward  # noqa: E402
from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config  # noqa: E402

for dp in (False, True):
    torch.manual_seed(0)
    cfg = GPT2Config()
    model = GPT2(cfg, dp=dp).cuda()
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
    idx = torch.randint(0, cfg.vocab, (8, 1025), device="cuda")
    x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()

    def step():
        opt.zero_grad(set_to_none=True)
        loss = model.loss(x, y)
        if dp:
            with GroupedDPBackward():
                loss.backward()
        else:
            loss.backward()
        opt.step()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            step()
        torch.cuda.synchronize()
    print("==== dp" if dp else "==== non-dp")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18, max_name_column_width=60))
