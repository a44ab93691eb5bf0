"""cProfile of the eager DataParallelStep (GPT-2 small, every parameter DP, B = 1):
where the host time of a small-batch step goes.

    python tools/host_profile_dps.py
"""
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_01154_b200.ddp import DataParallelStep  # noqa: E402
from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config  # noqa: E402

for dp in (False, True):
    torch.manual_seed(0)
    cfg = GPT2Config(seq=1024)
    model = GPT2(cfg, dp="full" if dp else False, tied=False, nondp_linear="fp32grad").cuda()
    step = DataParallelStep(model, dp=dp, lr=1e-4, global_batch=1)
    idx = torch.randint(0, cfg.vocab, (1, 1025), device="cuda")
    x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
    fn = (lambda: model.loss(x, y)) if dp else (lambda: model.loss(x, y))
    for i in range(5):
        step(i, fn)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(10):
        step(i, fn)
    host = (time.perf_counter() - t0) / 10
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for i in range(5):
        step(i, fn)
    pr.disable()
    torch.cuda.synchronize()
    sio = io.StringIO()
    pstats.Stats(pr, stream=sio).sort_stats("tottime").print_stats(30)
    print(f"=== dp={dp}: host {host * 1e3:.2f} ms/step")
    print(sio.getvalue()[:7000])
    del model, step
