"""Host-side (Python) cost of one GPT-2 training step, DP vs non-DP (cProfile): where the
CPU time goes when the step is host-bound (small batches).

    python tools/host_profile.py [--batch 1] [--full]
"""
import argparse
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_01154_b200.dplinear import GroupedDPBackward  # noqa: E402
from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--full", action="store_true")
    a = ap.parse_args()
    for dp in (False, True):
        torch.manual_seed(0)
        cfg = GPT2Config(seq=1024)
        model = GPT2(cfg, dp=dp, clip_c=1.0, sigma=1.0, tied=not a.full, nondp_linear="fp32grad").cuda()
        opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
        idx = torch.randint(0, cfg.vocab, (a.batch, 1025), device="cuda")
        x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
        layers = model.dp_modules()

        def step(i):
            for m in layers:
                m.set_step(i)
            opt.zero_grad(set_to_none=True)
            loss = model.loss(x, y)
            if dp:
                with GroupedDPBackward():
                    loss.backward()
            else:
                loss.backward()
            opt.step()

        for i in range(5):
            step(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(10):
            step(i)
        host = (time.perf_counter() - t0) / 10
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 10
        pr = cProfile.Profile()
        pr.enable()
        for i in range(5):
            step(i)
        pr.disable()
        torch.cuda.synchronize()
        sio = io.StringIO()
        pstats.Stats(pr, stream=sio).sort_stats("tottime").print_stats(25)
        print(f"=== dp={dp} batch={a.batch} full={a.full}: host enqueue {host*1e3:.2f} ms/step, wall {wall*1e3:.2f} ms/step")
        print(sio.getvalue()[:6000])
        del model, opt


if __name__ == "__main__":
    main()
