"""B=1 Llama-13B layer shapes: single-sample path vs ghost + reweight vs cuBLAS dW.

    python tools/single_parts.py            # event-timed, one JSON line per shape
    tools/ktimes.sh out.csv python tools/single_parts.py --once   # per-kernel split
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

SHAPES = [(5120, 5120), (5120, 13824), (13824, 5120)]


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def main():
    once = "--once" in sys.argv
    T = int(os.environ.get("SP_T", "2048"))
    B = int(os.environ.get("SP_B", "1"))
    g = torch.Generator(device="cuda").manual_seed(0)
    for P, D in SHAPES:
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
        row = {"B": B, "T": T, "P": P, "D": D}
        x2, y2 = x.view(-1, P), dy.view(-1, D)
        for name, kw in (("auto", {}), ("single", {"norm_phase": "single"} if B == 1 else None),
                         ("ghost", {"norm_phase": "ghost", "path": "two_phase"}),
                         ("recompute", {"norm_phase": "recompute", "path": "two_phase"})):
            if kw is None:
                continue
            c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", **kw)
            if once:
                c()
                torch.cuda.synchronize()
            else:
                row[name + "_us"] = round(timed(c), 1)
            del c
        if once:
            torch.mm(y2.t(), x2, out_dtype=torch.float32)
        else:
            row["cublas_us"] = round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32)), 1)
        torch.cuda.synchronize()
        if not once:
            print(json.dumps(row), flush=True)
        del x, dy
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
