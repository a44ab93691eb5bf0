"""Ghost-norm K-split sweep: two-phase layer time (ghost + reweight) for forced
(pair, split) vs the auto choice, on shapes where one operand's K dominates.

    python tools/ghost_split_sweep.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

SHAPES = [(8, 1024, 768, 50304), (1, 2048, 5120, 13824), (1, 2048, 4096, 32000), (1, 2048, 5120, 5120),
          (4, 2048, 4096, 32000)]


def timed(fn, n=5):
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
    g = torch.Generator(device="cuda").manual_seed(0)
    for B, T, P, D in SHAPES:
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
        row = {"B": B, "T": T, "P": P, "D": D}
        for pair in ("auto", "0", "1"):
            for split in ("auto", "1", "2", "3", "4", "6", "8", "12"):
                if pair == "auto" and split != "auto":
                    continue
                for k, v in (("FDP_GHOST_PAIR", pair), ("FDP_GHOST_SPLIT", split)):
                    if v == "auto":
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
                c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox",
                                         path="two_phase", norm_phase="ghost")
                row[f"p{pair}_s{split}"] = round(timed(c), 1)
                del c
        os.environ.pop("FDP_GHOST_PAIR", None)
        os.environ.pop("FDP_GHOST_SPLIT", None)
        x2, y2 = x.view(-1, P), dy.view(-1, D)
        row["cublas_us"] = round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32)), 1)
        print(json.dumps(row), flush=True)
        del x, dy
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
