"""Interleaved A/B timing of native-layer variants on single layers (any path).

    [AB_PATH=fused|two_phase] python tools/ab_layer.py "B,T,P,D[;B,T,P,D...]" VAR1 VAR2 ...   (VAR as in tools/ab.py)

Round-robin over variants with an idle gap before each measurement (same thermal
start); prints min / median per (shape, variant) as JSON lines.
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

ROUNDS = int(os.environ.get("AB_ROUNDS", "4"))
SLEEP = float(os.environ.get("AB_SLEEP", "0.5"))


def timed(fn, n=5):
    time.sleep(SLEEP)
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def parse(v):
    return {} if v == "base" else dict(kv.split("=", 1) for kv in v.split(","))


def main():
    shapes = [tuple(int(t) for t in s.split(",")) for s in sys.argv[1].split(";")]
    variants = sys.argv[2:] or ["base"]
    base_env = dict(os.environ)
    g = torch.Generator(device="cuda").manual_seed(0)
    for B, T, P, D in shapes:
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
        calls = {}
        for v in variants:
            os.environ.clear()
            os.environ.update(base_env)
            os.environ.update(parse(v))
            calls[v] = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox",
                                            path=os.environ.get("AB_PATH", "auto"))
        res = {v: [] for v in variants}
        for _ in range(ROUNDS):
            for v in variants:
                os.environ.clear()
                os.environ.update(base_env)
                os.environ.update(parse(v))
                res[v].append(timed(calls[v]))
        os.environ.clear()
        os.environ.update(base_env)
        for v in variants:
            print(json.dumps({"B": B, "T": T, "P": P, "D": D, "variant": v, "min_us": round(min(res[v]), 1),
                              "median_us": round(statistics.median(res[v]), 1)}), flush=True)
        del x, dy, calls
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
