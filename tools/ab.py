"""Interleaved A/B timing of native-layer variants on the 48-layer GPT-2 group.

    python tools/ab.py VAR1 VAR2 ...      e.g.  base FDP_DEBUG_NOSYNC=1 FDP_NO_PACK=1

Each variant is a comma-separated list of ENV=VALUE settings ("base" = none)
applied to os.environ before the timed launches (the native layer reads its
debug/planning environment per call). Variants are timed round-robin for
several rounds on the same buffers so that clock / thermal drift hits all of
them alike; the minimum and median over rounds are printed per variant.
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

TYPES = [("c_attn", 768, 2304), ("attn_proj", 768, 768), ("c_fc", 768, 3072), ("mlp_proj", 3072, 768)]
B = int(os.environ.get("AB_B", "8"))
T = int(os.environ.get("AB_T", "1024"))
ROUNDS = int(os.environ.get("AB_ROUNDS", "5"))
SLEEP = float(os.environ.get("AB_SLEEP", "1.0"))  # idle before each measurement: same thermal start
ITERS = int(os.environ.get("AB_ITERS", "10"))


def timed(fn, n=ITERS):
    time.sleep(SLEEP)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3  # us


def parse(v):
    if v == "base":
        return {}
    return dict(kv.split("=", 1) for kv in v.split(","))


def main():
    variants = sys.argv[1:] or ["base"]
    g = torch.Generator(device="cuda").manual_seed(0)
    layers, flops = [], 0
    for blk in range(12):
        for j, (name, P, D) in enumerate(TYPES):
            x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
            dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
            layers.append((x, dy, fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=blk * 4 + j)))
            flops += 2 * B * T * P * D
    grads = [torch.zeros(d.shape[2], x.shape[2], device="cuda") for x, d, _ in layers]
    groups = {}
    base_env = dict(os.environ)
    for v in variants:
        os.environ.clear()
        os.environ.update(base_env)
        os.environ.update(parse(v))
        groups[v] = fdp.PreparedGroup(layers, grads=grads, noise_impl="philox")
    x2 = [(x.view(-1, x.shape[2]), d.view(-1, d.shape[2])) for x, d, _ in layers]

    def cublas():
        for x, d in x2:
            torch.mm(d.t(), x, out_dtype=torch.float32)

    res = {v: [] for v in variants + ["cublas_nondp"]}
    for _ in range(ROUNDS):
        for v in variants:
            os.environ.clear()
            os.environ.update(base_env)
            os.environ.update(parse(v))
            res[v].append(timed(groups[v]))
        res["cublas_nondp"].append(timed(cublas))
    os.environ.clear()
    os.environ.update(base_env)
    for v, ts in res.items():
        print(json.dumps({"variant": v, "min_us": round(min(ts), 1), "med_us": round(statistics.median(ts), 1),
                          "tflops_at_min": round(flops / min(ts) / 1e6, 1), "all": [round(t, 1) for t in ts]}))


if __name__ == "__main__":
    main()
