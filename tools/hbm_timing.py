"""Warm timing (CUDA events) of the HBM-bound kernels: fp32 DP-Adam with shard noise,
without noise, with a deferred clip factor; the B = 1 clip + noise finalize (via the
single-sample path minus its GEMM); reports GB/s of the algorithmic bytes.

    python tools/hbm_timing.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402


def timed(fn, n=20):
    time.sleep(0.3)
    for _ in range(3):
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
    n = 1 << 27  # 134 M parameters: 3.75 GB of Adam traffic per step
    g = torch.Generator(device="cuda").manual_seed(0)
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=2)
    st = fdp.OptimizerState.fresh(torch.zeros(n, device="cuda"), eta=1e-4)
    grad = torch.randn(n, device="cuda", generator=g)
    scale = torch.full((1,), 0.5, device="cuda")
    bytes_adam = 28.0 * n
    row = {"lib": os.environ.get("FDP_LIB_PATH", "base")}
    for name, kw in (("adam_noise", dict(noise=cfg, layer_numel=n)), ("adam_plain", {}),
                     ("adam_scaled", dict(grad_scale=scale))):
        us = timed(lambda: fdp.dp_adam_step_(st, grad, **kw))
        row[name + "_us"] = round(us, 1)
        row[name + "_gbs"] = round(bytes_adam / us / 1e3, 0)
    # the one-launch bucketed DP-Adam over the same 134 M parameters (+ 64 small ones)
    from paper_2507_01154_b200.ddp import BucketedAdam, GradBuckets

    ps = [torch.nn.Parameter(torch.zeros(n, device="cuda"))] + [torch.nn.Parameter(torch.zeros(768, device="cuda"))
                                                               for _ in range(64)]
    bk = GradBuckets(ps, flat_params=True, hooks=False, isolate=ps[:1])
    bk.zero_grad()
    keys = {id(p_): (cfg, 0, p_.numel(), "philox") for p_ in ps}
    opt = BucketedAdam(bk, lr=1e-4, noise_keys=keys)
    it = [0]

    def multi():
        it[0] += 1
        opt.step(it[0])
    us = timed(multi)
    row["adam_multi_noise_us"] = round(us, 1)
    row["adam_multi_noise_gbs"] = round(28.0 * (n + 64 * 768) / us / 1e3, 0)
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
