"""Warm per-kernel durations and launch gaps of one layer's DP backward (torch.profiler /
CUPTI), next to the CUDA-event time per call: where the two-phase path's time goes at
small T (ghost norms, factor reduce, reweight) vs the non-DP GEMM.

    python tools/smallT_phases.py [B T P D ...]   (default: the small-T shapes of DESIGN §6)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

SHAPES = [(64, 128, 1024, 1024), (64, 128, 2048, 2048), (128, 128, 1024, 1024), (32, 256, 2048, 2048)]


def events_us(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def kernels(fn, n=20):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
    ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                key=lambda e: e.time_range.start)
    per = {}
    for e in ev:
        per.setdefault(e.name[:48], []).append(e.time_range.elapsed_us())
    span = (ev[-1].time_range.end - ev[0].time_range.start) / n if ev else 0.0
    return {k: round(sum(v) / len(v), 2) for k, v in per.items()}, round(span, 2)


def main():
    shapes = [tuple(int(v) for v in sys.argv[i:i + 4]) for i in range(1, len(sys.argv), 4)] or SHAPES
    g = torch.Generator(device="cuda").manual_seed(0)
    for B, T, P, D in shapes:
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        cfg = fdp.DPConfig(1.0, float(os.environ.get("PH_SIGMA", "1.0")), "mean", seed=1, layer_id=2)
        row = {"shape": [B, T, P, D]}
        for name, kind, path in (("two_phase", fdp.WorkflowKind.FLASHDP, "two_phase"),
                                 ("fused", fdp.WorkflowKind.FLASHDP, "fused"),
                                 ("nondp", fdp.WorkflowKind.NON_DP, "auto")):
            try:
                call = fdp.PreparedBackward(kind, x, dy, cfg if kind != fdp.WorkflowKind.NON_DP else None,
                                            path=path, noise_impl="philox")
            except Exception as e:  # noqa: BLE001  (fused may not fit)
                row[name] = {"error": repr(e)[:80]}
                continue
            k, span = kernels(call)
            row[name] = {"event_us": round(events_us(call), 2), "span_us": span, "kernels_us": k}
        a, b = torch.empty(B * T, D, device="cuda", dtype=torch.bfloat16), x.view(-1, P)
        row["cublas_us"] = round(events_us(lambda: torch.mm(dy.view(-1, D).t(), b, out_dtype=torch.float32)), 2)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
