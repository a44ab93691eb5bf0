"""Quick GPU diagnostics: run each path on small shapes, compare with the oracle.

    python tools/gpu_diag.py [case ...]

Each case runs in a child process with a timeout so one failure (or a trapped
kernel) does not hide the others. Prints one line per case.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    # name: (B, T, P, D, dtype, path, clip_c, sigma, reduction, kind)
    "nondp_tc_small": (2, 64, 128, 128, "bf16", "auto", 1.0, 0.0, "sum", "non_dp"),
    "fused_small": (2, 64, 128, 128, "bf16", "fused", 1.0, 0.0, "sum", "flashdp"),
    "fused_c1": (4, 128, 256, 256, "bf16", "fused", 1.0, 0.0, "sum", "flashdp"),
    "fused_c1_noise": (4, 128, 256, 256, "bf16", "fused", 1.0, 1.0, "sum", "flashdp"),
    "fused_ragged": (3, 100, 200, 136, "bf16", "fused", 0.05, 0.0, "mean", "flashdp"),
    "two_phase": (4, 128, 256, 384, "bf16", "two_phase", 1.0, 0.0, "sum", "flashdp"),
    "simt_f32": (3, 17, 13, 9, "f32", "simt", 0.5, 0.0, "sum", "flashdp"),
    "explicit": (4, 128, 256, 256, "bf16", "auto", 1.0, 1.0, "mean", "explicit_dp"),
    "implicit": (4, 128, 256, 256, "bf16", "auto", 1.0, 0.0, "sum", "implicit_dp"),
    "fused_gpt2_fc": (8, 1024, 768, 3072, "bf16", "fused", 1.0, 0.0, "sum", "flashdp"),
    "fused_gpt2_attnproj": (8, 1024, 768, 768, "bf16", "fused", 1.0, 0.0, "sum", "flashdp"),
}


def run_case(name: str) -> dict:
    import numpy as np
    import torch

    import paper_2507_01154_b200 as fdp
    from oracle import dp_oracle as O

    B, T, P, D, dt, path, C, sigma, red, kind = CASES[name]
    g = torch.Generator().manual_seed(1234)
    x = torch.randn(B, T, P, generator=g, dtype=torch.float32)
    dy = torch.randn(B, T, D, generator=g, dtype=torch.float32)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    xd, yd = x.to(tdt).cuda(), dy.to(tdt).cuda()
    xo, yo = xd.double().cpu().numpy(), yd.double().cpu().numpy()
    cfg = fdp.DPConfig(clip_c=C, sigma=sigma, reduction=red, seed=7, layer_id=3, step=11)
    ocfg = O.Cfg(C, sigma, red, 7, 3, 11)
    out = {"case": name}
    if kind == "flashdp":
        out["plan"] = fdp.execution_plan((B, T, P), (B, T, D), path=path)
    t0 = time.time()
    res = fdp.run_backward(fdp.WorkflowKind(kind), xd, yd, cfg, path=path)
    torch.cuda.synchronize()
    out["first_call_s"] = round(time.time() - t0, 4)
    gw = res.grad_w.double().cpu().numpy()
    if kind == "non_dp":
        want = O.nondp_backward(xo, yo)
    else:
        want, wn = O.dp_backward(xo, yo, ocfg, exact_noise=False)
        n = res.per_sample_norms_sq.double().cpu().numpy()
        out["norm_rel"] = float(np.max(np.abs(n - wn) / np.maximum(wn, 1e-30)))
    scale = float(np.max(np.abs(want))) or 1.0
    out["grad_rel"] = float(np.max(np.abs(gw - want)) / scale)
    # timing
    for _ in range(3):
        fdp.run_backward(fdp.WorkflowKind(kind), xd, yd, cfg, path=path)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n_it = 10
    for _ in range(n_it):
        fdp.run_backward(fdp.WorkflowKind(kind), xd, yd, cfg, path=path)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n_it
    out["ms"] = round(ms, 4)
    out["tflops"] = round(2 * B * T * P * D / (ms * 1e-3) / 1e12, 2)
    return out


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        try:
            print("RESULT " + json.dumps(run_case(sys.argv[2])), flush=True)
        except Exception as e:  # noqa: BLE001
            print("RESULT " + json.dumps({"case": sys.argv[2], "error": repr(e)[:400]}), flush=True)
        return
    names = sys.argv[1:] or list(CASES)
    for n in names:
        try:
            r = subprocess.run([sys.executable, __file__, "--child", n], capture_output=True, text=True, timeout=120)
            line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
            print(line[-1][7:] if line else json.dumps({"case": n, "rc": r.returncode,
                                                        "stderr": r.stderr[-600:]}), flush=True)
        except subprocess.TimeoutExpired:
            print(json.dumps({"case": n, "error": "timeout"}), flush=True)


if __name__ == "__main__":
    main()
