"""BASELINE config 5: DP-linear sweep d in {1024..8192}, B in {1..64}, T in {128..4096}.

For each point: the DP weight gradient through the auto-selected path (fused or
two-phase with ghost norms), the naive explicit (Opacus-style) baseline, and the
non-DP dW (cuBLAS), as TFLOP/s of the dense contraction F = 2 B T D P.

    python tools/layer_sweep.py [--quick] > profiles/layer_sweep.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3


def peak_tflops():
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["bf16_tflops"]), "measured bf16 burst (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 1617.0, "fallback"


def main():
    quick = "--quick" in sys.argv
    peak, peak_src = peak_tflops()
    print(json.dumps({"peak_tflops": peak, "peak_source": peak_src}), flush=True)
    points = []
    for d in (1024, 2048, 4096, 8192):
        for B, T in ((1, 4096), (8, 1024), (32, 512), (64, 128), (4, 2048)):
            points.append((B, T, d, d))
    points += [(4, 2048, 4096, 11008), (4, 2048, 11008, 4096), (2, 2048, 5120, 13824), (2, 2048, 13824, 5120)]
    if quick:
        points = points[::3]
    g = torch.Generator(device="cuda").manual_seed(0)
    for B, T, P, D in points:
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        F = 2.0 * B * T * P * D
        cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
        row = {"B": B, "T": T, "P": P, "D": D, "gflop": F / 1e9}
        c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox")
        row["dp_path"] = fdp._lib.PATH_NAMES[c.plan.path]
        row["dp_norm_phase"] = fdp._lib.NORM_PHASE_NAMES.get(c.plan.norm_phase, "-")
        row["dp_tile"] = [c.plan.tile_d, c.plan.tile_p, c.plan.groups]
        s = timed(c)
        row["dp_ms"] = s * 1e3
        row["dp_tflops"] = F / s / 1e12
        row["dp_frac_of_peak"] = row["dp_tflops"] / peak
        if B == 1:  # the training step's form: clip factor left to the optimizer / collective
            dfr = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", add_noise=False,
                                       grad_scale=torch.zeros(1, device="cuda"))
            s = timed(dfr)
            row["dp_deferred_tflops"] = F / s / 1e12
            row["dp_deferred_frac_of_peak"] = row["dp_deferred_tflops"] / peak
            del dfr
        x2, y2 = x.view(-1, P), dy.view(-1, D)
        s = timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32))
        row["nondp_cublas_tflops"] = F / s / 1e12
        row["dp_over_nondp"] = row["dp_tflops"] / row["nondp_cublas_tflops"]
        row["nondp_cublas_frac_of_peak"] = row["nondp_cublas_tflops"] / peak
        if B * D * P * 4 * 2 < 24e9:  # explicit materialises G and G' (fp32)
            e = fdp.PreparedBackward(fdp.WorkflowKind.EXPLICIT_DP, x, dy, cfg, noise_impl="philox")
            s = timed(e, 3)
            row["explicit_tflops"] = F / s / 1e12
            del e
        print(json.dumps(row), flush=True)
        del x, dy, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
