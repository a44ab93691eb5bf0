"""Per-layer timing sweep of the fused kernel (CUDA events around back-to-back
prepared calls; no host overhead in the numbers).

    python tools/perf_sweep.py [B] [T]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

SHAPES = {"c_attn": (768, 2304), "attn_proj": (768, 768), "c_fc": (768, 3072), "mlp_proj": (3072, 768)}
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1024


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3  # us


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    out = []
    for name, (P, D) in SHAPES.items():
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        flops = 2 * B * T * P * D
        x2, y2 = x.view(-1, P), dy.view(-1, D)
        us = timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32))
        out.append({"layer": name, "variant": "cublas_nondp", "us": round(us, 2), "tflops": round(flops / us / 1e6, 1)})
        nd = fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)
        us = timed(nd)
        out.append({"layer": name, "variant": "tcgen05_nondp", "us": round(us, 2), "tflops": round(flops / us / 1e6, 1)})
        for bn, cg in (("128", "1"), ("256", "1"), ("128", "2"), ("256", "2")):
            os.environ["FDP_FORCE_BN"] = bn
            os.environ["FDP_FORCE_CG"] = cg
            for noise, sigma in (("none", 0.0), ("philox", 1.0)):
                cfg = fdp.DPConfig(1.0, sigma, "mean", seed=1, layer_id=2)
                try:
                    c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, path="fused",
                                             noise_impl="keyed_f32" if noise == "none" else noise)
                    us = timed(c)
                    out.append({"layer": name, "variant": f"fused_bn{bn}_cg{cg}_{noise}", "us": round(us, 2),
                                "tflops": round(flops / us / 1e6, 1), "groups": c.plan.groups, "grid": c.plan.grid})
                except Exception as e:  # noqa: BLE001
                    out.append({"layer": name, "variant": f"fused_bn{bn}_cg{cg}_{noise}", "error": repr(e)[:200]})
            cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=2)
            try:
                c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, path="two_phase", noise_impl="philox")
                us = timed(c)
                out.append({"layer": name, "variant": f"two_phase_bn{bn}_cg{cg}_philox", "us": round(us, 2),
                            "tflops": round(flops / us / 1e6, 1)})
            except Exception as e:  # noqa: BLE001
                out.append({"layer": name, "variant": f"two_phase_bn{bn}", "error": repr(e)[:200]})
        os.environ.pop("FDP_FORCE_BN", None)
        os.environ.pop("FDP_FORCE_CG", None)
        for r in out[-14:]:
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
