"""Phase trace of the fused kernel (FDP_FLAG_TRACE): where does each CTA spend time?

    python tools/trace_fused.py [layer|PxD] [bn] [noise] [B] [T]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_01154_b200 import _lib  # noqa: E402

SHAPES = {"c_attn": (768, 2304), "attn_proj": (768, 768), "c_fc": (768, 3072), "mlp_proj": (3072, 768)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c_fc"
    bn = sys.argv[2] if len(sys.argv) > 2 else "128"
    noise = sys.argv[3] if len(sys.argv) > 3 else "none"
    B = int(sys.argv[4]) if len(sys.argv) > 4 else 8
    T = int(sys.argv[5]) if len(sys.argv) > 5 else 1024
    os.environ["FDP_FORCE_BN"] = bn
    P, D = SHAPES[name] if name in SHAPES else (int(v) for v in name.split("x"))  # "PxD" for any shape
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    desc = _lib.make_desc(B=B, T=T, P=P, D=D, reduction="mean", clip_c=1.0, sigma=0.0 if noise == "none" else 1.0,
                          noise_impl="keyed_f32" if noise == "none" else noise, path="fused", flags=4)
    lib = _lib.load()
    info = _lib.plan(desc, "flashdp")
    ws = torch.zeros(info.workspace_bytes, dtype=torch.uint8, device="cuda")
    grad = torch.empty(D, P, device="cuda")
    norms = torch.empty(B, device="cuda")
    for _ in range(3):
        _lib.check(lib.fdp_backward(3, ctypes.byref(desc), x.data_ptr(), dy.data_ptr(), grad.data_ptr(),
                                    norms.data_ptr(), ws.data_ptr(), ws.numel(), None))
    torch.cuda.synchronize()
    tr = ws[info.workspace_bytes - 1024 * info.grid:].view(torch.int64).view(info.grid, 128).cpu().numpy()
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = np.where(tr > 0, (tr - t0) / 1e3, np.nan)  # us
    n_units = (B + info.groups - 1) // info.groups
    out = {"layer": name, "bn": bn, "noise": noise, "groups": info.groups, "grid": info.grid,
           "start_us": [float(np.nanmin(rel[:, 0])), float(np.nanmax(rel[:, 0]))],
           "loop_end_us_med_max": [float(np.nanmedian(rel[:, 1])), float(np.nanmax(rel[:, 1]))],
           "final_end_us_med_max": [float(np.nanmedian(rel[:, 2])), float(np.nanmax(rel[:, 2]))]}
    units = []
    out["first_ready_med"] = round(float(np.nanmedian(rel[:, 9])), 2)

    def med(col):
        v = rel[:, col]
        return round(float(np.nanmedian(v)), 2) if np.isfinite(v).any() else None

    for u in range(n_units):
        # slots: 9+4u sample u ready (MMA done), 8+4u published + noise chunk u done, 10+4u factor u known
        units.append({"u": u, "ready": med(9 + 4 * u), "pass1": med(64 + 4 * u), "block_red": med(65 + 4 * u),
                      "published": med(8 + 4 * u), "factor": med(10 + 4 * u), "pass2": med(66 + 4 * u), "poll_exit": med(67 + 4 * u),
                      "factor_max": round(float(np.nanmax(rel[:, 10 + 4 * u])), 2),
                      "ready_max": round(float(np.nanmax(rel[:, 9 + 4 * u])), 2),
                      "published_max": round(float(np.nanmax(rel[:, 8 + 4 * u])), 2),
                      "ready_min": round(float(np.nanmin(rel[:, 9 + 4 * u])), 2),
                      "published_min": round(float(np.nanmin(rel[:, 8 + 4 * u])), 2),
                      "published_p90": round(float(np.nanpercentile(rel[:, 8 + 4 * u], 90)), 2),
                      "late_ctas": [int(i) for i in np.argsort(np.nan_to_num(rel[:, 8 + 4 * u], nan=-1))[-4:]]})
    out["units"] = units
    print(json.dumps(out))


if __name__ == "__main__":
    main()
