"""Per-layer timeline of the multi-layer fused launch (FDP_FLAG_TRACE).

    python tools/trace_group.py [noise] [B] [T]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402
from paper_2507_01154_b200 import _lib  # noqa: E402

GPT2 = [("c_attn", 768, 2304), ("attn_proj", 768, 768), ("c_fc", 768, 3072), ("mlp_proj", 3072, 768)]


def main():
    noise = sys.argv[1] if len(sys.argv) > 1 else "philox"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    sigma = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    g = torch.Generator(device="cuda").manual_seed(0)
    layers = []
    for blk in range(int(os.environ.get("TG_BLOCKS", "2"))):
        for j, (name, P, D) in enumerate(GPT2):
            x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
            dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
            layers.append((x, dy, fdp.DPConfig(1.0, sigma, "mean", seed=1, layer_id=blk * 4 + j)))
    grp = fdp.PreparedGroup(layers, noise_impl=noise)
    for i in range(len(layers)):
        grp.descs[i].flags = _lib.FLAG_TRACE
    nbytes = ctypes.c_size_t()
    _lib.check(_lib.load().fdp_group_workspace_bytes(len(layers), grp.descs, ctypes.byref(nbytes)))
    grp.workspace = torch.zeros(nbytes.value, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        grp()
    torch.cuda.synchronize()
    grid = 148
    raw = grp.workspace[nbytes.value - 2048 * grid:].view(torch.int64).cpu().numpy()
    # the trace region is sized for the launch grid; infer it from the nonzero rows
    tr = raw.reshape(-1, 256)[:grid]
    valid = tr[:, :128]
    big = valid[valid > 10**15]  # globaltimer values (ns since epoch)
    t0 = big.min()
    rel = np.where(valid > 10**15, (valid - t0) / 1e3, np.nan)
    names = ["first_ready", "loop_end", "noise_done", "groups_done", "round0", "stored", "noise_signal"]
    out = []
    for l in range(min(len(layers), 16)):
        cols = rel[:, 8 * l:8 * l + 7]
        if not np.isfinite(cols).any():
            continue
        row = {"layer": l, "name": GPT2[l % 4][0], "ctas": int(np.isfinite(cols[:, 0]).sum())}
        for k, nm in enumerate(names):
            v = cols[:, k]
            row[nm] = round(float(np.nanmedian(v)), 2) if np.isfinite(v).any() else None
            if nm in ("loop_end", "noise_signal", "stored"):
                row[nm + "_max"] = round(float(np.nanmax(v)), 2) if np.isfinite(v).any() else None
        out.append(row)
    mma = raw.reshape(-1, 256)[:grid, 248:252]
    lead = mma[mma[:, 3] > 0]
    mma_stats = {"ctas": int(len(lead)),
                 "wait_tmem_us_med": round(float(np.median(lead[:, 0])) / 1e3, 2),
                 "wait_operands_us_med": round(float(np.median(lead[:, 1])) / 1e3, 2),
                 "issue_span_us_med": round(float(np.median(lead[:, 2])) / 1e3, 2),
                 "units_med": float(np.median(lead[:, 3])),
                 # spread over the MMA-issuing CTAs: imbalance of the packed layer ranges
                 "issue_span_us_min": round(float(np.min(lead[:, 2])) / 1e3, 2),
                 "issue_span_us_max": round(float(np.max(lead[:, 2])) / 1e3, 2),
                 "wait_operands_us_max": round(float(np.max(lead[:, 1])) / 1e3, 2),
                 "units_min": float(np.min(lead[:, 3])), "units_max": float(np.max(lead[:, 3]))} if len(lead) else {}
    print(json.dumps({"noise": noise, "sigma": sigma, "B": B, "T": T, "layers": out, "mma_issuer": mma_stats}))


if __name__ == "__main__":
    main()
