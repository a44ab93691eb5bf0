"""DRAM bytes moved per workflow (north_star: report the fused path's memory
movement against the naive explicit per-sample-gradient (Opacus-style) kernel).

Run under ncu so every kernel's dram__bytes_{read,write}.sum is recorded, and the
L2 write / reduction sectors: ncu flushes the caches before each kernel (cold
reads), but lines a kernel writes can stay dirty in the 126 MB L2 past its end,
so dram__bytes_write under-counts what a kernel produces; the L2-side write and
reduction sectors (x 32 B) count every byte it writes:

    FDP_NO_COOP=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,\
lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum \
        --csv --log-file gpurun_out/bytes.csv python tools/bytes_moved.py

(FDP_NO_COOP=1: ncu's kernel replay cannot re-launch cooperative cluster grids; the
grids are co-resident either way.)
    python tools/bytes_moved.py --summarize gpurun_out/bytes.csv > profiles/r1_bytes_moved.json

Each workflow runs once on the same inputs, separated by marker kernels
(torch.cuda._sleep's spin kernel) so the CSV can be split per workflow.
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = [(8, 1024, 768, 3072), (4, 2048, 4096, 4096)]
KINDS = ["non_dp", "flashdp", "implicit_dp", "explicit_dp"]


def run():
    import torch

    import paper_2507_01154_b200 as fdp

    g = torch.Generator(device="cuda").manual_seed(0)
    for B, T, P, D in SHAPES:
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
        calls = {k: fdp.PreparedBackward(fdp.WorkflowKind(k), x, dy, None if k == "non_dp" else cfg,
                                         noise_impl="philox") for k in KINDS}
        for c in calls.values():  # warm-up (plans, workspaces) before any marker
            c()
        torch.cuda.synchronize()
        for k in KINDS:
            torch.cuda._sleep(100)  # split point (spin kernel): the kernels after it belong to this call
            calls[k]()
        torch.cuda._sleep(100)
        torch.cuda.synchronize()
        del x, dy, calls
        torch.cuda.empty_cache()


def summarize(path):
    rows = list(csv.reader(open(path)))
    h = None
    kern = []  # (id, name, metric, value)
    for r in rows:
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            kern.append((int(d["ID"]), d["Kernel Name"], d["Grid Size"], d["Metric Name"], d["Metric Unit"],
                         d["Metric Value"]))
    by_id = {}
    for i, name, grid, m, unit, v in kern:
        e = by_id.setdefault(i, {"name": name, "grid": grid})
        val = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(unit, 1.0)
        e[m] = val * scale
    ids = sorted(by_id)
    order = [(sh, k) for sh in SHAPES for k in KINDS + ["end"]]
    oi, cur, out = -1, None, []
    for i in ids:
        e = by_id[i]
        if "spin" in e["name"]:  # torch.cuda._sleep marker
            if cur is not None and cur["kind"] != "end":
                out.append(cur)
            oi += 1
            cur = {"shape": order[oi][0], "kind": order[oi][1], "kernels": 0, "dram_read": 0.0, "dram_write": 0.0,
                   "time_s": 0.0} if oi < len(order) else None
            continue
        if cur is None or "elementwise" in e["name"]:
            continue
        cur["kernels"] += 1
        cur["dram_read"] += e.get("dram__bytes_read.sum", 0.0)
        cur["dram_write"] += e.get("dram__bytes_write.sum", 0.0)
        cur["l2_write"] = cur.get("l2_write", 0.0) + 32.0 * (e.get("lts__t_sectors_op_write.sum", 0.0)
                                                             + e.get("lts__t_sectors_op_red.sum", 0.0)
                                                             + e.get("lts__t_sectors_op_atom.sum", 0.0))
        cur["time_s"] += e.get("gpu__time_duration.sum", 0.0)
    res = []
    for r in out:
        B, T, P, D = r["shape"]
        alg = 2 * B * T * (P + D) + 4 * D * P
        l2w = r.get("l2_write", 0.0)
        res.append({"B": B, "T": T, "P": P, "D": D, "kind": r["kind"], "kernels": r["kernels"],
                    "dram_bytes": r["dram_read"] + r["dram_write"], "dram_read": r["dram_read"],
                    "dram_write": r["dram_write"], "l2_write_bytes": l2w,
                    # every byte read from DRAM (cold) + every byte written (each eventually reaches DRAM)
                    "bytes_moved": r["dram_read"] + max(l2w, r["dram_write"]),
                    "algorithmic_bytes": alg, "ncu_time_us": r["time_s"] * 1e6})
    for sh in SHAPES:
        rows = {r["kind"]: r for r in res if (r["B"], r["T"], r["P"], r["D"]) == sh}
        for base in ("explicit_dp", "implicit_dp", "non_dp"):
            if base in rows and "flashdp" in rows:
                rows["flashdp"][f"bytes_moved_vs_{base}"] = rows["flashdp"]["bytes_moved"] / rows[base]["bytes_moved"]
                rows["flashdp"][f"dram_bytes_vs_{base}"] = rows["flashdp"]["dram_bytes"] / rows[base]["dram_bytes"]
    print(json.dumps({"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                                "lts__t_sectors_op_{write,red,atom}.sum (cold caches: ncu flushes before each "
                                "kernel; serialised); one call per workflow on the same inputs. bytes_moved = DRAM "
                                "reads + max(L2 write/reduce bytes, DRAM writes)",
                      "rows": res}, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        run()
