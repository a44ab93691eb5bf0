"""Summarise an ncu report (or a launch-list CSV) into profiles/.

    python tools/ncu_summary.py full   gpurun_out/prof.ncu-rep  profiles/ncu_<name>.json
    python tools/ncu_summary.py launch gpurun_out/launches.csv  profiles/launches_<name>.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        k = {"kernel": vals[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
        for m in FULL_METRICS:
            if m in h:
                i = h.index(m)
                k[m] = {"value": vals[i], "unit": units[i]}
        kernels.append(k)
    json.dump({"report": rep, "kernels": kernels}, open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1)[:3000])


def launch(path, out):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hdr], rows[hdr + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = defaultdict(list)
    seq = []
    for r in data:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        per[r[ki]].append(v)
        seq.append({"kernel": r[ki][:80], "ns": v})
    tot = sum(sum(v) for v in per.values())
    summary = [{"kernel": k[:120], "launches": len(v), "total_ns": sum(v), "mean_ns": sum(v) / len(v),
                "share": sum(v) / tot if tot else None} for k, v in sorted(per.items(), key=lambda x: -sum(x[1]))]
    json.dump({"source": path, "summary": summary, "launches": seq}, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    {"full": full, "launch": launch}[sys.argv[1]](sys.argv[2], sys.argv[3])
