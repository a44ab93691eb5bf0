#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "ghost or two_phase" 2>&1 | tail -3
FDP_NO_COOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/phase3.csv python tools/phase_times.py > /dev/null 2>&1
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/phase3.csv")))
h=None
for r in rows:
    if "Kernel Name" in r: h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        if d.get("Metric Name")=="gpu__time_duration.sum":
            n=d["Kernel Name"]
            if "elementwise" in n or "Fill" in n or "copy" in n or "reduce_norms" in n: continue
            print(d["ID"], n[:50], d["Metric Value"])
PY
