#!/bin/bash
# usage: tools/ktimes.sh OUT.csv cmd...   -> per-kernel durations (ncu launch list), FDP kernels + cuBLAS
out=$1; shift
FDP_NO_COOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out "$@" > /dev/null 2>&1
python - "$out" <<'PY'
import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
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
