#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python tools/trace_group.py philox 8 1024 1.0 > gpurun_out/trace_s1.json 2>&1
timeout 120 python tools/trace_group.py philox 8 1024 0.0 > gpurun_out/trace_s0.json 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/trace_s1.json", "gpurun_out/trace_s0.json"):
    d = json.load(open(f))
    print(f)
    for r in d["layers"]:
        print(r)
PY
