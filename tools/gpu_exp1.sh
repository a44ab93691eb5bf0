#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -k host_streamed -x -q > gpurun_out/pytest_hs.txt 2>&1; echo "hs rc=$?"
EXP_TAG=base timeout 300 python tools/group_exp.py > gpurun_out/exp_base.jsonl 2>&1
EXP_TAG=nosync FDP_DEBUG_NOSYNC=1 timeout 300 python tools/group_exp.py > gpurun_out/exp_nosync.jsonl 2>&1
timeout 600 python bench.py --steps 50 --no-cpu --no-nondp > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
tail -3 gpurun_out/pytest_hs.txt; cat gpurun_out/exp_base.jsonl gpurun_out/exp_nosync.jsonl; python -c "
import json; d=json.loads(open('gpurun_out/bench_e2e.json').read()); print(d['value'], d['e2e'])"
