#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
EXP_TAG=pack timeout 300 python tools/group_exp.py > gpurun_out/exp_pack.jsonl 2>&1
EXP_TAG=nopack FDP_NO_PACK=1 timeout 300 python tools/group_exp.py > gpurun_out/exp_nopack.jsonl 2>&1
timeout 600 python bench.py --steps 100 --no-cpu --no-e2e > gpurun_out/bench2.json 2> gpurun_out/bench2.err
tail -5 gpurun_out/pytest_gpu.txt; grep all48 gpurun_out/exp_pack.jsonl gpurun_out/exp_nopack.jsonl; python -c "
import json; d=json.loads(open('gpurun_out/bench2.json').read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['nondp'])"
