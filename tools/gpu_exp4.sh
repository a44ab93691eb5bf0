#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 0 1 2; do
EXP_TAG=dbg$v FDP_DEBUG_NOISE=$v timeout 300 python tools/group_exp.py > gpurun_out/exp_dbg$v.jsonl 2>&1
done
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 50 > gpurun_out/smi_trace.csv &
SMI=$!
timeout 300 python tools/group_exp.py > gpurun_out/exp_smi.jsonl 2>&1
kill $SMI
grep all48 gpurun_out/exp_dbg*.jsonl gpurun_out/exp_smi.jsonl
