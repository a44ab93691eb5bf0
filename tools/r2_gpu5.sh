#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SIG=0 timeout 300 python tools/debug_dp.py allreduce 0 > gpurun_out/dbg5_nondp.txt 2>&1
FDP_DDP_SYNC=1 SIG=0 timeout 300 python tools/debug_dp.py allreduce 0 > gpurun_out/dbg5_nondp_sync.txt 2>&1
FDP_DDP_SYNC=1 timeout 300 python tools/debug_dp.py allreduce 1 > gpurun_out/dbg5_dp_sync.txt 2>&1
AB_ROUNDS=5 timeout 600 python tools/ab.py base FDP_PF_AHEAD=-1 FDP_PF_AHEAD=1 > gpurun_out/ab_pf.jsonl 2> gpurun_out/ab_pf.err
echo done
