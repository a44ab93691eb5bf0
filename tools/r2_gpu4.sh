#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/debug_nondp.py > gpurun_out/dbg_nondp.txt 2>&1
timeout 300 python tools/debug_dp.py allreduce 1 > gpurun_out/dbg_dp_ar.txt 2>&1
SIG=0 timeout 300 python tools/debug_dp.py allreduce 1 > gpurun_out/dbg_dp_ar_s0.txt 2>&1
timeout 300 python tools/debug_dp.py allreduce 0 > gpurun_out/dbg_nondp_ar.txt 2>&1
echo done
