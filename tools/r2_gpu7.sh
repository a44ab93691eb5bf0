#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/debug_gloo.py > gpurun_out/dbg_gloo.txt 2>&1
echo done
