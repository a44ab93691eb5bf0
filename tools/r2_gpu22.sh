#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
AB_ROUNDS=3 timeout 1500 python tools/ab_layer.py "1,2048,13824,5120;1,2048,5120,13824;1,2048,5120,5120;1,2048,4096,4096;2,2048,5120,5120;2,2048,13824,5120" \
  base FDP_STREAM_SWIZZLE=4 FDP_STREAM_SWIZZLE=8 FDP_STREAM_SWIZZLE=16 FDP_STREAM_MC=0 FDP_STREAM_MC=0,FDP_STREAM_SWIZZLE=8 > gpurun_out/ab_swz.jsonl 2> gpurun_out/ab_swz.err
echo done
