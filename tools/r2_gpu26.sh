#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export FDP_NO_COOP=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tp_smallT.csv python tools/prof_shape.py 64 128 2048 2048 two_phase 2 > gpurun_out/tp_smallT.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dpdw_stream -s 1 -c 1 -o gpurun_out/stream_smallT -f python tools/prof_shape.py 64 128 2048 2048 two_phase 2 > gpurun_out/stream_smallT.log 2>&1
echo done
