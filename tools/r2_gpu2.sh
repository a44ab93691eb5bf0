#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
FDP_DEBUG=1 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/coop_debug.txt 2>&1
FDP_DEBUG=1 python tools/prof_shape.py 8 1024 768 3072 fused 2 >> gpurun_out/coop_debug.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.txt 2>&1
for s in "64 128 1024 1024" "64 128 2048 2048"; do
  tag=$(echo $s | tr ' ' '_')
  FDP_NO_COOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:dpdw -s 2 -c 1 \
    -o gpurun_out/r2_smallT_$tag -f python tools/prof_shape.py $s fused 3 > gpurun_out/ncu_smallT_$tag.log 2>&1
done
echo done
