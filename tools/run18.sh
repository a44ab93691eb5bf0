cd /root/repo/tools
timeout 120 python trace_group.py philox > ../gpurun_out/trace_group18.txt 2>&1
FDP_FORCE_CG=2 timeout 60 python trace_fused.py c_fc 256 philox > ../gpurun_out/trace18.txt 2>&1
cd /root/repo
timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench18.json 2> gpurun_out/bench18.err
echo done
