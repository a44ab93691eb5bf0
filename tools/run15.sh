cd /root/repo/tools
timeout 120 python trace_group.py philox > ../gpurun_out/trace_group15.txt 2>&1
FDP_FORCE_CG=2 timeout 60 python trace_fused.py c_fc 256 none > ../gpurun_out/trace15.txt 2>&1
FDP_FORCE_CG=2 timeout 60 python trace_fused.py c_fc 256 philox >> ../gpurun_out/trace15.txt 2>&1
cd /root/repo
timeout 600 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench15.json 2> gpurun_out/bench15.err
FDP_NO_COOP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dpdw -c 3 --csv python tools/prof_one.py c_fc 3 > gpurun_out/ncu15_cg2_nocoop.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu15.txt 2>&1
echo done
