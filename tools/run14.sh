cd /root/repo/tools
timeout 120 python trace_group.py philox > ../gpurun_out/trace_group14.txt 2>&1
cd /root/repo
FDP_DEBUG=1 timeout 60 python tools/prof_one.py c_fc 2 > gpurun_out/debug14.txt 2>&1
FDP_FORCE_CG=1 FDP_FORCE_BN=256 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dpdw -c 3 --csv python tools/prof_one.py c_fc 3 > gpurun_out/ncu14_cg1.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:dpdw -c 3 --csv python tools/prof_one.py c_fc 3 > gpurun_out/ncu14_cg2.txt 2>&1
echo done
