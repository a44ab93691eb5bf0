cd /root/repo/tools
timeout 120 python trace_group.py philox > ../gpurun_out/trace_group13.txt 2>&1
timeout 120 python trace_group.py keyed_f32 >> ../gpurun_out/trace_group13.txt 2>&1
echo done
