# ncu evidence for profiles/: launch list of the bench command + one full capture
# of the dominant kernel (grouped persistent kernel) and of one per-layer fused kernel.
# FDP_NO_COOP=1: ncu replay cannot relaunch cooperative cluster kernels; the grid is
# sized to co-residency so a plain launch is equivalent.
cd /root/repo
export FDP_NO_COOP=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpdw_group -s 2 -c 1 \
  -o gpurun_out/prof_group_r1 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-nondp \
  > gpurun_out/prof_group.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dpdw_tc -s 2 -c 1 \
  -o gpurun_out/prof_cfc_r1 -f python tools/prof_one.py c_fc 4 \
  > gpurun_out/prof_cfc.log 2>&1
echo prof-done
