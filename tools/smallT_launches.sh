# Per-kernel durations of the two-phase path at small T (ncu launch list; cold caches, serialised)
mkdir -p gpurun_out
export FDP_NO_COOP=1
for s in "64 128 1024 1024" "64 128 2048 2048" "128 128 1024 1024" "32 256 2048 2048"; do
  tag=$(echo $s | tr ' ' '_')
  ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --csv --log-file gpurun_out/smallT_launch_$tag.csv \
    python tools/prof_shape.py $s two_phase 3 > gpurun_out/smallT_launch_$tag.log 2>&1
  ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/smallT_nondp_$tag.csv \
    python tools/prof_shape.py $s auto 3 non_dp > gpurun_out/smallT_nondp_$tag.log 2>&1
done
