cd tools
for cg in 2 1; do for bn in 128 256; do
  FDP_FORCE_CG=$cg FDP_FORCE_BN=$bn timeout 120 python gpu_diag.py fused_small fused_c1 fused_ragged two_phase explicit fused_gpt2_fc fused_gpt2_attnproj > ../gpurun_out/diag_cg${cg}_bn${bn}.txt 2>&1
done; done
timeout 400 python perf_sweep.py > ../gpurun_out/sweep2.txt 2>&1
timeout 300 python mainloop.py > ../gpurun_out/mainloop2.txt 2>&1
cd ..
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.txt 2>&1
echo done
