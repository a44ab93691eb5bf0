cd /root/repo
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu11.txt 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench11.json 2> gpurun_out/bench11.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dpdw|k_|gemm|nvjet|cutlass|ghost" -c 200 --csv \
    --log-file gpurun_out/launches11.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-nondp > /dev/null 2> gpurun_out/ncu_launch11.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dpdw_tc -s 2 -c 1 \
    -o gpurun_out/prof11_fused_cfc -f python tools/prof_one.py c_fc 3 > gpurun_out/ncu_full11.log 2>&1
timeout 900 python tools/layer_sweep.py > gpurun_out/layer_sweep11.jsonl 2>&1
echo done
