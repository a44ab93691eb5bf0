cd /root/repo
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "group" > gpurun_out/pytest_gpu12.txt 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench12.json 2> gpurun_out/bench12.err
timeout 600 python bench.py --steps 100 --warmup 5 --noise keyed_f32 --no-e2e --no-cpu --no-nondp > gpurun_out/bench12_keyed.json 2>> gpurun_out/bench12.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu12_all.txt 2>&1
echo done
