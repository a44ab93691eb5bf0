# B = 2 per rank Llama steps after fresh bucket views are written (not reduce-added) + deferred-clip tests
mkdir -p gpurun_out
python -m pytest tests/test_gpu_deferred.py tests/test_gpu_ddp.py tests/test_gpu_shared_x.py tests/test_gpu_models.py -q > gpurun_out/pytest_b2.txt 2>&1
tail -2 gpurun_out/pytest_b2.txt
python tools/train_llama.py --model llama-7b --batch 2 --steps 4 --warmup 2 > gpurun_out/tl7_b2.json 2> gpurun_out/tl7_b2.err
python tools/train_llama.py --model llama-13b --layers 20 --zero1 --batch 2 --steps 4 --warmup 2 > gpurun_out/tl13_b2.json 2> gpurun_out/tl13_b2.err
