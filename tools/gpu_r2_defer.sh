# Deferred clip evidence (round 2): GPU tests of the path, Llama training steps with it on / off.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_deferred.py tests/test_gpu_ddp.py -q > gpurun_out/pytest_def.txt 2>&1
tail -3 gpurun_out/pytest_def.txt
for B in 1 2; do
python tools/train_llama.py --model llama-7b --batch $B --steps 4 --warmup 2 --defer-clip on > gpurun_out/tl7_on_b$B.json 2> gpurun_out/tl7_on_b$B.err
done
python tools/train_llama.py --model llama-7b --steps 4 --warmup 2 --defer-clip off > gpurun_out/tl7_off.json 2> gpurun_out/tl7_off.err
python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 --defer-clip on > gpurun_out/tl13_on.json 2> gpurun_out/tl13_on.err
python tools/train_llama.py --model llama-13b --layers 20 --zero1 --steps 4 --warmup 2 --defer-clip off > gpurun_out/tl13_off.json 2> gpurun_out/tl13_off.err
