# Deferred clip evidence (round 2): GPU tests of the path, Llama block dW with it, training steps.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_deferred.py -q > gpurun_out/pytest_def.txt 2>&1
tail -3 gpurun_out/pytest_def.txt
python tools/llama_block.py --batches 1 > gpurun_out/llama_blocks_def.jsonl 2> gpurun_out/llama_blocks_def.err
