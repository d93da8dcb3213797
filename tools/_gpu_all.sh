python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_multirank.py tests/test_gpu_volumes.py -q -rf 2>&1 | tail -8
TFB200_BENCH_FUNCTIONAL=1 timeout 900 python bench.py --gpus 2 --steps 4 --warmup 1 --no-extra --no-color --no-cpu-baseline > gpurun_out/bench_gpus2_functional.json 2> gpurun_out/bench_gpus2_functional.err; echo functional_rc=$?
tail -c 600 gpurun_out/bench_gpus2_functional.json
