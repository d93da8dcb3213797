python -m pytest tests/test_gpu_volumes.py -q -x 2>&1 | tail -2
( time python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full_v3.json 2> gpurun_out/bench_full_v3.err ) 2> gpurun_out/bench_full_v3.time; echo bench_rc=$?
( time python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_v3.json 2> gpurun_out/bench_ref_v3.err ) 2> gpurun_out/bench_ref_v3.time; echo ref_rc=$?
cat gpurun_out/bench_full_v3.time gpurun_out/bench_ref_v3.time
