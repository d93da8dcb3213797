python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_k20.json 2> gpurun_out/bench_r02_k20.err; echo bench20_rc=$?
python bench.py --steps 64 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/bench_r02_k64.json 2> gpurun_out/bench_r02_k64.err; echo bench64_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02_reference_arm.json 2> gpurun_out/bench_r02_reference_arm.err; echo ref_rc=$?
bash tools/_prof_r02.sh
