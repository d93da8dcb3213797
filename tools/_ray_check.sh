set -x
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -x -q 2>&1 | tail -4
python bench.py --steps 64 --warmup 5 --no-extra --no-cpu-baseline --no-color > gpurun_out/bench_ray1.json 2> gpurun_out/bench_ray1.err; echo rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_ray1.json').read().strip().splitlines()[-1])
print(d['frames_per_s'], d['breakdown_ms_per_step'], d['roofline']['frac'], d['e2e']['frames_per_s'])
PY
