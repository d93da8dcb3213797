python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-color > gpurun_out/dbg_mem.json 2> gpurun_out/dbg_mem.err; echo rc=$?
grep "bench:" gpurun_out/dbg_mem.err
python -c "
import json; d=json.loads(open('gpurun_out/dbg_mem.json').read().strip().splitlines()[-1]); print(json.dumps(d.get('config5'))[:1500])"
bash tools/ab_run.sh 2 cur3 eq6 eq8
for k in 20 21 64; do python bench.py --steps $k --warmup 5 --no-e2e --no-extra --no-cpu-baseline --no-color > gpurun_out/k$k.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/k$k.json').read().strip().splitlines()[-1]); print('K=$k', d['frames_per_s'], d['breakdown_ms_per_step'])"; done
