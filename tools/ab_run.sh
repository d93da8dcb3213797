#!/bin/bash
# A/B timing of libtfb200 variants built by tools/ab_build.py (developer tool):
#   bash tools/ab_run.sh ROUNDS SPEC1 SPEC2 ...   (on the GPU box)
# SPEC = NAME[:VAR=VAL[,VAR=VAL...]] -> TFB200_LIB=_ab/NAME.so plus the env.
# Each round runs the quick bench (config 3, K = 64) once per variant.
rounds=$1; shift
mkdir -p gpurun_out
for r in $(seq 1 $rounds); do
  for spec in "$@"; do
    v=${spec%%:*}; envs=""
    [[ "$spec" == *:* ]] && envs=$(echo "${spec#*:}" | tr ',' ' ')
    tag=$(echo "$spec" | tr ':,=' '___')
    e2e=--no-e2e; [ -n "$AB_E2E" ] && e2e=
    env $envs TFB200_LIB=_ab/$v.so python bench.py --steps 64 --warmup 5 $e2e --no-extra \
      --no-cpu-baseline --no-color > gpurun_out/ab_${tag}_${r}.json 2>/dev/null
    python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_${tag}_${r}.json').read().strip().splitlines()[-1])
b=d['breakdown_ms_per_step']
e=d.get('e2e',{}).get('frames_per_s',0.0)
print('%-28s fps %7.1f  e2e %7.1f  step %.4f  upd %.4f  scr %.4f  int %.4f  ray %.4f  coop %.4f' % ('$spec', d['frames_per_s'], e, d['ms_per_step'], b['integrate_update_kernel'], b.get('integrate_screen_overlapped', 0.0), b['integrate_total'], b['raycast'], d['raycast']['coop_pass_ms_per_frame']))
"
  done
done
