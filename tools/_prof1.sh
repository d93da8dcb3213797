set -e
CMD="python bench.py --steps 8 --warmup 3 --no-e2e --no-extra --no-cpu-baseline --no-color"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"raycast_kernel|brick_update_kernel|brick_free_kernel|exact_queue_kernel" -s 280 -c 4 -o gpurun_out/prof_r02a $CMD > gpurun_out/ncu_r02a.log 2>&1
echo done
