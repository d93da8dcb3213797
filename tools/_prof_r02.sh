CMD="python bench.py --steps 20 --warmup 5 --no-e2e --no-extra --no-cpu-baseline --no-color"
$CMD > gpurun_out/r02_plain.json 2> gpurun_out/r02_plain.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -s 990 -c 420 --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_launches.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"raycast_kernel|brick_update_kernel|brick_free_kernel|exact_queue_kernel|part_cull_kernel|raycast_coop_items" -s 414 -c 6 -o gpurun_out/r02_full $CMD > gpurun_out/r02_full.log 2>&1
echo full_rc=$?
