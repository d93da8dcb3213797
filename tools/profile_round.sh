#!/bin/bash
# Round-2 measurement set (current build): bench lines, reference arm, ncu launch list, ncu full capture.
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02d_k20.json 2> gpurun_out/bench_r02d_k20.err; echo bench20_rc=$?
python bench.py --steps 64 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/bench_r02d_k64.json 2> gpurun_out/bench_r02d_k64.err; echo bench64_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02d_reference_arm.json 2> gpurun_out/bench_r02d_reference_arm.err; echo ref_rc=$?
CMD="python bench.py --steps 20 --warmup 5 --no-e2e --no-extra --no-cpu-baseline --no-color"
$CMD > gpurun_out/r02d_plain.json 2> gpurun_out/r02d_plain.err; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -s 1040 -c 450 --csv --log-file gpurun_out/r02d_launches.csv $CMD > gpurun_out/r02d_launches.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"raycast_kernel|brick_update_kernel|brick_apply_kernel|exact_queue_kernel|part_cull_kernel|raycast_coop_items" -s 414 -c 6 -o gpurun_out/r02d_full $CMD > gpurun_out/r02d_full.log 2>&1
echo full_rc=$?
