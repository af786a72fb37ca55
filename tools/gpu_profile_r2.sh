#!/bin/bash
# round-2 evidence run (one gpurun call): sanitizers, launch list of the bench step, ncu --set full
# of the top kernels.  Outputs under gpurun_out/.
set -x
O=gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/r2_sanitize_$tool.txt 2>&1
  echo "exit $?" >> $O/r2_sanitize_$tool.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > $O/r2_launches_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_tc_kernel -c 1 -o $O/r2_sketch \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsr_kernel -s 2 -c 4 -o $O/r2_bsr \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -c 6 -o $O/r2_cpqr \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > /dev/null 2>&1
ls -la $O
