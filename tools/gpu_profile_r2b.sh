#!/bin/bash
# round-2 evidence run #2 (one gpurun call): sanitizers over every kernel family incl. the cluster
# CPQR and the GPU KD ordering, the launch list of one bench build, ncu --set full of the cluster CPQR
set -x
O=gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/r2b_sanitize_$tool.txt 2>&1
  echo "exit $?" >> $O/r2b_sanitize_$tool.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2b_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > $O/r2b_launches_bench.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cpqr_cluster_kernel -c 2 -o $O/r2b_cpqr_cluster \
  python tools/one_build.py > /dev/null 2>&1
ls -la $O
