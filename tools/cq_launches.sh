#!/bin/bash
# CPQR launch list of one C2 build per H2_CQ_CLUSTER setting (ncu, gpu__time_duration.sum)
for c in "$@"; do
  H2_CQ_CLUSTER=$c timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:cpqr --csv python tools/one_build.py > gpurun_out/cq_launches_$c.csv 2>&1
done
