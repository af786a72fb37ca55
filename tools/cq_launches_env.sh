#!/bin/bash
# CPQR launch list of one C2 build per environment setting (ncu, gpu__time_duration.sum):
#   tools/cq_launches_env.sh TAG 'ENV=..' [TAG 'ENV=..' ...]
while [ $# -gt 1 ]; do
  tag=$1; envs=$2; shift 2
  env $envs timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:cpqr --csv python tools/one_build.py > gpurun_out/cq_launches_$tag.csv 2>&1
done
