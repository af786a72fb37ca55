for v in 0 1; do
H2_CQ2=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches_cq$v.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > /dev/null 2>&1
done
H2_CQ2=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr2_kernel -s 4 -c 1 -o gpurun_out/r2i_cpqr2_src \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > /dev/null 2>&1
ls gpurun_out | grep r2i
