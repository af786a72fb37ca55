timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsr_kernel -s 1 -c 2 -o gpurun_out/r2d_bsr_src \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > gpurun_out/r2d_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > /dev/null 2>&1
ls -la gpurun_out | tail -5
