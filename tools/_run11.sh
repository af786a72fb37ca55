timeout 900 ncu --set full --clock-control none --import-source on -k regex:bsr2_kernel -c 3 -o gpurun_out/r2f_bsr2_src \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > gpurun_out/r2f_ncu.log 2>&1
tail -2 gpurun_out/r2f_ncu.log
