timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 2 -c 1 -o gpurun_out/r2g_cpqr_src \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-c3 > gpurun_out/r2g_ncu.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
tail -c 600 gpurun_out/r2g_bench.json
