python tools/ab_phases.py cov3d_256k 3 2 'H2_CQ_ONEBAR=0' 'H2_CQ_ONEBAR=1' 'H2_CQ_ONEBAR=2' 'H2_CQ_REG=1' 'H2_BSR_VAR=1' 'H2_BSR_VAR=4' > gpurun_out/r2_ab_cq.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
cat gpurun_out/r2_ab_cq.txt
