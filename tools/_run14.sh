timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedule.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > gpurun_out/r2h_test.txt 2>&1; tail -3 gpurun_out/r2h_test.txt
python tools/ab_phases.py cov3d_256k 3 2 'H2_CQ2=0' 'H2_CQ2=1' > gpurun_out/r2h_ab.txt 2>&1; cat gpurun_out/r2h_ab.txt
