timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_update.py -q -x > gpurun_out/r2j_test.txt 2>&1; tail -15 gpurun_out/r2j_test.txt
