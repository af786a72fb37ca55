timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise or build_parity" > gpurun_out/r2e_test.txt 2>&1; tail -3 gpurun_out/r2e_test.txt
python tools/ab_phases.py cov3d_256k 3 2 'H2_BSR2=0' 'H2_BSR2=1' 'H2_BSR2=2' 'H2_BSR2=3' > gpurun_out/r2e_ab.txt 2>&1; cat gpurun_out/r2e_ab.txt
