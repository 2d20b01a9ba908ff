timeout 900 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -5 > gpurun_out/paths.log
cat gpurun_out/paths.log
timeout 900 python scripts/pass_sweep.py --train - SVMB200_RPT=2 SVMB200_TMA=1 2>&1 | tee gpurun_out/sweep.log
