timeout 900 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -15 > gpurun_out/paths.log
cat gpurun_out/paths.log
timeout 900 python scripts/pass_sweep.py --train - SVMB200_NO_TMA=1 SVMB200_TMA_STAGES=2 SVMB200_TMA_STAGES=3 SVMB200_TMA_STAGES=6 SVMB200_TMA_STAGES=4,SVMB200_NO_L2PERSIST=1 2>&1 | tee gpurun_out/sweep.log
