timeout 900 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -4
timeout 900 python scripts/pass_sweep.py --train - SVMB200_CHUNK_ROWS=-1 SVMB200_CHUNK_ROWS=104 2>&1 | tee gpurun_out/sweep.log
SWEEP_CFG=c2 timeout 900 python scripts/pass_sweep.py --train - SVMB200_CHUNK_ROWS=-1 2>&1 | tee -a gpurun_out/sweep.log
