timeout 900 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -6
SVMB200_PROFILE=1 timeout 900 python scripts/pass_sweep.py --train - SVMB200_CACHE=0 SVMB200_CACHE=16384 2>&1 | grep -v "^\[svmb200\] pass-only" | tee gpurun_out/sweep.log
