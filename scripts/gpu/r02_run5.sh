timeout 900 python scripts/pass_sweep.py --train - SVMB200_NO_DBUF=1 2>&1 | tee gpurun_out/sweep.log
