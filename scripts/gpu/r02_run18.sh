timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "virtual or one_step or cache" 2>&1 | tail -2
SWEEP_CFG=c2 timeout 600 python scripts/pass_sweep.py --train - 2>&1 | tail -2
timeout 600 python scripts/pass_sweep.py --train - 2>&1 | tail -2
