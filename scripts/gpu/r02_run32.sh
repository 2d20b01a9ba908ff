timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "csr" 2>&1 | tail -2
SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 300 python scripts/pass_probe.py 2>&1 | tail -1
SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 300 python scripts/pass_probe.py 2>&1 | tail -1
SVMB200_CACHE=0 SWEEP_CFG=c5 ITERS=3000 timeout 600 python scripts/train_probe.py 2>&1 | tail -1
