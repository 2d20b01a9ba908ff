TOLS=1e-4 timeout 900 python scripts/golden_margin.py 2>&1 | tail -2
for cfg in c2 c4; do for q in 0 1; do SWEEP_CFG=$cfg SVMB200_QWW_MMA=$q timeout 600 python scripts/pass_sweep.py --train - 2>&1 | tail -1 | sed "s/^/$cfg qww_mma=$q /"; done; done
SVMB200_QWW_MMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -x -q -k "one_step or end_to_end or virtual" 2>&1 | tail -2
