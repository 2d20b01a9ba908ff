timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "csr or virtual" 2>&1 | tail -3
for m in staged sell; do
  if [ $m = staged ]; then export SVMB200_CSR_STAGED=1; else unset SVMB200_CSR_STAGED; fi
  SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 300 python scripts/pass_probe.py 2>&1 | tail -2
  SWEEP_CFG=c5 ITERS=3000 timeout 600 python scripts/train_probe.py 2>&1 | tail -1
done
unset SVMB200_CSR_STAGED
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
