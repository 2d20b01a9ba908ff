export ITERS=30000
for rep in 1 2; do
SVMB200_LIB=libsvmb200_head.so timeout 300 python scripts/train_probe.py 2>&1 | tail -1 | sed 's/^/head   /'
SVMB200_KWW_SPLIT=0 timeout 300 python scripts/train_probe.py 2>&1 | tail -1 | sed 's/^/split0 /'
SVMB200_KWW_SPLIT=1 timeout 300 python scripts/train_probe.py 2>&1 | tail -1 | sed 's/^/split1 /'
done
SWEEP_CFG=c2 ITERS=100000 SVMB200_LIB=libsvmb200_head.so timeout 300 python scripts/train_probe.py 2>&1 | tail -1 | sed 's/^/head   /'
SWEEP_CFG=c2 ITERS=100000 timeout 300 python scripts/train_probe.py 2>&1 | tail -1 | sed 's/^/cur    /'
SWEEP_CFG=c5 ITERS=2000 SVMB200_CACHE=0 SVMB200_KWW_SPLIT=0 timeout 300 python scripts/train_probe.py 2>&1 | tail -1 | sed 's/^/split0 /'
SWEEP_CFG=c5 ITERS=2000 SVMB200_CACHE=0 SVMB200_KWW_SPLIT=1 timeout 300 python scripts/train_probe.py 2>&1 | tail -1 | sed 's/^/split1 /'
timeout 900 python -m pytest tests/test_gpu_paths.py -q -x 2>&1 | tail -2
