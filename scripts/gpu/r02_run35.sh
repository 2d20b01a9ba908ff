timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x -k "csr or ragged" 2>&1 | tail -2
SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 300 python scripts/pass_probe.py 2>&1 | tail -1
cat > /tmp/c5cert.py <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c5")
t = [torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data, ds.y)]
t0 = time.time()
m = pkg.train_csr(*t, ds.d, gamma=1.0 / ds.d)
print("c5 train", time.time() - t0, "s; iterations", m.info.iterations, "loop_ms", m.info.loop_ms, "cert", m.info.certified)
PY
SVMB200_PROFILE=1 timeout 900 python /tmp/c5cert.py 2>&1 | grep -v "^\[svmb200\] loop" | tail -8
