timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -x -q -k "csr or virtual or cache or kernel_rows" 2>&1 | tail -2
SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 python scripts/pass_probe.py
python - <<'PY' 2>&1 | grep -E "^c5"
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c5", n=300000)
a = [torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data, ds.y)]
m = pkg.train_csr(a[0], a[1], a[2], a[3], ds.d, gamma=1.0 / ds.d)
print("c5 300k", m.info.iterations, round(m.info.loop_ms, 1), round(m.info.loop_ms * 1e3 / m.info.iterations, 1), "us/it", flush=True)
PY
