python - <<'PY' 2>&1 | tail -5
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c5", n=300000)
a = [torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data, ds.y)]
for cache in ("0", "auto"):
    if cache == "auto": os.environ.pop("SVMB200_CACHE", None)
    else: os.environ["SVMB200_CACHE"] = cache
    m = pkg.train_csr(a[0], a[1], a[2], a[3], ds.d, gamma=1.0 / ds.d)
    print("c5", cache, m.info.iterations, round(m.info.loop_ms, 1), m.info.cache_passes, flush=True)
PY
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -3
