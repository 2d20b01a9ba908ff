timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "cache or virtual" 2>&1 | tail -2
python - <<'PY' 2>&1 | grep -E "^c"
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c4")
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
for cache in ("4096", "0", "4096", "0"):
    os.environ["SVMB200_CACHE"] = cache
    m = pkg.train(X, y, gamma=1.0/ds.d)
    print("c4", cache, m.info.iterations, round(m.info.loop_ms, 1), round(m.info.train_ms, 1), m.info.cache_passes, flush=True)
PY
