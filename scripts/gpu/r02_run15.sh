./scripts/fma_rate
python - <<'PY' 2>&1 | grep -E "^c"
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c4")
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
for cache in ("0", "4096", "0", "4096"):
    os.environ["SVMB200_CACHE"] = cache
    m = pkg.train(X, y, gamma=1.0/ds.d)
    print("c4", cache, m.info.iterations, round(m.info.loop_ms, 1), round(m.info.train_ms, 1), m.info.cache_passes, flush=True)
ds = synth.make("c5", n=300000)
a = [torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data, ds.y)]
for cache in ("0", "-"):
    if cache == "-": os.environ.pop("SVMB200_CACHE", None)
    else: os.environ["SVMB200_CACHE"] = cache
    m = pkg.train_csr(*a[:3], a[3], ds.d, gamma=1.0 / ds.d)
    print("c5", cache, m.info.iterations, round(m.info.loop_ms, 1), m.info.cache_passes, flush=True)
PY
