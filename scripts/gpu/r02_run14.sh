timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
SVMB200_PROFILE=1 python - <<'PY' 2>&1 | grep -E "column cache|c5 "
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c5", n=300000)
a = [torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data, ds.y)]
for slots in ("0", "-"):
    if slots == "-": os.environ.pop("SVMB200_CACHE", None)
    else: os.environ["SVMB200_CACHE"] = slots
    m = pkg.train_csr(*a[:3], a[3], ds.d, gamma=1.0 / ds.d)
    print("c5 ", slots, m.info.iterations, m.info.loop_ms, m.info.cache_passes, flush=True)
PY
