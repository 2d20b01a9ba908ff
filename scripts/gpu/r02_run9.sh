python - <<'PY' 2>&1 | grep -E "svmb200\]|iters"
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
for cfg in ("c4", "c2"):
    ds = synth.make(cfg)
    X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
    for slots in (256, 1024, 4096, 16384):
        os.environ["SVMB200_CACHE_STATS"] = str(slots)
        m = pkg.train(X, y, gamma=1.0/ds.d, certify=0, svm_type="eps-regression" if ds.svm_type == 3 else "C-classification")
        print(cfg, slots, "iters", m.info.iterations, flush=True)
PY
