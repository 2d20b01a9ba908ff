export SVMB200_LIB=libsvmb200_prof.so SVMB200_PROFILE=1
python - <<'PY' 2>&1 | grep -E "svmb200\] [0-9]+ iters|worker|column|c4|c2"
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
for cfg in ("c4", "c2"):
    ds = synth.make(cfg)
    X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
    for cache in ("0", "4096"):
        os.environ["SVMB200_CACHE"] = cache
        m = pkg.train(X, y, gamma=1.0/ds.d, certify=0, svm_type="eps-regression" if ds.svm_type == 3 else "C-classification")
        print(cfg, cache, m.info.iterations, m.info.loop_ms, flush=True)
PY
