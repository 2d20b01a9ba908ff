"""One bounded training run for ncu profiling: python scripts/prof_train.py CFG[:n] [max_iter]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2:10000"
name, _, n = cfg.partition(":")
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ds = synth.make(name, n=int(n) if n else None)
reg = ds.svm_type == synth.EPS_REGRESSION
kw = dict(svm_type="eps-regression" if reg else "C-classification", gamma=1.0 / ds.d, max_iter=mi,
          certify=0)
if ds.is_csr:
    m = pkg.train_csr(torch.from_numpy(ds.indptr).cuda(), torch.from_numpy(ds.indices).cuda(),
                      torch.from_numpy(ds.data).cuda(), torch.from_numpy(ds.y).cuda(), ds.d, **kw)
else:
    m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), **kw)
i = m.info
print(f"{cfg}: iters {i.iterations} loop {i.loop_ms:.2f} ms us/iter {i.loop_ms*1e3/max(1,i.iterations):.2f}")
