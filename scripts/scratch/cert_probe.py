"""c4: certification time vs one decision pass over the training rows (same contraction)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
ds = synth.make(cfg)
X = torch.from_numpy(ds.X).cuda(); y = torch.from_numpy(ds.y).cuda()
reg = ds.svm_type == synth.EPS_REGRESSION
kw = dict(svm_type="eps-regression" if reg else "C-classification", gamma=1.0 / ds.d)
m = pkg.train(X, y, **kw)
i = m.info
print(f"{cfg}: iters {i.iterations} nsv {i.n_sv} loop {i.loop_ms:.1f} ms certify {i.certify_ms:.1f} ms train {i.train_ms:.1f} ms")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out, dec = m.predict(X, decision=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"  predict over the {ds.n} training rows: {(t1-t0)*1e3:.1f} ms")
