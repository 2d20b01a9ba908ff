"""Train a workload (no certification), then time predict of 50,000 held-out rows (CUDA events);
also the ncu target for the decision kernels: python scripts/predict_probe.py CFG [n]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
ds = synth.make(cfg, n=int(sys.argv[2]) if len(sys.argv) > 2 else None)
reg = ds.svm_type == synth.EPS_REGRESSION
m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(),
              svm_type="eps-regression" if reg else "C-classification", gamma=1.0 / ds.d, certify=0)
Xq = torch.from_numpy(synth.make(cfg, n=50000, heldout=True).X).cuda()
ts = []
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); m.predict(Xq); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{cfg}: nsv {m.info.n_sv} predict 50,000 rows: {min(ts[1:]):.2f} ms -> {50000 / min(ts[1:]) / 1e3:.2f} M rows/s")
