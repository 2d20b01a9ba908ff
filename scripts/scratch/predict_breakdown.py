"""Train a workload once, then time svm_predict of the held-out rows (device-resident queries) with
CUDA events; under ncu this gives the per-kernel launch list of one predict call.
python scripts/predict_breakdown.py CFG [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
retrain = len(sys.argv) > 3 and sys.argv[3] == "retrain"   # a new model before every predict (as bench.py)
ds = synth.make(cfg)
q = synth.make(cfg, n=min(ds.n, 100000), heldout=True)
reg = ds.svm_type == synth.EPS_REGRESSION
kw = dict(svm_type="eps-regression" if reg else "C-classification", gamma=1.0 / ds.d)
m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), **kw)
Xq = torch.from_numpy(q.X).cuda()
for r in range(reps):
    if retrain:
        m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); out = m.predict(Xq); e1.record(); torch.cuda.synchronize()
    print(f"{cfg} predict {Xq.shape[0]} rows x {m.info.n_sv} SVs: {e0.elapsed_time(e1)*1e3:8.1f} us "
          f"({Xq.shape[0] / e0.elapsed_time(e1) * 1e3 / 1e6:.2f} M rows/s)", flush=True)
