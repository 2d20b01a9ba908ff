"""Train the same workload several times and print each run's info (determinism / step spread)."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ds = synth.make(cfg)
reg = ds.svm_type == synth.EPS_REGRESSION
kw = dict(svm_type="eps-regression" if reg else "C-classification", gamma=1.0 / ds.d)
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for r in range(reps):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); m = pkg.train(X, y, **kw); e1.record(); torch.cuda.synchronize()
    i = m.info
    print(f"{cfg} run {r}: {e0.elapsed_time(e1):8.1f} ms  iters {i.iterations}  loop {i.loop_ms:8.1f}  certify {i.certify_ms:7.1f}  "
          f"setup {i.setup_ms:6.1f}  total {i.train_ms:8.1f}  dual {i.dual_objective:.9f}  viol {i.violation:.3e}", flush=True)
