"""Quick GPU probe: train configs through the C ABI and print timings (not a bench line)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth

cfgs = sys.argv[1:] or ["c1", "c2"]
for cfg in cfgs:
    name, _, n = cfg.partition(":")
    ds = synth.make(name, n=int(n) if n else None)
    reg = ds.svm_type == synth.EPS_REGRESSION
    X = torch.from_numpy(ds.X).cuda(); y = torch.from_numpy(ds.y).cuda()
    for rep in range(2):
        torch.cuda.synchronize(); t = time.time()
        m = pkg.train(X, y, svm_type="eps-regression" if reg else "C-classification",
                      gamma=1.0 / ds.d, certify=int(os.environ.get("CERT", "-1")))
        torch.cuda.synchronize(); dt = time.time() - t
        i = m.info
        print(f"{cfg} rep{rep}: {dt*1e3:.1f} ms wall, loop {i.loop_ms:.1f} ms, cert {i.certify_ms:.1f} ms, "
              f"setup {i.setup_ms:.1f}, iters {i.iterations}, us/iter {i.loop_ms*1e3/max(i.iterations,1):.2f}, "
              f"nsv {i.n_sv}, conv {i.converged}, cert {i.certified}, viol {i.violation:.3e}, dual {i.dual_objective:.6f}",
              flush=True)
    Xh = torch.from_numpy(synth.make(name, n=min(ds.n, 100000), heldout=True).X).cuda()
    torch.cuda.synchronize(); t = time.time()
    out = m.predict(Xh)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"{cfg} predict {Xh.shape[0]} rows: {dt*1e3:.1f} ms -> {Xh.shape[0]/dt:.0f} rows/s", flush=True)
