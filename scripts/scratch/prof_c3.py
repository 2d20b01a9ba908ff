import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c3")
cls = np.unique(ds.y)
y = np.where(ds.y == cls[0], 1.0, -1.0).astype(np.float32)
m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(y).cuda(), gamma=1.0/ds.d, certify=0, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
i = m.info
print(f"c3 class0: iters {i.iterations} loop {i.loop_ms:.2f} ms us/iter {i.loop_ms*1e3/max(1,i.iterations):.2f}")
