"""c3 class-0-vs-rest training with certification (d = 784: the tcgen05 fp16-split decision kernel
runs the certification pass) plus one predict of 20,000 held-out rows: the target of launch lists."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c3")
y = np.where(ds.y == 0, 1.0, -1.0).astype(np.float32)
m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(y).cuda(), gamma=1.0 / ds.d)
i = m.info
hq = synth.make("c3", n=20000, heldout=True)
out = m.predict(torch.from_numpy(hq.X).cuda())
torch.cuda.synchronize()
print(f"c3 class0: iters {i.iterations} loop {i.loop_ms:.2f} ms certify {i.certify_ms:.2f} ms nsv {i.n_sv}")
