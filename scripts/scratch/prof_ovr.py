"""Batched one-vs-rest training of c3 (10 classes, 60,000 x 784) for a bounded number of
iterations: the target of the k_ovr_pass / k_ovr_solve ncu captures."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c3")
it = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), gamma=1.0 / ds.d,
              certify=0, max_iter=it)
i = m.info
print(f"c3 batched: passes {i.passes} pass {i.pass_ms:.2f} ms ({i.pass_ms * 1e3 / max(1, i.passes):.1f} us/pass), "
      f"loop {i.loop_ms:.2f} ms, batched {i.batched}")
