"""A bounded c4 training for ncu: one persistent launch of ITERS iterations (no certification),
so that its DRAM bytes per iteration can be measured (profiles/traffic_<cfg>_n1.json)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_05544_b200 as pkg  # noqa: E402
from paper_1706_05544_b200 import synth  # noqa: E402

cfg = os.environ.get("SWEEP_CFG", "c4")
it = int(os.environ.get("ITERS", "3000"))
ds = synth.make(cfg)
kw = dict(gamma=1.0 / ds.d, svm_type="eps-regression" if ds.svm_type == 3 else "C-classification",
          max_iter=it, certify=0)
if ds.is_csr:
    m = pkg.train_csr(*(torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data)),
                      torch.from_numpy(ds.y).cuda(), ds.d, **kw)
else:
    m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), **kw)
print(f"{cfg}: {m.info.iterations} iterations, loop {m.info.loop_ms:.1f} ms, cache passes {m.info.cache_passes}")
