"""One pass-only launch of the a3 pass (for ncu): solver build, a 4-pass warm launch, then one
launch of PASSES passes (env, default 20).  SWEEP_CFG selects the config (c5: CSR, PROBE_N rows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05544_b200 as pkg  # noqa: E402
from paper_1706_05544_b200 import synth  # noqa: E402

cfg = os.environ.get("SWEEP_CFG", "c4")
n = int(os.environ["PROBE_N"]) if os.environ.get("PROBE_N") else None
ds = synth.make(cfg, n=n)
kw = dict(gamma=1.0 / ds.d, svm_type="eps-regression" if ds.svm_type == 3 else "C-classification")
if ds.is_csr:
    s = pkg.Solver(csr=tuple(torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data)),
                   y=torch.from_numpy(ds.y).cuda(), d=ds.d, **kw)
else:
    s = pkg.Solver(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), **kw)
rows = np.linspace(0, ds.n - 1, 16).astype(np.int64)
c = np.full(16, 1e-6, np.float32)
s.pass_bench(rows, c, 4)
p = int(os.environ.get("PASSES", "20"))
ms = s.pass_bench(rows, c, p)
print(f"{cfg} n={ds.n}: {p} passes: {ms:.3f} ms, {ms * 1e3 / p:.2f} us per pass")
