"""One pass-only launch of the c4 a3 pass (for ncu): solver build, a 4-pass warm launch, then one
launch of PASSES passes (env, default 20)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05544_b200 as pkg  # noqa: E402
from paper_1706_05544_b200 import synth  # noqa: E402

ds = synth.make(os.environ.get("SWEEP_CFG", "c4"))
s = pkg.Solver(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), gamma=1.0 / ds.d,
               svm_type="eps-regression" if ds.svm_type == 3 else "C-classification")
rows = np.linspace(0, ds.n - 1, 16).astype(np.int64)
c = np.full(16, 1e-6, np.float32)
s.pass_bench(rows, c, 4)
p = int(os.environ.get("PASSES", "20"))
ms = s.pass_bench(rows, c, p)
print(f"{p} passes: {ms:.3f} ms, {ms * 1e3 / p:.2f} us per pass")
