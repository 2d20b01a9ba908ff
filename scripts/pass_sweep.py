"""Pass-only (a3) and full-loop timing of the c4 workload under launch-variant env knobs.
Usage: python scripts/pass_sweep.py [--train] VAR=VAL,VAR=VAL ...   (one variant per argument;
"-" = defaults).  Prints one line per variant: us per pass, GB/s of algorithmic bytes, and with
--train the full training's loop time and us per iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05544_b200 as pkg  # noqa: E402
from paper_1706_05544_b200 import synth  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
train = "--train" in sys.argv
cfg = os.environ.get("SWEEP_CFG", "c4")
ds = synth.make(cfg)
X = torch.from_numpy(ds.X).cuda()
y = torch.from_numpy(ds.y).cuda()
kw = dict(gamma=1.0 / ds.d, svm_type="eps-regression" if ds.svm_type == 3 else "C-classification")
ncopy = 2 if ds.svm_type == 3 else 1
bpp = ds.n * (4 * ds.d + 4 + 9 * ncopy)
for var in args or ["-"]:
    env = {} if var == "-" else dict(kv.split("=") for kv in var.split(","))
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        s = pkg.Solver(X, y, **kw)
        rows = np.linspace(0, ds.n - 1, 16).astype(np.int64)
        c = np.full(16, 1e-6, np.float32)
        s.pass_bench(rows, c, 4)
        ms = min(s.pass_bench(rows, c, 200) for _ in range(3))
        line = f"{var:50s} pass {ms * 1e3 / 200:7.2f} us  {bpp * 200 / ms / 1e6:7.0f} GB/s"
        if train:
            m = pkg.train(X, y, **kw)
            inf = m.info
            line += (f"  | train loop {inf.loop_ms:8.1f} ms  {inf.iterations} it  "
                     f"{inf.loop_ms * 1e3 / inf.iterations:6.2f} us/it")
        print(line, flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
