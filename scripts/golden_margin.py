"""max |f_gpu - f_oracle| on the golden rows of a config as a function of the GPU's tolerance (the
oracle's golden is at 1e-3): separates the oracle's own distance from the optimum from the GPU's."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1706_05544_b200 as pkg  # noqa: E402
from paper_1706_05544_b200 import synth  # noqa: E402

cfg = os.environ.get("SWEEP_CFG", "c4")
g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", f"full_{cfg}.npz"))
ds = synth.make(cfg)
Xh = synth.make(cfg, n=g["f_heldout"].shape[0], heldout=True).X
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
for tol in [float(t) for t in os.environ.get("TOLS", "1e-3,5e-4,2.5e-4,1e-4").split(",")]:
    m = pkg.train(X, y, gamma=1.0 / ds.d, tolerance=tol,
                  svm_type="eps-regression" if ds.svm_type == 3 else "C-classification")
    ft = m.predict(ds.X[g["train_rows"]], decision=True)[1]
    fh = m.predict(Xh, decision=True)[1]
    d1 = np.abs(ft - g["f_train"]).max()
    d2 = np.abs(fh - g["f_heldout"]).max()
    q = np.quantile(np.abs(np.concatenate([ft - g["f_train"], fh - g["f_heldout"]])), [0.5, 0.99, 0.999])
    print(f"{cfg} gpu tol {tol:g}: iterations {m.info.iterations} train {m.info.train_ms:.0f} ms "
          f"max|df| train {d1:.2e} held {d2:.2e}  quantiles 50/99/99.9% {q[0]:.1e} {q[1]:.1e} {q[2]:.1e} "
          f"dual {m.info.dual_objective:.6f} (oracle {float(np.sum(g['dual'])):.6f})", flush=True)
