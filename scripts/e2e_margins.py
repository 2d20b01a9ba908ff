"""Margins of the end-to-end parity cases (tests/test_gpu_parity.py::test_end_to_end): max |f_gpu -
f_oracle| on training and held-out rows (bound 1e-3) and the relative dual difference (bound 1e-4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as ora
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
for cfg, n in (("c1", None), ("c2", 3000), ("c4", 3000)):
    ds = synth.make(cfg, n=n)
    reg = ds.svm_type == synth.EPS_REGRESSION
    m = pkg.train(ds.X, ds.y, svm_type="eps-regression" if reg else "C-classification", gamma=1.0 / ds.d)
    om = ora.train(ds.X, ds.y, svm_type=ora.EPS_REGRESSION if reg else ora.C_CLASSIFICATION, gamma=1.0 / ds.d)
    dd = abs(m.info.dual_objective - om.results[0]["dual"]) / abs(om.results[0]["dual"])
    Xh = synth.make(cfg, n=min(ds.n, 1000), heldout=True).X
    df = [np.abs(m.predict(Xq, decision=True)[1][:, 0] - om.decision_function(Xq)[:, 0]).max()
          for Xq in (ds.X[:1500], Xh)]
    print(f"{cfg} n={ds.n}: dual rel {dd:.2e}  max|df| train {df[0]:.2e} heldout {df[1]:.2e}  "
          f"iters gpu {m.info.iterations} ora {om.results[0]['iterations']}")
