"""End-to-end parity at BASELINE.json's FULL sizes against the fp64 oracle's own solutions.

The goldens (tests/golden/full_<cfg>.npz) were written by scripts/make_goldens.py, which imports
only oracle/ and the input generators: the oracle trained each config to tol = 1e-3 at the
BASELINE size (P:53 loop, P:59-69 problem) and stored its dual objective(s), iteration counts,
its model (SV indices + coefficients + biases), and its decision values on a fixed 10,000-row
training subset and on the first 10,000 held-out rows (seed + 100).  No value comes from the CUDA
path.  Bars (north_star; SURVEY 8(c) "End to end"):
  * dual objective within 1e-4 relative (summed over the one-vs-rest problems);
  * decision values within 1e-3 absolute on both subsets (every problem) -- except c4, where the
    bar is not met against the oracle's tol-1e-3 solution (reading R20: measured max
    1.35e-3, 99.9th percentile 1.009e-3); there the test asserts max <= 2 tol;
  * label agreement >= 99.9% over both subsets together;
  * the GPU solution's KKT violation, recomputed in fp64 by the oracle from the GPU model's
    support vectors (G = Q alpha + p) over the 10,000-row training subset plus every free
    support vector (0 < alpha < C; those set m_up / M_low), <= tol.
C5 (2,000,000 x 400) has no golden: the oracle does not finish on the host in a useful time
(tests/golden/dnf_c5.json records its measured iterations/s; SURVEY 8(d) "do not extrapolate").
"""
import os

import numpy as np
import pytest

import oracle as ora
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-3
# configs whose decision-value check follows DESIGN.md reading R20 (north_star's 1e-3 measured as
# not attainable against an oracle stopped at the same tolerance); the others assert max <= 1e-3
DF_READING = {"c4"}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pkg.lib()


def _golden(cfg):
    p = os.path.join(GOLD, f"full_{cfg}.npz")
    if not os.path.exists(p):
        pytest.skip(f"no golden for {cfg} (run scripts/make_goldens.py {cfg})")
    return np.load(p)


def _kkt_fp64(X, yv, reg, sv_idx, coef, rows, C, eps=0.1):
    """fp64 violation m_up - M_low over the duals of `rows` from the model's SVs (oracle kernels).
    SVC: G_i = -1 + y_i sum_s coef_s K(x_s, x_i); eps-SVR: G_{i+} = eps - z_i + g_i,
    G_{i-} = eps + z_i - g_i with g_i = sum_s beta_s K(x_s, x_i) (Eq. 1)."""
    ks = ora.kspec("rbf", 1.0 / X.shape[1], d=X.shape[1])
    g = ora.decision(X[sv_idx], coef, 0.0, ks, X[rows])
    c_row = np.zeros(X.shape[0])
    c_row[sv_idx] = coef
    s_up, s_low = [], []

    def add(yy, G, a):
        s = -yy * G
        up = np.where(yy > 0, a < C, a > 0)
        lo = np.where(yy > 0, a > 0, a < C)
        s_up.append(s[up])
        s_low.append(s[lo])

    cr = c_row[rows]
    if reg:
        z = yv[rows].astype(np.float64)
        add(np.ones_like(z), eps - z + g, np.maximum(cr, 0.0))
        add(-np.ones_like(z), eps + z - g, np.maximum(-cr, 0.0))
    else:
        yy = yv[rows].astype(np.float64)
        add(yy, -1.0 + yy * g, np.abs(cr))
    return np.concatenate(s_up).max() - np.concatenate(s_low).min()


def _check(cfg, m, gold, ds, ybins):
    """ybins: +-1 label vector of each problem (None for eps-SVR)."""
    info = m.info
    reg = ds.svm_type == synth.EPS_REGRESSION
    k = int(gold["n_problems"])
    assert info.n_problem == k
    assert info.converged == 1
    # ---- dual objective (sum over problems) ----
    d_ora = float(np.sum(gold["dual"]))
    rel = abs(info.dual_objective - d_ora) / abs(d_ora)
    # ---- decision values and labels on the golden's rows ----
    rows = gold["train_rows"]
    Xh = synth.make(cfg, n=gold["f_heldout"].shape[0], heldout=True).X
    lab_t, f_t = m.predict(ds.X[rows], decision=True)
    lab_h, f_h = m.predict(Xh, decision=True)
    df = max(np.abs(f_t - gold["f_train"]).max(), np.abs(f_h - gold["f_heldout"]).max())

    def ora_labels(f):
        if reg:
            return f[:, 0]
        if k == 1:
            pos, neg, first = gold["classes"]
            return np.where(f[:, 0] > 0, pos, np.where(f[:, 0] < 0, neg, first))
        return gold["classes"][np.argmax(f, axis=1)]

    agree = None
    if not reg:
        agree = np.concatenate([lab_t == ora_labels(gold["f_train"]),
                                lab_h == ora_labels(gold["f_heldout"])]).mean()
    # ---- fp64 KKT of the GPU solution: training subset + free SVs, per problem ----
    idx, coef = m.support()
    viols = []
    for p in range(k):
        cp = coef[p]
        nz = cp != 0
        si, sc = idx[nz], cp[nz]
        free = si[(np.abs(sc) > 1e-12) & (np.abs(sc) < 1.0 - 1e-12)]
        chk = np.unique(np.concatenate([rows, free[:20000]]))
        yv = ds.y if reg else ybins[p]
        viols.append(_kkt_fp64(ds.X, yv, reg, si, sc, chk, 1.0))
    print(f"\n[{cfg}] dual rel {rel:.2e} (oracle {d_ora:.6f}, gpu {info.dual_objective:.6f}); "
          f"max|df| {df:.2e}; labels {agree}; fp64 KKT max {max(viols):.3e}; "
          f"iterations gpu {info.iterations} oracle {int(np.sum(gold['iterations']))}; "
          f"abs df quantiles 99% / 99.9%: {np.quantile(np.abs(np.concatenate([(f_t - gold['f_train']).ravel(), (f_h - gold['f_heldout']).ravel()])), [0.99, 0.999])}")
    assert rel <= 1e-4, rel
    if cfg in DF_READING:
        # DESIGN.md reading R20: at full c4 size two tol-1e-3 solutions differ by more than 1e-3 on
        # a few rows (the oracle's own distance from the optimum: tightening the GPU to 5e-4 /
        # 2.5e-4 moves it further away, 1.5e-3 / 1.7e-3).  north_star's 1e-3 is NOT met here
        # (measured max 1.35e-3, 99.9th percentile 1.009e-3, 99th 7.3e-4); asserted: max <= 2 tol
        assert df <= 2 * TOL, df
    else:
        assert df <= 1e-3, df
    if agree is not None:
        assert agree >= 0.999, agree
    assert max(viols) <= TOL, viols


def _train(ds):
    import torch
    reg = ds.svm_type == synth.EPS_REGRESSION
    return pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(),
                     svm_type="eps-regression" if reg else "C-classification",
                     gamma=1.0 / ds.d, epsilon=0.1, tolerance=TOL)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c4"])
def test_full_size_vs_oracle(cfg):
    gold = _golden(cfg)
    ds = synth.make(cfg)
    m = _train(ds)
    yb = None if ds.svm_type == synth.EPS_REGRESSION else [ora.binary_labels(ds.y)[0]]
    _check(cfg, m, gold, ds, yb)


def test_full_size_c3_one_vs_rest_vs_oracle():
    """10 classes, batched one-vs-rest passes on tcgen05 (the c3 training path)."""
    gold = _golden("c3")
    ds = synth.make("c3")
    m = _train(ds)
    labels = np.array(m.info.labels[:10])
    np.testing.assert_array_equal(labels, gold["classes"])
    ybins = [np.where(ds.y == c, 1.0, -1.0).astype(np.float32) for c in labels]
    _check("c3", m, gold, ds, ybins)
