"""Full-size oracle goldens for the end-to-end parity tests (SURVEY.md 8(c) "End to end").

Imports ONLY ``oracle/`` and the input generators (``paper_1706_05544_b200.synth``, which holds
no arithmetic of the method).  For each BASELINE config it trains the fp64 oracle (the loop of
P:53 on the Eq. 2 instance) to tol = 1e-3 at the BASELINE size on this host's cores and
writes ``tests/golden/full_<cfg>.npz`` with:

  dual[k], iterations[k], b[k], m_up[k], M_low[k], converged[k]   per problem (k = 1 or 10 OvR)
  sv_index[k] (int32), sv_coef[k] (fp64)                          the oracle model
  train_rows (int64), f_train [rows x k]                           f on a fixed training subset
  f_heldout [rows x k]                                             f on the first rows of seed+100
  wall_s, threads                                                  the oracle's own time to tol

The subsets are drawn with a fixed seed here and stored, so the GPU test reads them back.  No
value comes from the CUDA path.  C5 (2,000,000 x 400) does not finish on the host in a useful
time; ``--dnf c5`` records the measured iterations/s over a bounded number of iterations with
``did_not_finish`` (SURVEY.md 8(d) "Oracle timing": do not extrapolate).

Usage: python scripts/make_goldens.py c2 c3 c4      (each config is independent)
       python scripts/make_goldens.py --dnf c5 --iters 200
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as ora  # noqa: E402
from paper_1706_05544_b200 import synth  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
N_SUB = 10000          # rows of the training subset and of the held-out set
SUB_SEED = 20260419    # seed of the training-subset draw


def golden_path(cfg: str) -> str:
    return os.path.join(GOLDEN, f"full_{cfg}.npz")


def make(cfg: str, tol: float = 1e-3) -> dict:
    ds = synth.make(cfg)
    X, y, n, d = ds.X, ds.y, ds.n, ds.d
    reg = ds.svm_type == synth.EPS_REGRESSION
    t0 = time.perf_counter()
    model = ora.train(X, y, svm_type=ora.EPS_REGRESSION if reg else ora.C_CLASSIFICATION,
                      C=ds.params["C"], gamma=ds.params["gamma"], epsilon=ds.params["epsilon"],
                      tol=tol)
    wall = time.perf_counter() - t0
    rows = np.sort(np.random.default_rng(SUB_SEED).choice(n, min(N_SUB, n), replace=False))
    Xh = synth.make(cfg, n=N_SUB, heldout=True).X
    t1 = time.perf_counter()
    f_train = model.decision_function(X[rows])
    f_held = model.decision_function(Xh)
    t_dec = time.perf_counter() - t1
    out = dict(cfg=cfg, tol=tol, n=n, d=d, threads=ora.num_threads(), wall_s=wall,
               decision_s=t_dec, train_rows=rows.astype(np.int64), f_train=f_train,
               f_heldout=f_held)
    k = len(model.coefs)
    out["classes"] = np.asarray(model.classes if model.classes is not None else [], np.float64)
    for key in ("dual", "iterations", "b", "m_up", "M_low", "converged", "inner_steps"):
        out[key] = np.asarray([r[key] for r in model.results])
    sv_idx, sv_coef, sv_ptr = [], [], [0]
    for c in model.coefs:
        nz = np.nonzero(c)[0]
        sv_idx.append(nz.astype(np.int32))
        sv_coef.append(c[nz])
        sv_ptr.append(sv_ptr[-1] + nz.size)
    out["sv_index"] = np.concatenate(sv_idx)
    out["sv_coef"] = np.concatenate(sv_coef)
    out["sv_ptr"] = np.asarray(sv_ptr, np.int64)
    out["n_problems"] = k
    return out


def dnf(cfg: str, iters: int, tol: float = 1e-3) -> dict:
    """Bounded oracle run for a config whose time to tol is out of reach on the host."""
    ds = synth.make(cfg)
    X = ds.dense()
    n, d = X.shape
    prob = ora.Problem(ora.C_CLASSIFICATION, ds.y, n)
    ks = ora.kspec("rbf", ds.params["gamma"], d=d)
    t0 = time.perf_counter()
    r = ora.train_dual(X, prob, ks, ds.params["C"], tol, 16, max_iter=iters)
    wall = time.perf_counter() - t0
    return dict(cfg=cfg, n=n, d=d, threads=ora.num_threads(), iterations=r["iterations"],
                wall_s=wall, iterations_per_s=r["iterations"] / wall,
                violation=r["m_up"] - r["M_low"], did_not_finish=True, tol=tol)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--dnf", action="store_true")
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    os.makedirs(GOLDEN, exist_ok=True)
    for cfg in a.configs:
        if a.dnf:
            rec = dnf(cfg, a.iters)
            with open(os.path.join(GOLDEN, f"dnf_{cfg}.json"), "w") as f:
                json.dump(rec, f, indent=1)
            print(json.dumps(rec), flush=True)
            continue
        rec = make(cfg)
        np.savez_compressed(golden_path(cfg), **rec)
        summ = {k: (v.tolist() if isinstance(v, np.ndarray) and v.size <= 16 else v)
                for k, v in rec.items() if not (isinstance(v, np.ndarray) and v.size > 16)}
        print(json.dumps(summ, default=float), flush=True)


if __name__ == "__main__":
    main()
