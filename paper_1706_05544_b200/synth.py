"""Seeded synthetic inputs shaped like the paper's workloads (SURVEY.md section 8(d) recipes).

This module holds NO arithmetic of the method: it only draws data.  It is the one module the
CUDA path's harness and the fp64 oracle's tests both import.  Every array is generated in fp64
with ``numpy.random.default_rng(seed)`` (PCG64) and cast ONCE to fp32; those fp32 arrays are the
inputs of both sides.  Held-out predict sets use ``seed + 100``.

Configs (BASELINE.json ``configs``; gamma = 1/d, C = 1, tol = 1e-3, |W| = 16 throughout):
  c1  binary C-SVC, two Gaussian blobs, n=2,000 d=20             (seed 1)
  c2  eps-SVR (eps=0.1), Friedman #1 in 100-d, n=50,000 d=100    (seed 2; Fig. 1 SVR analogue)
  c3  10-class one-vs-rest C-SVC, MNIST-shaped, n=60,000 d=784   (seed 3; Fig. 1 SVC analogue)
  c4  binary C-SVC, covertype-shaped, n=500,000 d=54             (seed 4)
  c5  binary C-SVC, genomics-shaped CSR ~10% density, n=2,000,000 d=400 (seed 5)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

C_CLASSIFICATION, EPS_REGRESSION = 0, 3


@dataclass
class Dataset:
    name: str
    svm_type: int
    X: np.ndarray | None            # dense row-major fp32 (n, d), or None for CSR
    y: np.ndarray                   # fp32 labels / targets
    d: int
    indptr: np.ndarray | None = None  # CSR (int64), indices (int32, sorted per row), data (fp32)
    indices: np.ndarray | None = None
    data: np.ndarray | None = None
    params: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.y.shape[0])

    @property
    def is_csr(self) -> bool:
        return self.X is None

    def dense(self) -> np.ndarray:
        if self.X is not None:
            return self.X
        out = np.zeros((self.n, self.d), np.float32)
        rows = np.repeat(np.arange(self.n), np.diff(self.indptr))
        out[rows, self.indices] = self.data
        return out


def blobs(n=2000, d=20, seed=1) -> Dataset:
    """c1: y = +1 for even i, -1 for odd i; x = y (1/sqrt d) 1 + N(0, I): centres 2 apart."""
    rng = np.random.default_rng(seed)
    y = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    X = y[:, None] * (1.0 / np.sqrt(d)) + rng.standard_normal((n, d))
    return Dataset("c1", C_CLASSIFICATION, X.astype(np.float32), y.astype(np.float32), d,
                   params=dict(C=1.0, gamma=1.0 / d, epsilon=0.1))


def friedman(n=50000, d=100, seed=2) -> Dataset:
    """c2: U ~ U[0,1]^d; z = 10 sin(pi u1 u2) + 20 (u3 - 1/2)^2 + 10 u4 + 5 u5 + N(0,1);
    X = (U - 1/2) sqrt(12); z standardised."""
    rng = np.random.default_rng(seed)
    U = rng.random((n, d))
    z = (10 * np.sin(np.pi * U[:, 0] * U[:, 1]) + 20 * (U[:, 2] - 0.5) ** 2 + 10 * U[:, 3]
         + 5 * U[:, 4] + rng.standard_normal(n))
    z = (z - z.mean()) / z.std()
    X = (U - 0.5) * np.sqrt(12.0)
    return Dataset("c2", EPS_REGRESSION, X.astype(np.float32), z.astype(np.float32), d,
                   params=dict(C=1.0, gamma=1.0 / d, epsilon=0.1))


def mnist_like(n=60000, d=784, seed=3, k=10) -> Dataset:
    """c3: label c_i = i mod 10; latent h = mu_c + N(0, I16), mu_c ~ 0.9 N(0, I16);
    x = logistic(A h) + 0.05 N(0, I_784), A ~ N(0, 1/16); columns standardised."""
    rng = np.random.default_rng(seed)
    lab = np.arange(n) % k
    mu = 0.9 * rng.standard_normal((k, 16))
    A = rng.standard_normal((d, 16)) / 4.0
    X = np.empty((n, d), np.float32)
    chunk = 8192
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        h = mu[lab[s:e]] + rng.standard_normal((e - s, 16))
        X[s:e] = 1.0 / (1.0 + np.exp(-(h @ A.T))) + 0.05 * rng.standard_normal((e - s, d))
    X64 = X.astype(np.float64)
    X = ((X64 - X64.mean(0)) / X64.std(0)).astype(np.float32)
    return Dataset("c3", C_CLASSIFICATION, X, lab.astype(np.float32), d,
                   params=dict(C=1.0, gamma=1.0 / d, epsilon=0.1))


def covertype_like(n=500000, d=54, seed=4) -> Dataset:
    """c4: 10 N(0,1) + one-hot(U{0..3}) + one-hot(U{0..39});
    y = sign(sin(1.5 x1) + 0.7 x2 x3 + 0.5 [soil < 20] - 0.25 + 0.3 N(0,1))."""
    assert d == 54
    rng = np.random.default_rng(seed)
    cont = rng.standard_normal((n, 10))
    area = rng.integers(0, 4, n)
    soil = rng.integers(0, 40, n)
    X = np.zeros((n, d))
    X[:, :10] = cont
    X[np.arange(n), 10 + area] = 1.0
    X[np.arange(n), 14 + soil] = 1.0
    score = (np.sin(1.5 * cont[:, 0]) + 0.7 * cont[:, 1] * cont[:, 2] + 0.5 * (soil < 20) - 0.25
             + 0.3 * rng.standard_normal(n))
    y = np.where(score > 0, 1.0, -1.0)
    return Dataset("c4", C_CLASSIFICATION, X.astype(np.float32), y.astype(np.float32), d,
                   params=dict(C=1.0, gamma=1.0 / d, epsilon=0.1))


def sparse_genomics(n=2000000, d=400, seed=5, density=0.1, chunk=20000) -> Dataset:
    """c5: mask ~ Bernoulli(0.1); v = 1 + Exp(mean 2); informative set S of 40 features with
    w_S ~ N(0,1); score = x.w/sqrt(40) + 0.5 tanh(x_S0 - 2) x_S1 + 0.5 N(0,1);
    y = +1 iff score > median.  CSR with sorted int32 columns."""
    rng = np.random.default_rng(seed)
    S = rng.choice(d, 40, replace=False)
    w = np.zeros(d)
    w[S] = rng.standard_normal(40)
    indptr = np.zeros(n + 1, np.int64)
    idx_parts, val_parts = [], []
    score = np.empty(n)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        mask = rng.random((e - s, d)) < density
        vals = 1.0 + rng.exponential(2.0, (e - s, d))
        Xc = np.where(mask, vals, 0.0)
        score[s:e] = (Xc @ w / np.sqrt(40.0) + 0.5 * np.tanh(Xc[:, S[0]] - 2.0) * Xc[:, S[1]]
                      + 0.5 * rng.standard_normal(e - s))
        r, c = np.nonzero(mask)
        idx_parts.append(c.astype(np.int32))
        val_parts.append(Xc[r, c].astype(np.float32))
        indptr[s + 1:e + 1] = indptr[s] + np.cumsum(mask.sum(1))
    y = np.where(score > np.median(score), 1.0, -1.0).astype(np.float32)
    return Dataset("c5", C_CLASSIFICATION, None, y, d, indptr=indptr,
                   indices=np.concatenate(idx_parts), data=np.concatenate(val_parts),
                   params=dict(C=1.0, gamma=1.0 / d, epsilon=0.1))


CONFIGS = {
    "c1": (blobs, dict(n=2000, d=20, seed=1)),
    "c2": (friedman, dict(n=50000, d=100, seed=2)),
    "c3": (mnist_like, dict(n=60000, d=784, seed=3)),
    "c4": (covertype_like, dict(n=500000, d=54, seed=4)),
    "c5": (sparse_genomics, dict(n=2000000, d=400, seed=5)),
}


def make(name: str, n: int | None = None, heldout: bool = False, **kw) -> Dataset:
    """Build config ``name`` (optionally at a reduced ``n``); ``heldout`` uses seed + 100."""
    fn, args = CONFIGS[name]
    args = dict(args)
    if n is not None:
        args["n"] = n
    if heldout:
        args["seed"] = args["seed"] + 100
    args.update(kw)
    return fn(**args)


def random_problem(rng: np.random.Generator, n: int, d: int, regression: bool = False):
    """Tiny random instances for brute-force pins (x ~ N(0, I), y = +-1 or z ~ N(0,1))."""
    X = rng.standard_normal((n, d)).astype(np.float32)
    if regression:
        return X, rng.standard_normal(n).astype(np.float32)
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    y[0], y[1] = 1.0, -1.0
    return X, y.astype(np.float32)
