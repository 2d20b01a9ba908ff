"""fp64 CPU oracle for the Rgtsvm working-set SMO path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import this package.  The product path (``paper_1706_05544_b200``) never
imports it; the two share no code.  The arithmetic lives in ``svm_oracle.c`` (plain C, fp64,
OpenMP over rows); this module is argument marshalling plus the plain host-side label logic of
S:296-325 (class order by first appearance, one-vs-rest per BASELINE config 3).

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, section 8(c) = SURVEY.md's oracle section.
Every function of svm_oracle.c is pinned by tests/test_oracle_*.py (closed forms, brute-force QP,
libsvm, finite differences, invariants); nothing here is "parity unpinned" except the
one-vs-rest multiclass scheme against the paper itself (the paper never names a scheme, P:39,
P:51; SURVEY 8(c) reading #9) -- it is pinned against per-class binary solves.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "svm_oracle.c")
_LIB = os.path.join(_HERE, "libsvm_oracle.so")

LINEAR, POLY, RBF, SIGMOID = 0, 1, 2, 3
KERNELS = {"linear": LINEAR, "polynomial": POLY, "poly": POLY, "radial": RBF, "rbf": RBF,
           "sigmoid": SIGMOID}
C_CLASSIFICATION, EPS_REGRESSION = 0, 3


def build(force: bool = False) -> str:
    """Compile svm_oracle.c (gcc -O2 -fopenmp, IEEE fp64: no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _KSpec(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("degree", ctypes.c_int32),
                ("gamma", ctypes.c_double), ("coef0", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        sig = {
            "ora_kernel": (f64, [P, P, i64, P]),
            "ora_build_problem": (i64, [i32, P, i64, f64, P, P, P]),
            "ora_violation": (None, [i64, P, P, P, f64, P, P]),
            "ora_select": (i32, [i64, P, P, P, f64, i32, P]),
            "ora_subproblem": (i32, [i32, P, P, P, P, f64, f64, i32]),
            "ora_gradient_update": (None, [P, i64, i64, P, P, i32, P, P, P, P]),
            "ora_bias": (f64, [i64, P, P, P, f64]),
            "ora_dual_objective": (f64, [i64, P, P, P]),
            "ora_train": (i64, [P, i64, i64, P, i64, P, P, P, f64, f64, i32, i64, f64, i32,
                                P, P, P]),
            "ora_step": (i32, [P, i64, P, i64, P, P, f64, i32, f64, i32, P, P, P, P, P]),
            "ora_coef": (None, [i32, i64, P, P, f64, P]),
            "ora_decision": (None, [P, i64, i64, P, f64, P, P, i64, P]),
            "ora_gradient_full": (None, [P, i64, P, i64, P, P, P, P, P]),
            "ora_num_threads": (i32, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def kspec(kernel="rbf", gamma=None, degree=3, coef0=0.0, d=1) -> _KSpec:
    k = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    g = (1.0 / d) if (gamma is None or gamma <= 0) else float(gamma)
    return _KSpec(k, int(degree), g, float(coef0))


def num_threads() -> int:
    return int(lib().ora_num_threads())


def kernel(u, v, ks: _KSpec) -> float:
    u = np.ascontiguousarray(u, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    return float(lib().ora_kernel(_p(u), _p(v), u.size, ctypes.byref(ks)))


def gram(X, ks: _KSpec) -> np.ndarray:
    """Dense Gram matrix from ora_kernel, upper triangle mirrored (test support)."""
    X = np.ascontiguousarray(X, np.float32)
    n = X.shape[0]
    K = np.empty((n, n))
    for i in range(n):
        for j in range(i, n):
            K[i, j] = K[j, i] = kernel(X[i], X[j], ks)
    return K


class Problem:
    """The Eq. 2 instance (y, p, map) built by ora_build_problem."""

    def __init__(self, svm_type: int, yz, n: int, epsilon: float = 0.1):
        yz = np.ascontiguousarray(yz, np.float32)
        mmax = n if svm_type == C_CLASSIFICATION else 2 * n
        self.y = np.empty(mmax, np.int8)
        self.p = np.empty(mmax)
        self.map = np.empty(mmax, np.int64)
        self.m = int(lib().ora_build_problem(int(svm_type), _p(yz), n, float(epsilon),
                                             _p(self.y), _p(self.p), _p(self.map)))
        self.type, self.n = svm_type, n


def inner_tol_for(tol: float) -> float:
    """SURVEY 8(c) reading #2: inner_tol = 0.1 tol floored at 1e-10."""
    return max(0.1 * tol, 1e-10)


def violation(prob: Problem, alpha, G, C):
    up, low = ctypes.c_double(), ctypes.c_double()
    lib().ora_violation(prob.m, _p(prob.y), _p(np.ascontiguousarray(alpha, np.float64)),
                        _p(np.ascontiguousarray(G, np.float64)), float(C),
                        ctypes.byref(up), ctypes.byref(low))
    return up.value, low.value


def select(prob: Problem, alpha, G, C, q=16):
    W = np.empty(q, np.int64)
    nw = lib().ora_select(prob.m, _p(prob.y), _p(np.ascontiguousarray(alpha, np.float64)),
                          _p(np.ascontiguousarray(G, np.float64)), float(C), int(q), _p(W))
    return W[:nw].copy()


def subproblem(yW, aW, GW, QW, C, inner_tol, max_steps):
    yW = np.ascontiguousarray(yW, np.int8)
    aW = np.array(aW, np.float64)
    GW = np.array(GW, np.float64)
    QW = np.ascontiguousarray(QW, np.float64)
    steps = lib().ora_subproblem(len(yW), _p(yW), _p(aW), _p(GW), _p(QW), float(C),
                                 float(inner_tol), int(max_steps))
    return aW, GW, int(steps)


def step(X, prob: Problem, ks, alpha, G, C, q=16, tol=1e-3, inner_max=None):
    """One outer iteration (steps 4-6) from a given state.  Returns (W, dalpha, alpha', G')."""
    X = np.ascontiguousarray(X, np.float32)
    alpha = np.array(alpha, np.float64)
    G = np.array(G, np.float64)
    W = np.empty(q, np.int64)
    dA = np.empty(q)
    steps = ctypes.c_int32()
    inner_max = 64 * q if inner_max is None else inner_max
    nw = lib().ora_step(_p(X), X.shape[1], ctypes.byref(ks), prob.m, _p(prob.y), _p(prob.map),
                        float(C), int(q), inner_tol_for(tol), int(inner_max), _p(alpha), _p(G),
                        _p(W), _p(dA), ctypes.byref(steps))
    return W[:nw].copy(), dA[:nw].copy(), alpha, G


def gradient_update(X, prob: Problem, ks, W, dalpha, G):
    """Step 6 applied to a given working set and alpha change: returns the new G."""
    X = np.ascontiguousarray(X, np.float32)
    W = np.ascontiguousarray(W, np.int64)
    dalpha = np.ascontiguousarray(dalpha, np.float64)
    Gn = np.array(G, np.float64)
    lib().ora_gradient_update(_p(X), X.shape[1], prob.m, _p(prob.y), _p(prob.map), len(W), _p(W),
                              _p(dalpha), ctypes.byref(ks), _p(Gn))
    return Gn


def gradient_full(X, prob: Problem, ks, alpha):
    X = np.ascontiguousarray(X, np.float32)
    G = np.empty(prob.m)
    lib().ora_gradient_full(_p(X), X.shape[1], ctypes.byref(ks), prob.m, _p(prob.y),
                            _p(prob.map), _p(np.ascontiguousarray(alpha, np.float64)),
                            _p(prob.p), _p(G))
    return G


def train_dual(X, prob: Problem, ks, C=1.0, tol=1e-3, q=16, max_iter=None, inner_max=None):
    """The loop of P:53 on an Eq. 2 instance.  Returns a dict with alpha, G, iterations, m_up,
    M_low, converged, b, dual, inner_steps."""
    X = np.ascontiguousarray(X, np.float32)
    n, d = X.shape
    if max_iter is None:
        max_iter = max(10 * prob.m, 10000)
    inner_max = 64 * q if inner_max is None else inner_max
    alpha = np.empty(prob.m)
    G = np.empty(prob.m)
    info = np.zeros(5)
    lib().ora_train(_p(X), n, d, ctypes.byref(ks), prob.m, _p(prob.y), _p(prob.p), _p(prob.map),
                    float(C), float(tol), int(q), int(max_iter), inner_tol_for(tol),
                    int(inner_max), _p(alpha), _p(G), _p(info))
    b = lib().ora_bias(prob.m, _p(prob.y), _p(alpha), _p(G), float(C))
    dual = lib().ora_dual_objective(prob.m, _p(alpha), _p(G), _p(prob.p))
    return dict(alpha=alpha, G=G, iterations=int(info[0]), m_up=info[1], M_low=info[2],
                converged=bool(info[3]), inner_steps=int(info[4]), b=float(b), dual=float(dual))


def coef(prob: Problem, alpha, C):
    out = np.empty(prob.n)
    lib().ora_coef(int(prob.type), prob.n, _p(prob.y), _p(np.ascontiguousarray(alpha, np.float64)),
                   float(C), _p(out))
    return out


def decision(SV, coefs, b, ks, Xq):
    SV = np.ascontiguousarray(SV, np.float32)
    Xq = np.ascontiguousarray(Xq, np.float32)
    coefs = np.ascontiguousarray(coefs, np.float64)
    f = np.empty(Xq.shape[0])
    lib().ora_decision(_p(SV), SV.shape[0], SV.shape[1], _p(coefs), float(b), ctypes.byref(ks),
                       _p(Xq), Xq.shape[0], _p(f))
    return f


class Model:
    """Oracle model: per-problem coefficient vectors over the training rows plus biases."""

    def __init__(self, svm_type, ks, X, classes, coefs, bs, results):
        self.type, self.ks, self.X = svm_type, ks, X
        self.classes = classes            # class labels (classification) or None
        self.coefs = coefs                # list of length-n coefficient arrays, one per problem
        self.bs = bs                      # list of biases
        self.results = results            # list of train_dual dicts

    def decision_function(self, Xq) -> np.ndarray:
        cols = [decision(self.X, c, b, self.ks, Xq) for c, b in zip(self.coefs, self.bs)]
        return np.stack(cols, axis=1)

    def predict(self, Xq) -> np.ndarray:
        f = self.decision_function(Xq)
        if self.type == EPS_REGRESSION:
            return f[:, 0]
        if len(self.coefs) == 1:          # binary: sign(f), f == 0 -> first class
            pos, neg, first = self.classes
            out = np.where(f[:, 0] > 0, pos, np.where(f[:, 0] < 0, neg, first))
            return out.astype(np.float64)
        return np.asarray(self.classes, np.float64)[np.argmax(f, axis=1)]  # OvR, ties -> lowest


def binary_labels(labels):
    """S:282/S:325 label handling: exactly {-1,+1} used as-is; otherwise the first-appearing
    label maps to +1.  Returns (y_pm1, (pos_label, neg_label, first_label))."""
    labels = np.asarray(labels, np.float64)
    uniq = list(dict.fromkeys(labels.tolist()))
    if set(uniq) == {-1.0, 1.0}:
        return labels.astype(np.float32), (1.0, -1.0, uniq[0])
    pos, neg = uniq[0], uniq[1]
    return np.where(labels == pos, 1.0, -1.0).astype(np.float32), (pos, neg, pos)


def train(X, yv, svm_type=C_CLASSIFICATION, kernel="rbf", C=1.0, gamma=None, degree=3,
          coef0=0.0, epsilon=0.1, tol=1e-3, q=16, max_iter=None) -> Model:
    """train dispatch: binary SVC, eps-SVR, or k > 2 classes one-vs-rest."""
    X = np.ascontiguousarray(X, np.float32)
    n, d = X.shape
    ks = kspec(kernel, gamma, degree, coef0, d)
    if svm_type == EPS_REGRESSION:
        prob = Problem(EPS_REGRESSION, yv, n, epsilon)
        r = train_dual(X, prob, ks, C, tol, q, max_iter)
        return Model(svm_type, ks, X, None, [coef(prob, r["alpha"], C)], [r["b"]], [r])
    uniq = list(dict.fromkeys(np.asarray(yv, np.float64).tolist()))
    if len(uniq) < 2:
        raise ValueError("degenerate labels")
    if len(uniq) == 2:
        ypm, cls = binary_labels(yv)
        prob = Problem(C_CLASSIFICATION, ypm, n)
        r = train_dual(X, prob, ks, C, tol, q, max_iter)
        return Model(svm_type, ks, X, cls, [coef(prob, r["alpha"], C)], [r["b"]], [r])
    coefs, bs, rs = [], [], []
    yv = np.asarray(yv, np.float64)
    for c in uniq:                        # one-vs-rest (BASELINE config 3)
        prob = Problem(C_CLASSIFICATION, np.where(yv == c, 1.0, -1.0), n)
        r = train_dual(X, prob, ks, C, tol, q, max_iter)
        coefs.append(coef(prob, r["alpha"], C))
        bs.append(r["b"])
        rs.append(r)
    return Model(svm_type, ks, X, uniq, coefs, bs, rs)
