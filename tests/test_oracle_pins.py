"""Pins for the fp64 oracle (oracle/svm_oracle.c) against things other than itself.

Each test names what fixes the expected value: a worked example of SPEC/PAPER (cited), a closed
form derived by hand (tests/golden/closed_forms.json, each entry with its derivation), brute-force
active-set QP (tests/qp_bruteforce.py), libsvm via scikit-learn (shrinking off), a
finite-difference gradient or an invariant of S:172-174.
Chosen so that a dropped term, a wrong sign or index, or a transposed operand fails one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle as ora
from paper_1706_05544_b200 import synth
from tests import qp_bruteforce as bf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")


def _ks(kernel, d, gamma=None, degree=3, coef0=0.0):
    return ora.kspec(kernel, gamma, degree, coef0, d)


# ----------------------------------------------------------------------------- kernels (step 2)
def test_kernel_spec_examples():
    """S:119-122 worked values."""
    assert ora.kernel([1, 2], [3, 4], _ks("linear", 2)) == 11.0
    assert ora.kernel([0.3, -2.0], [0.3, -2.0], _ks("rbf", 2, gamma=0.7)) == 1.0
    assert ora.kernel([1, 0], [0, 1], _ks("sigmoid", 2, gamma=1.0, coef0=0.0)) == 0.0
    assert ora.kernel([1, 1], [1, 1], _ks("poly", 2, gamma=1.0, degree=2, coef0=1.0)) == 9.0


@pytest.mark.parametrize("kernel", ["linear", "rbf", "poly", "sigmoid"])
def test_kernel_vs_sklearn(kernel):
    """Library routine: sklearn.metrics.pairwise_kernels with libsvm's parameterisation."""
    from sklearn.metrics.pairwise import pairwise_kernels
    rng = np.random.default_rng(7)
    X = rng.standard_normal((12, 5)).astype(np.float32)
    kw = {"linear": {}, "rbf": dict(gamma=0.3), "poly": dict(gamma=0.3, degree=3, coef0=1.5),
          "sigmoid": dict(gamma=0.2, coef0=-0.4)}[kernel]
    ref = pairwise_kernels(X.astype(np.float64), metric={"poly": "polynomial"}.get(kernel, kernel),
                           **kw)
    ks = _ks(kernel, 5, gamma=kw.get("gamma"), degree=kw.get("degree", 3), coef0=kw.get("coef0", 0.0))
    got = ora.gram(X, ks)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("kernel", ["linear", "rbf", "poly"])
def test_gram_psd_and_symmetric(kernel):
    """Gram PSD (min eig >= -1e-8 l) and exactly symmetric; rbf in (0, 1]."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        X = rng.standard_normal((15, 4)).astype(np.float32)
        K = ora.gram(X, _ks(kernel, 4, gamma=0.5, coef0=1.0))
        assert (K == K.T).all()
        assert np.linalg.eigvalsh(K).min() >= -1e-8 * 15
        if kernel == "rbf":
            assert (K > 0).all() and (K <= 1).all() and (np.diag(K) == 1).all()


# ----------------------------------------------------------------------------- problem (step 1)
def test_svr_problem_spec_example():
    """l=2, z=(3,-1), eps=0.5 -> p = (-2.5, 1.5, 3.5, -0.5); y = [+1,+1,-1,-1]."""
    pr = ora.Problem(ora.EPS_REGRESSION, [3.0, -1.0], 2, 0.5)
    assert pr.m == 4
    np.testing.assert_array_equal(pr.p, [-2.5, 1.5, 3.5, -0.5])
    np.testing.assert_array_equal(pr.y, [1, 1, -1, -1])
    np.testing.assert_array_equal(pr.map, [0, 1, 0, 1])


def test_svr_block_sign():
    """Q_{1,1+l} = -K(x1, x1) (Eq. 1's [[Q,-Q],[-Q,Q]] block through y)."""
    X = np.array([[0.5, 1.0], [2.0, -1.0]], np.float32)
    pr = ora.Problem(ora.EPS_REGRESSION, [1.0, 2.0], 2, 0.1)
    ks = _ks("linear", 2)
    Q = np.array([[pr.y[i] * pr.y[j] * ora.kernel(X[pr.map[i]], X[pr.map[j]], ks)
                   for j in range(4)] for i in range(4)])
    assert Q[0, 2] == -ora.kernel(X[0], X[0], ks)
    np.testing.assert_array_equal(Q[:2, :2], -Q[:2, 2:])
    np.testing.assert_array_equal(Q[:2, :2], Q[2:, 2:])


def test_svc_problem():
    """m = l, y = labels, p = -1."""
    pr = ora.Problem(ora.C_CLASSIFICATION, [-1.0, 1.0], 2)
    np.testing.assert_array_equal(pr.y, [-1, 1])
    np.testing.assert_array_equal(pr.p, [-1.0, -1.0])


# ----------------------------------------------------------------------------- selection (3-4)
def test_select_fresh_state_c1():
    """at alpha=0, -y_i G_i = y_i, so W = first 8 positives + first 8 negatives; C1's
    interleaved labels give W = {0..15}."""
    ds = synth.make("c1")
    pr = ora.Problem(ora.C_CLASSIFICATION, ds.y, ds.n)
    W = ora.select(pr, np.zeros(pr.m), pr.p.copy(), 1.0, 16)
    np.testing.assert_array_equal(W, np.arange(16))


def test_select_clamp_and_empty():
    """S:195 clamp (m=4, size 16 -> all eligible) and the up/low structure at alpha = 0."""
    pr = ora.Problem(ora.C_CLASSIFICATION, [1, -1, 1, -1], 4)
    W = ora.select(pr, np.zeros(4), pr.p.copy(), 1.0, 16)
    np.testing.assert_array_equal(W, [0, 1, 2, 3])
    # all at upper bound for y=+1 and lower for y=-1: I_up = {} -> only the low half
    alpha = np.array([1.0, 0.0, 1.0, 0.0])
    W = ora.select(pr, alpha, pr.p.copy(), 1.0, 2)
    assert len(W) == 1


def _select_bruteforce(y, alpha, G, C, q):
    s = -y * G
    up = [i for i in range(len(y)) if (y[i] > 0 and alpha[i] < C) or (y[i] < 0 and alpha[i] > 0)]
    low = [i for i in range(len(y)) if (y[i] > 0 and alpha[i] > 0) or (y[i] < 0 and alpha[i] < C)]
    up = sorted(up, key=lambda i: (-s[i], i))[:q // 2]          # full sort, (s, index) order
    low = sorted(low, key=lambda i: (s[i], i))[:q // 2]
    return sorted(set(up) | set(low))


def test_select_vs_full_sort():
    """Brute force: full sort by (s, index) on random states with many ties."""
    rng = np.random.default_rng(3)
    for trial in range(200):
        m = int(rng.integers(2, 60))
        y = np.where(rng.random(m) < 0.5, 1, -1).astype(np.int8)
        C = 1.0
        alpha = rng.choice([0.0, 0.5, 1.0], m)
        G = rng.choice([-1.0, -0.5, 0.0, 0.25], m) if trial % 2 else rng.standard_normal(m)
        pr = ora.Problem(ora.C_CLASSIFICATION, y.astype(np.float32), m)
        q = int(rng.choice([2, 4, 16]))
        got = ora.select(pr, alpha, G, C, q)
        np.testing.assert_array_equal(got, _select_bruteforce(y.astype(float), alpha, G, C, q))


# ----------------------------------------------------------------------------- subproblem (5)
def test_subproblem_two_point_closed_form():
    """dA = (0.5, 0.5) (C=1) and (0.25, 0.25) (C=0.25); y'a preserved."""
    yW = np.array([-1, 1], np.int8)
    QW = np.array([[1.0, 1.0], [1.0, 1.0]])          # y_a y_b x_a x_b with x = (-1, +1)
    for C, want in [(1.0, 0.5), (0.25, 0.25)]:
        aW, GW, steps = ora.subproblem(yW, [0, 0], [-1, -1], QW, C, 1e-12, 100)
        np.testing.assert_allclose(aW, [want, want], rtol=0, atol=1e-15)
        assert steps >= 1


@pytest.mark.parametrize("kernel", ["linear", "rbf", "poly"])
def test_subproblem_vs_bruteforce(kernel):
    """The subproblem restricted to W (alpha outside W fixed) solved to inner_tol 1e-12 equals the
    brute-force QP on W whose linear term is G_W - Q_WW a_W; y'a is preserved and
    the local KKT violation ends below inner_tol."""
    rng = np.random.default_rng(5)
    for trial in range(15):
        nw = int(rng.integers(2, 7))
        X = rng.standard_normal((nw, 3)).astype(np.float32)
        y = np.where(rng.random(nw) < 0.5, 1, -1).astype(np.int8)
        y[0], y[1] = 1, -1
        ks = _ks(kernel, 3, gamma=0.5, coef0=1.0, degree=2)
        Q = np.outer(y, y) * ora.gram(X, ks)
        C = float([0.1, 1.0, 10.0][trial % 3])
        a0 = np.zeros(nw)
        if trial % 2:
            a0[0] = a0[1] = C / 2            # y'a0 = 0, both free
        G0 = rng.standard_normal(nw)
        aW, GW, _ = ora.subproblem(y, a0, G0, Q, C, 1e-12, 100000)
        pl = G0 - Q @ a0
        obj_smo = 0.5 * aW @ Q @ aW + pl @ aW
        _, obj_bf = bf.solve(Q, pl, y.astype(float), C)
        assert abs(obj_smo - obj_bf) <= 1e-9 * max(1.0, abs(obj_bf))
        assert abs(y @ aW) <= 1e-12 * max(1.0, C)
        assert (aW >= 0).all() and (aW <= C).all()
        s = -y * GW
        up = np.array([(y[i] > 0 and aW[i] < C) or (y[i] < 0 and aW[i] > 0) for i in range(nw)])
        lo = np.array([(y[i] > 0 and aW[i] > 0) or (y[i] < 0 and aW[i] < C) for i in range(nw)])
        if up.any() and lo.any():
            assert s[up].max() - s[lo].min() <= 1e-9
        np.testing.assert_allclose(GW, G0 + Q @ (aW - a0), atol=1e-10)


# ----------------------------------------------------------------------------- gradient (6)
@pytest.mark.parametrize("svm_type", [ora.C_CLASSIFICATION, ora.EPS_REGRESSION])
def test_gradient_consistency_and_fd(svm_type):
    """after steps, G equals the dense Q a + p; G matches central finite
    differences of the dual objective (h = 1e-5, within 1e-5)."""
    rng = np.random.default_rng(9)
    X, yz = synth.random_problem(rng, 12, 3, regression=svm_type == ora.EPS_REGRESSION)
    pr = ora.Problem(svm_type, yz, 12, 0.2)
    ks = _ks("rbf", 3, gamma=0.4)
    alpha = np.zeros(pr.m)
    G = pr.p.copy()
    for _ in range(4):
        _, _, alpha, G = ora.step(X, pr, ks, alpha, G, 1.0, q=4, tol=1e-3)
    np.testing.assert_allclose(G, ora.gradient_full(X, pr, ks, alpha), rtol=1e-12, atol=1e-12)
    Q = np.array([[pr.y[i] * pr.y[j] * ora.kernel(X[pr.map[i]], X[pr.map[j]], ks)
                   for j in range(pr.m)] for i in range(pr.m)])

    def obj(a):
        return 0.5 * a @ Q @ a + pr.p @ a
    h = 1e-5
    fd = np.array([(obj(alpha + h * e) - obj(alpha - h * e)) / (2 * h) for e in np.eye(pr.m)])
    np.testing.assert_allclose(G, fd, atol=1e-5)


# ----------------------------------------------------------------------------- whole solve
def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c["name"])
def test_closed_forms(case):
    """tests/golden/closed_forms.json: hand-derived optima, each with its citation."""
    X = np.array(case["X"], np.float32)
    svm_type = case["type"]
    ks = _ks(case["kernel"], X.shape[1], gamma=case.get("gamma"))
    pr = ora.Problem(svm_type, np.array(case["y"], np.float32), X.shape[0], case.get("epsilon", 0.1))
    r = ora.train_dual(X, pr, ks, C=case["C"], tol=1e-10)
    assert r["converged"]
    np.testing.assert_allclose(r["dual"], case["dual"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(r["b"], case["b"], atol=1e-7)
    if "alpha" in case:
        np.testing.assert_allclose(r["alpha"], case["alpha"], atol=1e-7)
    if "coef" in case:
        np.testing.assert_allclose(ora.coef(pr, r["alpha"], case["C"]), case["coef"], atol=1e-7)


@pytest.mark.parametrize("kernel", ["linear", "rbf", "poly", "sigmoid"])
@pytest.mark.parametrize("svm_type", [ora.C_CLASSIFICATION, ora.EPS_REGRESSION])
def test_train_vs_bruteforce(kernel, svm_type):
    """S:538-539 acceptance 1-2: dual objective within max(1e-6, 1e-4|opt|) of the brute-force
    active-set QP, over seeded random problems, C in {0.1, 1, 100}."""
    rng = np.random.default_rng(100 + svm_type + 7 * ["linear", "rbf", "poly", "sigmoid"].index(kernel))
    for trial in range(6):
        C = [0.1, 1.0, 100.0][trial % 3]
        n = 4 if svm_type == ora.EPS_REGRESSION else int(rng.integers(3, 8))
        X, yz = synth.random_problem(rng, n, 2, regression=svm_type == ora.EPS_REGRESSION)
        ks = _ks(kernel, 2, gamma=0.5, coef0=0.5 if kernel == "poly" else -0.2, degree=2)
        pr = ora.Problem(svm_type, yz, n, 0.1)
        r = ora.train_dual(X, pr, ks, C=C, tol=1e-9, max_iter=200000)
        Q = np.array([[pr.y[i] * pr.y[j] * ora.kernel(X[pr.map[i]], X[pr.map[j]], ks)
                       for j in range(pr.m)] for i in range(pr.m)])
        if kernel == "sigmoid" and np.linalg.eigvalsh(Q).min() < -1e-9:
            continue   # non-convex: neither method is guaranteed a global optimum
        _, obj = bf.solve(Q, pr.p, pr.y.astype(float), C)
        assert r["dual"] <= obj + max(1e-6, 1e-4 * abs(obj)), (r["dual"], obj)
        assert r["dual"] >= obj - max(1e-6, 1e-4 * abs(obj))
        assert (r["alpha"] >= 0).all() and (r["alpha"] <= C).all()
        assert abs(pr.y @ r["alpha"]) <= 1e-10 * pr.m * C


def test_c1_vs_libsvm():
    """libsvm via scikit-learn (SVC, shrinking off, tol 1e-3) on C1: same dual objective to 1e-4
    relative, decision values within 2e-3 (both stop at KKT tol 1e-3), >= 99.9% label agreement.
    Pins the dual form, p = -1, coef = y a and the bias sign."""
    from sklearn.svm import SVC
    ds = synth.make("c1")
    X, y = ds.X, ds.y
    m = ora.train(X, y, kernel="rbf", C=1.0, gamma=1.0 / ds.d, tol=1e-3)
    r = m.results[0]
    sk = SVC(C=1.0, kernel="rbf", gamma=1.0 / ds.d, tol=1e-3, shrinking=False).fit(
        X.astype(np.float64), y)
    Xh = synth.make("c1", heldout=True).X
    f_ora = m.decision_function(Xh)[:, 0]
    f_sk = sk.decision_function(Xh.astype(np.float64))
    # sklearn orders classes ascending (-1, +1): its f is for +1 vs -1, same as ours
    assert np.abs(f_ora - f_sk).max() < 2e-3
    # sklearn's dual: 1/2 a'Qa - sum a  == ours
    coef_full = np.zeros(ds.n)
    coef_full[sk.support_] = sk.dual_coef_[0]
    Kq = ora.gram(X[sk.support_], ora.kspec("rbf", 1.0 / ds.d, d=ds.d))
    c = sk.dual_coef_[0]
    d_sk = 0.5 * c @ Kq @ c - np.abs(c).sum()
    assert abs(r["dual"] - d_sk) <= 1e-4 * abs(d_sk)
    assert (np.sign(f_ora) == np.sign(f_sk)).mean() >= 0.999


def test_svr_vs_libsvm():
    """libsvm eps-SVR (shrinking off) on a C2 subsample: dual within 1e-4 relative, f within
    2e-3.  Pins Eq. 1's pairing p = [eps - z; eps + z] with [alpha*; alpha]."""
    from sklearn.svm import SVR
    ds = synth.make("c2", n=800)
    m = ora.train(ds.X, ds.y, svm_type=ora.EPS_REGRESSION, kernel="rbf", C=1.0,
                  gamma=1.0 / ds.d, epsilon=0.1, tol=1e-3)
    sk = SVR(C=1.0, kernel="rbf", gamma=1.0 / ds.d, epsilon=0.1, tol=1e-3, shrinking=False).fit(
        ds.X.astype(np.float64), ds.y.astype(np.float64))
    Xh = synth.make("c2", n=300, heldout=True).X
    f_ora = m.decision_function(Xh)[:, 0]
    f_sk = sk.predict(Xh.astype(np.float64))
    assert np.abs(f_ora - f_sk).max() < 2e-3
    c = sk.dual_coef_[0]
    Kq = ora.gram(ds.X[sk.support_], ora.kspec("rbf", 1.0 / ds.d, d=ds.d))
    d_sk = 0.5 * c @ Kq @ c + 0.1 * np.abs(c).sum() - ds.y[sk.support_].astype(np.float64) @ c
    assert abs(m.results[0]["dual"] - d_sk) <= 1e-4 * abs(d_sk)


# ----------------------------------------------------------------------------- invariants
def test_invariants_along_the_path():
    """S:172-173 box + equality at every iterate; S:239 dual non-increasing; S:243 KKT at exit."""
    ds = synth.make("c1", n=300)
    pr = ora.Problem(ora.C_CLASSIFICATION, ds.y, ds.n)
    ks = ora.kspec("rbf", 1.0 / ds.d, d=ds.d)
    alpha, G = np.zeros(pr.m), pr.p.copy()
    prev = 0.0
    for it in range(2000):
        up, low = ora.violation(pr, alpha, G, 1.0)
        if up - low <= 1e-3:
            break
        _, _, alpha, G = ora.step(ds.X, pr, ks, alpha, G, 1.0, q=16, tol=1e-3)
        assert (alpha >= 0).all() and (alpha <= 1.0).all()
        assert abs(pr.y @ alpha) <= 1e-10 * pr.m
        D = 0.5 * alpha @ (G + pr.p)
        assert D <= prev + 1e-12
        prev = D
    assert up - low <= 1e-3
    # trajectory identical to ora_train
    r = ora.train_dual(ds.X, pr, ks, C=1.0, tol=1e-3)
    assert r["iterations"] == it
    np.testing.assert_array_equal(r["alpha"], alpha)


def test_working_set_size_invariance():
    """|W| = 2 vs 16 give dual objectives within 1e-6 (tight tol)."""
    ds = synth.make("c1", n=200)
    pr = ora.Problem(ora.C_CLASSIFICATION, ds.y, ds.n)
    ks = ora.kspec("rbf", 1.0 / ds.d, d=ds.d)
    r2 = ora.train_dual(ds.X, pr, ks, 1.0, 1e-7, q=2, max_iter=10 ** 6)
    r16 = ora.train_dual(ds.X, pr, ks, 1.0, 1e-7, q=16)
    assert abs(r2["dual"] - r16["dual"]) <= 1e-6


def test_svr_complementarity_and_label_flip():
    """not both alpha_i, alpha*_i > 1e-8 at the optimum; flipped labels negate f."""
    ds = synth.make("c2", n=300)
    m = ora.train(ds.X, ds.y, svm_type=ora.EPS_REGRESSION, gamma=1.0 / ds.d, tol=1e-6)
    a = m.results[0]["alpha"]
    n = ds.n
    assert not ((a[:n] > 1e-8) & (a[n:] > 1e-8)).any()
    c1 = synth.make("c1", n=200)
    m1 = ora.train(c1.X, c1.y, gamma=0.05, tol=1e-6)
    m2 = ora.train(c1.X, -c1.y, gamma=0.05, tol=1e-6)
    Xh = synth.make("c1", n=50, heldout=True).X
    np.testing.assert_allclose(m1.decision_function(Xh), -m2.decision_function(Xh), atol=1e-5)


def test_ovr_equals_independent_binaries():
    """One-vs-rest (BASELINE config 3, parity unpinned vs the paper): each class
    problem equals a binary solve of (label == c) vs rest; predict is argmax_c f_c."""
    ds = synth.make("c3", n=300, d=20)
    m = ora.train(ds.X, ds.y, gamma=1.0 / 20, tol=1e-3)
    assert len(m.coefs) == 10
    for c in (0, 3):
        yb = np.where(ds.y == c, 1.0, -1.0)
        mb = ora.train(ds.X, yb, gamma=1.0 / 20, tol=1e-3)
        np.testing.assert_array_equal(mb.coefs[0], m.coefs[c])
    pred = m.predict(ds.X)
    f = m.decision_function(ds.X)
    np.testing.assert_array_equal(pred, np.argmax(f, 1))
