"""GPU parity of every launch configuration a BASELINE config takes, and of the multi-rank path.

* One step from identical state (SURVEY 8(c) "Parity criteria"; north_star: "kernel rows and
  gradient within 1e-5 relative") through each production variant of the persistent kernel:
  X resident in shared memory, X streamed with 1 / 2 / 4 rows per thread (with and without the
  per-lane cp.async ring), wide rows through the bulk-copy pipeline (d >= 256), feature slices,
  CSR, and virtual ranks.  W must equal the oracle's exactly; G must equal the oracle's step 6
  ("calculating the gradient for all dual space coefficients") applied to the GPU's own
  dalpha within 1e-5 max(1, |G|).
* The pass-only diagnostic (svm_solver_pass_bench) against the same step 6: one pass with a fixed
  W through every row of the production launch.
* Virtual ranks (SURVEY 8(e) invariant): P ranks inside one launch run the
  multi-rank exchange (local merge, one 8+8 list per rank, owner-rank payload and row gathers)
  and must reproduce the one-rank alpha, G and iteration count bit for bit.
"""
import os
from contextlib import contextmanager

import numpy as np
import pytest

import oracle as ora
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    pkg.lib()


@contextmanager
def env(**kw):
    old = {k: os.environ.get(k) for k in kw}
    try:
        for k, v in kw.items():
            os.environ[k] = str(v)
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _csr(X):
    ip = np.concatenate([[0], np.cumsum((X != 0).sum(1))]).astype(np.int64)
    return ip, np.nonzero(X)[1].astype(np.int32), X[X != 0].astype(np.float32)


# (config, n, env, csr): every launch variant of smo_persistent that a BASELINE config takes
PATHS = {
    "xsmem": ("c1", 900, {}, False),                                   # c1 / c2: X in SMEM
    "stream_rpt1": ("c1", 1300, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=1), False),
    "stream_rpt2": ("c1", 1300, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=2), False),
    "stream_rpt4": ("c4", 2600, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=4), False),  # c4
    "stream_rpt4_noring": ("c4", 2600, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=4, SVMB200_XRING=0), False),
    "stream_rpt4_nodbuf": ("c4", 2600, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=4, SVMB200_NO_DBUF=1), False),
    "wide": ("c3", 1500, {}, False),                                   # c3 per class: bulk-copy ring
    "slices": ("c3", 1500, dict(SVMB200_NO_WIDE=1), False),           # feature-slice fallback
    "csr": ("c5", 3000, {}, True),                                     # c5: CSR staged pass
    "svr_stream_rpt2": ("c2", 1300, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=2), False),
}


def _problem(cfg, n):
    ds = synth.make(cfg, n=n)
    X = ds.dense()
    reg = ds.svm_type == synth.EPS_REGRESSION
    y = ds.y if reg or cfg != "c3" else np.where(ds.y == ds.y[0], 1.0, -1.0).astype(np.float32)
    svm_type = "eps-regression" if reg else "C-classification"
    prob = ora.Problem(ora.EPS_REGRESSION if reg else ora.C_CLASSIFICATION, y, n, 0.1)
    return ds, X, y, svm_type, prob


@pytest.mark.parametrize("path", list(PATHS))
def test_one_step_launch_paths(path):
    cfg, n, ev, csr = PATHS[path]
    ds, X, y, svm_type, prob = _problem(cfg, n)
    gamma, C, tol = 1.0 / ds.d, 1.0, 1e-3
    ks = ora.kspec("rbf", gamma, d=ds.d)
    alpha, G = np.zeros(prob.m), prob.p.copy()
    with env(**ev):
        s = (pkg.Solver(csr=_csr(X), y=y, d=ds.d, svm_type=svm_type, gamma=gamma)
             if csr else pkg.Solver(X, y, svm_type=svm_type, gamma=gamma))
        done = 0
        for steps in (0, 5, 30):
            for _ in range(steps - done):
                _, _, alpha, G = ora.step(X, prob, ks, alpha, G, C, q=16, tol=tol)
            done = steps
            G32 = G.astype(np.float32)
            W = ora.select(prob, alpha, G32.astype(np.float64), C, 16)
            s.set_state(alpha, G32)
            st = s.run(1)
            assert st.iterations == 1
            np.testing.assert_array_equal(np.array(st.last_w[:st.last_nw]), W)
            dg = np.array(st.last_dalpha[:st.last_nw])
            _, Gg = s.get_state()
            Gref = ora.gradient_update(X, prob, ks, W, dg, G32.astype(np.float64))
            err = np.abs(Gg - Gref) / np.maximum(1.0, np.abs(Gref))
            assert err.max() <= 1e-5, (path, steps, err.max())


@pytest.mark.parametrize("path", ["xsmem", "stream_rpt4", "stream_rpt2", "wide", "csr",
                                  "svr_stream_rpt2"])
def test_pass_only_diagnostic_matches_step6(path):
    """svm_solver_pass_bench (the a3 diagnostic bench.py times) computes the oracle's step 6."""
    cfg, n, ev, csr = PATHS[path]
    ds, X, y, svm_type, prob = _problem(cfg, n)
    gamma = 1.0 / ds.d
    ks = ora.kspec("rbf", gamma, d=ds.d)
    rows = np.array([3, 0, n - 1, n // 2, 17, 5, 11, n // 3, 40, 41, 42, 7, 8, 9, 99, 100])
    coef = np.linspace(-0.9, 0.8, len(rows)).astype(np.float32)
    with env(**ev):
        s = (pkg.Solver(csr=_csr(X), y=y, d=ds.d, svm_type=svm_type, gamma=gamma)
             if csr else pkg.Solver(X, y, svm_type=svm_type, gamma=gamma))
        _, G0 = s.get_state()
        ms = s.pass_bench(rows, coef, 1)
        assert ms > 0
        _, G1 = s.get_state()
    # step 6 with W = the rows' positive copies (y_w = prob.y) and y_w dalpha_w = coef_w
    W = rows.astype(np.int64)
    dalpha = coef.astype(np.float64) * prob.y[W]
    Gref = ora.gradient_update(X, prob, ks, W, dalpha, G0.astype(np.float64))
    err = np.abs(G1 - Gref) / np.maximum(1.0, np.abs(Gref))
    assert err.max() <= 1e-5, err.max()


@pytest.mark.parametrize("case", [("c4", 36864, {}, False, "C-classification"),
                                  ("c4", 36864, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=2), False,
                                   "C-classification"),
                                  ("c2", 18432, {}, False, "eps-regression"),
                                  ("c5", 36864, {}, True, "C-classification")])
def test_virtual_ranks_bit_identical(case):
    """P in {2, 4, 8} virtual ranks (144 CTAs) == one rank with the same 144 CTAs, bit for bit."""
    cfg, n, ev, csr, svm_type = case
    ds = synth.make(cfg, n=n)
    X = ds.dense()
    with env(SVMB200_NBLK=144, **ev):
        def solver():
            kw = dict(svm_type=svm_type, gamma=1.0 / ds.d)
            return (pkg.Solver(csr=(ds.indptr, ds.indices, ds.data), y=ds.y, d=ds.d, **kw)
                    if csr else pkg.Solver(X, ds.y, **kw))
        ref = solver()
        assert ref.geometry()[0] == 144
        r1 = ref.run(1000000)
        assert r1.converged
        a1, g1 = ref.get_state()
        for P in (2, 4, 8):
            s = solver()
            s.set_ranks(P)
            rp = s.run(1000000)
            ap, gp = s.get_state()
            assert rp.iterations == r1.iterations, (P, rp.iterations, r1.iterations)
            np.testing.assert_array_equal(ap, a1)
            np.testing.assert_array_equal(gp, g1)
            assert (rp.m_up, rp.M_low) == (r1.m_up, r1.M_low)


def test_virtual_ranks_one_step_vs_oracle():
    """One step through the multi-rank exchange (virtual ranks) against the oracle's step."""
    ds, X, y, svm_type, prob = _problem("c1", 2000)
    gamma, C = 1.0 / ds.d, 1.0
    ks = ora.kspec("rbf", gamma, d=ds.d)
    alpha, G = np.zeros(prob.m), prob.p.copy()
    for _ in range(9):
        _, _, alpha, G = ora.step(X, prob, ks, alpha, G, C)
    G32 = G.astype(np.float32)
    W = ora.select(prob, alpha, G32.astype(np.float64), C, 16)
    with env(SVMB200_NBLK=8):
        for P in (2, 4, 8):
            s = pkg.Solver(X, y, gamma=gamma)
            s.set_ranks(P)
            s.set_state(alpha, G32)
            st = s.run(1)
            np.testing.assert_array_equal(np.array(st.last_w[:st.last_nw]), W)
            _, Gg = s.get_state()
            Gref = ora.gradient_update(X, prob, ks, W, np.array(st.last_dalpha[:st.last_nw]),
                                       G32.astype(np.float64))
            assert (np.abs(Gg - Gref) <= 1e-5 * np.maximum(1.0, np.abs(Gref))).all()


def test_set_ranks_rejects_bad_counts():
    ds = synth.make("c1", n=900)
    with env(SVMB200_NBLK=4):
        s = pkg.Solver(ds.X, ds.y, gamma=1.0 / ds.d)
        for bad in (0, 3, 9):
            with pytest.raises(pkg.SvmError):
                s.set_ranks(bad)


def test_train_sharded_one_call_world1():
    """svm_train_sharded: the handle exchange over a one-rank NCCL communicator,
    then the shard path -- the same model as svm_train (same CTA partition: bit-identical)."""
    from paper_1706_05544_b200 import binding
    ds = synth.make("c1", n=3000)
    m1 = pkg.train(ds.X, ds.y, gamma=1.0 / ds.d)
    uid = binding.nccl_unique_id()
    assert len(uid) == 128
    ms = binding.train_sharded_nccl(ds.X, 0, ds.y, 0, 1, uid, gamma=1.0 / ds.d)
    i1, c1 = m1.support()
    i2, c2 = ms.support()
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(c1, c2)
    assert ms.info.iterations == m1.info.iterations
    dsc = synth.make("c5", n=4000)
    mc1 = pkg.train_csr(dsc.indptr, dsc.indices, dsc.data, dsc.y, dsc.d, gamma=1.0 / dsc.d)
    mc2 = binding.train_sharded_nccl_csr(dsc.indptr, dsc.indices, dsc.data, dsc.d, 0, dsc.y, 0, 1,
                                         binding.nccl_unique_id(), gamma=1.0 / dsc.d)
    np.testing.assert_array_equal(mc1.support()[1], mc2.support()[1])


@pytest.mark.parametrize("case", [("c4", 36864, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=4), False),
                                  ("c4", 20000, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=2), False),
                                  ("c2", 9000, dict(SVMB200_NO_XSMEM=1, SVMB200_RPT=1), False),
                                  ("c4", 36864, {}, True)])
def test_column_cache_bit_identical(case):
    """SURVEY 8(f) #3 / SPEC KernelRowCache ("a cached row equals a fresh recomputation
    exactly"): training with the kernel-column cache (cache passes read K columns instead of X)
    gives bit-identical alpha, G and iteration count to training without it."""
    cfg, n, ev, csr = case
    ds = synth.make(cfg, n=n)
    kw = dict(svm_type="eps-regression" if ds.svm_type == synth.EPS_REGRESSION else "C-classification",
              gamma=1.0 / ds.d)
    sp = _csr(ds.X) if csr else None   # c4's rows as CSR (one-hot blocks: 12 of 54 nonzero)

    def run(slots):
        with env(SVMB200_CACHE=slots, **ev):
            s = (pkg.Solver(csr=sp, y=ds.y, d=ds.d, **kw) if csr else pkg.Solver(ds.X, ds.y, **kw))
            st = s.run(10 ** 7)
            return st, s.get_state()
    st0, (a0, g0) = run(0)
    st1, (a1, g1) = run(1024)
    assert st0.converged and st0.cache_passes == 0
    assert st1.iterations == st0.iterations
    np.testing.assert_array_equal(a1, a0)
    np.testing.assert_array_equal(g1, g0)
    if cfg != "c2":   # (eps-SVR working sets rarely repeat all 16 rows: no cache passes needed)
        assert st1.cache_passes > 0


@pytest.mark.parametrize("n,vr", [(20000, 1), (9000, 1), (30000, 2)])
def test_csr_slice_copy_bit_identical(n, vr):
    """The CSR pass streams each 32-row chunk from the library's slice copy (SmoArgs::sell_*,
    DESIGN.md §4) instead of staging the chunk's nonzeros through shared memory: same per-row
    order and masked updates, so alpha, G and the iteration count are bit-identical to the staged
    path (SVMB200_CSR_STAGED=1), with one rank and with virtual ranks (global CTA slices)."""
    ds = synth.make("c5", n=n)
    sp = (ds.indptr, ds.indices, ds.data)

    def run(staged):
        ev = dict(SVMB200_CSR_STAGED=1) if staged else {}
        with env(**ev):
            s = pkg.Solver(csr=sp, y=ds.y, d=ds.d, gamma=1.0 / ds.d)
        if vr > 1:
            s.set_ranks(vr)
        st = s.run(3000)
        return st, s.get_state()
    st0, (a0, g0) = run(True)
    st1, (a1, g1) = run(False)
    assert st1.iterations == st0.iterations > 0
    np.testing.assert_array_equal(a1, a0)
    np.testing.assert_array_equal(g1, g0)


@pytest.mark.parametrize("n,d,P", [(1100, 40, 3), (700, 200, 4)])
def test_batched_pass_one_step_vs_oracle(n, d, P):
    """one batched iteration (k_ovr_solve + the tcgen05 k_ovr_pass with 3 fp16-split
    MMAs) from the same fp32-representable state as the oracle, for every problem: W exact and the
    new G within 1e-5 max(1, |G|) of the oracle's step 6 applied to the GPU's dalpha."""
    from paper_1706_05544_b200 import binding
    ds = synth.mnist_like(n=n, d=d, k=P)
    classes = list(dict.fromkeys(ds.y.tolist()))
    Y = np.stack([np.where(ds.y == c, 1.0, -1.0) for c in classes]).astype(np.float32)
    gamma, C = 1.0 / d, 1.0
    ks = ora.kspec("rbf", gamma, d=d)
    b = binding.BatchSolver(ds.X, Y, gamma=gamma)
    probs = [ora.Problem(ora.C_CLASSIFICATION, Y[p], n) for p in range(P)]
    states = []
    for p in range(P):   # a different number of oracle steps per problem
        alpha, G = np.zeros(n), probs[p].p.copy()
        for _ in range(3 * p):
            _, _, alpha, G = ora.step(ds.X, probs[p], ks, alpha, G, C)
        G32 = G.astype(np.float32)
        b.set_state(p, alpha, G32)
        states.append((alpha, G32))
    it = b.run(1)
    assert (it == 1).all(), it
    for p in range(P):
        alpha, G32 = states[p]
        W = ora.select(probs[p], alpha, G32.astype(np.float64), C, 16)
        ag, Gg = b.get_state(p)
        dA = ag - alpha
        Wg = np.nonzero(dA)[0]
        assert set(Wg.tolist()) <= set(W.tolist())        # only W moved (a1)
        Gref = ora.gradient_update(ds.X, probs[p], ks, W, dA[W], G32.astype(np.float64))
        err = np.abs(Gg - Gref) / np.maximum(1.0, np.abs(Gref))
        assert err.max() <= 1e-5, (p, err.max())


def test_process_state_restored_after_training():
    """The library raises the persisting-L2 set-aside for its own launch only (DESIGN.md §4
    "Process-wide state"): after training and predicting, the caller's limit is back, and a second
    model trained in the same process on the same data gives the same result (no stale scratch)."""
    import torch
    try:
        from cuda.bindings import runtime as rt
    except ImportError:
        from cuda import cudart as rt
    lim = rt.cudaLimit.cudaLimitPersistingL2CacheSize
    err, before = rt.cudaDeviceGetLimit(lim)
    assert int(err) == 0
    ds = synth.make("c4", n=20000)
    X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
    m1 = pkg.train(X, y, gamma=1.0 / ds.d)
    f1 = m1.predict(ds.X[:500], decision=True)[1]
    err, after = rt.cudaDeviceGetLimit(lim)
    assert int(err) == 0 and after == before, (before, after)
    m2 = pkg.train(X, y, gamma=1.0 / ds.d)
    f2 = m2.predict(ds.X[:500], decision=True)[1]
    assert m1.info.iterations == m2.info.iterations
    np.testing.assert_array_equal(f1, f2)


def _kkt_fp64_svc(X, ybin, sv_idx, coef, rows, gamma, C=1.0):
    """fp64 m_up - M_low over the duals of `rows`, G_i = -1 + y_i sum_s coef_s K(x_s, x_i) from
    the model's SVs (oracle kernels)."""
    ks = ora.kspec("rbf", gamma, d=X.shape[1])
    f = ora.decision(X[sv_idx], coef, 0.0, ks, X[rows])
    c = np.zeros(X.shape[0])
    c[sv_idx] = coef
    a = np.abs(c[rows])
    y = ybin[rows].astype(np.float64)
    s = -y * (-1.0 + y * f)
    up = np.where(y > 0, a < C, a > 0)
    lo = np.where(y > 0, a > 0, a < C)
    return s[up].max() - s[lo].min()


def test_incremental_recertification():
    """A resumed loop is certified again from the rows whose coefficient changed since the previous
    certification (F += sum_s (coef_s - coef'_s) K(x_s, .), fp64 sums): with resumptions forced
    (SVMB200_CERT_MARGIN = 0.6: the certification target drops to 0.6 tol) the result agrees with
    full re-certifications (SVMB200_FULL_RECERT=1), and the certified violation holds against the
    oracle's fp64 recomputation from the model's support vectors."""
    ds = synth.make("c4", n=20000)
    gamma = 1.0 / ds.d

    def run(full):
        ev = dict(SVMB200_CERT_MARGIN=0.6)
        if full:
            ev["SVMB200_FULL_RECERT"] = 1
        with env(**ev):
            return pkg.train(ds.X, ds.y, gamma=gamma)
    mi, mf = run(False), run(True)
    assert mi.info.certifications >= 2 and mf.info.certifications >= 2
    assert mi.info.converged == 1 and mf.info.converged == 1
    assert abs(mi.info.dual_objective - mf.info.dual_objective) <= 1e-7 * abs(mf.info.dual_objective)
    idx, coef = mi.support()
    ybin = ora.binary_labels(ds.y)[0]
    rows = np.arange(0, ds.n, 4)
    viol = _kkt_fp64_svc(ds.X, ybin, idx, coef[0], rows, gamma)
    assert viol <= 0.6e-3 + 2e-5, viol
    m0 = pkg.train(ds.X, ds.y, gamma=gamma)   # default margin: the counter is at least 1
    assert m0.info.certifications >= 1
    # the sharded path (one rank) re-certifies the same way: the same model bit for bit
    from paper_1706_05544_b200 import binding
    with env(SVMB200_CERT_MARGIN=0.6):
        ms = binding.train_sharded_nccl(ds.X, 0, ds.y, 0, 1, binding.nccl_unique_id(), gamma=gamma)
    assert ms.info.certifications == mi.info.certifications
    assert ms.info.iterations == mi.info.iterations
    np.testing.assert_array_equal(ms.support()[1], mi.support()[1])
