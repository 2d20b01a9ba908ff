"""ctypes binding of libsvmb200.so -- argument marshalling only.

Every step of the path (problem build, selection, subproblem, fused kernel-row + gradient pass,
certification, bias, model extraction, predict) runs inside the CUDA library behind
``include/svmb200.h``.  This module converts numpy arrays (host) or torch CUDA tensors (device)
into pointers, calls the C ABI with the same names, and raises ``SvmError`` on a negative status.
There is no CPU fallback: if the shared library is missing, importing this module fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("SVMB200_LIB", "libsvmb200.so"))

SVM_OK, SVM_EINVAL, SVM_EDEGENERATE, SVM_ENONFINITE = 0, -1, -2, -3
SVM_ENOMEM, SVM_ECUDA, SVM_EPEER, SVM_ETIMEOUT, SVM_ENCCL = -4, -5, -6, -7, -8
C_CLASSIFICATION, EPS_REGRESSION = 0, 3
LINEAR, POLYNOMIAL, RADIAL, SIGMOID = 0, 1, 2, 3
ROW_MAJOR, COL_MAJOR = 0, 1
KERNELS = {"linear": LINEAR, "polynomial": POLYNOMIAL, "poly": POLYNOMIAL, "radial": RADIAL,
           "rbf": RADIAL, "sigmoid": SIGMOID}
TYPES = {"C-classification": C_CLASSIFICATION, "eps-regression": EPS_REGRESSION}
SHARD_HANDLE_BYTES = 1024


class SvmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class svm_params(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("kernel", ctypes.c_int32), ("cost", ctypes.c_double),
                ("gamma", ctypes.c_double), ("degree", ctypes.c_int32), ("coef0", ctypes.c_double),
                ("epsilon", ctypes.c_double), ("tolerance", ctypes.c_double),
                ("working_set", ctypes.c_int32), ("max_iter", ctypes.c_int64),
                ("layout", ctypes.c_int32), ("certify", ctypes.c_int32),
                ("stream", ctypes.c_void_p)]


class svm_model_info(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int32), ("kernel", ctypes.c_int32), ("degree", ctypes.c_int32),
                ("gamma", ctypes.c_double), ("coef0", ctypes.c_double),
                ("n_features", ctypes.c_int64), ("n_train", ctypes.c_int64),
                ("n_sv", ctypes.c_int64), ("n_class", ctypes.c_int32),
                ("n_problem", ctypes.c_int32), ("labels", ctypes.c_double * 64),
                ("b", ctypes.c_double * 64), ("iterations", ctypes.c_int64),
                ("violation", ctypes.c_double), ("converged", ctypes.c_int32),
                ("certified", ctypes.c_int32), ("dual_objective", ctypes.c_double),
                ("train_ms", ctypes.c_double), ("loop_ms", ctypes.c_double),
                ("setup_ms", ctypes.c_double), ("certify_ms", ctypes.c_double),
                ("passes", ctypes.c_int64), ("pass_ms", ctypes.c_double),
                ("batched", ctypes.c_int32), ("exchange_ms", ctypes.c_double),
                ("exchange_p50_us", ctypes.c_double), ("exchange_p99_us", ctypes.c_double),
                ("cache_passes", ctypes.c_int64), ("certifications", ctypes.c_int32)]


class svm_solver_stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("m_up", ctypes.c_double),
                ("M_low", ctypes.c_double), ("converged", ctypes.c_int32),
                ("last_nw", ctypes.c_int32), ("last_w", ctypes.c_int64 * 16),
                ("last_dalpha", ctypes.c_double * 16), ("last_inner", ctypes.c_int32),
                ("loop_ms", ctypes.c_double), ("cache_passes", ctypes.c_int64)]


class svm_cv_result(ctypes.Structure):
    _fields_ = [("nfold", ctypes.c_int32), ("failed", ctypes.c_int32), ("metric", ctypes.c_double),
                ("pearson", ctypes.c_double), ("gamma", ctypes.c_double), ("cost", ctypes.c_double),
                ("iterations", ctypes.c_int64), ("converged", ctypes.c_int32)]


# name -> (restype, argtypes); the names are exactly those of include/svmb200.h
_P = ctypes.c_void_p
_i64, _i32 = ctypes.c_int64, ctypes.c_int32
SIGNATURES = {
    "svm_params_default": (ctypes.c_int, [ctypes.POINTER(svm_params), _i64]),
    "svm_train": (ctypes.c_int, [_P, _P, _i64, _i64, ctypes.POINTER(svm_params),
                                 ctypes.POINTER(_P)]),
    "svm_train_csr": (ctypes.c_int, [_P, _P, _P, _P, _i64, _i64, ctypes.POINTER(svm_params),
                                     ctypes.POINTER(_P)]),
    "svm_predict": (ctypes.c_int, [_P, _P, _i64, _i64, _i32, _P, _P]),
    "svm_predict_csr": (ctypes.c_int, [_P, _P, _P, _P, _i64, _i64, _P, _P]),
    "svm_model_get_info": (ctypes.c_int, [_P, ctypes.POINTER(svm_model_info)]),
    "svm_model_get_sv": (ctypes.c_int, [_P, _P, _P]),
    "svm_free_model": (None, [_P]),
    "svm_last_error": (ctypes.c_char_p, []),
    "svm_launch_count": (ctypes.c_int64, []),
    "svm_solver_create": (ctypes.c_int, [_P, _P, _i64, _i64, ctypes.POINTER(svm_params),
                                         ctypes.POINTER(_P)]),
    "svm_solver_create_csr": (ctypes.c_int, [_P, _P, _P, _P, _i64, _i64,
                                             ctypes.POINTER(svm_params), ctypes.POINTER(_P)]),
    "svm_solver_size": (ctypes.c_int, [_P, ctypes.POINTER(_i64)]),
    "svm_solver_set_state": (ctypes.c_int, [_P, _P, _P]),
    "svm_solver_get_state": (ctypes.c_int, [_P, _P, _P]),
    "svm_solver_run": (ctypes.c_int, [_P, _i64, ctypes.POINTER(svm_solver_stats)]),
    "svm_solver_kernel_rows": (ctypes.c_int, [_P, _P, _i32, _P]),
    "svm_solver_set_ranks": (ctypes.c_int, [_P, _i32]),
    "svm_solver_geometry": (ctypes.c_int, [_P, ctypes.POINTER(_i32), ctypes.POINTER(_i64)]),
    "svm_solver_pass_bench": (ctypes.c_int, [_P, _P, _i32, _P, _i64, ctypes.POINTER(ctypes.c_double)]),
    "svm_solver_free": (None, [_P]),
    "svm_shard_create": (ctypes.c_int, [_P, _i64, _i64, _i64, _P, _i64, _i32, _i32,
                                        ctypes.POINTER(svm_params), ctypes.POINTER(_P)]),
    "svm_shard_create_csr": (ctypes.c_int, [_P, _P, _P, _i64, _i64, _i64, _P, _i64, _i32, _i32,
                                            ctypes.POINTER(svm_params), ctypes.POINTER(_P)]),
    "svm_shard_handle": (ctypes.c_int, [_P, _P]),
    "svm_shard_connect": (ctypes.c_int, [_P, _P]),
    "svm_shard_train": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "svm_shard_free": (None, [_P]),
    "svm_nccl_unique_id": (ctypes.c_int, [_P]),
    "svm_batch_create": (ctypes.c_int, [_P, _P, _i32, _i64, _i64, ctypes.POINTER(svm_params),
                                        ctypes.POINTER(_P)]),
    "svm_batch_set_state": (ctypes.c_int, [_P, _i32, _P, _P]),
    "svm_batch_get_state": (ctypes.c_int, [_P, _i32, _P, _P]),
    "svm_batch_run": (ctypes.c_int, [_P, _i64, _P]),
    "svm_batch_free": (None, [_P]),
    "svm_cross_validate": (ctypes.c_int, [_P, _P, _i64, _i64, ctypes.POINTER(svm_params), _i32, _P,
                                          _i32, _P, _P, ctypes.POINTER(svm_cv_result), _P]),
    "svm_train_sharded": (ctypes.c_int, [_P, _i64, _i64, _i64, _P, _i64, _i32, _i32, _P,
                                         ctypes.POINTER(svm_params), ctypes.POINTER(_P)]),
    "svm_train_sharded_csr": (ctypes.c_int, [_P, _P, _P, _i64, _i64, _i64, _P, _i64, _i32, _i32,
                                             _P, ctypes.POINTER(svm_params), ctypes.POINTER(_P)]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libsvmb200.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1706_05544_b200._build` "
                              "(the CUDA path has no CPU fallback)")
        _lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def launch_count() -> int:
    """Kernels launched by libsvmb200.so so far (svm_launch_count)."""
    return int(lib().svm_launch_count())


def _check(rc: int):
    if rc != SVM_OK:
        raise SvmError(rc, lib().svm_last_error().decode())


# ---------------------------------------------------------------- array marshalling
class _Arr:
    """Keeps a contiguous array alive and exposes its pointer (numpy host or torch device)."""

    def __init__(self, a, dtype):
        self.obj = None
        if a is None:
            self.ptr = None
            return
        if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):      # torch tensor
            import torch
            tdt = {np.float32: torch.float32, np.float64: torch.float64, np.int64: torch.int64,
                   np.int32: torch.int32}[dtype]
            t = a.contiguous() if a.dtype == tdt else a.to(tdt).contiguous()
            self.obj = t
            self.ptr = t.data_ptr()
        else:
            arr = np.ascontiguousarray(a, dtype=dtype)
            self.obj = arr
            self.ptr = arr.ctypes.data

    @property
    def p(self):
        return ctypes.c_void_p(self.ptr) if self.ptr is not None else None


def params(d: int, svm_type="C-classification", kernel="radial", cost=1.0, gamma=None, degree=3,
           coef0=0.0, epsilon=0.1, tolerance=1e-3, working_set=16, max_iter=0, layout=ROW_MAJOR,
           certify=-1, stream=None) -> svm_params:
    p = svm_params()
    _check(lib().svm_params_default(ctypes.byref(p), int(d)))
    p.type = TYPES.get(svm_type, svm_type) if isinstance(svm_type, str) else int(svm_type)
    p.kernel = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    p.cost = float(cost)
    p.gamma = float(gamma) if gamma is not None else 1.0 / d
    p.degree, p.coef0, p.epsilon = int(degree), float(coef0), float(epsilon)
    p.tolerance, p.working_set, p.max_iter = float(tolerance), int(working_set), int(max_iter)
    p.layout, p.certify = int(layout), int(certify)
    p.stream = stream
    return p


def _shape(X, layout):
    n, d = X.shape
    return int(n), int(d)


class Model:
    """A trained model (owns the C handle)."""

    def __init__(self, handle):
        self._h = ctypes.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.svm_free_model(self._h)
            self._h = ctypes.c_void_p(None)

    @property
    def info(self) -> svm_model_info:
        inf = svm_model_info()
        _check(lib().svm_model_get_info(self._h, ctypes.byref(inf)))
        return inf

    def support(self):
        """(training-row indices int64[n_sv], coefficients fp64[n_problem, n_sv])."""
        inf = self.info
        idx = np.empty(inf.n_sv, np.int64)
        coef = np.empty((inf.n_problem, inf.n_sv), np.float64)
        _check(lib().svm_model_get_sv(self._h, idx.ctypes.data_as(_P), coef.ctypes.data_as(_P)))
        return idx, coef

    def predict(self, Xq, layout=ROW_MAJOR, decision=False):
        """Returns labels / values (fp32[nq]) and, if decision, decision values [nq, n_problem]."""
        nq, d = (int(Xq.shape[0]), int(Xq.shape[1])) if layout == ROW_MAJOR else \
            (int(Xq.shape[1]), int(Xq.shape[0]))
        x = _Arr(Xq, np.float32)
        dev = x.obj is not None and hasattr(x.obj, "is_cuda") and x.obj.is_cuda
        npb = self.info.n_problem
        if dev:
            import torch
            out = torch.empty(nq, dtype=torch.float32, device=x.obj.device)
            dec = torch.empty((nq, npb), dtype=torch.float32, device=x.obj.device)
            op, dp = ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(dec.data_ptr())
        else:
            out = np.empty(nq, np.float32)
            dec = np.empty((nq, npb), np.float32)
            op, dp = out.ctypes.data_as(_P), dec.ctypes.data_as(_P)
        _check(lib().svm_predict(self._h, x.p, nq, d, int(layout), dp if decision else None, op))
        return (out, dec) if decision else out

    def predict_csr(self, indptr, indices, data, d, decision=False):
        nq = int(len(indptr) - 1)
        a, b, c = _Arr(indptr, np.int64), _Arr(indices, np.int32), _Arr(data, np.float32)
        npb = self.info.n_problem
        out = np.empty(nq, np.float32)
        dec = np.empty((nq, npb), np.float32)
        _check(lib().svm_predict_csr(self._h, a.p, b.p, c.p, nq, int(d),
                                     dec.ctypes.data_as(_P) if decision else None,
                                     out.ctypes.data_as(_P)))
        return (out, dec) if decision else out


def train(X, y, layout=ROW_MAJOR, **kw) -> Model:
    """svm_train: dense X (numpy host array or torch CUDA tensor), labels / targets y."""
    n, d = (int(X.shape[0]), int(X.shape[1])) if layout == ROW_MAJOR else \
        (int(X.shape[1]), int(X.shape[0]))
    p = params(d, layout=layout, **kw)
    x, yy = _Arr(X, np.float32), _Arr(y, np.float32)
    h = ctypes.c_void_p()
    _check(lib().svm_train(x.p, yy.p, n, d, ctypes.byref(p), ctypes.byref(h)))
    return Model(h.value)


def train_csr(indptr, indices, data, y, d, **kw) -> Model:
    n = int(len(indptr) - 1)
    p = params(d, **kw)
    a, b, c, yy = (_Arr(indptr, np.int64), _Arr(indices, np.int32), _Arr(data, np.float32),
                   _Arr(y, np.float32))
    h = ctypes.c_void_p()
    _check(lib().svm_train_csr(a.p, b.p, c.p, yy.p, n, int(d), ctypes.byref(p), ctypes.byref(h)))
    return Model(h.value)


class Solver:
    """Stepwise access to one binary / regression problem (svm_solver_* API)."""

    def __init__(self, X=None, y=None, csr=None, d=None, **kw):
        h = ctypes.c_void_p()
        if csr is not None:
            indptr, indices, data = csr
            n = int(len(indptr) - 1)
            p = params(d, **kw)
            a, b, c, yy = (_Arr(indptr, np.int64), _Arr(indices, np.int32),
                           _Arr(data, np.float32), _Arr(y, np.float32))
            _check(lib().svm_solver_create_csr(a.p, b.p, c.p, yy.p, n, int(d), ctypes.byref(p),
                                               ctypes.byref(h)))
        else:
            n, dd = int(X.shape[0]), int(X.shape[1])
            p = params(dd, **kw)
            x, yy = _Arr(X, np.float32), _Arr(y, np.float32)
            _check(lib().svm_solver_create(x.p, yy.p, n, dd, ctypes.byref(p), ctypes.byref(h)))
        self._h = h
        m = ctypes.c_int64()
        _check(lib().svm_solver_size(self._h, ctypes.byref(m)))
        self.m = int(m.value)
        self.n = n

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.svm_solver_free(self._h)
            self._h = ctypes.c_void_p(None)

    def set_state(self, alpha, G):
        a, g = _Arr(alpha, np.float64), _Arr(G, np.float32)
        _check(lib().svm_solver_set_state(self._h, a.p, g.p))

    def get_state(self):
        alpha = np.empty(self.m, np.float64)
        G = np.empty(self.m, np.float32)
        _check(lib().svm_solver_get_state(self._h, alpha.ctypes.data_as(_P),
                                          G.ctypes.data_as(_P)))
        return alpha, G

    def run(self, max_iter: int) -> svm_solver_stats:
        st = svm_solver_stats()
        _check(lib().svm_solver_run(self._h, int(max_iter), ctypes.byref(st)))
        return st

    def set_ranks(self, vranks: int):
        """svm_solver_set_ranks: run the next svm_solver_run calls as `vranks` virtual ranks."""
        _check(lib().svm_solver_set_ranks(self._h, int(vranks)))

    def geometry(self):
        """(nblk, rows_per_cta) of the persistent launch (svm_solver_geometry)."""
        nb, rpc = ctypes.c_int32(), ctypes.c_int64()
        _check(lib().svm_solver_geometry(self._h, ctypes.byref(nb), ctypes.byref(rpc)))
        return int(nb.value), int(rpc.value)

    def pass_bench(self, rows, coef, passes: int) -> float:
        """svm_solver_pass_bench: device ms of `passes` fused a3 passes with W fixed."""
        r = np.ascontiguousarray(rows, np.int64)
        c = np.ascontiguousarray(coef, np.float32)
        ms = ctypes.c_double()
        _check(lib().svm_solver_pass_bench(self._h, r.ctypes.data_as(_P), len(r),
                                           c.ctypes.data_as(_P), int(passes), ctypes.byref(ms)))
        return float(ms.value)

    def kernel_rows(self, rows):
        rows = np.ascontiguousarray(rows, np.int64)
        K = np.empty((self.n, len(rows)), np.float32)
        _check(lib().svm_solver_kernel_rows(self._h, rows.ctypes.data_as(_P), len(rows),
                                            K.ctypes.data_as(_P)))
        return K


def _shard_run(sh, world, all_gather_bytes) -> Model:
    try:
        blob = ctypes.create_string_buffer(SHARD_HANDLE_BYTES)
        _check(lib().svm_shard_handle(sh, blob))
        blobs = all_gather_bytes(blob.raw)
        allh = ctypes.create_string_buffer(b"".join(blobs), SHARD_HANDLE_BYTES * world)
        _check(lib().svm_shard_connect(sh, allh))
        h = ctypes.c_void_p()
        _check(lib().svm_shard_train(sh, ctypes.byref(h)))
        return Model(h.value)
    finally:
        lib().svm_shard_free(sh)


def train_sharded_csr(indptr, indices, data, d: int, row0: int, y_global, rank: int, world: int,
                      all_gather_bytes, **kw) -> Model:
    """svm_shard_create_csr: as train_sharded, this rank's rows [row0, row0 + n_local) in CSR
    (indptr of the local rows, starting at 0)."""
    n_local = int(len(indptr)) - 1
    n_global = int(len(y_global))
    p = params(int(d), **kw)
    a, b, c = _Arr(indptr, np.int64), _Arr(indices, np.int32), _Arr(data, np.float32)
    yy = _Arr(y_global, np.float32)
    sh = ctypes.c_void_p()
    _check(lib().svm_shard_create_csr(a.p, b.p, c.p, n_local, int(d), int(row0), yy.p, n_global,
                                      int(rank), int(world), ctypes.byref(p), ctypes.byref(sh)))
    return _shard_run(sh, world, all_gather_bytes)


def train_sharded(X_local, row0: int, y_global, rank: int, world: int, all_gather_bytes,
                  layout=ROW_MAJOR, **kw) -> Model:
    """svm_shard_*: row-sharded training over `world` GPUs (one process per GPU).

    X_local: this rank's rows [row0, row0 + n_local) (numpy host or torch CUDA tensor);
    y_global: labels / targets of all rows; all_gather_bytes(b: bytes) -> list[bytes] must
    return every rank's handle blob in rank order (e.g. torch.distributed.all_gather_object).
    Every rank returns the identical model."""
    n_local, d = (int(X_local.shape[0]), int(X_local.shape[1])) if layout == ROW_MAJOR else \
        (int(X_local.shape[1]), int(X_local.shape[0]))
    n_global = int(len(y_global))
    p = params(d, layout=layout, **kw)
    x, yy = _Arr(X_local, np.float32), _Arr(y_global, np.float32)
    sh = ctypes.c_void_p()
    _check(lib().svm_shard_create(x.p, n_local, d, int(row0), yy.p, n_global, int(rank),
                                  int(world), ctypes.byref(p), ctypes.byref(sh)))
    return _shard_run(sh, world, all_gather_bytes)


def nccl_unique_id() -> bytes:
    """svm_nccl_unique_id: a fresh 128-byte ncclUniqueId (call on rank 0, share with all ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().svm_nccl_unique_id(buf))
    return buf.raw


def train_sharded_nccl(X_local, row0: int, y_global, rank: int, world: int, nccl_id: bytes,
                       layout=ROW_MAJOR, **kw) -> Model:
    """svm_train_sharded: the one-call sharded training (handles exchanged over NCCL inside)."""
    n_local, d = (int(X_local.shape[0]), int(X_local.shape[1])) if layout == ROW_MAJOR else \
        (int(X_local.shape[1]), int(X_local.shape[0]))
    p = params(d, layout=layout, **kw)
    x, yy = _Arr(X_local, np.float32), _Arr(y_global, np.float32)
    idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
    h = ctypes.c_void_p()
    _check(lib().svm_train_sharded(x.p, n_local, d, int(row0), yy.p, int(len(y_global)), int(rank),
                                   int(world), idb, ctypes.byref(p), ctypes.byref(h)))
    return Model(h.value)


def train_sharded_nccl_csr(indptr, indices, data, d: int, row0: int, y_global, rank: int,
                           world: int, nccl_id: bytes, **kw) -> Model:
    """svm_train_sharded_csr: as train_sharded_nccl for this rank's CSR rows."""
    p = params(int(d), **kw)
    a, b, c = _Arr(indptr, np.int64), _Arr(indices, np.int32), _Arr(data, np.float32)
    yy = _Arr(y_global, np.float32)
    idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
    h = ctypes.c_void_p()
    _check(lib().svm_train_sharded_csr(a.p, b.p, c.p, int(len(indptr)) - 1, int(d), int(row0), yy.p,
                                       int(len(y_global)), int(rank), int(world), idb,
                                       ctypes.byref(p), ctypes.byref(h)))
    return Model(h.value)


def kfold_split(n: int, k: int, seed: int = 0, labels=None) -> np.ndarray:
    """Fold id per row (host plumbing, SPEC kfold_split): a seeded shuffle, then round-robin
    assignment; with labels, the round robin runs per class (stratified)."""
    if not (2 <= k <= n):
        raise ValueError("need 2 <= k <= n")
    rng = np.random.default_rng(seed)
    fold = np.empty(n, np.int32)
    if labels is None:
        perm = rng.permutation(n)
        fold[perm] = np.arange(n) % k
        return fold
    labels = np.asarray(labels)
    start = 0
    for c in dict.fromkeys(labels.tolist()):
        idx = np.nonzero(labels == c)[0]
        perm = idx[rng.permutation(idx.size)]
        fold[perm] = (np.arange(idx.size) + start) % k
        start += idx.size
    return fold


def cross_validate(X, y, nfold: int, fold=None, gammas=None, costs=None, decision=False, **kw):
    """svm_cross_validate: K-fold CV over a (gamma, C) grid on one device copy of X.
    Returns a list of per-cell dicts and, if decision, the held-out decision values
    [ngrid, n, n_problem]."""
    n, d = int(X.shape[0]), int(X.shape[1])
    p = params(d, **kw)
    ng = max(len(gammas) if gammas is not None else 1, len(costs) if costs is not None else 1)
    g = None if gammas is None else np.ascontiguousarray(np.broadcast_to(gammas, (ng,)), np.float64)
    c = None if costs is None else np.ascontiguousarray(np.broadcast_to(costs, (ng,)), np.float64)
    x, yy = _Arr(X, np.float32), _Arr(y, np.float32)
    fo = None if fold is None else _Arr(fold, np.int32)
    res = (svm_cv_result * ng)()
    yv = np.asarray(y.cpu().numpy() if hasattr(y, "cpu") else y)
    nprob = 1
    if p.type == C_CLASSIFICATION:
        ncls = len(set(yv.tolist()))
        nprob = ncls if ncls > 2 else 1
    dec = np.empty((ng, n, nprob), np.float64) if decision else None
    _check(lib().svm_cross_validate(x.p, yy.p, n, d, ctypes.byref(p), int(nfold),
                                    fo.p if fo is not None else None, ng,
                                    g.ctypes.data_as(_P) if g is not None else None,
                                    c.ctypes.data_as(_P) if c is not None else None, res,
                                    dec.ctypes.data_as(_P) if dec is not None else None))
    out = [{f: getattr(r, f) for f, _ in svm_cv_result._fields_} for r in res]
    return (out, dec) if decision else out


class BatchSolver:
    """svm_batch_*: P binary C-SVC problems on one dense X, stepwise (the batched tcgen05 pass)."""

    def __init__(self, X, Y, **kw):
        n, d = int(X.shape[0]), int(X.shape[1])
        Y = np.ascontiguousarray(Y, np.float32)
        self.P, self.n = int(Y.shape[0]), n
        p = params(d, **kw)
        x = _Arr(X, np.float32)
        h = ctypes.c_void_p()
        _check(lib().svm_batch_create(x.p, Y.ctypes.data_as(_P), self.P, n, d, ctypes.byref(p),
                                      ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.svm_batch_free(self._h)
            self._h = ctypes.c_void_p(None)

    def set_state(self, p, alpha, G):
        a, g = _Arr(alpha, np.float64), _Arr(G, np.float32)
        _check(lib().svm_batch_set_state(self._h, int(p), a.p, g.p))

    def get_state(self, p):
        alpha = np.empty(self.n, np.float64)
        G = np.empty(self.n, np.float32)
        _check(lib().svm_batch_get_state(self._h, int(p), alpha.ctypes.data_as(_P),
                                         G.ctypes.data_as(_P)))
        return alpha, G

    def run(self, max_iter: int):
        it = np.zeros(self.P, np.int64)
        _check(lib().svm_batch_run(self._h, int(max_iter), it.ctypes.data_as(_P)))
        return it
