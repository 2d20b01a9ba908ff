"""CPU checks of the boundary: libsvmb200.so loads and exports every function include/svmb200.h
declares; the binding's names equal the header's; host-side errors (no GPU work) are reported
with the documented codes.  No compute call is made here."""
import ctypes
import os
import re

import pytest

import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "svmb200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(svm_\w+)\s*\(", src, flags=re.M)
    assert len(names) >= 20
    return names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(binding.LIB_PATH)
    for name in header_functions():
        assert hasattr(lib, name), f"{name} declared in svmb200.h but not exported"


def test_binding_names_match_header():
    assert set(binding.SIGNATURES) == set(header_functions())


def test_struct_layouts():
    # the ctypes mirrors must match the C layout sizes (offsets of the last fields)
    assert ctypes.sizeof(binding.svm_params) == 88
    assert binding.svm_model_info.certify_ms.offset + 8 == ctypes.sizeof(binding.svm_model_info)
    assert ctypes.sizeof(binding.svm_solver_stats) % 8 == 0


def test_params_default_and_invalid_arguments():
    p = pkg.params(20)
    assert p.gamma == pytest.approx(1 / 20) and p.working_set == 16 and p.tolerance == 1e-3
    assert p.cost == 1.0 and p.epsilon == 0.1 and p.degree == 3 and p.kernel == binding.RADIAL
    lib = pkg.lib()
    assert lib.svm_params_default(None, 3) == binding.SVM_EINVAL
    assert lib.svm_params_default(ctypes.byref(binding.svm_params()), 0) == binding.SVM_EINVAL
    h = ctypes.c_void_p()
    bad = pkg.params(4, working_set=3)
    assert lib.svm_train(None, None, 10, 4, ctypes.byref(bad), ctypes.byref(h)) == binding.SVM_EINVAL
    assert "working_set" in lib.svm_last_error().decode()
    bad = pkg.params(4, cost=0.0)
    assert lib.svm_train(None, None, 10, 4, ctypes.byref(bad), ctypes.byref(h)) == binding.SVM_EINVAL
    ok = pkg.params(4)
    assert lib.svm_train(None, None, 1, 4, ctypes.byref(ok), ctypes.byref(h)) == binding.SVM_EINVAL
    assert lib.svm_shard_create(None, 1, 4, 0, None, 10, 3, 2, ctypes.byref(ok),
                                ctypes.byref(h)) == binding.SVM_EINVAL
    assert h.value is None
