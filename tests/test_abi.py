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


def test_struct_layouts(tmp_path):
    """The ctypes mirrors match the C layouts of include/svmb200.h: sizes and every field offset,
    as the host C compiler lays them out."""
    import shutil
    import subprocess
    structs = [binding.svm_params, binding.svm_model_info, binding.svm_solver_stats]
    if shutil.which("gcc") is None:
        assert ctypes.sizeof(binding.svm_params) == 88
        return
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "svmb200.h"', "int main(void) {"]
    for st in structs:
        name = st.__name__
        src.append(f'printf("{name} sizeof %zu\\n", sizeof({name}));')
        for f, _ in st._fields_:
            src.append(f'printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    src.append("return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    inc = os.path.join(ROOT, "include")
    subprocess.run(["gcc", "-I", inc, "-I", "/usr/local/cuda/include", str(c), "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for st in structs:
        name = st.__name__
        assert got[(name, "sizeof")] == ctypes.sizeof(st), name
        for f, _ in st._fields_:
            assert got[(name, f)] == getattr(st, f).offset, (name, f)


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
