"""B200-native working-set SVM (Rgtsvm, arXiv 1706.05544): C-SVC and eps-SVR training by the
16-coefficient working-set iteration of P:53 and batched predict, as a C-ABI CUDA library
(``libsvmb200.so``, declared in ``include/svmb200.h``) with a thin ctypes binding.

    from paper_1706_05544_b200 import train
    model = train(X, y, kernel="radial", cost=1.0)      # numpy host arrays or torch CUDA tensors
    labels = model.predict(Xq)

The package holds no arithmetic of the method in Python; ``synth`` only draws seeded inputs.
"""
from .binding import (Model, Solver, SvmError, launch_count, lib, params, train,  # noqa: F401
                      train_csr)

__all__ = ["Model", "Solver", "SvmError", "launch_count", "lib", "params", "train", "train_csr"]
