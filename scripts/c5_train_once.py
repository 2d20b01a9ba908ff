"""One full-size c5 training (CSR, 2,000,000 x 400) through the public API, for profiling runs
(SVMB200_PROFILE=1 prints the certification phases)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1706_05544_b200 as pkg  # noqa: E402
from paper_1706_05544_b200 import synth  # noqa: E402

ds = synth.make("c5")
t = [torch.from_numpy(v).cuda() for v in (ds.indptr, ds.indices, ds.data, ds.y)]
t0 = time.time()
m = pkg.train_csr(*t, ds.d, gamma=1.0 / ds.d)
print(f"c5 train {time.time() - t0:.2f} s; iterations {m.info.iterations}, loop {m.info.loop_ms:.0f} ms, "
      f"certify {m.info.certify_ms:.0f} ms in {m.info.certifications} certifications, certified {m.info.certified}")
