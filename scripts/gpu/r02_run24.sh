SVMB200_CSR_IL=1 timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -x -q -k "csr or c5" 2>&1 | tail -2
python - <<'PY'
import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c5", n=40000)
res = []
for il in ("0", "1"):
    os.environ["SVMB200_CSR_IL"] = il
    s = pkg.Solver(csr=(ds.indptr, ds.indices, ds.data), y=ds.y, d=ds.d, gamma=1.0 / ds.d)
    st = s.run(10 ** 7)
    res.append((st.iterations, *s.get_state()))
print("bit-identical IL vs staged:", res[0][0] == res[1][0], np.array_equal(res[0][1], res[1][1]), np.array_equal(res[0][2], res[1][2]), res[0][0])
PY
for il in 0 1; do SVMB200_CSR_IL=$il SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 python scripts/pass_probe.py | sed "s/^/IL=$il /"; done
