timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cv.py tests/test_gpu_golden.py tests/test_gpu_paths.py -x -q -k "ovr or cv or c3 or batched or cross" 2>&1 | tail -3
python - <<'PY' 2>&1 | grep -E "^c3|batched OvR"
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c3")
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
for v in ("0", "1", "0", "1"):
    if v == "1": os.environ["SVMB200_NO_COMPACT"] = "1"
    else: os.environ.pop("SVMB200_NO_COMPACT", None)
    m = pkg.train(X, y, gamma=1.0 / ds.d)
    inf = m.info
    print("c3 nocompact=%s train %.1f ms loop %.1f ms passes %d pass_ms %.1f iters %d" % (v, inf.train_ms, inf.loop_ms, inf.passes, inf.pass_ms, inf.iterations), flush=True)
PY
