export SVMB200_LIB=libsvmb200_prof.so SVMB200_PROFILE=1
python - <<'PY' 2>&1 | grep -E "k_ovr|batched OvR|c3"
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c3")
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
for rep in range(2):
    m = pkg.train(X, y, gamma=1.0 / ds.d)
    print("c3", m.info.loop_ms, m.info.passes, m.info.pass_ms, flush=True)
PY
