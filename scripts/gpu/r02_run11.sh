timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "cache" 2>&1 | tail -3
python - <<'PY' 2>&1 | grep -v "^\[svmb200\]"
import os, sys, torch, time
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c4")
X, y = torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda()
for slots in ("0", "2048", "4096", "8192", "16384", "4096"):
    os.environ["SVMB200_CACHE"] = slots
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        m = pkg.train(X, y, gamma=1.0/ds.d)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        inf = m.info
        print(f"slots {slots:>6s} wall {1e3*(t1-t0):8.1f} ms train_ms {inf.train_ms:8.1f} loop {inf.loop_ms:8.1f} it {inf.iterations} cache_passes {inf.cache_passes}", flush=True)
PY
