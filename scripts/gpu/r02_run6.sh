(export SVMB200_LIB=libsvmb200_prof.so SVMB200_PROFILE=1
python scripts/pass_probe.py 2>&1 | tail -3
python - <<'PY' 2>&1 | grep svmb200 | tail -4
import os, sys, torch
sys.path.insert(0, '.')
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
ds = synth.make("c4")
m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(), gamma=1.0/ds.d, certify=0)
PY
)
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_paths.py -x -q -s -k "c3 or sharded" 2>&1 | tail -8
