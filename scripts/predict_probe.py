"""One predict of 50,000 c2 held-out rows (tcgen05 path) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1706_05544_b200 as pkg
from paper_1706_05544_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
ds = synth.make(cfg, n=int(sys.argv[2]) if len(sys.argv) > 2 else None)
reg = ds.svm_type == synth.EPS_REGRESSION
m = pkg.train(torch.from_numpy(ds.X).cuda(), torch.from_numpy(ds.y).cuda(),
              svm_type="eps-regression" if reg else "C-classification", gamma=1.0 / ds.d, certify=0)
Xq = torch.from_numpy(synth.make(cfg, n=50000, heldout=True).X).cuda()
for _ in range(3):
    m.predict(Xq)
torch.cuda.synchronize()
print("nsv", m.info.n_sv)
