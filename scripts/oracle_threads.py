"""The 'plain' CPU baseline of SURVEY 8(d) "Oracle timing": the fp64 oracle with 1 thread and
with every host thread (OpenMP), on C1 (trained to tol) and C2 (its first ITERS iterations,
iterations/s; the full run is in tests/golden/full_c2.npz).  Writes profiles/oracle_threads.json
with the host's lscpu record.  Imports only oracle/ and the generators."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, time
sys.path.insert(0, %r)
import oracle as ora
from paper_1706_05544_b200 import synth
out = {"threads": ora.num_threads()}
ds = synth.make("c1")
t = time.perf_counter()
m = ora.train(ds.X, ds.y, gamma=1.0 / ds.d)
out["c1_to_tol_s"] = time.perf_counter() - t
out["c1_iterations"] = m.results[0]["iterations"]
ds = synth.make("c2")
prob = ora.Problem(ora.EPS_REGRESSION, ds.y, ds.n, 0.1)
ks = ora.kspec("rbf", 1.0 / ds.d, d=ds.d)
t = time.perf_counter()
r = ora.train_dual(ds.X, prob, ks, 1.0, 1e-3, 16, max_iter=%d)
el = time.perf_counter() - t
out["c2_sample_iterations"] = r["iterations"]
out["c2_sample_s"] = el
out["c2_iterations_per_s"] = r["iterations"] / el
print(json.dumps(out))
"""


def lscpu():
    rec = {}
    for ln in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
        k, _, v = ln.partition(":")
        if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)"):
            rec[k.strip()] = v.strip()
    return rec


def main():
    iters = int(os.environ.get("ITERS", "300"))
    runs = []
    for th in ("1", str(os.cpu_count())):
        env = dict(os.environ, OMP_NUM_THREADS=th, OMP_PROC_BIND="close")
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, iters)], env=env,
                           capture_output=True, text=True, check=True)
        runs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    rec = {"host": lscpu(), "runs": runs,
           "note": "fp64 oracle (oracle/svm_oracle.c, gcc -O2 -fopenmp) as it stands; C2's full run "
                   "to tol: tests/golden/full_c2.npz (wall_s, threads)"}
    with open(os.path.join(ROOT, "profiles", "oracle_threads.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
