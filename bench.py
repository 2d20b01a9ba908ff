#!/usr/bin/env python
"""bench.py -- the driver's benchmark of the working-set SVM hot path on B200.

One step = one pass of the whole hot path over the bench workload:
  svm_train to KKT tolerance (problem build, selection, subproblem, fused kernel-row + gradient
  pass, certification, bias, model extraction) + svm_predict of the held-out rows.
Workload (default): c4 = binary C-SVC, RBF, covertype-shaped, n = 500,000 x d = 54 dense
(BASELINE.json configs[3]) -- the largest dense config that fits one GPU and the one north_star
names for HBM evidence and 1/2/4/8-GPU scaling (BASELINE.json's metric names no config).  gamma =
1/d, C = 1, tol = 1e-3, |W| = 16; held-out predict set n_q = 100,000 (seed + 100).  Data: seeded
synthetic (paper_1706_05544_b200.synth).  --config c1..c5 selects another BASELINE config.

metric/value: BASELINE.json's metric; value = train time to KKT tol [s] (mean over timed steps,
  CUDA events on the library's stream, max over ranks); lower is better.
e2e: one full step through the public API from pinned HOST buffers: svm_train (H2D of X and y
  inside) + svm_predict of the held-out rows (H2D of Xq, D2H of the labels) [s].
roofline: the persistent working-set kernel (the dominant kernel): algorithmic bytes of the fused
  pass (n (4d + 13) B per iteration for C-SVC) x iterations / its device time.  "pass_only": the
  same fused a3 pass timed in isolation (svm_solver_pass_bench: W fixed, no exchange, no
  subproblem) -- the north_star "fused kernel-row + gradient step" GB/s.
cpu_baseline: the fp64 oracle (oracle/) on the host cores: a bounded sample (the first k SMO
  iterations of the same workload), scaled to the metric with the ORACLE's own iteration count to
  tol (tests/golden/full_<cfg>.npz, written by scripts/make_goldens.py from oracle/ alone).
--impl reference: the oracle arm of the contract (rank 0 only), the same sample and scaling.

Multi-GPU (torchrun, N > 1): rows are sharded (svm_shard_*), candidates exchanged over NVLink peer
memory inside the kernel; the model is identical on all ranks; predict shards the query rows.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train time to KKT tol & fused kernel-row GB/s vs HBM peak; predict rows/s"
ROOF_NOTES = {
    "c1": "2,000 rows on 8 CTAs: launch/serial latency bound; see DESIGN.md",
    "c2": "X is SMEM-resident for c2 (135 KB per CTA): the per-iteration chain (exchange, merge, "
          "fp64 subproblem) bounds it, not HBM; see DESIGN.md",
    "c3": "batched one-vs-rest: X (188 MB > L2) read once per batched iteration for all 10 "
          "problems; see DESIGN.md",
    "c4": "X (108 MB) streamed from HBM/L2 through per-lane cp.async rings; see DESIGN.md",
    "c5": "CSR pass: 32-row slices streamed from the lane-interleaved copy (SELL), masked X_W groups "
          "in shared memory (issue / shared-pipe bound, not HBM); algorithmic bytes 8 nnz + 17 n "
          "per iteration; see DESIGN.md",
}
WORKLOADS = {
    "c1": "binary C-SVC, RBF, two Gaussian blobs, n=2,000 d=20 dense",
    "c2": "eps-SVR, RBF, Friedman #1, n=50,000 d=100 dense (m=100,000 duals)",
    "c3": "10-class one-vs-rest C-SVC, RBF, MNIST-shaped, n=60,000 d=784 dense",
    "c4": "binary C-SVC, RBF, covertype-shaped, n=500,000 d=54 dense",
    "c5": "binary C-SVC, RBF, genomics-shaped, n=2,000,000 d=400 CSR-sparse (~10% density)",
}
CLOCK_FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c4", choices=list(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pass", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={CLOCK_FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's start-up (NVML init) holds driver locks for tens of ms and used to
            # stall the host launches of the first timed steps (c3: 141 -> 200+ ms): wait for its
            # first sample, so that the timed region starts with the sampler already running
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def fused_bytes_per_iter(cfg, n_rows, d, ncopy, nnz=None):
    """Algorithmic bytes of one fused kernel-row + gradient pass: X (4d per row
    dense; 8 per nonzero + 8 of indptr per row CSR), |x|^2 (4), G read + write (8 per dual),
    status (1 per dual)."""
    if nnz is not None:
        return 8 * nnz + n_rows * (8 + 4 + 9 * ncopy)
    return n_rows * (4 * d + 4 + 9 * ncopy)


def oracle_to_tol(cfg):
    """The oracle's own run to tol at the full BASELINE size (tests/golden/full_<cfg>.npz, written
    by scripts/make_goldens.py, which imports only oracle/ and synth): iterations summed over the
    problems, wall seconds and threads of that run.  None when the config has no golden."""
    path = os.path.join(ROOT, "tests", "golden", f"full_{cfg}.npz")
    if not os.path.exists(path):
        return None
    import numpy as np
    g = np.load(path)
    return {"iterations": int(np.sum(g["iterations"])), "wall_s": float(g["wall_s"]),
            "threads": int(g["threads"]), "source": os.path.relpath(path, ROOT)}


def cpu_baseline(ds, kw, seconds):
    """The fp64 oracle as it stands, on a bounded sample: the first k SMO iterations of the same
    workload (first problem; k sized to ~`seconds`).  Returns (seconds, k, threads)."""
    import oracle as ora
    reg = kw["svm_type"] == "eps-regression"
    if reg:
        yb = ds.y
    elif len(set(ds.y.tolist())) > 2:          # one-vs-rest: the first class against the rest
        yb = (ds.y == ds.y[0]).astype("float32") * 2 - 1
    else:
        yb = ora.binary_labels(ds.y)[0]
    prob = ora.Problem(ora.EPS_REGRESSION if reg else ora.C_CLASSIFICATION, yb, ds.n,
                       kw.get("epsilon", 0.1))
    ks = ora.kspec("rbf", kw["gamma"], d=ds.d)
    X = ds.X if ds.X is not None else ds.dense()   # c5: the oracle takes the densified rows
    t = time.perf_counter()
    ora.train_dual(X, prob, ks, C=kw["cost"], tol=kw["tolerance"], max_iter=2)
    per = (time.perf_counter() - t) / 2
    k = max(2, min(20000, int(seconds / max(per, 1e-6))))
    t = time.perf_counter()
    r = ora.train_dual(X, prob, ks, C=kw["cost"], tol=kw["tolerance"], max_iter=k)
    el = time.perf_counter() - t
    return el, max(1, r["iterations"]), ora.num_threads()


def host_cpu():
    """lscpu-style record of the host the oracle ran on (model, sockets, cores)."""
    rec = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            k, v = k.strip(), v.strip()
            if k in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                rec[k] = v
    except (OSError, subprocess.SubprocessError):
        pass
    return rec


def cpu_record(cfg, el, k, cores):
    """cpu_baseline object: the sample's iterations/s, scaled to train time to tol with the
    oracle's own iteration count (no GPU number enters); did_not_finish when none exists."""
    ref = oracle_to_tol(cfg)
    rec = {"unit": "s", "cores": cores, "kind": "oracle", "iterations_per_s": k / el,
           "host": host_cpu(),
           "sample": f"first {k} SMO iterations of {cfg} at full size in {el:.1f} s"}
    if ref is None:
        rec.update(value=None, did_not_finish=True,
                   note="no oracle run to tol at this size (SURVEY 8(d)): iterations/s only")
    else:
        rec.update(value=el / k * ref["iterations"],
                   scaled_to=f"{ref['iterations']} iterations to tol of the oracle's own full "
                             f"run ({ref['source']}: {ref['wall_s']:.0f} s on {ref['threads']} "
                             "threads of the build host)")
    return rec


def config_object(cfg, ds, hq_n, kw, world):
    """The `config` object of both arms (identical keys and values)."""
    ncopy = 2 if kw["svm_type"] == "eps-regression" else 1
    return {"workload": f"{cfg}: {WORKLOADS[cfg]}", "n": ds.n, "d": ds.d, "duals": ds.n * ncopy,
            "heldout_rows": hq_n, "C": kw["cost"], "gamma": kw["gamma"],
            "epsilon": kw["epsilon"], "tolerance": kw["tolerance"], "working_set": 16,
            "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
            "l2": "flushed (256 MB write) before every timed step"}


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    from paper_1706_05544_b200 import synth
    ds = synth.make(args.config)
    hq_n = min(ds.n, 100000)
    kw = workload_params(ds)
    vals, walls, recs = [], [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        el, k, cores = cpu_baseline(ds, kw, args.cpu_seconds)
        wall = time.perf_counter() - t0
        if i >= args.warmup:
            rec = cpu_record(args.config, el, k, cores)
            recs.append(rec)
            walls.append(wall)
            vals.append(rec["value"])
    rec = recs[-1]
    v = statistics.mean(vals) if vals[0] is not None else None
    if v is not None:
        rec["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(walls) * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_object(args.config, ds, hq_n, kw, args.gpus),
            "projected": v is not None,
            "ms_per_step_is": "wall time of the bounded oracle sample each step ran",
            "cpu_baseline": rec,
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def pass_only(pkg, X, y, kw, ncopy, n, d, peaks, passes=200):
    """The fused a3 pass (kernel rows + G update + candidate selection) in its production launch,
    timed in isolation: svm_solver_pass_bench with W = 16 fixed rows, `passes` passes in one
    launch (CUDA events on the library's stream).  Algorithmic bytes per pass: n (4d + 4 + 9 ncopy)."""
    import numpy as np
    s = pkg.Solver(X, y, **kw)
    rows = np.linspace(0, n - 1, 16).astype(np.int64)
    coef = np.full(16, 1e-6, np.float32)   # tiny: G stays near p over the passes
    s.pass_bench(rows, coef, 4)            # warm
    ms = s.pass_bench(rows, coef, passes)
    bpp = n * (4 * d + 4 + 9 * ncopy)
    gbs = bpp * passes / (ms / 1e3) / 1e9
    return {"kernel": "smo_persistent, pass-only mode (svm_solver_pass_bench)",
            "passes": passes, "us_per_pass": ms * 1e3 / passes,
            "algorithmic_bytes_per_pass": bpp, "achieved": gbs, "unit": "GB/s",
            "peak": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"]}


def batched_roofline(info, n, d, peaks, peak_src):
    """Batched one-vs-rest: the dominant kernel is k_ovr_pass, the dense
    contraction D = X X_U^T (n x d x |U|, |U| = 16 per problem) on tcgen05 plus the fused kernel /
    gradient / selection epilogue.  fp32-accurate products come from three kind::f16 MMAs per
    product (operands pre-split into fp16 hi + lo pairs with a power-of-two scale), so
    the peak is the f16 dense rate / 3, the f16 rate being the measured bf16 peak (same tensor rate,
    B200_PROFILING.md).  Algorithmic FLOPs per pass = 2 n d |U|.  Timing: CUDA event pairs on the
    library's stream around every 8th k_ovr_pass launch (an event between the solve and the pass
    would serialise the programmatic dependent launch of the others): info.pass_ms = mean sampled
    duration x info.passes."""
    nu = 16 * info.n_problem
    flops = 2.0 * n * d * nu
    per_launch_s = info.pass_ms / 1e3 / max(1, info.passes)
    peak = peaks["bf16_tflops"] / 3.0
    achieved = flops / per_launch_s / 1e12 if per_launch_s > 0 else 0.0
    xbytes = 4.0 * n * d + n * (4 + 9 * info.n_problem)
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": None,
            "algorithmic_flops_per_launch": flops, "launches": info.passes,
            "us_per_launch": per_launch_s * 1e6,
            "hbm_gbs_per_launch": xbytes / per_launch_s / 1e9 if per_launch_s > 0 else 0.0,
            "hbm_frac": (xbytes / per_launch_s / 1e9) / peaks["hbm_gbs"] if per_launch_s > 0 else 0.0,
            "kernel": "k_ovr_pass (batched one-vs-rest pass: tcgen05 3xFP16-split X X_U^T + fused epilogue)",
            "peak_source": f"{peak_src} bf16_tflops (MEASURED_PEAKS.json) / 3 (three f16 MMAs per "
                           "fp32-accurate product)",
            "note": "X (188 MB > L2) read once per batched iteration for all 10 problems"}


def workload_params(ds):
    reg = ds.svm_type == 3
    return dict(svm_type="eps-regression" if reg else "C-classification", kernel="radial",
                cost=1.0, gamma=1.0 / ds.d, epsilon=0.1, tolerance=1e-3, working_set=16)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch

    import paper_1706_05544_b200 as pkg
    from paper_1706_05544_b200 import synth

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    pkg.lib()

    # (SVMB200_BENCH_N: debugging only -- a reduced n is not the BASELINE workload)
    ds = synth.make(args.config, n=int(os.environ["SVMB200_BENCH_N"]) if os.environ.get("SVMB200_BENCH_N") else None)
    hq = synth.make(args.config, n=min(ds.n, 100000), heldout=True)
    kw = workload_params(ds)
    ncopy = 2 if kw["svm_type"] == "eps-regression" else 1
    n, d, nq = ds.n, ds.d, hq.n
    from paper_1706_05544_b200.dist import all_gather_bytes, shard_bounds
    r0, r1 = shard_bounds(n, world, rank)
    q0, q1 = shard_bounds(nq, world, rank)
    csr = ds.is_csr
    y = torch.from_numpy(ds.y).to(dev)
    if csr:   # c5: CSR training rows (this rank's slice re-based at 0) and CSR held-out rows
        ip = ds.indptr
        loc = (ip[r0:r1 + 1] - ip[r0]).astype(np.int64)
        csr_l = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                      for a in (loc, ds.indices[ip[r0]:ip[r1]], ds.data[ip[r0]:ip[r1]]))
        qip = hq.indptr
        q_csr = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                      for a in ((qip[q0:q1 + 1] - qip[q0]).astype(np.int64),
                                hq.indices[qip[q0]:qip[q1]], hq.data[qip[q0]:qip[q1]]))
        X = Xl = csr_l
        Xq = q_csr
    else:
        X = torch.from_numpy(ds.X).to(dev)
        Xq = torch.from_numpy(hq.X[q0:q1]).to(dev)
        Xl = X[r0:r1].contiguous()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def train(Xa, ya):
        if csr:
            if world == 1:
                return pkg.train_csr(*Xa, ya, d, **kw)
            return pkg.binding.train_sharded_csr(*Xa, d, r0, ya, rank, world, all_gather_bytes, **kw)
        if world == 1:
            return pkg.train(Xa, ya, **kw)
        return pkg.binding.train_sharded(Xa, r0, ya, rank, world, all_gather_bytes, **kw)

    def predict(m, Xqa):
        return m.predict_csr(*Xqa, d) if csr else m.predict(Xqa)

    def step(Xa, ya, Xqa):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        m = train(Xa, ya)
        e1.record()
        out = predict(m, Xqa)
        e2.record()
        torch.cuda.synchronize()
        return m, out, e0.elapsed_time(e1), e1.elapsed_time(e2)

    for _ in range(args.warmup):
        flush.zero_()
        step(Xl if world > 1 else X, y, Xq)
    # ---- timed region (device-resident inputs) ---------------------------------------------
    barrier()
    torch.cuda.synchronize()
    l0 = pkg.launch_count()
    tr, pr, infos = [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            m, out, t_ms, p_ms = step(Xl if world > 1 else X, y, Xq)
            tr.append(t_ms)
            pr.append(p_ms)
            infos.append(m.info)
        torch.cuda.synchronize()
        barrier()
    launches = (pkg.launch_count() - l0) / args.steps
    train_s = statistics.mean(tr) / 1e3
    pred_s = statistics.mean(pr) / 1e3
    step_ms = statistics.mean(a + b for a, b in zip(tr, pr))
    info = infos[-1]
    # per-iteration candidate exchange (the collective of SURVEY 8(e), fused into the persistent
    # kernel): CTA 0's publish -> every slot staged, as a share of the device-timed loop
    exch_us = info.exchange_ms * 1e3 / max(1, info.iterations)
    p50, p99 = info.exchange_p50_us, info.exchange_p99_us
    if world > 1:
        t = torch.tensor([train_s, pred_s, step_ms, exch_us, p50, p99], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        train_s, pred_s, step_ms, exch_us, p50, p99 = t.tolist()
    # ---- roofline of the persistent working-set kernel ---------------------------------------
    peaks, peak_src = measured_peaks()
    n_rows_local = r1 - r0
    bpi = fused_bytes_per_iter(args.config, n_rows_local, d, ncopy,
                               nnz=int(ds.indptr[r1] - ds.indptr[r0]) if csr else None)
    loop_s = info.loop_ms / 1e3
    # kernel-column cache passes read 16 cached K values per row instead of X
    cpi = n_rows_local * (4 * 16 + 4 + 9 * ncopy) if not csr else n_rows_local * (4 * 16 + 8 + 4 + 9 * ncopy)
    alg_bytes = bpi * (info.iterations - info.cache_passes) + cpi * info.cache_passes
    achieved = alg_bytes / loop_s / 1e9 if loop_s > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}_n{world}.json")
    if os.path.exists(tf):
        with open(tf) as f:
            tj = json.load(f)
        if "dram_bytes_per_launch" in tj:
            traffic = tj["dram_bytes_per_launch"]
        elif "dram_bytes_per_iter" in tj:   # streamed X: traffic scales with the iterations
            traffic = tj["dram_bytes_per_iter"] * info.iterations
    if getattr(info, "batched", 0):
        roofline = batched_roofline(info, n, d, peaks, peak_src)
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                  "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                  "algorithmic_bytes_per_launch": alg_bytes,
                  "algorithmic_bytes_per_iteration": {"pass": bpi, "cache_pass": cpi},
                  "cache_passes": info.cache_passes, "iterations": info.iterations,
                  "kernel": "smo_persistent (a1+a2+a3 fused, one cooperative launch per training)",
                  "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)",
                  "note": ROOF_NOTES.get(args.config, "")}
    # ---- e2e: pinned host buffers through the C ABI ------------------------------------------
    e2e = None
    if not args.no_e2e:
        yh = torch.from_numpy(ds.y).pin_memory()
        ya = yh.numpy()
        if csr:
            xa = tuple(t.cpu().pin_memory().numpy() for t in Xl)
            qa = tuple(t.cpu().pin_memory().numpy() for t in Xq)
        else:
            xa = torch.from_numpy(ds.X[r0:r1] if world > 1 else ds.X).pin_memory().numpy()
            qa = torch.from_numpy(hq.X[q0:q1]).pin_memory().numpy()
        step(xa, ya, qa)  # warm
        barrier()
        et, ep, ea = [], [], []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m = train(xa, ya)                 # H2D of X, y inside
            t1 = time.perf_counter()
            out = predict(m, qa)              # H2D of Xq, D2H of the labels (host array)
            t2 = time.perf_counter()
            et.append(t1 - t0)
            ep.append(t2 - t1)
            ea.append(t2 - t0)
        barrier()
        nb = (lambda a: sum(x.nbytes for x in a)) if csr else (lambda a: a.nbytes)
        nqr = (len(qa[0]) - 1) if csr else qa.shape[0]
        e = statistics.mean(ea)
        if world > 1:
            t = torch.tensor([e], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e = t.item()
        e2e = {"value": e, "unit": "s",
               "h2d_bytes_per_step": int(nb(xa) + ya.nbytes + nb(qa)),
               "d2h_bytes_per_step": int(out.nbytes),
               "includes": "svm_train + svm_predict of the held-out rows from pinned host "
                           "buffers (wall clock, synchronous API)",
               "train_s": statistics.mean(et), "predict_s": statistics.mean(ep),
               "predict_rows_per_s": nqr / statistics.mean(ep)}
    # ---- CPU baseline (rank 0, N = 1 only) ---------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        el, k, cores = cpu_baseline(ds, kw, args.cpu_seconds)
        cpu = cpu_record(args.config, el, k, cores)
    # ---- pass-only diagnostic of the fused a3 step (rank 0, dense single-problem workloads) --
    if (rank == 0 and world == 1 and not csr and not getattr(info, "batched", 0)
            and not args.no_pass and roofline.get("bound") == "hbm"):
        roofline["pass_only"] = pass_only(pkg, X, y, dict(kw), ncopy, n, d, peaks)
    if rank == 0:
        line = {
            "metric": METRIC, "value": train_s, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_object(args.config, ds, nq, kw, world),
            "iterations": info.iterations, "iterations_per_s": info.iterations / loop_s,
            "train_breakdown_ms": {"setup": info.setup_ms, "loop": info.loop_ms,
                                   "certify": info.certify_ms, "total": info.train_ms,
                                   "per_step_train_ms": tr},
            "us_per_iteration": loop_s / max(1, info.iterations) * 1e6,
            "predict_rows_per_s": nq / pred_s, "n_sv": info.n_sv,
            "converged": bool(info.converged), "certified": bool(info.certified),
            "final_violation": info.violation, "dual_objective": info.dual_objective,
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clk.summary(),
        }
        if not getattr(info, "batched", 0):
            line["exchange"] = {
                "us_per_iteration": exch_us, "p50_us": p50, "p99_us": p99,
                "frac_of_loop": exch_us * info.iterations / 1e3 / max(info.loop_ms, 1e-9),
                "measured": "clock64 on CTA 0 (max over ranks): its candidate publish -> every CTA's "
                            "keys staged (transport + wait for the slowest CTA); in-kernel NVLink "
                            "peer-memory exchange, no NCCL call per iteration"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
