cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for c in c2 c3 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  tail -c 400 gpurun_out/bench_$c.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo "ref rc=$?"; tail -c 300 gpurun_out/ref_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
