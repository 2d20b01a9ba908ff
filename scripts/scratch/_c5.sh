cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python bench.py --config c5 --steps 1 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
tail -c 400 gpurun_out/bench_c5.json
