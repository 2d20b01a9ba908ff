cd $GRAFT_REPO_ROOT
python -m pytest tests -q -x -m gpu 2>&1 | tail -3
python bench.py --no-cpu > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; tail -c 1500 gpurun_out/b_c2.json
timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; tail -c 1500 gpurun_out/b_c3.json; tail -5 gpurun_out/b_c3.err
