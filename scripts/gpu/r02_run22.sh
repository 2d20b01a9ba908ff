timeout 1200 python -m pytest tests/test_gpu_golden.py -x -q -s 2>&1 | grep -E "^\[c|passed|failed|Error" | head -12
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err; head -c 1500 gpurun_out/ref_c4.json
