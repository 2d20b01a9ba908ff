timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x -k "increment or sharded or world1" 2>&1 | tail -3
