timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "sharded" > gpurun_out/pytest_shard.log 2>&1; echo shard_rc=$?; tail -15 gpurun_out/pytest_shard.log
export SVMB200_PROFILE=1
timeout 900 python scripts/prof_train.py c5:200000 300 2>&1 | tail -3
timeout 900 python scripts/prof_train.py c5 100 2>&1 | tail -3
