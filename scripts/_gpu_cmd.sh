export SVMB200_PROFILE=1
timeout 900 python scripts/prof_train.py c4 2000 > gpurun_out/c4_2000.log 2>&1; echo c4_rc=$?; tail -3 gpurun_out/c4_2000.log
timeout 900 python scripts/prof_train.py c3:20000 300 > gpurun_out/c3_300.log 2>&1; echo c3_rc=$?; tail -4 gpurun_out/c3_300.log
unset SVMB200_PROFILE
timeout 600 python scripts/prof_train.py c4 300 > gpurun_out/c4_300_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:smo_persistent -c 1 -o gpurun_out/smo_c4_300 python scripts/prof_train.py c4 300 > gpurun_out/ncu_c4.log 2>&1; echo ncu_rc=$?
