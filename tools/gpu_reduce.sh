#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_collectives.py tests/test_gpu_regressions.py -x -q > gpurun_out/red_tests.log 2>&1
echo "rc=$?" >> gpurun_out/red_tests.log
python tools/reduce_ab.py > gpurun_out/red_ab.log 2>&1
for v in minb20 minb18; do FC2_LIB=variants/$v/libfc2.so python tools/reduce_ab.py 2>&1 | sed "s/^/$v /" >> gpurun_out/red_ab.log; done
ncu --set full --import-source on --clock-control none -k regex:k_reduce_run -c 1 -o gpurun_out/red_run python tools/reduce_ab.py > gpurun_out/red_ncu.log 2>&1
tail -3 gpurun_out/red_tests.log; cat gpurun_out/red_ab.log
