#!/bin/bash
# One gpurun call: GPU tests, the N=1 bench line, the reference arm, an N=2 smoke of the
# multi-rank bench path (2 ranks sharing GPU 0 over gloo + CUDA IPC), and the ncu launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench rc=$?" >> gpurun_out/bench_n1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_n1.json 2> gpurun_out/bench_ref_n1.err
echo "ref rc=$?" >> gpurun_out/bench_ref_n1.err
timeout 900 python bench.py --gpus 2 --backend gloo --steps 3 --warmup 3 --sweep-max 4194304 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "bench2 rc=$?" >> gpurun_out/bench_n2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/bench_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/bench_ncu.log
tail -3 gpurun_out/gputest.log
