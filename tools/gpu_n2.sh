#!/bin/bash
# N=2 bench arms on one GPU (2 ranks share GPU 0 over gloo + CUDA IPC) + one reduce-kernel ncu capture (dev tool)
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --sweep-max 4194304 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "bench2 rc=$?" >> gpurun_out/bench_n2.err
timeout 900 python bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_ref_n2.json 2> gpurun_out/bench_ref_n2.err
echo "ref2 rc=$?" >> gpurun_out/bench_ref_n2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_reduce_run -c 1 -o gpurun_out/red_run -f python tools/reduce_ab.py > gpurun_out/red_ncu.log 2>&1
tail -2 gpurun_out/bench_n2.err gpurun_out/bench_ref_n2.err; cat gpurun_out/bench_ref_n2.json | cut -c1-600
