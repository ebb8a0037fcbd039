#!/bin/bash
# bench lines only (dev tool): N=1, reference N=1, N=2 on one GPU over gloo
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench rc=$?" >> gpurun_out/bench_n1.err
timeout 900 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --sweep-max 4194304 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "bench2 rc=$?" >> gpurun_out/bench_n2.err
tail -n 1 gpurun_out/bench_n1.err; tail -n 1 gpurun_out/bench_n2.err
