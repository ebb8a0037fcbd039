#!/bin/bash
# small-message codec latency (dev tool): ncu kernel durations + event timing at 64 KiB .. 4 MiB
mkdir -p gpurun_out
: > gpurun_out/small.log
for k in 64 256 1024 4096; do
  KIB=$k timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -k "regex:k_(encode|decode)" python tools/ncu_enc.py 2>&1 | grep -E "k_encode|k_decode|gpu__time|grid_size|block_size" | sed "s/^/$k KiB /" >> gpurun_out/small.log
done
cat gpurun_out/small.log
