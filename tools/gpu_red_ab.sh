#!/bin/bash
# stage-2 reducer A/B (dev tool): current build vs variants/<v>
mkdir -p gpurun_out
: > gpurun_out/red_ab.log
timeout 300 python tools/reduce_ab.py 2>&1 | sed "s/^/cur /" >> gpurun_out/red_ab.log
for v in ${VARIANTS}; do FC2_LIB=variants/$v/libfc2.so timeout 300 python tools/reduce_ab.py 2>&1 | sed "s/^/$v /" >> gpurun_out/red_ab.log; done
cat gpurun_out/red_ab.log
