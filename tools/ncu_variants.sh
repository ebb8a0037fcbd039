#!/bin/bash
# Instruction count + duration of the codec kernels for each variants/*/libfc2.so (dev tool).
for d in variants/*/; do
  echo "== $d"
  FC2_LIB=$d/libfc2.so ncu --clock-control none -k regex:"k_encode_grp|k_decode_fast" -s 2 -c 2 \
    --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    python tools/prof_codec.py 2>&1 | grep -E "k_encode|k_decode|inst_executed|duration|issue_active|warps_active" | grep -v "^==PROF" | sed 's/(fc2::.*//'
done
