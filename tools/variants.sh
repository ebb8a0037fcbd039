#!/bin/bash
# Run the brief bench against each kernel-variant build under variants/ (dev tool).
for d in variants/*/; do
  echo "== $d"
  FC2_LIB=$d/libfc2.so bash tools/bench_brief.sh
done
