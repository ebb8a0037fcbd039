#!/bin/bash
# encoder A/B on one GPU (dev tool): round-1 kernel vs the pipelined variants
mkdir -p gpurun_out
out=gpurun_out/enc_ab.log
: > $out
FC2_ENC=grp timeout 300 python tools/enc_ab.py --tag grp >> $out 2>&1
timeout 300 python tools/enc_ab.py --tag c8s12 >> $out 2>&1
for v in ${VARIANTS:-c20s26 c6s8 c4s6 c9s13}; do
  FC2_LIB=variants/$v/libfc2.so timeout 300 python tools/enc_ab.py --tag $v --cells 4sr,4rtn >> $out 2>&1
done
timeout 300 python -m pytest tests/test_gpu_codec.py -x -q -k "bf16 or full or encode" > gpurun_out/enc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/enc_tests.log
cat $out; tail -2 gpurun_out/enc_tests.log
