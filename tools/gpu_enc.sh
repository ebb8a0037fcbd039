#!/bin/bash
# encoder iteration on one GPU (dev tool): A/B timing vs variants/base, codec parity tests, one ncu capture
mkdir -p gpurun_out
: > gpurun_out/enc_ab.log
for v in ${VARIANTS:-base}; do
  FC2_LIB=variants/$v/libfc2.so timeout 300 python tools/enc_ab.py --tag $v --sizes ${SIZES:-64,256} --cells ${CELLS:-4sr,4rtn,3sr,2sr} >> gpurun_out/enc_ab.log 2>&1
done
timeout 300 python tools/enc_ab.py --tag new --sizes ${SIZES:-64,256} --cells ${CELLS:-4sr,4rtn,3sr,2sr} >> gpurun_out/enc_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fullsize.py ${EXTRA_TESTS} -x -q > gpurun_out/enc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/enc_tests.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_encode_grp -s 1 -c 1 -o gpurun_out/enc_full -f python tools/ncu_enc.py > gpurun_out/ncu_enc.log 2>&1
cat gpurun_out/enc_ab.log; tail -3 gpurun_out/enc_tests.log
