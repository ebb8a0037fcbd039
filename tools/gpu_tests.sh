#!/bin/bash
# run a subset of the GPU tests (dev tool): FILES="tests/a.py tests/b.py" K="expr"
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-1800} python -m pytest ${FILES:-tests} -m gpu -x -q ${K:+-k "$K"} > gpurun_out/tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tests.log
tail -30 gpurun_out/tests.log
