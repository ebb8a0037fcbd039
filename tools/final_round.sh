#!/bin/bash
# Final measurement call of a round (dev tool): gpu_round.sh (tests, N=1 bench, reference
# arm, N=2 one-GPU smoke, launch list) plus --set full captures of the encoder and the
# stage-2 reducer.
PYTEST_ARGS="${PYTEST_ARGS:--n 4}" bash tools/gpu_round.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_encode_grp -s 1 -c 1 -o gpurun_out/enc_full -f python tools/ncu_enc.py > gpurun_out/ncu_enc.log 2>&1
echo "enc ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_reduce_run -c 1 -o gpurun_out/red_run -f python tools/reduce_ab.py > gpurun_out/red_ncu.log 2>&1
echo "red ncu rc=$?"
for f in gpurun_out/bench_n1.err gpurun_out/bench_ref_n1.err gpurun_out/bench_n2.err gpurun_out/bench_ncu.log; do tail -n 1 "$f"; done
