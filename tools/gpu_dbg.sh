mkdir -p gpurun_out
timeout 600 python tools/n2_repro.py > gpurun_out/n2_repro.log 2>&1
echo "repro rc=$?" >> gpurun_out/n2_repro.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_encode_grp -s 1 -c 1 -o gpurun_out/enc_full -f python tools/ncu_enc.py > gpurun_out/ncu_enc.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_enc.log
grep -v Warning gpurun_out/n2_repro.log | tail -30; tail -3 gpurun_out/ncu_enc.log
