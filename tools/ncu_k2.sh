set -x
B="python tools/exp_k1.py base"
$B > gpurun_out/plain_k2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_check -s 8 -c 1 -o gpurun_out/k2b $B > gpurun_out/ncu_k2b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 8 -c 1 -o gpurun_out/k1p2 $B > gpurun_out/ncu_k1p2.log 2>&1
cat gpurun_out/plain_k2.log
