set -x
B="python tools/exp_k1.py base"
$B > gpurun_out/plain_y.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ymarch -s 8 -c 1 -o gpurun_out/k1y_prot $B > gpurun_out/ncu_y1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ymarch -s 50 -c 1 -o gpurun_out/k1y_unprot $B > gpurun_out/ncu_y2.log 2>&1
cat gpurun_out/plain_y.log; tail -3 gpurun_out/ncu_y1.log
