# ncu of the protected / unprotected K1 and K2 (cfg4), after a plain run of the same command
set -x
B="python tools/exp_k1.py base"
$B > gpurun_out/plain_exp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 8 -c 1 -o gpurun_out/k1prot2 $B > gpurun_out/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 50 -c 1 -o gpurun_out/k1unprot2 $B > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_check -s 8 -c 1 -o gpurun_out/k2b $B > gpurun_out/ncu_c.log 2>&1
ls gpurun_out
