set -x
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 4 -c 1 -o gpurun_out/k1prot $B > gpurun_out/ncu_k1p.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_sweep -s 17 -c 1 -o gpurun_out/k1unprot $B > gpurun_out/ncu_k1u.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_check -s 4 -c 1 -o gpurun_out/k2 $B > gpurun_out/ncu_k2.log 2>&1
ls -la gpurun_out
