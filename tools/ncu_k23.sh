B="python tools/exp_modes.py base"
$B > gpurun_out/plain_k23.log 2>&1
N="--set full --clock-control none --import-source on --kernel-name-base mangled -c 1"
timeout 600 ncu $N -k regex:k2_check -s 400 -o gpurun_out/k2L $B > gpurun_out/ncu_k2L.log 2>&1
timeout 600 ncu $N -k regex:k3_lazy -s 20 -o gpurun_out/k3L $B > gpurun_out/ncu_k3L.log 2>&1
timeout 600 ncu $N -k regex:k1_sweepIfLi4ELi2ELb0E -s 20 -o gpurun_out/k1L $B > gpurun_out/ncu_k1L.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k23.csv $B > /dev/null 2>&1
