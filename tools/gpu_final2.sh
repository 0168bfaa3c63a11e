B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
mkdir -p gpurun_out/n
timeout 600 $B > gpurun_out/n/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n/launches.csv $B > gpurun_out/n/ncu_list.log 2>&1
N="--set full --clock-control none --kernel-name-base mangled -c 1"
timeout 300 ncu $N --import-source on -k regex:k1_sweepIfLi4ELi2ELi0E -s 2 -o gpurun_out/n/k1_lazy $B > gpurun_out/n/ncu_a.log 2>&1
timeout 300 ncu $N -k regex:k1_sweepIfLi4ELi0ELi0E -s 2 -o gpurun_out/n/k1_none $B > gpurun_out/n/ncu_c.log 2>&1
timeout 300 ncu $N -k regex:k2_check -s 4 -o gpurun_out/n/k2 $B > gpurun_out/n/ncu_d.log 2>&1
du -sh gpurun_out/n; ls -la gpurun_out/n
