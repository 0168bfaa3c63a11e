# bench + launch list + ncu captures of the kernels of one protected sweep (cfg4), campaign
set -x
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -2 gpurun_out/bench.log
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e"
timeout 900 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
N="--set full --clock-control none --import-source on --kernel-name-base mangled -c 1"
timeout 600 ncu $N -k regex:k1_sweepIfLi4ELi2ELi0E -s 2 -o gpurun_out/k1_lazy $B > gpurun_out/ncu_a.log 2>&1
timeout 600 ncu $N -k regex:k1_sweepIfLi4ELi1ELi0E -s 2 -o gpurun_out/k1_both $B > gpurun_out/ncu_b.log 2>&1
timeout 600 ncu $N -k regex:k1_sweepIfLi4ELi0ELi0E -s 2 -o gpurun_out/k1_none $B > gpurun_out/ncu_c.log 2>&1
timeout 600 ncu $N -k regex:k2_check -s 4 -o gpurun_out/k2 $B > gpurun_out/ncu_d.log 2>&1
timeout 600 ncu $N -k regex:k3_lazy -s 4 -o gpurun_out/k3 $B > gpurun_out/ncu_e.log 2>&1
timeout 1500 python campaign.py --reps 100 --out gpurun_out/campaign.json > gpurun_out/campaign.log 2>&1
ls -la gpurun_out
