B="python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e"
timeout 900 $B > gpurun_out/plain_cfg5.log 2>&1
N="--set full --clock-control none --import-source on --kernel-name-base mangled -c 1"
timeout 900 ncu $N -k regex:k1_sweepIdLi3ELi0ELi0E -s 2 -o gpurun_out/k1_box27_none $B > gpurun_out/ncu_c5a.log 2>&1
timeout 900 ncu $N -k regex:k1_sweepIdLi3ELi1ELi0E -s 1 -o gpurun_out/k1_box27_ab $B > gpurun_out/ncu_c5b.log 2>&1
tail -1 gpurun_out/plain_cfg5.log | cut -c1-600
