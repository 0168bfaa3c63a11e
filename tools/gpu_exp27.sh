python tools/exp_build.py ct256 -DABFT_CHECK_THREADS=256 > /dev/null 2>&1
python tools/exp_build.py ct256k2 -DABFT_CHECK_THREADS=256 -DABFT_KU=2 > /dev/null 2>&1
python tools/exp_build.py ct64 -DABFT_CHECK_THREADS=64 > /dev/null 2>&1
B="python tools/exp_modes.py"
N="--metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base mangled -k regex:k2_check|k3_lazy"
for l in base ct256 ct256k2 ct64; do timeout 600 ncu $N --log-file gpurun_out/k2_$l.csv $B $l cfg4 20 > /dev/null 2>&1; done
ls gpurun_out/k2_*.csv
