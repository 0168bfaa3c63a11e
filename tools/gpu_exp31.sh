python tools/exp_build.py hlds -DABFT_HALO_LDS=1 > /dev/null 2>&1
for l in base hlds base hlds; do timeout 300 python tools/exp_modes.py $l cfg5 40 128 >> gpurun_out/exp31.log 2>&1; done
