python tools/exp_build.py defer -DABFT_ROWS_DEFERRED=1
for l in base defer base defer; do python tools/exp_modes.py $l >> gpurun_out/exp17.log 2>&1; done
