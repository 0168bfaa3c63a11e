for pp in 1 2 4; do ABFT_K2_PARTS=$pp timeout 300 python tools/exp_modes.py base cfg4 100 >> gpurun_out/exp30.log 2>&1; echo "parts $pp" >> gpurun_out/exp30.log; done
