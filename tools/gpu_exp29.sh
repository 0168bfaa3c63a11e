for zc in 28 20 16 12; do ABFT_ZCHUNK=$zc timeout 300 python tools/exp_modes.py base cfg4 100 >> gpurun_out/exp29.log 2>&1; echo "zchunk $zc" >> gpurun_out/exp29.log; done
