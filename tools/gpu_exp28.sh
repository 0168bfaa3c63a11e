for zc in 103 64 37 28; do ABFT_ZCHUNK=$zc timeout 300 python tools/exp_modes.py base cfg4 100 >> gpurun_out/exp28.log 2>&1; echo "zchunk $zc" >> gpurun_out/exp28.log; done
