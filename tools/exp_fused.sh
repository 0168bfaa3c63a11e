timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/t5.log 2>&1; tail -15 gpurun_out/t5.log
ABFT_FUSED_CHECK=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -p no:cacheprovider -x -k "cfg2 or cfg3 or slab" > gpurun_out/t5b.log 2>&1; tail -3 gpurun_out/t5b.log
python tools/exp_k1.py base; ABFT_FUSED_CHECK=0 python tools/exp_k1.py base; python tools/exp_k1.py base
