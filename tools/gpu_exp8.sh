set -x
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p.L2_cache_size if hasattr(p,'L2_cache_size') else p)"
python tools/exp_modes.py base > gpurun_out/exp8.log 2>&1
ABFT_L2_PERSIST=0 python tools/exp_modes.py base >> gpurun_out/exp8.log 2>&1
cat gpurun_out/exp8.log
