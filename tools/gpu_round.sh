# GPU round (run through gpurun from the repo root): every GPU test, then the
# measurements of tools/gpu_final.sh (smoke, bench lines, reference arm, launch
# lists, ncu --set full of the top kernels -- each capture after its command
# ran clean without ncu)
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=12 > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest.log | tail -8
bash tools/gpu_final.sh
# the multi-rank bench path (CUDA IPC halo) with ranks sharing the one GPU
for n in 2 3; do
ABFT_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 3 --warmup 3 --no-cpu --nz-per-gpu 256 > gpurun_out/bench_mr$n.json 2> gpurun_out/bench_mr$n.err; echo mr${n}_rc=$?; tail -c 600 gpurun_out/bench_mr$n.json
done
timeout 1800 python campaign.py --exp e1,e3 --reps 20 --out gpurun_out/campaign.json > gpurun_out/campaign.log 2>&1; echo campaign_rc=$?
python tools/campaign_summary.py gpurun_out/campaign.json > gpurun_out/campaign_summary.md 2>&1
# recovery of dirty offline windows on the cfg5 slab: ROLLBACK vs PARTIAL, 1-4 flips per window
timeout 600 python tools/exp_partial.py 3 > gpurun_out/exp_partial.txt 2>&1; echo exp_partial_rc=$?
