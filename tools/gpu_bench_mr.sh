# the multi-rank bench path (CUDA IPC) on a one-GPU box: 2 and 3 ranks share cuda:0
set -x
for n in 2 3; do
ABFT_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus $n --steps 3 --warmup 3 --no-cpu --nz-per-gpu 256 > gpurun_out/bench_mr$n.json 2> gpurun_out/bench_mr$n.err; echo rc=$?; tail -c 1500 gpurun_out/bench_mr$n.json; tail -5 gpurun_out/bench_mr$n.err
done
ABFT_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --config cfg5 --steps 3 --warmup 3 --no-cpu --nz-per-gpu 32 > gpurun_out/bench_mr5.json 2> gpurun_out/bench_mr5.err; echo rc=$?; tail -c 1200 gpurun_out/bench_mr5.json; tail -5 gpurun_out/bench_mr5.err
