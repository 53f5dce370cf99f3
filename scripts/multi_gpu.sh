# torchrun N-GPU bench lines (degraded step, fault-free, exchange) on one box.
N=${1:-4}
mkdir -p gpurun_out/multi
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus $N > gpurun_out/multi/bench_n$N.json 2> gpurun_out/multi/bench_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus $N --scenario c2 > gpurun_out/multi/c2_n$N.json 2> gpurun_out/multi/c2_n$N.err
