# torchrun N-GPU bench line and the reference arm under torchrun (rank 0 only prints).
N=${1:-4}
mkdir -p gpurun_out/multi
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 \
  bench.py --gpus $N > gpurun_out/multi/final_n$N.json 2> gpurun_out/multi/final_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29515 \
  bench.py --gpus $N --impl reference --steps 2 --warmup 1 > gpurun_out/multi/ref_n$N.json 2> gpurun_out/multi/ref_n$N.err
echo "ref exit $?" >> gpurun_out/multi/ref_n$N.err
