export PYTHONPATH=$PWD; mkdir -p gpurun_out/r2p; O=gpurun_out/r2p
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 ${@:3}; }
run 4 29601 --model 130M --scenario c2 --steps 100 > $O/c2_130M_n4.json 2> $O/c2_130M_n4.err
run 4 29602 --model 350M --scenario c3 --steps 60 --fail-prob 0.02 > $O/c3_350M_n4.json 2> $O/c3_350M_n4.err
for r in 64 128 256; do run 4 $((29610 + r)) --model 1B --rank $r --steps 10 --no-memory > $O/1b_r${r}_n4.json 2> $O/1b_r${r}_n4.err; done
run 2 29820 --model 1B --rank 128 --steps 10 --no-memory > $O/1b_r128_n2.json 2> $O/1b_r128_n2.err
ls -la $O
