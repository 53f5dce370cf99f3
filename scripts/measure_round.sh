# One measurement pass on a B200: GPU parity suite, the default bench line,
# the ncu launch list of one timed degraded step and an ncu --set full of the
# QKV (+RoPE) GEMM and the dominant kernel. Outputs under gpurun_out/.
set -x
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo EXIT $? >> gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/plain_profile_only.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
python scripts/fwd_probe.py > gpurun_out/fwd_plain.txt 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:gemm_tc_kernel<256, true, true, 1, 1, true>' -s 2 -c 1 -o gpurun_out/qkv \
    python scripts/fwd_probe.py > gpurun_out/ncu_qkv.log 2>&1
