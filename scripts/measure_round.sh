# One measurement pass on a B200: GPU parity suite, smoke, the default bench
# line, and the ncu launch list of one timed degraded step. Outputs under gpurun_out/final/.
set -x
export PYTHONPATH=$PWD
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/gputest.log 2>&1; echo EXIT $? >> gpurun_out/final/gputest.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/final/plain_profile_only.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/final/launches.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/final/ncu_launch.log 2>&1
