# One measurement pass on a B200: GPU parity suite, smoke, the default bench
# line, the reference arm, the ncu launch list of one timed degraded step and
# an ncu --set full of the dominant kernel. Outputs under gpurun_out/final/.
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
python scripts/fwd_probe.py > gpurun_out/final/fwd_plain.txt 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k "regex:swiglu_bwd_dual2sm" -s 2 -c 1 -o /tmp/dual python scripts/fwd_probe.py > gpurun_out/final/ncu_dual.log 2>&1
ncu -i /tmp/dual.ncu-rep --page raw --csv > gpurun_out/final/dual_raw.csv 2>&1
ncu -i /tmp/dual.ncu-rep --page details --csv > gpurun_out/final/dual_details.csv 2>&1
