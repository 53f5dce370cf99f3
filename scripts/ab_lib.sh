# A/B the product library against the timing build (MECEFO_LIB) on the same box:
# GPU suite first, then the bench for both (twice, interleaved).
set -x
export PYTHONPATH=$PWD
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo EXIT $? >> gpurun_out/ab/gputest.log
grep -q "EXIT 0" gpurun_out/ab/gputest.log || exit 1
for rep in 1 2; do
for lab in prod timing; do
  if [ $lab = timing ]; then export MECEFO_LIB=paper_2510_16415_b200/libmecefo_timing.so; else unset MECEFO_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/ab/bench_${lab}_$rep.json 2> gpurun_out/ab/bench_${lab}_$rep.err
done
done
