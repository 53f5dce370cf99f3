# A/B the product library against the timing build (MECEFO_LIB) on the same box:
# parity tests first, then the per-layer probe and the bench for both.
set -x
export PYTHONPATH=$PWD
timeout 400 python -m pytest tests/test_gemm_gpu.py tests/test_c1_parity_gpu.py tests/test_block_parity_gpu.py -x -q > gpurun_out/t_ab.log 2>&1; echo EXIT $? >> gpurun_out/t_ab.log
grep -q "EXIT 0" gpurun_out/t_ab.log || exit 1
for lab in prod timing; do
  if [ $lab = timing ]; then export MECEFO_LIB=paper_2510_16415_b200/libmecefo_timing.so; fi
  timeout 120 python scripts/fwd_probe.py $lab > gpurun_out/fwd_$lab.txt 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/bench_$lab.json 2> gpurun_out/bench_$lab.err
done
unset MECEFO_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo EXIT $? >> gpurun_out/gputest.log
