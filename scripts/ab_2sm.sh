set -x
timeout 400 python -m pytest tests/test_gemm_gpu.py tests/test_c1_parity_gpu.py -x -q > gpurun_out/t_gemm.log 2>&1; echo EXIT $? >> gpurun_out/t_gemm.log
tail -3 gpurun_out/t_gemm.log
grep -q "EXIT 0" gpurun_out/t_gemm.log || exit 1
export PYTHONPATH=$PWD
TL=paper_2510_16415_b200/libmecefo_timing.so
for lab in 2sm no2sm all2sm; do
  if [ $lab = no2sm ]; then export MECEFO_LIB=$TL MECEFO_NO_2SM=1; fi
  if [ $lab = all2sm ]; then unset MECEFO_NO_2SM; export MECEFO_LIB=$TL MECEFO_2SM_MIN_K=0; fi
  timeout 120 python scripts/fwd_probe.py $lab > gpurun_out/fwd_$lab.txt 2>&1
  timeout 120 python scripts/head_probe.py $lab > gpurun_out/head_$lab.txt 2>&1
  timeout 120 python scripts/exact_probe.py > gpurun_out/exact_$lab.txt 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/bench_$lab.json 2> gpurun_out/bench_$lab.err
done
unset MECEFO_LIB MECEFO_NO_2SM
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo EXIT $? >> gpurun_out/gputest.log
