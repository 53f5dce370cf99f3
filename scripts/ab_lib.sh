# A/B the product library against the timing build (MECEFO_LIB) on the same box:
# parity tests first, then the per-layer probe and the bench for both (interleaved twice).
set -x
export PYTHONPATH=$PWD
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_block_parity_gpu.py tests/test_c1_parity_gpu.py tests/test_attention_gpu.py tests/test_engine_gpu.py tests/test_padding_gpu.py -x -q > gpurun_out/ab/t.log 2>&1; echo EXIT $? >> gpurun_out/ab/t.log
cp gpurun_out/c1_parity_*.json gpurun_out/ab/
grep -q "EXIT 0" gpurun_out/ab/t.log || exit 1
for rep in 1 2; do
for lab in prod timing; do
  if [ $lab = timing ]; then export MECEFO_LIB=paper_2510_16415_b200/libmecefo_timing.so; else unset MECEFO_LIB; fi
  python scripts/fwd_probe.py $lab > gpurun_out/ab/fwd_${lab}_$rep.txt 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/ab/bench_${lab}_$rep.json 2> gpurun_out/ab/bench_${lab}_$rep.err
done
done
