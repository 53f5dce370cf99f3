# Fused recompute epilogue: product vs the timing build (compute-then-release epilogue), same box.
export PYTHONPATH=$PWD
mkdir -p gpurun_out/epw
TL=paper_2510_16415_b200/libmecefo_timing.so
timeout 300 python -m pytest tests/test_block_parity_gpu.py tests/test_c1_parity_gpu.py tests/test_padding_gpu.py -x -q > gpurun_out/epw/t.log 2>&1; echo EXIT $? >> gpurun_out/epw/t.log
tail -n 2 gpurun_out/epw/t.log
grep -q "EXIT 0" gpurun_out/epw/t.log || exit 1
for rep in 1 2; do
  timeout 120 python scripts/fwd_probe.py prod | grep fused_recompute
  MECEFO_LIB=$TL timeout 120 python scripts/fwd_probe.py old8 | grep fused_recompute
done
timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/epw/bench_prod.json 2> gpurun_out/epw/bench_prod.err
MECEFO_LIB=$TL timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/epw/bench_old.json 2> gpurun_out/epw/bench_old.err
for f in gpurun_out/epw/bench_prod.json gpurun_out/epw/bench_old.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); print('$f', d['value'], d['value_steady'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
