# Residual+norm GEMM: windows spread over all SMs (default) vs one 128-row block per CTA.
export PYTHONPATH=$PWD
mkdir -p gpurun_out/gn
TL=paper_2510_16415_b200/libmecefo_timing.so
timeout 600 python -m pytest tests/test_block_parity_gpu.py tests/test_c1_parity_gpu.py tests/test_engine_gpu.py tests/test_harness_gpu.py tests/test_reference_shim_gpu.py -x -q > gpurun_out/gn/t.log 2>&1; echo EXIT $? >> gpurun_out/gn/t.log
tail -n 2 gpurun_out/gn/t.log
grep -q "EXIT 0" gpurun_out/gn/t.log || exit 1
for rep in 1 2; do
  MECEFO_LIB=$TL timeout 120 python scripts/fwd_probe.py spread | grep residual
  MECEFO_LIB=$TL MECEFO_GN_NOSPREAD=1 timeout 120 python scripts/fwd_probe.py blocks | grep residual
done
timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/gn/bench_spread.json 2> gpurun_out/gn/bench_spread.err
MECEFO_LIB=$TL MECEFO_GN_NOSPREAD=1 timeout 300 python bench.py --no-cpu-baseline --no-memory > gpurun_out/gn/bench_blocks.json 2> gpurun_out/gn/bench_blocks.err
for f in gpurun_out/gn/bench_spread.json gpurun_out/gn/bench_blocks.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); ks={k['tag']:round(k['ms_total']/d['steps']*1000,1) for k in d['kernels']}
print('$f', d['value'], d['value_steady'], d['fault_free_tokens_per_s'], ks.get('fwd.o_residual_norm'), ks.get('fwd.down_residual_norm'), d['clocks']['sm_mhz'])"; done
