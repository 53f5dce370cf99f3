# BN of the grouped low-rank launches (timing build), per-tag times from the bench's profiled leg.
export PYTHONPATH=$PWD MECEFO_LIB=paper_2510_16415_b200/libmecefo_timing.so
mkdir -p gpurun_out/lr
for v in base lowrank.up_proj=64 lowrank.up_proj=256 lowrank.P=64 lowrank.P=128 lowrank.P=256; do
  if [ $v = base ]; then unset MECEFO_BN_FOR; else export MECEFO_BN_FOR=$v; fi
  timeout 300 python bench.py --no-cpu-baseline --no-memory --no-fault-free --steps 30 > gpurun_out/lr/$v.json 2> gpurun_out/lr/$v.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/lr/$v.json').read().splitlines()[-1])
ks={k['tag']:round(k['ms_total']/30*1000,1) for k in d['kernels']}
print('$v', d['value_steady'], {t:ks.get(t) for t in ['lowrank.up_proj','lowrank.P','lowrank.Q']})
"
done
