# QKV / K=512 GEMM timing knobs (timing build): tile order, B box split, no outputs.
export PYTHONPATH=$PWD MECEFO_LIB=paper_2510_16415_b200/libmecefo_timing.so
mkdir -p gpurun_out/knobs
python scripts/fwd_probe.py base > gpurun_out/knobs/base.txt 2>&1
MECEFO_NFAST_FOR=fwd.qkv=0 python scripts/fwd_probe.py nfast0 > gpurun_out/knobs/nfast0.txt 2>&1
MECEFO_B_SPLIT=1 python scripts/fwd_probe.py bsplit > gpurun_out/knobs/bsplit.txt 2>&1
MECEFO_B_SPLIT=1 MECEFO_NFAST_FOR=fwd.qkv=0 python scripts/fwd_probe.py both > gpurun_out/knobs/both.txt 2>&1
MECEFO_DBG_NOEPI=1 MECEFO_NFAST_FOR=fwd.qkv=0 python scripts/fwd_probe.py noepi_nf0 > gpurun_out/knobs/noepi_nf0.txt 2>&1
MECEFO_DBG_NOEPI=1 MECEFO_B_SPLIT=1 python scripts/fwd_probe.py noepi_bs > gpurun_out/knobs/noepi_bs.txt 2>&1
python scripts/head_probe.py base > gpurun_out/knobs/head_base.txt 2>&1
MECEFO_B_SPLIT=1 python scripts/head_probe.py bsplit > gpurun_out/knobs/head_bsplit.txt 2>&1
grep -h "fwd.qkv\|gu_swiglu\|d_h2\|TOTAL\|head\|residual" gpurun_out/knobs/*.txt | sort -k2,2 -k1,1
