# ncu --set full of the QKV (+RoPE) GEMM and the LM-head logits GEMM (reports
# exported to CSV; the .ncu-rep stays on the box), plus the C1 parity test on
# the timing build with the CTA-pair GEMM mode off (error baseline).
set -x
export PYTHONPATH=$PWD
mkdir -p gpurun_out/ncu gpurun_out/no2sm
MECEFO_LIB=paper_2510_16415_b200/libmecefo_timing.so MECEFO_NO_2SM=1 timeout 300 python -m pytest tests/test_c1_parity_gpu.py -x -q > gpurun_out/no2sm/t_c1.log 2>&1
cp gpurun_out/c1_parity_*.json gpurun_out/no2sm/
for spec in "qkv fwd_probe Li1ELi1ELb1EE 2" "logits head_probe ILi256ELb1ELb1ELi2ELi1ELb0EE 1"; do
  set -- $spec
  python scripts/$2.py > gpurun_out/ncu/$1_plain.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k "regex:$3" -s $4 -c 1 -o /tmp/$1 python scripts/$2.py > gpurun_out/ncu/$1_ncu.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/ncu/$1_details.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv > gpurun_out/ncu/$1_source.csv 2>&1
done
du -sh gpurun_out/ncu
