#!/usr/bin/env bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over the
# engine's kernels at C0 shapes: the smoke step (lean block fwd,
# neighbour bwd fp32 + bf16, fused two-microbatch engine step incl. CE, AdamW,
# budgeted refresh) and the small-shape GPU parity tests. The caching allocator
# is disabled so out-of-bounds accesses are not hidden inside pooled blocks.
# Usage (GPU box): bash scripts/sanitize.sh [outdir]   -> outdir/sanitize_*.log
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
cs=/usr/local/cuda/bin/compute-sanitizer
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
smoke='import __graft_entry__ as g; g.smoke()'
tests="tests/test_block_parity_gpu.py tests/test_engine_gpu.py tests/test_status_gpu.py tests/test_cross_entropy_gpu.py"
for tool in memcheck racecheck synccheck initcheck; do
  log="$out/sanitize_${tool}.log"
  : > "$log"
  echo "== $tool: smoke" >> "$log"
  timeout 900 $cs --tool $tool --error-exitcode 9 --print-limit 50 python -c "$smoke" >> "$log" 2>&1
  echo "rc=$? (smoke)" >> "$log"
  if [ "$tool" = memcheck ] || [ "$tool" = synccheck ]; then
    echo "== $tool: tests" >> "$log"
    timeout 1500 $cs --tool $tool --error-exitcode 9 --print-limit 50 python -m pytest -x -q -p no:cacheprovider \
      $tests -k "not c1 and not 4096" >> "$log" 2>&1
    echo "rc=$? (tests)" >> "$log"
  fi
  grep -E "ERROR SUMMARY|^rc=" "$log" | sed "s/^/[$tool] /"
done
