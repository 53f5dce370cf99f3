"""Print the per-kernel table of a bench JSON line (per-step ms)."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st = d["steps"]
print("value", d["value"], "steady", d.get("value_steady"), "ms/step", d["ms_per_step"])
for k in d["kernels"]:
    print(f"  {k['tag']:34s} {k['ms_total'] / st:7.3f} ms  {k['tflops']}  {k['gbs']}")
