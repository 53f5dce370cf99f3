"""Summarize an ncu launch list (gpu__time_duration.sum CSV) by kernel name."""
import csv
import sys
from collections import defaultdict


def main(path, out=None):
    lines_in = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines_in))
    agg = defaultdict(lambda: [0.0, 0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        tmpl = r["Kernel Name"]
        key = name if "gemm_tc_kernel" not in name else tmpl.split("(")[0] + tmpl[tmpl.find("<"):tmpl.find(">") + 1]
        agg[key][0] += float(r["Metric Value"]) / 1e3
        agg[key][1] += 1
    total = sum(v[0] for v in agg.values())
    lines = [f"launches: {sum(v[1] for v in agg.values())}, total device time {total:.1f} us (cold-cache, serialised)",
             f"{'kernel':70s} {'launches':>8s} {'us':>10s} {'share':>7s}"]
    for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"{k[:70]:70s} {n:8d} {us:10.1f} {100 * us / total:6.1f}%")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
