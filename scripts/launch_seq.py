"""Print an ncu launch list (gpu__time_duration.sum CSV) in launch order."""
import csv, sys
rows = list(csv.DictReader([l for l in open(sys.argv[1]) if l.startswith('"')]))
tot = 0.0
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    n = r["Kernel Name"]
    short = n.split("(")[0].replace("void ", "").replace("mecefo::", "")
    if "<" in n and "gemm" in short:
        short = short + n[n.find("<"):n.find(">") + 1] if "<" not in short else short
    us = float(r["Metric Value"]) / 1e3
    tot += us
    print(f"{r['ID']:>5s} {us:9.2f} {short[:60]:60s} grid={r.get('Grid Size', '')}")
print("total us", round(tot, 1))
