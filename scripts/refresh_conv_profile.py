"""Converged batched refresh of every layer's gate/up/down (C1 LLaMA-60M by
default; argv[1] in 60M/350M/1B), r=128, tol 1e-9: wall time and device
time per kernel tag."""
import ctypes, sys, time, torch
from collections import defaultdict
from paper_2510_16415_b200 import _lib, linalg, model as mdl
DIMS = {"60M": (512, 1376, 8, 8), "350M": (1024, 2736, 16, 24), "1B": (2048, 5461, 32, 24)}
m_, f_, H_, L_ = DIMS[sys.argv[1] if len(sys.argv) > 1 else "60M"]
cfg = mdl.ModelConfig(vocab=32000, hidden=m_, heads=H_, ffn_intermediate=f_, layers=L_, seq_len=256)
w = mdl.init_weights(cfg, 0, precision="bf16")
ws, ranks = [], []
for lw in w.layers:
    for k in ("gate", "up", "down"):
        m = lw.kind(k); ws.append(m); ranks.append(min(128, m.shape[1]))
svd = linalg.SvdConfig(rank=128, tolerance=1e-9, max_iterations=3000, seed=23)
linalg.refresh_bases(ws, ranks, svd); torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter(); info = []
    linalg.refresh_bases(ws, ranks, svd, info=info); torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("wall ms", [round(x, 2) for x in ts], "products", max(i["products"] for i in info),
      "rr_steps", max(i["rr_steps"] for i in info), "jacobi_sweeps", max(i["jacobi_sweeps"] for i in info))
lib = _lib.load()
lib.mecefo_profile_enable(1)
linalg.refresh_bases(ws, ranks, svd); torch.cuda.synchronize()
agg = defaultdict(lambda: [0.0, 0])
fl_ = defaultdict(float)
for i in range(lib.mecefo_profile_count()):
    tag, ms, fl, by = ctypes.c_char_p(), ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
    lib.mecefo_profile_record(i, ctypes.byref(tag), ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by))
    agg[tag.value.decode()][0] += ms.value; agg[tag.value.decode()][1] += 1; fl_[tag.value.decode()] += fl.value
lib.mecefo_profile_enable(0)
tot = sum(v[0] for v in agg.values())
print(f"device total {tot:.2f} ms")
for k, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:24s} {ms:8.3f} ms  {n} launches  {fl_[k] / (ms / 1e3) / 1e12 if ms else 0:.2f} TFLOP/s")
