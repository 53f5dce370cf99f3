"""Time the batched projection refresh on the bench model (C1 LLaMA-60M,
8 layers x gate/up/down, r=128) and attribute it per kernel tag."""
import ctypes, time, torch, numpy as np
from collections import defaultdict
from paper_2510_16415_b200 import _lib, linalg, model as mdl
cfg = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=8, seq_len=256)
w = mdl.init_weights(cfg, 0, precision="bf16")
ws, ranks = [], []
for lw in w.layers:
    for k in ("gate", "up", "down"):
        m = lw.kind(k); ws.append(m); ranks.append(min(128, m.shape[1]))
def t(f, n=3):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
for it in (1, 30):
    print("iters", it, "ms", round(t(lambda: linalg.top_r_right_singular_vectors_batched(ws, ranks, it, 23)), 2))
lib = _lib.load()
lib.mecefo_profile_enable(1)
linalg.top_r_right_singular_vectors_batched(ws, ranks, 30, 23); torch.cuda.synchronize()
agg = defaultdict(lambda: [0.0, 0])
for i in range(lib.mecefo_profile_count()):
    tag, ms, fl, by = ctypes.c_char_p(), ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
    lib.mecefo_profile_record(i, ctypes.byref(tag), ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by))
    agg[tag.value.decode()][0] += ms.value; agg[tag.value.decode()][1] += 1
lib.mecefo_profile_enable(0)
for k, (ms, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:24s} {ms:8.3f} ms  {n} launches")
