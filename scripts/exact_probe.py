"""Per-kernel device time of one LLaMA-60M block forward (full cache) + exact
backward at 16384 tokens (the healthy ranks' / fault-free path), from the
engine's launch profiler; median over repetitions. For ncu: --once."""
import ctypes, sys, torch, numpy as np
from collections import defaultdict
from paper_2510_16415_b200 import _lib, model as mdl
cfg = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=1, seq_len=256)
w = mdl.init_weights(cfg, 0, precision="bf16")
x = torch.randn(64 * 256, 512, device="cuda") * 0.5
dy = torch.randn(64 * 256, 512, device="cuda") * 0.01
lib = _lib.load()
once = "--once" in sys.argv
agg = defaultdict(list)
for it in range(2 if once else 25):
    lib.mecefo_profile_enable(0 if once else 1)
    y, cache = mdl.forward_block(cfg, w.layers[0], x, mdl.CACHE_FULL)
    dx, g = mdl.backward_block_exact(cfg, w.layers[0], cache, dy)
    torch.cuda.synchronize()
    if once:
        continue
    per = defaultdict(float)
    for i in range(lib.mecefo_profile_count()):
        tag, ms, fl, by = ctypes.c_char_p(), ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
        lib.mecefo_profile_record(i, ctypes.byref(tag), ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by))
        per[tag.value.decode()] += ms.value
    lib.mecefo_profile_enable(0)
    if it >= 5:
        for k, v in per.items(): agg[k].append(v)
tot = 0.0
for k, v in sorted(agg.items(), key=lambda kv: -np.median(kv[1])):
    med = np.median(v) * 1000
    tot += med
    print(f"{k:34s} {med:8.1f} us")
print(f"{'TOTAL':34s} {tot:8.1f} us")
