"""Per-GEMM device time of one LLaMA-60M block forward + lean neighbour
backward at 16384 tokens (the fused doubled microbatch), from the engine's
launch profiler; median over repetitions."""
import ctypes, sys, torch, numpy as np
from collections import defaultdict
from paper_2510_16415_b200 import _lib, approx, model as mdl
from paper_2510_16415_b200.linalg import SvdConfig
cfg = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=1, seq_len=256)
w = mdl.init_weights(cfg, 0, precision="bf16")
x = torch.randn(64 * 256, 512, device="cuda") * 0.5
dy = torch.randn(64 * 256, 512, device="cuda") * 0.01
proj = approx.ProjectionCache(rank=128, refresh_period=10**9, step=1)
rng = np.random.Generator(np.random.PCG64(9))
for k, n in (("gate", 512), ("up", 512), ("down", 1376)):
    proj.set_basis(k, np.linalg.qr(rng.normal(size=(n, 128)))[0])
lib = _lib.load()
agg = defaultdict(list)
for it in range(25):
    lib.mecefo_profile_enable(1)
    y, cache = mdl.forward_block(cfg, w.layers[0], x, mdl.CACHE_FFN_INPUT_ONLY)
    dx, g = approx.backward_block_neighbor(cfg, w.layers[0], cache, dy, proj=proj, svd=SvdConfig(rank=128))
    torch.cuda.synchronize()
    per = defaultdict(float)
    for i in range(lib.mecefo_profile_count()):
        tag, ms, fl, by = ctypes.c_char_p(), ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
        lib.mecefo_profile_record(i, ctypes.byref(tag), ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by))
        per[tag.value.decode()] += ms.value
    lib.mecefo_profile_enable(0)
    if it >= 5:
        for k, v in per.items(): agg[k].append(v)
label = sys.argv[1] if len(sys.argv) > 1 else ""
tot = 0.0
for k, v in sorted(agg.items(), key=lambda kv: -np.median(kv[1])):
    med = np.median(v) * 1000
    tot += med
    print(f"{label:10s} {k:34s} {med:8.1f} us")
print(f"{label:10s} {'TOTAL':34s} {tot:8.1f} us")
