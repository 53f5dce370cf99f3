"""Per-kernel device time of the LM head (logits, CE, d_xf, g_unemb) at 16384 tokens x 32000 vocab."""
import ctypes, sys, torch, numpy as np
from collections import defaultdict
from paper_2510_16415_b200 import _lib, engine as E, model as mdl
cfg = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=1, seq_len=256)
eng = E.StepEngine(cfg, precision="bf16", seqs_per_microbatch=32, r=128, tau=10**6)
lib = _lib.load()
rng = np.random.Generator(np.random.PCG64(1))
mbs = [E.Microbatch(rank=j, tokens=torch.from_numpy(rng.integers(0, 32000, size=(32, 256))).cuda(),
                    targets=torch.from_numpy(rng.integers(0, 32000, size=(32, 256))).cuda(),
                    lean=[False], alpha_mha=[0.5], alpha_ffn=0.5, alpha_global=0.5) for j in range(2)]
agg = defaultdict(list)
for it in range(12):
    lib.mecefo_profile_enable(1)
    eng._body(mbs, torch.zeros(2, device="cuda"))
    torch.cuda.synchronize()
    per = defaultdict(float)
    for i in range(lib.mecefo_profile_count()):
        tag, ms, fl, by = ctypes.c_char_p(), ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
        lib.mecefo_profile_record(i, ctypes.byref(tag), ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by))
        per[tag.value.decode()] += ms.value
    lib.mecefo_profile_enable(0)
    if it >= 4:
        for k, v in per.items(): agg[k].append(v)
label = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in sorted(agg.items(), key=lambda kv: -np.median(kv[1])):
    if k.startswith("head") or k.startswith("cross"):
        print(f"{label:8s} {k:30s} {np.median(v) * 1000:8.1f} us")
