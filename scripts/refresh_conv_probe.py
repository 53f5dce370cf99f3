"""Converged device refresh at bench scale: every lean layer's gate/up/down of
a model (one batched solve) at several oversamples; time, products,
residuals, and the per-phase device time of the default setting."""
import ctypes
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_16415_b200 import _lib, model as mdl  # noqa: E402
from paper_2510_16415_b200.linalg import SvdConfig, refresh_bases  # noqa: E402

DIMS = {"60M": (512, 1376, 8, 8), "130M": (768, 2048, 12, 12), "350M": (1024, 2736, 16, 24),
        "1B": (2048, 5472, 32, 24)}


def profile(fn):
    lib = _lib.load()
    lib.mecefo_profile_enable(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    agg = {}
    for i in range(lib.mecefo_profile_count()):
        tag, kms, fl, by = ctypes.c_char_p(), ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
        _lib.check(lib.mecefo_profile_record(i, ctypes.byref(tag), ctypes.byref(kms), ctypes.byref(fl),
                                             ctypes.byref(by)))
        a = agg.setdefault(tag.value.decode(), [0.0, 0, 0.0])
        a[0] += kms.value
        a[1] += 1
        a[2] += fl.value
    lib.mecefo_profile_enable(0)
    return {"wall_ms": round(1000 * wall, 2),
            "phases": {k: {"ms": round(v[0], 3), "n": v[1],
                           "tflops": round(v[2] / (v[0] / 1e3) / 1e12, 2) if v[2] else None}
                       for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])}}


for name in sys.argv[1:] or ["60M"]:
    m, f, H, L = DIMS[name]
    r = 128
    cfg = mdl.ModelConfig(vocab=32000, hidden=m, heads=H, ffn_intermediate=f, layers=L, seq_len=256)
    w = mdl.init_weights(cfg, 0, precision="bf16")
    mats = [w.layers[l].kind(k) for l in range(L) for k in ("gate", "up", "down")]
    svd = SvdConfig(rank=r, tolerance=1e-9, max_iterations=3000, seed=23)
    for os_ in (4, 16, 32):
        for rep in range(2):
            info = []
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            refresh_bases(mats, [r] * len(mats), svd, info=info, oversample=os_)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        sw = [i["jacobi_sweeps"] / max(1, i["rr_steps"]) for i in info]
        print(json.dumps({"model": name, "oversample": os_, "matrices": len(mats), "seconds": round(dt, 4),
                          "products_max": max(i["products"] for i in info),
                          "products_mean": sum(i["products"] for i in info) / len(info),
                          "residual_max": max(i["residual"] for i in info), "rr_steps_max": max(i["rr_steps"] for i in info), "sweeps_per_rr_mean": sum(sw) / len(sw)}), flush=True)
    print(json.dumps(profile(lambda: refresh_bases(mats, [r] * len(mats), svd, oversample=4))), flush=True)
