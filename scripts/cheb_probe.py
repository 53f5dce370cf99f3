"""Converged refresh under one Chebyshev amplification setting (MECEFO_CHEB,
read at library load by the timing build: run with
MECEFO_LIB=paper_2510_16415_b200/libmecefo_timing.so): wall time, products, RR steps, residuals, and the
projector distance of the bases to a reference solve saved by the first run
(/tmp/cheb_ref_<model>.pt)."""
import json, os, sys, time, torch
sys.path.insert(0, ".")
from paper_2510_16415_b200 import model as mdl
from paper_2510_16415_b200.linalg import SvdConfig, refresh_bases
DIMS = {"60M": (512, 1376, 8, 8), "350M": (1024, 2736, 16, 24), "1B": (2048, 5461, 32, 24)}
name = sys.argv[1]
m, f, H, L = DIMS[name]
cfg = mdl.ModelConfig(vocab=32000, hidden=m, heads=H, ffn_intermediate=f, layers=L, seq_len=256)
w = mdl.init_weights(cfg, 0, precision="bf16")
mats = [w.layers[l].kind(k) for l in range(L) for k in ("gate", "up", "down")]
svd = SvdConfig(rank=128, tolerance=1e-9, max_iterations=3000, seed=23)
refresh_bases(mats, [128] * len(mats), svd)
torch.cuda.synchronize()
t0 = time.perf_counter(); info = []
out = refresh_bases(mats, [128] * len(mats), svd, info=info)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
ref_path = f"/tmp/cheb_ref_{name}.pt"
dist = None
if os.path.exists(ref_path):
    ref = torch.load(ref_path)
    dist = 0.0
    for a, b in zip(out, ref):
        a64, b64 = a.double(), b.double().to(a.device)
        s = torch.linalg.svdvals(a64.T @ b64)
        dist = max(dist, float(torch.sqrt(torch.clamp(1 - s.min() ** 2, min=0))))
else:
    torch.save([o.cpu() for o in out], ref_path)
print(json.dumps({"model": name, "cheb": os.environ.get("MECEFO_CHEB", "default"), "ms": round(1000 * dt, 1),
                  "products_max": max(i["products"] for i in info), "rr_steps_max": max(i["rr_steps"] for i in info),
                  "residual_max": max(i["residual"] for i in info), "all_converged": all(i["converged"] for i in info),
                  "proj_dist_to_default": dist}), flush=True)
