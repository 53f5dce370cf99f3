"""Reference top-r right singular bases at C1 (LLaMA-60M) init weights.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_svd_golden.py

Runs the REFERENCE's linalg.top_r_right_singular_vectors (linalg.py:97-142)
with the harness's SvdConfig(rank=r, tolerance=1e-9, max_iterations=3000,
seed=run.seed + 23) (harness.py:367) on layer 0's gate / up / down matrices of
init_weights(C1, seed=0), r = 128 (approx.py:79: min(r, in)). Writes
tests/golden/c1_svd_l0.npz (float32 bases) and c1_svd_l0.json (iterations the
reference needed, wall time). tests/test_refresh_gpu.py compares the device
refresh against these by projector distance.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from faultsim import linalg, model as mdl  # noqa: E402
from faultsim.linalg import SvdConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
C1 = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=8, seq_len=256, rope=True)


class _Count:
    """Counts the reference's QR calls (one per iteration, linalg.py:121)."""

    def __init__(self):
        self.n = 0
        self._qr = np.linalg.qr

    def __call__(self, a, *args, **kw):
        self.n += 1
        return self._qr(a, *args, **kw)


def main():
    w = mdl.init_weights(C1, seed=0)
    lw = w.layers[0]
    out, meta = {}, {}
    for kind in ("gate", "up", "down"):
        mat = lw.kind(kind)
        cfg = SvdConfig(rank=min(128, mat.shape[1]), tolerance=1e-9, max_iterations=3000, seed=23)
        cnt = _Count()
        np.linalg.qr = cnt
        t0 = time.perf_counter()
        try:
            v1 = linalg.top_r_right_singular_vectors(mat, cfg)
        finally:
            np.linalg.qr = cnt._qr
        dt = time.perf_counter() - t0
        out[f"v1.{kind}"] = v1.astype(np.float32)
        meta[kind] = {"shape": list(mat.shape), "rank": cfg.rank, "iterations": cnt.n - 1, "seconds": round(dt, 2)}
        print(kind, meta[kind], flush=True)
    np.savez_compressed(os.path.join(OUT, "c1_svd_l0.npz"), **out)
    with open(os.path.join(OUT, "c1_svd_l0.json"), "w") as f:
        json.dump({"config": "C1 layer 0, init_weights seed 0, SvdConfig(r, 1e-9, 3000, seed 23)", "kinds": meta}, f,
                  indent=1)


if __name__ == "__main__":
    main()
