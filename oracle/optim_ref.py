"""ORACLE (test infrastructure only): AdamW, apply_step with skips, lr schedule.

optim.py:24-31 (defaults), :75-93 (adamw_step, per-parameter step count),
:96-103 (apply_step in canonical order, skip list), :106-117 (lr_at).
"""

from __future__ import annotations

import math

import numpy as np


class Adam:
    def __init__(self, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01):
        self.b1, self.b2, self.eps, self.wd = b1, b2, eps, wd
        self.m: dict[str, np.ndarray] = {}
        self.v: dict[str, np.ndarray] = {}
        self.t: dict[str, int] = {}

    def update(self, name, w, g, lr):
        if not np.isfinite(g).all():
            raise FloatingPointError(f"non-finite gradient for {name!r}")
        m = self.m.setdefault(name, np.zeros_like(w))
        v = self.v.setdefault(name, np.zeros_like(w))
        t = self.t.get(name, 0) + 1
        m[...] = self.b1 * m + (1 - self.b1) * g
        v[...] = self.b2 * v + (1 - self.b2) * g * g
        mh = m / (1 - self.b1 ** t)
        vh = v / (1 - self.b2 ** t)
        w -= lr * (mh / (np.sqrt(vh) + self.eps) + self.wd * w)
        self.t[name] = t

    def apply(self, params: dict, grads: dict, lr: float, skip=()):
        skip = set(skip)
        for name, w in params.items():
            if name not in skip:
                self.update(name, w, grads[name], lr)


def lr_at(step: int, total: int, base: float, floor_fraction: float = 0.1) -> float:
    warm = math.ceil(0.1 * total)
    if step <= warm:
        return base * (step / warm) if warm > 0 else base
    prog = (step - warm) / (total - warm)
    lo = floor_fraction * base
    return lo + (base - lo) * 0.5 * (1.0 + math.cos(math.pi * prog))
