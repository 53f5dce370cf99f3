"""Optimizers and the lr schedule — drop-in for faultsim.optim (optim.py:1-117).

`apply_step` runs the fused multi-tensor AdamW kernel over the model's flat
fp32 buffer: one launch updates every non-skipped parameter, its m/v state
and (bf16 mode) the bf16 operand shadow. Step counts are per parameter
(optim.py:83,93), so a parameter skipped by Eq. (1) keeps both its weights
and its bias correction untouched (optim.py:96-103). The synthetic-objective
convergence harness of optim.py:120-224 is out of scope.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, runtime
from .errors import ConfigError, ContractViolation, NumericalFailure

MOMENTUM_SGD = "momentum_sgd"
ADAMW = "adamw"


@dataclass
class OptimConfig:
    """optim.py:24-37."""

    kind: str = ADAMW
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01

    def __post_init__(self):
        if self.kind not in (MOMENTUM_SGD, ADAMW):
            raise ConfigError(f"unknown optimizer {self.kind!r}")
        if not 0.0 <= self.beta1 < 1.0 or not 0.0 <= self.beta2 < 1.0:
            raise ConfigError("betas must be in [0, 1)")


@dataclass
class OptimState:
    """optim.py:40-52: first/second moments live in flat device buffers
    parallel to the model's parameter buffer; `step` is per parameter name."""

    cfg: OptimConfig
    step: dict = field(default_factory=dict)
    m: torch.Tensor | None = None
    v: torch.Tensor | None = None
    _flag: torch.Tensor | None = None

    def ensure_flat(self, total: int, device) -> None:
        if self.m is None or self.m.numel() != total:
            self.m = torch.zeros(total, dtype=torch.float32, device=device)
            self.v = torch.zeros(total, dtype=torch.float32, device=device) if self.cfg.kind == ADAMW else None
            self._flag = torch.zeros(1, dtype=torch.int32, device=device)


def lr_at(step: int, total_steps: int, base_lr: float, floor_fraction: float = 0.1) -> float:
    """optim.py:106-117."""
    if not 0 <= step <= total_steps:
        raise ContractViolation(f"step {step} outside 0..{total_steps}")
    warmup = math.ceil(0.1 * total_steps)
    if step <= warmup:
        return base_lr * (step / warmup) if warmup > 0 else base_lr
    span = total_steps - warmup
    progress = (step - warmup) / span
    floor = floor_fraction * base_lr
    return floor + (base_lr - floor) * 0.5 * (1.0 + math.cos(math.pi * progress))


def adam_segments(weights, state: OptimState, lr_t: float, skip=()) -> tuple[np.ndarray, int, list]:
    """Host side of apply_step: per-parameter bias corrections for the
    parameters that step this iteration. Returns (segments, total numel,
    names); the caller advances the counters of `names`."""
    cfg = state.cfg
    skip = set(skip)
    segs = []
    names = []
    total_numel = 0
    for name, shape, off in weights.layout:
        if name in skip:
            continue
        t = state.step.get(name, 0) + 1
        n = int(np.prod(shape))
        segs.append((off, n, lr_t / (1.0 - cfg.beta1 ** t), 1.0 / (1.0 - cfg.beta2 ** t), lr_t * cfg.weight_decay))
        names.append(name)
        total_numel += n
    arr = np.zeros(len(segs), dtype=[("offset", "<i8"), ("numel", "<i8"), ("step_size", "<f4"), ("inv_bc2", "<f4"),
                                     ("lr_wd", "<f4"), ("pad", "<i4")])
    for k, s in enumerate(segs):
        arr[k] = (*s, 0)
    return arr, total_numel, names


def apply_flat(weights, state: OptimState, flat_grad: torch.Tensor, lr_t: float, skip=(), check: bool = True,
               stream=None) -> None:
    """One optimizer step from a flat fp32 gradient buffer (same layout as
    weights.master). check=True syncs once to raise NumericalFailure on
    non-finite gradients before any update (optim.py:55-57)."""
    if lr_t <= 0:
        raise ContractViolation("learning rate must be > 0")
    state.ensure_flat(weights.total, weights.master.device)
    sp = runtime.stream_ptr(stream)
    if check:
        state._flag.zero_()
        _lib.call("mecefo_nonfinite", flat_grad.data_ptr(), flat_grad.numel(), state._flag.data_ptr(), sp)
        if int(state._flag.item()) != 0:
            raise NumericalFailure("non-finite gradient")
    cfg = state.cfg
    if cfg.kind == MOMENTUM_SGD:
        skip = set(skip)
        for name, shape, off in weights.layout:
            if name in skip:
                continue
            n = int(np.prod(shape))
            mp = state.m.data_ptr() + 4 * off
            _lib.call("mecefo_scale_accumulate", flat_grad.data_ptr() + 4 * off, mp, n, 1.0 - cfg.beta1, cfg.beta1, sp)
            _lib.call("mecefo_scale_accumulate", mp, weights.master.data_ptr() + 4 * off, n, -lr_t, 1.0, sp)
            state.step[name] = state.step.get(name, 0) + 1
        weights.sync_shadow()
        return
    arr, total_numel, names = adam_segments(weights, state, lr_t, skip)
    if len(names) == 0:
        return
    segs = torch.from_numpy(arr.view(np.uint8)).to(weights.master.device, non_blocking=True)
    eng = runtime.engine_for(weights.cfg, weights.precision)
    shadow = weights.shadow.data_ptr() if weights.precision != "fp32" else None
    _lib.call("mecefo_adamw_step", eng.handle, segs.data_ptr(), len(names), total_numel, weights.master.data_ptr(),
              flat_grad.data_ptr(), state.m.data_ptr(), state.v.data_ptr(), shadow, cfg.beta1, cfg.beta2, cfg.eps, sp)
    for name in names:
        state.step[name] = state.step.get(name, 0) + 1


def apply_step(weights, state: OptimState, grads: dict, lr_t: float, skip=()) -> None:
    """optim.py:96-103: one step over named parameters in canonical order;
    names in `skip` keep weights and optimizer state untouched."""
    skip = set(skip)
    flat = torch.zeros(weights.total, dtype=torch.float32, device=weights.master.device)
    for name, _, _ in weights.layout:
        if name in skip:
            continue
        if name not in grads:
            raise ContractViolation(f"missing gradient for {name!r}")
        g = grads[name]
        dst = weights.view(flat, name)  # reference shape (FFN padding stays zero)
        if tuple(g.shape) != tuple(dst.shape):
            raise ContractViolation(f"shape mismatch for {name!r}: {tuple(dst.shape)} vs {tuple(g.shape)}")
        dst.copy_(torch.as_tensor(g).reshape(dst.shape))
    apply_flat(weights, state, flat, lr_t, skip)


def adamw_step(w, state: OptimState, name: str, g, lr_t: float, weights=None) -> None:
    """optim.py:75-93 for one named parameter of `weights`."""
    if weights is None:
        raise ContractViolation("adamw_step needs the owning ModelWeights on the device engine")
    others = [n for n, _, _ in weights.layout if n != name]
    apply_step(weights, state, {name: g}, lr_t, skip=others)
