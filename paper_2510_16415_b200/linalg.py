"""Linear-algebra helpers — mirror of faultsim.linalg (linalg.py:1-142).

* seeded_gaussian: host PCG64 draws, bit-identical to the reference (used for
  weight init and the subspace-iteration start block).
* top_r_right_singular_vectors: the reference's block power iteration on
  W^T W (oversample 4, QR, Rayleigh-Ritz, relative-residual stop). The two
  large products per iteration (W^T W once, then B V) run on the engine's
  fp32 GEMM; the k x k factorizations (k = r + 4) run in host float64, as in
  the reference. This is the tau-amortised projection refresh
  (approx.py:66-87), not part of the per-step hot path; SURVEY.md §8(f) row 3
  lists a fully on-device refresh as the next step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import runtime
from .errors import ContractViolation, SvdConvergenceError

__all__ = ["SvdConfig", "check_matrix", "seeded_gaussian", "top_r_right_singular_vectors"]

# fp32 device products bound the attainable relative residual; tolerances
# tighter than this are clamped (the reference runs in float64).
FP32_RESIDUAL_FLOOR = 2e-6
_OVERSAMPLE = 4  # linalg.py:94


def seeded_gaussian(rows: int, cols: int, mean: float = 0.0, stddev: float = 1.0, seed: int = 0) -> np.ndarray:
    """linalg.py:46-62 (host draw; same stream as the reference)."""
    if rows < 1 or cols < 1:
        raise ContractViolation(f"rows/cols must be >= 1, got {rows}x{cols}")
    if stddev < 0:
        raise ContractViolation(f"stddev must be >= 0, got {stddev}")
    return np.random.Generator(np.random.PCG64(seed)).normal(mean, stddev, size=(rows, cols))


@dataclass(frozen=True)
class SvdConfig:
    """linalg.py:65-88."""

    rank: int
    tolerance: float = 1e-12
    max_iterations: int = 2000
    seed: int = 0

    def __post_init__(self):
        if self.rank < 1:
            raise ContractViolation(f"rank must be >= 1, got {self.rank}")
        if self.tolerance <= 0:
            raise ContractViolation("tolerance must be > 0")
        if self.max_iterations < 1:
            raise ContractViolation("max_iterations must be >= 1")

    def validate_for(self, shape) -> None:
        if self.rank > shape[1]:
            raise ContractViolation(f"rank {self.rank} exceeds the column count of {tuple(shape)}")


def check_matrix(a: torch.Tensor, name: str = "matrix") -> torch.Tensor:
    """linalg.py:25-32 on device: 2-D and finite (one device reduction)."""
    if a.ndim != 2:
        raise ContractViolation(f"{name} must be 2-D, got shape {tuple(a.shape)}")
    if not bool(torch.isfinite(a).all()):
        raise ContractViolation(f"{name} contains non-finite entries")
    return a


def _fp32_engine():
    key = runtime.EngineKey(vocab=8, hidden=8, heads=1, ffn=8, layers=1, seq_len=1, rope=False, precision="fp32")
    eng = runtime._ENGINES.get(key)
    if eng is None:
        eng = runtime.Engine(key)
        runtime._ENGINES[key] = eng
    return eng


def top_r_right_singular_vectors(w: torch.Tensor, cfg: SvdConfig, budgeted: bool = False) -> torch.Tensor:
    """Orthonormal (cols x r) basis of the top-r right singular subspace of w
    (linalg.py:97-142). Returns a float32 CUDA tensor.

    budgeted=True stops after cfg.max_iterations without raising (used for
    throughput runs, where the basis quality does not affect timing)."""
    if w.ndim != 2:
        raise ContractViolation(f"w must be 2-D, got shape {tuple(w.shape)}")
    cfg.validate_for(w.shape)
    n = w.shape[1]
    r = cfg.rank
    eng = _fp32_engine()
    wd = w.detach().to(device="cuda", dtype=torch.float32).contiguous()
    check_matrix(wd, "w")
    B = torch.empty(n, n, dtype=torch.float32, device=wd.device)
    # B = W^T W: A(i, k) = W[k, i] and B(j, k) = W[k, j], both MN-major.
    runtime.gemm(eng, wd, False, wd, False, n, n, wd.shape[0], B)
    scale = float(torch.linalg.matrix_norm(B.double()).item())
    if scale == 0.0:
        return torch.eye(n, device=wd.device)[:, :r].contiguous()
    k = min(n, r + _OVERSAMPLE)
    tol = max(cfg.tolerance, FP32_RESIDUAL_FLOOR)
    V, _ = np.linalg.qr(seeded_gaussian(n, k, 0.0, 1.0, cfg.seed))
    Vd = torch.empty(n, k, dtype=torch.float32, device=wd.device)
    Zd = torch.empty(n, k, dtype=torch.float32, device=wd.device)
    last = np.inf
    for _ in range(cfg.max_iterations):
        Vd.copy_(torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)))
        # Z = B V: A = B (K-major, symmetric), B-operand(n=j, k) = V[k, j] MN-major
        runtime.gemm(eng, B, True, Vd, False, n, k, n, Zd)
        V, _ = np.linalg.qr(Zd.double().cpu().numpy())
        Vd.copy_(torch.from_numpy(np.ascontiguousarray(V, dtype=np.float32)))
        runtime.gemm(eng, B, True, Vd, False, n, k, n, Zd)
        BV = Zd.double().cpu().numpy()
        small = V.T @ BV
        theta, s = np.linalg.eigh(0.5 * (small + small.T))
        order = np.argsort(theta)[::-1]
        theta = theta[order]
        V = V @ s[:, order]
        top = V[:, :r]
        resid = BV @ s[:, order][:, :r] - top * theta[:r]
        last = float(np.max(np.linalg.norm(resid, axis=0)) / max(theta[0], np.finfo(float).tiny))
        if last <= tol:
            return torch.from_numpy(np.ascontiguousarray(top)).to(wd.device, torch.float32)
    if budgeted:
        return torch.from_numpy(np.ascontiguousarray(V[:, :r])).to(wd.device, torch.float32)
    raise SvdConvergenceError(
        f"subspace iteration did not converge within {cfg.max_iterations} iterations (last residual {last:.3e})",
        residual=last,
    )
