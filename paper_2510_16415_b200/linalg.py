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


_START_CACHE: dict = {}


def _start_block(n: int, k: int, seed: int, device) -> torch.Tensor:
    """Orthonormalised seeded Gaussian start block (linalg.py:117), cached:
    every refresh with the same (n, k, seed) starts from the same block."""
    key = (n, k, seed, str(device))
    if key not in _START_CACHE:
        v, _ = np.linalg.qr(seeded_gaussian(n, k, 0.0, 1.0, seed))
        _START_CACHE[key] = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(device)
    return _START_CACHE[key]


def top_r_right_singular_vectors_batched(ws: list, ranks: list, iterations: int, seed: int,
                                         return_values: bool = False):
    """Budgeted block power iteration for many matrices at once (the
    tau-amortised projection refresh of every due (rank, layer, kind)).

    Same iteration as linalg.py:97-142 — start block linalg.py:117, Z = B V,
    re-orthonormalise, Rayleigh-Ritz (linalg.py:124-129), keep the top r —
    with two changes that keep it entirely on the GPU: QR is CholeskyQR
    (fp32 Gram matrix, fp64 k x k Cholesky and triangular inverse on the
    device) and the Ritz rotation (fp64 Jacobi eigensolve on the device) is
    taken once at the end, since it only rotates within the spanned
    subspace. One launch per phase for ALL matrices, no host round trip
    (mecefo_subspace_iteration_batched). Runs a fixed number of iterations
    (the reference cost model charges SVD_CHARGED_ITERATIONS = 30,
    costmodel.py:41); used for throughput runs. Parity tests inject the
    reference's converged bases."""
    from . import _lib

    if not ws:
        return ([], []) if return_values else []
    eng = _fp32_engine()
    dev = ws[0].device if ws[0].is_cuda else torch.device("cuda")
    jobs = (_lib.SubspaceJob * len(ws))()
    keep, outs, thetas = [], [], []
    for i, (w, r) in enumerate(zip(ws, ranks)):
        wd = w.detach()
        if wd.device != dev or wd.dtype != torch.float32 or wd.stride(1) != 1:
            wd = wd.to(device=dev, dtype=torch.float32).contiguous()
        rows, n = wd.shape
        if not 1 <= r <= n:
            raise ContractViolation(f"rank {r} outside [1, {n}] for shape {tuple(wd.shape)}")
        k = min(n, r + _OVERSAMPLE)
        V = _start_block(n, k, seed, dev).clone()
        v1 = torch.empty(n, r, dtype=torch.float32, device=dev)
        th = torch.empty(r, dtype=torch.float32, device=dev) if return_values else None
        jobs[i] = _lib.SubspaceJob(wd.data_ptr(), rows, n, wd.stride(0), k, r, V.data_ptr(), v1.data_ptr(),
                                   th.data_ptr() if th is not None else None)
        keep += [wd, V]
        outs.append(v1)
        thetas.append(th)
    nbytes = _lib.load().mecefo_subspace_workspace_bytes(jobs, len(ws))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.call("mecefo_subspace_iteration_batched", eng.handle, jobs, len(ws), iterations, scratch.data_ptr(), nbytes,
              runtime.stream_ptr())
    # the caching allocator may hand `scratch`/`keep` to later work on this
    # stream only after the queued kernels, so no synchronisation is needed
    del keep, scratch
    return (outs, thetas) if return_values else outs


def _lib_gemm_into(eng, X, Y, rows, cols, inner, out):
    """out (rows x cols, ld = out.stride(0)) = X^T Y with X (inner x rows), Y (inner x cols)."""
    from . import _lib

    _lib.call("mecefo_gemm", eng.handle, rows, cols, inner, X.data_ptr(), X.shape[1], 0, Y.data_ptr(), Y.shape[1],
              0, out.data_ptr(), out.stride(0), 1.0, 0.0, runtime.stream_ptr())
