"""Linear-algebra helpers — mirror of faultsim.linalg (linalg.py:1-142).

* seeded_gaussian: host PCG64 draws, bit-identical to the reference (used for
  weight init and the subspace-iteration start block).
* top_r_right_singular_vectors / refresh_bases: the top-r right singular
  subspace of W to the reference's stopping rule (residual <= tol * theta_max,
  SvdConvergenceError otherwise; linalg.py:97-142), computed entirely on the
  device in float64 (mecefo_refresh_converged: Chebyshev-filtered block
  subspace iteration + Rayleigh-Ritz, all due matrices of a refresh batched;
  csrc/refresh.cu). This is the tau-amortised projection refresh
  (approx.py:66-87).
* top_r_right_singular_vectors_batched: the budgeted fixed-iteration variant
  (30 iterations, the cost model's charge, costmodel.py:41) kept for
  throughput comparisons; it does NOT meet the stopping rule.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import runtime
from .errors import ContractViolation, SvdConvergenceError

__all__ = ["SvdConfig", "check_matrix", "seeded_gaussian", "top_r_right_singular_vectors"]

_OVERSAMPLE = 4  # linalg.py:94 (the minimum; see oversample_for)


def oversample_for(r: int, n: int) -> int:
    """Extra block columns of the converged refresh (Gram dimension n). The
    reference carries 4 (linalg.py:94). A wider block widens the gap the
    filter separates (lambda_r vs lambda_k) and cuts the block products, but
    past k = 132 the device Ritz eigensolve leaves shared memory
    (csrc/refresh.cuh): measured on B200, 4 is fastest for the 512-wide C1
    Grams (61 vs 96 ms per refresh) and 32 for the 2048-wide 1B Grams (0.86 vs
    1.41 s), where the products dominate. Only span(V[:, :r]) is returned, so
    the computed object is unchanged."""
    return _OVERSAMPLE if n <= 1024 else max(_OVERSAMPLE, min(r // 4, 32))


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


_START64: dict = {}


def _start_block64(n: int, k: int, seed: int, device) -> torch.Tensor:
    """QR of the seeded Gaussian start block (linalg.py:117), float64, cached
    per (n, k, seed) — every refresh with the same SvdConfig starts there."""
    key = (n, k, seed, str(device))
    if key not in _START64:
        v, _ = np.linalg.qr(seeded_gaussian(n, k, 0.0, 1.0, seed))
        _START64[key] = torch.from_numpy(np.ascontiguousarray(v)).to(device)
    return _START64[key]


def refresh_bases(ws: list, ranks: list, svd: SvdConfig, oversample: int | None = None, info: list | None = None,
                  want_f64: bool = False):
    """Converged top-r right singular bases of several matrices at once
    (linalg.py:97-142 per matrix, batched like approx.py:66-87 refreshes
    every kind). Returns fp32 (cols, r) CUDA tensors (and fp64 copies with
    want_f64). Raises SvdConvergenceError(residual) if any matrix misses
    svd.tolerance within svd.max_iterations block products. `info`, if
    given, receives one dict per matrix (residual, products, k)."""
    from . import _lib

    if not ws:
        return []
    dev = torch.device("cuda", torch.cuda.current_device())
    jobs = (_lib.RefreshJob * len(ws))()
    keep, outs, outs64 = [], [], []
    for i, (w, r) in enumerate(zip(ws, ranks)):
        if w.ndim != 2:
            raise ContractViolation(f"w must be 2-D, got shape {tuple(w.shape)}")
        wd = torch.as_tensor(w).detach()
        if wd.device != dev or wd.dtype != torch.float32 or wd.stride(1) != 1:
            wd = wd.to(device=dev, dtype=torch.float32).contiguous()
        rows, n = wd.shape
        if not 1 <= r <= n:
            raise ContractViolation(f"rank {r} exceeds the column count of {tuple(wd.shape)}")
        k = min(n, r + (oversample if oversample is not None else oversample_for(r, min(rows, n) if rows >= r + 4 else n)))
        v0 = _start_block64(n, k, svd.seed, dev)
        v1 = torch.empty(n, r, dtype=torch.float32, device=dev)
        v64 = torch.empty(n, r, dtype=torch.float64, device=dev) if want_f64 else None
        jobs[i] = _lib.RefreshJob(wd.data_ptr(), rows, n, wd.stride(0), r, k, v0.data_ptr(), v1.data_ptr(),
                                  v64.data_ptr() if v64 is not None else None, None, 0.0, 0, 0, 0, 0)
        keep += [wd, v0]
        outs.append(v1)
        outs64.append(v64)
    lib = _lib.load()
    nbytes = int(lib.mecefo_refresh_workspace_bytes(jobs, len(ws)))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    rc = lib.mecefo_refresh_converged(None, jobs, len(ws), float(svd.tolerance), int(svd.max_iterations),
                                      scratch.data_ptr(), nbytes, runtime.stream_ptr())
    if info is not None:
        info.extend({"residual": jobs[i].residual, "products": jobs[i].products, "k": jobs[i].k,
                     "converged": bool(jobs[i].converged), "rr_steps": jobs[i].rr_steps,
                     "jacobi_sweeps": jobs[i].jacobi_sweeps} for i in range(len(ws)))
    if rc == 3:
        worst = max(jobs[i].residual for i in range(len(ws)) if not jobs[i].converged)
        raise SvdConvergenceError(
            f"subspace iteration did not converge within {svd.max_iterations} iterations "
            f"(last residual {worst:.3e})", residual=worst)
    _lib.check(rc)
    del keep, scratch
    return (outs, outs64) if want_f64 else outs


def top_r_right_singular_vectors(w: torch.Tensor, cfg: SvdConfig, budgeted: bool = False) -> torch.Tensor:
    """Orthonormal (cols x r) basis of the top-r right singular subspace of w
    (linalg.py:97-142), float32 CUDA tensor. Converged to cfg.tolerance on the
    device (refresh_bases); budgeted=True instead runs exactly
    cfg.max_iterations iterations of the budgeted batched iteration without a
    stopping rule (throughput comparisons only)."""
    if w.ndim != 2:
        raise ContractViolation(f"w must be 2-D, got shape {tuple(w.shape)}")
    cfg.validate_for(w.shape)
    if budgeted:
        return top_r_right_singular_vectors_batched([w], [cfg.rank], cfg.max_iterations, cfg.seed)[0]
    return refresh_bases([w], [cfg.rank], cfg)[0]


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
