"""Device runtime around libmecefo.so: engine handles, workspaces, streams.

PyTorch supplies device memory and streams (plumbing); every computation
goes through the C-ABI (`_lib`). Tensors passed to the engine must be CUDA,
contiguous and of the documented dtype; violations raise ContractViolation.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ContractViolation

PRECISIONS = {"fp32": _lib.PREC_F32, "bf16": _lib.PREC_BF16}


def compute_dtype(precision: str) -> torch.dtype:
    return torch.bfloat16 if precision == "bf16" else torch.float32


def ptr(t: torch.Tensor | None) -> int | None:
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ContractViolation("engine tensors must live on a CUDA device")
    return t.data_ptr()


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise _lib.EngineUnavailable("the MeCeFO engine needs a CUDA device (B200, sm_100a); none is visible")
    _lib.load()


@dataclass(frozen=True)
class EngineKey:
    vocab: int
    hidden: int
    heads: int
    ffn: int
    layers: int
    seq_len: int
    rope: bool
    precision: str


class Engine:
    """Owns one mecefo_engine handle and a growable workspace."""

    def __init__(self, key: EngineKey, device: torch.device | None = None):
        require_cuda()
        self.key = key
        self.precision = key.precision
        self.dtype = compute_dtype(key.precision)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        dims = _lib.Dims(key.vocab, key.hidden, key.heads, key.ffn, key.layers, key.seq_len, int(key.rope),
                         PRECISIONS[key.precision])
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.call("mecefo_engine_create", ctypes.byref(handle), ctypes.byref(dims))
        self.handle = handle
        self._ws: torch.Tensor | None = None

    def workspace(self, tokens: int, rank_pad: int = 16) -> tuple[int, int]:
        need = int(_lib.load().mecefo_workspace_bytes(self.handle, tokens, rank_pad))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws.data_ptr(), self._ws.numel()

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.load().mecefo_engine_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_ENGINES: dict[EngineKey, Engine] = {}


def engine_for(cfg, precision: str) -> Engine:
    """Cached engine for a ModelConfig-like object and precision."""
    if precision not in PRECISIONS:
        raise ContractViolation(f"unknown precision {precision!r}")
    key = EngineKey(cfg.vocab, cfg.hidden, cfg.heads, cfg.ffn_intermediate, cfg.layers, cfg.seq_len, bool(cfg.rope),
                    precision)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = Engine(key)
        _ENGINES[key] = eng
    return eng


def gemm(eng: Engine, a: torch.Tensor, a_kmajor: bool, b: torch.Tensor, b_kmajor: bool, M: int, N: int, K: int,
         out: torch.Tensor, alpha: float = 1.0, beta: float = 0.0) -> torch.Tensor:
    """out[M,N] = alpha * A B^T + beta * out on the engine's GEMM path."""
    lda = a.shape[1]
    ldb = b.shape[1]
    _lib.call("mecefo_gemm", eng.handle, M, N, K, ptr(a), lda, int(a_kmajor), ptr(b), ldb, int(b_kmajor), ptr(out),
              out.shape[1], alpha, beta, stream_ptr())
    return out
