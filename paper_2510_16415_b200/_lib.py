"""ctypes binding of the C-ABI in include/mecefo.h (libmecefo.so).

The shared library is the product: there is no Python or CPU fallback. If the
library is missing or cannot be loaded, every entry point raises
`EngineUnavailable` (a RuntimeError) instead of computing anything.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_size_t, c_void_p

from . import errors

LIB_NAME = "libmecefo.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

MECEFO_OK = 0
PREC_F32 = 0
PREC_BF16 = 1
CACHE_FULL = 0
CACHE_FFN_INPUT_ONLY = 1
FWD_H1_READY = 1  # mecefo_forward_block_chained flags
STATUS_BAD_TOKEN = 1
STATUS_BAD_TARGET = 2
STATUS_NONFINITE_GRAD = 4


class EngineUnavailable(RuntimeError):
    """libmecefo.so is missing or unusable; the engine has no fallback path."""


class Dims(ctypes.Structure):
    _fields_ = [
        ("vocab", c_int64),
        ("hidden", c_int64),
        ("heads", c_int64),
        ("ffn", c_int64),
        ("layers", c_int64),
        ("seq_len", c_int64),
        ("rope", c_int32),
        ("precision", c_int32),
    ]


class LayerWeights(ctypes.Structure):
    _fields_ = [
        ("w_qkv", c_void_p),
        ("w_o", c_void_p),
        ("norm_mha", c_void_p),
        ("w_gu", c_void_p),
        ("w_down", c_void_p),
        ("norm_ffn", c_void_p),
        ("w_qkv_c", c_void_p),
        ("w_o_c", c_void_p),
        ("w_gu_c", c_void_p),
        ("w_down_c", c_void_p),
    ]


class BlockCache(ctypes.Structure):
    _fields_ = [
        ("x", c_void_p),
        ("x1", c_void_p),
        ("h1", c_void_p),
        ("inv1", c_void_p),
        ("qkv", c_void_p),
        ("ctx", c_void_p),
        ("lse", c_void_p),
        ("h2", c_void_p),
        ("inv2", c_void_p),
        ("gu", c_void_p),
        ("act", c_void_p),
    ]


class LayerGrads(ctypes.Structure):
    _fields_ = [
        ("qkv", c_void_p),
        ("o", c_void_p),
        ("norm_mha", c_void_p),
        ("alpha_mha", c_float),
        ("gu", c_void_p),
        ("down", c_void_p),
        ("norm_ffn", c_void_p),
        ("alpha_ffn", c_float),
    ]


class Projection(ctypes.Structure):
    _fields_ = [
        ("rank", c_int32 * 3),
        ("rank_pad", c_int32),
        ("v1", c_void_p * 3),
        ("v1t", c_void_p * 3),
        ("v1_gu", c_void_p),
        ("v1t_gu", c_void_p),
    ]


class AdamSegment(ctypes.Structure):
    _fields_ = [
        ("offset", c_int64),
        ("numel", c_int64),
        ("step_size", c_float),
        ("inv_bc2", c_float),
        ("lr_wd", c_float),
        ("pad", c_int32),
    ]


class SubspaceJob(ctypes.Structure):
    _fields_ = [
        ("w", c_void_p),
        ("rows", c_int64),
        ("cols", c_int64),
        ("ldw", c_int64),
        ("k", c_int32),
        ("r", c_int32),
        ("v", c_void_p),
        ("v1", c_void_p),
        ("theta", c_void_p),
    ]


class RefreshJob(ctypes.Structure):
    _fields_ = [
        ("w", c_void_p),
        ("rows", c_int64),
        ("cols", c_int64),
        ("ldw", c_int64),
        ("r", c_int32),
        ("k", c_int32),
        ("v0", c_void_p),
        ("v1", c_void_p),
        ("v1_f64", c_void_p),
        ("theta", c_void_p),
        ("residual", ctypes.c_double),
        ("products", c_int32),
        ("converged", c_int32),
        ("rr_steps", c_int32),
        ("jacobi_sweeps", c_int32),
    ]


class FfnSaved(ctypes.Structure):
    _fields_ = [("h2", c_void_p), ("act", c_void_p), ("dcat", c_void_p)]


class LowrankJob(ctypes.Structure):
    _fields_ = [
        ("dy_c", c_void_p),
        ("saved", FfnSaved),
        ("proj", POINTER(Projection)),
        ("grad_gu", c_void_p),
        ("grad_down", c_void_p),
        ("alpha", c_float),
    ]


# name -> (restype, argtypes)
_SIGNATURES = {
    "mecefo_last_error": (c_char_p, []),
    "mecefo_version": (c_char_p, []),
    "mecefo_launch_count": (c_int64, []),
    "mecefo_padded_ffn": (c_int64, [c_int64]),
    "mecefo_engine_create": (c_int, [POINTER(c_void_p), POINTER(Dims)]),
    "mecefo_engine_destroy": (c_int, [c_void_p]),
    "mecefo_workspace_bytes": (c_size_t, [c_void_p, c_int64, c_int32]),
    "mecefo_status_device": (c_int, [c_void_p, POINTER(c_void_p)]),
    "mecefo_status_reset": (c_int, [c_void_p, c_void_p]),
    "mecefo_status_snapshot": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mecefo_memset_zero": (c_int, [c_void_p, c_size_t, c_void_p]),
    "mecefo_forward_block": (
        c_int,
        [c_void_p, POINTER(LayerWeights), POINTER(BlockCache), c_void_p, c_void_p, c_int64, c_int32, c_void_p,
         c_size_t, c_void_p],
    ),
    "mecefo_forward_block_chained": (
        c_int,
        [c_void_p, POINTER(LayerWeights), POINTER(BlockCache), c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p,
         c_void_p, c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_backward_block_neighbor": (
        c_int,
        [c_void_p, POINTER(LayerWeights), POINTER(BlockCache), c_void_p, c_void_p, c_void_p, c_void_p,
         POINTER(LayerGrads), POINTER(Projection), c_int64, c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_backward_block_exact": (
        c_int,
        [c_void_p, POINTER(LayerWeights), POINTER(BlockCache), c_void_p, c_void_p, c_void_p, c_void_p,
         POINTER(LayerGrads), c_int64, c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_recompute_ffn": (
        c_int,
        [c_void_p, POINTER(LayerWeights), c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_lowrank_wgrad": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64, c_float, c_void_p,
         c_size_t, c_void_p],
    ),
    "mecefo_embedding_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "mecefo_head_forward_loss": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_head_forward_loss_grouped": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_head_logits": (
        c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "mecefo_cross_entropy": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_size_t, c_void_p]),
    "mecefo_cross_entropy_grouped": (
        c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_head_backward": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         c_void_p, c_float, c_int64, c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_embedding_backward": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_int64, c_void_p]),
    "mecefo_scale_accumulate": (c_int, [c_void_p, c_void_p, c_int64, c_float, c_float, c_void_p]),
    "mecefo_cast": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "mecefo_nonfinite": (c_int, [c_void_p, c_int64, c_void_p, c_void_p]),
    "mecefo_cast_bf16": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "mecefo_widen_bf16": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "mecefo_adamw_step": (
        c_int,
        [c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_float,
         c_float, c_void_p],
    ),
    "mecefo_profile_enable": (c_int, [c_int32]),
    "mecefo_profile_count": (c_int64, []),
    "mecefo_profile_record": (
        c_int, [c_int64, POINTER(c_char_p), POINTER(c_float), POINTER(ctypes.c_double), POINTER(ctypes.c_double)],
    ),
    "mecefo_gemm": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_int32, c_void_p,
         c_int64, c_float, c_float, c_void_p],
    ),
    "mecefo_backward_block_neighbor_main": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
         c_size_t, c_void_p],
    ),
    "mecefo_lowrank_batched_workspace_bytes": (c_size_t, [c_void_p, c_int64, c_int32, c_int32]),
    "mecefo_lowrank_wgrads_batched": (c_int, [c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_size_t, c_void_p]),
    "mecefo_subspace_workspace_bytes": (c_size_t, [c_void_p, c_int32]),
    "mecefo_refresh_workspace_bytes": (c_size_t, [c_void_p, c_int32]),
    "mecefo_refresh_converged": (
        c_int, [c_void_p, c_void_p, c_int32, ctypes.c_double, c_int32, c_void_p, c_size_t, c_void_p],
    ),
    "mecefo_subspace_iteration_batched": (c_int, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_size_t, c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_LIB = None


def load(path: str | None = None):
    """Load libmecefo.so once; raise EngineUnavailable if it cannot be used."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = path or os.environ.get("MECEFO_LIB") or LIB_PATH  # MECEFO_LIB: A/B a second in-tree build
    if not os.path.exists(p):
        raise EngineUnavailable(
            f"{LIB_NAME} not found at {p}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        lib = ctypes.CDLL(p)
    except OSError as exc:  # pragma: no cover - depends on the host
        raise EngineUnavailable(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


_ERROR_CLASSES = {
    1: errors.ContractViolation,
    2: errors.NumericalFailure,
    4: errors.UnrecoverableRankError,
    5: errors.ConsistencyError,
    6: errors.ConfigError,
    7: errors.CudaError,
}


def check(rc: int) -> None:
    """Map a status code to the reference's exception classes (errors.py)."""
    if rc == MECEFO_OK:
        return
    msg = load().mecefo_last_error().decode("utf-8", "replace")
    if rc == 3:
        raise errors.SvdConvergenceError(msg, residual=float("nan"))
    raise _ERROR_CLASSES.get(rc, RuntimeError)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
