"""ctypes binding of include/mecefo_ctl.h (libmecefo_ctl.so): the native PCG64
streams of the host control plane.

`Pcg64Generator(seed)` / `Pcg64Generator((seed, a, i))` draw the same values as
`np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))` for the
calls the degraded-step control plane makes (reference
pkg/src/faultsim/cluster.py:98,149,164; data.py:96,104): `random()` and
`integers(low, high, size)`; plus the ring-successor takeover
(`ring_route`, cluster.py:207-218). There is no numpy fallback: a missing library
raises `EngineUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_size_t, c_uint32, c_uint64

import numpy as np

from . import errors
from ._lib import EngineUnavailable

LIB_NAME = "libmecefo_ctl.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

SYMBOLS = {
    "mecefo_pcg64_seed": [ctypes.c_void_p, POINTER(c_uint64), c_int32],
    "mecefo_pcg64_next_u64": [ctypes.c_void_p, POINTER(c_uint64), c_size_t],
    "mecefo_pcg64_next_u32": [ctypes.c_void_p, POINTER(c_uint32), c_size_t],
    "mecefo_pcg64_random": [ctypes.c_void_p, POINTER(c_double), c_size_t],
    "mecefo_pcg64_integers": [ctypes.c_void_p, c_int64, c_int64, POINTER(c_int64), c_size_t],
    "mecefo_ring_route": [c_int32, POINTER(ctypes.c_uint8), POINTER(c_int32)],
    "mecefo_cluster_create": [POINTER(ctypes.c_void_p), ctypes.c_void_p],
    "mecefo_cluster_destroy": [ctypes.c_void_p],
    "mecefo_cluster_arrays": [ctypes.c_void_p, POINTER(ctypes.c_void_p), POINTER(ctypes.c_void_p)],
    "mecefo_cluster_rng": [ctypes.c_void_p, POINTER(ctypes.c_void_p)],
    "mecefo_cluster_next_failure_time": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    "mecefo_cluster_down_until": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, c_int32, POINTER(c_int32)],
    "mecefo_cluster_set_down_until": [ctypes.c_void_p, c_int32, c_int32, ctypes.c_void_p],
    "mecefo_cluster_inject": [ctypes.c_void_p, c_double, c_int32, ctypes.c_void_p, c_int32, POINTER(c_int32)],
    "mecefo_cluster_due_recoveries": [ctypes.c_void_p, c_double, c_int32, ctypes.c_void_p, c_int32,
                                      POINTER(c_int32)],
    "mecefo_cluster_recover": [ctypes.c_void_p, c_int32, c_int32, c_double, c_int32, ctypes.c_void_p, c_int32,
                               POINTER(c_int32)],
    "mecefo_cluster_reassign": [ctypes.c_void_p, c_double, c_int32, ctypes.c_void_p, c_int32, POINTER(c_int32)],
    "mecefo_cluster_validate": [ctypes.c_void_p],
    "mecefo_cluster_step": [ctypes.c_void_p, c_double, c_int32, ctypes.c_void_p, c_int32, POINTER(c_int32)],
    "mecefo_iteration_cost": [ctypes.c_void_p, c_int64, c_int64, c_int32, c_int64, c_int64, c_int64,
                              POINTER(c_int64), POINTER(c_int32), POINTER(c_int64)],
}
MECEFO_CTL_UNRECOVERABLE = 2


class ClusterConfigC(ctypes.Structure):
    _fields_ = [("dp", c_int32), ("pp", c_int32), ("layers", c_int32), ("stage_boundaries", ctypes.c_void_p),
                ("kind", c_int32), ("probability", c_double), ("recovery_iterations", c_int32),
                ("failure_interval_s", c_double), ("recovery_time_s", c_double), ("victims", ctypes.c_void_p),
                ("n_victims", c_int32), ("seed", c_uint64)]


class ClusterEventC(ctypes.Structure):
    _fields_ = [("time", c_double), ("iteration", c_int32), ("kind", c_int32), ("node_rank", c_int32),
                ("node_stage", c_int32), ("stage", c_int32), ("from_rank", c_int32), ("from_stage", c_int32)]


class _State(ctypes.Structure):
    _fields_ = [("state_hi", c_uint64), ("state_lo", c_uint64), ("inc_hi", c_uint64), ("inc_lo", c_uint64),
                ("has_uint32", c_int32), ("uinteger", c_uint32)]


_LIB = None


def load():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise EngineUnavailable(f"{LIB_NAME} not built (run python -m paper_2510_16415_b200.build)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, argtypes in SYMBOLS.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = c_int32
        _LIB = lib
    return _LIB


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise errors.ContractViolation(f"{what}: invalid arguments")


def _entropy_words(entropy) -> list:
    ints = [entropy] if isinstance(entropy, (int, np.integer)) else list(entropy)
    out = []
    for v in ints:
        v = int(v)
        if v < 0 or v >= 1 << 64:
            raise errors.ContractViolation(f"seed entropy {v} outside [0, 2**64)")
        out.append(v)
    return out


class Pcg64Generator:
    """Generator(PCG64(SeedSequence(entropy))) restricted to the control
    plane's draws; copy.copy forks the stream."""

    def __init__(self, entropy):
        words = _entropy_words(entropy)
        self._s = _State()
        arr = (c_uint64 * len(words))(*words)
        _check(load().mecefo_pcg64_seed(ctypes.byref(self._s), arr, len(words)), "mecefo_pcg64_seed")

    def __copy__(self):
        g = Pcg64Generator.__new__(Pcg64Generator)
        g._s = _State()
        ctypes.pointer(g._s)[0] = self._s
        return g

    def __deepcopy__(self, memo):
        return self.__copy__()

    @property
    def state(self) -> dict:
        """Same layout as numpy's PCG64.state['state'] / has_uint32 / uinteger."""
        s = self._s
        return {"state": (s.state_hi << 64) | s.state_lo, "inc": (s.inc_hi << 64) | s.inc_lo,
                "has_uint32": int(s.has_uint32), "uinteger": int(s.uinteger)}

    def random(self, size=None):
        n = 1 if size is None else int(np.prod(size))
        out = np.empty(n, dtype=np.float64)
        _check(load().mecefo_pcg64_random(ctypes.byref(self._s), out.ctypes.data_as(POINTER(c_double)), n),
               "mecefo_pcg64_random")
        return float(out[0]) if size is None else out.reshape(size)

    def integers(self, low, high=None, size=None):
        if high is None:
            low, high = 0, low
        n = 1 if size is None else int(np.prod(size))
        out = np.empty(n, dtype=np.int64)
        _check(load().mecefo_pcg64_integers(ctypes.byref(self._s), int(low), int(high),
                                            out.ctypes.data_as(POINTER(c_int64)), n), "mecefo_pcg64_integers")
        return np.int64(out[0]) if size is None else out.reshape(size)

    def next_uint64(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        _check(load().mecefo_pcg64_next_u64(ctypes.byref(self._s), out.ctypes.data_as(POINTER(c_uint64)), n),
               "mecefo_pcg64_next_u64")
        return out

    def next_uint32(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        _check(load().mecefo_pcg64_next_u32(ctypes.byref(self._s), out.ctypes.data_as(POINTER(c_uint32)), n),
               "mecefo_pcg64_next_u32")
        return out



def ring_route(n: int, failed) -> list | None:
    """mecefo_ring_route: executor list, or None when unrecoverable."""
    if n < 1:
        raise errors.ContractViolation(f"ring of {n} members")
    mask = np.zeros(n, dtype=np.uint8)
    for s in failed:
        mask[int(s)] = 1
    ex = np.empty(n, dtype=np.int32)
    rc = load().mecefo_ring_route(n, mask.ctypes.data_as(POINTER(ctypes.c_uint8)), ex.ctypes.data_as(POINTER(c_int32)))
    if rc == MECEFO_CTL_UNRECOVERABLE:
        return None
    _check(rc, "mecefo_ring_route")
    return [int(v) for v in ex]
