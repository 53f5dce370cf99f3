"""Cluster control plane — drop-in for faultsim.cluster (cluster.py:1-322).

Host-side, replicated identically in every rank process (so skip lists and
active sets need no communication). The state machine is native C++
(libmecefo_ctl.so, include/mecefo_ctl.h: mecefo_cluster_*): the small
integer arrays `_st[i, s]` (0 healthy, 1 failed, 2 doubled) and `_ex[i, s]`
(executing stage within DP rank i) are numpy views of its memory;
`status` / `executor` expose the reference's dict-of-tuples view. Integer semantics (draw order, recovery-before-
injection, descending-failed NDB takeover with cascading) are bit-exact with
the reference and tested against its logs (tests/test_cluster_product.py).

Two placements share this module:
  * reference-native (Flavour A): ClusterConfig(dp, pp, layers) verbatim;
  * DP ring (Flavour B): R logical DP ranks on a ring of GPUs is
    ClusterConfig(dp=1, pp=R, layers=R); `ring_route` gives microbatch -> GPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .errors import ConfigError, ConsistencyError, ContractViolation, UnrecoverableRankError
from . import pcg as _pcg
from .pcg import Pcg64Generator

HEALTHY = "healthy"
FAILED = "failed"
DOUBLED = "doubled"
_NAMES = (HEALTHY, FAILED, DOUBLED)
_CODE = {HEALTHY: 0, FAILED: 1, DOUBLED: 2}

SCENARIO_NONE = "none"
SCENARIO_PER_ITERATION = "per_iteration"
SCENARIO_SCHEDULED = "scheduled"

MHA_GRAD_KINDS = ("q", "k", "v", "o", "norm_mha")
FFN_GRAD_KINDS = ("gate", "up", "down", "norm_ffn")
GLOBAL_GRAD_NAMES = ("embedding", "final_norm", "unembedding")


@dataclass(frozen=True)
class ClusterConfig:
    """cluster.py:37-66."""

    dp: int
    pp: int
    layers: int
    stage_boundaries: tuple | None = None

    def __post_init__(self):
        if self.dp < 1 or self.pp < 1:
            raise ConfigError("dp and pp must be >= 1")
        if self.layers < self.pp:
            raise ConfigError("need at least one layer per stage")
        if self.stage_boundaries is not None and len(self.stage_boundaries) != self.pp + 1:
            raise ConfigError("stage_boundaries must have pp+1 entries")

    def boundaries(self) -> tuple:
        if self.stage_boundaries is not None:
            return tuple(self.stage_boundaries)
        return tuple(round(s * self.layers / self.pp) for s in range(self.pp + 1))

    def stage_of_layer(self, layer: int) -> int:
        b = self.boundaries()
        idx = int(np.searchsorted(np.asarray(b[1:]), layer, side="right"))
        if not (0 <= layer < self.layers) or idx >= self.pp or not (b[idx] <= layer < b[idx + 1]):
            raise ContractViolation(f"layer {layer} outside 0..{self.layers - 1}")
        return idx

    def layers_of_stage(self, stage: int) -> range:
        b = self.boundaries()
        return range(b[stage], b[stage + 1])


@dataclass(frozen=True)
class FailureScenario:
    """cluster.py:69-89."""

    kind: str = SCENARIO_NONE
    probability: float = 0.0
    recovery_iterations: int = 1
    failure_interval_s: float = 1800.0
    recovery_time_s: float = 7200.0
    victims: tuple | None = None
    seed: int = 0

    def __post_init__(self):
        if self.kind not in (SCENARIO_NONE, SCENARIO_PER_ITERATION, SCENARIO_SCHEDULED):
            raise ConfigError(f"unknown scenario kind {self.kind!r}")
        if not 0.0 <= self.probability <= 1.0:
            raise ConfigError("probability must be in [0, 1]")
        if self.kind == SCENARIO_SCHEDULED and (self.failure_interval_s <= 0 or self.recovery_time_s <= 0):
            raise ConfigError("scheduled intervals must be > 0")
        if self.recovery_iterations < 1:
            raise ConfigError("recovery_iterations must be >= 1")


class _StatusView:
    def __init__(self, st):
        self._st = st

    def __getitem__(self, node):
        return _NAMES[self._st[node[0], node[1]]]

    def __setitem__(self, node, value):
        self._st[node[0], node[1]] = _CODE[value]

    def __iter__(self):
        return iter(self.keys())

    def __len__(self):
        return self._st.size

    def keys(self):
        return [(i, s) for i in range(self._st.shape[0]) for s in range(self._st.shape[1])]

    def values(self):
        return [self[n] for n in self.keys()]

    def items(self):
        return [(n, self[n]) for n in self.keys()]


class _ExecutorView:
    def __init__(self, ex):
        self._ex = ex

    def __getitem__(self, node):
        return (node[0], int(self._ex[node[0], node[1]]))

    def __setitem__(self, node, value):
        if value[0] != node[0]:
            raise ConsistencyError(f"stage {node} cannot be executed by foreign rank {value}")
        self._ex[node[0], node[1]] = value[1]

    def __iter__(self):
        return iter([(i, s) for i in range(self._ex.shape[0]) for s in range(self._ex.shape[1])])


class _DownUntil:
    """`ClusterState.down_until` (cluster.py:101): (rank, stage) -> recovery
    deadline, stored in the native state (mutable-mapping view)."""

    def __init__(self, state: "ClusterState"):
        self._s = state

    def _items(self) -> list:
        lib, h = _pcg.load(), self._s._h
        n = ctypes.c_int32()
        lib.mecefo_cluster_down_until(h, None, None, 0, ctypes.byref(n))
        k = n.value
        nodes = np.zeros(2 * max(k, 1), dtype=np.int32)
        until = np.zeros(max(k, 1), dtype=np.float64)
        lib.mecefo_cluster_down_until(h, nodes.ctypes.data, until.ctypes.data, k, ctypes.byref(n))
        return [((int(nodes[2 * j]), int(nodes[2 * j + 1])), float(until[j])) for j in range(k)]

    def __getitem__(self, node):
        for k, v in self._items():
            if k == tuple(node):
                return v
        raise KeyError(node)

    def __setitem__(self, node, value):
        v = ctypes.c_double(float(value))
        if _pcg.load().mecefo_cluster_set_down_until(self._s._h, int(node[0]), int(node[1]), ctypes.byref(v)):
            raise ContractViolation(f"node {tuple(node)} outside the cluster")

    def pop(self, node, *default):
        try:
            v = self[node]
        except KeyError:
            if default:
                return default[0]
            raise
        _pcg.load().mecefo_cluster_set_down_until(self._s._h, int(node[0]), int(node[1]), None)
        return v

    def __contains__(self, node):
        return any(k == tuple(node) for k, _ in self._items())

    def __len__(self):
        return len(self._items())

    def __iter__(self):
        return iter([k for k, _ in self._items()])

    def items(self):
        return self._items()

    def keys(self):
        return [k for k, _ in self._items()]


_KIND_CODE = {SCENARIO_NONE: 0, SCENARIO_PER_ITERATION: 1, SCENARIO_SCHEDULED: 2}


class ClusterState:
    """cluster.py:92-123, held by the native state machine (libmecefo_ctl.so,
    include/mecefo_ctl.h mecefo_cluster_*): `_st` / `_ex` are numpy views of
    its arrays, `down_until` and `next_failure_time` live there, and the
    failure stream is its PCG64(seed) (cluster.py:98)."""

    native = True

    def __init__(self, cfg: ClusterConfig, scenario: FailureScenario):
        self.cfg = cfg
        self.scenario = scenario
        lib = _pcg.load()
        bounds = (ctypes.c_int32 * (cfg.pp + 1))(*cfg.boundaries())
        self._bounds = bounds
        vic = None
        nv = 0
        if scenario.victims is not None:
            flat = [int(x) for v in scenario.victims for x in v]
            vic = (ctypes.c_int32 * max(1, len(flat)))(*flat)
            nv = len(flat) // 2
        self._vic = vic
        conf = _pcg.ClusterConfigC(cfg.dp, cfg.pp, cfg.layers, ctypes.cast(bounds, ctypes.c_void_p),
                                   _KIND_CODE[scenario.kind], float(scenario.probability),
                                   int(scenario.recovery_iterations), float(scenario.failure_interval_s),
                                   float(scenario.recovery_time_s),
                                   ctypes.cast(vic, ctypes.c_void_p) if vic is not None else None, nv,
                                   int(scenario.seed))
        h = ctypes.c_void_p()
        if lib.mecefo_cluster_create(ctypes.byref(h), ctypes.byref(conf)):
            raise ConfigError("invalid cluster configuration")
        self._h = h
        sp, ep = ctypes.c_void_p(), ctypes.c_void_p()
        lib.mecefo_cluster_arrays(h, ctypes.byref(sp), ctypes.byref(ep))
        n = cfg.dp * cfg.pp
        self._st = np.ctypeslib.as_array((ctypes.c_int8 * n).from_address(sp.value)).reshape(cfg.dp, cfg.pp)
        self._ex = np.ctypeslib.as_array((ctypes.c_int32 * n).from_address(ep.value)).reshape(cfg.dp, cfg.pp)
        self.down_until = _DownUntil(self)
        self._victims = None if scenario.victims is None else {tuple(v) for v in scenario.victims}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _pcg.load().mecefo_cluster_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def rng(self) -> Pcg64Generator:
        """The failure stream (a view of the native PCG64 state)."""
        p = ctypes.c_void_p()
        _pcg.load().mecefo_cluster_rng(self._h, ctypes.byref(p))
        g = Pcg64Generator.__new__(Pcg64Generator)
        g._s = _pcg._State.from_address(p.value)
        g._owner = self
        return g

    @property
    def next_failure_time(self) -> float:
        v = ctypes.c_double()
        _pcg.load().mecefo_cluster_next_failure_time(self._h, None, ctypes.byref(v))
        return v.value

    @next_failure_time.setter
    def next_failure_time(self, value: float) -> None:
        v = ctypes.c_double(float(value))
        _pcg.load().mecefo_cluster_next_failure_time(self._h, ctypes.byref(v), None)

    @property
    def status(self):
        return _StatusView(self._st)

    @property
    def executor(self):
        return _ExecutorView(self._ex)

    def nodes(self) -> Iterable:
        return [(i, s) for i in range(self.cfg.dp) for s in range(self.cfg.pp)]

    def healthy_nodes(self) -> list:
        ii, ss = np.nonzero(self._st == 0)
        return [(int(i), int(s)) for i, s in zip(ii, ss)]  # row-major == sorted

    def executing_stages(self, node) -> list:
        i, s = node
        return [int(t) for t in np.nonzero(self._ex[i] == s)[0]]

    def lean_mask(self) -> np.ndarray:
        """(dp, pp) bool: stage's executor is not healthy (harness.py:392-400)."""
        rows = np.arange(self.cfg.dp)[:, None]
        return self._st[rows, self._ex] != 0

    def affected_ranks(self) -> list:
        """cluster.py:115-123."""
        return [int(i) for i in np.nonzero(self.lean_mask().any(axis=1))[0]]


def _event(time, iteration, kind, node, **details) -> dict:
    return {"time": float(time), "iteration": int(iteration), "kind": kind, "node": [int(node[0]), int(node[1])],
            "details": details}


def _native_events(state: ClusterState, fn, *args) -> list:
    """Call a native cluster entry point and convert its event records to the
    reference's event dicts (cluster.py:126-133)."""
    cap = 3 * state.cfg.dp * state.cfg.pp + 16
    buf = (_pcg.ClusterEventC * cap)()
    n = ctypes.c_int32()
    rc = fn(state._h, *args, buf, cap, ctypes.byref(n))
    out = []
    for e in buf[: n.value]:
        node = (e.node_rank, e.node_stage)
        if e.kind == 0:
            out.append(_event(e.time, e.iteration, "fail", node))
        elif e.kind == 1:
            out.append(_event(e.time, e.iteration, "recover", node, fetched_from=[e.from_rank, e.from_stage]))
        else:
            out.append(_event(e.time, e.iteration, "adopt", node, stage=e.stage,
                              layers=list(state.cfg.layers_of_stage(e.stage)), fetched_from_rank=e.from_rank))
    if rc == _pcg.MECEFO_CTL_UNRECOVERABLE:
        failed = {i: sorted(int(s) for s in np.nonzero(state._st[i] == 1)[0]) for i in range(state.cfg.dp)}
        bad = [i for i, f in failed.items() if f and _pcg.ring_route(state.cfg.pp, f) is None]
        i = bad[0] if bad else 0
        raise UnrecoverableRankError(f"DP rank {i}: no eligible adopter for stage (failed stages {failed[i]})")
    if rc == 3:
        raise ConsistencyError("cluster state violates the partition / status invariants")
    if rc:
        raise ContractViolation("invalid control-plane request")
    return out


def inject_failures(state: ClusterState, scenario: FailureScenario, sim_time: float, iteration: int) -> list:
    """cluster.py:136-168 (native). Only healthy (and, if listed, victim)
    nodes draw; `scenario` must be the state's own."""
    if scenario is not state.scenario and scenario != state.scenario:
        raise ContractViolation("inject_failures: scenario differs from the state's")
    return _native_events(state, _pcg.load().mecefo_cluster_inject, float(sim_time), int(iteration))


def due_recoveries(state: ClusterState, sim_time: float, iteration: int) -> list:
    """cluster.py:171-173 (native)."""
    lib = _pcg.load()
    cap = state.cfg.dp * state.cfg.pp
    nodes = np.zeros(2 * max(cap, 1), dtype=np.int32)
    n = ctypes.c_int32()
    lib.mecefo_cluster_due_recoveries(state._h, float(sim_time), int(iteration), nodes.ctypes.data, cap,
                                      ctypes.byref(n))
    return [(int(nodes[2 * j]), int(nodes[2 * j + 1])) for j in range(n.value)]


def recover_node(state: ClusterState, node, sim_time: float, iteration: int) -> list:
    """cluster.py:176-187 (native)."""
    i, s = node
    if not (0 <= i < state.cfg.dp and 0 <= s < state.cfg.pp) or state._st[i, s] != 1:
        raise ContractViolation(f"node {tuple(node)} is not failed")
    return _native_events(state, lambda h, *a: _pcg.load().mecefo_cluster_recover(h, int(i), int(s), *a),
                          float(sim_time), int(iteration))


def ring_route(n: int, failed) -> list | None:
    """Ring-successor takeover on one ring of n members (cluster.py:207-218):
    failed members in descending order each take the first following member
    that is neither failed nor already adopting. Returns executor[j] for every
    member, or None if some failed member has no eligible adopter. Runs in
    the native control library (mecefo_ring_route, libmecefo_ctl.so)."""
    return _pcg.ring_route(n, failed)


def reassign_takeover(state: ClusterState, sim_time: float = 0.0, iteration: int = 0) -> list:
    """cluster.py:190-239 (native): per DP rank, failed stages in descending
    order take the first ring successor that is neither failed nor adopting."""
    return _native_events(state, _pcg.load().mecefo_cluster_reassign, float(sim_time), int(iteration))


def validate_state(state: ClusterState) -> None:
    """cluster.py:253-271 (native): partition and status-coupling invariants."""
    if _pcg.load().mecefo_cluster_validate(state._h):
        raise ConsistencyError("cluster state violates the partition / status invariants")


def step_cluster(state: ClusterState, sim_time: float, iteration: int) -> list:
    """cluster.py:242-250 (native): recoveries, then failures, then
    reassignment, then the invariants — one call into libmecefo_ctl.so."""
    return _native_events(state, _pcg.load().mecefo_cluster_step, float(sim_time), int(iteration))


def active_set(state: ClusterState, layer: int, kind: str) -> list:
    """cluster.py:274-289."""
    if kind in MHA_GRAD_KINDS:
        s = state.cfg.stage_of_layer(layer)
        lean = state.lean_mask()[:, s]
        return [int(i) for i in np.nonzero(~lean)[0]]
    if kind in FFN_GRAD_KINDS:
        return list(range(state.cfg.dp))
    raise ContractViolation(f"unknown per-layer gradient kind {kind!r}")


def aggregate_gradients(per_rank: list, active: dict, layers: int):
    """cluster.py:292-322 on the device: per-rank gradients (torch tensors or
    the reference's numpy arrays) -> fp32 CUDA averages, ascending-rank
    accumulation of g_i / |N|; empty active sets are skipped (excluded ranks
    are never read, so non-finite values there cannot leak); missing
    gradients raise ConsistencyError."""
    import torch

    from . import _lib, runtime

    n = len(per_rank)
    averaged, skipped = {}, []

    def mean_over(name, ranks):
        for i in ranks:
            if name not in per_rank[i]:
                raise ConsistencyError(f"rank {i} is missing gradient {name!r}")
        k = 1.0 / len(ranks)
        grads = [torch.as_tensor(per_rank[i][name]).detach().to("cuda", torch.float32).contiguous() for i in ranks]
        out = torch.zeros_like(grads[0])
        for g in grads:  # ascending rank order; out += g / |N| (never aliased)
            if tuple(g.shape) != tuple(out.shape):
                raise ConsistencyError(f"gradient {name!r} has shape {tuple(g.shape)} on one rank, "
                                       f"{tuple(out.shape)} on another")
            _lib.call("mecefo_scale_accumulate", runtime.ptr(g), runtime.ptr(out), out.numel(), k, 1.0,
                      runtime.stream_ptr())
        return out

    for name in GLOBAL_GRAD_NAMES:
        averaged[name] = mean_over(name, list(range(n)))
    for layer in range(layers):
        for kind in MHA_GRAD_KINDS + FFN_GRAD_KINDS:
            name = f"layers.{layer}.{kind}"
            ranks = active[(layer, kind)]
            if not ranks:
                skipped.append(name)
                continue
            averaged[name] = mean_over(name, ranks)
    return averaged, skipped
