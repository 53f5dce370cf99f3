"""Cluster control plane — drop-in for faultsim.cluster (cluster.py:1-322).

Host-side, replicated identically in every rank process (so skip lists and
active sets need no communication). State is kept in small integer arrays:
`_st[i, s]` (0 healthy, 1 failed, 2 doubled) and `_ex[i, s]` (executing
stage within DP rank i); `status` / `executor` expose the reference's
dict-of-tuples view. Integer semantics (draw order, recovery-before-
injection, descending-failed NDB takeover with cascading) are bit-exact with
the reference and tested against its logs (tests/test_cluster_product.py).

Two placements share this module:
  * reference-native (Flavour A): ClusterConfig(dp, pp, layers) verbatim;
  * DP ring (Flavour B): R logical DP ranks on a ring of GPUs is
    ClusterConfig(dp=1, pp=R, layers=R); `ring_route` gives microbatch -> GPU.
"""

from __future__ import annotations

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


class ClusterState:
    """cluster.py:92-123."""

    def __init__(self, cfg: ClusterConfig, scenario: FailureScenario):
        self.cfg = cfg
        self.scenario = scenario
        # native PCG64 (libmecefo_ctl.so), draw-for-draw == Generator(PCG64(seed)) of cluster.py:98
        self.rng = Pcg64Generator(scenario.seed)
        self._st = np.zeros((cfg.dp, cfg.pp), dtype=np.int8)
        self._ex = np.tile(np.arange(cfg.pp, dtype=np.int32), (cfg.dp, 1))
        self.down_until: dict = {}
        self.next_failure_time = scenario.failure_interval_s
        self._victims = None if scenario.victims is None else {tuple(v) for v in scenario.victims}

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


def inject_failures(state: ClusterState, scenario: FailureScenario, sim_time: float, iteration: int) -> list:
    """cluster.py:136-168. Only healthy (and, if listed, victim) nodes draw."""
    events = []
    if scenario.kind == SCENARIO_NONE:
        return events
    if scenario.kind == SCENARIO_PER_ITERATION:
        if scenario.probability == 0.0:
            return events
        for i, s in state.nodes():
            if state._st[i, s] != 0:
                continue
            if state._victims is not None and (i, s) not in state._victims:
                continue
            if state.rng.random() < scenario.probability:
                state._st[i, s] = 1
                state.down_until[(i, s)] = iteration + scenario.recovery_iterations
                events.append(_event(sim_time, iteration, "fail", (i, s)))
        return events
    while sim_time >= state.next_failure_time:
        boundary = state.next_failure_time
        state.next_failure_time += scenario.failure_interval_s
        cands = state.healthy_nodes()
        if state._victims is not None:
            cands = [n for n in cands if n in state._victims]
        if not cands:
            continue
        node = cands[int(state.rng.integers(len(cands)))]
        state._st[node] = 1
        state.down_until[node] = boundary + scenario.recovery_time_s
        events.append(_event(boundary, iteration, "fail", node))
    return events


def due_recoveries(state: ClusterState, sim_time: float, iteration: int) -> list:
    """cluster.py:171-173."""
    clock = iteration if state.scenario.kind == SCENARIO_PER_ITERATION else sim_time
    return sorted(n for n, until in state.down_until.items() if clock >= until)


def recover_node(state: ClusterState, node, sim_time: float, iteration: int) -> list:
    """cluster.py:176-187."""
    i, s = node
    if state._st[i, s] != 1:
        raise ContractViolation(f"node {tuple(node)} is not failed")
    old = int(state._ex[i, s])
    state._st[i, s] = 0
    state.down_until.pop((i, s), None)
    state._ex[i, s] = s
    if old != s and state._st[i, old] == 2 and int((state._ex[i] == old).sum()) == 1:
        state._st[i, old] = 0
    return [_event(sim_time, iteration, "recover", (i, s), fetched_from=[i, old])]


def ring_route(n: int, failed) -> list | None:
    """Ring-successor takeover on one ring of n members (cluster.py:207-218):
    failed members in descending order each take the first following member
    that is neither failed nor already adopting. Returns executor[j] for every
    member, or None if some failed member has no eligible adopter. Runs in
    the native control library (mecefo_ring_route, libmecefo_ctl.so)."""
    return _pcg.ring_route(n, failed)


def reassign_takeover(state: ClusterState, sim_time: float = 0.0, iteration: int = 0) -> list:
    """cluster.py:190-239."""
    cfg = state.cfg
    events = []
    for i in range(cfg.dp):
        failed = [int(s) for s in np.nonzero(state._st[i] == 1)[0]]
        route = ring_route(cfg.pp, failed)
        if route is None:
            raise UnrecoverableRankError(f"DP rank {i}: no eligible adopter for stage "
                                         f"(failed stages {sorted(failed)})")
        adopters = {route[s] for s in failed}
        for s in range(cfg.pp):
            if s not in failed:
                state._ex[i, s] = s
        for s in sorted(failed, reverse=True):
            if int(state._ex[i, s]) != route[s]:
                state._ex[i, s] = route[s]
                events.append(_event(sim_time, iteration, "adopt", (i, route[s]), stage=s,
                                     layers=list(cfg.layers_of_stage(s)),
                                     fetched_from_rank=(i + 1) % cfg.dp if cfg.dp > 1 else i))
        for s in range(cfg.pp):
            if s not in failed:
                state._st[i, s] = 2 if s in adopters else 0
    return events


def validate_state(state: ClusterState) -> None:
    """cluster.py:253-271: partition and status-coupling invariants."""
    cfg = state.cfg
    for i in range(cfg.dp):
        for s in range(cfg.pp):
            if state._st[i, int(state._ex[i, s])] == 1:
                raise ConsistencyError(f"stage ({i},{s}) assigned to failed node ({i},{int(state._ex[i, s])})")
        counts = np.bincount(state._ex[i], minlength=cfg.pp)
        for s in range(cfg.pp):
            want = {0: 1, 1: 0, 2: 2}[int(state._st[i, s])]
            if counts[s] != want:
                raise ConsistencyError(f"{_NAMES[state._st[i, s]]} node ({i},{s}) executes {counts[s]} stages")


def step_cluster(state: ClusterState, sim_time: float, iteration: int) -> list:
    """cluster.py:242-250: recoveries, then failures, then reassignment."""
    events = []
    for node in due_recoveries(state, sim_time, iteration):
        events.extend(recover_node(state, node, sim_time, iteration))
    events.extend(inject_failures(state, state.scenario, sim_time, iteration))
    events.extend(reassign_takeover(state, sim_time, iteration))
    validate_state(state)
    return events


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
