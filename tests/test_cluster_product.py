"""CPU: the product control plane (paper_2510_16415_b200.cluster) is bit-exact
with the reference — replayed against the reference's own logs (goldens) and
the reference test suite's cases (pkg/tests/test_cluster.py)."""

import json
import os

import pytest
from hypothesis import given, settings, strategies as st

from oracle import cluster_ref
from paper_2510_16415_b200 import cluster as cl
from paper_2510_16415_b200.errors import ConsistencyError, ContractViolation, UnrecoverableRankError

G = os.path.join(os.path.dirname(__file__), "golden")


def make_state(dp=4, pp=4, layers=4, **kw):
    return cl.ClusterState(cl.ClusterConfig(dp=dp, pp=pp, layers=layers),
                           cl.FailureScenario(**kw) if kw else cl.FailureScenario())


def fail(state, rank, stage, until=10**9):
    state.status[(rank, stage)] = cl.FAILED
    state.down_until[(rank, stage)] = until


def test_replays_reference_logs_bit_exactly():
    logs = json.load(open(os.path.join(G, "cluster_logs.json")))
    for name, rec in logs.items():
        c = rec["config"]
        sc = dict(rec["scenario"])
        if sc.get("victims") is not None:
            sc["victims"] = tuple(tuple(v) for v in sc["victims"])
        state = cl.ClusterState(cl.ClusterConfig(dp=c["dp"], pp=c["pp"], layers=c["layers"]),
                                cl.FailureScenario(**sc))
        sim = 0.0
        for it, snap in enumerate(rec["iterations"]):
            evs = cl.step_cluster(state, sim, it)
            assert json.loads(json.dumps(evs)) == snap["events"], (name, it)
            assert [state.status[(i, s)] for i in range(c["dp"]) for s in range(c["pp"])] == snap["status"]
            assert [list(state.executor[(i, s)]) for i in range(c["dp"]) for s in range(c["pp"])] == snap["executor"]
            assert state.affected_ranks() == snap["affected"]
            assert [cl.active_set(state, l, "q") for l in range(c["layers"])] == snap["active_mha"]
            sim += c["dt"]
        if "unrecoverable_at" in rec:
            with pytest.raises(UnrecoverableRankError):
                cl.step_cluster(state, sim, len(rec["iterations"]))


def test_ring_route_matches_reference_router():
    router = json.load(open(os.path.join(G, "router.json")))
    for n, table in router.items():
        for pattern, expect in table.items():
            failed = {s for s in range(int(n)) if int(pattern) >> s & 1}
            assert cl.ring_route(int(n), failed) == expect, (n, pattern)


@pytest.mark.parametrize("n", [2, 3, 5, 8, 9])
def test_ring_route_exhaustive_against_oracle(n):
    for pattern in range(1 << n):
        failed = {s for s in range(n) if pattern >> s & 1}
        want = cluster_ref.ring_takeover(n, failed)
        got = cl.ring_route(n, failed)
        if want is None:
            assert got is None
        else:
            assert got == [want.get(s, s) for s in range(n)]


def test_single_failure_ring_successor():
    state = make_state()
    fail(state, 0, 2)
    cl.reassign_takeover(state)
    assert state.executor[(0, 2)] == (0, 3)
    assert state.status[(0, 3)] == cl.DOUBLED


def test_two_adjacent_failures_frozen_expectation():
    state = make_state()
    fail(state, 0, 1)
    fail(state, 0, 2)
    cl.reassign_takeover(state)
    assert state.executor[(0, 2)] == (0, 3) and state.executor[(0, 1)] == (0, 0)
    assert state.status[(0, 3)] == cl.DOUBLED and state.status[(0, 0)] == cl.DOUBLED


def test_infeasible_rank_aborts():
    state = make_state(pp=2, layers=2)
    fail(state, 1, 0)
    fail(state, 1, 1)
    with pytest.raises(UnrecoverableRankError):
        cl.reassign_takeover(state)


def test_recovery_round_trip_and_partial():
    state = make_state()
    fail(state, 2, 1, until=5)
    cl.reassign_takeover(state)
    ev = cl.recover_node(state, (2, 1), 0.0, 5)
    cl.reassign_takeover(state)
    assert ev[0]["kind"] == "recover"
    assert all(state.executor[n] == n for n in state.nodes())
    state = make_state()
    fail(state, 0, 1)
    fail(state, 0, 2)
    cl.reassign_takeover(state)
    cl.recover_node(state, (0, 1), 0.0, 0)
    cl.reassign_takeover(state)
    assert state.status[(0, 0)] == cl.HEALTHY and state.status[(0, 3)] == cl.DOUBLED
    cl.validate_state(state)
    with pytest.raises(ContractViolation):
        cl.recover_node(state, (1, 1), 0.0, 0)


@given(st.lists(st.tuples(st.booleans(), st.integers(0, 15)), min_size=1, max_size=40))
@settings(max_examples=60, deadline=None)
def test_random_sequences_preserve_partition(ops):
    state = make_state(dp=2, pp=4, layers=4)
    ref = cluster_ref.Cluster(2, 4, 4)
    for is_fail, pick in ops:
        if is_fail:
            healthy = state.healthy_nodes()
            if not healthy:
                continue
            node = healthy[pick % len(healthy)]
            before_st = state._st.copy()
            before_ex = state._ex.copy()
            fail(state, *node)
            try:
                cl.reassign_takeover(state)
            except UnrecoverableRankError:
                state._st[:] = before_st
                state._ex[:] = before_ex
                state.down_until.pop(node, None)
                continue
        else:
            failed = sorted(n for n in state.nodes() if state.status[n] == cl.FAILED)
            if not failed:
                continue
            cl.recover_node(state, failed[pick % len(failed)], 0.0, 0)
            cl.reassign_takeover(state)
        cl.validate_state(state)
        for i in range(2):
            stages = {s for s in range(4) if state.status[(i, s)] == cl.FAILED}
            take = cluster_ref.ring_takeover(4, stages)
            assert take is not None
            assert [state.executor[(i, s)][1] for s in range(4)] == [take.get(s, s) for s in range(4)]


def test_injection_edge_cases():
    state = make_state(kind="per_iteration", probability=0.0, seed=1)
    assert cl.inject_failures(state, state.scenario, 0.0, 0) == []
    state = make_state(dp=4, pp=8, layers=8, kind="per_iteration", probability=1.0, seed=1)
    assert len(cl.inject_failures(state, state.scenario, 0.0, 0)) == 32
    state = make_state(dp=2, pp=4, layers=4, kind="per_iteration", probability=1.0, victims=((1, 2),), seed=1)
    evs = cl.inject_failures(state, state.scenario, 0.0, 0)
    assert [e["node"] for e in evs] == [[1, 2]]


def test_active_sets_and_validation():
    state = make_state(dp=3, pp=2, layers=4)
    fail(state, 1, 0)
    cl.reassign_takeover(state)
    assert cl.active_set(state, 0, "q") == [0, 2]
    assert cl.active_set(state, 3, "q") == [0, 2]  # stage 1 of rank 1 is run by the doubled node
    assert cl.active_set(state, 0, "gate") == [0, 1, 2]
    with pytest.raises(ContractViolation):
        cl.active_set(state, 0, "bogus")
    state._ex[0, 1] = 0  # break the partition: node (0,0) now runs 2 stages while healthy
    with pytest.raises(ConsistencyError):
        cl.validate_state(state)


def test_stage_boundaries_match_reference_rounding():
    for L in range(1, 17):
        for pp in range(1, L + 1):
            c = cl.ClusterConfig(dp=1, pp=pp, layers=L)
            assert c.boundaries() == cluster_ref.boundaries(L, pp)
            for l in range(L):
                assert c.stage_of_layer(l) == cluster_ref.stage_of(l, c.boundaries())


def test_ring_plan_eq1_weights():
    from paper_2510_16415_b200.engine import ring_plan

    route, lean, a_mha, skip = ring_plan(2, {1}, 3)
    assert route == [0, 0] and lean == [True, True] and a_mha is None and len(skip) == 15
    route, lean, a_mha, skip = ring_plan(8, {3}, 2)
    assert route[3] == 4 and lean == [False, False, False, True, True, False, False, False]
    assert a_mha == pytest.approx(1 / 6) and skip == []
    with pytest.raises(UnrecoverableRankError):
        ring_plan(2, {0, 1}, 2)


def test_control_plane_is_native_and_matches_python_accounting():
    """step_cluster / inject / recover / reassign / validate run in the native
    state machine (libmecefo_ctl.so); iteration_cost's native FLOP accounting
    equals the Python restatement on random degraded states."""
    import numpy as np

    from paper_2510_16415_b200 import costmodel as cm, model as mdl

    assert cl.ClusterState.native
    mcfg = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=8, seq_len=64)
    rng = np.random.default_rng(3)
    for trial in range(40):
        dp, pp = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        state = make_state(dp=dp, pp=pp, layers=8, kind="per_iteration", probability=0.3, recovery_iterations=2,
                           seed=trial)
        for it in range(6):
            try:
                cl.step_cluster(state, 0.0, it)
            except UnrecoverableRankError:
                break
            for policy in (cm.POLICY_APPROX, cm.POLICY_NAIVE):
                args = (state, mcfg, policy, 32, 100, 256)
                assert cm.iteration_cost(*args) == cm.iteration_cost_py(*args)
