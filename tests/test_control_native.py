"""Native control-plane streams (libmecefo_ctl.so, include/mecefo_ctl.h) are
draw-for-draw identical to numpy's Generator(PCG64(SeedSequence(...))), which
is what the reference's failure injection (pkg/src/faultsim/cluster.py:98,149,164)
and sampler (data.py:96,104) draw from. numpy is the checker here. CPU only."""

import copy
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2510_16415_b200 import cluster, errors, pcg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SEEDS = [0, 1, 7, 23, 2**32 - 1, 2**32, 123456789012345, 2**64 - 1, (0, 0xDA7A, 3), (5, 0x5E7, 1), (2**40, 0, 0, 9)]


def _np(entropy):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "mecefo_ctl.h")).read()
    declared = set(re.findall(r"^int (mecefo_\w+)\(", hdr, re.M))
    assert declared == set(pcg.SYMBOLS)
    lib = ctypes.CDLL(pcg.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name


@pytest.mark.parametrize("entropy", SEEDS)
def test_seed_state_matches_numpy(entropy):
    g, r = pcg.Pcg64Generator(entropy), _np(entropy)
    st = r.bit_generator.state
    assert g.state["state"] == st["state"]["state"] and g.state["inc"] == st["state"]["inc"]
    assert np.array_equal(g.next_uint64(257), r.bit_generator.random_raw(257).astype(np.uint64))


@pytest.mark.parametrize("entropy", SEEDS)
def test_interleaved_draws_match_numpy(entropy):
    """random / integers over 32-bit (buffered next_uint32) and 64-bit ranges,
    scalar and vector, interleaved so numpy's uint32 buffer carries across calls."""
    g, r = pcg.Pcg64Generator(entropy), _np(entropy)
    rs = np.random.Generator(np.random.PCG64(0))
    for step in range(60):
        op = int(rs.integers(6))
        n = int(rs.integers(1, 40))
        if op == 0:
            assert g.random() == r.random()
        elif op == 1:
            assert np.array_equal(g.random(n), r.random(n))
        elif op == 2:
            hi = int(rs.integers(1, 10))
            assert g.integers(hi) == r.integers(hi)
        elif op == 3:
            assert np.array_equal(g.integers(0, 32000, size=(n, 3)), r.integers(0, 32000, size=(n, 3)))
        elif op == 4:
            lo, hi = -5, 2**40 + 3
            assert np.array_equal(g.integers(lo, hi, size=n), r.integers(lo, hi, size=n))
        else:
            assert np.array_equal(g.integers(0, 2**32, size=n), r.integers(0, 2**32, size=n))
        assert g.state["has_uint32"] == r.bit_generator.state["has_uint32"], step


def test_edge_ranges_and_contract():
    g, r = pcg.Pcg64Generator(3), _np(3)
    assert np.array_equal(g.integers(4, 5, size=5), r.integers(4, 5, size=5))  # single value: no draw
    assert np.array_equal(g.integers(0, 2**63 - 1, size=5), r.integers(0, 2**63 - 1, size=5))
    assert np.array_equal(g.integers(-(2**63), 2**63 - 1, size=5), r.integers(-(2**63), 2**63 - 1, size=5))
    with pytest.raises(errors.ContractViolation):
        g.integers(3, 3)
    with pytest.raises(errors.ContractViolation):
        pcg.Pcg64Generator(-1)


def test_copy_forks_stream():
    g = pcg.Pcg64Generator(11)
    g.integers(7)
    h = copy.deepcopy(g)
    assert np.array_equal(g.integers(0, 100, size=50), h.integers(0, 100, size=50))


def test_cluster_state_uses_native_stream():
    st = cluster.ClusterState(cluster.ClusterConfig(dp=4, pp=2, layers=2), cluster.FailureScenario(kind="per_iteration",
                                                                                        probability=0.5, seed=7))
    assert isinstance(st.rng, pcg.Pcg64Generator)


def _sampler_golden():
    import json

    return json.load(open(os.path.join(ROOT, "tests", "golden", "sampler.json")))


@pytest.mark.parametrize("source", ["teacher", "corpus"])
def test_sharded_sampler_matches_reference_batches(source):
    """data.ShardedSampler == reference faultsim.data.ShardedSampler
    (tests/golden/make_sampler_golden.py): same shards, same window starts
    from the native (seed, 0xDA7A, rank) streams, bit-exact token ids."""
    from paper_2510_16415_b200 import data

    rec = _sampler_golden()[source]
    args = dict(rec["args"])
    if source == "corpus":
        args["text"] = rec["text"]
    s = data.ShardedSampler(**args)
    for call in rec["calls"]:
        x, y = s.batch(call["rank"], call["batch"])
        assert x.dtype == np.int64 and x.shape == (call["batch"], args["seq_len"])
        assert x.tolist() == call["inputs"] and y.tolist() == call["targets"]
    ex, ey = s.eval_windows(0, 5)
    assert ex.tolist() == rec["eval"]["inputs"] and ey.tolist() == rec["eval"]["targets"]


def test_sharded_sampler_contract():
    from paper_2510_16415_b200 import data

    with pytest.raises(errors.ConfigError):
        data.ShardedSampler(2, 8, 16, 0, source="corpus")  # no corpus given
    with pytest.raises(errors.ConfigError):
        data.ShardedSampler(2, 8, 2, 0, source="corpus", text="abcabc" * 20)  # vocab too small
    with pytest.raises(errors.ConfigError):
        data.ShardedSampler(2, 40, 16, 0, source="corpus", text="ab" * 30)  # shard too short
    with pytest.raises(errors.ConfigError):
        data.ShardedSampler(2, 8, 16, 0, source="bogus")
    with pytest.raises(errors.ConfigError):
        data.encode("abz", {"a": 0, "b": 1})
