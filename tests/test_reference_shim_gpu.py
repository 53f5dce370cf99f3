"""GPU: the reference's OWN harness driving the engine (Callers).

numpy_shim.install() replaces the three block operators the reference looks up
by module attribute (faultsim/model.py:461-463, faultsim/harness.py:226-235)
with the device bridge. The reference (faultsim, installed into oracle/_ref by
oracle/build_ref.sh; it travels with the repo) then runs unchanged:
`harness._rank_pass` (harness.py:243-249) and a short `harness.run_training`
with a permanently failed rank (the pattern of pkg/tests/test_harness.py:
87-102). Its results must match the same reference run without the bridge
(float64 numpy) within the north-star fp32 tolerance, tensor_rel_err <= 1e-4
(pkg/tests/oracles.py:147-149), and every integer column bit-exactly.
"""

import copy
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


@pytest.fixture
def fs():
    if not os.path.isdir(os.path.join(REF, "faultsim")):
        pytest.skip("reference not installed into oracle/_ref (oracle/build_ref.sh)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import faultsim
    import faultsim.approx
    import faultsim.harness
    import faultsim.model

    return faultsim


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _caches(fs, cfg, r, bases):
    out = {}
    for l in range(cfg.layers):
        pc = fs.approx.ProjectionCache(rank=r, refresh_period=100, step=1)
        pc.basis = {k: v.copy() for k, v in bases[l].items()}
        out[l] = pc
    return out


@pytest.mark.parametrize("lean", [True, False])
def test_rank_pass_through_the_reference_harness(cuda, fs, monkeypatch, lean):
    from paper_2510_16415_b200 import numpy_shim

    cfg = fs.model.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64)
    w = fs.model.init_weights(cfg, seed=0)
    rng = np.random.Generator(np.random.PCG64(11))
    tokens = rng.integers(0, 64, size=(4, 64))
    targets = rng.integers(0, 64, size=(4, 64))
    mode = fs.model.CACHE_FFN_INPUT_ONLY if lean else fs.model.CACHE_FULL
    modes = [mode] * cfg.layers
    bases = {l: {k: np.linalg.qr(rng.normal(size=(n, 32)))[0] for k, n in (("gate", 128), ("up", 128),
                                                                           ("down", 344))}
             for l in range(cfg.layers)}
    svd = fs.linalg.SvdConfig(rank=32, tolerance=1e-9, max_iterations=3000, seed=23)
    pc_ref = _caches(fs, cfg, 32, bases)
    loss_ref, g_ref = fs.harness._rank_pass(w, tokens, targets, modes, pc_ref if lean else None, svd)

    numpy_shim.install(fs, "fp32", monkeypatch)
    pc = _caches(fs, cfg, 32, bases)
    loss, g = fs.harness._rank_pass(w, tokens, targets, modes, pc if lean else None, svd)

    assert abs(loss - loss_ref) <= 1e-4 * abs(loss_ref)
    assert set(g) == set(g_ref)
    errs = {k: rel(g[k], g_ref[k]) for k in g_ref}
    assert max(errs.values()) <= 1e-4, errs
    if lean:  # the reference's ProjectionCache side effects (approx.py:132-133)
        assert [pc[l].step for l in pc] == [pc_ref[l].step for l in pc_ref]
        assert [pc[l].refreshes for l in pc] == [pc_ref[l].refreshes for l in pc_ref]


def test_run_training_with_a_failed_rank_through_the_bridge(cuda, fs, monkeypatch):
    """The reference's whole failure-handling loop (NDB takeover, lean modes,
    adoption resets -> device refreshes, Eq. (1), AdamW) with the engine as
    its block operators."""
    from paper_2510_16415_b200 import numpy_shim

    raw = {"model": {"vocab": 64, "hidden": 32, "heads": 4, "ffn_intermediate": 64, "layers": 2, "seq_len": 16},
           "cluster": {"dp": 4, "pp": 2, "layers": 2},
           "scenario": {"kind": "per_iteration", "probability": 1.0, "victims": [[1, 0]],
                        "recovery_iterations": 10**9},
           "optimizer": {"kind": "adamw", "lr": 1e-3},
           "run": {"iterations": 4, "global_batch": 8, "seed": 3, "r": 8}}
    ref = fs.harness.run_training(fs.harness.config_from_dict(copy.deepcopy(raw)))
    numpy_shim.install(fs, "fp32", monkeypatch)
    got = fs.harness.run_training(fs.harness.config_from_dict(copy.deepcopy(raw)))

    assert len(got.rows) == len(ref.rows) == 4
    for a, b in zip(got.rows, ref.rows):
        for key, v in b.items():
            if key == "loss":
                assert abs(a[key] - v) <= 1e-4 * abs(v), (key, a[key], v)
            elif isinstance(v, float) and key not in ("sim_time_s", "lr"):
                assert a[key] == pytest.approx(v, rel=1e-3, abs=1e-6), key
            else:
                assert a[key] == v, key  # iteration, events, affected ranks, lr, simulated clock
    assert any(r["affected_ranks"] for r in got.rows)
    errs = {n: rel(arr, ref.weights.get(n)) for n, arr in got.weights.named()}
    assert max(errs.values()) <= 1e-4, sorted(errs.items(), key=lambda kv: -kv[1])[:4]
