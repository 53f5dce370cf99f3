"""CPU: host-side logic that needs no GPU — cost-model clock, lr schedule,
AdamW bias-correction segments, weight layout, and the C-ABI library's
exported symbols (loaded, never called)."""

import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

from oracle import model_ref, optim_ref
from paper_2510_16415_b200 import _lib, cluster as cl, costmodel as cm, model as mdl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


class _Cfg:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def test_linear_flops_known_answers():
    # pkg/tests/test_costmodel.py:12-18 known answers
    assert cm.linear_flops(8, 64, 128, cm.FPROP) == 131072
    assert cm.linear_flops(8, 64, 128, cm.APPROX_WGRAD, r=4) == 2 * 4 * (8 * 128 + 8 * 64 + 64 * 128)


def test_sim_clock_reproduces_reference_run():
    """harness.py:442-446: sim_time advances by worst-node flops / node_flops
    + fetch events * fetch_cost; must match the reference rows exactly."""
    rec = json.load(open(os.path.join(G, "c0_training.json")))
    model = _Cfg(hidden=128, ffn_intermediate=344, heads=4, seq_len=64, vocab=64, layers=2)
    state = cl.ClusterState(cl.ClusterConfig(dp=2, pp=2, layers=2),
                            cl.FailureScenario(kind="per_iteration", probability=1.0, recovery_iterations=10**9,
                                               victims=((0, 1),), seed=7))
    sim = 0.0
    for it, row in enumerate(rec["rows"]):
        evs = cl.step_cluster(state, sim, it)
        worst, _, _, _ = cm.iteration_cost(state, model, cm.POLICY_APPROX, 32, 100, 4 * 64)
        fetches = sum(1 for e in evs if e["kind"] in ("adopt", "recover"))
        sim += worst / 1e12 + fetches * 1.0
        assert sim == row["sim_time_s"], it
        assert len(state.affected_ranks()) == row["affected_ranks"]


def test_lr_schedule_matches_oracle():
    from paper_2510_16415_b200.optim import lr_at

    for total in (1, 4, 10, 123):
        for step in range(total + 1):
            assert lr_at(step, total, 1e-3) == optim_ref.lr_at(step, total, 1e-3)


def test_adam_segments_bias_correction():
    from paper_2510_16415_b200 import optim as op

    class W:
        layout = [("a", (3,), 0), ("b", (2, 2), 64)]

    st = op.OptimState(op.OptimConfig())
    arr, mx, names = op.adam_segments(W, st, 1e-3, skip=("b",))
    assert names == ["a"] and mx == 3
    assert arr[0]["step_size"] == pytest.approx(1e-3 / (1 - 0.9))
    assert arr[0]["inv_bc2"] == pytest.approx(1 / (1 - 0.999))
    st.step["a"] = 4
    arr, _, _ = op.adam_segments(W, st, 2e-3)
    assert arr[0]["step_size"] == pytest.approx(2e-3 / (1 - 0.9 ** 5))
    assert arr[1]["step_size"] == pytest.approx(2e-3 / (1 - 0.9))


def test_param_layout_is_canonical_and_packs_qkv_and_gate_up():
    from paper_2510_16415_b200.model import ModelConfig, _param_layout

    cfg = ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64)
    layout, total = _param_layout(cfg)
    d = model_ref.Dims(64, 128, 4, 344, 2, 64)
    assert [n for n, _, _ in layout] == [n for n, _ in model_ref.param_shapes(d)]
    off = {n: (o, s) for n, s, o in layout}
    for l in range(2):
        q, k, v = (off[f"layers.{l}.{x}"] for x in "qkv")
        assert k[0] == q[0] + 128 * 128 and v[0] == k[0] + 128 * 128
        g, u = off[f"layers.{l}.gate"], off[f"layers.{l}.up"]
        assert u[0] == g[0] + 344 * 128
    assert all(o % 64 == 0 for n, (o, s) in off.items() if not n.endswith((".k", ".v", ".up")))
    assert total >= max(o + int(np.prod(s)) for o, s in off.values())


def test_flop_formulas_match_survey():
    c1 = _Cfg(hidden=512, ffn_intermediate=1376, layers=8, seq_len=256, vocab=32000)
    assert abs(cm.standard_flops_per_token(c1) / 1e6 - 256.4) < 0.1
    assert abs(cm.lean_flops_per_token(c1, 128, 8192) / 1e6 - 219.5) < 0.2


def test_c_abi_library_exports_every_declared_symbol():
    """include/mecefo.h declarations == symbols exported by libmecefo.so ==
    the ctypes binding table (no compute calls without a GPU)."""
    hdr = open(os.path.join(ROOT, "include", "mecefo.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(mecefo_\w+)\(", hdr, flags=re.M))
    assert "mecefo_backward_block_neighbor" in declared and len(declared) >= 20
    assert declared == set(_lib.EXPORTED_SYMBOLS)
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.mecefo_version()


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(_lib.EngineUnavailable):
        _lib.load(str(tmp_path / "nope.so"))


def test_padded_ffn_layout_and_wire_format_round_trip():
    """f = 5461 (LLaMA-1B) is stored padded to 5464; the reference-facing
    views and the final_weights wire format keep the reference's shapes."""
    from paper_2510_16415_b200 import harness

    cfg = mdl.ModelConfig(vocab=16, hidden=32, heads=4, ffn_intermediate=5461, layers=1, seq_len=8)
    layout, total = mdl._param_layout(cfg)
    shapes = {n: s for n, s, _ in layout}
    assert mdl.ffn_storage(cfg) == 5464
    assert shapes["layers.0.gate"] == (5464, 32) and shapes["layers.0.down"] == (32, 5464)
    assert mdl.logical_shape(cfg, "layers.0.down", shapes["layers.0.down"]) == (32, 5461)
    rng = np.random.default_rng(0)
    host = np.zeros(total, dtype=np.float32)
    ref = {}
    for name, shape, off in layout:
        blk = mdl.logical_view(cfg, name, host[off: off + int(np.prod(shape))].reshape(shape))
        ref[name] = rng.normal(size=blk.shape).astype(np.float32)
        blk[...] = ref[name]
    blob, manifest = harness.pack_weights(layout, host, cfg)
    assert [tuple(p["shape"]) for p in manifest["params"]] == [ref[n].shape for n, _, _ in layout]
    assert blob.size == sum(v.size for v in ref.values())
    back = harness.unpack_weights(layout, total, blob, manifest, cfg)
    assert np.array_equal(back, host)  # pads come back as zero
