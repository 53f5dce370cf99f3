"""CPU: pin the oracle restatement against the reference's own outputs.

The golden files were produced by running the reference (faultsim) in the
build container (tests/golden/make_golden.py). If the oracle agrees with them,
it can stand in for the reference on the GPU box, where the reference does
not exist.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import cluster_ref, model_ref as R, optim_ref

G = os.path.join(os.path.dirname(__file__), "golden")
C0 = R.Dims(vocab=64, hidden=128, heads=4, ffn=344, layers=2, seq_len=64)
TINY = R.Dims(vocab=16, hidden=16, heads=4, ffn=32, layers=1, seq_len=6)


def _npz(name):
    return np.load(os.path.join(G, name))


def test_init_params_bit_identical_to_reference():
    shas = json.load(open(os.path.join(G, "weights_sha.json")))
    for key, d, seed, std in (("c0", C0, 0, 0.02), ("tiny5", TINY, 5, 0.1)):
        w = R.init_params(d, seed, std)
        assert list(w) == list(shas[key]) or set(w) == set(shas[key])
        for name, a in w.items():
            assert hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest() == shas[key][name], name


@pytest.mark.parametrize("fixture,dims,seed,std,tol", [
    ("tiny_block.npz", TINY, 5, 0.1, 1e-10),
    ("c0_block.npz", C0, 0, 0.02, 2e-5),
])
def test_block_math_matches_reference(fixture, dims, seed, std, tol):
    z = _npz(fixture)
    W = R.init_params(dims, seed, std)
    x = z["x"].astype(np.float64)
    x3 = x.reshape(-1, dims.seq_len, dims.hidden)
    dy3 = z["dy"].astype(np.float64).reshape(x3.shape)
    y, lean = R.block_fwd(dims, W, 0, x3, lean=True)
    assert R.rel_err(y.reshape(x.shape), z["y"]) < tol
    assert R.rel_err(lean["x1"].reshape(x.shape), z["x1"]) < tol
    basis = {k: z[f"v1.{k}"].astype(np.float64) for k in ("gate", "up", "down")}
    dx, g = R.block_bwd_neighbor(dims, W, 0, lean, dy3, basis)
    assert R.rel_err(dx.reshape(x.shape), z["dx_lowrank"]) < tol * 10
    for k in ("gate", "up", "down", "norm_ffn"):
        assert R.rel_err(g[k], z[f"g_lowrank.{k}"]) < tol * 10, k
    dx, g = R.block_bwd_neighbor(dims, W, 0, lean, dy3, None)
    assert R.rel_err(dx.reshape(x.shape), z["dx_exact_neighbor"]) < tol
    for k in g:
        assert R.rel_err(g[k], z[f"g_exact_neighbor.{k}"]) < tol, k
    _, full = R.block_fwd(dims, W, 0, x3, lean=False)
    dx, g = R.block_bwd_exact(dims, W, 0, full, dy3)
    assert R.rel_err(dx.reshape(x.shape), z["dx_full"]) < tol
    for k in g:
        assert R.rel_err(g[k], z[f"g_full.{k}"]) < tol, k


def test_rank_pass_matches_reference():
    z = _npz("c0_rank_pass.npz")
    W = R.init_params(C0, 0)
    bases = {l: {k: z[f"v1.{l}.{k}"].astype(np.float64) for k in ("gate", "up", "down")} for l in range(2)}
    loss, g = R.rank_pass(C0, W, z["tokens"], z["targets"], ["ffn_input_only"] * 2, bases)
    assert abs(loss - float(z["loss_lean"])) < 1e-9
    for name, v in g.items():
        assert R.rel_err(v, z[f"lean.{name}"]) < 1e-5, name
    loss, g = R.rank_pass(C0, W, z["tokens"], z["targets"], ["full"] * 2)
    assert abs(loss - float(z["loss_full"])) < 1e-9
    for name, v in g.items():
        assert R.rel_err(v, z[f"full.{name}"]) < 1e-5, name


def test_subspace_iteration_reproduces_reference_bases():
    z = _npz("c0_rank_pass.npz")
    W = R.init_params(C0, 0)
    for l in range(2):
        for k in ("gate", "up", "down"):
            w = W[f"layers.{l}.{k}"]
            v = R.subspace_top_r(w, min(32, w.shape[1]), tol=1e-9, max_iter=3000, seed=23)
            assert R.rel_err(v, z[f"v1.{l}.{k}"]) < 1e-6


def test_cluster_control_plane_replays_reference_logs():
    logs = json.load(open(os.path.join(G, "cluster_logs.json")))
    for name, rec in logs.items():
        c = rec["config"]
        sc = dict(rec["scenario"])
        cl = cluster_ref.Cluster(c["dp"], c["pp"], c["layers"], kind=sc["kind"], p=sc.get("probability", 0.0),
                                 rec_iters=sc.get("recovery_iterations", 1),
                                 interval=sc.get("failure_interval_s", 1800.0),
                                 rec_time=sc.get("recovery_time_s", 7200.0), victims=sc.get("victims"),
                                 seed=sc["seed"])
        sim = 0.0
        for it, snap in enumerate(rec["iterations"]):
            evs = cl.step(sim, it)
            assert json.loads(json.dumps(evs)) == snap["events"], (name, it)
            assert [cl.st[(i, s)] for i in range(c["dp"]) for s in range(c["pp"])] == snap["status"]
            assert [list(cl.ex[(i, s)]) for i in range(c["dp"]) for s in range(c["pp"])] == snap["executor"]
            assert cl.affected() == snap["affected"]
            assert [cl.active(l, "q") for l in range(c["layers"])] == snap["active_mha"]
            sim += c["dt"]
        if "unrecoverable_at" in rec:
            with pytest.raises(RuntimeError):
                cl.step(sim, len(rec["iterations"]))


def test_ring_router_matches_reference():
    router = json.load(open(os.path.join(G, "router.json")))
    for R_, table in router.items():
        n = int(R_)
        for pattern, expect in table.items():
            failed = {s for s in range(n) if int(pattern) >> s & 1}
            take = cluster_ref.ring_takeover(n, failed)
            if expect is None:
                assert take is None
            else:
                got = [take.get(s, s) if s in failed else s for s in range(n)]
                assert got == expect


def test_training_loop_replays_reference_run():
    """harness.run_training (C0, dp2 x pp2, permanent victim (0,1)) replayed
    with the oracle: losses, lr and final weights."""
    rec = json.load(open(os.path.join(G, "c0_training.json")))
    final = _npz("c0_training_weights.npz")
    W = R.init_params(C0, 0)
    opt = optim_ref.Adam()
    cl = cluster_ref.Cluster(2, 2, 2, kind="per_iteration", p=1.0, rec_iters=10**9, victims=[[0, 1]], seed=7)
    bases = {}
    for it, row in enumerate(rec["rows"]):
        evs = cl.step(0.0, it)
        for ev in evs:
            if ev["kind"] == "adopt":
                for l in ev["details"]["layers"]:
                    bases.pop((ev["node"][0], l), None)
        per_rank, losses = [], []
        for i in range(2):
            toks, tgts = (np.array(a) for a in rec["batches"][it][i])
            modes = ["ffn_input_only" if cl.lean(i, l) else "full" for l in range(2)]
            bl = {}
            for l in range(2):
                if modes[l] != "full":
                    if (i, l) not in bases:  # refresh at step 0 (tau=100 > iterations)
                        bases[(i, l)] = {k: R.subspace_top_r(W[f"layers.{l}.{k}"], 32, 1e-9, 3000, 23)
                                         for k in ("gate", "up", "down")}
                    bl[l] = bases[(i, l)]
            loss, g = R.rank_pass(C0, W, toks, tgts, modes, bl)
            losses.append(loss)
            per_rank.append(g)
        loss = sum(losses) / 2
        assert abs(loss - row["loss"]) < 1e-9 * max(1.0, abs(loss)), it
        active = {(l, k): cl.active(l, k) for l in range(2) for k in cluster_ref.MHA + cluster_ref.FFN}
        avg, skipped = cluster_ref.aggregate(per_rank, active, 2)
        lr = optim_ref.lr_at(it + 1, len(rec["rows"]), 1e-3)
        assert lr == row["lr"]
        opt.apply(W, avg, lr, skip=skipped)
    for name, v in W.items():
        assert R.rel_err(v, final[name]) < 1e-6, name
