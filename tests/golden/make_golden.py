"""Generate golden vectors by running the REFERENCE (faultsim) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed here
as small fixtures. Nothing at test/bench time imports the reference.

Outputs (tests/golden/):
  tiny_block.npz     test_approx.py CFG (hidden 16, f 32, T 6): forward,
                     neighbor backward at full rank, exact-Wgrad neighbor and
                     exact full-cache backward, float64
  c0_block.npz       C0 dims (hidden 128, f 344, H 4, T 64), layer 0, r=32
                     bases from the reference SVD (seed 23), float32
  c0_rank_pass.npz   C0 two-layer rank pass, all-lean (low-rank) and all-full
  weights_sha.json   sha256 of every initial parameter (init_weights seed 0)
  cluster_logs.json  step_cluster event logs / executors / modes / active sets
  router.json        Flavour-B ring routing: reassign_takeover on dp=1, pp=R
  c0_training.json   run_training (C0, dp2 x pp2, victim (0,1)) rows + events
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from faultsim import approx, cluster as cl, harness, model as mdl  # noqa: E402
from faultsim.errors import UnrecoverableRankError  # noqa: E402
from faultsim.linalg import SvdConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

C0 = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64, rope=True)
TINY = mdl.ModelConfig(vocab=16, hidden=16, heads=4, ffn_intermediate=32, layers=1, seq_len=6)


def _grads(prefix, g, dtype):
    return {f"{prefix}.{k}": np.asarray(v, dtype=dtype) for k, v in g.items()}


def block_fixture(cfg, seed, std, batch, rank, svd, dtype, x_scale, dy_scale):
    weights = mdl.init_weights(cfg, seed=seed, std=std)
    lw = weights.layers[0]
    rng = np.random.Generator(np.random.PCG64(seed + 100))
    x = rng.normal(size=(batch * cfg.seq_len, cfg.hidden)) * x_scale
    dy = rng.normal(size=(batch * cfg.seq_len, cfg.hidden)) * dy_scale
    y, cache_lean = mdl.forward_block(cfg, lw, x, mdl.CACHE_FFN_INPUT_ONLY)
    _, cache_full = mdl.forward_block(cfg, lw, x, mdl.CACHE_FULL)
    proj = approx.ProjectionCache(rank=rank, refresh_period=1)
    dx_lr, g_lr = approx.backward_block_neighbor(cfg, lw, cache_lean, dy, proj=proj, svd=svd)
    dx_ex, g_ex = approx.backward_block_neighbor(cfg, lw, cache_lean, dy, proj=None)
    dx_full, g_full = mdl.backward_block_exact(cfg, lw, cache_full, dy)
    out = {
        "x": x, "dy": dy, "y": y, "x1": cache_lean.x1.reshape(x.shape),
        "dx_lowrank": dx_lr, "dx_exact_neighbor": dx_ex, "dx_full": dx_full,
    }
    for k in ("gate", "up", "down"):
        out[f"v1.{k}"] = proj.basis[k]
    out.update(_grads("g_lowrank", g_lr, np.float64))
    out.update(_grads("g_exact_neighbor", g_ex, np.float64))
    out.update(_grads("g_full", g_full, np.float64))
    meta = {"seed": seed, "std": std, "batch": batch, "rank": rank, "x_scale": x_scale, "dy_scale": dy_scale}
    return {k: np.asarray(v, dtype=dtype) for k, v in out.items()}, meta


def main():
    # ---- tiny block (float64): the tests/test_approx.py configuration ----
    tiny, meta = block_fixture(TINY, seed=5, std=0.1, batch=2, rank=32,
                               svd=SvdConfig(rank=1, tolerance=1e-13, max_iterations=3000, seed=0),
                               dtype=np.float64, x_scale=1.0, dy_scale=1.0)
    np.savez_compressed(os.path.join(OUT, "tiny_block.npz"), meta=json.dumps(meta), **tiny)

    # ---- C0 block (float32 storage) ----
    svd = SvdConfig(rank=32, tolerance=1e-9, max_iterations=3000, seed=23)
    c0b, meta = block_fixture(C0, seed=0, std=0.02, batch=4, rank=32, svd=svd, dtype=np.float32, x_scale=0.5,
                              dy_scale=0.01)
    np.savez_compressed(os.path.join(OUT, "c0_block.npz"), meta=json.dumps(meta), **c0b)

    # ---- initial weight hashes ----
    shas = {}
    for cfg_name, cfg, seed in (("c0", C0, 0), ("tiny5", TINY, 5)):
        w = mdl.init_weights(cfg, seed=seed, std=0.1 if cfg is TINY else 0.02)
        shas[cfg_name] = {name: hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()
                          for name, a in w.named()}
    with open(os.path.join(OUT, "weights_sha.json"), "w") as f:
        json.dump(shas, f, indent=1, sort_keys=True)

    # ---- C0 rank pass: all-lean (low-rank, refreshed bases) and all-full ----
    weights = mdl.init_weights(C0, seed=0)
    rng = np.random.Generator(np.random.PCG64(42))
    tokens = rng.integers(0, C0.vocab, size=(4, C0.seq_len))
    targets = rng.integers(0, C0.vocab, size=(4, C0.seq_len))
    lean = [mdl.CACHE_FFN_INPUT_ONLY] * C0.layers
    projs = {l: approx.ProjectionCache(rank=32, refresh_period=100) for l in range(C0.layers)}
    loss_lean, g_lean = harness._rank_pass(weights, tokens, targets, lean, projs, svd)
    loss_full, g_full = harness._rank_pass(weights, tokens, targets, None)
    rp = {"tokens": tokens, "targets": targets, "loss_lean": np.float64(loss_lean),
          "loss_full": np.float64(loss_full)}
    for l in range(C0.layers):
        for k in ("gate", "up", "down"):
            rp[f"v1.{l}.{k}"] = projs[l].basis[k].astype(np.float32)
    rp.update({f"lean.{k}": v.astype(np.float32) for k, v in g_lean.items()})
    rp.update({f"full.{k}": v.astype(np.float32) for k, v in g_full.items()})
    np.savez_compressed(os.path.join(OUT, "c0_rank_pass.npz"), **rp)

    # ---- cluster control-plane logs ----
    scenarios = {
        "per_iter_dp4_pp4": dict(dp=4, pp=4, layers=8, scen=dict(kind="per_iteration", probability=0.05,
                                                                 recovery_iterations=3, seed=7), iters=300, dt=1.0),
        "per_iter_dp2_pp8": dict(dp=2, pp=8, layers=8, scen=dict(kind="per_iteration", probability=0.03,
                                                                 recovery_iterations=5, seed=11), iters=300, dt=1.0),
        "scheduled_dp2_pp4": dict(dp=2, pp=4, layers=6, scen=dict(kind="scheduled", failure_interval_s=1800.0,
                                                                  recovery_time_s=5000.0, seed=3), iters=200,
                                  dt=700.0),
        "victims_c0": dict(dp=2, pp=2, layers=2, scen=dict(kind="per_iteration", probability=1.0,
                                                           recovery_iterations=10**9, victims=((0, 1),), seed=7),
                           iters=20, dt=1.0),
        "ring_dp1_pp8": dict(dp=1, pp=8, layers=8, scen=dict(kind="per_iteration", probability=0.08,
                                                             recovery_iterations=2, seed=5), iters=400, dt=1.0),
    }
    logs = {}
    for name, sc in scenarios.items():
        state = cl.ClusterState(cl.ClusterConfig(dp=sc["dp"], pp=sc["pp"], layers=sc["layers"]),
                                cl.FailureScenario(**sc["scen"]))
        rec = {"config": {k: v for k, v in sc.items() if k != "scen"}, "scenario": sc["scen"], "iterations": []}
        sim = 0.0
        for it in range(sc["iters"]):
            try:
                evs = cl.step_cluster(state, sim, it)
            except UnrecoverableRankError as exc:
                rec["unrecoverable_at"] = it
                rec["error"] = str(exc)
                break
            rec["iterations"].append({
                "events": evs,
                "status": [state.status[(i, s)] for i in range(sc["dp"]) for s in range(sc["pp"])],
                "executor": [list(state.executor[(i, s)]) for i in range(sc["dp"]) for s in range(sc["pp"])],
                "affected": state.affected_ranks(),
                "active_mha": [cl.active_set(state, l, "q") for l in range(sc["layers"])],
            })
            sim += sc["dt"]
        logs[name] = rec
    with open(os.path.join(OUT, "cluster_logs.json"), "w") as f:
        json.dump(logs, f, separators=(",", ":"))

    # ---- Flavour-B routing: R logical DP ranks on a ring ----
    router = {}
    for R in (2, 3, 4, 8):
        table = {}
        for pattern in range(1 << R):
            failed = [s for s in range(R) if pattern >> s & 1]
            state = cl.ClusterState(cl.ClusterConfig(dp=1, pp=R, layers=R), cl.FailureScenario())
            for s in failed:
                state.status[(0, s)] = cl.FAILED
            try:
                cl.reassign_takeover(state)
                table[str(pattern)] = [state.executor[(0, s)][1] for s in range(R)]
            except UnrecoverableRankError:
                table[str(pattern)] = None
        router[str(R)] = table
    with open(os.path.join(OUT, "router.json"), "w") as f:
        json.dump(router, f, separators=(",", ":"))

    # ---- end-to-end run_training at C0 with a permanent victim ----
    raw = {
        "model": dict(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64),
        "cluster": dict(dp=2, pp=2, layers=2),
        "scenario": dict(kind="per_iteration", probability=1.0, recovery_iterations=10**9, victims=[[0, 1]]),
        "run": dict(iterations=4, global_batch=8, seed=0, r=32, tau=100, probe_interval=0),
    }
    cfg = harness.config_from_dict(raw)
    sampler = harness.dt.ShardedSampler(n_ranks=2, seq_len=64, vocab_size=64, seed=0)
    batches = [[[b.tolist() for b in sampler.batch(i, 4)] for i in range(2)] for _ in range(4)]
    res = harness.run_training(cfg)
    final = {name: np.asarray(a, dtype=np.float32) for name, a in res.weights.named()}
    np.savez_compressed(os.path.join(OUT, "c0_training_weights.npz"), **final)
    with open(os.path.join(OUT, "c0_training.json"), "w") as f:
        json.dump({"config": raw, "rows": res.rows, "events": res.events, "batches": batches}, f)
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
