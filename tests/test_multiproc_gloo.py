"""CPU, world_size 2 (gloo): the N>1 host path.

Every process runs the replicated control plane and builds its own ring plan;
the plans must agree bit for bit (all-gathered hash), and the Eq. (1)
"pre-weight locally, all-reduce(sum)" exchange the engine performs on its
flat gradient buffer must equal the reference's subset average
(cluster.py:292-322, restated in oracle/cluster_ref.aggregate)."""

import hashlib
import json
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cluster_ref
from paper_2510_16415_b200 import cluster as cl
from paper_2510_16415_b200.engine import ring_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, R=4):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = 3
    # replicated control plane: same scenario, same seed on every process
    state = cl.ClusterState(cl.ClusterConfig(dp=1, pp=R, layers=R),
                            cl.FailureScenario(kind="per_iteration", probability=0.1, recovery_iterations=2, seed=11))
    digests = []
    rng = np.random.Generator(np.random.PCG64(5))
    names = ["embedding"] + [f"layers.{l}.{k}" for l in range(L) for k in cluster_ref.MHA + cluster_ref.FFN] + \
            ["final_norm", "unembedding"]
    results = []
    for it in range(12):
        try:
            cl.step_cluster(state, 0.0, it)
        except Exception:
            break
        failed = {s for s in range(R) if state.status[(0, s)] == cl.FAILED}
        route, lean, a_mha, skip = ring_plan(R, failed, L)
        digests.append(hashlib.sha256(json.dumps([route, lean, a_mha, skip]).encode()).hexdigest())
        # synthetic per-rank gradients; lean ranks produce no MHA gradients
        per_rank = []
        for j in range(R):
            g = {n: rng.normal(size=3) for n in names}
            if lean[j]:
                for l in range(L):
                    for k in cluster_ref.MHA:
                        g[f"layers.{l}.{k}"] = np.full(3, np.nan)  # poison: must never leak
            per_rank.append(g)
        # this process executes the ranks routed to GPU == process rank (R logical ranks on `world` procs: j % world)
        local = {n: torch.zeros(3, dtype=torch.float64) for n in names}
        for j in range(R):
            if route[j] % world != rank:
                continue
            for n in names:
                is_mha = n.startswith("layers.") and n.split(".")[2] in cluster_ref.MHA
                if is_mha and lean[j]:
                    continue  # select, not multiply
                alpha = a_mha if is_mha else 1.0 / R
                local[n] += alpha * torch.from_numpy(per_rank[j][n])
        flat = torch.cat([local[n] for n in names])
        dist.all_reduce(flat)
        active = {(l, k): [j for j in range(R) if not lean[j]] if k in cluster_ref.MHA else list(range(R))
                  for l in range(L) for k in cluster_ref.MHA + cluster_ref.FFN}
        avg, skipped = cluster_ref.aggregate(per_rank, active, L)
        assert sorted(skipped) == sorted(skip)
        off = 0
        for n in names:
            got = flat[off: off + 3].numpy()
            off += 3
            if n in skipped:
                assert np.all(got == 0.0)
            else:
                assert np.allclose(got, avg[n], rtol=1e-12, atol=1e-12), n
        results.append(it)
    gathered = [None] * world
    dist.all_gather_object(gathered, digests)
    assert all(g == gathered[0] for g in gathered)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump({"iterations": results, "digests": digests}, f)
    dist.destroy_process_group()


def test_two_process_plan_agreement_and_eq1_exchange(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r0 = json.load(open(tmp_path / "rank0.json"))
    r1 = json.load(open(tmp_path / "rank1.json"))
    assert r0 == r1 and len(r0["iterations"]) >= 5


def test_four_process_eight_rank_plan_agreement_and_eq1_exchange(tmp_path):
    """The 8-rank ring (the 8-GPU layout's control plane) on 4 processes."""
    world = 4
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), 8), nprocs=world, join=True)
    docs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    assert all(d == docs[0] for d in docs) and len(docs[0]["iterations"]) >= 5
