"""ORACLE (test infrastructure only): restatement of the cluster control plane.

cluster.py: ring-successor NDB takeover (:190-239), failure injection
(:136-168), recovery (:171-187), step order (:242-250), invariants
(:253-271), active sets (:274-289) and Eq. (1) aggregation (:292-322).
State is plain dicts keyed by (dp_rank, stage).
"""

from __future__ import annotations

import numpy as np

H, F, D = "healthy", "failed", "doubled"
MHA = ("q", "k", "v", "o", "norm_mha")
FFN = ("gate", "up", "down", "norm_ffn")
GLOBAL = ("embedding", "final_norm", "unembedding")


def ring_takeover(pp: int, failed: set[int]) -> dict[int, int] | None:
    """Failed stage -> adopter stage; descending failed order, first ring
    successor that is neither failed nor already adopting (cluster.py:207-218)."""
    adopter_of: dict[int, int] = {}
    busy: set[int] = set()
    for s in sorted(failed, reverse=True):
        t = next(((s + h) % pp for h in range(1, pp) if (s + h) % pp not in failed and (s + h) % pp not in busy),
                 None)
        if t is None:
            return None
        busy.add(t)
        adopter_of[s] = t
    return adopter_of


def boundaries(layers: int, pp: int, explicit=None):
    """cluster.py:56-62: round(s * L / pp) (Python banker's rounding)."""
    return tuple(explicit) if explicit is not None else tuple(round(s * layers / pp) for s in range(pp + 1))


def stage_of(layer: int, bounds) -> int:
    return next(s for s in range(len(bounds) - 1) if bounds[s] <= layer < bounds[s + 1])


class Cluster:
    """Minimal restatement of ClusterState + step_cluster."""

    def __init__(self, dp, pp, layers, kind="none", p=0.0, rec_iters=1, interval=1800.0, rec_time=7200.0,
                 victims=None, seed=0, bounds=None):
        self.dp, self.pp, self.layers = dp, pp, layers
        self.kind, self.p, self.rec_iters = kind, p, rec_iters
        self.interval, self.rec_time = interval, rec_time
        self.victims = None if victims is None else {tuple(v) for v in victims}
        self.rng = np.random.Generator(np.random.PCG64(seed))
        self.st = {(i, s): H for i in range(dp) for s in range(pp)}
        self.ex = {n: n for n in self.st}
        self.until: dict = {}
        self.next_fail = interval
        self.bounds = boundaries(layers, pp, bounds)

    def _ev(self, t, it, kind, node, **det):
        return {"time": float(t), "iteration": int(it), "kind": kind, "node": list(node), "details": det}

    def step(self, t, it):
        evs = []
        clock = it if self.kind == "per_iteration" else t
        for n in sorted(n for n, u in self.until.items() if clock >= u):  # recoveries first (:244-246)
            old = self.ex[n]
            self.st[n] = H
            del self.until[n]
            self.ex[n] = n
            if old != n and self.st[old] == D and sum(1 for s in range(self.pp) if self.ex[(n[0], s)] == old) == 1:
                self.st[old] = H
            evs.append(self._ev(t, it, "recover", n, fetched_from=list(old)))
        if self.kind == "per_iteration" and self.p != 0.0:  # (:141-152)
            for n in sorted(self.st):
                if self.st[n] != H or (self.victims is not None and n not in self.victims):
                    continue
                if self.rng.random() < self.p:
                    self.st[n] = F
                    self.until[n] = it + self.rec_iters
                    evs.append(self._ev(t, it, "fail", n))
        elif self.kind == "scheduled":  # (:154-168)
            while t >= self.next_fail:
                b = self.next_fail
                self.next_fail += self.interval
                cands = [n for n in sorted(self.st) if self.st[n] == H]
                if self.victims is not None:
                    cands = [n for n in cands if n in self.victims]
                if not cands:
                    continue
                n = cands[int(self.rng.integers(len(cands)))]
                self.st[n] = F
                self.until[n] = b + self.rec_time
                evs.append(self._ev(b, it, "fail", n))
        for i in range(self.dp):  # NDB reassignment (:190-239)
            failed = {s for s in range(self.pp) if self.st[(i, s)] == F}
            take = ring_takeover(self.pp, failed)
            if take is None:
                raise RuntimeError(f"unrecoverable DP rank {i}")
            for s in range(self.pp):
                if s not in failed:
                    self.ex[(i, s)] = (i, s)
            for s in sorted(failed, reverse=True):
                new = (i, take[s])
                if self.ex[(i, s)] != new:
                    self.ex[(i, s)] = new
                    lay = list(range(self.bounds[s], self.bounds[s + 1]))
                    evs.append(self._ev(t, it, "adopt", new, stage=s, layers=lay,
                                        fetched_from_rank=(i + 1) % self.dp if self.dp > 1 else i))
            adopters = set(take.values())
            for s in range(self.pp):
                if self.st[(i, s)] != F:
                    self.st[(i, s)] = D if s in adopters else H
        return evs

    def lean(self, i, layer) -> bool:
        """harness.py:392-400: layer is lean iff its executor is not healthy."""
        return self.st[self.ex[(i, stage_of(layer, self.bounds))]] != H

    def active(self, layer, kind):
        """cluster.py:274-289."""
        if kind in FFN:
            return list(range(self.dp))
        s = stage_of(layer, self.bounds)
        return [i for i in range(self.dp) if self.st[self.ex[(i, s)]] == H]

    def affected(self):
        """cluster.py:115-123."""
        return [i for i in range(self.dp) if any(self.st[self.ex[(i, s)]] != H for s in range(self.pp))]


def aggregate(per_rank: list[dict], active: dict, layers: int):
    """cluster.py:292-322: ascending-rank sums / |N|; empty sets -> skipped."""
    n = len(per_rank)
    out, skipped = {}, []
    for name in GLOBAL:
        out[name] = sum(per_rank[i][name] for i in range(n)) / n
    for l in range(layers):
        for kind in MHA + FFN:
            ranks = active[(l, kind)]
            name = f"layers.{l}.{kind}"
            if not ranks:
                skipped.append(name)
                continue
            acc = per_rank[ranks[0]][name].copy()
            for i in ranks[1:]:
                acc = acc + per_rank[i][name]
            out[name] = acc / len(ranks)
    return out, skipped
