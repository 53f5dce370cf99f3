"""Training driver — drop-in for the step path of faultsim.harness.

`run_training` is harness.py:362-470 on the B200 engine: the replicated
control plane decides failures, NDB takeover, per-(rank, layer) cache modes,
Eq. (1) active sets and skip lists exactly as the reference does; the fused
StepEngine then runs every logical DP rank's microbatch (lean layers through
the neighbour backward), accumulates Eq. (1)-weighted gradients in one flat
buffer and applies the fused AdamW. Metrics rows, event records and the
simulated clock follow harness.py:24,382-464. The rho1/rho2 probes
(harness.py:473-514), finite-difference checks and weight dumps are outside
this tier and are not computed (rho columns stay empty).

`backward_model` / `_rank_pass` mirror harness.py:209-249 per rank (gradient
dicts), built from the block-level engine API.
"""

from __future__ import annotations

import json
import os
import tempfile
from dataclasses import dataclass, field, fields as dc_fields

import numpy as np
import torch

from . import approx, cluster as cl, costmodel as cm, engine as E, model as mdl, optim as op
from .errors import ConfigError, NumericalFailure
from .linalg import SvdConfig
from .pcg import Pcg64Generator

METRICS_HEADER = "iteration,loss,perplexity,rho1,rho2,lr,sim_time_s,affected_ranks"


# ---------------------------------------------------------------------------
# Configuration (harness.py:32-128)
# ---------------------------------------------------------------------------


@dataclass
class RunSettings:
    iterations: int = 200
    global_batch: int = 8
    seed: int = 0
    r: int = 4
    tau: int = 100
    probe_interval: int = 0
    probe_only_under_faults: bool = True
    full_batch_interval: int = 50
    full_batch_windows: int = 8
    flush_interval: int = 50
    base_lr: float | None = None


@dataclass
class CostSettings:
    node_flops_per_s: float = 1e12
    fetch_cost_s: float = 1.0


@dataclass
class DataSettings:
    """harness.py:54-56: the reference default is the embedded char corpus.
    "synthetic" (uniform tokens) is this engine's explicit opt-in."""
    source: str = "corpus"
    path: str | None = None


@dataclass
class RunConfig:
    model: mdl.ModelConfig = field(default_factory=mdl.ModelConfig)
    cluster: cl.ClusterConfig = field(default_factory=lambda: cl.ClusterConfig(dp=4, pp=2, layers=4))
    scenario: cl.FailureScenario = field(default_factory=cl.FailureScenario)
    optimizer: op.OptimConfig = field(default_factory=op.OptimConfig)
    run: RunSettings = field(default_factory=RunSettings)
    cost: CostSettings = field(default_factory=CostSettings)
    data: DataSettings = field(default_factory=DataSettings)

    def __post_init__(self):
        if self.cluster.layers != self.model.layers:
            raise ConfigError("cluster layer count must match the model")
        if self.run.global_batch % self.cluster.dp != 0:
            raise ConfigError("global batch must divide evenly across DP ranks")
        if self.data.path is not None and not os.path.exists(self.data.path):  # harness.py:74-75
            raise ConfigError(f"dataset path does not exist: {self.data.path}")

    @property
    def per_rank_batch(self) -> int:
        return self.run.global_batch // self.cluster.dp

    @property
    def tokens_per_rank(self) -> int:
        return self.per_rank_batch * self.model.seq_len


_SECTIONS = {"model": mdl.ModelConfig, "cluster": cl.ClusterConfig, "scenario": cl.FailureScenario,
             "optimizer": op.OptimConfig, "run": RunSettings, "cost": CostSettings, "data": DataSettings}


def config_from_dict(raw: dict) -> RunConfig:
    """harness.py:111-128: unknown keys rejected; scenario seed = seed*31+7
    unless pinned."""
    unknown = set(raw) - set(_SECTIONS)
    if unknown:
        raise ConfigError(f"unknown top-level key(s): {sorted(unknown)}")
    kwargs = {}
    for section, cls in _SECTIONS.items():
        if section not in raw:
            continue
        sec = raw[section]
        if not isinstance(sec, dict):
            raise ConfigError(f"section {section!r} must be an object")
        bad = set(sec) - {f.name for f in dc_fields(cls)}
        if bad:
            raise ConfigError(f"unknown key(s) in {section!r}: {sorted(bad)}")
        sec = dict(sec)
        if section == "scenario" and sec.get("victims") is not None:
            sec["victims"] = tuple(tuple(v) for v in sec["victims"])
        if section == "cluster" and sec.get("stage_boundaries") is not None:
            sec["stage_boundaries"] = tuple(sec["stage_boundaries"])
        kwargs[section] = cls(**sec)
    cfg = RunConfig(**kwargs)
    if "seed" not in raw.get("scenario", {}):
        sc = cfg.scenario
        cfg.scenario = cl.FailureScenario(kind=sc.kind, probability=sc.probability,
                                          recovery_iterations=sc.recovery_iterations,
                                          failure_interval_s=sc.failure_interval_s,
                                          recovery_time_s=sc.recovery_time_s, victims=sc.victims,
                                          seed=cfg.run.seed * 31 + 7)
    return cfg


def load_config(path: str) -> RunConfig:
    """harness.py:153-159."""
    try:
        with open(path, "r", encoding="utf-8") as f:
            raw = json.load(f)
    except (OSError, json.JSONDecodeError) as exc:
        raise ConfigError(f"cannot read config {path}: {exc}") from exc
    return config_from_dict(raw)


def replace_scenario_seed(cfg: RunConfig, seed: int) -> RunConfig:
    """harness.py:131-150: same run, failure stream reseeded."""
    sc = cfg.scenario
    new_sc = cl.FailureScenario(kind=sc.kind, probability=sc.probability, recovery_iterations=sc.recovery_iterations,
                                failure_interval_s=sc.failure_interval_s, recovery_time_s=sc.recovery_time_s,
                                victims=sc.victims, seed=seed)
    return RunConfig(model=cfg.model, cluster=cfg.cluster, scenario=new_sc, optimizer=cfg.optimizer, run=cfg.run,
                     cost=cfg.cost, data=cfg.data)


def make_sampler(cfg: RunConfig):
    """harness.py:300-307: data.source "corpus"/"teacher" -> data.ShardedSampler
    (bit-exact batches); "synthetic" (this engine's default) -> SyntheticSampler."""
    if cfg.data.source == "synthetic":
        return SyntheticSampler(cfg.cluster.dp, cfg.model.seq_len, cfg.model.vocab, cfg.run.seed)
    from . import data as dt

    return dt.ShardedSampler(n_ranks=cfg.cluster.dp, seq_len=cfg.model.seq_len, vocab_size=cfg.model.vocab,
                             seed=cfg.run.seed, source=cfg.data.source, corpus_path=cfg.data.path)


# ---------------------------------------------------------------------------
# Crash-consistent writers (harness.py:167-201)
# ---------------------------------------------------------------------------


class AtomicFileWriter:
    def __init__(self, path: str | None, header: str | None = None):
        self.path, self.header, self.lines = path, header, []

    def add(self, line: str) -> None:
        self.lines.append(line)

    def flush(self) -> None:
        if self.path is None:
            return
        d = os.path.dirname(os.path.abspath(self.path))
        os.makedirs(d, exist_ok=True)
        fd, tmp = tempfile.mkstemp(dir=d, suffix=".tmp")
        try:
            with os.fdopen(fd, "w", encoding="utf-8") as f:
                if self.header is not None:
                    f.write(self.header + "\n")
                f.writelines(line + "\n" for line in self.lines)
            os.replace(tmp, self.path)
        finally:
            if os.path.exists(tmp):
                os.unlink(tmp)


def _fmt(v) -> str:
    if v is None:
        return ""
    return repr(v) if isinstance(v, float) else str(v)


# ---------------------------------------------------------------------------
# Per-rank mirror API (harness.py:209-249)
# ---------------------------------------------------------------------------


def backward_model(weights, tokens, caches, final_cache, dlogits, modes, proj_caches=None, svd=None) -> dict:
    cfg = weights.cfg
    if modes is None:
        modes = [mdl.CACHE_FULL] * cfg.layers
    dx, grads = mdl.head_backward(weights, final_cache, dlogits)
    for layer in reversed(range(cfg.layers)):
        lw = weights.layers[layer]
        if modes[layer] == mdl.CACHE_FULL:
            dx, lg = mdl.backward_block_exact(cfg, lw, caches[layer], dx)
        else:
            proj = proj_caches.get(layer) if proj_caches is not None else None
            dx, lg = approx.backward_block_neighbor(cfg, lw, caches[layer], dx, proj=proj, svd=svd)
        for kind, g in lg.items():
            grads[f"layers.{layer}.{kind}"] = g
    grads["embedding"] = mdl.embedding_backward(weights, tokens, dx)
    return grads


def _rank_pass(weights, tokens, targets, modes, proj_caches=None, svd=None):
    logits, caches, final_cache = mdl.forward_model(weights, tokens, modes)
    loss, dlogits = mdl.cross_entropy(logits, np.asarray(targets).reshape(-1), cfg=weights.cfg,
                                      precision=weights.precision)
    grads = backward_model(weights, tokens, caches, final_cache, dlogits, modes, proj_caches, svd)
    return loss, grads


# ---------------------------------------------------------------------------
# Training loop (harness.py:362-470)
# ---------------------------------------------------------------------------


@dataclass
class RunResult:
    rows: list
    events: list
    weights: mdl.ModelWeights
    summary: dict


class SyntheticSampler:
    """LLaMA-shaped synthetic batches: uniform tokens, next-token targets,
    one native PCG64 stream per DP rank. The reference's corpus/teacher sampler
    is data.ShardedSampler; any object with .batch(rank, n) -> (tokens, targets)
    plugs in."""

    def __init__(self, n_ranks: int, seq_len: int, vocab: int, seed: int):
        self.T, self.V = seq_len, vocab
        self.rngs = [Pcg64Generator((seed, 0x5E7, i)) for i in range(n_ranks)]  # native PCG64 streams

    def batch(self, rank: int, n: int):
        x = self.rngs[rank].integers(0, self.V, size=(n, self.T + 1))
        return x[:, :-1], x[:, 1:]


def _summary(rows):
    if not rows:
        return {"iterations": 0}
    tail = rows[-min(50, len(rows)):]
    return {"iterations": len(rows), "final_loss": float(np.mean([r["loss"] for r in tail])),
            "last_loss": rows[-1]["loss"], "max_rho1": None, "sim_time_s": rows[-1]["sim_time_s"]}


def run_training(cfg: RunConfig, out_dir: str | None = None, quiet: bool = True, precision: str = "fp32",
                 sampler=None, svd: SvdConfig | None = None, svd_budgeted: bool = False) -> RunResult:
    """The fault-tolerant loop (harness.py:362-470) on the B200 engine."""
    if cfg.run.probe_interval > 0:
        raise ConfigError("rho probes (harness.py:473-514) are outside this engine's scope; set probe_interval=0")
    n = cfg.cluster.dp
    weights = mdl.init_weights(cfg.model, seed=cfg.run.seed, precision=precision)
    svd = svd or SvdConfig(rank=cfg.run.r, tolerance=1e-9, max_iterations=3000, seed=cfg.run.seed + 23)
    eng = E.StepEngine(cfg.model, precision=precision, seqs_per_microbatch=cfg.per_rank_batch, r=cfg.run.r,
                       tau=cfg.run.tau, optim_cfg=cfg.optimizer, weights=weights, svd=svd,
                       svd_budgeted=svd_budgeted)
    state = cl.ClusterState(cfg.cluster, cfg.scenario)
    if sampler is None:
        sampler = make_sampler(cfg)
    base_lr = cfg.run.base_lr if cfg.run.base_lr is not None else cfg.optimizer.lr
    metrics = AtomicFileWriter(os.path.join(out_dir, "metrics.csv") if out_dir else None, METRICS_HEADER)
    events_out = AtomicFileWriter(os.path.join(out_dir, "events.jsonl") if out_dir else None)
    L = cfg.model.layers
    stage_of = [cfg.cluster.stage_of_layer(l) for l in range(L)]
    rows, all_events = [], []
    sim_time = 0.0
    try:
        for it in range(cfg.run.iterations):
            events = cl.step_cluster(state, sim_time, it)
            for ev in events:
                if ev["kind"] == "adopt":
                    for layer in ev["details"]["layers"]:
                        eng.reset_projection(ev["node"][0], layer)  # harness.py:384-388
                all_events.append(ev)
                events_out.add(json.dumps(ev))
            lean_stage = state.lean_mask()  # (dp, pp): executor not healthy
            lean = [[bool(lean_stage[i, stage_of[l]]) for l in range(L)] for i in range(n)]
            n_mha = [sum(1 for i in range(n) if not lean[i][l]) for l in range(L)]  # cluster.py:280-284
            skip = [f"layers.{l}.{k}" for l in range(L) if n_mha[l] == 0 for k in cl.MHA_GRAD_KINDS]
            lr = op.lr_at(it + 1, cfg.run.iterations, base_lr)
            mbs = []
            for i in range(n):
                tk, tg = sampler.batch(i, cfg.per_rank_batch)
                mbs.append(E.Microbatch(
                    rank=i, tokens=torch.as_tensor(np.asarray(tk), dtype=torch.int64).cuda(),
                    targets=torch.as_tensor(np.asarray(tg), dtype=torch.int64).cuda(), lean=lean[i],
                    alpha_mha=[None if lean[i][l] else 1.0 / n_mha[l] for l in range(L)], alpha_ffn=1.0 / n,
                    alpha_global=1.0 / n))
            losses = eng.step(mbs, n, lr, skip=skip, check=True).cpu().numpy().astype(np.float64)
            loss = float(sum(losses.tolist()) / n)
            if not np.isfinite(loss):
                raise NumericalFailure(f"non-finite loss at iteration {it}")
            affected = state.affected_ranks()
            worst, _, _, _ = cm.iteration_cost(state, cfg.model, cm.POLICY_APPROX, cfg.run.r, cfg.run.tau,
                                               cfg.tokens_per_rank)
            fetches = sum(1 for ev in events if ev["kind"] in ("adopt", "recover"))
            sim_time += worst / cfg.cost.node_flops_per_s + fetches * cfg.cost.fetch_cost_s
            row = {"iteration": it, "loss": loss, "perplexity": float(np.exp(loss)), "rho1": None, "rho2": None,
                   "lr": lr, "sim_time_s": sim_time, "affected_ranks": len(affected)}
            rows.append(row)
            metrics.add(",".join(_fmt(row[k]) for k in METRICS_HEADER.split(",")))
            if out_dir and (it + 1) % cfg.run.flush_interval == 0:
                metrics.flush()
                events_out.flush()
            if not quiet and (it + 1) % 100 == 0:
                print(f"[train] iter {it + 1}/{cfg.run.iterations} loss {loss:.4f}")
    finally:
        metrics.flush()
        events_out.flush()
    if out_dir:
        dump_weights(weights, out_dir)  # harness.py:468-469
    return RunResult(rows=rows, events=all_events, weights=weights, summary=_summary(rows))


# --- weight wire format (harness.py:635-665: final_weights.bin + .json) -----

def pack_weights(layout, master: np.ndarray, cfg: mdl.ModelConfig | None = None):
    """Canonical-order dense little-endian float64 blob + manifest from the
    aligned flat parameter store (padding between groups — and, given cfg,
    the FFN-width padding inside gate/up/down — dropped: reference shapes)."""
    params, chunks, off = [], [], 0
    for name, shape, src in layout:
        block = master[src: src + int(np.prod(shape))].reshape(shape)
        if cfg is not None:
            block = mdl.logical_view(cfg, name, block)
        n = block.size
        params.append({"name": name, "shape": list(block.shape), "offset_elems": off})
        chunks.append(np.ascontiguousarray(block).reshape(-1))
        off += n
    blob = np.concatenate(chunks).astype("<f8") if chunks else np.zeros(0, "<f8")
    return blob, {"dtype": "<f8", "total_elems": off, "params": params}


def unpack_weights(layout, total: int, blob: np.ndarray, manifest: dict,
                   cfg: mdl.ModelConfig | None = None) -> np.ndarray:
    """Inverse of pack_weights into an aligned fp32 flat store; names and
    shapes must match the model's (reference) shapes (ContractViolation
    otherwise); FFN padding stays zero."""
    from .errors import ContractViolation

    want = {name: (tuple(mdl.logical_shape(cfg, name, shape)) if cfg is not None else tuple(shape), shape, src)
            for name, shape, src in layout}
    host = np.zeros(total, dtype=np.float32)
    seen = set()
    for e in manifest["params"]:
        name, shape = e["name"], tuple(e["shape"])
        if name not in want or want[name][0] != shape:
            raise ContractViolation(f"final_weights.json: unexpected parameter {name} {shape}")
        n = int(np.prod(shape))
        start = int(e["offset_elems"])
        if start + n > blob.size:
            raise ContractViolation(f"final_weights.bin too short for {name}")
        _, sshape, src = want[name]
        block = host[src: src + int(np.prod(sshape))].reshape(sshape)
        if cfg is not None:
            block = mdl.logical_view(cfg, name, block)
        block[...] = blob[start: start + n].reshape(shape)
        seen.add(name)
    missing = set(want) - seen
    if missing:
        raise ContractViolation(f"final_weights.json lacks {sorted(missing)[:3]}")
    return host


def dump_weights(weights: mdl.ModelWeights, out_dir: str) -> None:
    """harness.py:635-651: one device->host copy of the fp32 master store,
    written as final_weights.bin (<f8, canonical order) + final_weights.json."""
    os.makedirs(out_dir, exist_ok=True)
    blob, manifest = pack_weights(weights.layout, weights.master.detach().cpu().numpy(), weights.cfg)
    tmp = os.path.join(out_dir, "final_weights.bin.tmp")
    blob.tofile(tmp)
    os.replace(tmp, os.path.join(out_dir, "final_weights.bin"))
    with open(os.path.join(out_dir, "final_weights.json"), "w", encoding="utf-8") as f:
        json.dump(manifest, f, indent=2)


def load_weights(cfg: mdl.ModelConfig, out_dir: str, precision: str = "fp32") -> mdl.ModelWeights:
    """harness.py:654-665: read the dump back into a device store (one
    host->device copy, then the compute-precision shadow is refreshed)."""
    with open(os.path.join(out_dir, "final_weights.json"), "r", encoding="utf-8") as f:
        manifest = json.load(f)
    blob = np.fromfile(os.path.join(out_dir, "final_weights.bin"), dtype="<f8")
    w = mdl.ModelWeights(cfg, precision)
    host = unpack_weights(w.layout, w.total, blob, manifest, cfg)
    w.master.copy_(torch.from_numpy(host).to(w.device))
    w.sync_shadow()
    return w
