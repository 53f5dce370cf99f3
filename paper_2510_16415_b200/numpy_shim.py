"""numpy <-> device bridge: runs the reference's block operators on the B200
engine from inside the reference's own harness (Callers).

The reference dispatches its block operators by module-attribute lookup —
`forward_model` calls `forward_block` (faultsim/model.py:461-463),
`backward_model` calls `mdl.backward_block_exact` and
`approx.backward_block_neighbor` (faultsim/harness.py:226-235) — so pointing a
reference training loop at the engine is a matter of replacing those three
attributes. `install(faultsim)` does exactly that: each replacement takes the
reference's argument types (float64 numpy activations, a faultsim
LayerWeights, a faultsim BlockCache, a faultsim ProjectionCache/SvdConfig),
uploads them, runs the engine's C-ABI through this package's mirror
(`model.forward_block`, `model.backward_block_exact`,
`approx.backward_block_neighbor`) and hands float64 numpy results back, with
the reference's side effects (ProjectionCache step / basis / counters).

The host numpy weights stay the source of truth (the reference updates them
in place, faultsim/optim.py:71,92), so a layer is uploaded on each call; the
device caches ride inside the returned BlockCache objects. Heads, loss,
embedding and the optimizer stay the reference's. No CPU fallback: without
the CUDA library every call raises EngineUnavailable.
"""

from __future__ import annotations

import numpy as np
import torch

from . import approx, linalg, model as mdl
from .errors import ContractViolation


class _BridgedCache:
    """Stands in for faultsim.model.BlockCache (model.py:376-381): the
    reference fields (mode, x, x1 as float64 numpy, full = None or a marker)
    plus the engine's device cache."""

    def __init__(self, mode: str, x: np.ndarray, x1: np.ndarray, dev: mdl.BlockCache):
        self.mode = mode
        self.x = x
        self.x1 = x1
        self.full = {"device": True} if mode == mdl.CACHE_FULL else None
        self.dev = dev


class DeviceBridge:
    """Block operators with the reference's signatures, computed on cuda."""

    def __init__(self, fs, precision: str = "fp32"):
        self.fs = fs
        self.precision = precision
        self._cfgs: dict = {}

    # -- conversions ---------------------------------------------------------
    def _cfg(self, cfg_ref) -> mdl.ModelConfig:
        key = (cfg_ref.vocab, cfg_ref.hidden, cfg_ref.heads, cfg_ref.ffn_intermediate, cfg_ref.seq_len,
               cfg_ref.rope)
        if key not in self._cfgs:
            # one layer, vocab 1: the block operators never touch the embeddings
            self._cfgs[key] = mdl.ModelConfig(vocab=1, hidden=cfg_ref.hidden, heads=cfg_ref.heads,
                                              ffn_intermediate=cfg_ref.ffn_intermediate, layers=1,
                                              seq_len=cfg_ref.seq_len, rope=cfg_ref.rope)
        return self._cfgs[key]

    def _layer(self, cfg: mdl.ModelConfig, lw_ref) -> mdl.LayerWeights:
        arrays = {f"layers.0.{k}": lw_ref.kind(k) for k in mdl.LAYER_PARAM_KINDS}
        arrays["embedding"] = np.zeros((1, cfg.hidden))
        arrays["final_norm"] = np.ones(cfg.hidden)
        arrays["unembedding"] = np.zeros((1, cfg.hidden))
        return mdl.from_numpy(cfg, arrays, precision=self.precision).layers[0]

    @staticmethod
    def _dev(x) -> torch.Tensor:
        return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to("cuda", torch.float32)

    @staticmethod
    def _host(t: torch.Tensor, like: np.ndarray) -> np.ndarray:
        return t.detach().to(torch.float64).cpu().numpy().reshape(like.shape)

    # -- faultsim.model.forward_block (model.py:398-418) ---------------------
    def forward_block(self, cfg_ref, lw_ref, x, mode=mdl.CACHE_FULL):
        if mode not in (mdl.CACHE_FULL, mdl.CACHE_FFN_INPUT_ONLY):
            raise ContractViolation(f"unknown cache mode {mode!r}")
        x = np.asarray(x)
        x3 = self.fs.model._to_btm(cfg_ref, x)  # the reference's own shape contract
        cfg = self._cfg(cfg_ref)
        y, dev = mdl.forward_block(cfg, self._layer(cfg, lw_ref), self._dev(x3), mode)
        x1 = self._host(dev.x1, x3)
        return self._host(y, x), _BridgedCache(mode, x3, x1, dev)

    # -- faultsim.model.backward_block_exact (model.py:421-437) --------------
    def backward_block_exact(self, cfg_ref, lw_ref, cache, dy):
        if cache.mode != mdl.CACHE_FULL:
            raise ContractViolation("exact backward requires a full activation cache")
        dy = np.asarray(dy)
        cfg = self._cfg(cfg_ref)
        dx, g = mdl.backward_block_exact(cfg, self._layer(cfg, lw_ref), cache.dev,
                                         self._dev(self.fs.model._to_btm(cfg_ref, dy)))
        return self._host(dx, dy), {k: v.detach().to(torch.float64).cpu().numpy() for k, v in g.items()}

    # -- faultsim.approx.backward_block_neighbor (approx.py:99-134) ----------
    def backward_block_neighbor(self, cfg_ref, lw_ref, cache, dy, proj=None, svd=None):
        if cache.mode != mdl.CACHE_FFN_INPUT_ONLY:
            raise ContractViolation("neighbor backward requires an ffn-input-only cache")
        dy = np.asarray(dy)
        cfg = self._cfg(cfg_ref)
        lw = self._layer(cfg, lw_ref)
        pc = None
        sv = None
        if proj is not None:
            if svd is None:
                raise ContractViolation("projection refresh needs an SvdConfig")
            # the reference cache's schedule decides (approx.py:74-75); a due
            # refresh runs on the device and is written back to the reference
            # cache with its counters (approx.py:76-87)
            pc = approx.ProjectionCache(rank=proj.rank, refresh_period=proj.refresh_period, step=proj.step)
            for kind, v in proj.basis.items():
                pc.set_basis(kind, v)
            sv = linalg.SvdConfig(rank=svd.rank, tolerance=svd.tolerance, max_iterations=svd.max_iterations,
                                  seed=svd.seed)
        dx, g = approx.backward_block_neighbor(cfg, lw, cache.dev, self._dev(self.fs.model._to_btm(cfg_ref, dy)),
                                               proj=pc, svd=sv)
        if proj is not None:
            if pc.refreshes:
                proj.refreshes += pc.refreshes
                proj.svd_calls += pc.svd_calls
                for kind, v in pc.basis.items():
                    proj.basis[kind] = v.detach().to(torch.float64).cpu().numpy()
            proj.step += 1
        return self._host(dx, dy), {k: v.detach().to(torch.float64).cpu().numpy() for k, v in g.items()}


def install(fs, precision: str = "fp32", monkeypatch=None) -> DeviceBridge:
    """Point a reference faultsim package at the engine: replaces
    faultsim.model.forward_block / backward_block_exact and
    faultsim.approx.backward_block_neighbor (the attributes its harness looks
    up, harness.py:226-235, model.py:461-463). With a pytest `monkeypatch`
    the replacement is undone at test teardown."""
    br = DeviceBridge(fs, precision)
    targets = ((fs.model, "forward_block", br.forward_block),
               (fs.model, "backward_block_exact", br.backward_block_exact),
               (fs.approx, "backward_block_neighbor", br.backward_block_neighbor))
    for mod, name, fn in targets:
        if monkeypatch is not None:
            monkeypatch.setattr(mod, name, fn)
        else:
            setattr(mod, name, fn)
    return br
