"""Cheap backward for nodes running a doubled workload — mirror of faultsim.approx.

(i) the attention backward is skipped (identity path only), (ii) the FFN
intermediates are recomputed from x1 on the tensor cores with SwiGLU fused
into the GEMM epilogue, (iii) FFN weight gradients are projected onto the
top-r right singular subspace, G = d2^T (inp2 V1) V1^T (approx.py:24-42),
with per-(rank, layer) bases refreshed every `refresh_period` local steps.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib, model as mdl, runtime
from .errors import ContractViolation
from .linalg import SvdConfig, refresh_bases, top_r_right_singular_vectors

FFN_KINDS = mdl.FFN_WEIGHT_KINDS


def _pad16(r: int) -> int:
    return max(16, (r + 15) // 16 * 16)


def lowrank_wgrad(g_y: torch.Tensor, x: torch.Tensor, v1: torch.Tensor, precision: str = "fp32") -> torch.Tensor:
    """approx.py:24-42: g_y (out, b), x (in, b), v1 (in, r) -> (out, in) fp32,
    computed as g_y (x^T v1) v1^T in exactly that association order."""
    for name, t in (("g_y", g_y), ("x", x), ("v1", v1)):
        if t.ndim != 2:
            raise ContractViolation(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if g_y.shape[1] != x.shape[1]:
        raise ContractViolation(f"g_y and x batch dims differ: {tuple(g_y.shape)} vs {tuple(x.shape)}")
    if v1.shape[0] != x.shape[0]:
        raise ContractViolation(f"v1 rows must match x rows: {tuple(v1.shape)} vs {tuple(x.shape)}")
    n_out, b = g_y.shape
    n_in, r = v1.shape
    cfg = mdl.ModelConfig(vocab=8, hidden=8, heads=1, ffn_intermediate=8, layers=1, seq_len=1)
    eng = runtime.engine_for(cfg, precision)
    dt = eng.dtype
    # Zero-pad every dim to 16-byte rows for TMA (exact: zero rows/columns
    # contribute nothing and the padded output block is sliced away).
    p8 = lambda n: (n + 7) // 8 * 8
    bp, rp, op_, ip = p8(b), p8(r), p8(n_out), p8(n_in)
    gp = torch.zeros(op_, bp, dtype=dt, device="cuda")
    xp = torch.zeros(ip, bp, dtype=dt, device="cuda")
    vp = torch.zeros(ip, rp, dtype=dt, device="cuda")
    gp[:n_out, :b] = g_y.to("cuda", dt)
    xp[:n_in, :b] = x.to("cuda", dt)
    vp[:n_in, :r] = v1.to("cuda", dt)
    out = torch.zeros(op_, ip, dtype=torch.float32, device="cuda")
    ws, wn = eng.workspace(max(bp, op_, ip), _pad16(rp))
    _lib.call("mecefo_lowrank_wgrad", eng.handle, gp.data_ptr(), xp.data_ptr(), vp.data_ptr(), out.data_ptr(), op_,
              ip, bp, rp, 1.0, ws, wn, runtime.stream_ptr())
    return out[:n_out, :n_in].contiguous()


@dataclass
class ProjectionCache:
    """approx.py:45-63. `basis[kind]` is V1 (in, r_kind) fp32 on device; the
    engine operands (compute precision, rank padded to 16) are derived lazily."""

    rank: int
    refresh_period: int
    step: int = 0
    basis: dict = field(default_factory=dict)
    svd_calls: int = 0
    refreshes: int = 0
    # provenance of the current basis: equal tokens <=> bitwise-equal bases
    # (lets the engine fuse microbatches whose ranks share a basis)
    token: object = None
    _packed: dict = field(default_factory=dict, repr=False)

    def reset(self) -> None:
        """Adoption (harness.py:384-388): forget the basis and the step count.
        The packed engine operands are kept (and overwritten in place by the
        next refresh) so captured CUDA graphs of recurring plans stay valid."""
        self._shapes = {k: tuple(v.shape) for k, v in self.basis.items()}
        self.step = 0
        self.basis.clear()
        self.token = None

    def set_basis(self, kind: str, v1) -> None:
        """Inject a basis (e.g. the reference's seeded V1 for parity)."""
        t = torch.as_tensor(v1).to("cuda", torch.float32).contiguous()
        self.token = ("inject", object())
        old = self.basis.get(kind)
        old_shape = tuple(old.shape) if old is not None else getattr(self, "_shapes", {}).get(kind)
        self.basis[kind] = t
        if old_shape == tuple(t.shape) and self._packed:
            # refresh in place: packed engine operands keep their addresses
            # (captured CUDA graphs read them by pointer)
            for (prec, rp), (_, keep) in self._packed.items():
                i = FFN_KINDS.index(kind)
                v, vt = keep[2 + 2 * i], keep[3 + 2 * i]
                v.zero_()
                v[:t.shape[0], :t.shape[1]] = t.to(v.dtype)
                vt.copy_(v.t())
                if kind in ("gate", "up") and keep[1] is not None:
                    keep[1][:, i * rp:(i + 1) * rp].copy_(v)
            return
        self._packed.clear()

    def packed(self, precision: str, down_rows: int | None = None):
        """Projection struct + keep-alive tensors for the engine. down_rows:
        the stored FFN width (V1_down's rows zero-padded to it, model.ffn_storage)."""
        ranks = [int(self.basis[k].shape[1]) for k in FFN_KINDS]
        rp = _pad16(max(ranks))
        key = (precision, rp)
        if key not in self._packed:
            dt = runtime.compute_dtype(precision)
            dev = self.basis["gate"].device
            n_gu = self.basis["gate"].shape[0]
            # gate/up transposed bases stacked: one GEMM forms [P_gate | P_up]
            vt_gu = torch.zeros(2 * rp, n_gu, dtype=dt, device=dev)
            tensors = {}
            for i, k in enumerate(FFN_KINDS):
                b = self.basis[k]
                n_in, r = b.shape
                rows = down_rows if (k == "down" and down_rows) else n_in
                v = torch.zeros(rows, rp, dtype=dt, device=dev)
                v[:n_in, :r] = b.to(dt)
                if k in ("gate", "up") and n_in == n_gu:
                    vt = vt_gu[i * rp:(i + 1) * rp]
                    vt.copy_(v.t())
                else:
                    vt = v.t().contiguous()
                tensors[k] = (v, vt)
            packed_gu = self.basis["up"].shape[0] == n_gu
            # [V1_gate | V1_up] side by side for the merged up-projection
            v1_gu = torch.cat([tensors["gate"][0], tensors["up"][0]], dim=1).contiguous() if packed_gu else None
            keep = [vt_gu, v1_gu] + [t for k in FFN_KINDS for t in tensors[k]]
            st = _lib.Projection((ctypes.c_int32 * 3)(*ranks), rp,
                                 (ctypes.c_void_p * 3)(*[tensors[k][0].data_ptr() for k in FFN_KINDS]),
                                 (ctypes.c_void_p * 3)(*[tensors[k][1].data_ptr() for k in FFN_KINDS]),
                                 v1_gu.data_ptr() if packed_gu else None, vt_gu.data_ptr() if packed_gu else None)
            self._packed[key] = (st, keep)
        st, keep = self._packed[key]
        return st, keep, rp


def refresh_projections(cache: ProjectionCache, lw: mdl.LayerWeights, svd: SvdConfig, budgeted: bool = False) -> None:
    """approx.py:66-87: refresh iff step % period == 0 or no basis; does not
    advance the step counter."""
    if cache.refresh_period < 1:
        raise ContractViolation("refresh_period must be >= 1")
    if cache.step % cache.refresh_period != 0 and cache.basis:
        return
    if cache.basis and getattr(cache, "_fresh_step", None) == cache.step:
        return  # already refreshed for this step by a batched pre-refresh
    cache.refreshes += 1
    mats = [lw.kind(kind) for kind in FFN_KINDS]
    ranks = [min(cache.rank, w.shape[1]) for w in mats]
    if budgeted:
        for kind, w, rank in zip(FFN_KINDS, mats, ranks):
            cfg = SvdConfig(rank=rank, tolerance=svd.tolerance, max_iterations=svd.max_iterations, seed=svd.seed)
            cache.set_basis(kind, top_r_right_singular_vectors(w, cfg, budgeted=True))
            cache.svd_calls += 1
        return
    # the three kinds in one batched device solve (each is linalg.py:97-142
    # with SvdConfig(rank=min(r, in), svd.tolerance, svd.max_iterations, svd.seed))
    for kind, v1 in zip(FFN_KINDS, refresh_bases(mats, ranks, svd)):
        cache.set_basis(kind, v1)
        cache.svd_calls += 1


def recompute_ffn(lw: mdl.LayerWeights, x1) -> dict:
    """approx.py:90-96: same kernel as the forward, so bit-identical."""
    return mdl.ffn_forward(lw, x1)


def backward_block_neighbor(cfg: mdl.ModelConfig, lw: mdl.LayerWeights, cache: mdl.BlockCache, dy,
                            proj: ProjectionCache | None = None, svd: SvdConfig | None = None):
    """approx.py:99-134. Returns (dx, {gate, up, down, norm_ffn}); advances
    proj.step by one."""
    if cache.mode != mdl.CACHE_FFN_INPUT_ONLY:
        raise ContractViolation("neighbor backward requires an ffn-input-only cache")
    dy2 = mdl._to_2d(cfg, dy)
    eng = runtime.engine_for(cfg, lw.precision)
    b = dy2.shape[0]
    pst, keep, rp = None, None, 16
    if proj is not None:
        if svd is None:
            raise ContractViolation("projection refresh needs an SvdConfig")
        refresh_projections(proj, lw, svd)
        pst, keep, rp = proj.packed(lw.precision, down_rows=mdl.ffn_storage(cfg))
    dx = torch.empty_like(dy2)
    g = mdl._grad_buffers(cfg, dy2.device, mha=False)
    ws, wn = eng.workspace(b, rp)
    _lib.call("mecefo_backward_block_neighbor", eng.handle, ctypes.byref(lw.struct()), ctypes.byref(cache.struct()),
              dy2.data_ptr(), None, dx.data_ptr(), None, ctypes.byref(mdl._grads_struct(g)),
              ctypes.byref(pst) if pst is not None else None, b, ws, wn, runtime.stream_ptr())
    del keep
    if proj is not None:
        proj.step += 1
    return dx.reshape(dy.shape), mdl._unpack_grads(cfg, g)
