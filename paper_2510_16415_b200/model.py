"""Decoder-only transformer on the B200 engine — mirror of faultsim.model.

Same names, argument order, shapes and cache-mode semantics as
pkg/src/faultsim/model.py, on CUDA tensors. All arithmetic runs in
libmecefo.so (tcgen05 GEMMs in bf16 mode, fp32 FFMA in fp32 mode); this
module only allocates outputs and marshals pointers.

HBM layout: the parameters live in ONE flat fp32 buffer in the reference's
canonical order (model.py:35,101-108), each group aligned to 64 elements, so
q|k|v and gate|up are contiguous (3m, m) and (2f, m) matrices the engine
reads as single operands. bf16 mode keeps a flat bf16 operand shadow with the
same offsets, refreshed by the fused AdamW kernel.

The FFN width is stored padded to fp = mecefo_padded_ffn(f) (a multiple of 8,
16-byte bf16 rows; LLaMA-1B's f = 5461 -> 5464): gate/up are (fp, m) blocks
whose first f rows are the parameter, down is (m, fp) whose first f columns
are. The pads are zero and stay zero (zero rows/columns contribute nothing,
their gradients are zero, AdamW keeps a zero weight at zero), so the step is
exactly the unpadded one; every reference-facing accessor returns the
logical (f-wide) view.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, runtime
from .errors import ContractViolation
from .linalg import seeded_gaussian

RMS_EPS = 1e-6
INIT_STD = 0.02

CACHE_FULL = "full"
CACHE_FFN_INPUT_ONLY = "ffn_input_only"

MHA_WEIGHT_KINDS = ("q", "k", "v", "o")
FFN_WEIGHT_KINDS = ("gate", "up", "down")
MATRIX_KINDS = MHA_WEIGHT_KINDS + FFN_WEIGHT_KINDS
LAYER_PARAM_KINDS = ("q", "k", "v", "o", "norm_mha", "gate", "up", "down", "norm_ffn")

_MODE_CODE = {CACHE_FULL: _lib.CACHE_FULL, CACHE_FFN_INPUT_ONLY: _lib.CACHE_FFN_INPUT_ONLY}
_ALIGN = 64


@dataclass(frozen=True)
class ModelConfig:
    """model.py:40-61."""

    vocab: int = 64
    hidden: int = 32
    heads: int = 4
    ffn_intermediate: int = 64
    layers: int = 4
    seq_len: int = 32
    rope: bool = True

    def __post_init__(self):
        for name in ("vocab", "hidden", "heads", "ffn_intermediate", "layers", "seq_len"):
            if getattr(self, name) < 1:
                raise ContractViolation(f"{name} must be >= 1")
        if self.hidden % self.heads != 0:
            raise ContractViolation("hidden must be divisible by heads")
        if self.rope and (self.hidden // self.heads) % 2 != 0:
            raise ContractViolation("rotary positions need an even head dim")

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def ffn_storage(cfg: ModelConfig) -> int:
    """Stored FFN width (include/mecefo.h mecefo_padded_ffn)."""
    return (cfg.ffn_intermediate + 7) // 8 * 8


def logical_shape(cfg: ModelConfig, name: str, shape: tuple) -> tuple:
    """The reference's shape of a parameter stored as `shape`."""
    f, fp = cfg.ffn_intermediate, ffn_storage(cfg)
    if fp == f or not name.startswith("layers."):
        return tuple(shape)
    kind = name.rsplit(".", 1)[1]
    if kind in ("gate", "up"):
        return (f, shape[1])
    if kind == "down":
        return (shape[0], f)
    return tuple(shape)


def logical_view(cfg: ModelConfig, name: str, storage: torch.Tensor) -> torch.Tensor:
    """Reference-shaped view of a parameter's storage block (slices off the
    FFN padding; a strided view for down)."""
    f, fp = cfg.ffn_intermediate, ffn_storage(cfg)
    if fp == f or not name.startswith("layers."):
        return storage
    kind = name.rsplit(".", 1)[1]
    if kind in ("gate", "up"):
        return storage[:f]
    if kind == "down":
        return storage[:, :f]
    return storage


def _param_layout(cfg: ModelConfig):
    """(name, storage shape, offset) in canonical order; groups aligned to 64
    elements, q|k|v and gate|up packed back to back; FFN width padded."""
    m, f, v = cfg.hidden, ffn_storage(cfg), cfg.vocab
    shapes = {"q": (m, m), "k": (m, m), "v": (m, m), "o": (m, m), "norm_mha": (m,), "gate": (f, m), "up": (f, m),
              "down": (m, f), "norm_ffn": (m,)}
    out = []
    off = 0

    def add(name, shape, align=True):
        nonlocal off
        if align:
            off = (off + _ALIGN - 1) // _ALIGN * _ALIGN
        out.append((name, shape, off))
        off += int(np.prod(shape))

    add("embedding", (v, m))
    for l in range(cfg.layers):
        for kind in LAYER_PARAM_KINDS:
            add(f"layers.{l}.{kind}", shapes[kind], align=kind not in ("k", "v", "up"))
    add("final_norm", (m,))
    add("unembedding", (v, m))
    total = (off + _ALIGN - 1) // _ALIGN * _ALIGN
    return out, total


class LayerWeights:
    """Views of one layer inside ModelWeights (model.py:64-90)."""

    def __init__(self, owner: "ModelWeights", layer: int):
        self._owner = owner
        self.layer = layer

    def kind(self, name: str) -> torch.Tensor:
        return self._owner.get(f"layers.{self.layer}.{name}")

    w_q = property(lambda self: self.kind("q"))
    w_k = property(lambda self: self.kind("k"))
    w_v = property(lambda self: self.kind("v"))
    w_o = property(lambda self: self.kind("o"))
    w_gate = property(lambda self: self.kind("gate"))
    w_up = property(lambda self: self.kind("up"))
    w_down = property(lambda self: self.kind("down"))
    norm_mha = property(lambda self: self.kind("norm_mha"))
    norm_ffn = property(lambda self: self.kind("norm_ffn"))

    @property
    def precision(self) -> str:
        return self._owner.precision

    @property
    def cfg(self) -> ModelConfig:
        return self._owner.cfg

    def struct(self) -> _lib.LayerWeights:
        o = self._owner
        p = f"layers.{self.layer}."
        mp = lambda n: o.master.data_ptr() + 4 * o.offsets[p + n]
        cp = lambda n: o.shadow.data_ptr() + o.shadow.element_size() * o.offsets[p + n]
        return _lib.LayerWeights(mp("q"), mp("o"), mp("norm_mha"), mp("gate"), mp("down"), mp("norm_ffn"),
                                 cp("q"), cp("o"), cp("gate"), cp("down"))


class ModelWeights:
    """Flat-buffer parameter store (model.py:93-135)."""

    def __init__(self, cfg: ModelConfig, precision: str = "fp32", device=None):
        runtime.require_cuda()
        self.cfg = cfg
        self.precision = precision
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        layout, total = _param_layout(cfg)
        self.layout = layout
        self.offsets = {n: off for n, _, off in layout}
        self.shapes = {n: shp for n, shp, _ in layout}
        self.total = total
        self.master = torch.zeros(total, dtype=torch.float32, device=self.device)
        self.shadow = self.master if precision == "fp32" else torch.zeros(total, dtype=torch.bfloat16,
                                                                          device=self.device)
        self.layers = [LayerWeights(self, l) for l in range(cfg.layers)]

    # --- reference-style accessors (logical, reference-shaped views) ----
    def view(self, flat: torch.Tensor, name: str) -> torch.Tensor:
        """Reference-shaped view of parameter `name` inside any flat buffer
        with this layout (master weights, gradients, optimizer moments)."""
        off = self.offsets[name]
        shape = self.shapes[name]
        return logical_view(self.cfg, name, flat[off: off + int(np.prod(shape))].view(shape))

    def named(self):
        for name, _, _ in self.layout:
            yield name, self.view(self.master, name)

    def get(self, name: str) -> torch.Tensor:
        return self.view(self.master, name)

    def set(self, name: str, value) -> None:
        t = torch.as_tensor(np.asarray(value) if not torch.is_tensor(value) else value)
        self.get(name).copy_(t.to(self.device, torch.float32))
        self.sync_shadow(name)

    def shadow_view(self, name: str) -> torch.Tensor:
        return self.view(self.shadow, name)

    def sync_shadow(self, name: str | None = None) -> None:
        """Refresh the compute-precision operand copy (bf16 mode)."""
        if self.precision == "fp32":
            return
        eng = runtime.engine_for(self.cfg, self.precision)
        if name is None:
            _lib.call("mecefo_cast", eng.handle, self.master.data_ptr(), self.shadow.data_ptr(), self.total,
                      runtime.stream_ptr())
        else:
            off = self.offsets[name]
            n = int(np.prod(self.shapes[name]))
            _lib.call("mecefo_cast", eng.handle, self.master.data_ptr() + 4 * off,
                      self.shadow.data_ptr() + 2 * off, n, runtime.stream_ptr())

    @property
    def embedding(self):
        return self.get("embedding")

    @property
    def final_norm(self):
        return self.get("final_norm")

    @property
    def unembedding(self):
        return self.get("unembedding")

    def copy(self) -> "ModelWeights":
        out = ModelWeights(self.cfg, self.precision, self.device)
        out.master.copy_(self.master)
        if self.precision != "fp32":
            out.shadow.copy_(self.shadow)
        return out

    def to_numpy(self) -> dict[str, np.ndarray]:
        return {n: t.detach().double().cpu().numpy() for n, t in self.named()}


def _host_view(w: "ModelWeights", host: np.ndarray, name: str) -> np.ndarray:
    off = w.offsets[name]
    shape = w.shapes[name]
    return logical_view(w.cfg, name, host[off: off + int(np.prod(shape))].reshape(shape))


def init_weights(cfg: ModelConfig, seed: int, std: float = INIT_STD, precision: str = "fp32",
                 device=None) -> ModelWeights:
    """model.py:138-167, bit-identical draws (host PCG64), uploaded once."""
    m, f, v = cfg.hidden, cfg.ffn_intermediate, cfg.vocab
    w = ModelWeights(cfg, precision, device)
    host = np.zeros(w.total, dtype=np.float32)
    counter = seed * 1000
    draws = []
    for l in range(cfg.layers):
        for kind, shp in (("q", (m, m)), ("k", (m, m)), ("v", (m, m)), ("o", (m, m)), ("gate", (f, m)),
                          ("up", (f, m)), ("down", (m, f))):
            draws.append((f"layers.{l}.{kind}", shp))
    draws += [("embedding", (v, m)), ("unembedding", (v, m))]
    for name, (r, c) in draws:
        counter += 1
        _host_view(w, host, name)[...] = seeded_gaussian(r, c, 0.0, std, counter)
    for name, shape, off in w.layout:
        if name.endswith("norm_mha") or name.endswith("norm_ffn") or name == "final_norm":
            host[off: off + shape[0]] = 1.0
    w.master.copy_(torch.from_numpy(host))
    w.sync_shadow()
    return w


def from_numpy(cfg: ModelConfig, arrays: dict, precision: str = "fp32", device=None) -> ModelWeights:
    """Upload reference-layout arrays (e.g. faultsim ModelWeights.named())."""
    w = ModelWeights(cfg, precision, device)
    host = np.zeros(w.total, dtype=np.float32)
    for name, _, _ in w.layout:
        _host_view(w, host, name)[...] = np.asarray(arrays[name], dtype=np.float64).reshape(
            logical_shape(cfg, name, w.shapes[name]))
    w.master.copy_(torch.from_numpy(host))
    w.sync_shadow()
    return w


# ---------------------------------------------------------------------------
# Block-level forward/backward
# ---------------------------------------------------------------------------


@dataclass
class BlockCache:
    """model.py:376-381: x and x1 always; the rest only in CACHE_FULL."""

    mode: str
    x: torch.Tensor
    x1: torch.Tensor
    full: dict | None = field(default=None, repr=False)

    def struct(self) -> _lib.BlockCache:
        f = self.full or {}
        p = lambda k: runtime.ptr(f.get(k))
        return _lib.BlockCache(self.x.data_ptr(), self.x1.data_ptr(), p("h1"), p("inv1"), p("qkv"), p("ctx"),
                               p("lse"), p("h2"), p("inv2"), p("gu"), p("act"))


def _to_2d(cfg: ModelConfig, x: torch.Tensor) -> torch.Tensor:
    """model.py:381-395 _to_btm contract, returned flattened to (tokens, m)."""
    if not torch.is_tensor(x) or not x.is_cuda:
        raise ContractViolation("activations must be CUDA tensors")
    if x.ndim == 2:
        n_tok, m = x.shape
        if m != cfg.hidden or n_tok % cfg.seq_len != 0:
            raise ContractViolation(f"activations of shape {tuple(x.shape)} do not match hidden={cfg.hidden}, "
                                    f"seq_len={cfg.seq_len}")
    elif x.ndim == 3:
        if x.shape[1] != cfg.seq_len or x.shape[2] != cfg.hidden:
            raise ContractViolation(f"activations of shape {tuple(x.shape)} do not match the config")
    else:
        raise ContractViolation(f"activations must be 2-D or 3-D, got {x.ndim}-D")
    return x.reshape(-1, cfg.hidden).to(torch.float32).contiguous()


def _alloc_full_cache(cfg: ModelConfig, b: int, dtype, device) -> dict:
    m, f, H = cfg.hidden, ffn_storage(cfg), cfg.heads
    e = lambda *s, dt=dtype: torch.empty(*s, dtype=dt, device=device)
    return {"h1": e(b, m), "inv1": e(b, dt=torch.float32), "qkv": e(b, 3 * m), "ctx": e(b, m),
            "lse": e(b, H, dt=torch.float32), "h2": e(b, m), "inv2": e(b, dt=torch.float32), "gu": e(b, 2 * f),
            "act": e(b, f)}


def forward_block(cfg: ModelConfig, lw: LayerWeights, x, mode: str = CACHE_FULL):
    """model.py:398-418. Output identical across cache modes."""
    if mode not in _MODE_CODE:
        raise ContractViolation(f"unknown cache mode {mode!r}")
    x2 = _to_2d(cfg, x)
    eng = runtime.engine_for(cfg, lw.precision)
    b = x2.shape[0]
    x1 = torch.empty_like(x2)
    y = torch.empty_like(x2)
    full = _alloc_full_cache(cfg, b, eng.dtype, x2.device) if mode == CACHE_FULL else None
    cache = BlockCache(mode=mode, x=x2, x1=x1, full=full)
    cs = cache.struct()
    ws, wn = eng.workspace(b)
    _lib.call("mecefo_forward_block", eng.handle, ctypes.byref(lw.struct()), ctypes.byref(cs), y.data_ptr(), None,
              b, _MODE_CODE[mode], ws, wn, runtime.stream_ptr())
    return y.reshape(x.shape), cache


def _grad_buffers(cfg: ModelConfig, device, mha: bool):
    m, f = cfg.hidden, ffn_storage(cfg)
    z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=device)
    g = {"gu": z(2 * f, m), "down": z(m, f), "norm_ffn": z(m)}
    if mha:
        g.update({"qkv": z(3 * m, m), "o": z(m, m), "norm_mha": z(m)})
    return g


def _grads_struct(g: dict, alpha_mha=1.0, alpha_ffn=1.0) -> _lib.LayerGrads:
    p = lambda k: runtime.ptr(g.get(k))
    return _lib.LayerGrads(p("qkv"), p("o"), p("norm_mha"), alpha_mha, p("gu"), p("down"), p("norm_ffn"), alpha_ffn)


def _unpack_grads(cfg: ModelConfig, g: dict) -> dict:
    m, f, fp = cfg.hidden, cfg.ffn_intermediate, ffn_storage(cfg)
    out = {"gate": g["gu"][:f], "up": g["gu"][fp:fp + f], "down": g["down"][:, :f], "norm_ffn": g["norm_ffn"]}
    if "qkv" in g:
        out.update({"q": g["qkv"][:m], "k": g["qkv"][m:2 * m], "v": g["qkv"][2 * m:], "o": g["o"],
                    "norm_mha": g["norm_mha"]})
    return out


def backward_block_exact(cfg: ModelConfig, lw: LayerWeights, cache: BlockCache, dy):
    """model.py:421-437. Requires a full cache; returns (dx, grads)."""
    if cache.mode != CACHE_FULL:
        raise ContractViolation("exact backward requires a full activation cache")
    dy2 = _to_2d(cfg, dy)
    eng = runtime.engine_for(cfg, lw.precision)
    b = dy2.shape[0]
    dx = torch.empty_like(dy2)
    g = _grad_buffers(cfg, dy2.device, mha=True)
    ws, wn = eng.workspace(b)
    _lib.call("mecefo_backward_block_exact", eng.handle, ctypes.byref(lw.struct()), ctypes.byref(cache.struct()),
              dy2.data_ptr(), None, dx.data_ptr(), None, ctypes.byref(_grads_struct(g)), b, ws, wn,
              runtime.stream_ptr())
    return dx.reshape(dy.shape), _unpack_grads(cfg, g)


def ffn_forward(lw: LayerWeights, x1) -> dict:
    """model.py:207-225 (shared with recompute, so recomputation is bit-identical)."""
    cfg = lw.cfg
    x2 = _to_2d(cfg, x1)
    eng = runtime.engine_for(cfg, lw.precision)
    b, m, f = x2.shape[0], cfg.hidden, ffn_storage(cfg)
    dt = eng.dtype
    out = {"h2": torch.empty(b, m, dtype=dt, device=x2.device),
           "inv_rms2": torch.empty(b, 1, dtype=torch.float32, device=x2.device),
           "gate": torch.empty(b, f, dtype=dt, device=x2.device), "up": torch.empty(b, f, dtype=dt, device=x2.device),
           "act": torch.empty(b, f, dtype=dt, device=x2.device),
           "down": torch.empty(b, m, dtype=torch.float32, device=x2.device)}
    ws, wn = eng.workspace(b)
    _lib.call("mecefo_recompute_ffn", eng.handle, ctypes.byref(lw.struct()), x2.data_ptr(), b, out["h2"].data_ptr(),
              out["inv_rms2"].data_ptr(), out["gate"].data_ptr(), out["up"].data_ptr(), out["act"].data_ptr(),
              out["down"].data_ptr(), ws, wn, runtime.stream_ptr())
    lead = x1.shape[:-1]
    fl = cfg.ffn_intermediate
    return {k: (v[:, :fl] if k in ("gate", "up", "act") else v).reshape(*lead, -1) for k, v in out.items()}


# ---------------------------------------------------------------------------
# Whole-model forward, loss, head/embedding backward
# ---------------------------------------------------------------------------


def _check_tokens(cfg: ModelConfig, tokens) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(tokens) if not torch.is_tensor(tokens) else tokens)
    if t.ndim != 2 or t.shape[1] != cfg.seq_len:
        raise ContractViolation(f"tokens must be (batch, {cfg.seq_len})")
    if int(t.min()) < 0 or int(t.max()) >= cfg.vocab:
        raise ContractViolation("token id out of vocabulary")
    return t.to(device="cuda", dtype=torch.int64).contiguous()


def forward_model(weights: ModelWeights, tokens, modes=None):
    """model.py:445-473: (logits (B*T, vocab) in compute precision, caches, final cache)."""
    cfg = weights.cfg
    tok = _check_tokens(cfg, tokens)
    if modes is None:
        modes = [CACHE_FULL] * cfg.layers
    if len(modes) != cfg.layers:
        raise ContractViolation("one cache mode per layer required")
    eng = runtime.engine_for(cfg, weights.precision)
    b = tok.numel()
    x = torch.empty(b, cfg.hidden, dtype=torch.float32, device=tok.device)
    _lib.call("mecefo_embedding_forward", eng.handle, tok.data_ptr(), weights.master.data_ptr() +
              4 * weights.offsets["embedding"], x.data_ptr(), b, runtime.stream_ptr())
    caches = []
    for lw, mode in zip(weights.layers, modes):
        x, cache = forward_block(cfg, lw, x, mode)
        caches.append(cache)
    xf = torch.empty(b, cfg.hidden, dtype=eng.dtype, device=tok.device)
    inv_f = torch.empty(b, 1, dtype=torch.float32, device=tok.device)
    logits = torch.empty(b, cfg.vocab, dtype=eng.dtype, device=tok.device)
    _lib.call("mecefo_head_logits", eng.handle, x.data_ptr(), weights.get("final_norm").data_ptr(),
              weights.shadow_view("unembedding").data_ptr(), b, xf.data_ptr(), inv_f.data_ptr(), logits.data_ptr(),
              runtime.stream_ptr())
    final_cache = {"x_last": x, "inv_rms_f": inv_f, "xf2": xf}
    return logits, caches, final_cache


def cross_entropy(logits: torch.Tensor, targets, cfg: ModelConfig | None = None, precision: str | None = None):
    """model.py:492-509: (loss, dlogits = (softmax - onehot)/n). Returns the
    loss as a Python float and dlogits in the logits' precision."""
    if logits.ndim != 2:
        raise ContractViolation("logits/targets shapes are inconsistent")
    t = torch.as_tensor(np.asarray(targets) if not torch.is_tensor(targets) else targets).reshape(-1)
    if t.shape[0] != logits.shape[0]:
        raise ContractViolation("logits/targets shapes are inconsistent")
    t = t.to(device=logits.device, dtype=torch.int64).contiguous()
    prec = precision or ("bf16" if logits.dtype == torch.bfloat16 else "fp32")
    if cfg is None:
        cfg = ModelConfig(vocab=logits.shape[1], hidden=8, heads=1, ffn_intermediate=8, layers=1, seq_len=1)
    eng = runtime.engine_for(cfg, prec)
    d = logits.to(eng.dtype).clone().contiguous()
    loss = torch.empty(1, dtype=torch.float32, device=logits.device)
    ws, wn = eng.workspace(d.shape[0])
    _lib.call("mecefo_cross_entropy", eng.handle, d.data_ptr(), t.data_ptr(), d.shape[0], loss.data_ptr(), ws, wn,
              runtime.stream_ptr())
    return float(loss.item()), d


def head_backward(weights: ModelWeights, final_cache: dict, dlogits: torch.Tensor):
    """model.py:476-483: (dx_last, {"final_norm", "unembedding"})."""
    cfg = weights.cfg
    eng = runtime.engine_for(cfg, weights.precision)
    x_last = final_cache["x_last"]
    b = x_last.shape[0]
    dx = torch.empty_like(x_last)
    g_final = torch.zeros(cfg.hidden, dtype=torch.float32, device=x_last.device)
    g_un = torch.zeros(cfg.vocab, cfg.hidden, dtype=torch.float32, device=x_last.device)
    ws, wn = eng.workspace(b)
    _lib.call("mecefo_head_backward", eng.handle, x_last.data_ptr(), weights.get("final_norm").data_ptr(),
              final_cache["inv_rms_f"].data_ptr(), final_cache["xf2"].data_ptr(), dlogits.contiguous().data_ptr(),
              weights.shadow_view("unembedding").data_ptr(), dx.data_ptr(), None, g_final.data_ptr(),
              g_un.data_ptr(), 1.0, b, ws, wn, runtime.stream_ptr())
    return dx, {"final_norm": g_final, "unembedding": g_un}


def embedding_backward(weights: ModelWeights, tokens, dx0: torch.Tensor) -> torch.Tensor:
    """model.py:486-489 (scatter-add by token id)."""
    cfg = weights.cfg
    tok = torch.as_tensor(np.asarray(tokens) if not torch.is_tensor(tokens) else tokens)
    tok = tok.reshape(-1).to(device=dx0.device, dtype=torch.int64).contiguous()
    g = torch.zeros(cfg.vocab, cfg.hidden, dtype=torch.float32, device=dx0.device)
    eng = runtime.engine_for(cfg, weights.precision)
    _lib.call("mecefo_embedding_backward", eng.handle, tok.data_ptr(), dx0.contiguous().data_ptr(), g.data_ptr(),
              1.0, tok.numel(), runtime.stream_ptr())
    return g
