"""ORACLE (test infrastructure only): float64 restatement of the model math.

Weights are a flat dict keyed by the reference's canonical parameter names
("embedding", "layers.{l}.{kind}", "final_norm", "unembedding";
model.py:35,101-108). Each function cites the reference lines it restates.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

EPS = 1e-6  # model.py:27
LAYER_KINDS = ("q", "k", "v", "o", "norm_mha", "gate", "up", "down", "norm_ffn")  # model.py:35
FFN_KINDS = ("gate", "up", "down")  # approx.py:22


def _mm_f64(a, b):
    return np.matmul(a, b)


# Every matrix product of the restatement goes through MM (BLAS-backed
# np.matmul in float64). tests/golden/make_bf16_calibration.py swaps in a
# PyTorch bf16 matmul to measure the error of a bf16-autocast implementation
# of the same step; nothing else touches it.
MM = _mm_f64


def mm(a, b):
    return MM(a, b)


@dataclass(frozen=True)
class Dims:
    vocab: int
    hidden: int
    heads: int
    ffn: int
    layers: int
    seq_len: int
    rope: bool = True

    @property
    def hd(self) -> int:
        return self.hidden // self.heads


def gaussian(rows: int, cols: int, std: float, seed: int) -> np.ndarray:
    """linalg.py:46-62: N(0, std^2) from Generator(PCG64(seed)).normal."""
    return np.random.Generator(np.random.PCG64(seed)).normal(0.0, std, size=(rows, cols))


def param_shapes(d: Dims) -> list[tuple[str, tuple[int, ...]]]:
    m, f, v = d.hidden, d.ffn, d.vocab
    per = {"q": (m, m), "k": (m, m), "v": (m, m), "o": (m, m), "norm_mha": (m,), "gate": (f, m), "up": (f, m),
           "down": (m, f), "norm_ffn": (m,)}
    out = [("embedding", (v, m))]
    for l in range(d.layers):
        out += [(f"layers.{l}.{k}", per[k]) for k in LAYER_KINDS]
    out += [("final_norm", (m,)), ("unembedding", (v, m))]
    return out


def init_params(d: Dims, seed: int, std: float = 0.02) -> dict[str, np.ndarray]:
    """model.py:138-167. Draw order: per layer q,k,v,o,gate,up,down (seeds
    seed*1000+1, +2, ...), then embedding, then unembedding; norms are ones."""
    counter = seed * 1000
    w: dict[str, np.ndarray] = {}
    draws = []
    for l in range(d.layers):
        for k in ("q", "k", "v", "o", "gate", "up", "down"):
            draws.append(f"layers.{l}.{k}")
    draws += ["embedding", "unembedding"]
    shapes = dict(param_shapes(d))
    for name in draws:
        counter += 1
        r, c = shapes[name]
        w[name] = gaussian(r, c, std, counter)
    for name, shp in shapes.items():
        if name not in w:
            w[name] = np.ones(shp)
    return {name: w[name] for name, _ in param_shapes(d)}


# ----------------------------------------------------------------- kernels

def rms_fwd(x, g):
    """model.py:183-186."""
    inv = 1.0 / np.sqrt((x * x).mean(axis=-1, keepdims=True) + EPS)
    return x * inv * g, inv


def rms_bwd(x, g, inv, dy):
    """model.py:189-195."""
    red = tuple(range(x.ndim - 1))
    dg = (dy * x * inv).sum(axis=red)
    a = dy * g
    proj = (a * x).sum(axis=-1, keepdims=True) / x.shape[-1]
    return a * inv - x * inv ** 3 * proj, dg


def sigm(z):
    return 1.0 / (1.0 + np.exp(-z))


def silu(z):
    """model.py:198-199."""
    return z * sigm(z)


def dsilu(z):
    """model.py:202-204."""
    s = sigm(z)
    return s * (1.0 + z * (1.0 - s))


def ffn_fwd(W, l, x1):
    """model.py:207-225 (== approx.recompute_ffn, approx.py:90-96)."""
    p = f"layers.{l}."
    h2, inv2 = rms_fwd(x1, W[p + "norm_ffn"])
    gate = mm(h2, W[p + "gate"].T)
    up = mm(h2, W[p + "up"].T)
    act = silu(gate) * up
    down = mm(act, W[p + "down"].T)
    return dict(h2=h2, inv2=inv2, gate=gate, up=up, act=act, down=down)


def ffn_bwd(W, l, x1, it, dout, wgrad=None):
    """model.py:232-261 with the `wgrad(kind, d2, inp2)` hook."""
    p = f"layers.{l}."
    n = int(np.prod(dout.shape[:-1]))
    flat = lambda a: a.reshape(n, a.shape[-1])
    if wgrad is None:
        wgrad = lambda kind, d2, inp: mm(d2.T, inp)
    g = {"down": wgrad("down", flat(dout), flat(it["act"]))}
    dact = mm(dout, W[p + "down"])
    dup = dact * silu(it["gate"])
    dgate = dact * it["up"] * dsilu(it["gate"])
    g["gate"] = wgrad("gate", flat(dgate), flat(it["h2"]))
    g["up"] = wgrad("up", flat(dup), flat(it["h2"]))
    dh2 = mm(dgate, W[p + "gate"]) + mm(dup, W[p + "up"])
    dx1, g["norm_ffn"] = rms_bwd(x1, W[p + "norm_ffn"], it["inv2"], dh2)
    return dx1, {k: g[k] for k in ("gate", "up", "down", "norm_ffn")}


def rope_tables(T, hd):
    """model.py:268-278: theta_j = 10000^(-2j/hd), angle = t * theta_j."""
    j = np.arange(hd // 2)
    ang = np.outer(np.arange(T), 10000.0 ** (-2.0 * j / hd))
    return np.cos(ang), np.sin(ang)


def rope(x, cos, sin, inverse=False):
    """model.py:281-298: rotate interleaved (even, odd) pairs."""
    s = -sin if inverse else sin
    e, o = x[..., 0::2], x[..., 1::2]
    y = np.empty_like(x)
    y[..., 0::2] = e * cos - o * s
    y[..., 1::2] = e * s + o * cos
    return y


def heads_split(x, H):
    B, T, m = x.shape
    return x.reshape(B, T, H, m // H).transpose(0, 2, 1, 3)


def heads_merge(x):
    B, H, T, d = x.shape
    return x.transpose(0, 2, 1, 3).reshape(B, T, H * d)


def attn_fwd(d: Dims, W, l, h1):
    """model.py:317-333."""
    p = f"layers.{l}."
    q = heads_split(mm(h1, W[p + "q"].T), d.heads)
    k = heads_split(mm(h1, W[p + "k"].T), d.heads)
    v = heads_split(mm(h1, W[p + "v"].T), d.heads)
    T = h1.shape[1]
    if d.rope:
        c, s = rope_tables(T, d.hd)
        q, k = rope(q, c, s), rope(k, c, s)
    sc = mm(q, k.swapaxes(-1, -2)) / math.sqrt(d.hd)
    sc = np.where(np.triu(np.ones((T, T), bool), 1), -np.inf, sc)
    sc = sc - sc.max(-1, keepdims=True)
    pr = np.exp(sc)
    pr /= pr.sum(-1, keepdims=True)
    ctx = heads_merge(mm(pr, v))
    return dict(q=q, k=k, v=v, probs=pr, ctx=ctx, out=mm(ctx, W[p + "o"].T))


def attn_bwd(d: Dims, W, l, h1, a, dout):
    """model.py:336-368."""
    p = f"layers.{l}."
    B, T, m = h1.shape
    n = B * T
    g = {"o": mm(dout.reshape(n, m).T, a["ctx"].reshape(n, m))}
    dctx = heads_split(mm(dout, W[p + "o"]), d.heads)
    pr = a["probs"]
    dpr = mm(dctx, a["v"].swapaxes(-1, -2))
    dv = mm(pr.swapaxes(-1, -2), dctx)
    ds = pr * (dpr - (dpr * pr).sum(-1, keepdims=True))
    sc = 1.0 / math.sqrt(d.hd)
    dq = mm(ds, a["k"]) * sc
    dk = mm(ds.swapaxes(-1, -2), a["q"]) * sc
    if d.rope:
        c, s = rope_tables(T, d.hd)
        dq, dk = rope(dq, c, s, inverse=True), rope(dk, c, s, inverse=True)
    mq, mk, mv = (heads_merge(t).reshape(n, m) for t in (dq, dk, dv))
    h = h1.reshape(n, m)
    g["q"], g["k"], g["v"] = mm(mq.T, h), mm(mk.T, h), mm(mv.T, h)
    dh1 = (mm(mq, W[p + "q"]) + mm(mk, W[p + "k"]) + mm(mv, W[p + "v"])).reshape(B, T, m)
    return dh1, g


def block_fwd(d: Dims, W, l, x3, lean: bool):
    """model.py:398-418. Returns (y, cache)."""
    p = f"layers.{l}."
    h1, inv1 = rms_fwd(x3, W[p + "norm_mha"])
    a = attn_fwd(d, W, l, h1)
    x1 = x3 + a["out"]
    it = ffn_fwd(W, l, x1)
    y = x1 + it["down"]
    cache = dict(x=x3, x1=x1)
    if not lean:
        cache.update(h1=h1, inv1=inv1, attn=a, ffn=it)
    return y, cache


def block_bwd_exact(d: Dims, W, l, cache, dy):
    """model.py:421-437."""
    p = f"layers.{l}."
    dx1f, g = ffn_bwd(W, l, cache["x1"], cache["ffn"], dy)
    dx1 = dy + dx1f
    dh1, ga = attn_bwd(d, W, l, cache["h1"], cache["attn"], dx1)
    dxn, g["norm_mha"] = rms_bwd(cache["x"], W[p + "norm_mha"], cache["inv1"], dh1)
    g.update(ga)
    return dx1 + dxn, g


def lowrank(g_y, x, v1):
    """approx.py:24-42: g_y (x^T v1) v1^T in exactly that association order."""
    return mm(mm(g_y, mm(x.T, v1)), v1.T)


def block_bwd_neighbor(d: Dims, W, l, cache, dy, basis=None):
    """approx.py:99-134 (basis = ProjectionCache.basis or None for exact)."""
    wg = None
    if basis is not None:
        wg = lambda kind, d2, inp: lowrank(d2.T, inp.T, basis[kind])
    it = ffn_fwd(W, l, cache["x1"])
    dx1f, g = ffn_bwd(W, l, cache["x1"], it, dy, wg)
    return dy + dx1f, g


def subspace_top_r(w, r, tol=1e-12, max_iter=2000, seed=0):
    """linalg.py:97-142: block power iteration on w^T w (oversample 4),
    QR + Rayleigh-Ritz per step, relative residual stopping rule."""
    n = w.shape[1]
    B = w.T @ w
    if np.linalg.norm(B) == 0.0:
        return np.eye(n)[:, :r].copy()
    k = min(n, r + 4)
    V, _ = np.linalg.qr(gaussian(n, k, 1.0, seed))
    for _ in range(max_iter):
        V, _ = np.linalg.qr(B @ V)
        S = V.T @ B @ V
        lam, U = np.linalg.eigh(0.5 * (S + S.T))
        idx = np.argsort(lam)[::-1]
        lam, V = lam[idx], V @ U[:, idx]
        top = V[:, :r]
        res = np.linalg.norm(B @ top - top * lam[:r], axis=0).max() / max(lam[0], np.finfo(float).tiny)
        if res <= tol:
            return np.ascontiguousarray(top)
    raise RuntimeError(f"subspace iteration did not converge (residual {res:.3e})")


def cross_entropy(logits, targets):
    """model.py:492-509."""
    n = logits.shape[0]
    z = logits - logits.max(axis=1, keepdims=True)
    lp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    t = targets.reshape(-1)
    loss = -float(lp[np.arange(n), t].mean())
    dl = np.exp(lp)
    dl[np.arange(n), t] -= 1.0
    return loss, dl / n


def rank_pass(d: Dims, W, tokens, targets, modes, bases=None):
    """harness.py:243-249 + forward_model (model.py:445-473) + backward_model
    (harness.py:209-240). modes[l] in {"full", "ffn_input_only"}; bases maps
    layer -> {kind: V1} for lean layers (None -> exact Wgrads)."""
    x = W["embedding"][tokens]
    caches = []
    for l in range(d.layers):
        x, c = block_fwd(d, W, l, x, modes[l] != "full")
        caches.append(c)
    xf, invf = rms_fwd(x, W["final_norm"])
    xf2 = xf.reshape(-1, d.hidden)
    logits = mm(xf2, W["unembedding"].T)
    loss, dl = cross_entropy(logits, targets)
    g = {"unembedding": mm(dl.T, xf2)}
    dx, g["final_norm"] = rms_bwd(x, W["final_norm"], invf, mm(dl, W["unembedding"]).reshape(x.shape))
    for l in reversed(range(d.layers)):
        if modes[l] == "full":
            dx, gl = block_bwd_exact(d, W, l, caches[l], dx)
        else:
            dx, gl = block_bwd_neighbor(d, W, l, caches[l], dx, None if bases is None else bases.get(l))
        for k, v in gl.items():
            g[f"layers.{l}.{k}"] = v
    ge = np.zeros_like(W["embedding"])
    np.add.at(ge, tokens.reshape(-1), dx.reshape(-1, d.hidden))
    g["embedding"] = ge
    return loss, g


def rel_err(a, b, floor=1e-12):
    """tests/oracles.py:147-149 tensor_rel_err."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    s = max(float(np.abs(a).max(initial=0.0)), float(np.abs(b).max(initial=0.0)), floor)
    return float(np.abs(a - b).max(initial=0.0)) / s
