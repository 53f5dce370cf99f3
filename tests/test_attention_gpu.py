"""GPU: head_dim-64 / T=256 block (the LLaMA-60M..1B attention shape) against
the float64 oracle — exercises the tcgen05 attention forward (bf16), the RoPE
GEMM epilogue and the SIMT exact backward on pre-rotated q/k."""

import numpy as np
import pytest
import torch

from oracle import model_ref as R
from paper_2510_16415_b200 import approx, model as mdl

pytestmark = pytest.mark.gpu

BF16_TOL = 5e-2


def _setup(hidden=512, heads=8, ffn=1376, T=256, seqs=2, seed=0):
    cfg = mdl.ModelConfig(vocab=64, hidden=hidden, heads=heads, ffn_intermediate=ffn, layers=1, seq_len=T)
    d = R.Dims(64, hidden, heads, ffn, 1, T)
    W = R.init_params(d, seed)
    rng = np.random.Generator(np.random.PCG64(seed + 1))
    x = rng.normal(size=(seqs * T, hidden)) * 0.5
    dy = rng.normal(size=(seqs * T, hidden)) * 0.01
    return cfg, d, W, x, dy


@pytest.mark.parametrize("prec,tol", [("bf16", BF16_TOL), ("fp32", 1e-4)])
@pytest.mark.parametrize("T,seqs", [(256, 2), (128, 3), (192, 2)])
def test_forward_block_hd64(cuda, prec, tol, T, seqs):
    cfg, d, W, x, dy = _setup(T=T, seqs=seqs)
    y_ref, c_ref = R.block_fwd(d, W, 0, x.reshape(seqs, T, -1), lean=False)
    w = mdl.init_weights(cfg, 0, precision=prec)
    xt = torch.tensor(x, dtype=torch.float32, device="cuda")
    y, cache = mdl.forward_block(cfg, w.layers[0], xt, mdl.CACHE_FULL)
    assert R.rel_err(y.cpu().numpy(), y_ref.reshape(x.shape)) < tol
    assert R.rel_err(cache.x1.cpu().numpy(), c_ref["x1"].reshape(x.shape)) < tol
    # cached q/k are post-RoPE, like the reference's full cache (model.py:323-326)
    q_ref = R.heads_merge(c_ref["attn"]["q"]).reshape(x.shape)
    k_ref = R.heads_merge(c_ref["attn"]["k"]).reshape(x.shape)
    qkv = cache.full["qkv"].float().cpu().numpy()
    assert R.rel_err(qkv[:, :512], q_ref) < tol
    assert R.rel_err(qkv[:, 512:1024], k_ref) < tol
    assert R.rel_err(cache.full["ctx"].float().cpu().numpy(), c_ref["attn"]["ctx"].reshape(x.shape)) < tol
    # lean forward gives the identical output (model.py:398-418)
    y2, lean = mdl.forward_block(cfg, w.layers[0], xt, mdl.CACHE_FFN_INPUT_ONLY)
    assert torch.equal(y, y2)


@pytest.mark.parametrize("prec,tol", [("bf16", BF16_TOL), ("fp32", 1e-4)])
@pytest.mark.parametrize("T,seqs", [(256, 2), (128, 3)])
def test_exact_backward_hd64(cuda, prec, tol, T, seqs):
    """bf16: tcgen05 attention backward (T in {128, 256}); fp32: SIMT path."""
    cfg, d, W, x, dy = _setup(T=T, seqs=seqs)
    _, c_ref = R.block_fwd(d, W, 0, x.reshape(seqs, T, -1), lean=False)
    dx_ref, g_ref = R.block_bwd_exact(d, W, 0, c_ref, dy.reshape(seqs, T, -1))
    w = mdl.init_weights(cfg, 0, precision=prec)
    _, cache = mdl.forward_block(cfg, w.layers[0], torch.tensor(x, dtype=torch.float32, device="cuda"),
                                 mdl.CACHE_FULL)
    dx, g = mdl.backward_block_exact(cfg, w.layers[0], cache, torch.tensor(dy, dtype=torch.float32, device="cuda"))
    assert R.rel_err(dx.cpu().numpy(), dx_ref.reshape(x.shape)) < tol
    for k in g:
        assert R.rel_err(g[k].cpu().numpy(), g_ref[k]) < tol, k


@pytest.mark.parametrize("seqs", [2, 16])
def test_lean_backward_hd64_lowrank_r128(cuda, seqs):
    """seqs=16 (4096 tokens): many tiles per CTA, so the fused recompute
    kernel's TMEM ring wraps (d_act of tile i+1 overlapping tile i's epilogue)."""
    cfg, d, W, x, dy = _setup(seqs=seqs)
    rng = np.random.Generator(np.random.PCG64(9))
    basis = {k: np.linalg.qr(rng.normal(size=(n, 128)))[0] for k, n in (("gate", 512), ("up", 512), ("down", 1376))}
    _, lean_ref = R.block_fwd(d, W, 0, x.reshape(seqs, 256, -1), lean=True)
    dx_ref, g_ref = R.block_bwd_neighbor(d, W, 0, lean_ref, dy.reshape(seqs, 256, -1), basis)
    w = mdl.init_weights(cfg, 0, precision="bf16")
    _, cache = mdl.forward_block(cfg, w.layers[0], torch.tensor(x, dtype=torch.float32, device="cuda"),
                                 mdl.CACHE_FFN_INPUT_ONLY)
    proj = approx.ProjectionCache(rank=128, refresh_period=10**9, step=1)
    for k, v in basis.items():
        proj.set_basis(k, v)
    from paper_2510_16415_b200.linalg import SvdConfig
    dx, g = approx.backward_block_neighbor(cfg, w.layers[0], cache,
                                           torch.tensor(dy, dtype=torch.float32, device="cuda"), proj=proj,
                                           svd=SvdConfig(rank=128))
    assert R.rel_err(dx.cpu().numpy(), dx_ref.reshape(x.shape)) < BF16_TOL
    for k in g:
        assert R.rel_err(g[k].cpu().numpy(), g_ref[k]) < BF16_TOL, k


@pytest.mark.parametrize("hidden,heads,ffn,r", [(768, 12, 2048, 128), (1024, 16, 2736, 128),
                                                (2048, 32, 5472, 64), (2048, 32, 5472, 256)])
def test_lean_backward_llama_shapes(cuda, hidden, heads, ffn, r):
    """SURVEY configs C2 (130M), C3 (350M) and C4 (1B, r in {64, 256}) block
    shapes: one lean block forward + neighbour backward in bf16 vs the fp64
    oracle. ffn 2736 / 5472 leave partial 128-column tiles; r = 256 makes the
    transposed low-rank contraction's diagonal blocks two tiles tall."""
    cfg, d, W, x, dy = _setup(hidden=hidden, heads=heads, ffn=ffn, T=256, seqs=1)
    rng = np.random.Generator(np.random.PCG64(21))
    basis = {k: np.linalg.qr(rng.normal(size=(n, r)))[0] for k, n in (("gate", hidden), ("up", hidden),
                                                                         ("down", ffn))}
    _, lean_ref = R.block_fwd(d, W, 0, x.reshape(1, 256, -1), lean=True)
    dx_ref, g_ref = R.block_bwd_neighbor(d, W, 0, lean_ref, dy.reshape(1, 256, -1), basis)
    w = mdl.init_weights(cfg, 0, precision="bf16")
    _, cache = mdl.forward_block(cfg, w.layers[0], torch.tensor(x, dtype=torch.float32, device="cuda"),
                                 mdl.CACHE_FFN_INPUT_ONLY)
    proj = approx.ProjectionCache(rank=r, refresh_period=10**9, step=1)
    for k, v in basis.items():
        proj.set_basis(k, v)
    from paper_2510_16415_b200.linalg import SvdConfig
    dx, g = approx.backward_block_neighbor(cfg, w.layers[0], cache,
                                           torch.tensor(dy, dtype=torch.float32, device="cuda"), proj=proj,
                                           svd=SvdConfig(rank=r))
    assert R.rel_err(dx.cpu().numpy(), dx_ref.reshape(x.shape)) < BF16_TOL
    for k in g:
        assert R.rel_err(g[k].cpu().numpy(), g_ref[k]) < BF16_TOL, k


def test_forward_block_fused_residual_norm_at_bench_size(cuda):
    """16384 tokens at C1 dims (the fused doubled microbatch): the O projection
    and the following RMSNorm run as ONE kernel (gemm_norm.cuh, one CTA per
    128-row block owning all 512 columns). x1, h2, inv2 and the block output
    against the float64 oracle; the lean forward gives the identical output."""
    seqs = 64
    cfg, d, W, x, dy = _setup(T=256, seqs=seqs, seed=3)
    y_ref, c_ref = R.block_fwd(d, W, 0, x.reshape(seqs, 256, -1), lean=False)
    w = mdl.init_weights(cfg, 3, precision="bf16")
    xt = torch.tensor(x, dtype=torch.float32, device="cuda")
    y, cache = mdl.forward_block(cfg, w.layers[0], xt, mdl.CACHE_FULL)
    assert R.rel_err(cache.x1.cpu().numpy(), c_ref["x1"].reshape(x.shape)) < BF16_TOL
    assert R.rel_err(cache.full["h2"].float().cpu().numpy(), c_ref["ffn"]["h2"].reshape(x.shape)) < BF16_TOL
    assert R.rel_err(cache.full["inv2"].cpu().numpy(), c_ref["ffn"]["inv2"].reshape(-1)) < 1e-2
    assert R.rel_err(y.cpu().numpy(), y_ref.reshape(x.shape)) < BF16_TOL
    y2, _ = mdl.forward_block(cfg, w.layers[0], xt, mdl.CACHE_FFN_INPUT_ONLY)
    assert torch.equal(y, y2)


def test_chained_forward_matches_per_block_calls(cuda):
    """mecefo_forward_block_chained (the step engine's forward: block l's down
    projection also writes block l+1's h1 / inv1, fused into one kernel at
    hidden 512 and 16384 tokens) against plain per-block calls, two lean
    blocks: same outputs up to fp32 summation order / bf16 rounding ties."""
    import ctypes

    from paper_2510_16415_b200 import _lib, runtime

    seqs = 64
    cfg = mdl.ModelConfig(vocab=64, hidden=512, heads=8, ffn_intermediate=1376, layers=2, seq_len=256)
    w = mdl.init_weights(cfg, 5, precision="bf16")
    rng = np.random.Generator(np.random.PCG64(9))
    x0 = torch.tensor(rng.normal(size=(seqs * 256, 512)) * 0.5, dtype=torch.float32, device="cuda")
    eng = runtime.engine_for(cfg, "bf16")
    b = x0.shape[0]
    ws, wn = eng.workspace(b)
    s = runtime.stream_ptr()
    lean = _lib.CACHE_FFN_INPUT_ONLY

    def run(chained):
        xs = [x0.clone(), torch.empty_like(x0), torch.empty_like(x0)]
        x1s = [torch.empty_like(x0) for _ in range(2)]
        h1 = torch.empty(b, 512, dtype=torch.bfloat16, device="cuda")
        inv1 = torch.empty(b, dtype=torch.float32, device="cuda")
        for l in range(2):
            cs = mdl.BlockCache(mode=mdl.CACHE_FFN_INPUT_ONLY, x=xs[l], x1=x1s[l]).struct()
            if not chained:
                _lib.call("mecefo_forward_block", eng.handle, ctypes.byref(w.layers[l].struct()), ctypes.byref(cs),
                          xs[l + 1].data_ptr(), None, b, lean, ws, wn, s)
                continue
            if l == 1:
                cs.h1, cs.inv1 = h1.data_ptr(), inv1.data_ptr()
            gain = w.get("layers.1.norm_mha").data_ptr() if l == 0 else None
            _lib.call("mecefo_forward_block_chained", eng.handle, ctypes.byref(w.layers[l].struct()),
                      ctypes.byref(cs), xs[l + 1].data_ptr(), b, lean, _lib.FWD_H1_READY if l == 1 else 0, gain,
                      h1.data_ptr() if l == 0 else None, inv1.data_ptr() if l == 0 else None, ws, wn, s)
        torch.cuda.synchronize()
        return xs, x1s

    xs_a, x1s_a = run(False)
    xs_b, x1s_b = run(True)
    for t_a, t_b in ((x1s_a[0], x1s_b[0]), (xs_a[1], xs_b[1]), (x1s_a[1], x1s_b[1]), (xs_a[2], xs_b[2])):
        assert R.rel_err(t_b.cpu().numpy(), t_a.cpu().numpy()) < 2e-3
