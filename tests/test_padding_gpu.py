"""GPU: FFN widths that are not a multiple of 8 (LLaMA-1B: f = 5461,
reference model.py:40-61 accepts any width). The engine stores f padded to
mecefo_padded_ffn(f) with zero pad rows/columns; results must equal the
unpadded reference math and the pads must stay exactly zero through
backward and AdamW."""

import numpy as np
import pytest
import torch

from oracle import cluster_ref, model_ref as R
from paper_2510_16415_b200 import _lib, approx, engine as E, model as mdl
from paper_2510_16415_b200.linalg import SvdConfig

pytestmark = pytest.mark.gpu


def test_padded_ffn_width():
    assert _lib.load().mecefo_padded_ffn(5461) == 5464
    assert _lib.load().mecefo_padded_ffn(1376) == 1376


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 5e-2)])
def test_1b_shape_lean_block_f5461_matches_oracle(cuda, prec, tol):
    """LLaMA-1B block shapes (hidden 2048, 32 heads, f 5461, T 256) at r=128:
    lean forward + neighbour backward (skip-MHA, recompute, low-rank Wgrad)."""
    cfg = mdl.ModelConfig(vocab=64, hidden=2048, heads=32, ffn_intermediate=5461, layers=1, seq_len=256)
    d = R.Dims(64, 2048, 32, 5461, 1, 256)
    W = R.init_params(d, 0)
    w = mdl.init_weights(cfg, 0, precision=prec)
    assert w.get("layers.0.down").shape == (2048, 5461) and w.get("layers.0.gate").shape == (5461, 2048)
    assert np.array_equal(w.get("layers.0.down").cpu().numpy(), W["layers.0.down"].astype(np.float32))
    rng = np.random.Generator(np.random.PCG64(9))
    x = rng.normal(size=(256, 2048)) * 0.5
    dy = rng.normal(size=(256, 2048)) * 0.01
    basis = {k: np.linalg.qr(rng.normal(size=(n, 128)))[0] for k, n in (("gate", 2048), ("up", 2048),
                                                                          ("down", 5461))}
    y_ref, lean_ref = R.block_fwd(d, W, 0, x.reshape(1, 256, 2048), lean=True)
    dx_ref, g_ref = R.block_bwd_neighbor(d, W, 0, lean_ref, dy.reshape(1, 256, 2048), basis)
    y, cache = mdl.forward_block(cfg, w.layers[0], torch.tensor(x, dtype=torch.float32, device="cuda"),
                                 mdl.CACHE_FFN_INPUT_ONLY)
    proj = approx.ProjectionCache(rank=128, refresh_period=10**9, step=1)
    for k, v in basis.items():
        proj.set_basis(k, v)
    dx, g = approx.backward_block_neighbor(cfg, w.layers[0], cache,
                                           torch.tensor(dy, dtype=torch.float32, device="cuda"), proj=proj,
                                           svd=SvdConfig(rank=128))
    assert R.rel_err(y.cpu().numpy(), y_ref.reshape(256, 2048)) < tol
    assert R.rel_err(dx.cpu().numpy(), dx_ref.reshape(256, 2048)) < tol
    for k in ("gate", "up", "down", "norm_ffn"):
        assert tuple(g[k].shape) == g_ref[k].shape, k
        assert R.rel_err(g[k].cpu().numpy(), g_ref[k]) < tol, k


def test_1b_shape_exact_block_f5461_fp32(cuda):
    cfg = mdl.ModelConfig(vocab=64, hidden=2048, heads=32, ffn_intermediate=5461, layers=1, seq_len=256)
    d = R.Dims(64, 2048, 32, 5461, 1, 256)
    W = R.init_params(d, 0)
    w = mdl.init_weights(cfg, 0, precision="fp32")
    rng = np.random.Generator(np.random.PCG64(10))
    x = rng.normal(size=(256, 2048)) * 0.5
    dy = rng.normal(size=(256, 2048)) * 0.01
    y_ref, full_ref = R.block_fwd(d, W, 0, x.reshape(1, 256, 2048), lean=False)
    dx_ref, g_ref = R.block_bwd_exact(d, W, 0, full_ref, dy.reshape(1, 256, 2048))
    y, cache = mdl.forward_block(cfg, w.layers[0], torch.tensor(x, dtype=torch.float32, device="cuda"),
                                 mdl.CACHE_FULL)
    dx, g = mdl.backward_block_exact(cfg, w.layers[0], cache, torch.tensor(dy, dtype=torch.float32, device="cuda"))
    assert R.rel_err(dx.cpu().numpy(), dx_ref.reshape(256, 2048)) < 1e-4
    for k, v in g_ref.items():
        assert R.rel_err(g[k].cpu().numpy(), v) < 1e-4, k


def test_engine_step_with_odd_ffn_keeps_pads_zero(cuda):
    """A fused 2-rank MeCeFO step + AdamW at f = 683 (pads to 688): Eq. (1)
    gradients equal the oracle's, and every pad element of the weights,
    gradients and optimizer moments is still exactly zero."""
    cfg = mdl.ModelConfig(vocab=64, hidden=256, heads=4, ffn_intermediate=683, layers=2, seq_len=64)
    d = R.Dims(64, 256, 4, 683, 2, 64)
    eng = E.StepEngine(cfg, precision="fp32", seqs_per_microbatch=2, r=32, tau=10**6)
    rng = np.random.Generator(np.random.PCG64(12))
    bases = {}
    for l in range(2):
        bases[l] = {k: np.linalg.qr(rng.normal(size=(n, 32)))[0] for k, n in (("gate", 256), ("up", 256),
                                                                              ("down", 683))}
        for j in range(2):
            pc = eng.proj(j, l)
            for k, v in bases[l].items():
                pc.set_basis(k, v)
            pc.step = 1
        eng.proj(1, l).token = eng.proj(0, l).token
    batches = [(rng.integers(0, 64, size=(2, 64)), rng.integers(0, 64, size=(2, 64))) for _ in range(2)]
    route, lean, a_mha, skip = E.ring_plan(2, {1}, 2)
    mbs = [E.Microbatch(rank=j, tokens=torch.from_numpy(batches[j][0]).cuda(),
                        targets=torch.from_numpy(batches[j][1]).cuda(), lean=[True] * 2, alpha_mha=[None] * 2,
                        alpha_ffn=0.5, alpha_global=0.5) for j in range(2)]
    losses = torch.zeros(2, device="cuda")
    eng._body(mbs, losses)
    torch.cuda.synchronize()
    W = R.init_params(d, 0)
    per_rank = [R.rank_pass(d, W, batches[j][0], batches[j][1], ["ffn_input_only"] * 2, bases)[1] for j in range(2)]
    active = {(l, k): ([] if k in cluster_ref.MHA else [0, 1]) for l in range(2)
              for k in cluster_ref.MHA + cluster_ref.FFN}
    avg, skipped = cluster_ref.aggregate(per_rank, active, 2)
    for name in avg:
        got = eng.weights.view(eng.grad, name).cpu().numpy()
        assert got.shape == avg[name].shape, name
        assert R.rel_err(got, avg[name]) < 1e-4, name
    from paper_2510_16415_b200 import optim as op

    op.apply_flat(eng.weights, eng.opt, eng.grad, 1e-3, skip=skip, check=True)
    torch.cuda.synchronize()
    fp = mdl.ffn_storage(cfg)
    for l in range(2):
        for buf in (eng.weights.master, eng.grad, eng.opt.m, eng.opt.v):
            for k in ("gate", "up"):
                off = eng.weights.offsets[f"layers.{l}.{k}"]
                blk = buf[off: off + fp * 256].view(fp, 256)
                assert not blk[683:].any(), (l, k)
            off = eng.weights.offsets[f"layers.{l}.down"]
            assert not buf[off: off + 256 * fp].view(256, fp)[:, 683:].any(), l
