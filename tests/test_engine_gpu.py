"""GPU: the fused step engine (flat Eq. (1)-weighted gradient buffer, fused
AdamW, CUDA-graph replay) against the oracle's per-rank rank passes plus the
reference aggregation (cluster.py:292-322) and AdamW (optim.py:75-103)."""

import numpy as np
import pytest
import torch

from oracle import cluster_ref, model_ref as R, optim_ref
from paper_2510_16415_b200 import engine as E, model as mdl

pytestmark = pytest.mark.gpu

C0 = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64)
D0 = R.Dims(64, 128, 4, 344, 2, 64)


def _batches(n_ranks, seqs, seed=0):
    rng = np.random.Generator(np.random.PCG64(seed))
    return [(rng.integers(0, 64, size=(seqs, 64)), rng.integers(0, 64, size=(seqs, 64))) for _ in range(n_ranks)]


def _engine(prec, seqs):
    eng = E.StepEngine(C0, precision=prec, seqs_per_microbatch=seqs, r=32, tau=10**6)
    rng = np.random.Generator(np.random.PCG64(11))
    bases = {}
    for j in range(4):
        for l in range(2):
            pc = eng.proj(j, l)
            bl = {k: np.linalg.qr(rng.normal(size=(n, 32)))[0] for k, n in (("gate", 128), ("up", 128),
                                                                              ("down", 344))}
            for k, v in bl.items():
                pc.set_basis(k, v)
            pc.step = 1  # injected: no refresh due
            bases[(j, l)] = bl
    return eng, bases


def _plan(R_, failed, batches):
    route, lean, a_mha, skip = E.ring_plan(R_, set(failed), 2)
    mbs = []
    for j in range(R_):
        tk, tg = batches[j]
        mbs.append(E.Microbatch(rank=j, tokens=torch.from_numpy(tk).cuda(), targets=torch.from_numpy(tg).cuda(),
                                lean=[lean[j]] * 2, alpha_mha=[None if lean[j] else a_mha] * 2, alpha_ffn=1.0 / R_,
                                alpha_global=1.0 / R_))
    return mbs, lean, skip


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 5e-2)])
@pytest.mark.parametrize("R_,failed", [(2, {1}), (4, {2}), (3, ())])
def test_eq1_weighted_gradients_match_reference_aggregation(cuda, prec, tol, R_, failed):
    batches = _batches(R_, 2)
    eng, bases = _engine(prec, 2)
    mbs, lean, skip = _plan(R_, failed, batches)
    losses = torch.zeros(R_, device="cuda")
    eng._body(mbs, losses)  # all ranks on this GPU: the local flat buffer is the full Eq. (1) sum
    torch.cuda.synchronize()
    W = R.init_params(D0, 0)
    per_rank, ref_losses = [], []
    for j in range(R_):
        modes = ["ffn_input_only" if lean[j] else "full"] * 2
        loss, g = R.rank_pass(D0, W, batches[j][0], batches[j][1], modes,
                              {l: bases[(j, l)] for l in range(2)} if lean[j] else None)
        per_rank.append(g)
        ref_losses.append(loss)
    active = {(l, k): ([j for j in range(R_) if not lean[j]] if k in cluster_ref.MHA else list(range(R_)))
              for l in range(2) for k in cluster_ref.MHA + cluster_ref.FFN}
    avg, skipped = cluster_ref.aggregate(per_rank, active, 2)
    assert sorted(skipped) == sorted(skip)
    assert np.allclose(losses.cpu().numpy(), ref_losses, rtol=tol, atol=tol)
    for name, shape, off in eng.weights.layout:
        got = eng.grad[off: off + int(np.prod(shape))].view(shape).cpu().numpy()
        if name in skipped:
            assert not got.any(), name  # never accumulated (select, not multiply)
        else:
            assert R.rel_err(got, avg[name]) < tol, name


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 5e-2)])
def test_step_with_adamw_matches_reference(cuda, prec, tol):
    """Three MeCeFO steps. Each step's Eq. (1) gradients are checked against
    the oracle (gradient tolerance), then the oracle's AdamW (optim.py:75-103)
    applies the ENGINE's gradient to the float64 weights, so the weight
    comparison isolates the fused optimizer: <= 1% of elements may differ by
    more than 1e-3 of the update scale (fp32 vs fp64 arithmetic)."""
    from paper_2510_16415_b200 import optim as op

    batches = _batches(2, 2, seed=3)
    eng, bases = _engine(prec, 2)
    mbs, lean, skip = _plan(2, {1}, batches)
    W = R.init_params(D0, 0)
    opt = optim_ref.Adam()
    losses = torch.zeros(2, device="cuda")
    for it in range(3):
        lr = optim_ref.lr_at(it + 1, 3, 1e-3)
        eng._body(mbs, losses)
        torch.cuda.synchronize()
        got = {name: eng.grad[off: off + int(np.prod(shape))].view(shape).double().cpu().numpy()
               for name, shape, off in eng.weights.layout}
        op.apply_flat(eng.weights, eng.opt, eng.grad, lr, skip=skip, check=True)
        per_rank = [R.rank_pass(D0, W, batches[j][0], batches[j][1], ["ffn_input_only"] * 2,
                                {l: bases[(j, l)] for l in range(2)})[1] for j in range(2)]
        active = {(l, k): ([] if k in cluster_ref.MHA else [0, 1]) for l in range(2)
                  for k in cluster_ref.MHA + cluster_ref.FFN}
        avg, skipped = cluster_ref.aggregate(per_rank, active, 2)
        for name in avg:
            assert R.rel_err(got[name], avg[name]) < tol, (it, name)
        opt.apply(W, {n: got[n] for n in avg}, lr, skip=skipped)
    torch.cuda.synchronize()
    W0 = R.init_params(D0, 0)
    for name, t in eng.weights.named():
        if name in skipped:
            continue  # checked exactly below
        w = t.cpu().numpy().astype(np.float64)
        err = np.abs(w - W[name])
        step = np.abs(W[name] - W0[name]).max() + 1e-6 * np.abs(W0[name]).max()  # + fp32 rounding of w
        assert err.max() <= 0.05 * step, name
        frac_bad = float((err > 1e-3 * step).mean())
        assert frac_bad <= 1e-2, (name, frac_bad)
    # skipped MHA params never moved, and their step counters never advanced
    assert np.array_equal(eng.weights.get("layers.0.q").cpu().numpy(),
                          R.init_params(D0, 0)["layers.0.q"].astype(np.float32))
    assert "layers.0.q" not in eng.opt.step and eng.opt.step["layers.0.gate"] == 3


def test_graph_replay_matches_eager(cuda):
    batches = _batches(2, 2, seed=5)
    outs = []
    for graph in (False, True):
        eng, _ = _engine("bf16", 2)
        mbs, lean, skip = _plan(2, {1}, batches)
        eng.step(mbs, 2, 1e-3, skip=skip, check=False)
        if graph:
            eng.capture(mbs, 2, skip)
        for _ in range(3):
            if graph:
                eng.replay(1e-3)
            else:
                eng.step(mbs, 2, 1e-3, skip=skip, check=False)
        torch.cuda.synchronize()
        outs.append((eng.weights.master.clone(), eng.losses.clone(), dict(eng.opt.step),
                     {k: pc.step for k, pc in eng.projs.items()}))
    (w0, l0, s0, p0), (w1, l1, s1, p1) = outs
    assert s0 == s1 and p0 == p1
    assert torch.allclose(l0, l1, rtol=1e-3, atol=1e-4)
    assert R.rel_err(w0.cpu().numpy(), w1.cpu().numpy()) < 1e-3


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 5e-2)])
def test_fused_lean_microbatches_match_reference(cuda, prec, tol):
    """The doubled GPU's two lean microbatches run as ONE stacked pass when
    their ranks share projection bases; Eq. (1) gradients and per-rank losses
    are those of the reference's separate rank passes."""
    batches = _batches(2, 2, seed=7)
    eng, bases = _engine(prec, 2)
    for l in range(2):  # rank 1 adopts rank 0's bases (same provenance token)
        for k, v in bases[(0, l)].items():
            eng.proj(1, l).set_basis(k, v)
        eng.proj(1, l).token = eng.proj(0, l).token
        bases[(1, l)] = bases[(0, l)]
    mbs, lean, skip = _plan(2, {1}, batches)
    assert eng._fusable(mbs)
    losses = torch.zeros(2, device="cuda")
    eng._body(mbs, losses)
    torch.cuda.synchronize()
    W = R.init_params(D0, 0)
    per_rank, ref_losses = [], []
    for j in range(2):
        loss, g = R.rank_pass(D0, W, batches[j][0], batches[j][1], ["ffn_input_only"] * 2,
                              {l: bases[(j, l)] for l in range(2)})
        per_rank.append(g)
        ref_losses.append(loss)
    active = {(l, k): ([] if k in cluster_ref.MHA else [0, 1]) for l in range(2)
              for k in cluster_ref.MHA + cluster_ref.FFN}
    avg, skipped = cluster_ref.aggregate(per_rank, active, 2)
    assert np.allclose(losses.cpu().numpy(), ref_losses, rtol=tol, atol=tol)
    for name, shape, off in eng.weights.layout:
        got = eng.grad[off: off + int(np.prod(shape))].view(shape).cpu().numpy()
        if name in skipped:
            assert not got.any(), name
        else:
            assert R.rel_err(got, avg[name]) < tol, name
    assert all(eng.proj(j, l).step == 2 for j in range(2) for l in range(2))


@pytest.mark.parametrize("fused", [True, False])
def test_deferred_grouped_lowrank_wgrads_match_reference(cuda, fused):
    """bf16 with r = 128 (rank_pad a multiple of the 128-row tile): every lean
    layer's low-rank FFN Wgrads are deferred and run as grouped launches
    (mecefo_lowrank_wgrads_batched); the Eq. (1) gradients equal the
    reference's per-rank passes + aggregation. fused=False keeps one pass per
    microbatch (distinct bases per rank -> separate jobs)."""
    tol = 5e-2
    batches = _batches(2, 2, seed=13)
    eng = E.StepEngine(C0, precision="bf16", seqs_per_microbatch=2, r=128, tau=10**6)
    rng = np.random.Generator(np.random.PCG64(17))
    bases = {}
    for j in range(2):
        for l in range(2):
            pc = eng.proj(j, l)
            src = (0, l) if fused else (j, l)
            if src not in bases:
                bases[src] = {k: np.linalg.qr(rng.normal(size=(n, 128)))[0]
                              for k, n in (("gate", 128), ("up", 128), ("down", 344))}
            for k, v in bases[src].items():
                pc.set_basis(k, v)
            pc.step = 1
            if fused and j == 1:
                pc.token = eng.proj(0, l).token
    mbs, lean, skip = _plan(2, {1}, batches)
    assert eng._fusable(mbs) == fused
    losses = torch.zeros(2, device="cuda")
    eng._body(mbs, losses)
    torch.cuda.synchronize()
    W = R.init_params(D0, 0)
    per_rank, ref_losses = [], []
    for j in range(2):
        src = (lambda l: (0, l)) if fused else (lambda l: (j, l))
        loss, g = R.rank_pass(D0, W, batches[j][0], batches[j][1], ["ffn_input_only"] * 2,
                              {l: bases[src(l)] for l in range(2)})
        per_rank.append(g)
        ref_losses.append(loss)
    active = {(l, k): ([] if k in cluster_ref.MHA else [0, 1]) for l in range(2)
              for k in cluster_ref.MHA + cluster_ref.FFN}
    avg, skipped = cluster_ref.aggregate(per_rank, active, 2)
    assert np.allclose(losses.cpu().numpy(), ref_losses, rtol=tol, atol=tol)
    for name, shape, off in eng.weights.layout:
        got = eng.grad[off: off + int(np.prod(shape))].view(shape).cpu().numpy()
        if name in skipped:
            assert not got.any(), name
        else:
            assert R.rel_err(got, avg[name]) < tol, name


def test_batched_refresh_finds_dominant_subspace(cuda):
    """linalg.top_r_right_singular_vectors_batched: the subspace it returns
    for matrices with a spectral gap at r matches numpy's SVD (projector
    distance), and it is orthonormal (linalg.py:97-142 semantics)."""
    from paper_2510_16415_b200.linalg import top_r_right_singular_vectors_batched

    rng = np.random.Generator(np.random.PCG64(3))
    mats, refs = [], []
    # odd k (r=33), k == cols (20 x 18), and the C1 down-projection shape
    for (out, n, r) in ((344, 128, 32), (128, 344, 33), (512, 256, 64), (40, 20, 18), (512, 1376, 128)):
        q = min(out, n)
        u, _ = np.linalg.qr(rng.normal(size=(out, q)))
        v, _ = np.linalg.qr(rng.normal(size=(n, q)))
        s = np.concatenate([np.linspace(10, 5, r), np.linspace(1, 0.1, q - r)])
        w = (u * s) @ v.T
        mats.append(torch.tensor(w, dtype=torch.float32, device="cuda"))
        refs.append((v[:, :r], s[:r], r))
    got, theta = top_r_right_singular_vectors_batched(mats, [r for *_, r in refs], iterations=30, seed=23,
                                                      return_values=True)
    for v1, th, (vref, sref, r) in zip(got, theta, refs):
        v1 = v1.double().cpu().numpy()
        th = th.double().cpu().numpy()
        assert v1.shape == vref.shape
        assert np.abs(v1.T @ v1 - np.eye(r)).max() < 1e-4
        assert np.abs(v1 @ v1.T - vref @ vref.T).max() < 1e-3
        # Ritz values: descending, = sigma^2 (linalg.py:127-129)
        assert np.all(np.diff(th) <= 0)
        assert np.abs(th - sref ** 2).max() < 1e-3 * sref[0] ** 2
        # each Ritz vector matches its singular vector up to sign
        assert np.abs(np.abs(np.sum(v1 * vref, axis=0)) - 1).max() < 1e-3


def test_engine_budgeted_refresh_runs_and_is_shared(cuda):
    eng = E.StepEngine(C0, precision="bf16", seqs_per_microbatch=2, r=32, tau=3,
                       svd=__import__("paper_2510_16415_b200.linalg", fromlist=["SvdConfig"]).SvdConfig(
                           rank=32, tolerance=1e-3, max_iterations=10, seed=23), svd_budgeted=True)
    mbs, lean, skip = _plan(2, {1}, _batches(2, 2, seed=9))
    for it in range(5):
        losses = eng.step(mbs, 2, 1e-3, skip=skip, check=True)
        assert bool(torch.isfinite(losses).all())
    pcs = [eng.proj(j, l) for j in range(2) for l in range(2)]
    assert all(pc.refreshes == 2 for pc in pcs)  # iterations 0 and 3 (tau = 3)
    assert eng.proj(0, 0).token == eng.proj(1, 0).token  # shared basis -> fused pass
    assert eng._fusable(mbs)
