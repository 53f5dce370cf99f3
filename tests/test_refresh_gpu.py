"""GPU: the converged device projection refresh (linalg.py:97-142 with the
harness's SvdConfig(r, 1e-9, 3000, seed + 23), approx.py:66-87).

It must compute the reference's object: the bases are compared with bases
produced by the REFERENCE itself (tests/golden/c0_rank_pass.npz at C0 and
tests/golden/c1_svd_l0.npz at C1, made by make_golden.py / make_svd_golden.py)
by projector distance ||V1 V1^T - V2 V2^T||_2 (sine of the largest principal
angle), and every returned basis must satisfy the reference's stopping rule
||W^T W v - theta v|| <= tol * theta_max, re-checked here in float64 numpy.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import model_ref as R
from paper_2510_16415_b200 import approx, engine as E, model as mdl
from paper_2510_16415_b200.errors import ContractViolation, SvdConvergenceError
from paper_2510_16415_b200.linalg import SvdConfig, refresh_bases, top_r_right_singular_vectors

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SVD = SvdConfig(rank=128, tolerance=1e-9, max_iterations=3000, seed=23)


def proj_dist(a, b):
    a = np.linalg.qr(np.asarray(a, np.float64))[0]
    b = np.linalg.qr(np.asarray(b, np.float64))[0]
    s = np.linalg.svd(a.T @ b, compute_uv=False)
    return float(np.sqrt(max(0.0, 1.0 - s.min() ** 2)))


def ref_residual(w, v):
    """linalg.py:131-135 on the returned basis (Ritz values of v)."""
    w = np.asarray(w, np.float64)
    v = np.asarray(v, np.float64)
    b = w.T @ w
    th = np.einsum("ij,ij->j", v, b @ v)
    res = np.linalg.norm(b @ v - v * th, axis=0).max()
    return res / np.linalg.eigvalsh(b)[-1]


def test_c0_bases_match_reference(cuda):
    d = R.Dims(64, 128, 4, 344, 2, 64)
    W = R.init_params(d, 0)
    gold = np.load(os.path.join(GOLD, "c0_rank_pass.npz"))
    mats, names = [], []
    for l in range(2):
        for k in ("gate", "up", "down"):
            mats.append(torch.tensor(W[f"layers.{l}.{k}"], dtype=torch.float32, device="cuda"))
            names.append(f"v1.{l}.{k}")
    info = []
    got = refresh_bases(mats, [32] * 6, SvdConfig(rank=32, tolerance=1e-9, max_iterations=3000, seed=23), info=info)
    for g, n, m, inf in zip(got, names, mats, info):
        assert inf["converged"] and inf["residual"] <= 1e-9, (n, inf)
        assert proj_dist(g.cpu().numpy(), gold[n]) < 1e-3, n
        assert ref_residual(m.cpu().numpy(), g.cpu().numpy()) < 1e-7, n  # fp32 output rounding of V


def test_c1_bases_match_reference(cuda):
    """C1 (LLaMA-60M) init matrices: gate/up are tall (1376 x 512, iterated on
    W^T W), down is wide (512 x 1376, iterated on W W^T and checked on W^T W).
    The reference needs hundreds of iterations here (c1_svd_l0.json)."""
    gold = np.load(os.path.join(GOLD, "c1_svd_l0.npz"))
    with open(os.path.join(GOLD, "c1_svd_l0.json")) as f:
        meta = json.load(f)["kinds"]
    cfg = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=8, seq_len=256)
    w = mdl.init_weights(cfg, 0, precision="bf16")
    mats = [w.layers[0].kind(k) for k in ("gate", "up", "down")]
    info = []
    got = refresh_bases(mats, [128] * 3, SVD, info=info)
    for k, g, m, inf in zip(("gate", "up", "down"), got, mats, info):
        assert inf["converged"] and inf["residual"] <= 1e-9, (k, inf)
        assert inf["products"] < meta[k]["iterations"], (k, inf, meta[k])
        dist = proj_dist(g.cpu().numpy(), gold[f"v1.{k}"])
        assert dist < 1e-3, (k, dist)
        assert ref_residual(m.cpu().numpy(), g.cpu().numpy()) < 1e-7, k


@pytest.mark.parametrize("shape,r", [((300, 96), 16), ((96, 300), 16), ((64, 64), 64), ((200, 130), 128),
                                     ((37, 91), 20), ((1376, 512), 256)])
def test_random_matrices_vs_numpy_svd(cuda, shape, r):
    rng = np.random.Generator(np.random.PCG64(shape[0] * 7 + r))
    # decaying spectrum with a gap at r (the subspace is well defined)
    u = np.linalg.qr(rng.normal(size=(shape[0], min(shape))))[0]
    v = np.linalg.qr(rng.normal(size=(shape[1], min(shape))))[0]
    s = np.linspace(2.0, 1.0, min(shape))
    s[r:] *= 0.5
    w = (u * s) @ v.T
    info = []
    got = refresh_bases([torch.tensor(w, dtype=torch.float32, device="cuda")], [r],
                        SvdConfig(rank=r, tolerance=1e-9, max_iterations=3000, seed=1), info=info)[0]
    ref = np.linalg.svd(w.astype(np.float32).astype(np.float64))[2][:r].T
    assert info[0]["converged"], info
    assert proj_dist(got.cpu().numpy(), ref) < 1e-4, (shape, r)
    g = got.cpu().numpy().astype(np.float64)
    assert np.abs(g.T @ g - np.eye(r)).max() < 1e-5  # orthonormal


def test_zero_matrix_returns_standard_basis(cuda):
    z = torch.zeros(40, 24, device="cuda")
    got = top_r_right_singular_vectors(z, SvdConfig(rank=5, tolerance=1e-9, max_iterations=10, seed=0))
    assert torch.equal(got.cpu(), torch.eye(24)[:, :5])


def test_nonconvergence_raises_svd_error(cuda):
    cfg = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=8, seq_len=256)
    w = mdl.init_weights(cfg, 0, precision="bf16").layers[0].kind("gate")
    with pytest.raises(SvdConvergenceError) as ei:
        top_r_right_singular_vectors(w, SvdConfig(rank=128, tolerance=1e-12, max_iterations=3, seed=23))
    assert ei.value.residual > 1e-12


def test_rank_exceeding_columns_is_a_contract_violation(cuda):
    with pytest.raises(ContractViolation):
        top_r_right_singular_vectors(torch.ones(8, 4, device="cuda"), SvdConfig(rank=5))


def test_engine_refresh_is_the_converged_reference_basis(cuda):
    """A StepEngine with no injected bases refreshes every lean layer at its
    first neighbour backward (approx.py:74-75) with the converged device solve:
    the bases equal the reference's (c0_rank_pass.npz) to projector distance
    1e-3, and refresh counters follow approx.py:76-87."""
    c0 = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64)
    gold = np.load(os.path.join(GOLD, "c0_rank_pass.npz"))
    eng = E.StepEngine(c0, precision="fp32", seqs_per_microbatch=2, r=32, tau=100,
                       svd=SvdConfig(rank=32, tolerance=1e-9, max_iterations=3000, seed=23))
    rng = np.random.Generator(np.random.PCG64(0))
    tk = torch.from_numpy(rng.integers(0, 64, size=(2, 64))).cuda()
    mbs = [E.Microbatch(rank=j, tokens=tk, targets=tk, lean=[True] * 2, alpha_mha=[None] * 2, alpha_ffn=0.5,
                        alpha_global=0.5) for j in range(2)]
    eng._body(mbs, torch.zeros(2, device="cuda"))  # before any update: bases of the init weights
    torch.cuda.synchronize()
    for l in range(2):
        pc = eng.proj(0, l)
        assert pc.refreshes == 1 and pc.svd_calls == 3 and pc.step == 1
        for k in approx.FFN_KINDS:
            assert proj_dist(pc.basis[k].cpu().numpy(), gold[f"v1.{l}.{k}"]) < 1e-3, (l, k)
    assert all(i["converged"] for i in eng.refresh_info)
