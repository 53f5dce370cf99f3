"""GPU: bad inputs and non-finite gradients raise what the reference raises,
through the engine's device status word (never an out-of-range access):

  * token / target ids outside [0, vocab): the reference's gather and CE
    raise IndexError (model.py:463, 505) -> ContractViolation here;
  * non-finite gradient: optim.py:55-57 _check_grad -> NumericalFailure,
    fused into the AdamW read of g and read at the iteration boundary;
  * aggregate_gradients (cluster.py:292-322) on the reference's numpy dicts.
"""

import numpy as np
import pytest
import torch

from oracle import cluster_ref, model_ref as R
from paper_2510_16415_b200 import cluster as cl, engine as E, model as mdl
from paper_2510_16415_b200.errors import ConsistencyError, ContractViolation, NumericalFailure

pytestmark = pytest.mark.gpu

C0 = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64)


def _engine():
    eng = E.StepEngine(C0, precision="bf16", seqs_per_microbatch=2, r=32, tau=10**6)
    rng = np.random.Generator(np.random.PCG64(11))
    for j in range(2):
        for l in range(2):
            pc = eng.proj(j, l)
            for k, n in (("gate", 128), ("up", 128), ("down", 344)):
                pc.set_basis(k, np.linalg.qr(rng.normal(size=(n, 32)))[0])
            pc.step = 1
    return eng


def _mbs(tok0, tgt0, device=True):
    rng = np.random.Generator(np.random.PCG64(2))
    out = []
    for j in range(2):
        tk = torch.from_numpy(tok0 if j == 0 else rng.integers(0, 64, size=(2, 64)))
        tg = torch.from_numpy(tgt0 if j == 0 else rng.integers(0, 64, size=(2, 64)))
        if device:
            tk, tg = tk.cuda(), tg.cuda()
        out.append(E.Microbatch(rank=j, tokens=tk, targets=tg, lean=[True] * 2, alpha_mha=[None] * 2,
                                alpha_ffn=0.5, alpha_global=0.5))
    return out


def _skip():
    return E.ring_plan(2, {1}, 2)[3]


@pytest.mark.parametrize("device", [True, False])
@pytest.mark.parametrize("what", ["token", "target"])
def test_out_of_vocab_ids_raise_contract_violation(cuda, device, what):
    rng = np.random.Generator(np.random.PCG64(1))
    tok, tgt = rng.integers(0, 64, size=(2, 64)), rng.integers(0, 64, size=(2, 64))
    (tok if what == "token" else tgt)[1, 7] = 64 if what == "token" else -3
    eng = _engine()
    w0 = eng.weights.master.clone()
    with pytest.raises(ContractViolation, match=what):
        eng.step(_mbs(tok, tgt, device), 2, 1e-3, skip=_skip(), check=False)
        eng.check_status(sync=True)
    torch.cuda.synchronize()  # no fault: every access stayed in range
    if not device:  # host ids are validated before anything is launched
        assert torch.equal(eng.weights.master, w0)
    # the engine stays usable after the error
    eng.step(_mbs(rng.integers(0, 64, size=(2, 64)), rng.integers(0, 64, size=(2, 64))), 2, 1e-3, skip=_skip(),
             check=False)
    eng.check_status(sync=True)
    assert bool(torch.isfinite(eng.losses).all())


def test_nonfinite_gradient_raises_numerical_failure_without_extra_pass(cuda):
    """check=False (the bench path) still does _check_grad: the flag comes
    from the fused AdamW read of g."""
    rng = np.random.Generator(np.random.PCG64(4))
    eng = _engine()
    eng.weights.master[eng.weights.offsets["layers.1.down"]] = float("nan")
    eng.weights.sync_shadow()
    with pytest.raises(NumericalFailure):
        eng.step(_mbs(rng.integers(0, 64, size=(2, 64)), rng.integers(0, 64, size=(2, 64))), 2, 1e-3,
                 skip=_skip(), check=False)
        eng.check_status(sync=True)


def test_nonfinite_gradient_checked_mode_raises_before_update(cuda):
    rng = np.random.Generator(np.random.PCG64(5))
    eng = _engine()
    eng.weights.master[eng.weights.offsets["layers.0.gate"] + 5] = float("inf")
    eng.weights.sync_shadow()
    w0 = eng.weights.master.clone()
    with pytest.raises(NumericalFailure):
        eng.step(_mbs(rng.integers(0, 64, size=(2, 64)), rng.integers(0, 64, size=(2, 64))), 2, 1e-3,
                 skip=_skip(), check=True)
    assert torch.equal(eng.weights.master, w0)  # optim.py: raised before any update


def test_aggregate_gradients_matches_reference_on_numpy_dicts(cuda):
    rng = np.random.Generator(np.random.PCG64(8))
    L, R_ = 2, 3
    names = list(cluster_ref.GLOBAL) + [f"layers.{l}.{k}" for l in range(L)
                                        for k in cluster_ref.MHA + cluster_ref.FFN]
    per_rank = [{n: rng.normal(size=(4, 5)) for n in names} for _ in range(R_)]
    per_rank[1]["layers.0.q"][:] = np.nan  # rank 1 is excluded from layer 0's MHA set: must not leak
    active = {(l, k): ([0, 2] if (k in cluster_ref.MHA and l == 0) else ([] if k in cluster_ref.MHA else
                                                                       [0, 1, 2]))
              for l in range(L) for k in cluster_ref.MHA + cluster_ref.FFN}
    ref, ref_skip = cluster_ref.aggregate(per_rank, active, L)
    got, skip = cl.aggregate_gradients(per_rank, active, L)
    assert sorted(skip) == sorted(ref_skip) and "layers.1.q" in skip
    for n, v in ref.items():
        g = got[n].cpu().numpy()
        assert np.isfinite(g).all(), n
        assert R.rel_err(g, v) < 1e-6, n
    missing = [dict(d) for d in per_rank]
    del missing[2]["layers.1.gate"]
    with pytest.raises(ConsistencyError):
        cl.aggregate_gradients(missing, active, L)
