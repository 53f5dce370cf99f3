"""GPU parity on the exact benchmarked path (configs[1], LLaMA-60M / C1).

1. The 2-CTA TMA-multicast tcgen05 GEMM (chosen for >= 1024-tile unpaired
   GEMMs: the LM-head logits at bench size) against torch fp32 on the same
   bf16-valued operands: the bench's 16384 x 32000 x 512 logits shape, an odd
   M-tile count, every operand-major combination and the beta=1 accumulate
   epilogue; plus the head-backward GEMMs d_xf / g_unemb at bench size.
2. One full StepEngine degraded step at C1 dims (V 32000, 8 lean layers,
   T 256, r 128 with injected bases; two logical ranks of 3 sequences, rank 1
   failed): fused (one stacked 1536-row pass -> logits on the cluster GEMM,
   grouped CE, 8-job grouped low-rank launches) and unfused (two passes),
   against the float64 oracle's rank passes (harness.py:243-249) + Eq. (1)
   aggregation (cluster.py:292-322). Per-tensor bound: 2x the error of a
   PyTorch bf16-autocast implementation of the same step
   (tests/golden/c1_bf16_calibration.json, tests/golden/make_bf16_calibration.py),
   with a 2e-3 floor.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import cluster_ref, model_ref as R
from paper_2510_16415_b200 import engine as E, model as mdl, runtime

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
C1 = mdl.ModelConfig(vocab=32000, hidden=512, heads=8, ffn_intermediate=1376, layers=8, seq_len=256)
D1 = R.Dims(32000, 512, 8, 1376, 8, 256)
SEQS, RANK = 3, 128
FLOOR = 2e-3


def _engine_bf16():
    key = runtime.EngineKey(vocab=32000, hidden=512, heads=8, ffn=1376, layers=8, seq_len=256, rope=True,
                            precision="bf16")
    return runtime.Engine(key)


def _operand(rows, k, kmajor, gen, scale=1.0):
    full = (torch.randn(rows, k, generator=gen, device="cuda") * scale).to(torch.bfloat16)
    stored = full.contiguous() if kmajor else full.t().contiguous()
    return full.float(), stored


def _rel(out, ref):
    return (out - ref).abs().max().item() / max(ref.abs().max().item(), 1e-12)


@pytest.mark.parametrize("a_km,b_km", [(True, True), (True, False), (False, True), (False, False)])
@pytest.mark.parametrize("shape", [(16384, 32000, 512), (4224, 8192, 128)])  # 16000 tiles; 33 x 32 (odd M tiles)
def test_cluster_multicast_gemm_matches_torch(cuda, shape, a_km, b_km):
    M, N, K = shape
    if shape[0] == 16384 and not (a_km and b_km):
        pytest.skip("bench orientation (K-major x K-major) covers the big shape; majors run at the odd shape")
    eng = _engine_bf16()
    gen = torch.Generator(device="cuda").manual_seed(M + N + K)
    a_full, a = _operand(M, K, a_km, gen)
    b_full, b = _operand(N, K, b_km, gen)
    out = torch.full((M, N), 3.0, device="cuda")
    runtime.gemm(eng, a, a_km, b, b_km, M, N, K, out)
    ref = a_full @ b_full.t()
    torch.cuda.synchronize()
    assert _rel(out, ref) < 2e-5
    runtime.gemm(eng, a, a_km, b, b_km, M, N, K, out, alpha=0.5, beta=1.0)  # accumulate epilogue
    torch.cuda.synchronize()
    assert _rel(out, 1.5 * ref) < 3e-5
    del out, ref


def test_head_backward_gemms_at_bench_size(cuda):
    """d_xf = dlogits W_un (K = 32000) and g_unemb = dlogits^T xf (K = 16384,
    split-K accumulate) at the bench's 16384-row stacked pass."""
    from paper_2510_16415_b200 import _lib

    eng = _engine_bf16()
    b, V, m = 16384, 32000, 512
    gen = torch.Generator(device="cuda").manual_seed(5)
    dl = (torch.randn(b, V, generator=gen, device="cuda") * 1e-3).to(torch.bfloat16)
    xf = torch.randn(b, m, generator=gen, device="cuda").to(torch.bfloat16)
    wun = (torch.randn(V, m, generator=gen, device="cuda") * 0.02).to(torch.bfloat16)
    dxf = torch.empty(b, m, device="cuda")
    runtime.gemm(eng, dl, True, wun, False, b, m, V, dxf)  # B(n, k) = Wun[k, n]: MN-major
    ref = dl.float() @ wun.float()
    torch.cuda.synchronize()
    assert _rel(dxf, ref) < 5e-5
    # the engine's head backward (split-K accumulate into g_unemb, alpha-scaled)
    ws_n = _lib.load().mecefo_workspace_bytes(eng.handle, b, 128)
    ws = torch.empty(int(ws_n), dtype=torch.uint8, device="cuda")
    x_last = torch.randn(b, m, generator=gen, device="cuda")
    fnorm = torch.ones(m, device="cuda")
    inv_f = torch.rsqrt((x_last * x_last).mean(1) + 1e-6)
    g_un = torch.full((V, m), 0.25, device="cuda")
    g_fn = torch.zeros(m, device="cuda")
    dx = torch.empty(b, m, device="cuda")
    _lib.call("mecefo_head_backward", eng.handle, x_last.data_ptr(), fnorm.data_ptr(), inv_f.data_ptr(),
              xf.data_ptr(), dl.data_ptr(), wun.data_ptr(), dx.data_ptr(), None, g_fn.data_ptr(), g_un.data_ptr(),
              0.5, b, ws.data_ptr(), ws.numel(), runtime.stream_ptr())
    ref_g = 0.25 + 0.5 * (dl.float().t() @ xf.float())
    torch.cuda.synchronize()
    assert _rel(g_un, ref_g) < 5e-5


def _calibration():
    with open(os.path.join(HERE, "golden", "c1_bf16_calibration.json")) as f:
        return json.load(f)


def _inputs():
    """tests/golden/make_bf16_calibration.py inputs()."""
    rng = np.random.Generator(np.random.PCG64(2024))
    batches = [(rng.integers(0, D1.vocab, size=(SEQS, D1.seq_len)),
                rng.integers(0, D1.vocab, size=(SEQS, D1.seq_len))) for _ in range(2)]
    brng = np.random.Generator(np.random.PCG64(11))
    bases = {}
    for j in range(2):
        for l in range(D1.layers):
            bases[(j, l)] = {k: np.linalg.qr(brng.normal(size=(n, RANK)))[0]
                             for k, n in (("gate", D1.hidden), ("up", D1.hidden), ("down", D1.ffn))}
    return batches, bases


@pytest.mark.parametrize("fused", [True, False])
def test_c1_degraded_step_matches_oracle(cuda, fused):
    batches, bases = _inputs()
    eng = E.StepEngine(C1, precision="bf16", seqs_per_microbatch=SEQS, r=RANK, tau=10**6)
    for j in range(2):
        for l in range(C1.layers):
            pc = eng.proj(j, l)
            for k, v in bases[(0 if fused else j, l)].items():
                pc.set_basis(k, v)
            pc.step = 1
    if fused:
        for l in range(C1.layers):
            eng.proj(1, l).token = eng.proj(0, l).token
    route, lean, a_mha, skip = E.ring_plan(2, {1}, C1.layers)
    mbs = [E.Microbatch(rank=j, tokens=torch.from_numpy(batches[j][0]).cuda(),
                        targets=torch.from_numpy(batches[j][1]).cuda(), lean=[True] * C1.layers,
                        alpha_mha=[None] * C1.layers, alpha_ffn=0.5, alpha_global=0.5) for j in range(2)]
    assert eng._fusable(mbs) == fused
    losses = torch.zeros(2, device="cuda")
    eng._body(mbs, losses)
    torch.cuda.synchronize()
    eng.check_status(sync=True)

    W = R.init_params(D1, 0)
    per_rank, ref_losses = [], []
    for j in range(2):
        loss, g = R.rank_pass(D1, W, batches[j][0], batches[j][1], ["ffn_input_only"] * C1.layers,
                              {l: bases[(0 if fused else j, l)] for l in range(C1.layers)})
        per_rank.append(g)
        ref_losses.append(loss)
    active = {(l, k): ([] if k in cluster_ref.MHA else [0, 1]) for l in range(C1.layers)
              for k in cluster_ref.MHA + cluster_ref.FFN}
    avg, skipped = cluster_ref.aggregate(per_rank, active, C1.layers)
    cal = _calibration()["fused" if fused else "unfused"]
    assert sorted(skipped) == sorted(skip) == sorted(cal["skipped"])
    errs, bad = {}, {}
    for name, shape, off in eng.weights.layout:
        got = eng.grad[off: off + int(np.prod(shape))].view(shape).cpu().numpy()
        if name in skipped:
            assert not got.any(), name  # select, not multiply
            continue
        e = R.rel_err(got, avg[name])
        errs[name] = e
        bound = max(2.0 * cal["grad_rel_err"][name], FLOOR)
        if not e <= bound:
            bad[name] = (e, bound)
    loss_err = [abs(float(a) - b) for a, b in zip(losses.cpu().numpy(), ref_losses)]
    report = {"fused": fused, "grad_rel_err": errs, "loss_abs_err": loss_err,
              "calibration": cal["grad_rel_err"], "calibration_loss_abs_err": cal["loss_abs_err"]}
    out_dir = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, f"c1_parity_{'fused' if fused else 'unfused'}.json"), "w") as f:
            json.dump(report, f, indent=1, sort_keys=True)
    assert not bad, bad
    for a, c in zip(loss_err, cal["loss_abs_err"]):
        assert a <= max(2.0 * c, 1e-3), (loss_err, cal["loss_abs_err"])
