"""GPU: the GEMM engine (tcgen05/TMA bf16 and fp32 SIMT) against torch fp32.

bf16 operands are exactly representable in fp32, so the only difference to
a float32 matmul of the same (bf16-valued) operands is the summation order:
the tolerance is fp32-accumulation level, not bf16 level.
"""

import pytest
import torch

from paper_2510_16415_b200 import _lib, runtime

pytestmark = pytest.mark.gpu

# (4696, 1000, 1096) takes BN = 256 and (K >= 1024) the CTA-pair
# cta_group::2 path, with an odd M-tile count (the last pair's
# second CTA has no rows), a ragged last N tile and a partial k-block;
# (8192, 512, 512) the single-CTA BN = 256 path
SHAPES = [(128, 64, 64), (256, 256, 128), (296, 200, 104), (1000, 768, 520), (64, 16, 16), (8192, 512, 512),
          (512, 128, 8192), (4696, 1000, 1096)]


def _engine(precision):
    key = runtime.EngineKey(vocab=64, hidden=128, heads=4, ffn=344, layers=1, seq_len=64, rope=True,
                            precision=precision)
    return runtime.Engine(key)


def _operand(rows, k, kmajor, dtype, gen):
    full = torch.randn(rows, k, generator=gen, device="cuda").to(dtype)
    stored = full.contiguous() if kmajor else full.t().contiguous()
    return full.float(), stored


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("a_km", [True, False])
@pytest.mark.parametrize("b_km", [True, False])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_matches_torch(cuda, precision, a_km, b_km, shape):
    M, N, K = shape
    if precision == "fp32" and M * N * K > 2**31:
        pytest.skip("large fp32 SIMT case covered elsewhere")
    eng = _engine(precision)
    dt = runtime.compute_dtype(precision)
    gen = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    a_full, a = _operand(M, K, a_km, dt, gen)
    b_full, b = _operand(N, K, b_km, dt, gen)
    out = torch.full((M, N), 7.0, device="cuda")
    runtime.gemm(eng, a, a_km, b, b_km, M, N, K, out)
    ref = a_full @ b_full.t()
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item() / max(ref.abs().max().item(), 1e-12)
    assert err < 2e-5, (err, shape, a_km, b_km)
    # beta = 1 accumulates
    runtime.gemm(eng, a, a_km, b, b_km, M, N, K, out, alpha=0.5, beta=1.0)
    err2 = (out - 1.5 * ref).abs().max().item() / max(ref.abs().max().item(), 1e-12)
    assert err2 < 3e-5


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("dims", [(64, 48, 256, 16), (1376, 512, 8192, 128), (512, 1376, 4096, 128), (16, 32, 24, 16)])
def test_lowrank_wgrad_association_order(cuda, precision, dims):
    """approx.py:24-42: out = g_y (x^T v1) v1^T, split-K long contraction."""
    n_out, n_in, b, r = dims
    eng = _engine(precision)
    dt = runtime.compute_dtype(precision)
    gen = torch.Generator(device="cuda").manual_seed(n_out + n_in + b + r)
    g_y = torch.randn(n_out, b, generator=gen, device="cuda").to(dt)
    x = torch.randn(n_in, b, generator=gen, device="cuda").to(dt)
    v1, _ = torch.linalg.qr(torch.randn(n_in, r, generator=gen, device="cuda", dtype=torch.float64))
    v1 = v1.to(dt).contiguous()
    out = torch.zeros(n_out, n_in, device="cuda")
    wsp, wsn = eng.workspace(b, r)
    _lib.call("mecefo_lowrank_wgrad", eng.handle, g_y.data_ptr(), x.data_ptr(), v1.data_ptr(), out.data_ptr(),
              n_out, n_in, b, r, 1.0, wsp, wsn, runtime.stream_ptr())
    ref = (g_y.double() @ (x.double().t() @ v1.double())) @ v1.double().t()
    torch.cuda.synchronize()
    err = (out.double() - ref).abs().max().item() / ref.abs().max().item()
    tol = 1e-2 if precision == "bf16" else 1e-5  # bf16: P and Q are rounded to bf16 between the GEMMs
    assert err < tol, err
