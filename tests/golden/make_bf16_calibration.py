"""bf16 tolerance calibration for the C1 (LLaMA-60M) degraded step.

    python tests/golden/make_bf16_calibration.py

SURVEY.md §7.4-2: the bf16 engine's tolerance is k x the error of a PyTorch
bf16-autocast implementation of the same step against the float64 oracle,
measured with tensor_rel_err (pkg/tests/oracles.py:147-149). This script runs
the oracle's rank pass (oracle/model_ref.rank_pass = harness._rank_pass,
pinned to the reference by tests/test_oracle_golden.py) twice on identical
inputs:

  * float64 (np.matmul), and
  * with every matrix product replaced by a PyTorch bf16 matmul (operands and
    output in bf16, fp32 accumulation — what torch.autocast(bfloat16) does to
    matmul/linear), everything else float64;

aggregates both ranks with Eq. (1) (cluster.py:292-322) and records, per
gradient tensor and per rank loss, the bf16 run's error against float64. The
GPU test tests/test_c1_parity_gpu.py bounds the engine's error by 2x these.

Workload: C1 dims (V 32000, hidden 512, 8 heads, ffn 1376, 8 layers, seq 256),
two logical ranks of 3 sequences each, rank 1 failed -> both lean with r=128
low-rank FFN Wgrads (injected orthonormal bases, seed 11), MHA kinds skipped.
"fused": both ranks share the bases (the engine stacks them in one pass);
"unfused": distinct bases per rank (two passes).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import cluster_ref, model_ref as R  # noqa: E402

D = R.Dims(vocab=32000, hidden=512, heads=8, ffn=1376, layers=8, seq_len=256)
SEQS = 3
RANK = 128


def inputs():
    """Same seeds as tests/test_c1_parity_gpu.py."""
    rng = np.random.Generator(np.random.PCG64(2024))
    batches = [(rng.integers(0, D.vocab, size=(SEQS, D.seq_len)), rng.integers(0, D.vocab, size=(SEQS, D.seq_len)))
               for _ in range(2)]
    brng = np.random.Generator(np.random.PCG64(11))
    bases = {}
    for j in range(2):
        for l in range(D.layers):
            bases[(j, l)] = {k: np.linalg.qr(brng.normal(size=(n, RANK)))[0]
                             for k, n in (("gate", D.hidden), ("up", D.hidden), ("down", D.ffn))}
    return batches, bases


def step(W, batches, bases, fused):
    per_rank, losses = [], []
    for j in range(2):
        src = 0 if fused else j
        loss, g = R.rank_pass(D, W, batches[j][0], batches[j][1], ["ffn_input_only"] * D.layers,
                              {l: bases[(src, l)] for l in range(D.layers)})
        per_rank.append(g)
        losses.append(loss)
    active = {(l, k): ([] if k in cluster_ref.MHA else [0, 1]) for l in range(D.layers)
              for k in cluster_ref.MHA + cluster_ref.FFN}
    avg, skipped = cluster_ref.aggregate(per_rank, active, D.layers)
    return avg, skipped, losses


def mm_bf16(a, b):
    ta = torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16)
    tb = torch.from_numpy(np.ascontiguousarray(b)).to(torch.bfloat16)
    return torch.matmul(ta, tb).to(torch.float64).numpy()


def main():
    torch.set_num_threads(os.cpu_count() or 1)
    W = R.init_params(D, 0)
    batches, bases = inputs()
    out = {"config": {"dims": D.__dict__, "seqs_per_rank": SEQS, "rank": RANK, "ranks": 2, "failed": [1],
                      "token_seed": 2024, "basis_seed": 11, "weights_seed": 0,
                      "bf16_model": "torch.matmul in bfloat16 (operands + output bf16, fp32 accumulate) for every "
                                    "matrix product; float64 elsewhere",
                      "metric": "tensor_rel_err = max|a-b| / max(max|a|, max|b|) (pkg/tests/oracles.py:147-149)"}}
    for fused in (True, False):
        R.MM = R._mm_f64
        ref, skipped, ref_loss = step(W, batches, bases, fused)
        R.MM = mm_bf16
        low, _, low_loss = step(W, batches, bases, fused)
        R.MM = R._mm_f64
        errs = {n: R.rel_err(low[n], ref[n]) for n in ref}
        out["fused" if fused else "unfused"] = {
            "grad_rel_err": errs, "skipped": skipped,
            "loss_abs_err": [abs(a - b) for a, b in zip(low_loss, ref_loss)], "loss_ref": ref_loss}
        print(("fused" if fused else "unfused"), "max grad err", max(errs.values()), "loss err",
              out["fused" if fused else "unfused"]["loss_abs_err"], flush=True)
    with open(os.path.join(HERE, "c1_bf16_calibration.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
