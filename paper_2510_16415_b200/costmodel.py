"""Analytic FLOP accounting — the subset of faultsim.costmodel the step needs.

Two uses: (1) the reference's simulated clock
(harness.py:442-446) drives *scheduled* failure times, so a drop-in
run_training must reproduce `iteration_cost` exactly; (2) algorithmic FLOPs
for the roofline (bench.py). The timeline simulator / policies of
costmodel.py:241-357 are out of scope.
"""

from __future__ import annotations

from . import cluster as cl

FPROP, WGRAD, DGRAD, RCOMP, APPROX_WGRAD = "fprop", "wgrad", "dgrad", "rcomp", "approx_wgrad"
MODE_STANDARD, MODE_NEIGHBOR_APPROX, MODE_NEIGHBOR_NAIVE = "standard", "neighbor_approx", "neighbor_naive"
POLICY_APPROX, POLICY_NAIVE, POLICY_CHECKPOINT = "approx", "naive", "checkpoint"
SVD_CHARGED_ITERATIONS = 30  # costmodel.py:41


def linear_flops(b: int, m: int, n: int, op: str, r: int | None = None) -> int:
    """costmodel.py:47-57: 2bmn, or 2brn + 2brm + 2rmn for the projected Wgrad."""
    if op == APPROX_WGRAD:
        return 2 * r * (b * n + b * m + m * n)
    return 2 * b * m * n


def svd_flops(m: int, n: int, r: int, iterations: int = SVD_CHARGED_ITERATIONS) -> int:
    """costmodel.py:60-64."""
    k = min(n, r + 4)
    return 2 * m * n * n + iterations * (2 * n * n * k + 2 * n * k * k)


def block_flops(cfg, mode: str, r: int, tau: int, tokens: int) -> int:
    """Total of costmodel.block_cost (:103-139) — the seven linear layers only."""
    m, f = cfg.hidden, cfg.ffn_intermediate
    mats = [(m, m)] * 4 + [(f, m), (f, m), (m, f)]
    total = sum(2 * tokens * a * b for a, b in mats)  # Fprop
    if mode in (MODE_STANDARD, MODE_NEIGHBOR_NAIVE):
        return total + 2 * sum(2 * tokens * a * b for a, b in mats)  # Wgrad + Dgrad
    for a, b in mats[4:]:
        re = min(r, b)
        total += 2 * tokens * a * b * 2  # Rcomp + Dgrad
        total += linear_flops(tokens, a, b, APPROX_WGRAD, re)
        total += svd_flops(a, b, re) // tau
    return total


def iteration_cost(state: cl.ClusterState, model_cfg, policy: str, r: int, tau: int, tokens_per_rank: int):
    """costmodel.py:206-238: (worst node flops, its first stage, total, 0),
    computed natively on the cluster state (mecefo_iteration_cost,
    libmecefo_ctl.so). Activation bytes are not tracked here (always 0)."""
    import ctypes

    from . import pcg

    worst, stage, total = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
    rc = pcg.load().mecefo_iteration_cost(state._h, int(model_cfg.hidden), int(model_cfg.ffn_intermediate),
                                          1 if policy == POLICY_APPROX else 0, int(r), int(tau),
                                          int(tokens_per_rank), ctypes.byref(worst), ctypes.byref(stage),
                                          ctypes.byref(total))
    if rc:
        from .errors import ContractViolation

        raise ContractViolation("iteration_cost: invalid arguments")
    return worst.value, stage.value, total.value, 0


def iteration_cost_py(state: cl.ClusterState, model_cfg, policy: str, r: int, tau: int, tokens_per_rank: int):
    """The same accounting in Python (cross-check of the native version)."""
    cfg = state.cfg
    doubled = MODE_NEIGHBOR_APPROX if policy == POLICY_APPROX else MODE_NEIGHBOR_NAIVE
    per_mode = {}
    worst, worst_stage, total = 0, 0, 0
    for node in state.nodes():
        stages = state.executing_stages(node)
        if not stages:
            continue
        mode = MODE_STANDARD if state.status[node] == cl.HEALTHY else doubled
        if mode not in per_mode:
            per_mode[mode] = block_flops(model_cfg, mode, r, tau, tokens_per_rank)
        node_flops = sum(len(cfg.layers_of_stage(s)) for s in stages) * per_mode[mode]
        total += node_flops
        if node_flops > worst:
            worst, worst_stage = node_flops, stages[0]
    return worst, worst_stage, total, 0


# ----------------------------------------------------------------------------
# Required-work FLOPs per token for the roofline: the cost
# model's linear layers plus attention core and LM head; the lean step skips
# the down-projection recompute (model.py:243-259 never reads `down`).
# ----------------------------------------------------------------------------

def standard_flops_per_token(cfg) -> int:
    m, f, L, T, V = cfg.hidden, cfg.ffn_intermediate, cfg.layers, cfg.seq_len, cfg.vocab
    return L * (24 * m * m + 18 * m * f + 6 * T * m) + 6 * m * V


def lean_flops_per_token(cfg, r: int, tokens: int) -> int:
    """Per token of one lean microbatch of `tokens` rows (incl. the up-projection
    2 r out in per matrix, amortised over the microbatch)."""
    m, f, L, T, V = cfg.hidden, cfg.ffn_intermediate, cfg.layers, cfg.seq_len, cfg.vocab
    rm, rf = min(r, m), min(r, f)
    per_tok = 8 * m * m + 2 * T * m  # forward attention side (QKV, O, scores/PV)
    per_tok += 6 * m * f  # forward FFN (gate, up, down)
    per_tok += 4 * m * f + 4 * m * f + 2 * m * f  # recompute gate|up, Dgrad (d_act, d_h2)
    per_tok += 2 * rm * (m + f) * 2 + 2 * rf * (f + m)  # P and Q contractions
    up_proj = 2 * (rm * f * m) * 2 + 2 * rf * m * f  # Q V1^T per matrix, per microbatch
    return L * per_tok + L * up_proj // tokens + 6 * m * V
