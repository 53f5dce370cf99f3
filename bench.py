#!/usr/bin/env python
"""MeCeFO degraded-step throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): LLaMA-60M (vocab 32000, hidden 512,
8 heads, FFN 1376, 8 layers), seq 256, 32 sequences (8192 tokens) per
microbatch, low-rank FFN Wgrads r=128, bf16 operands / fp32 accumulation.

A "step" is one MeCeFO training iteration of the whole job: R logical DP
ranks (R = max(2, N) with N GPUs), rank 1 failed, so its ring neighbour runs
BOTH microbatches with the approximate backward (skip-MHA, FFN recompute,
low-rank Wgrad), every other GPU runs its own microbatch exactly; Eq. (1)
all-reduce over NVLink (N > 1) and the fused AdamW step (with the fused
_check_grad flag) with the Eq. (1) skip list. At N = 1 the GPU is the
neighbour of an (emulated) failed rank.

value  = R * 8192 tokens per step / (step time + converged projection
         refresh / tau) — device-timed, max over ranks, inputs resident in
         HBM; the refresh is the device solve to the reference's stopping rule
         (residual <= 1e-9 theta_max, linalg.py:119-142), due every tau = 100.
e2e    = same through the public API with tokens copied from pinned host
         memory every step and the loss read back every step.
Also reported: the fault-free step and the instantaneous / refresh-amortised
MeCeFO drop, the dominant kernel's roofline (CUDA events in the timed
region), peak memory of the degraded vs fault-free GPU, the reference's own
CPU step (faultsim._rank_pass from oracle/_ref) on this host, clocks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model 60M|130M|350M|1B] [--rank R] [--precision bf16|fp32]
                    [--scenario c2|c3] [--defer-layers G] [--budgeted-refresh]
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))

import argparse  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s (8×B200) fault-free vs under failures; MeCeFO throughput drop %"
# SURVEY.md §8 size table: C1 (60M) is the bench workload; C2-C4 dims via --model.
# f = 5461 for 1B is the reference's own shape (padded internally to 5464).
MODELS = {"60M": dict(vocab=32000, hidden=512, heads=8, ffn=1376, layers=8, seq_len=256),
          "130M": dict(vocab=32000, hidden=768, heads=12, ffn=2048, layers=12, seq_len=256),
          "350M": dict(vocab=32000, hidden=1024, heads=16, ffn=2736, layers=24, seq_len=256),
          "1B": dict(vocab=32000, hidden=2048, heads=32, ffn=5461, layers=24, seq_len=256)}
SEQS = 32
FAILED = (1,)
TAU = 100
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def workload(model: str, rank: int) -> str:
    base = f"LLaMA-{model} synthetic seq 256, neighbour runs 2 microbatches with low-rank FFN grads r={rank}"
    if model == "60M" and rank == 128:
        return base + " (configs[1])"
    return base + " (SURVEY.md §8 dims; not the configs[1] bench workload)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------
# CPU reference: the reference's own _rank_pass (oracle/_ref), else the port
# --------------------------------------------------------------------------

def _import_reference():
    """faultsim from oracle/_ref (oracle/build_ref.sh installs it there from
    /root/reference; it travels to the GPU box with the repo). None if absent."""
    if os.path.isdir(os.path.join(REF_DIR, "faultsim")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import faultsim.harness  # noqa: F401
            import faultsim

            return faultsim
        except Exception:
            return None
    return None


def host_info() -> dict:
    info = {"cores": os.cpu_count(), "numpy": np.__version__,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["cpu"] = line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info

        blas = [f"{d.get('internal_api')} {d.get('version')} ({d.get('num_threads')} threads)"
                for d in threadpool_info() if d.get("user_api") == "blas"]
        info["blas"] = blas
    except Exception:
        pass
    return info


class CpuReference:
    """One C1-shaped rank pass on the host: faultsim.harness._rank_pass
    (harness.py:243-249) with injected orthonormal V1 (all layers lean,
    ProjectionCache not due -> SVD excluded) or all layers exact; the oracle
    port (oracle/model_ref.rank_pass) when the reference is not installed.
    Weights, bases and tokens are built once, outside any timing."""

    def __init__(self, dims: dict, rank: int, seqs: int = 2):
        self.fs = _import_reference()
        self.seqs, self.T = seqs, dims["seq_len"]
        rng = np.random.Generator(np.random.PCG64(7))
        self.tokens = rng.integers(0, dims["vocab"], size=(seqs, dims["seq_len"]))
        self.targets = rng.integers(0, dims["vocab"], size=(seqs, dims["seq_len"]))
        L, m, f = dims["layers"], dims["hidden"], dims["ffn"]
        self.bases = {l: {k: np.linalg.qr(rng.normal(size=(n, min(rank, n))))[0]
                          for k, n in (("gate", m), ("up", m), ("down", f))} for l in range(L)}
        self.L = L
        if self.fs is not None:
            from faultsim import model as fm
            from faultsim.linalg import SvdConfig

            cfg = fm.ModelConfig(vocab=dims["vocab"], hidden=m, heads=dims["heads"], ffn_intermediate=f,
                                 layers=L, seq_len=dims["seq_len"])
            self.weights = fm.init_weights(cfg, seed=0)
            self.svd = SvdConfig(rank=rank, tolerance=1e-9, max_iterations=3000, seed=23)
            self.kind = "reference"
        else:
            from oracle import model_ref as R

            self.d = R.Dims(vocab=dims["vocab"], hidden=m, heads=dims["heads"], ffn=f, layers=L,
                            seq_len=dims["seq_len"])
            self.weights = R.init_params(self.d, 0)
            self.kind = "port"

    def rank_pass(self, lean: bool) -> float:
        t0 = time.perf_counter()
        if self.fs is not None:
            from faultsim import approx, harness, model as fm

            modes = [fm.CACHE_FFN_INPUT_ONLY if lean else fm.CACHE_FULL] * self.L
            projs = None
            if lean:
                projs = {}
                for l in range(self.L):
                    pc = approx.ProjectionCache(rank=self.svd.rank, refresh_period=10**9, step=1)
                    pc.basis.update(self.bases[l])
                    projs[l] = pc
            harness._rank_pass(self.weights, self.tokens, self.targets, modes, projs, self.svd)
        else:
            from oracle import model_ref as R

            modes = ["ffn_input_only" if lean else "full"] * self.L
            R.rank_pass(self.d, self.weights, self.tokens, self.targets, modes, self.bases if lean else None)
        return time.perf_counter() - t0

    def baseline(self, reps: int = 5) -> dict:
        lean = min(self.rank_pass(True) for _ in range(reps))
        exact = min(self.rank_pass(False) for _ in range(reps))
        tok = self.seqs * self.T
        return {"value": tok / lean, "unit": "tokens/s", "cores": os.cpu_count(), "kind": self.kind,
                "exact_tokens_per_s": round(tok / exact, 2),
                "sample": f"{'faultsim.harness._rank_pass' if self.kind == 'reference' else 'oracle port'} at "
                          f"C1 shapes, {self.seqs} seq x {self.T} tok, all layers lean (injected V1, SVD excluded; "
                          f"value) and all exact (exact_tokens_per_s), best of {reps} each, fp64, "
                          f"OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS')}",
                "host": host_info()}


def run_reference(args, rank: int, dims: dict):
    if rank != 0:
        return
    ref = CpuReference(dims, args.rank)
    for _ in range(max(0, args.warmup)):
        ref.rank_pass(True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.rank_pass(True)
    dt = time.perf_counter() - t0
    v = args.steps * ref.seqs * ref.T / dt
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / max(1, args.steps),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (uniform tokens, PCG64)",
           "config": {"workload": workload(args.model, args.rank),
                      "sample": f"one lean rank pass of {ref.seqs} sequences per step (the degraded "
                                "neighbour's per-microbatch work at C1 shapes, bounded)"},
           "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": ref.kind,
                            "sample": f"{'faultsim.harness._rank_pass' if ref.kind == 'reference' else 'oracle port'}"
                                      f", all layers lean, {ref.seqs} seq/step", "host": host_info()},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    o = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                        "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                    parts = [p.strip() for p in o.stdout.strip().split(",")]
                    if len(parts) >= 6:
                        self.samples.append(parts)
                except Exception:
                    pass
                self._stop.wait(0.05)

        self._th = threading.Thread(target=run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _profile_records(lib):
    """Aggregate the engine's launch-profiler records by tag and stop it."""
    import ctypes

    from paper_2510_16415_b200 import _lib

    agg = {}
    for i in range(lib.mecefo_profile_count()):
        tag, kms, fl, by = ctypes.c_char_p(), ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
        _lib.check(lib.mecefo_profile_record(i, ctypes.byref(tag), ctypes.byref(kms), ctypes.byref(fl),
                                             ctypes.byref(by)))
        a = agg.setdefault(tag.value.decode(), [0.0, 0, 0.0, 0.0])
        a[0] += kms.value
        a[1] += 1
        a[2] += fl.value
        a[3] += by.value
    lib.mecefo_profile_enable(0)
    return agg


class Job:
    """One bench job: the engine, the synthetic per-rank batches and the
    timing helpers shared by the static and scenario runs."""

    def __init__(self, args, dims, world, rank, local, group):
        import torch

        from paper_2510_16415_b200 import _lib, engine as E, model as mdl
        from paper_2510_16415_b200.linalg import SvdConfig

        self.torch, self.E = torch, E
        self.args, self.world, self.rank, self.group = args, world, rank, group
        self.cfg = mdl.ModelConfig(vocab=dims["vocab"], hidden=dims["hidden"], heads=dims["heads"],
                                   ffn_intermediate=dims["ffn"], layers=dims["layers"], seq_len=dims["seq_len"])
        self.R = max(2, world)
        self.b = SEQS * self.cfg.seq_len
        # the harness's SvdConfig (harness.py:367); the budgeted variant only on request
        svd = (SvdConfig(rank=args.rank, tolerance=1e-3, max_iterations=30, seed=23) if args.budgeted_refresh
               else SvdConfig(rank=args.rank, tolerance=1e-9, max_iterations=3000, seed=23))
        self.eng = E.StepEngine(self.cfg, precision=args.precision, seqs_per_microbatch=SEQS, r=args.rank, tau=TAU,
                                seed=0, svd=svd, svd_budgeted=args.budgeted_refresh, group=group,
                                defer_layers=args.defer_layers, grad_comm=args.grad_comm,
                                overlap_comm=not args.no_overlap)
        self.lib = _lib.load()
        self.host_batches, self.dev_batches = {}, {}
        for j in range(self.R):
            g = np.random.Generator(np.random.PCG64(1000 + j))
            tk = torch.from_numpy(g.integers(0, self.cfg.vocab, size=(SEQS, self.cfg.seq_len))).pin_memory()
            tg = torch.from_numpy(g.integers(0, self.cfg.vocab, size=(SEQS, self.cfg.seq_len))).pin_memory()
            self.host_batches[j] = (tk, tg)
            self.dev_batches[j] = (tk.cuda(), tg.cuda())
        self.lr = 1e-4
        self.graph_launches = {}

    def plan(self, failed, batches):
        route, lean, alpha_mha, skip = self.E.ring_plan(self.R, set(failed), self.cfg.layers)
        mbs = []
        for j in range(self.R):
            if route[j] != self.rank:
                continue  # at N = 1, logical rank j >= 1 lives on the absent GPU j unless adopted
            tk, tg = batches[j]
            mbs.append(self.E.Microbatch(rank=j, tokens=tk, targets=tg, lean=[lean[j]] * self.cfg.layers,
                                         alpha_mha=[None if lean[j] else alpha_mha] * self.cfg.layers,
                                         alpha_ffn=1.0 / self.R, alpha_global=1.0 / self.R))
        return mbs, skip

    def barrier(self):
        if self.group is not None:
            import torch.distributed as dist

            dist.barrier()

    def min_over_ranks(self, v: int) -> int:
        if self.group is None:
            return v
        import torch.distributed as dist

        t = self.torch.tensor([float(min(v, 10**9))], device="cuda", dtype=self.torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return int(t.item())

    def max_over_ranks(self, v: float) -> float:
        if self.group is None:
            return v
        import torch.distributed as dist

        t = self.torch.tensor([v], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def clear_refresh(self, mbs, skip, steps):
        """Run untimed steps past any projection refresh that would otherwise
        fall inside the next timed leg (refresh cost is measured separately,
        amortised over tau)."""
        # collective: every step carries the Eq. (1) all-reduces, so all ranks
        # run the same number of extra steps — until no rank's refresh falls
        # inside the leg (a rank without lean layers never needs one)
        for _ in range(4):  # (legs longer than tau cannot avoid a refresh: bounded)
            k = self.min_over_ranks(self.eng.steps_until_refresh(mbs))
            if k > steps + 1:
                break
            for _ in range(k + 1):
                self.eng.step(mbs, self.R, self.lr, skip=skip, check=False)
            self.torch.cuda.synchronize()

    def capture(self, mbs, skip):
        """Eager step (warms descriptors / caches) then capture the plan."""
        self.eng.step(mbs, self.R, self.lr, skip=skip, check=False)
        n0 = self.lib.mecefo_launch_count()
        self.eng.capture(mbs, self.R, skip)
        self.graph_launches[self.eng.plan_key(mbs, skip)] = (self.lib.mecefo_launch_count() - n0) // 2

    def timed(self, mbs, skip, steps, e2e=False, profile=False, graph=False):
        """K steps bracketed by barrier + synchronize; device time (CUDA events
        on the launching stream), max over ranks."""
        torch = self.torch
        self.clear_refresh(mbs, skip, steps)
        self.barrier()
        torch.cuda.synchronize()
        if profile:
            self.lib.mecefo_profile_enable(1)
        n0 = self.lib.mecefo_launch_count()
        replays = 0
        t_wall = time.perf_counter()
        # e2e: every step's losses are copied to pinned host memory and read by
        # the host (two slots: the host reads step i-2's values while step i
        # is queued, as a training loop logging its loss would; the last two
        # are read after the final synchronize, inside the timed region)
        if e2e:
            hbuf = [torch.empty(self.R, dtype=torch.float32).pin_memory() for _ in range(2)]
            hev = [torch.cuda.Event() for _ in range(2)]
            self.e2e_losses = []
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        for i in range(steps):
            if graph and not self.eng.projections_due(mbs):
                losses = self.eng.replay(self.lr, mbs, skip)
                replays += 1
            else:
                losses = self.eng.step(mbs, self.R, self.lr, skip=skip, check=False)
            if e2e:  # D2H read of the step's result
                j = i % 2
                if i >= 2:
                    hev[j].synchronize()
                    self.e2e_losses.append(hbuf[j].tolist())
                hbuf[j].copy_(losses, non_blocking=True)
                hev[j].record()
        en.record()
        torch.cuda.synchronize()
        if e2e:
            for i in range(max(0, steps - 2), steps):
                self.e2e_losses.append(hbuf[i % 2].tolist())
        wall = time.perf_counter() - t_wall
        launches = self.lib.mecefo_launch_count() - n0 + replays * self.graph_launches.get(
            self.eng.plan_key(mbs, skip), 0)
        ms = st.elapsed_time(en)
        self.barrier()
        self.eng.check_status(sync=True)  # _check_grad / bad ids of the timed steps
        return self.max_over_ranks(ms), launches, wall


def measure_memory(args, dims, job) -> dict:
    """Peak device memory of one eager iteration: the doubled neighbour
    (2 lean microbatches, low-rank Wgrads deferred in groups of
    `defer_layers`), the same with every layer's Wgrads deferred to the end,
    and a fault-free GPU (1 exact microbatch, full caches) — fresh engines
    on the bench's weights (weights + optimizer state are the common base)."""
    import torch

    from paper_2510_16415_b200 import engine as E
    from paper_2510_16415_b200.linalg import SvdConfig

    cfg, b, L = job.cfg, job.b, job.cfg.layers
    out = {}
    w = job.eng.weights
    for name, failed, defer in (("degraded", FAILED, args.defer_layers), ("degraded_defer_all", FAILED, None),
                                ("fault_free", (), args.defer_layers)):
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        eng = E.StepEngine(cfg, precision=args.precision, seqs_per_microbatch=SEQS, r=args.rank, tau=TAU,
                           weights=w, svd=SvdConfig(rank=args.rank, tolerance=1e-9, max_iterations=3000, seed=23),
                           defer_layers=defer)
        mbs, skip = job.plan(failed, job.dev_batches)
        eng.step(mbs, job.R, job.lr, skip=skip, check=False)
        torch.cuda.synchronize()
        out[name + "_gb"] = round((torch.cuda.max_memory_allocated() - base) / 1e9, 3)
        del eng
    m, f = cfg.hidden, cfg.ffn_intermediate
    out["lean_cache_per_microbatch_gb"] = round(L * 2 * b * m * 4 / 1e9, 3)  # {x, x1} fp32 (model.py:416-417)
    out["deferred_wgrad_buffers_per_layer_gb"] = round(2 * b * 2 * (2 * m + 3 * f) / 1e9, 3)
    out["note"] = ("device bytes above the weights' own (fp32 master, bf16 shadow): optimizer state, gradients, "
                   "activations, workspaces; one eager iteration each")
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def run_scenario(args, dims, world, rank, local, group):
    """C2 / C3 (SURVEY.md §8(d) Scenarios): the control plane (cluster.step_cluster,
    cluster.py:242-250, on ClusterConfig(dp=1, pp=R): ring-successor takeover,
    harness.py:382-446 semantics) is driven EVERY iteration; adoptions reset the
    adopted rank's projection caches (harness.py:384-388), which forces a
    converged refresh at its next lean backward. Plans are replayed from a
    plan-keyed CUDA-graph cache (a plan that persists 3 iterations is captured
    once and replayed whenever it recurs; short-lived plans and iterations
    with a due refresh launch eagerly). value = R * 8192 tokens per iteration /
    wall time of the whole loop (refreshes, captures and host control plane
    included); time-averaged drop against the fault-free step."""
    import torch

    from paper_2510_16415_b200 import cluster as cl
    from paper_2510_16415_b200.errors import UnrecoverableRankError

    job = Job(args, dims, world, rank, local, group)
    R, L = job.R, job.cfg.layers
    if args.scenario == "c2":  # rank 1 fails at iteration 20% and recovers 40% later
        k0 = max(1, args.steps // 5)
        fail_at = {k0: [1]}
        recover_at = {k0 + max(1, (2 * args.steps) // 5): [1]}
        sc = cl.FailureScenario(kind="none")
    else:  # c3: rotating failures, per-iteration p with recovery after 2 iterations
        fail_at, recover_at = {}, {}
        victims = tuple((0, s) for s in range(R)) if world > 1 else ((0, 1),)
        sc = cl.FailureScenario(kind="per_iteration", probability=args.fail_prob, recovery_iterations=2,
                                victims=victims, seed=7)
    state = cl.ClusterState(cl.ClusterConfig(dp=1, pp=R, layers=R), sc)
    ff_mbs, ff_skip = job.plan((), job.dev_batches)
    # fault-free reference step (graph replay)
    for _ in range(max(3, args.warmup)):
        job.eng.step(ff_mbs, R, job.lr, skip=ff_skip, check=False)
    job.capture(ff_mbs, ff_skip)
    ms_ff, _, _ = job.timed(ff_mbs, ff_skip, args.steps, graph=True)
    ff_tps = R * job.b * args.steps / (ms_ff / 1000.0)

    # Pre-capture (untimed, like the warm-up): the graphs of every single-failure
    # plan this scenario's victims can produce, so a failure in the timed loop
    # replays a ready graph instead of paying a capture. The projection caches
    # are then reset for every rank: the loop starts cold and pays every
    # converged refresh the reference's schedule asks for (harness.py:384-388).
    precaptured = []
    if not args.no_precapture:
        stages = sorted({v[1] for v in sc.victims} if args.scenario == "c3" else {1})
        for s_ in stages:  # every rank captures every plan (the graphs hold the collectives)
            mbs_p, skip_p = job.plan((s_,), job.dev_batches)
            job.eng.step(mbs_p, R, job.lr, skip=skip_p, check=False)
            job.capture(mbs_p, skip_p)
            precaptured.append([s_])
        for j in range(R):
            for l in range(L):
                job.eng.reset_projection(j, l)
        torch.cuda.synchronize()

    degraded_iters, refreshes, captures, events_log = 0, 0, 0, []
    kinds, marks, refresh_log = [], [], []
    aborted = None  # the reference aborts on an unrecoverable state (cli exit 4): measured up to there
    run_len, last_key = 0, None
    job.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for it in range(args.steps):
        mk = torch.cuda.Event(enable_timing=True)
        mk.record()
        marks.append(mk)
        if args.scenario == "c2":  # scripted fail / recover through the same state machine
            evs = []
            for s in recover_at.get(it, []):
                evs += cl.recover_node(state, (0, s), 0.0, it)
            for s in fail_at.get(it, []):
                state._st[0, s] = 1
                evs.append(cl._event(0.0, it, "fail", (0, s)))
            evs += cl.reassign_takeover(state, 0.0, it)
            cl.validate_state(state)
        else:
            try:
                evs = cl.step_cluster(state, 0.0, it)
            except UnrecoverableRankError as exc:  # every process sees it at the same iteration
                aborted = {"iteration": it, "error": str(exc)}
                marks.pop()
                break
        for ev in evs:
            if ev["kind"] == "adopt":  # harness.py:384-388: the adopted rank's layers start fresh bases
                j = ev["details"]["stage"]
                for l in range(L):
                    job.eng.reset_projection(j, l)
        events_log += [(ev["iteration"], ev["kind"], ev["node"][1]) for ev in evs]
        failed = [s for s in range(R) if state._st[0, s] == 1]
        degraded_iters += bool(failed)
        mbs, skip = job.plan(failed, job.dev_batches)
        key = (tuple(failed), len(mbs))
        run_len = run_len + 1 if key == last_key else 1
        last_key = key
        if job.eng.projections_due(mbs):
            refreshes += 1
            kinds.append("refresh")
            job.eng.step(mbs, R, job.lr, skip=skip, check=False)
            ri = [i for i in job.eng.refresh_info if i]
            refresh_log.append((it, len(ri), max((i["products"] for i in ri), default=0), job.eng._fusable(mbs),
                                round(1000 * getattr(job.eng, "last_refresh_s", 0.0), 2)))
        elif job.eng.has_graph(mbs, skip):
            kinds.append("replay_degraded" if failed else "replay_fault_free")
            job.eng.replay(job.lr, mbs, skip)
        elif run_len >= 3:  # a plan that persists: capture it (reused whenever it recurs)
            captures += 1
            kinds.append("capture")
            job.eng.step(mbs, R, job.lr, skip=skip, check=False)
            job.eng.capture(mbs, R, skip)
        else:  # short-lived plan: eager launches (a capture costs ~2 host-side iterations)
            kinds.append("eager")
            job.eng.step(mbs, R, job.lr, skip=skip, check=False)
    en.record()
    marks.append(en)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = job.max_over_ranks(max(st.elapsed_time(en), 1000 * wall))
    job.eng.check_status(sync=True)
    done = len(kinds)
    tps = R * job.b * done / (ms / 1000.0) if done else 0.0
    breakdown = {}
    for k_, a_, b_ in zip(kinds, marks[:-1], marks[1:]):  # device time between iteration boundaries
        e_ = breakdown.setdefault(k_, [0, 0.0])
        e_[0] += 1
        e_[1] += a_.elapsed_time(b_)
    breakdown = {k_: {"iterations": v[0], "ms_total": round(v[1], 2), "ms_mean": round(v[1] / v[0], 3)}
                 for k_, v in breakdown.items()}
    if rank == 0:
        out = {"metric": METRIC, "value": round(tps, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms / max(1, done), 3), "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "impl": "ours",
               "data": "synthetic (uniform tokens, PCG64)", "iterations_completed": done, "aborted": aborted,
               "config": {"workload": workload(args.model, args.rank), "model": f"LLaMA-{args.model}",
                          "scenario": args.scenario, "logical_ranks": R, "microbatch_tokens": job.b,
                          "fail_prob": args.fail_prob if args.scenario == "c3" else None,
                          "recovery_iterations": 2 if args.scenario == "c3" else None,
                          "refresh_period": TAU, "svd": "converged" if not args.budgeted_refresh else "budgeted"},
               "fault_free_tokens_per_s": round(ff_tps, 1),
               "drop_pct_time_averaged": round(100.0 * (1.0 - tps / ff_tps), 2),
               "degraded_iteration_fraction": round(degraded_iters / max(1, done), 3),
               "eager_refresh_iterations": refreshes, "graph_captures": captures,
               "graphs_cached": len(getattr(job.eng, "_graph_cache", {})),
               "precaptured_failure_plans": precaptured,
               "refreshes": [{"iteration": a_, "matrices": b_, "products_max": c_, "fused": d_, "solve_ms": e_}
                             for a_, b_, c_, d_, e_ in refresh_log[:32]], "iteration_breakdown": breakdown,
               "events": events_log[:64]}
        emit(out)
    _finish(group, job.eng)


_JSON_OUT = None


def _stdout_to_stderr():
    """Route everything written to fd 1 (library banners such as NCCL's
    version line) to stderr; the JSON line still goes to the real stdout."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def emit(obj):
    """The one JSON line of this run, on the real stdout."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--model", default="60M", choices=sorted(MODELS),
                    help="LLaMA dims (SURVEY.md §8 C1-C4); the bench workload is 60M (configs[1])")
    ap.add_argument("--rank", type=int, default=128, help="low-rank r (C4 sweep: 64/128/256)")
    ap.add_argument("--scenario", default=None, choices=["c2", "c3"],
                    help="drive the failure control plane every iteration (SURVEY.md §8(d) C2/C3)")
    ap.add_argument("--fail-prob", type=float, default=0.03)
    ap.add_argument("--defer-layers", type=int, default=4,
                    help="lean layers whose low-rank Wgrads are grouped (bounds the deferred buffers)")
    ap.add_argument("--grad-comm", default="fp32", choices=["fp32", "bf16"],
                    help="dtype of the Eq. (1) gradient all-reduce buckets")
    ap.add_argument("--no-overlap", action="store_true",
                    help="all-reduce the gradient buckets on the compute stream (no overlap with backward)")
    ap.add_argument("--budgeted-refresh", action="store_true",
                    help="30-iteration budgeted projection refresh instead of the converged one")
    ap.add_argument("--no-precapture", action="store_true",
                    help="scenarios: capture failure plans lazily inside the timed loop")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fault-free", action="store_true")
    ap.add_argument("--no-memory", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--eager", action="store_true", help="launch kernels eagerly instead of CUDA-graph replay")
    args = ap.parse_args()
    dims = MODELS[args.model]
    args.warmup = max(args.warmup, 3) if not args.profile_only else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, dims)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        _stdout_to_stderr()  # NCCL's own banner lines must not precede the JSON line
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD

    if args.scenario:
        run_scenario(args, dims, world, rank, local, group)
        return

    job = Job(args, dims, world, rank, local, group)
    eng, lib, R, b, cfg = job.eng, job.lib, job.R, job.b, job.cfg
    degraded, skip_d = job.plan(FAILED, job.dev_batches)
    fault_free, skip_f = job.plan((), job.dev_batches)
    degraded_e2e, _ = job.plan(FAILED, job.host_batches)

    # warm-up (includes the first, converged projection refresh of every lean layer)
    for _ in range(args.warmup):
        eng.step(degraded, R, job.lr, skip=skip_d, check=False)
    torch.cuda.synchronize()
    refresh_info = list(eng.refresh_info)
    if args.profile_only:
        torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off captures only the timed steps
        ms, _, _ = job.timed(degraded, skip_d, args.steps)
        torch.cuda.cudart().cudaProfilerStop()
        if rank == 0:
            emit({"profile_only": True, "ms_per_step": ms / args.steps})
        return

    # value: CUDA-graph replay of the degraded iteration, inputs resident in HBM
    use_graph = not args.eager
    if use_graph:
        job.capture(degraded, skip_d)
    with ClockSampler(local) as clk:
        ms, launches, wall = job.timed(degraded, skip_d, args.steps, graph=use_graph)
    tokens_per_step = R * b
    value_steady = tokens_per_step * args.steps / (ms / 1000.0)
    # the projection refresh of this GPU's lean layers, due once per tau steps:
    # timed separately (median of 3, device-synchronised) and amortised into
    # `value` — the timed legs themselves never contain a refresh
    t_refresh = float(np.median([eng.refresh_cost(degraded) for _ in range(3)])) if degraded else 0.0
    t_refresh = job.max_over_ranks(t_refresh)
    refresh_s_per_step = t_refresh / eng.tau
    value = tokens_per_step / ((ms / args.steps) / 1000.0 + refresh_s_per_step)
    t_budget = None
    if not args.budgeted_refresh and degraded:  # the budgeted 30-iteration variant, for comparison only
        from paper_2510_16415_b200.linalg import top_r_right_singular_vectors_batched

        mats = [eng.weights.layers[l].kind(k) for l in range(cfg.layers) for k in ("gate", "up", "down")]
        rks = [min(args.rank, m_.shape[1]) for m_ in mats]
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            top_r_right_singular_vectors_batched(mats, rks, 30, 23)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t_budget = float(np.median(ts))
    # per-kernel attribution: the same degraded iteration, eager, with CUDA
    # events around every kernel group (own timed region of K steps)
    ms_prof, _, _ = job.timed(degraded, skip_d, args.steps, profile=True)

    agg = _profile_records(lib)
    hbm, bf16, bf16_sus, peak_src = _peaks()
    top = sorted(agg.items(), key=lambda kv: -kv[1][0])
    roofline = None
    kernels = []
    kernel_ms = sum(v[0] for v in agg.values())
    for tag, (tms, cnt, fl, by) in top[:18]:
        kernels.append({"tag": tag, "ms_total": round(tms, 3), "launches": cnt, "share": round(tms / ms_prof, 4),
                        "tflops": round(fl / (tms / 1e3) / 1e12, 1) if fl else None,
                        "gbs": round(by / (tms / 1e3) / 1e9, 1)})
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            ncu_traffic = json.load(f)
    except Exception:
        ncu_traffic = {}
    if top:
        tag, (tms, cnt, fl, by) = top[0]
        avg_s = tms / cnt / 1e3
        if fl > 0:
            ach = fl / cnt / avg_s / 1e12
            roofline = {"kernel": tag, "bound": "tensor", "achieved": round(ach, 1), "peak": bf16,
                        "unit": "TFLOP/s", "frac": round(ach / bf16, 4),
                        "frac_of_sustained": round(ach / bf16_sus, 4),
                        "traffic": ncu_traffic.get(tag, {}).get("bytes"),
                        "per_launch": f"{fl / cnt / 1e9:.3f} GFLOP algorithmic (2*M*N*K)",
                        "peak_source": f"{peak_src} bf16 burst (kernel timed alone per launch)",
                        "share_of_step": round(tms / ms_prof, 4)}
        else:
            ach = by / cnt / avg_s / 1e9
            roofline = {"kernel": tag, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "traffic": ncu_traffic.get(tag, {}).get("bytes"),
                        "per_launch": f"{by / cnt / 1e6:.2f} MB algorithmic", "peak_source": peak_src,
                        "share_of_step": round(tms / ms_prof, 4)}

    # fault-free step (every GPU one exact microbatch) and instantaneous drop
    ff_value = None
    kernels_ff = None
    if not args.no_fault_free:
        for _ in range(2):
            eng.step(fault_free, R, job.lr, skip=skip_f, check=False)
        if use_graph:
            job.capture(fault_free, skip_f)
        ms_ff, _, _ = job.timed(fault_free, skip_f, args.steps, graph=use_graph)
        ff_value = tokens_per_step * args.steps / (ms_ff / 1000.0)
        ms_ffp, _, _ = job.timed(fault_free, skip_f, args.steps, profile=True)
        agg_ff = _profile_records(lib)
        kernels_ff = [{"tag": t, "ms_per_step": round(v[0] / args.steps, 3), "share": round(v[0] / ms_ffp, 4)}
                      for t, v in sorted(agg_ff.items(), key=lambda kv: -kv[1][0])[:10]]

    # end-to-end through the public API: H2D of inputs + D2H of the loss per step
    if use_graph:
        job.capture(degraded_e2e, skip_d)
    else:
        eng.step(degraded_e2e, R, job.lr, skip=skip_d, check=False)
    ms_e2e, _, _ = job.timed(degraded_e2e, skip_d, args.steps, e2e=True, graph=use_graph)
    e2e_value = tokens_per_step / ((ms_e2e / args.steps) / 1000.0 + refresh_s_per_step)
    h2d = sum(2 * mb.tokens.numel() * 8 for mb in degraded_e2e)
    loss_ok = bool(torch.isfinite(eng.losses).all().item())

    exchange = None
    if group is not None:  # the Eq. (1) all-reduce alone: NCCL bus bandwidth of the whole flat buffer
        nbytes = eng.grad.numel() * (2 if args.grad_comm == "bf16" else 4)
        buf = eng.grad if args.grad_comm == "fp32" else torch.empty(eng.grad.numel(), dtype=torch.bfloat16,
                                                                     device="cuda")
        for _ in range(3):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        job.barrier()
        st_, en_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st_.record()
        for _ in range(10):
            dist.all_reduce(buf)
        en_.record()
        torch.cuda.synchronize()
        t_ar = job.max_over_ranks(st_.elapsed_time(en_) / 10)
        exchange = {"mode": ("bucketed, overlapped with backward on a communication stream"
                             if not args.no_overlap else "bucketed, on the compute stream"),
                    "dtype": args.grad_comm, "bytes": nbytes, "buckets": 2 + -(-cfg.layers // args.defer_layers),
                    "allreduce_whole_buffer_ms": round(t_ar, 3),
                    "busbw_gbs": round(2 * (world - 1) / world * nbytes / (t_ar / 1e3) / 1e9, 1)}

    memory = None
    if world == 1 and not args.no_memory:
        eng.drop_graphs()
        try:
            memory = measure_memory(args, dims, job)
        except Exception as exc:  # pragma: no cover
            memory = {"error": str(exc)}

    if rank != 0:
        _finish(group, eng)
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = CpuReference(dims if args.model == "60M" else MODELS["60M"], 128).baseline()
        except Exception as exc:  # pragma: no cover
            cpu = {"error": str(exc)}
    conv = [i for i in refresh_info if i]
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps + 1000 * refresh_s_per_step, 3),
        "value_steady": round(value_steady, 1), "ms_per_step_steady": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "impl": "ours",
        "data": "synthetic (uniform tokens in [0,32000), PCG64 seeds 1000+j; weights = reference init_weights seed 0)",
        "config": {"workload": workload(args.model, args.rank), "model": f"LLaMA-{args.model}",
                   "global_batch": R * SEQS, "seq_len": cfg.seq_len, "microbatch_tokens": b, "logical_ranks": R,
                   "failed_ranks": list(FAILED), "rank_r": args.rank, "ffn": dims["ffn"],
                   "parallelism": f"dp{world} (MeCeFO ring, NDB neighbour)", "l2": "inputs larger than L2 "
                   "(per-step activations + logits > 126 MB)", "refresh_period": TAU,
                   "defer_layers": args.defer_layers},
        "projection_refresh": {
            "ms": round(1000 * t_refresh, 2), "refresh_period": eng.tau,
            "ms_per_step_amortised": round(1000 * refresh_s_per_step, 3),
            "kind": "budgeted (30 iterations, no stopping rule)" if args.budgeted_refresh else
                    "converged: every lean layer's gate/up/down basis to residual <= 1e-9 theta_max "
                    "(linalg.py:119-142), float64 on the device, one batched solve",
            "products_max": max((i["products"] for i in conv), default=None),
            "residual_max": max((i["residual"] for i in conv), default=None),
            "budgeted_30_iteration_ms": round(1000 * t_budget, 2) if t_budget else None},
        "fault_free_tokens_per_s": round(ff_value, 1) if ff_value else None,
        "kernels_fault_free": kernels_ff,
        "drop_pct_instantaneous": round(100.0 * (1.0 - value_steady / ff_value), 2) if ff_value else None,
        "drop_pct_amortised": round(100.0 * (1.0 - value / ff_value), 2) if ff_value else None,
        "e2e": {"value": round(e2e_value, 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "losses_read_per_rank": len(getattr(job, "e2e_losses", [])),
                "d2h_bytes_per_step": 4 * R},
        "gpu_launches": int(launches), "roofline": roofline, "kernels": kernels,
        "profiled_kernel_ms_per_step": round(kernel_ms / args.steps, 3),
        "gpu_busy_frac_eager": round(kernel_ms / ms_prof, 4),
        "ms_per_step_eager_profiled": round(ms_prof / args.steps, 3),
        "launch_mode": "cuda_graph" if use_graph else "eager", "exchange": exchange, "memory": memory,
        "cpu_baseline": cpu,
        "clocks": clk.summary(), "loss_finite": loss_ok, "wall_s_timed": round(wall, 3),
    }
    emit(out)
    _finish(group, eng)


def _finish(group, eng):
    """Multi-process teardown: drop the captured graphs (they hold NCCL work),
    synchronize, meet at a barrier and exit without destroying the NCCL
    communicator (its destruction with graph-captured collectives can hang)."""
    if group is None:
        return
    import torch
    import torch.distributed as dist

    eng.drop_graphs()
    torch.cuda.synchronize()
    dist.barrier()
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
