"""Fused MeCeFO training step on one GPU (one process per GPU).

The reference runs every logical DP rank sequentially in one process, keeps
per-rank gradient dicts and averages them afterwards (harness.py:406-428,
cluster.py:292-322). Here each process owns persistent HBM buffers and runs
the microbatches assigned to its GPU by the replicated control plane:

  * activations: the residual stream x_0..x_L and x1_l (fp32) — the whole lean
    cache — plus full caches only for layers run exactly;
  * gradients: ONE flat fp32 buffer with the parameter layout. Every backward
    kernel accumulates g += alpha * dW straight into it, alpha being the
    Eq. (1) weight 1/|N_{l,#}| of that microbatch (or nothing at all when the
    microbatch is outside the active set: select, not multiply);
  * exchange: one NCCL all-reduce(sum) of the flat buffer over NVLink turns the
    pre-weighted local sums into the Eq. (1) averages on every GPU;
  * update: one fused multi-tensor AdamW launch with per-parameter step
    counts and the Eq. (1) skip list, which also refreshes the bf16 shadow.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, approx, model as mdl, optim as op, runtime
from .errors import ContractViolation, NumericalFailure
from .linalg import SvdConfig


@dataclass
class Microbatch:
    """One logical DP rank's work this iteration (harness.py:406-418)."""

    rank: int                 # logical DP rank j
    tokens: torch.Tensor      # (B, T) int64, device or pinned host
    targets: torch.Tensor     # (B, T) int64
    lean: list                # per layer: True -> CACHE_FFN_INPUT_ONLY + neighbor backward
    alpha_mha: list           # per layer: Eq. (1) weight for MHA grads, or None (not in N_MHA)
    alpha_ffn: float          # 1/|N_FFN| = 1/R
    alpha_global: float       # 1/R (global params average over all ranks)


class StepEngine:
    def __init__(self, cfg: mdl.ModelConfig, precision: str = "bf16", seqs_per_microbatch: int = 32, r: int = 128,
                 tau: int = 100, optim_cfg: op.OptimConfig | None = None, seed: int = 0,
                 weights: mdl.ModelWeights | None = None, svd: SvdConfig | None = None, svd_budgeted: bool = False,
                 group=None, fuse_lean: bool = True, max_group: int = 2, defer_layers: int | None = 4,
                 grad_comm: str = "fp32", overlap_comm: bool = True):
        runtime.require_cuda()
        self.cfg = cfg
        self.precision = precision
        self.weights = weights if weights is not None else mdl.init_weights(cfg, seed, precision=precision)
        self.device = self.weights.master.device
        self.eng = runtime.engine_for(cfg, precision)
        self.dtype = self.eng.dtype
        self.seqs = seqs_per_microbatch
        self.b = seqs_per_microbatch * cfg.seq_len
        self.r = r
        self.tau = tau
        self.svd = svd if svd is not None else SvdConfig(rank=r, tolerance=1e-9, max_iterations=3000, seed=seed + 23)
        self.svd_budgeted = svd_budgeted
        # every due basis of an iteration is refreshed in ONE batched device
        # solve (converged to svd.tolerance, or the budgeted fixed iteration)
        self.batched_refresh = True
        self.refresh_info: list = []
        self.group = group
        self.opt = op.OptimState(optim_cfg or op.OptimConfig())
        self.opt.ensure_flat(self.weights.total, self.device)
        self.grad = torch.zeros(self.weights.total, dtype=torch.float32, device=self.device)
        self.lws = [lw.struct() for lw in self.weights.layers]
        # Lean microbatches of one GPU can run as ONE pass over stacked rows
        # (all row-wise / token-parallel kernels; per-rank losses kept apart):
        # buffers are sized for `max_group` microbatches.
        self.fuse_lean = fuse_lean
        self.max_group = max(1, max_group)
        self.iter = 0
        b, m, L = self.b * self.max_group, cfg.hidden, cfg.layers
        f32 = dict(dtype=torch.float32, device=self.device)
        self.xs = [torch.empty(b, m, **f32) for _ in range(L + 1)]
        self.x1s = [torch.empty(b, m, **f32) for _ in range(L)]
        self.full = None
        self.dx = [torch.empty(b, m, **f32) for _ in range(2)]
        self.dx_c = [torch.empty(b, m, dtype=self.dtype, device=self.device) for _ in range(2)] \
            if precision != "fp32" else [None, None]
        # bf16: the lean blocks' low-rank FFN Wgrads are deferred and run for
        # all lean layers at once (grouped launches, mecefo_lowrank_wgrads_batched);
        # each lean layer keeps its output gradient (bf16) and FFN intermediates.
        self.defer_wgrads = precision == "bf16"
        # ... in groups of `defer_layers` consecutive layers (None: all), so
        # the deferred buffers (h2, act, [d_gate|d_up], dy) exist for at most
        # that many layers at once (2 b (2m + 3f) bytes per layer)
        self.defer_layers = L if defer_layers is None else max(1, min(int(defer_layers), L))
        self._dyc = {}
        self._saved = {}
        # Eq. (1) exchange (cluster.py:292-322): the pre-weighted flat gradient
        # is all-reduced in buckets, in backward order (head, layer groups of
        # `defer_layers` from the top, embedding), each on a communication
        # stream as soon as its gradients are final — overlapped with the rest
        # of the backward. grad_comm "bf16" casts each bucket to bf16 for the
        # wire (and back to fp32 for the optimizer); "fp32" reduces in place.
        if grad_comm not in ("fp32", "bf16"):
            raise ContractViolation(f"grad_comm must be fp32 or bf16, got {grad_comm!r}")
        self.grad_comm = grad_comm
        self.overlap_comm = overlap_comm
        self._comm = torch.cuda.Stream(device=self.device) if group is not None else None
        self._gbf16 = None
        self._ws_lr = None
        self.xf = torch.empty(b, m, dtype=self.dtype, device=self.device)
        self.inv_f = torch.empty(b, **f32)
        self.logits = torch.empty(b, cfg.vocab, dtype=self.dtype, device=self.device)
        self.tok = torch.empty(b, dtype=torch.int64, device=self.device)
        self.tgt = torch.empty(b, dtype=torch.int64, device=self.device)
        self._loss_tmp = torch.zeros(self.max_group, dtype=torch.float32, device=self.device)
        self.rp = approx._pad16(r)
        nbytes = int(_lib.load().mecefo_workspace_bytes(self.eng.handle, b, self.rp))
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.projs: dict = {}
        self._keep = []
        self.losses = None
        self.graphs = []
        # device status word (bad token / bad target / non-finite gradient):
        # kernels set bits, a copy lands in pinned host memory after every
        # optimizer launch, the host checks it at the next iteration boundary
        sp = ctypes.c_void_p()
        _lib.call("mecefo_status_device", self.eng.handle, ctypes.byref(sp))
        self._status_dev = sp.value
        _lib.call("mecefo_status_reset", self.eng.handle, runtime.stream_ptr())
        self._status_host = torch.zeros(4, dtype=torch.int32).pin_memory()

    # ------------------------------------------------------------------ utils
    def _gp(self, name: str) -> int:
        return self.grad.data_ptr() + 4 * self.weights.offsets[name]

    def _layer_grads(self, l: int, alpha_mha, alpha_ffn: float) -> _lib.LayerGrads:
        p = f"layers.{l}."
        if alpha_mha is None:
            return _lib.LayerGrads(None, None, None, 0.0, self._gp(p + "gate"), self._gp(p + "down"),
                                   self._gp(p + "norm_ffn"), alpha_ffn)
        return _lib.LayerGrads(self._gp(p + "q"), self._gp(p + "o"), self._gp(p + "norm_mha"), alpha_mha,
                               self._gp(p + "gate"), self._gp(p + "down"), self._gp(p + "norm_ffn"), alpha_ffn)

    def _memset0(self, t: torch.Tensor) -> None:
        _lib.call("mecefo_memset_zero", t.data_ptr(), t.numel() * t.element_size(), runtime.stream_ptr())

    def _status_copy(self, stream_ptr: int) -> None:
        _lib.call("mecefo_status_snapshot", self.eng.handle, self._status_host.data_ptr(), stream_ptr)

    def check_status(self, sync: bool = False) -> None:
        """Raise what the reference raises for the iteration whose status word
        reached the host: non-finite gradient -> NumericalFailure
        (optim.py:55-57); token / target outside the vocabulary ->
        ContractViolation (model.py:463, 505 raise IndexError there). Without
        `sync` this reads the latest snapshot (one or two iterations behind);
        with it, the current one."""
        if sync:
            torch.cuda.synchronize()
        w = int(self._status_host[0])
        if not w:
            return
        _lib.call("mecefo_status_reset", self.eng.handle, runtime.stream_ptr())
        torch.cuda.synchronize()
        self._status_host.zero_()
        if w & _lib.STATUS_NONFINITE_GRAD:
            raise NumericalFailure("non-finite gradient")
        what = "token" if w & _lib.STATUS_BAD_TOKEN else "target"
        raise ContractViolation(f"{what} id outside [0, {self.cfg.vocab})")

    @staticmethod
    def _check_host_ids(t: torch.Tensor, vocab: int, what: str) -> None:
        if not t.is_cuda and t.numel():
            lo, hi = int(t.min()), int(t.max())
            if lo < 0 or hi >= vocab:
                raise ContractViolation(f"{what} id outside [0, {vocab}): range [{lo}, {hi}]")

    def _dy_buffer(self, k: int) -> torch.Tensor:
        """Compute-precision gradient of layer k's input (k = L: the head's
        output). defer_layers + 1 rotating buffers: a deferred Wgrad job of
        layer l reads dy(l + 1) until its group is flushed."""
        slot = k % (self.defer_layers + 1)
        if slot not in self._dyc:
            self._dyc[slot] = torch.empty(self.b * self.max_group, self.cfg.hidden, dtype=self.dtype,
                                          device=self.device)
        return self._dyc[slot]

    def _saved_buffers(self, l: int):
        slot = l % self.defer_layers
        if slot not in self._saved:
            b, m, f = self.b * self.max_group, self.cfg.hidden, mdl.ffn_storage(self.cfg)
            mk = lambda n: torch.empty(b, n, dtype=self.dtype, device=self.device)
            self._saved[slot] = (mk(m), mk(f), mk(2 * f))
        return self._saved[slot]

    def _layers_range(self, lo: int, hi: int) -> tuple:
        """Flat-buffer element range holding every parameter of layers lo..hi."""
        first = self.weights.offsets[f"layers.{lo}.q"]
        name = f"layers.{hi}.norm_ffn"
        return first, self.weights.offsets[name] + int(np.prod(self.weights.shapes[name]))

    def _exchange(self, start: int, end: int) -> None:
        """All-reduce(sum) of flat gradient elements [start, end) on the
        communication stream, ordered after everything enqueued so far on the
        compute stream (graph-capturable fork)."""
        if self.group is None or end <= start:
            return
        import torch.distributed as dist

        main = torch.cuda.current_stream()
        if not self.overlap_comm:
            dist.all_reduce(self.grad[start:end], op=dist.ReduceOp.SUM, group=self.group)
            return
        self._comm.wait_stream(main)
        with torch.cuda.stream(self._comm):
            g = self.grad[start:end]
            if self.grad_comm == "bf16":
                if self._gbf16 is None:
                    self._gbf16 = torch.empty(self.weights.total, dtype=torch.bfloat16, device=self.device)
                cs = self._comm.cuda_stream
                bb = self._gbf16[start:end]
                _lib.call("mecefo_cast_bf16", g.data_ptr(), bb.data_ptr(), end - start, cs)
                dist.all_reduce(bb, op=dist.ReduceOp.SUM, group=self.group)
                _lib.call("mecefo_widen_bf16", bb.data_ptr(), g.data_ptr(), end - start, cs)
            else:
                dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group)

    def _flush_lowrank(self, jobs: list, b: int, s: int) -> None:
        """The deferred low-rank FFN Wgrads of a group of lean layers, as
        grouped launches (mecefo_lowrank_wgrads_batched)."""
        if not jobs:
            return
        arr = (_lib.LowrankJob * len(jobs))(*jobs)
        wsl, wnl = self._lowrank_ws(b, len(jobs))
        _lib.call("mecefo_lowrank_wgrads_batched", self.eng.handle, arr, len(jobs), b, wsl, wnl, s)
        jobs.clear()

    def _h1_scratch(self, k: int, b: int):
        """Compute-precision h1 (b x m) and fp32 inv1 (b) of a lean block in a
        chain (two alternating pairs: a block reads one and writes the next
        block's into the other)."""
        if not hasattr(self, "_h1s"):
            self._h1s = {}
        key = (k, b)
        if key not in self._h1s:
            self._h1s[key] = (torch.empty(b, self.cfg.hidden, dtype=self.dtype, device=self.device),
                              torch.empty(b, dtype=torch.float32, device=self.device))
        return self._h1s[key]

    def _lowrank_ws(self, b: int, count: int):
        n = int(_lib.load().mecefo_lowrank_batched_workspace_bytes(self.eng.handle, b, self.rp, count))
        if self._ws_lr is None or self._ws_lr.numel() < n:
            self._ws_lr = torch.empty(n, dtype=torch.uint8, device=self.device)
        return self._ws_lr.data_ptr(), self._ws_lr.numel()

    def _full_cache(self, l: int) -> dict:
        if self.full is None:
            self.full = [None] * self.cfg.layers
        if self.full[l] is None:
            self.full[l] = mdl._alloc_full_cache(self.cfg, self.b, self.dtype, self.device)  # never fused
        return self.full[l]

    def proj(self, rank: int, layer: int) -> approx.ProjectionCache:
        key = (rank, layer)
        if key not in self.projs:
            self.projs[key] = approx.ProjectionCache(rank=self.r, refresh_period=self.tau)
        return self.projs[key]

    def reset_projection(self, rank: int, layer: int) -> None:
        """harness.py:384-388: adopted layers start a fresh basis."""
        if (rank, layer) in self.projs:
            self.projs[(rank, layer)].reset()

    # ---------------------------------------------------------- microbatch
    def _fusable(self, mbs: list) -> bool:
        """Several lean microbatches can share one pass iff every layer is lean
        for all of them, their Eq. (1) weights agree and, per layer, their
        projection bases are (or will be, after a common refresh) identical."""
        if not self.fuse_lean or len(mbs) < 2 or len(mbs) > self.max_group:
            return False
        m0 = mbs[0]
        for mb in mbs:
            if not all(mb.lean) or any(a is not None for a in mb.alpha_mha):
                return False
            if mb.alpha_ffn != m0.alpha_ffn or mb.alpha_global != m0.alpha_global:
                return False
        for l in range(self.cfg.layers):
            pcs = [self.proj(mb.rank, l) for mb in mbs]
            due = [(not pc.basis) or pc.step % pc.refresh_period == 0 for pc in pcs]
            if any(d != due[0] for d in due):
                return False
            if not due[0] and (pcs[0].token is None or any(pc.token != pcs[0].token for pc in pcs)):
                return False
        return True

    def _projection(self, mbs: list, l: int):
        """Refresh (if due) the basis of every rank in the group — computed once
        and shared — and return the packed operands of the group's basis."""
        pcs = [self.proj(mb.rank, l) for mb in mbs]
        lead = pcs[0]
        before = lead.refreshes
        approx.refresh_projections(lead, self.weights.layers[l], self.svd, budgeted=self.svd_budgeted)
        if lead.refreshes != before:
            lead.token = ("svd", self.iter, l, self.r, self.svd)
            for pc in pcs[1:]:  # same weights, same SvdConfig -> same basis
                for k, v in lead.basis.items():
                    pc.set_basis(k, v)
                pc.token = lead.token
                pc.refreshes += 1
                pc.svd_calls += len(lead.basis)
        return lead.packed(self.precision, down_rows=mdl.ffn_storage(self.cfg))

    def microbatch(self, mb: Microbatch, loss_ptr: int, comm: bool = False) -> None:
        self._run([mb], loss_ptr, comm)

    def _run(self, mbs: list, loss_ptr: int, comm: bool = False) -> None:
        """Forward + backward of len(mbs) microbatches stacked into one pass;
        loss_ptr receives len(mbs) consecutive per-microbatch mean losses.
        comm: this is the GPU's last pass of the iteration, so each gradient
        bucket is final once this pass has produced it: exchange it."""
        cfg, eng, s = self.cfg, self.eng, runtime.stream_ptr()
        n, b1 = len(mbs), self.b
        b = n * b1
        mb = mbs[0]
        w = self.weights
        ws, wn = self.ws.data_ptr(), self.ws.numel()
        for i, m_ in enumerate(mbs):
            self._check_host_ids(m_.tokens, cfg.vocab, "token")
            self._check_host_ids(m_.targets, cfg.vocab, "target")
            self.tok[i * b1:(i + 1) * b1].copy_(m_.tokens.reshape(-1), non_blocking=True)
            self.tgt[i * b1:(i + 1) * b1].copy_(m_.targets.reshape(-1), non_blocking=True)
        _lib.call("mecefo_embedding_forward", eng.handle, self.tok.data_ptr(),
                  w.master.data_ptr() + 4 * w.offsets["embedding"], self.xs[0].data_ptr(), b, s)
        caches = []
        # the blocks run as a chain: block l's residual down-projection also
        # writes block l+1's normalised input h1 / inv1 (fused into one kernel
        # at hidden 512) — into block l+1's full cache, or into a scratch pair
        # for a lean block (the lean cache stays {x, x1})
        structs = []
        for l in range(cfg.layers):
            full = None if mb.lean[l] else self._full_cache(l)
            cache = mdl.BlockCache(mode=mdl.CACHE_FFN_INPUT_ONLY if mb.lean[l] else mdl.CACHE_FULL,
                                   x=self.xs[l], x1=self.x1s[l], full=full)
            cs = cache.struct()
            if mb.lean[l] and l > 0:  # lean h1 scratch (alternating: block l reads one, writes the other)
                h1s, inv1s = self._h1_scratch(l % 2, b)
                cs.h1, cs.inv1 = h1s.data_ptr(), inv1s.data_ptr()
            structs.append(cs)
            caches.append(cs)
        for l in range(cfg.layers):
            cs = structs[l]
            nxt = structs[l + 1] if l + 1 < cfg.layers else None
            _lib.call("mecefo_forward_block_chained", eng.handle, ctypes.byref(self.lws[l]), ctypes.byref(cs),
                      self.xs[l + 1].data_ptr(), b, _lib.CACHE_FFN_INPUT_ONLY if mb.lean[l] else _lib.CACHE_FULL,
                      _lib.FWD_H1_READY if l > 0 else 0,
                      w.get(f"layers.{l + 1}.norm_mha").data_ptr() if nxt is not None else None,
                      nxt.h1 if nxt is not None else None, nxt.inv1 if nxt is not None else None, ws, wn, s)
        _lib.call("mecefo_head_forward_loss_grouped", eng.handle, self.xs[cfg.layers].data_ptr(),
                  w.get("final_norm").data_ptr(), w.shadow_view("unembedding").data_ptr(), self.tgt.data_ptr(), b, b1,
                  self.xf.data_ptr(), self.inv_f.data_ptr(), self.logits.data_ptr(), loss_ptr, ws, wn, s)
        cur = 0
        defer = self.defer_wgrads and any(mb.lean)
        dxc = (lambda k: self._dy_buffer(k)) if defer else None  # gradient of layer k's input (k = L: head)
        _lib.call("mecefo_head_backward", eng.handle, self.xs[cfg.layers].data_ptr(), w.get("final_norm").data_ptr(),
                  self.inv_f.data_ptr(), self.xf.data_ptr(), self.logits.data_ptr(),
                  w.shadow_view("unembedding").data_ptr(), self.dx[cur].data_ptr(),
                  runtime.ptr(dxc(cfg.layers) if defer else self.dx_c[cur]),
                  self._gp("final_norm"), self._gp("unembedding"), mb.alpha_global, b, ws, wn, s)
        if comm:  # head bucket: final_norm + unembedding (the flat buffer's tail)
            self._exchange(self.weights.offsets["final_norm"], self.weights.total)
        jobs, keeps = [], []
        since_flush = 0
        pending_hi = cfg.layers - 1
        for l in reversed(range(cfg.layers)):
            nxt = 1 - cur
            dyc_in = dxc(l + 1) if defer else self.dx_c[cur]
            dxc_out = dxc(l) if defer else self.dx_c[nxt]
            g = self._layer_grads(l, mb.alpha_mha[l], mb.alpha_ffn)
            if mb.lean[l]:
                pst, keep, rp = self._projection(mbs, l)
                keeps.append((pst, keep))
                if defer:
                    h2, act, dcat = self._saved_buffers(l)
                    saved = _lib.FfnSaved(h2.data_ptr(), act.data_ptr(), dcat.data_ptr())
                    _lib.call("mecefo_backward_block_neighbor_main", eng.handle, ctypes.byref(self.lws[l]),
                              ctypes.byref(caches[l]), self.dx[cur].data_ptr(), runtime.ptr(dyc_in),
                              self.dx[nxt].data_ptr(), runtime.ptr(dxc_out), ctypes.byref(g), ctypes.byref(saved), b,
                              ws, wn, s)
                    jobs.append(_lib.LowrankJob(dyc_in.data_ptr(), saved, ctypes.pointer(pst),
                                                self._gp(f"layers.{l}.gate"), self._gp(f"layers.{l}.down"),
                                                mb.alpha_ffn))
                else:
                    _lib.call("mecefo_backward_block_neighbor", eng.handle, ctypes.byref(self.lws[l]),
                              ctypes.byref(caches[l]), self.dx[cur].data_ptr(), runtime.ptr(dyc_in),
                              self.dx[nxt].data_ptr(), runtime.ptr(dxc_out), ctypes.byref(g), ctypes.byref(pst), b,
                              ws, wn, s)
                for m_ in mbs:
                    self.proj(m_.rank, l).step += 1
            else:
                _lib.call("mecefo_backward_block_exact", eng.handle, ctypes.byref(self.lws[l]),
                          ctypes.byref(caches[l]), self.dx[cur].data_ptr(), runtime.ptr(dyc_in),
                          self.dx[nxt].data_ptr(), runtime.ptr(dxc_out), ctypes.byref(g), b, ws, wn, s)
            cur = nxt
            since_flush += 1
            if since_flush == self.defer_layers:  # rotating buffers are about to be reused
                if defer:
                    self._flush_lowrank(jobs, b, s)
                if comm:  # layers l .. pending_hi are final
                    self._exchange(*self._layers_range(l, pending_hi))
                    pending_hi = l - 1
                since_flush = 0
        if defer:
            self._flush_lowrank(jobs, b, s)
        if comm and pending_hi >= 0:
            self._exchange(*self._layers_range(0, pending_hi))
        self._keep = keeps
        _lib.call("mecefo_embedding_backward", eng.handle, self.tok.data_ptr(), self.dx[cur].data_ptr(),
                  self._gp("embedding"), mb.alpha_global, b, s)
        if comm:
            e0 = self.weights.offsets["embedding"]
            self._exchange(e0, e0 + int(np.prod(self.weights.shapes["embedding"])))

    # ------------------------------------------------------------ optimizer
    def _seg_slot(self, slot: int, nseg: int):
        """Pinned host + device segment tables (two slots: one step of host
        look-ahead without racing the copy of the previous step)."""
        if not hasattr(self, "_segs"):
            n = len(self.weights.layout)
            nbytes = n * ctypes.sizeof(_lib.AdamSegment)
            self._segs = [(torch.empty(nbytes, dtype=torch.uint8).pin_memory(),
                           torch.empty(nbytes, dtype=torch.uint8, device=self.device),
                           torch.cuda.Event()) for _ in range(2)]
            self._seg_k = 0
        return self._segs[slot]

    def _adam_launch(self, lr: float, skip, slot: int, stream_ptr: int, fill: bool = True,
                     record: bool = True) -> None:
        host, dev, ev = self._seg_slot(slot, 0)
        if fill:
            ev.synchronize()  # the copy that last read this slot has executed
            arr, total_numel, names = op.adam_segments(self.weights, self.opt, lr, skip)
            host.numpy()[: arr.nbytes] = arr.view(np.uint8)
            for name in names:
                self.opt.step[name] = self.opt.step.get(name, 0) + 1
            self._adam_meta = (len(names), total_numel)
        nseg, total_numel = self._adam_meta
        dev.copy_(host, non_blocking=True)
        if record:
            ev.record()
        if nseg:
            cfg = self.opt.cfg
            shadow = self.weights.shadow.data_ptr() if self.precision != "fp32" else None
            _lib.call("mecefo_adamw_step", self.eng.handle, dev.data_ptr(), nseg, total_numel,
                      self.weights.master.data_ptr(), self.grad.data_ptr(), self.opt.m.data_ptr(),
                      self.opt.v.data_ptr(), shadow, cfg.beta1, cfg.beta2, cfg.eps, stream_ptr)
        self._status_copy(stream_ptr)

    # ---------------------------------------------------------------- step
    def _prerefresh(self, mbs: list) -> None:
        """Batched projection refresh: every lean (rank, layer) whose refresh
        is due this iteration (approx.py:74-75) is refreshed at once; ranks
        sharing a basis provenance share the result."""
        if not self.batched_refresh:
            return
        due = {}
        for mb in mbs:
            for l in range(self.cfg.layers):
                if not mb.lean[l]:
                    continue
                pc = self.proj(mb.rank, l)
                if pc.basis and pc.step % pc.refresh_period != 0:
                    continue
                if pc.basis and getattr(pc, "_fresh_step", None) == pc.step:
                    continue
                due.setdefault(l, []).append(pc)
        if not due:
            return
        mats, ranks, owners = [], [], []
        for l, pcs in due.items():
            for kind in approx.FFN_KINDS:
                w = self.weights.layers[l].kind(kind)
                mats.append(w)
                ranks.append(min(self.r, w.shape[1]))
                owners.append((l, kind))
        import time

        t0 = time.perf_counter()
        bases = self._solve_bases(mats, ranks)
        torch.cuda.current_stream().synchronize()  # the solve reads its convergence flags on the host anyway
        self.last_refresh_s = time.perf_counter() - t0
        for (l, kind), v1 in zip(owners, bases):
            for pc in due[l]:
                pc.set_basis(kind, v1)
        for l, pcs in due.items():
            tok = ("svd", self.iter, l, self.r, self.svd)
            for pc in pcs:
                pc.token = tok
                pc.refreshes += 1
                pc.svd_calls += len(approx.FFN_KINDS)
                pc._fresh_step = pc.step

    def _solve_bases(self, mats: list, ranks: list) -> list:
        from .linalg import refresh_bases, top_r_right_singular_vectors_batched

        if self.svd_budgeted:
            return top_r_right_singular_vectors_batched(mats, ranks, self.svd.max_iterations, self.svd.seed)
        info = []
        out = refresh_bases(mats, ranks, self.svd, info=info)
        self.refresh_info = info
        return out

    def _body(self, mbs: list, losses: torch.Tensor) -> None:
        self._prerefresh(mbs)
        self._memset0(self.grad)
        self._memset0(losses)
        comm = self.group is not None
        if self._fusable(mbs):
            ranks = [mb.rank for mb in mbs]
            if ranks == list(range(ranks[0], ranks[0] + len(ranks))):
                self._run(mbs, losses.data_ptr() + 4 * ranks[0], comm)  # per-rank losses land in place
            else:
                self._run(mbs, self._loss_tmp.data_ptr(), comm)
                for i, j in enumerate(ranks):  # device-to-device, graph-capturable
                    losses[j:j + 1].copy_(self._loss_tmp[i:i + 1])
        else:
            for k, mb in enumerate(mbs):
                self.microbatch(mb, losses.data_ptr() + 4 * mb.rank, comm and k == len(mbs) - 1)
        if comm and not mbs:  # a GPU with no microbatch (its rank failed) still joins every bucket
            self._exchange(self.weights.offsets["final_norm"], self.weights.total)
            for hi in range(self.cfg.layers - 1, -1, -self.defer_layers):
                self._exchange(*self._layers_range(max(0, hi - self.defer_layers + 1), hi))
            e0 = self.weights.offsets["embedding"]
            self._exchange(e0, e0 + int(np.prod(self.weights.shapes["embedding"])))
        self.iter += 1
        if comm:
            import torch.distributed as dist

            if self.overlap_comm:
                torch.cuda.current_stream().wait_stream(self._comm)  # join before the optimizer
            dist.all_reduce(losses, op=dist.ReduceOp.SUM, group=self.group)

    def step(self, mbs: list, n_ranks: int, lr: float, skip=(), check: bool = True) -> torch.Tensor:
        """Run this GPU's microbatches, exchange, update (eager launches).
        Returns the (n_ranks,) device vector of per-rank losses."""
        self.check_status()
        if self.losses is None or self.losses.numel() != n_ranks:
            self.losses = torch.zeros(n_ranks, dtype=torch.float32, device=self.device)
        self._body(mbs, self.losses)
        if check:
            op.apply_flat(self.weights, self.opt, self.grad, lr, skip=skip, check=True)
            self._status_copy(runtime.stream_ptr())
            self.check_status(sync=True)
        else:
            self.opt.ensure_flat(self.weights.total, self.device)
            slot = self._seg_k = (getattr(self, "_seg_k", 0) + 1) % 2
            self._adam_launch(lr, skip, slot, runtime.stream_ptr())
        return self.losses

    def plan_key(self, mbs: list, skip=()) -> tuple:
        """Identity of an iteration's plan: everything a captured graph bakes
        in — microbatch ranks, per-layer modes and Eq. (1) weights, input
        buffers, the skip list, whether the lean microbatches run fused, and
        the addresses of the projection operands (stable across in-place
        refreshes, new after an adoption reset)."""
        ops = []
        for mb in mbs:
            for l in range(self.cfg.layers):
                if mb.lean[l] and (mb.rank, l) in self.projs:
                    pk = self.projs[(mb.rank, l)]._packed
                    ops.append(tuple(sorted((k, v[1][2].data_ptr()) for k, v in pk.items())))
        return (tuple((mb.rank, tuple(mb.lean), tuple(mb.alpha_mha), mb.alpha_ffn, mb.alpha_global,
                       mb.tokens.data_ptr(), mb.targets.data_ptr()) for mb in mbs), tuple(sorted(skip)),
                self._fusable(mbs), tuple(ops))

    def has_graph(self, mbs: list, skip=()) -> bool:
        return self.plan_key(mbs, skip) in getattr(self, "_graph_cache", {})

    def capture(self, mbs: list, n_ranks: int, skip=()) -> None:
        """Capture one whole iteration of this plan (both microbatches'
        forward/backward, the Eq. (1) all-reduce and the fused AdamW) as CUDA
        graphs, one per optimizer-segment slot, into a plan-keyed cache (a
        rotating failure plan reuses its graphs when the plan recurs). Call
        after an eager step with the same plan (projections refreshed,
        descriptors and kernel attributes warm)."""
        if self.losses is None or self.losses.numel() != n_ranks:
            self.losses = torch.zeros(n_ranks, dtype=torch.float32, device=self.device)
        if not hasattr(self, "_graph_cache"):
            self._graph_cache = {}
            self._graph_pool = torch.cuda.graph_pool_handle()
        self._seg_slot(0, 0)
        arr, total_numel, names = op.adam_segments(self.weights, self.opt, 1e-4, skip)
        meta = (len(names), total_numel)
        self._adam_meta = meta
        torch.cuda.synchronize()
        steps = {k: pc.step for k, pc in self.projs.items()}
        graphs = []
        for slot in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self._graph_pool):
                self._body(mbs, self.losses)
                self._adam_launch(0.0, skip, slot, runtime.stream_ptr(), fill=False, record=False)
            graphs.append(g)
        for k, v in steps.items():  # capture ran the host bookkeeping once; undo it
            self.projs[k].step = v
        self.iter -= 2
        key = self.plan_key(mbs, skip)
        self._graph_cache[key] = (graphs, (list(mbs), n_ranks, tuple(skip)), meta)
        self._graph_key = key
        self.graphs = graphs
        self._graph_plan = (list(mbs), n_ranks, tuple(skip))
        torch.cuda.synchronize()

    def drop_graphs(self) -> None:
        self._graph_cache = {}
        self.graphs = []

    def replay(self, lr: float, mbs: list | None = None, skip=()) -> torch.Tensor:
        """One captured iteration: host bookkeeping (optimizer scalars,
        projection step counters) then a single graph launch. mbs=None
        replays the most recently captured plan."""
        self.check_status()
        key = self._graph_key if mbs is None else self.plan_key(mbs, skip)
        graphs, (mbs_c, n_ranks, skip_c), meta = self._graph_cache[key]
        self._adam_meta = meta
        slot = self._seg_k = (getattr(self, "_seg_k", 0) + 1) % 2
        host, dev, ev = self._segs[slot]
        ev.synchronize()
        arr, _, names = op.adam_segments(self.weights, self.opt, lr, skip_c)
        host.numpy()[: arr.nbytes] = arr.view(np.uint8)
        for name in names:
            self.opt.step[name] = self.opt.step.get(name, 0) + 1
        for mb in mbs_c:
            for l in range(self.cfg.layers):
                if mb.lean[l]:
                    self.proj(mb.rank, l).step += 1
        self.iter += 1
        graphs[slot].replay()
        ev.record()
        return self.losses

    def steps_until_refresh(self, mbs: list) -> int:
        """Iterations until the first lean layer's projection refresh is due
        (0 = due now; approx.py:74-75)."""
        best = 10**9
        for mb in mbs:
            for l in range(self.cfg.layers):
                if mb.lean[l]:
                    pc = self.proj(mb.rank, l)
                    best = min(best, 0 if not pc.basis else (-pc.step) % pc.refresh_period)
        return best

    def refresh_cost(self, mbs: list) -> float:
        """Seconds for one refresh of every lean layer's bases of these
        microbatches (the tau-amortised work), measured on a scratch copy of
        the caches so the run's own schedule is untouched."""
        import time

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        seen = set()
        mats, ranks = [], []
        for mb in mbs:
            for l in range(self.cfg.layers):
                if mb.lean[l] and (self.proj(mb.rank, l).token, l) not in seen:
                    seen.add((self.proj(mb.rank, l).token, l))
                    if self.batched_refresh:
                        for kind in approx.FFN_KINDS:
                            w = self.weights.layers[l].kind(kind)
                            mats.append(w)
                            ranks.append(min(self.r, w.shape[1]))
                    else:
                        pc = approx.ProjectionCache(rank=self.r, refresh_period=self.tau)
                        approx.refresh_projections(pc, self.weights.layers[l], self.svd, budgeted=self.svd_budgeted)
        if mats:
            self._solve_bases(mats, ranks)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    def projections_due(self, mbs: list) -> bool:
        """True if any lean layer's projection refresh is due next iteration
        (approx.py:74-75); graph replay must then fall back to an eager step."""
        for mb in mbs:
            for l in range(self.cfg.layers):
                if mb.lean[l]:
                    pc = self.proj(mb.rank, l)
                    if not pc.basis or pc.step % pc.refresh_period == 0:
                        return True
        return False


def ring_plan(n_ranks: int, failed, layers: int, gpu_of_rank=None):
    """Flavour-B plan: R logical DP ranks on a ring; a failed
    rank's microbatch goes to its ring successor (cluster.ring_route), which
    then runs BOTH microbatches lean on all layers (harness.py:395 predicate
    at microbatch granularity). Returns (executor, lean_by_rank, alpha_mha,
    skip) where alpha_mha[l] is 1/|N_MHA| (N_MHA = ranks run exactly) and
    skip lists the MHA parameters whose active set is empty."""
    from . import cluster as cl
    from .errors import UnrecoverableRankError

    route = cl.ring_route(n_ranks, failed)
    if route is None:
        raise UnrecoverableRankError(f"ring of {n_ranks}: failed ranks {sorted(failed)} leave no adopter")
    doubled = {route[j] for j in failed}
    lean = [route[j] in doubled for j in range(n_ranks)]
    exact = [j for j in range(n_ranks) if not lean[j]]
    alpha_mha = (1.0 / len(exact)) if exact else None
    skip = []
    if not exact:
        skip = [f"layers.{l}.{k}" for l in range(layers) for k in ("q", "k", "v", "o", "norm_mha")]
    return route, lean, alpha_mha, skip
