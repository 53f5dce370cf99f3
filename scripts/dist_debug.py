"""Staged multi-GPU diagnostic for the engine step (prints per-rank progress)."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"]); local = int(os.environ["LOCAL_RANK"])
t0 = time.time()


os.makedirs("gpurun_out", exist_ok=True)
_log = open(f"gpurun_out/dist_r{rank}.log", "w")


def say(msg):
    line = f"[r{rank} {time.time() - t0:6.1f}s] {msg}"
    print(line, flush=True)
    _log.write(line + "\n")
    _log.flush()


torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
say("pg up")
x = torch.ones(4, device="cuda")
dist.all_reduce(x)
say(f"allreduce ok {x[0].item()}")
from paper_2510_16415_b200 import engine as E, model as mdl
from paper_2510_16415_b200.linalg import SvdConfig

cfg = mdl.ModelConfig(vocab=64, hidden=128, heads=4, ffn_intermediate=344, layers=2, seq_len=64)
eng = E.StepEngine(cfg, precision="bf16", seqs_per_microbatch=2, r=32, tau=100,
                   svd=SvdConfig(rank=32, tolerance=1e-3, max_iterations=4, seed=23), svd_budgeted=True,
                   group=dist.group.WORLD)
say("engine up")
R = max(2, world)
route, lean, a_mha, skip = E.ring_plan(R, {1}, cfg.layers)
mbs = []
for j in range(R):
    if route[j] != rank:
        continue
    tk = torch.from_numpy(np.random.default_rng(j).integers(0, 64, size=(2, 64))).cuda()
    mbs.append(E.Microbatch(rank=j, tokens=tk, targets=tk, lean=[lean[j]] * 2,
                            alpha_mha=[None if lean[j] else a_mha] * 2, alpha_ffn=1 / R, alpha_global=1 / R))
say(f"plan: {len(mbs)} microbatches, route {route}")
for i in range(2):
    l = eng.step(mbs, R, 1e-3, skip=skip, check=False)
    torch.cuda.synchronize()
    say(f"eager step {i} losses {l.tolist()}")
eng.capture(mbs, R, skip)
say("captured")
for i in range(2):
    l = eng.replay(1e-3)
    torch.cuda.synchronize()
    say(f"replay {i} losses {l.tolist()}")
dist.barrier()
say("done")
eng.graphs = []
torch.cuda.synchronize()
dist.barrier()
say("exiting")
os._exit(0)
