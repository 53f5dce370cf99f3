"""Time the fused softmax-CE kernel on the bench head shape (16384 x 32000 bf16)."""
import os, sys, torch
from paper_2510_16415_b200 import _lib, model as mdl, runtime
b, V = 16384, 32000
cfg = mdl.ModelConfig(vocab=V, hidden=8, heads=1, ffn_intermediate=8, layers=1, seq_len=1)
eng = runtime.engine_for(cfg, "bf16")
g = torch.Generator(device="cuda").manual_seed(0)
base = (torch.randn(b, V, device="cuda", generator=g) * 3).to(torch.bfloat16)
t = torch.randint(0, V, (b,), device="cuda", generator=g)
d = base.clone()
loss = torch.empty(1, device="cuda")
ws, wn = eng.workspace(b)
def run():
    _lib.call("mecefo_cross_entropy", eng.handle, d.data_ptr(), t.data_ptr(), b, loss.data_ptr(), ws, wn,
              runtime.stream_ptr())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
times = []
for i in range(12):
    d.copy_(base); flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); run(); e.record(); torch.cuda.synchronize()
    times.append(s.elapsed_time(e))
ms = sorted(times[2:])[len(times[2:]) // 2]
print(f"{os.environ.get('MECEFO_CE_WARP') and 'warp' or 'row'} ce ms {ms:.3f}  GB/s(2 passes) {2*b*V*2/ms/1e6:.0f}  loss {loss.item():.5f}")
