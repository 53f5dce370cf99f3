"""All-reduce timing for the flat gradient buffer (LLaMA-60M: 58.1M fp32) across the local GPUs."""
import os, time, torch, torch.distributed as dist
dist.init_process_group("nccl")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", r)))
n = 58_100_000
for dt in (torch.float32, torch.bfloat16):
    x = torch.ones(n, dtype=dt, device="cuda")
    for _ in range(3):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        dist.all_reduce(x)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    if r == 0:
        nbytes = n * x.element_size()
        print(f"world {w} {dt} all_reduce {nbytes/1e6:.0f} MB: {ms:.3f} ms  busbw {2*(w-1)/w*nbytes/ms/1e6:.0f} GB/s", flush=True)
    # graph-captured
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        dist.all_reduce(x)
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    s.record()
    for _ in range(10):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    if r == 0:
        print(f"   graph replay: {s.elapsed_time(e)/10:.3f} ms", flush=True)
dist.barrier()
os._exit(0)
