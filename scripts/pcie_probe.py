"""PCIe probe: pinned H2D alone, D2H alone, and both concurrently (two streams), 1 GiB each, CUDA events."""
import json
import torch

n = 1 << 28  # 1 GiB of fp32
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3
def h2d():
    d_a.copy_(h_in, non_blocking=True)
def d2h():
    h_out.copy_(d_b, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
gb = n * 4 / 1e9
r = {"h2d_GBps": gb / timed(h2d), "d2h_GBps": gb / timed(d2h), "both_each_GBps": gb / timed(both)}
print(json.dumps(r))
