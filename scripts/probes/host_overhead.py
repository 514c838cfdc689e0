"""Host-side cost of one tem_step_host call (CPU time per call, GPU kept busy) vs the GPU step."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import datagen
from paper_1906_06496_b200 import tem

B = 16
s = tem.TemSession(tem.SessionConfig(batch_per_rank=B, lr=0.01), datagen.init_params())
xh = [torch.from_numpy(datagen.features(B, batch_idx=k)).pin_memory() for k in range(2)]
lh = [torch.from_numpy(datagen.labels(B, batch_idx=k)).pin_memory() for k in range(2)]
loss = torch.zeros(4).pin_memory()
for i in range(10):
    s.step_host(xh[i % 2], lh[i % 2], loss)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for i in range(n):
    s.step_host(xh[i % 2], lh[i % 2], loss)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / n:.1f} us/call, wall {1e6 * (t2 - t0) / n:.1f} us/step "
      f"-> {B * n / (t2 - t0):.0f} samples/s (no flush)")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
t0 = time.perf_counter()
for i in range(n):
    flush.zero_()
    s.step_host(xh[i % 2], lh[i % 2], loss)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"with flush: host {1e6 * (t1 - t0) / n:.1f} us/iter, wall {1e6 * (t2 - t0) / n:.1f} us/iter")

# H2D bandwidth alone, and the device-buffer step alone
xd = torch.empty_like(xh[0], device="cuda")
cs = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(cs):
    e0.record(cs)
    for i in range(n):
        xd.copy_(xh[i % 2], non_blocking=True)
    e1.record(cs)
torch.cuda.synchronize()
print(f"H2D {xh[0].numel() * 4 / 1e6:.2f} MB: {1e3 * e0.elapsed_time(e1) / n:.1f} us/copy "
      f"({xh[0].numel() * 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s)")
xs = [torch.from_numpy(datagen.features(B, batch_idx=k)).cuda() for k in range(2)]
ls = [torch.from_numpy(datagen.labels(B, batch_idx=k)).cuda() for k in range(2)]
for i in range(10):
    s.step(xs[i % 2], ls[i % 2])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    s.step(xs[i % 2], ls[i % 2])
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"device-buffer steps back to back: {1e6 * (t2 - t0) / n:.1f} us/step")
