"""End-to-end (host-buffer) step rate under different preceding activity (diagnostics)."""
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
xs = [torch.from_numpy(datagen.features(B, batch_idx=k)).cuda() for k in range(8)]
ls = [torch.from_numpy(datagen.labels(B, batch_idx=k)).cuda() for k in range(8)]
loss = torch.zeros(4).pin_memory()
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(tag, n=200, warm=20):
    for i in range(warm):
        s.step_host(xh[i % 2], lh[i % 2], loss)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for i in range(n):
        s.step_host(xh[i % 2], lh[i % 2], loss)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{tag}: event {1e3*ms/n:.1f} us/step ({B*n/(ms/1e3):.0f}/s), host enqueue {1e6*(t1-t0)/n:.1f} us/call")


run("first")
run("second")
for i in range(300):  # the bench's device loop: pool of 8 batches (16 graphs), flush between steps
    flush.zero_()
    s.step(xs[i % 8], ls[i % 8])
torch.cuda.synchronize()
run("after device loop")
s.timing_begin(20)
for i in range(20):
    flush.zero_()
    s.step(xs[i % 8], ls[i % 8])
torch.cuda.synchronize()
s.timing_end()
run("after timing pass")
run("again")
