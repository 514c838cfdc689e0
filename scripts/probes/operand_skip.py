"""Mainloop sensitivity to operand traffic (diagnostics, wrong numerics): per-kernel event times
of c2 steps with the FWD/DGRAD A-window loads and/or B loads skipped (probe_skip bits)."""
import ctypes
import sys

import torch

sys.path.insert(0, "/root/repo")
import datagen  # noqa: E402
from paper_1906_06496_b200 import tem  # noqa: E402

B = 16
for bits in [int(a) for a in sys.argv[1:]] or (0, 1, 2, 3):
    s = tem.TemSession(tem.SessionConfig(batch_per_rank=B, lr=0.0), datagen.init_params())
    x = torch.from_numpy(datagen.features(B)).cuda()
    lab = torch.from_numpy(datagen.labels(B)).cuda()
    nb = ctypes.c_int64(0)
    tem.lib().tem_debug_buffer(tem._P(s.ctx), 0, f"probe_skip:{bits}".encode(), ctypes.byref(nb))
    for _ in range(3):
        s.step(x, lab)
    torch.cuda.synchronize()
    s.timing_begin(20)
    for _ in range(20):
        s.step(x, lab)
    torch.cuda.synchronize()
    ms, n = s.timing_end()
    keys = ("conv1_fwd", "conv2_fwd", "conv2_dgrad", "conv2_wgrad", "conv1_wgrad")
    print(f"skip={bits}: " + "  ".join(f"{k} {1e3 * ms[k] / n:5.1f}" for k in keys))
    tem.lib().tem_debug_buffer(tem._P(s.ctx), 0, b"probe_skip:0", ctypes.byref(nb))
    s.sync()
    s.close()
