#!/usr/bin/env python
"""Per-task timeline of the persistent backward (bwd_kernel; diagnostics build, needs a GPU).

    TEM_NO_GRAPH=1 python scripts/probes/bwd_timeline.py [--workload c2]

Stamps per CTA: task k's MMA start (8 + k) and epilogue end (k).  Prints per task type the
start / end distribution and the CTAs' last end (the kernel's makespan), us after the first
MMA start."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--warm", type=int, default=3)
    args = ap.parse_args()
    os.environ["TEM_DIAG_LIB"] = "1"
    import numpy as np
    import torch
    import datagen
    from paper_1906_06496_b200 import tem
    B = {"c1": 4, "c2": 16}[args.workload]
    sc = tem.SessionConfig(world_size=1, rank=0, local_ranks=1, batch_per_rank=B, precision=0, lr=0.01)
    s = tem.TemSession(sc, datagen.init_params())
    x = torch.from_numpy(datagen.features(B)).cuda()
    lab = torch.from_numpy(datagen.labels(B)).cuda()
    lib = tem.lib()
    nb = ctypes.c_int64(0)
    for _ in range(args.warm):
        s.step(x, lab)
    torch.cuda.synchronize()
    slot = lib.tem_timing_slots(tem._P(s.ctx)) - 1  # SLOT_BWD is the last slot
    lib.tem_debug_buffer(tem._P(s.ctx), 0, f"tstamp_slot:{slot}".encode(), ctypes.byref(nb))
    s.step(x, lab)
    torch.cuda.synchronize()
    ptr = lib.tem_debug_buffer(tem._P(s.ctx), 0, b"tstamp", ctypes.byref(nb))

    class _Arr:
        __cuda_array_interface__ = {"shape": (nb.value // 8,), "typestr": "<i8", "data": (ptr, False), "version": 3}
    raw = torch.as_tensor(_Arr(), device="cuda").cpu().numpy().reshape(1024, 16).astype(np.float64)
    ws = lib.tem_debug_buffer(tem._P(s.ctx), 0, b"bwd_tasks", ctypes.byref(nb))
    tasks = None
    if ws:
        class _T:
            __cuda_array_interface__ = {"shape": (nb.value // 4,), "typestr": "<i4", "data": (ws, False), "version": 3}
        tasks = torch.as_tensor(_T(), device="cuda").cpu().numpy().reshape(-1, 8)
    starts = raw[:, 8:16]
    t0 = starts[starts > 0].min()
    names = {0: "DG", 1: "W2", 2: "W1"}
    rows = {}
    last = []
    for c in range(raw.shape[0]):
        if raw[c, 8] <= 0:
            continue
        ends = [raw[c, k] for k in range(8) if raw[c, k] > 0]
        last.append((max(ends) - t0) / 1e3)
        for k in range(8):
            if raw[c, 8 + k] > 0 and raw[c, k] > 0:
                ty = names.get((int(tasks[c, k]) >> 24) & 0xFF, "?") if tasks is not None else "?"
                rows.setdefault((k, ty), []).append(((raw[c, 8 + k] - t0) / 1e3, (raw[c, k] - t0) / 1e3))
    print(f"{len(last)} CTAs; makespan (last epilogue end) median {np.median(last):.2f} max {max(last):.2f} us")
    q = np.quantile(last, [0.0, 0.1, 0.25, 0.5, 0.75, 0.9, 1.0])
    print("  CTA end quantiles (0/10/25/50/75/90/100 %): " + " ".join(f"{v:.2f}" for v in q))
    for (k, ty), v in sorted(rows.items()):
        a = np.array(v)
        print(f"  task {k} {ty:>2}: n={len(a):3d} start {np.median(a[:, 0]):6.2f}/{a[:, 0].max():6.2f}  "
              f"end {np.median(a[:, 1]):6.2f}/{a[:, 1].max():6.2f}  dur {np.median(a[:, 1] - a[:, 0]):5.2f}")
    s.close()


if __name__ == "__main__":
    main()
