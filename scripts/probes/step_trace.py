#!/usr/bin/env python
"""GPU-side kernel spans of one graph-replayed tem_step (diagnostics; needs a GPU).

    python scripts/probes/step_trace.py [--workload c2] [--reps 5]

Each traced kernel records min(CTA start) / max(CTA end) globaltimer (tem_debug_buffer
"trace_on"); prints per kernel the median start / end / duration over `reps` steps (us,
relative to the step's first kernel start) -- the critical path of the graph as executed.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--flush", action="store_true", help="write 256 MiB (L2 flush) before every traced step, as bench.py")
    args = ap.parse_args()
    os.environ["TEM_DIAG_LIB"] = "1"  # traces / phase stamps exist only in the diagnostics build
    import numpy as np
    import torch
    import datagen
    from paper_1906_06496_b200 import tem
    B, prec = {"c1": (4, 0), "c2": (16, 0), "c3": (256, 1), "c5": (16, 0)}[args.workload]
    P = datagen.PEM_P if args.workload == "c5" else 0
    sc = tem.SessionConfig(world_size=1, rank=0, local_ranks=1, batch_per_rank=B, precision=prec, lr=0.01,
                           pem_proposals=P)
    p0 = datagen.init_params() if not P else np.concatenate([datagen.init_params(), datagen.init_pem_params()])
    s = tem.TemSession(sc, p0)
    xs = datagen.features(B)
    x = torch.from_numpy(datagen.to_bf16_bits(xs).view(np.int16)).cuda() if prec == 1 else torch.from_numpy(xs).cuda()
    lab = torch.from_numpy(datagen.labels(B)).cuda()
    if P:
        fd = torch.from_numpy(datagen.bsp_features(B)).cuda()
        gd = torch.from_numpy(datagen.iou_targets(B)).cuda()
        step = lambda: s.step_pem(x, lab, fd, gd)  # noqa: E731
    else:
        step = lambda: s.step(x, lab)  # noqa: E731
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    lib = tem.lib()
    nb = ctypes.c_int64(0)
    ptr = lib.tem_debug_buffer(tem._P(s.ctx), 0, b"trace_on", ctypes.byref(nb))

    class _Arr:
        __cuda_array_interface__ = {"shape": (nb.value // 8,), "typestr": "<u8", "data": (ptr, False), "version": 3}
    buf = torch.as_tensor(_Arr(), device="cuda")
    nslots = lib.tem_timing_slots(tem._P(s.ctx))
    names = [lib.tem_timing_slot_name(tem._P(s.ctx), i).decode() for i in range(nslots)]
    runs, heads = [], []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.reps):
        init = torch.zeros(nb.value // 8, dtype=torch.int64)
        init[0:2 * nslots:2] = -1  # 0xFFFF... as u64: min() identity
        buf.copy_(init.view(torch.uint64) if hasattr(torch, "uint64") else init)
        if args.flush:
            flush.zero_()
        torch.cuda.synchronize()
        step()
        torch.cuda.synchronize()
        allv = buf.cpu().view(torch.int64).numpy().astype(np.float64)
        runs.append(allv[:2 * nslots].reshape(nslots, 2))
        heads.append(allv[2 * nslots:].reshape(4096, 8))
    lib.tem_debug_buffer(tem._P(s.ctx), 0, b"trace_off", ctypes.byref(nb))
    torch.cuda.synchronize()
    rows = []
    for i, nm in enumerate(names):
        st, en = [], []
        for r in runs:
            t0 = min(v for v in r[:, 0] if v > 0)
            if r[i, 1] > 0:
                st.append((r[i, 0] - t0) / 1e3)
                en.append((r[i, 1] - t0) / 1e3)
        if st:
            rows.append((np.median(st), np.median(en), nm))
    ends = [r[1] for r in rows]
    print(f"{args.workload}: step span {max(ends):.1f} us (median of {args.reps}, GPU timeline)")
    for a, b, nm in sorted(rows):
        print(f"  {nm:>20}: {a:7.1f} -> {b:7.1f}  ({b - a:6.1f} us)")
    hp = heads[-1]
    hp = hp[hp[:, 0] > 0]
    if len(hp):
        t0 = hp[:, 0].min()
        print(f"  head_rows phases ({len(hp)} CTAs; us after the first CTA passed pdl_wait): median / max")
        for k, nm in enumerate(["pdl_wait", "labels+loads", "phase1", "phase2", "rp-combine", "end"]):
            d = (hp[:, k] - t0) / 1e3
            print(f"    {nm:>14}: {np.median(d):6.2f} / {d.max():6.2f}")
    s.close()


if __name__ == "__main__":
    main()
