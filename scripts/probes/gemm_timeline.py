#!/usr/bin/env python
"""Phase timeline of a FWD/DGRAD GEMM launch (diagnostics; needs a GPU).

    TEM_NO_GRAPH=1 [TEM_SPLITK=1] python scripts/probes/split_timeline.py [--workload c2] [--kernel halo|split]

Runs steps, enables the kernel's globaltimer stamps for the last one, and prints the per-phase
times (us after the earliest CTA entry; median / max over CTAs) of the step's last FWD/DGRAD
launch (conv2 dgrad).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

PHASES = {"split": ["entry", "pdl_wait", "prod_firstA", "mma_fullA", "mma_fullB", "mma_done", "epi_tfull",
                    "cluster1", "packed", "received", "done"],
          "halo": ["entry", "pdl_wait", "mma_fullA0", "tile0_mma_done", "last_mma_done", "acc_ready", "epi_done"],
          # conv2 FWD with the fused head (stamps 8..13; conv2 dgrad overwrites 0..6)
          "head": ["-"] * 8 + ["head_start", "cluster1", "dz_done", "dA2_done", "colsum_done",
                               "c0_tmem", "c0_math", "c0_stored"],
          "wgrad1": ["entry", "prologue", "mma_full0", "mma_done", "-", "acc_ready", "epi_done", "-"]
                    + [f"chunk{i}" for i in range(8)],
          "fwd1": ["entry", "pdl_wait", "mma_fullA0", "tile0_mma_done", "last_mma_done", "acc_ready", "epi_done", "-"]
                  + [f"chunk{i}" for i in range(4)],
          "wgrad2": ["entry", "prologue", "mma_full0", "mma_done", "-", "acc_ready", "epi_done"],
          # conv2 FWD + fused head, one launch (slot stamps)
          "fwd2": ["entry", "pdl_wait", "mma_fullA0", "tile0_mma_done", "-", "acc_ready", "epi_done", "-",
                   "head_start", "cluster1", "dz_done", "dA2_done", "colsum_done", "c0_tmem", "c0_math",
                   "c0_stored"]}
SLOTS = {"wgrad2": 6, "wgrad1": 8, "fwd1": 1, "fwd2": 2}  # Slot enum (kernels.h)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--kernel", default="halo", choices=["halo", "split", "head", "wgrad1", "wgrad2", "fwd1", "fwd2"])
    ap.add_argument("--warm", type=int, default=3, help="steps before the stamped one")
    ap.add_argument("--skip", type=int, default=0, help="probe_skip bits: 1 A-window loads, 2 B-tap loads")
    args = ap.parse_args()
    os.environ["TEM_DIAG_LIB"] = "1"  # traces / phase stamps exist only in the diagnostics build
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
    if args.skip:
        lib.tem_debug_buffer(tem._P(s.ctx), 0, f"probe_skip:{args.skip}".encode(), ctypes.byref(nb))
    def step():
        try:
            s.step(x, lab)
        except tem.TemError:  # skipped operand loads: garbage operands, non-finite loss
            if not args.skip:
                raise
    for _ in range(args.warm):
        step()
    torch.cuda.synchronize()
    on = b"tstamp_on" if args.kernel not in SLOTS else f"tstamp_slot:{SLOTS[args.kernel]}".encode()
    lib.tem_debug_buffer(tem._P(s.ctx), 0, on, ctypes.byref(nb))
    step()
    torch.cuda.synchronize()
    ptr = lib.tem_debug_buffer(tem._P(s.ctx), 0, b"tstamp", ctypes.byref(nb))
    class _Arr:  # wrap the raw device pointer (a __device__ symbol, outside the workspace)
        __cuda_array_interface__ = {"shape": (nb.value // 8,), "typestr": "<i8", "data": (ptr, False), "version": 3}
    raw = torch.as_tensor(_Arr(), device="cuda").cpu().numpy().reshape(1024, 16)
    used = raw[:, 0] > 0
    raw = raw[used]
    t0 = raw[:, 0].min() if args.kernel != "head" else raw[:, 8][raw[:, 8] > 0].min()
    print(f"{used.sum()} CTAs stamped")
    for k, name in enumerate(PHASES[args.kernel]):
        col = raw[:, k]
        col = col[col > 0]
        if len(col) and name != "-":
            d = (col - t0) / 1e3
            print(f"{name:>12}: median {np.median(d):7.2f} us  max {d.max():7.2f} us  (n={len(col)})")
    if args.kernel in ("fwd1", "fwd2"):
        ml = (raw[:, 3] - raw[:, 2]) / 1e3
        print(f"    mainloop: median {np.median(ml):7.2f} us  max {ml.max():7.2f} us")
        cptr = lib.tem_debug_buffer(tem._P(s.ctx), 0, b"tclk", ctypes.byref(nb))
        class _C:
            __cuda_array_interface__ = {"shape": (nb.value // 8,), "typestr": "<i8", "data": (cptr, False), "version": 3}
        clk = torch.as_tensor(_C(), device="cuda").cpu().numpy().reshape(1024, 4)[used]
        cyc = clk[:, 1] - clk[:, 0]
        kpairs = {"fwd1": 7 * 12, "fwd2": 8 * 12}[args.kernel]
        print(f"    mainloop: median {np.median(cyc):8.0f} clk = {np.median(cyc) / kpairs:6.1f} clk per K-step pair, "
              f"clock {np.median(cyc / (ml * 1e3)):.3f} GHz")
    if args.skip:
        lib.tem_debug_buffer(tem._P(s.ctx), 0, b"probe_skip:0", ctypes.byref(nb))
    s.close()


if __name__ == "__main__":
    main()
