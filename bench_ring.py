#!/usr/bin/env python
"""bench_ring.py -- BASELINE.json configs[3]: ring-allreduce bandwidth sweep vs NCCL.

    torchrun --nproc-per-node N bench_ring.py [--sizes ...] [--iters 50]

For each message size S (64 KiB .. 256 MiB, plus the TEM gradient 5,613,580 B) it times, with
CUDA events on each rank and the max over ranks:
  * ours : ring_allreduce (KR1) of S/4 fp32 elements, Sum; and the NVSwitch
           two-shot (same result bits, 2 phases instead of 2(N-1) rounds);
  * ps   : the parameter-server comparator at the TEM gradient size;
  * nccl : torch.distributed.all_reduce (NCCL), with whatever algorithm NCCL picks; run the
           script again with NCCL_ALGO=Ring for NCCL's ring.
and prints one JSON line per (impl, size): algbw = S/t, busbw = algbw * 2(N-1)/N (NCCL's
convention), and busbw as a fraction of 900 GB/s per direction.

With a single process and --emulate N, the N ranks run as CTA groups of one cooperative
launch on one GPU (the parity-test configuration): that measures the kernel, not NVLink.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TEM_BYTES = 1403395 * 4
NVLINK_GBS = 900.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--max-mib", type=int, default=256)
    ap.add_argument("--emulate", type=int, default=0, help="single-GPU emulation of N ranks")
    ap.add_argument("--no-nccl", action="store_true")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist
    import datagen
    from paper_1906_06496_b200 import dist as tdist
    from paper_1906_06496_b200 import metrics, tem

    rank, world, local = tdist.env_world()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    emulate = args.emulate if world == 1 else 0
    if world > 1:
        tdist.init_from_env("nccl", dev)
    N = emulate if emulate else world
    sizes = [1 << k for k in range(16, 29) if (1 << k) <= (args.max_mib << 20)]
    sizes = sorted(set(sizes + [TEM_BYTES]))
    maxK = max(sizes) // 4
    sc = tem.SessionConfig(world_size=N, rank=rank if not emulate else 0, local_ranks=N if emulate else 1,
                           batch_per_rank=1, max_allreduce_elems=maxK)
    sess = tem.TemSession(sc, datagen.init_params(), device=local)
    rng = np.random.default_rng(rank)
    stream = torch.cuda.current_stream()

    def timeit(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / args.iters / 1e3
        return tdist.max_over_ranks(t)

    out = []
    for S in sizes:
        K = S // 4
        for l in range(N if emulate else 1):
            sess.user(l, K).copy_(torch.from_numpy(rng.standard_normal(K).astype(np.float32) * 1e-3))
        t = timeit(lambda: sess.allreduce(K, tem.TEM_SUM))
        code, _ = sess.sync()
        assert code == 0, tem.status_string(code)
        out.append(("ours-ring", S, t))
        t = timeit(lambda: sess.twoshot_allreduce(K, tem.TEM_SUM))
        code, _ = sess.sync()
        assert code == 0, tem.status_string(code)
        out.append(("ours-twoshot", S, t))
        if S == TEM_BYTES:
            t = timeit(lambda: sess.ps_allreduce(K, tem.TEM_SUM))
            out.append(("ours-ps", S, t))
        if world > 1 and not args.no_nccl:
            buf = torch.randn(K, device=dev)
            t = timeit(lambda: dist.all_reduce(buf))
            out.append((f"nccl-{os.environ.get('NCCL_ALGO', 'default')}", S, t))
    if rank == 0:
        for impl, S, t in out:
            bus = metrics.busbw(S, t, N) / 1e9
            kpad = (S // 4 + 4 * N - 1) // (4 * N) * 4 * N
            print(json.dumps({"metric": "allreduce bus bandwidth", "impl": impl, "bytes": S, "n_ranks": N,
                              "emulated": bool(emulate), "time_us": t * 1e6, "algbw_GBs": S / t / 1e9,
                              "busbw_GBs": bus, "frac_of_900GBs": bus / NVLINK_GBS,
                              "ring_bytes_sent_per_rank": metrics.ring_bytes_per_rank(kpad, N)}))
    sess.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
