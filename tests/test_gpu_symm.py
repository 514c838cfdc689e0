"""The production host path of a one-process-per-GPU job, as two processes sharing the one GPU
of this pool: process-group rendezvous (gloo), the symmetric-configuration check, torch
symmetric-memory heaps and their rendezvous (the peer pointers tem_init receives), tem_init with
local_ranks = 1, and a tem_compute in each process.  No collective kernel runs -- ranks whose
kernels wait on one another must not share a GPU (B200_PROFILING.md); the data plane of that
launch is tests/test_gpu_wire.py.  Checked: each process sees the other's heap through the
mapped peer pointer (a marker written by the peer), and both computes match the oracle."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": "0",
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        import datagen
        import oracle
        from paper_1906_06496_b200 import dist as tdist
        from paper_1906_06496_b200 import tem
        tdist.init_from_env("gloo")
        B = 2
        sc = tem.SessionConfig(world_size=world, rank=rank, local_ranks=1, batch_per_rank=B, lr=0.05)
        try:
            s = tem.TemSession(sc, datagen.init_params())
        except Exception as e:  # symmetric memory unavailable for two processes on one device
            q.put((rank, "skip", repr(e)))
            return
        marker = float(1000 + rank)
        s.user(0, 1024).fill_(marker)
        torch.cuda.synchronize()
        dist.barrier()
        peer = (rank + 1) % world
        ptr = s._symm[1].buffer_ptrs[peer] + s.user_off

        class _Arr:
            __cuda_array_interface__ = {"shape": (1024,), "typestr": "<f4", "data": (ptr, False), "version": 3}
        seen = torch.as_tensor(_Arr(), device="cuda").clone().cpu().numpy()
        x = datagen.features(B, rank=rank, batch_idx=0)
        lab = datagen.labels(B, rank=rank, batch_idx=0)
        loss = s.compute(torch.from_numpy(x).cuda()[None], torch.from_numpy(lab).cuda()[None])
        code, _ = s.sync()
        g = s.local_grad(0).cpu().numpy()[:s.K]
        ref = oracle.tem_fwd_bwd(x, datagen.init_params(), lab, (1.0, 1.0, 1.0), prec=0)
        gerr = float(np.abs(g - ref["grad"]).max() / np.abs(ref["grad"]).max())
        lerr = float(np.abs(loss[0].cpu().numpy() - ref["loss"]).max() / np.abs(ref["loss"]).max())
        dist.barrier()
        s.close()
        q.put((rank, "ok", {"peer_marker": float(seen[0]), "peer_all": bool(np.all(seen == seen[0])),
                            "code": code, "gerr": gerr, "lerr": lerr, "expect": float(1000 + peer)}))
    except Exception as e:
        q.put((rank, "err", repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_processes_symmetric_heaps_on_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, status, out = q.get(timeout=300)
        res[r] = (status, out)
    for p in procs:
        p.join(timeout=60)
    if any(st == "skip" for st, _ in res.values()):
        pytest.skip(f"symmetric memory across two processes on one GPU unavailable: {res}")
    for r, (st, out) in res.items():
        assert st == "ok", (r, out)
        assert out["code"] == 0
        assert out["peer_marker"] == out["expect"] and out["peer_all"], out
        assert out["gerr"] <= 1e-4 and out["lerr"] <= 1e-4, out
