"""The host path of a one-process-per-GPU job, as two processes sharing the one GPU of this pool:
process-group rendezvous (gloo), the symmetric-configuration check, the heaps and their
exchange (the peer pointers tem_init receives), tem_init with local_ranks = 1, and a tem_compute
in each process.  torch symmetric memory refuses two processes on one device, so the heaps are
exchanged as CUDA IPC handles (TemSession(heap="ipc")); the symmetric-memory rendezvous itself
needs two GPUs.  No collective kernel runs -- ranks whose
kernels wait on one another must not share a GPU (B200_PROFILING.md); the data plane of that
launch is tests/test_gpu_wire.py.  Checked: each process sees the other's heap through the
mapped peer pointer (a marker written by the peer), and both computes match the oracle per
tensor."""
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
        s = tem.TemSession(sc, datagen.init_params(), heap="ipc")
        marker = float(1000 + rank)
        s.user(0, 1024).fill_(marker)
        torch.cuda.synchronize()
        dist.barrier()
        peer = (rank + 1) % world
        ptr = s._ptr_arr[peer] + s.user_off  # the peer's heap as mapped in this process

        class _Arr:
            __cuda_array_interface__ = {"shape": (1024,), "typestr": "<f4", "data": (ptr, False), "version": 3}
        seen = torch.as_tensor(_Arr(), device="cuda").clone().cpu().numpy()
        x = datagen.features(B, rank=rank, batch_idx=0)
        lab = datagen.labels(B, rank=rank, batch_idx=0)
        loss = s.compute(torch.from_numpy(x).cuda()[None], torch.from_numpy(lab).cuda()[None])
        code, _ = s.sync()
        g = s.local_grad(0).cpu().numpy()[:s.K].copy()
        z = s.logits(0).cpu().numpy().copy()
        # per tensor against the fp64 oracle, ReLU decisions in the ambiguity band taken from the
        # GPU (the parity tests' rule, test_gpu_parity.py)
        from test_gpu_parity import TOL, check_tensors, oracle_with_gpu_decisions
        ref = oracle_with_gpu_decisions(oracle, s, 0, x, datagen.init_params(), lab, (1.0, 1.0, 1.0), 0)
        parity = "ok"
        try:
            check_tensors(oracle, g, z, loss[0].cpu().numpy().copy(), ref, TOL[0])
        except AssertionError as e:
            parity = repr(e)
        dist.barrier()
        s.close()
        q.put((rank, "ok", {"peer_marker": float(seen[0]), "peer_all": bool(np.all(seen == seen[0])),
                            "code": code, "parity": parity, "expect": float(1000 + peer)}))
    except Exception as e:
        q.put((rank, "err", repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_processes_ipc_heaps_on_one_gpu():
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
    for r, (st, out) in res.items():
        assert st == "ok", (r, out)
        assert out["code"] == 0
        assert out["peer_marker"] == out["expect"] and out["peer_all"], out
        assert out["parity"] == "ok", out


def _ring_worker(rank, world, port, q):
    """One rank of a 2-process ring_allreduce over IPC-mapped heaps, run in turn (never two
    kernels waiting on each other): rank 0 first, against rank 1's messages written by rank 1's
    process from the oracle (the wire protocol of include/tem.h); then rank 1's kernel, against
    the messages rank 0's kernel actually stored into its heap."""
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
        import test_gpu_wire as W
        from paper_1906_06496_b200 import dist as tdist
        from paper_1906_06496_b200 import tem
        tdist.init_from_env("gloo")
        K, op = 40000 + 7, 1  # TEM_MEAN, K < K_pad: the tail is masked
        sc = tem.SessionConfig(world_size=world, rank=rank, local_ranks=1, batch_per_rank=1, ring_channels=W.G,
                               max_allreduce_elems=K)
        s = tem.TemSession(sc, datagen.init_params(), heap="ipc")
        Kp = oracle.kpad(K, world)
        rng = np.random.default_rng(7)
        g = np.zeros((world, Kp), np.float32)
        g[:, :K] = rng.standard_normal((world, K)).astype(np.float32)
        final = oracle.ring_allreduce(g, op)[0][0].copy()
        final[K:] = 0.0
        s.user(0, Kp).copy_(torch.from_numpy(g[rank]))
        torch.cuda.synchronize()
        out = {}
        # phase A: rank 1's process writes, through its mapping of rank 0's heap, everything
        # rank 0 will receive; rank 0 runs
        if rank == 1:
            W.transcript_in(oracle, s, g, final, 0, 1, K, op, 0)
            torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            s.allreduce(K, op)
            code, _ = s.sync()
            out["code_a"] = code
            out["result_a"] = bool(np.array_equal(s.user(0, K).cpu().numpy(), final[:K]))
        dist.barrier()
        if rank == 1:  # rank 0's sends, as they arrived in this process's heap
            W.check_transcript_out(oracle, s, g, final, 0, 1)
            out["sent_a"] = True
        dist.barrier()
        # phase B: rank 1 runs against what rank 0's kernel stored
        if rank == 1:
            s.allreduce(K, op)
            code, _ = s.sync()
            out["code_b"] = code
            out["result_b"] = bool(np.array_equal(s.user(0, K).cpu().numpy(), final[:K]))
        dist.barrier()
        if rank == 0:
            W.check_transcript_out(oracle, s, g, final, 1, 1)
            out["sent_b"] = True
        dist.barrier()
        s.close()
        q.put((rank, "ok", out))
    except Exception as e:
        import traceback
        q.put((rank, "err", traceback.format_exc()[-2000:]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_process_ring_through_ipc_heaps():
    """The production non-cooperative ring kernel in two processes, with every message crossing
    between the processes' IPC-mapped heaps: both results bit-exact against the oracle's ring
    replay (TEM_MEAN), and every message each kernel sent equal to the oracle's transcript."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ring_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, status, out = q.get(timeout=300)
        res[r] = (status, out)
    for p in procs:
        p.join(timeout=60)
    for r, (st, out) in res.items():
        assert st == "ok", (r, out)
    a, b = res[0][1], res[1][1]
    assert a["code_a"] == 0 and a["result_a"] and b["sent_a"], res
    assert b["code_b"] == 0 and b["result_b"] and a["sent_b"], res


def _step_worker(rank, world, port, q):
    """One rank of a 2-process data-parallel tem_step (compute + ring + mean + SGD) over
    IPC-mapped heaps, the two ranks' steps run in turn (see _ring_worker)."""
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
        import test_gpu_wire as W
        from paper_1906_06496_b200 import dist as tdist
        from paper_1906_06496_b200 import tem
        tdist.init_from_env("gloo")
        B, lr, lam = 2, 0.05, (2.0, 1.0, 1.0)
        sc = tem.SessionConfig(world_size=world, rank=rank, local_ranks=1, batch_per_rank=B, lr=lr,
                               loss_weight=lam, ring_channels=W.G)
        s = tem.TemSession(sc, datagen.init_params(), heap="ipc")
        Kp = s.Kpad
        xd = torch.from_numpy(datagen.features(B, rank=rank, batch_idx=0)).cuda()[None]
        ld = torch.from_numpy(datagen.labels(B, rank=rank, batch_idx=0)).cuda()[None]
        w0 = s.params(0).cpu().numpy().copy()
        s.compute(xd, ld)  # the step recomputes this gradient bit for bit (deterministic kernels)
        assert s.sync()[0] == 0
        g_all = [None] * world
        dist.all_gather_object(g_all, s.local_grad(0).cpu().numpy().copy())
        g = np.stack(g_all)
        fin = oracle.ring_sgd(g, w0, lr)
        assert np.array_equal(fin[0], fin[1])
        expect = fin[0]
        out = {}
        if rank == 1:  # rank 0's inbound messages, from the real gradients
            W.transcript_in(oracle, s, g, expect, 0, 1, Kp, 1, 1)
            torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            s.step(xd, ld)
            out["code_a"] = s.sync()[0]
        dist.barrier()
        if rank == 1:
            W.check_transcript_out(oracle, s, g, expect, 0, 1)
            s.step(xd, ld)  # against the messages rank 0's kernel stored into this heap
            out["code_b"] = s.sync()[0]
        dist.barrier()
        if rank == 0:
            W.check_transcript_out(oracle, s, g, expect, 1, 1)
        w = s.params(0).cpu().numpy()
        out["params_ok"] = bool(np.array_equal(w, expect))
        w_all = [None] * world
        dist.all_gather_object(w_all, w.copy())
        out["replicas_equal"] = bool(np.array_equal(w_all[0], w_all[1]))
        dist.barrier()
        s.close()
        q.put((rank, "ok", out))
    except Exception:
        import traceback
        q.put((rank, "err", traceback.format_exc()[-2000:]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_process_dp_step_through_ipc_heaps():
    """A 2-process data-parallel tem_step (each process its own shard: compute, ring allreduce,
    1/N mean, SGD fused in the owner) with the two steps run in turn over
    IPC-mapped heaps: both ranks' parameters bitwise equal to the oracle's ring replay of the
    two GPU gradients, the replicas identical, every message as the oracle's transcript."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, status, out = q.get(timeout=300)
        res[r] = (status, out)
    for p in procs:
        p.join(timeout=60)
    for r, (st, out) in res.items():
        assert st == "ok", (r, out)
        assert out["params_ok"] and out["replicas_equal"], (r, out)
    assert res[0][1]["code_a"] == 0 and res[1][1]["code_b"] == 0, res
