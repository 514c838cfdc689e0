"""World-size-2 tests of the N > 1 host path on CPU (gloo): rendezvous from env, the
symmetric-configuration check, max-over-ranks timing, per-rank sharding, and the
data-parallel identity the ring implements (mean of per-rank gradients == gradient of the
global batch), with the oracle standing in for the per-rank compute."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    from paper_1906_06496_b200 import dist as tdist
    try:
        tdist.init_from_env("gloo")
        out = globals()[fn_name](rank, world)
        q.put((rank, "ok", out))
    except Exception as e:  # report to the parent
        q.put((rank, "err", repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def run(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, status, out = q.get(timeout=240)
        res[r] = (status, out)
    for p in procs:
        p.join(timeout=60)
    return res


# ---------------------------------------------------------------- worker bodies
def body_env_and_max(rank, world):
    from paper_1906_06496_b200 import dist as tdist
    r, w, l = tdist.env_world()
    assert (r, w, l) == (rank, world, rank)
    return tdist.max_over_ranks(1.5 + rank)


def body_symmetric_ok(rank, world):
    from paper_1906_06496_b200 import dist as tdist
    from paper_1906_06496_b200.tem import SessionConfig
    tdist.check_symmetric(SessionConfig(world_size=world, rank=rank, batch_per_rank=16))
    return True


def body_symmetric_bad(rank, world):
    from paper_1906_06496_b200 import dist as tdist
    from paper_1906_06496_b200.tem import SessionConfig
    try:
        tdist.check_symmetric(SessionConfig(world_size=world, rank=rank, batch_per_rank=16 + rank))
    except tdist.ConfigMismatch:
        return "mismatch"
    return "no-error"


def body_dp_identity(rank, world):
    """Each rank computes the oracle gradient of its shard (seeded per rank); the mean over
    ranks equals the oracle gradient of the concatenated global batch."""
    import datagen
    import oracle
    from paper_1906_06496_b200 import dist as tdist
    rng = np.random.default_rng(0)
    Cin, C, T = 8, 16, 6
    K = C * 3 * Cin + C + C * 3 * C + C + 3 * C + 3
    p = (rng.standard_normal(K) * 0.3).astype(np.float32)
    Bg = 4
    x_all = rng.standard_normal((Bg, T, Cin)).astype(np.float32)
    lab_all = rng.uniform(0, 1, size=(Bg, 3, T)).astype(np.float32)
    idx = list(tdist.shard_batch_indices(Bg, world, rank))
    g = oracle.tem_fwd_bwd(x_all[idx], p, lab_all[idx], prec=0, C=C)["grad"]
    t = torch.from_numpy(g.copy())
    dist.all_reduce(t)
    t /= world
    full = oracle.tem_fwd_bwd(x_all, p, lab_all, prec=0, C=C)["grad"]
    err = float(np.abs(t.numpy() - full).max() / np.abs(full).max())
    # the per-rank synthetic shards the bench uses are distinct
    xs = datagen.features(2, T, Cin, rank=rank, batch_idx=0)
    other = [None] * world
    dist.all_gather_object(other, float(xs.sum()))
    return err, len(set(other)) == world


# ---------------------------------------------------------------- tests
def test_env_rendezvous_and_max_over_ranks():
    res = run("body_env_and_max")
    assert all(s == "ok" for s, _ in res.values()), res
    assert all(v == 2.5 for _, v in res.values())


def test_symmetric_config_check():
    res = run("body_symmetric_ok")
    assert all(s == "ok" and v for s, v in res.values()), res
    res = run("body_symmetric_bad")
    assert all(s == "ok" and v == "mismatch" for s, v in res.values()), res


def test_data_parallel_identity_two_ranks():
    res = run("body_dp_identity")
    assert all(s == "ok" for s, _ in res.values()), res
    for _, (err, distinct) in res.values():
        assert err < 1e-12 and distinct


def test_shard_indices():
    from paper_1906_06496_b200 import dist as tdist
    assert list(tdist.shard_batch_indices(8, 2, 1)) == [4, 5, 6, 7]
    with pytest.raises(ValueError):
        tdist.shard_batch_indices(7, 2, 0)
