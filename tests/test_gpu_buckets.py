"""GPU parity of the bucketed exchange (reading R25): exchange_buckets = 2
splits the gradient at bnd = roundup(off_W2, 4N) and exchanges [bnd, K_pad) and [0, bnd) each
with R9's partition of its own length, so every rank's params after a step equal the oracle's
ring replay applied to each bucket, bitwise (N ranks emulated on one device; with one rank per
process the [bnd, K_pad) bucket is launched inside the compute, beside conv1 wgrad)."""
import numpy as np
import pytest
import torch

import datagen
from test_gpu_parity import make_inputs, session, tem, to_dev_x  # noqa: F401

pytestmark = pytest.mark.gpu

OFF_W2 = 512 * 3 * 400 + 512  # [W1 | b1] (reading R3)


def bound(N):
    q = 4 * N
    return (OFF_W2 + q - 1) // q * q


@pytest.mark.parametrize("N,B,prec,exchange", [(2, 2, 0, 0), (3, 1, 0, 0), (4, 1, 1, 0), (3, 1, 0, 2),
                                               (4, 1, 0, 2), (8, 1, 0, 0)])
def test_bucketed_sgd_bitexact(tem, orc, N, B, prec, exchange):
    lr = 0.05
    s, _ = session(tem, N, B, prec, lr=lr, exchange=exchange, exchange_buckets=2)
    bnd = bound(N)
    for it in range(2):
        x, lab = make_inputs(N, B, prec, batch_idx=it)
        w0 = s.params(0).cpu().numpy().copy()
        s.step(to_dev_x(x, prec), torch.from_numpy(lab).cuda())
        assert s.sync()[0] == 0
        g = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
        expect = np.concatenate([orc.ring_sgd(g[:, :bnd], w0[:bnd], lr), orc.ring_sgd(g[:, bnd:], w0[bnd:], lr)],
                                axis=1)
        for r in range(N):
            assert np.array_equal(s.params(r).cpu().numpy(), expect[r]), (it, r)
    s.close()


def test_bucketed_adam_bitexact(tem, orc):
    """Adam state follows the buckets (pointer offsets); beta^t advances once per step."""
    N, B, lr = 3, 1, 1e-3
    s, _ = session(tem, N, B, 0, lr=lr, exchange_buckets=2, optimizer=tem.TEM_OPT_ADAM)
    bnd = bound(N)
    w = s.params(0).cpu().numpy().copy()
    m = np.zeros_like(w)
    v = np.zeros_like(w)
    sc = np.ones(2, np.float32)
    for it in range(3):
        x, lab = make_inputs(N, B, 0, batch_idx=it + 3)
        s.step(to_dev_x(x, 0), torch.from_numpy(lab).cuda())
        assert s.sync()[0] == 0
        g = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
        w0, m0, v0, sc1 = orc.ring_adam(g[:, :bnd], w[:bnd], m[:bnd], v[:bnd], sc, lr)
        w1, m1, v1, _ = orc.ring_adam(g[:, bnd:], w[bnd:], m[bnd:], v[bnd:], sc, lr)
        w, m, v, sc = np.concatenate([w0, w1]), np.concatenate([m0, m1]), np.concatenate([v0, v1]), sc1
        for r in range(N):
            assert np.array_equal(s.params(r).cpu().numpy(), w), (it, r)
    s.close()


def test_bucketed_pem_joint_step(tem, orc):
    """The joint [TEM | PEM] gradient: PEM's elements lie in the [bnd, K_pad) bucket."""
    from test_gpu_pem import pem_inputs
    N, B, lr = 2, 2, 0.05
    sc = tem.SessionConfig(world_size=N, rank=0, local_ranks=N, batch_per_rank=B, lr=lr, loss_weight=(2.0, 1.0, 1.0),
                           pem_proposals=datagen.PEM_P, exchange_buckets=2)
    s = tem.TemSession(sc, np.concatenate([datagen.init_params(), datagen.init_pem_params()]))
    x, lab = make_inputs(N, B, 0)
    f, gt = pem_inputs(N, B)
    w0 = s.params(0).cpu().numpy().copy()
    s.step_pem(to_dev_x(x, 0), torch.from_numpy(lab).cuda(), torch.from_numpy(f).cuda(), torch.from_numpy(gt).cuda())
    assert s.sync()[0] == 0
    g = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
    bnd = bound(N)
    expect = np.concatenate([orc.ring_sgd(g[:, :bnd], w0[:bnd], lr), orc.ring_sgd(g[:, bnd:], w0[bnd:], lr)], axis=1)
    for r in range(N):
        assert np.array_equal(s.params(r).cpu().numpy(), expect[r]), r
    s.close()


def test_single_bucket_is_the_paper_ring(tem, orc):
    """exchange_buckets = 1 is the default single ring (same bits as exchange_buckets = 0)."""
    N, B, lr = 3, 1, 0.05
    s, _ = session(tem, N, B, 0, lr=lr, exchange_buckets=1)
    x, lab = make_inputs(N, B, 0)
    w0 = s.params(0).cpu().numpy().copy()
    s.step(to_dev_x(x, 0), torch.from_numpy(lab).cuda())
    assert s.sync()[0] == 0
    g = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
    expect = orc.ring_sgd(g, w0, lr)
    for r in range(N):
        assert np.array_equal(s.params(r).cpu().numpy(), expect[r])
    s.close()
