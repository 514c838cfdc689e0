"""GPU parity of the NVSwitch two-shot allreduce: same partition
(reading R9) and chain order as the ring, so its result must equal the oracle's ring replay bit
for bit -- for allreduce, for the hand-derived order witness, and for the fused mean + SGD of
tem_step (N ranks emulated on one device, as the ring tests)."""
import json
import os

import numpy as np
import pytest
import torch

from test_gpu_parity import make_inputs, session, tem, to_dev_x  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("K", [1, 7, 65537, 1403395])
def test_twoshot_allreduce_bitexact(tem, orc, N, K):
    s, _ = session(tem, N, 1, 0, max_allreduce_elems=1403395)
    rng = np.random.default_rng(K * 10 + N + 7)
    Kp = orc.kpad(K, N)
    g = np.zeros((N, Kp), np.float32)
    g[:, :K] = rng.standard_normal((N, K)).astype(np.float32)
    for op in (0, 1):
        sentinel = np.float32(-77.25)
        for r in range(N):
            u = s.user(r, Kp)
            u.copy_(torch.from_numpy(g[r]))
            if Kp > K:
                u[K:] = float(sentinel)
        s.twoshot_allreduce(K, op)
        assert s.sync()[0] == 0
        expect, _ = orc.ring_allreduce(g, op)
        for r in range(N):
            out = s.user(r, Kp).cpu().numpy()
            assert np.array_equal(out[:K], expect[r][:K]), (r, op)
            assert np.all(out[K:] == sentinel)
    s.close()


@pytest.mark.parametrize("N", [3, 4, 8])
def test_twoshot_order_witness(tem, orc, N):
    w = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "order_witness.json")))
    K = 4096
    s, _ = session(tem, N, 1, 0, max_allreduce_elems=K)
    Bk = orc.kpad(K, N) // N
    for r in range(N):
        s.user(r, K).fill_(w["big"] if r == 0 else (-w["big"] if r == 1 else 1.0))
    s.twoshot_allreduce(K, 0)
    assert s.sync()[0] == 0
    expect = np.repeat(np.asarray(w["ring"][str(N)], np.float32), Bk)[:K]
    for r in range(N):
        assert np.array_equal(s.user(r, K).cpu().numpy(), expect)
    s.close()


def test_twoshot_repeated_and_interleaved_with_ring(tem, orc):
    """Epoch flags survive many collectives of both kinds and changing K."""
    N = 4
    s, _ = session(tem, N, 1, 0, max_allreduce_elems=200000)
    rng = np.random.default_rng(3)
    for it, K in enumerate([1000, 200000, 17, 65536, 1000, 3]):
        Kp = orc.kpad(K, N)
        g = np.zeros((N, Kp), np.float32)
        g[:, :K] = rng.standard_normal((N, K)).astype(np.float32)
        for r in range(N):
            s.user(r, Kp).copy_(torch.from_numpy(g[r]))
        (s.twoshot_allreduce if it % 2 == 0 else s.allreduce)(K, 1)
        assert s.sync()[0] == 0
        expect, _ = orc.ring_allreduce(g, 1)
        for r in range(N):
            assert np.array_equal(s.user(r, Kp).cpu().numpy()[:K], expect[r][:K]), (it, r)
    s.close()


@pytest.mark.parametrize("N,B,prec", [(2, 2, 0), (4, 1, 0), (3, 1, 1)])
def test_tem_step_twoshot_exchange(tem, orc, N, B, prec):
    """tem_step with exchange = TWOSHOT: params after the step equal the oracle's ring replay
    (mean + SGD) on the GPU's own local gradients, bitwise, on every rank."""
    lr = 0.05
    s, _ = session(tem, N, B, prec, lr=lr, exchange=tem.TEM_EXCHANGE_TWOSHOT)
    x, lab = make_inputs(N, B, prec)
    w0 = s.params(0).cpu().numpy().copy()
    s.step(to_dev_x(x, prec), torch.from_numpy(lab).cuda())
    assert s.sync()[0] == 0
    grads = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
    expect = orc.ring_sgd(grads, w0, lr)
    for r in range(N):
        assert np.array_equal(s.params(r).cpu().numpy(), expect[r]), r
    if prec == 1:  # bf16 operand copies refreshed on every rank: a second step agrees across ranks
        s.step(to_dev_x(x, prec), torch.from_numpy(lab).cuda())
        assert s.sync()[0] == 0
        for r in range(1, N):
            assert np.array_equal(s.params(r).cpu().numpy(), s.params(0).cpu().numpy())
    s.close()
