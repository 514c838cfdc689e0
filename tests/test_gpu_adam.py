"""GPU parity of the Adam owner update (reading R22) through the C ABI.

Every exchange (ring, two-shot, parameter server) and the N = 1 update kernels apply Adam with
single-rounded fp32 operations in the oracle's order, so after each step the parameters on every
rank equal the oracle's replay (orc.ring_adam, whose arithmetic is pinned in
tests/test_oracle_ring.py against textbook float64 Adam) on the GPU's own local gradients, bit
for bit.  The oracle carries m, v and beta^t across steps; the GPU keeps its own, so agreement
after several steps also checks the moments and the bias-correction products."""
import numpy as np
import pytest
import torch

from test_gpu_parity import make_inputs, session, tem, to_dev_x  # noqa: F401

pytestmark = pytest.mark.gpu

LR, B1, B2, EPS = 1e-3, 0.9, 0.999, 1e-8


def adam_session(tem, N, B, prec, exchange):
    return session(tem, N, B, prec, lr=LR, exchange=exchange, optimizer=tem.TEM_OPT_ADAM, beta1=B1, beta2=B2,
                   eps=EPS)


def oracle_step(orc, tem, exchange, grads, w, st):
    m, v, sc = st
    if exchange == tem.TEM_EXCHANGE_PS:  # ascending-rank mean, then the server's Adam
        gbar = orc.ps_allreduce(grads, orc.MEAN)
        return orc.ring_adam(gbar[None, :], w, m, v, sc, LR, B1, B2, EPS)
    return orc.ring_adam(grads, w, m, v, sc, LR, B1, B2, EPS)


@pytest.mark.parametrize("N,B,prec,exchange", [(1, 4, 0, 0), (1, 2, 1, 0), (2, 2, 0, 0), (3, 1, 0, 0),
                                               (4, 1, 1, 0), (2, 2, 0, 2), (4, 1, 0, 2), (3, 1, 0, 1)])
def test_adam_steps_bitexact(tem, orc, N, B, prec, exchange):
    s, _ = adam_session(tem, N, B, prec, exchange)
    Kp = s.Kpad
    w = s.params(0).cpu().numpy().copy()
    st = (np.zeros(Kp, np.float32), np.zeros(Kp, np.float32), np.ones(2, np.float32))
    for it in range(3):
        x, lab = make_inputs(N, B, prec, batch_idx=it)
        s.step(to_dev_x(x, prec), torch.from_numpy(lab).cuda())
        assert s.sync()[0] == 0
        grads = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
        w, m, v, sc = oracle_step(orc, tem, exchange, grads, w, st)
        st = (m, v, sc)
        for r in range(N):
            got = s.params(r).cpu().numpy()
            bad = np.nonzero(got != w)[0]
            assert bad.size == 0, (it, r, bad[:5], got[bad[:5]], w[bad[:5]])
    s.close()


def test_adam_compute_then_exchange(tem, orc):
    """N = 1 through tem_compute + tem_exchange (the unfused update kernel) == tem_step's."""
    B = 4
    s, _ = adam_session(tem, 1, B, 0, 0)
    w = s.params(0).cpu().numpy().copy()
    st = (np.zeros(s.Kpad, np.float32), np.zeros(s.Kpad, np.float32), np.ones(2, np.float32))
    for it in range(2):
        x, lab = make_inputs(1, B, 0, batch_idx=5 + it)
        s.compute(to_dev_x(x, 0), torch.from_numpy(lab).cuda())
        s.exchange()
        assert s.sync()[0] == 0
        w, m, v, sc = orc.ring_adam(s.local_grad(0).cpu().numpy()[None, :], w, *st, LR, B1, B2, EPS)
        st = (m, v, sc)
        assert np.array_equal(s.params(0).cpu().numpy(), w), it
    s.close()


def test_adam_graph_and_eager_identical(tem, monkeypatch):
    """The beta^t kernel is captured in the step graph: replayed and eager steps agree bitwise."""
    def run():
        s, _ = adam_session(tem, 1, 8, 0, 0)
        x, lab = make_inputs(1, 8, 0, batch_idx=6)
        xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
        for _ in range(4):
            s.step(xd, ld)
        assert s.sync()[0] == 0
        w = s.params(0).cpu().numpy().copy()
        s.close()
        return w
    w_graph = run()
    monkeypatch.setenv("TEM_NO_GRAPH", "1")
    assert np.array_equal(w_graph, run())


MU = 0.9


@pytest.mark.parametrize("N,B,prec,exchange", [(1, 4, 0, 0), (1, 2, 1, 0), (2, 2, 0, 0), (3, 1, 0, 0),
                                               (4, 1, 0, 2), (3, 1, 0, 1)])
def test_momentum_steps_bitexact(tem, orc, N, B, prec, exchange):
    """Heavy-ball momentum (reading R23) in every exchange: params after each of 3 steps equal
    orc.ring_momentum's replay on the GPU's own local gradients, bitwise, on every rank."""
    lr = 0.02
    s, _ = session(tem, N, B, prec, lr=lr, exchange=exchange, optimizer=tem.TEM_OPT_MOMENTUM, momentum=MU)
    w = s.params(0).cpu().numpy().copy()
    u = np.zeros(s.Kpad, np.float32)
    for it in range(3):
        x, lab = make_inputs(N, B, prec, batch_idx=10 + it)
        s.step(to_dev_x(x, prec), torch.from_numpy(lab).cuda())
        assert s.sync()[0] == 0
        grads = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
        if exchange == tem.TEM_EXCHANGE_PS:
            grads = orc.ps_allreduce(grads, orc.MEAN)[None, :]
        w, u = orc.ring_momentum(grads, w, u, lr, MU)
        for r in range(N):
            assert np.array_equal(s.params(r).cpu().numpy(), w), (it, r)
    s.close()
