"""End-to-end training sanity on the GPU: repeated tem_step calls on a fixed batch drive the
BSN-TEM loss down (the gradient, the exchange and the owner update compose into descent), for
SGD, momentum and Adam, with N = 2 emulated ranks kept bitwise identical throughout."""
import numpy as np
import pytest
import torch

from test_gpu_parity import make_inputs, session, tem, to_dev_x  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("opt,lr", [(0, 0.5), (2, 0.1), (1, 1e-3)])
def test_loss_decreases(tem, opt, lr):
    N, B, steps = 2, 4, 60
    s, _ = session(tem, N, B, 0, lr=lr, lam=(1.0, 1.0, 1.0), optimizer=opt, momentum=0.9)
    x, lab = make_inputs(N, B, 0, batch_idx=11)
    xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
    losses = []
    for _ in range(steps):
        loss = s.step(xd, ld)
        losses.append(float(loss[:, 0].sum().cpu()))
    assert s.sync()[0] == 0
    assert np.all(np.isfinite(losses))
    first, last = np.mean(losses[:5]), np.mean(losses[-5:])
    assert last < 0.8 * first, (first, last)
    p0 = s.params(0).cpu().numpy()
    assert np.array_equal(p0, s.params(1).cpu().numpy())  # replicas stay identical
    s.close()


def test_joint_pem_loss_decreases(tem):
    """TEM + PEM joint steps (configs[4]): both losses fall on a fixed batch."""
    from test_gpu_pem import pem_inputs, pem_session
    N, B = 2, 2
    s, _ = pem_session(tem, N, B, lr=0.5, lam=(1.0, 1.0, 1.0))
    x, lab = make_inputs(N, B, 0, batch_idx=12)
    f, g = pem_inputs(N, B, batch_idx=12)
    xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
    fd, gd = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    tl, pl = [], []
    for _ in range(60):
        a, b = s.step_pem(xd, ld, fd, gd)
        tl.append(float(a[:, 0].sum().cpu()))
        pl.append(float(b.sum().cpu()))
    assert s.sync()[0] == 0
    assert np.mean(tl[-5:]) < 0.8 * np.mean(tl[:5])
    assert np.mean(pl[-5:]) < np.mean(pl[:5])
    s.close()
