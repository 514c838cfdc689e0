"""GPU parity of the joint TEM + PEM step (BASELINE configs[4]; readings R19-R21) through the
C ABI: the PEM gradient and loss against the fp64 PEM oracle (1e-4, ReLU decisions handled as
in reading R7b), the TEM part against the TEM oracle, and the exchange of the concatenated
gradient bit-exact against the oracle's ring replay."""
import numpy as np
import pytest
import torch

import datagen
from test_gpu_parity import (TOL, check_tensors, make_inputs, oracle_with_gpu_decisions, rel_err,  # noqa: F401
                             tem, to_dev_x)

pytestmark = pytest.mark.gpu

P, F, H = datagen.PEM_P, datagen.PEM_F, datagen.PEM_H
KINK_TAU_PEM = 2.0 ** -16  # fp32 dot product of 32 terms: ~F u relative to sum|terms|


def pem_session(tem, N, B, prec=0, lr=0.05, lam=(2.0, 1.0, 1.0)):
    sc = tem.SessionConfig(world_size=N, rank=0, local_ranks=N, batch_per_rank=B, precision=prec, lr=lr,
                           loss_weight=lam, pem_proposals=P, pem_features=F, pem_hidden=H)
    p = np.concatenate([datagen.init_params(), datagen.init_pem_params()])
    return tem.TemSession(sc, p), p


def pem_inputs(N, B, batch_idx=0):
    f = np.stack([datagen.bsp_features(B, rank=r, batch_idx=batch_idx) for r in range(N)])
    g = np.stack([datagen.iou_targets(B, rank=r, batch_idx=batch_idx) for r in range(N)])
    return f, g


def pem_oracle_with_gpu_decisions(orc, s, l, f, p_pem, g):
    ref = orc.pem_fwd_bwd(f, p_pem, g, kink_tau=KINK_TAU_PEM, kinks_cap=1 << 20)
    gdec = s.pem_relu_decisions(l).cpu().numpy()
    diff = np.nonzero(gdec != ref["decisions"])[0]
    if diff.size == 0:
        return ref
    assert np.all(np.isin(diff, ref["kinks"])), "PEM ReLU decision differs outside the ambiguity band"
    return orc.pem_fwd_bwd(f, p_pem, g, flips=diff)


def test_num_params(tem):
    s, _ = pem_session(tem, 1, 2)
    assert s.K == datagen.num_params() + datagen.pem_num_params() == 1420804
    s.close()


@pytest.mark.parametrize("prec", [0, 1])
def test_pem_compute_single_rank(tem, orc, prec):
    B, lam = 4, (2.0, 1.0, 1.0)
    s, p = pem_session(tem, 1, B, prec, lam=lam)
    s.pem_record_decisions()
    x, lab = make_inputs(1, B, prec)
    f, g = pem_inputs(1, B)
    tl, pl = s.compute_pem(to_dev_x(x, prec), torch.from_numpy(lab).cuda(), torch.from_numpy(f).cuda(),
                           torch.from_numpy(g).cuda())
    assert s.sync()[0] == 0
    grad = s.local_grad(0).cpu().numpy()
    Kt = datagen.num_params()
    # TEM part: unchanged contract
    ref = oracle_with_gpu_decisions(orc, s, 0, x[0], p[:Kt], lab[0], lam, prec)
    check_tensors(orc, grad[:Kt], s.logits(0).cpu().numpy(), tl[0].cpu().numpy(), ref, TOL[prec])
    # PEM part: fp32 on both precisions
    pref = pem_oracle_with_gpu_decisions(orc, s, 0, f[0].reshape(B * P, F), p[Kt:], g[0].ravel())
    for name, sl in orc.pem_param_slices(F, H).items():
        e = rel_err(grad[Kt:Kt + datagen.pem_num_params()][sl], pref["grad"][sl])
        assert e <= TOL[0], (name, e)
    assert abs(float(pl[0]) - pref["loss"]) <= TOL[0] * pref["loss"]
    s.close()


@pytest.mark.parametrize("N,B", [(2, 2), (3, 1)])
def test_pem_joint_step_emulated(tem, orc, N, B):
    """Joint step on N emulated ranks: every rank's params after the fused ring + SGD equal the
    oracle's ring replay on the GPU's own concatenated local gradients, bit for bit."""
    lr = 0.05
    s, p = pem_session(tem, N, B, lr=lr)
    x, lab = make_inputs(N, B, 0)
    f, g = pem_inputs(N, B)
    w0 = s.params(0).cpu().numpy().copy()
    s.step_pem(to_dev_x(x, 0), torch.from_numpy(lab).cuda(), torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda())
    assert s.sync()[0] == 0
    grads = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
    expect = orc.ring_sgd(grads, w0, lr)
    for r in range(N):
        assert np.array_equal(s.params(r).cpu().numpy(), expect[r]), r
    s.close()


def test_pem_step_matches_compute_plus_update(tem, orc):
    """N = 1 graph-replayed joint steps (PEM on the side stream, fused split-K reduction in the
    update): the update equals the oracle SGD on the local gradient, bitwise, every step."""
    B, lr = 8, 0.05
    s, p = pem_session(tem, 1, B, lr=lr)
    x, lab = make_inputs(1, B, 0, batch_idx=2)
    f, g = pem_inputs(1, B, batch_idx=2)
    xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
    fd, gd = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    for _ in range(3):
        w0 = s.params(0).cpu().numpy().copy()
        s.step_pem(xd, ld, fd, gd)
        assert s.sync()[0] == 0
        grad = s.local_grad(0).cpu().numpy()
        assert np.array_equal(s.params(0).cpu().numpy(), orc.ring_sgd(grad[None, :], w0, lr)[0])
    s.close()


def test_tem_only_calls_rejected_on_pem_config(tem):
    s, _ = pem_session(tem, 1, 2)
    x, lab = make_inputs(1, 2, 0)
    with pytest.raises(tem.TemError):
        s.step(to_dev_x(x, 0), torch.from_numpy(lab).cuda())
    s.close()


def test_pem_bench_config_steps(tem, orc):
    """The configs[4] call bench.py times (B = 16 videos x 128 proposals, fp32, N = 1, graph-
    replayed tem_step_pem; the fp32 backward runs as the persistent bwd_kernel at this size):
    per step, the TEM tensors and the PEM tensors against their oracles at that step's weights,
    and the new weights bitwise equal to the oracle's SGD on the GPU's own gradient."""
    B, lr, lam = 16, 0.05, (2.0, 1.0, 1.0)
    s, p = pem_session(tem, 1, B, lr=lr, lam=lam)
    s.pem_record_decisions()
    Kt = datagen.num_params()
    for it in range(2):
        x, lab = make_inputs(1, B, 0, batch_idx=it)
        f, g = pem_inputs(1, B, batch_idx=it)
        w0 = s.params(0).cpu().numpy().copy()
        tl, pl = s.step_pem(to_dev_x(x, 0), torch.from_numpy(lab).cuda(), torch.from_numpy(f).cuda(),
                            torch.from_numpy(g).cuda())
        assert s.sync()[0] == 0
        grad = s.local_grad(0).cpu().numpy().copy()
        ref = oracle_with_gpu_decisions(orc, s, 0, x[0], w0[:Kt], lab[0], lam, 0)
        check_tensors(orc, grad[:Kt], s.logits(0).cpu().numpy(), tl[0].cpu().numpy(), ref, TOL[0])
        pref = pem_oracle_with_gpu_decisions(orc, s, 0, f[0].reshape(B * P, F), w0[Kt:s.K], g[0].ravel())
        for name, sl in orc.pem_param_slices(F, H).items():
            e = rel_err(grad[Kt:Kt + datagen.pem_num_params()][sl], pref["grad"][sl])
            assert e <= TOL[0], (it, name, e)
        assert abs(float(pl[0]) - pref["loss"]) <= TOL[0] * pref["loss"]
        assert np.array_equal(s.params(0).cpu().numpy(), orc.ring_sgd(grad[None, :], w0, lr)[0]), it
    s.close()
