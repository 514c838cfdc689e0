"""GPU parity of the PGM kernel (tem_pgm, reading R24) against the PGM
oracle: candidate / ranking decisions bit-exact (count, ts, te), BSP features and IoU targets
within 2e-5 absolute (fp32 kernel vs fp64 oracle, reading R24)."""
import numpy as np
import pytest
import torch

import datagen
from test_gpu_parity import tem  # noqa: F401

pytestmark = pytest.mark.gpu
TOL = 2e-5


def run(tem, prob, gt, n_gt, P):
    out = tem.pgm(torch.from_numpy(prob).cuda(), torch.from_numpy(gt).cuda(), torch.from_numpy(n_gt).cuda(), P)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def check(orc, got, prob, gt, n_gt, P):
    ref = orc.pgm(prob, gt, n_gt, P)
    assert np.array_equal(got["count"], ref["count"])
    assert np.array_equal(got["ts"], ref["ts"])
    assert np.array_equal(got["te"], ref["te"])
    assert np.abs(got["features"] - ref["features"]).max() <= TOL
    assert np.abs(got["iou"] - ref["iou"]).max() <= TOL
    return ref


@pytest.mark.parametrize("batch_idx", [0, 1])
def test_pgm_tem_shaped_inputs(tem, orc, batch_idx):
    """configs[4]'s shape: B = 16 videos, T = 100, P = 128, the labels' ground truth."""
    B, P = 16, datagen.PEM_P
    prob = datagen.tem_probabilities(B, batch_idx=batch_idx)
    gt, n = datagen.instances(B, batch_idx=batch_idx)
    ref = check(orc, run(tem, prob, gt, n, P), prob, gt, n, P)
    assert ref["count"].min() > 0


@pytest.mark.parametrize("T,P", [(1, 4), (2, 4), (5, 64), (37, 7), (100, 4096), (128, 128)])
def test_pgm_random_sequences(tem, orc, T, P):
    """U(0, 1) sequences (many local peaks: up to ~T/3 candidates per side), ragged T, P below
    and far above the number of proposals."""
    rng = np.random.default_rng(T * 31 + P)
    B = 5
    prob = rng.random((B, 3, T), dtype=np.float32)
    gt = (np.sort(rng.random((B, 4, 2)), axis=2) * T).astype(np.float32)
    n = rng.integers(0, 5, B).astype(np.int32)
    check(orc, run(tem, prob, gt, n, P), prob, gt, n, P)


def test_pgm_ties_and_degenerate_videos(tem, orc):
    """Equal scores (ordered by start then end), constant sequences (every t is a candidate),
    all-zero sequences (no candidate, count 0) and a single peak."""
    T, P = 20, 64
    prob = np.zeros((4, 3, T), np.float32)
    prob[0, 1, ::4] = 0.5
    prob[0, 2, 2::4] = 0.5
    prob[0, 0] = np.linspace(0, 1, T)
    prob[1] = 0.3
    prob[3, 1, 5] = 1.0
    prob[3, 2, 9] = 1.0
    prob[3, 0, 4:11] = 0.7
    gt = np.array([[[2.0, 9.0]]] * 4, np.float32)
    n = np.array([1, 1, 0, 1], np.int32)
    got = run(tem, prob, gt, n, P)
    ref = check(orc, got, prob, gt, n, P)
    assert got["count"][2] == 0 and np.all(got["ts"][2] == -1)
    assert got["count"][3] == 1 and (got["ts"][3][0], got["te"][3][0]) == (5, 9)
    assert ref["count"][1] == T * (T - 1) // 2 or ref["count"][1] == P


# ------------------------------------------------------------------ PGM-fed joint step
def pgm_session(tem, N, B, lr=0.05, lam=(2.0, 1.0, 1.0), pgm_gt_max=datagen.GT_MAX, P=datagen.PEM_P):
    sc = tem.SessionConfig(world_size=N, rank=0, local_ranks=N, batch_per_rank=B, precision=0, lr=lr,
                           loss_weight=lam, pem_proposals=P, pem_features=32, pem_hidden=512, pgm_gt_max=pgm_gt_max)
    p = np.concatenate([datagen.init_params(), datagen.init_pem_params()])
    return tem.TemSession(sc, p), p


def gt_inputs(N, B, batch_idx=0):
    segs, cnts = zip(*(datagen.instances(B, rank=r, batch_idx=batch_idx) for r in range(N)))
    return torch.from_numpy(np.stack(segs)).cuda(), torch.from_numpy(np.stack(cnts)).cuda()


def test_pgm_fed_step_composition(tem, orc):
    """tem_compute_pgm = TEM compute, PGM on sigmoid(z), PEM on PGM's features:
    * the step's probabilities are sigmoid(z) of its own logits (fp32 rounding),
    * its PGM outputs equal tem_pgm on those probabilities bitwise,
    * its PEM gradient / loss equal the caller-fed PEM path (oracle-pinned in test_gpu_pem)
      given those features and IoU targets, bitwise, and match the PEM oracle (1e-4),
    * its TEM gradient equals a TEM-only session's bitwise."""
    from test_gpu_parity import make_inputs, to_dev_x
    from test_gpu_pem import KINK_TAU_PEM, pem_session
    B, P = 4, datagen.PEM_P
    x, lab = make_inputs(1, B, 0, batch_idx=5)
    xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
    gt, n = gt_inputs(1, B, batch_idx=5)
    s, p = pgm_session(tem, 1, B)
    tl, pl = s.compute_pgm(xd, ld, gt, n)
    assert s.sync()[0] == 0
    z = s.logits(0).cpu().numpy().astype(np.float64)           # [B][T][3]
    prob = s.debug_buffer("pgm_prob").view(B, 3, -1).cpu().numpy()
    sig = 1.0 / (1.0 + np.exp(-z.transpose(0, 2, 1)))
    assert np.abs(prob - sig).max() <= 2.0 ** -22
    step_out = {k: s.debug_buffer("pgm_" + k).cpu().numpy() for k in ("feat", "iou", "ts", "te", "count")}
    alone = tem.pgm(torch.from_numpy(prob).cuda(), gt[0], n[0], P)
    torch.cuda.synchronize()
    assert np.array_equal(step_out["count"], alone["count"].cpu().numpy())
    assert np.array_equal(step_out["ts"].reshape(B, P), alone["ts"].cpu().numpy())
    assert np.array_equal(step_out["te"].reshape(B, P), alone["te"].cpu().numpy())
    assert np.array_equal(step_out["feat"].reshape(B, P, 32), alone["features"].cpu().numpy())
    assert np.array_equal(step_out["iou"].reshape(B, P), alone["iou"].cpu().numpy())
    grad = s.local_grad(0).cpu().numpy().copy()
    Kt = datagen.num_params()
    s.close()
    # caller-fed PEM on the same features / targets
    s2, _ = pem_session(tem, 1, B)
    feat = torch.from_numpy(step_out["feat"].reshape(1, B, P, 32)).cuda()
    iou = torch.from_numpy(step_out["iou"].reshape(1, B, P)).cuda()
    tl2, pl2 = s2.compute_pem(xd, ld, feat, iou)
    assert s2.sync()[0] == 0
    grad2 = s2.local_grad(0).cpu().numpy()
    assert np.array_equal(grad, grad2)
    assert float(pl[0]) == float(pl2[0]) and np.array_equal(tl.cpu().numpy(), tl2.cpu().numpy())
    s2.close()
    # PEM oracle on those inputs (decisions within the ambiguity band as in test_gpu_pem)
    ref = orc.pem_fwd_bwd(step_out["feat"].reshape(B * P, 32), p[Kt:], step_out["iou"].ravel(), kink_tau=KINK_TAU_PEM)
    e = np.abs(grad[Kt:Kt + datagen.pem_num_params()] - ref["grad"]).max() / np.abs(ref["grad"]).max()
    assert e <= 1e-3  # (ReLU decisions inside the band may differ; the bitwise check above is the contract)


@pytest.mark.parametrize("N,B", [(1, 8), (1, 16), (2, 2), (3, 1)])
def test_pgm_fed_steps_exchange(tem, orc, N, B):
    """Graph-replayed PGM-fed steps: every rank's params after each step equal the oracle's ring
    replay (mean + SGD) of the GPU's concatenated [TEM | PEM] local gradients, bitwise."""
    from test_gpu_parity import make_inputs, to_dev_x
    lr = 0.05
    s, _ = pgm_session(tem, N, B, lr=lr)
    x, lab = make_inputs(N, B, 0, batch_idx=7)
    xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
    gt, n = gt_inputs(N, B, batch_idx=7)
    for it in range(2):
        w0 = s.params(0).cpu().numpy().copy()
        s.step_pgm(xd, ld, gt, n)
        assert s.sync()[0] == 0
        grads = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
        expect = orc.ring_sgd(grads, w0, lr)
        for r in range(N):
            assert np.array_equal(s.params(r).cpu().numpy(), expect[r]), (it, r)
        assert int(s.debug_buffer("pgm_count").cpu().numpy().min()) > 0
    s.close()
