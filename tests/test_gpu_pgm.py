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
