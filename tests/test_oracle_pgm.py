"""Pins of the PGM oracle (oracle/proposals.py, reading R24) against hand-derived values.

Every expected value below is worked out in the comments from the definitions of reading
R24 (candidates, ranking, BSP sampling, IoU), not by calling the oracle."""
import numpy as np
import pytest

import oracle.proposals as pgm


def f32(a):
    return np.asarray(a, np.float32)


def test_candidates_threshold_and_strict_peaks():
    # p_s: max 0.6 -> threshold fl32(0.9 * 0.6) = 0.54: t = 7 is "high"; strict interior peaks
    # at t = 1 (0.5 > 0.1, 0.2) and t = 4 (0.3 > 0.2, 0.1); t = 3 is a plateau (0.2 = 0.2) and
    # t = 0 an endpoint below the threshold.
    assert pgm.candidates(f32([0.1, 0.5, 0.2, 0.2, 0.3, 0.1, 0.05, 0.6])) == [1, 4, 7]
    # p_e: threshold 0.81 keeps t = 6 only (0.8 <= 0.81); peaks at 3 and 6; t = 1 ties 0.1 = 0.1
    assert pgm.candidates(f32([0.0, 0.1, 0.1, 0.4, 0.2, 0.3, 0.9, 0.8])) == [3, 6]
    # all equal and positive: every t exceeds 0.9 * max
    assert pgm.candidates(f32([0.5] * 5)) == [0, 1, 2, 3, 4]
    # all zero: nothing exceeds 0, no strict peak
    assert pgm.candidates(f32([0.0] * 5)) == []


def test_proposals_ranked_by_score_then_boundaries():
    T = 8
    prob = np.zeros((3, T), np.float32)
    prob[1] = [0.1, 0.5, 0.2, 0.2, 0.3, 0.1, 0.05, 0.6]  # S = {1, 4, 7}
    prob[2] = [0.0, 0.1, 0.1, 0.4, 0.2, 0.3, 0.9, 0.8]  # E = {3, 6}
    # pairs t_s < t_e: (1,3) c = 0.5*0.4 = 0.2, (1,6) 0.45, (4,6) 0.27; start 7 has no end after it
    n, ts, te, _, _ = pgm.pgm_video(prob, np.zeros((0, 2)), 0, 5)
    assert n == 3
    assert ts.tolist() == [1, 4, 1, -1, -1] and te.tolist() == [6, 6, 3, -1, -1]
    n, ts, te, _, _ = pgm.pgm_video(prob, np.zeros((0, 2)), 0, 2)  # P truncates
    assert n == 2 and ts.tolist() == [1, 4] and te.tolist() == [6, 6]


def test_equal_scores_ordered_by_start_then_end():
    prob = np.zeros((3, 5), np.float32)
    prob[1] = [0, 0.5, 0, 0.5, 0]  # S = {1, 3}
    prob[2] = [0, 0, 0.5, 0, 0.5]  # E = {2, 4}
    # (1,2), (1,4), (3,4) all score 0.25
    n, ts, te, _, _ = pgm.pgm_video(prob, np.zeros((0, 2)), 0, 8)
    assert n == 3 and ts[:3].tolist() == [1, 1, 3] and te[:3].tolist() == [2, 4, 4]


def test_bsp_feature_of_a_linear_sequence():
    # p_a[t] = 0.1 + t/10 on [0, T-1]: linear interpolation reproduces the line, so every
    # sample inside [0, T-1] equals 0.1 + x/10 at its position x.
    T = 8
    pa = f32(0.1 + np.arange(T) / 10)
    # proposal (1, 6), d = 5: start region [0, 2], 8 midpoints 0.125, 0.375, ..., 1.875;
    # centre [1, 6], 16 midpoints 1 + (k + 1/2) 5/16; end region [5, 7], midpoints 5.125 ... 6.875
    xs = ([2 * (k + 0.5) / 8 for k in range(8)] + [1 + (k + 0.5) * 5 / 16 for k in range(16)]
          + [5 + 2 * (k + 0.5) / 8 for k in range(8)])
    got = pgm.bsp_feature(pa, 1, 6)
    assert got.shape == (32,)
    np.testing.assert_allclose(got, 0.1 + np.asarray(xs) / 10, rtol=0, atol=1e-7)


def test_interpolation_is_zero_extended():
    pa = f32([0.1, 0.2, 0.3])
    # left of 0: between the virtual 0 at -1 and p[0] = 0.1 -> 0.1 (x + 1)
    assert pgm.interp(pa, -0.25) == pytest.approx(0.1 * 0.75, abs=1e-7)
    assert pgm.interp(pa, -1.5) == 0.0
    # right of T-1 = 2: between p[2] = 0.3 and the virtual 0 at 3 -> 0.3 (3 - x)
    assert pgm.interp(pa, 2.5) == pytest.approx(0.15, abs=1e-7)
    # integer positions hit the samples (float32 inputs, compare in float32)
    assert pgm.interp(pa, 1.0) == pytest.approx(float(np.float32(0.2)), abs=1e-7)


def test_iou_target():
    # proposal (1, 6) spans snippet centres [1.5, 6.5] (length 5)
    assert pgm.iou(1, 6, [[1.5, 6.5]], 1) == pytest.approx(1.0)
    assert pgm.iou(1, 6, [[6.5, 8.0]], 1) == 0.0          # touching
    # [4, 9]: intersection 2.5, union 5 + 5 - 2.5 = 7.5 -> 1/3; the max over instances is taken
    assert pgm.iou(1, 6, [[6.5, 8.0], [4.0, 9.0]], 2) == pytest.approx(1 / 3)
    assert pgm.iou(1, 6, [[4.0, 9.0]], 0) == 0.0          # no instances


def test_batch_shapes_and_padding():
    prob = np.zeros((2, 3, 6), np.float32)
    prob[0, 1] = [0, 1, 0, 0, 0, 0]
    prob[0, 2] = [0, 0, 0, 1, 0, 0]
    out = pgm.pgm(prob, np.zeros((2, 1, 2), np.float32), np.zeros(2, np.int32), 4)
    assert out["count"].tolist() == [1, 0]  # video 1: all-zero sequences give no candidates
    assert out["ts"][0].tolist() == [1, -1, -1, -1] and out["te"][0].tolist() == [3, -1, -1, -1]
    assert np.all(out["features"][1] == 0) and np.all(out["features"][0, 1:] == 0)
