"""Training-time metrics pinned to the paper's fitted values."""
import json
import os

import numpy as np
import pytest

from paper_1906_06496_b200 import metrics as M

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_predictions_at_n2():
    g = GOLD["predictions"]
    assert abs(M.predict_time(M.PAPER_PS, 2) - g["ps_n2"]) < 1e-9
    assert abs(M.predict_time(M.PAPER_RING, 2) - g["ring_n2"]) < 1e-9
    assert M.predict_time(M.CostModel(M.PS, 100, 0, 0), 4) == 25.0
    with pytest.raises(ValueError):
        M.predict_time(M.PAPER_RING, 1)


@pytest.mark.parametrize("model", [M.PAPER_PS, M.PAPER_RING])
def test_fit_recovery(model):
    ns = np.arange(2, 9)
    rep = M.fit_cost_model(zip(ns, M.predict_time(model, ns)), model.kind)
    for a, b in ((rep.model.T, model.T), (rep.model.C, model.C), (rep.model.P, model.P)):
        assert abs(a - b) <= 1e-6 * abs(b)
    assert rep.residual_rms < 1e-9 and rep.valid


def test_wrong_basis_has_residual():
    """fitting ring-model data with the PS basis leaves a residual.  (SURVEY 4 defect 1:
    on noiseless model data the fitted C is positive, so only the residual is asserted.)"""
    ns = np.arange(2, 9)
    rep = M.fit_cost_model(zip(ns, M.predict_time(M.PAPER_RING, ns)), M.PS)
    assert rep.residual_rms > 0.5


def test_crossover_and_asymptote():
    assert M.crossover(M.PAPER_PS, M.PAPER_RING, 64) == GOLD["crossover"]["n"]
    assert M.crossover(M.PAPER_PS, M.PAPER_PS.__class__(M.RING, 4223.8, 12.1, 290.8)) == 2
    assert M.crossover(M.CostModel(M.PS, 1, 0, 0), M.CostModel(M.RING, 1, 1e9, 0), 64) is None
    big = M.predict_time(M.PAPER_RING, 10 ** 6)
    assert abs(big - (M.PAPER_RING.P + M.PAPER_RING.C)) <= 0.01 * (M.PAPER_RING.P + M.PAPER_RING.C)


def test_volumes_and_ratio():
    v = GOLD["volume_examples"]
    for K, N, e in v["ring"]:
        assert M.ring_bytes_per_rank(K, N, elem_bytes=1) == e
    for K, N, e in v["ps_uplink"]:
        assert M.ps_server_bytes(K, N, elem_bytes=1) == e
    assert M.ring_bytes_per_rank(1000, 1) == 0
    assert M.speed_ratio(100, 50) == 2.0
    with pytest.raises(ValueError):
        M.speed_ratio(0, 1)


def test_fit_rejects_degenerate():
    with pytest.raises(ValueError):
        M.fit_cost_model([(2, 1.0), (2, 1.0), (3, 1.0)], M.PS)
    with pytest.raises(ValueError):
        M.fit_cost_model([(1, 1.0), (2, 1.0), (3, 1.0)], M.PS)
