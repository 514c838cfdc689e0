"""The paper's training-time metrics.

Host-side reporting logic; no GPU work.  Units are whatever the
samples are in (the paper never states them, P:170 -- reading R15).

  Eq. (1), PS:  t = T/n + C*n       + P
  Eq. (2), ring:  t = T/n + C*n/(n-1) + P   (fitted as printed -- reading R14:
        the text's t2 ~ (n-1)/n = 1 - 1/n is collinear with {1/n, 1} and cannot
        identify three parameters)
  speed ratio:      t0 / t
  t = t1 + t2 + t3 decomposition.
"""
from __future__ import annotations

from dataclasses import dataclass, asdict
from typing import Iterable, Sequence

import numpy as np

PS, RING = "ps", "ring"


@dataclass
class CostModel:
    kind: str
    T: float
    C: float
    P: float

    @property
    def valid(self) -> bool:  # P:212 "C=-3.8<0, which is obviously unreasonable"
        return self.T > 0 and self.C >= 0 and self.P >= 0


@dataclass
class FitReport:
    model: CostModel
    residual_rms: float
    residuals: list
    valid: bool

    def to_json(self) -> dict:
        d = asdict(self)
        d["model"] = asdict(self.model)
        return d


def comm_basis(kind: str, n):
    n = np.asarray(n, dtype=np.float64)
    if kind == PS:
        return n
    if kind == RING:
        if np.any(n <= 1):
            raise ValueError("Eq. (2) is singular at n = 1 (defined for n = 2, 3, ...)")
        return n / (n - 1.0)
    raise ValueError(f"unknown architecture {kind!r}")


def predict_time(model: CostModel, n):
    """Eq. (1) / Eq. (2)."""
    n = np.asarray(n, dtype=np.float64)
    return model.T / n + model.C * comm_basis(model.kind, n) + model.P


def fit_cost_model(samples: Iterable[tuple[float, float]], kind: str) -> FitReport:
    """OLS over the basis {1/n, g(n), 1} ("use the number of GPUs ... as the
    independent variable and the training time as the dependent variable to fit")."""
    s = np.asarray(list(samples), dtype=np.float64)
    if s.ndim != 2 or s.shape[1] != 2:
        raise ValueError("samples must be (n, t) pairs")
    n, t = s[:, 0], s[:, 1]
    if np.any(n < 2):
        raise ValueError("fit samples need n >= 2 (n = 1 is only t0 for the speed ratio)")
    if len(np.unique(n)) < 3:
        raise ValueError("need >= 3 distinct n for 3 unknowns")
    A = np.stack([1.0 / n, comm_basis(kind, n), np.ones_like(n)], axis=1)
    Q, R = np.linalg.qr(A)
    coef = np.linalg.solve(R, Q.T @ t)
    res = t - A @ coef
    m = CostModel(kind, float(coef[0]), float(coef[1]), float(coef[2]))
    return FitReport(m, float(np.sqrt(np.mean(res ** 2))), res.tolist(), m.valid)


def speed_ratio(t0: float, t: float) -> float:
    """Speed ratio = t0 / t."""
    if t0 <= 0 or t <= 0:
        raise ValueError("times must be positive")
    return t0 / t


def crossover(ps: CostModel, ring: CostModel, n_max: int = 64):
    """Smallest n in [2, n_max] with ring time <= PS time, else None."""
    for n in range(2, n_max + 1):
        if predict_time(ring, n) <= predict_time(ps, n):
            return n
    return None


def ring_bytes_per_rank(K_pad: int, N: int, elem_bytes: int = 4) -> int:
    """every GPU sends K/n per round for n-1 scatter + n-1 gather rounds."""
    return 0 if N <= 1 else 2 * (K_pad // N) * (N - 1) * elem_bytes


def ps_server_bytes(K: int, N: int, elem_bytes: int = 4) -> int:
    """server volume N*M (uplink)."""
    return N * K * elem_bytes


def busbw(nbytes: float, seconds: float, N: int) -> float:
    """Allreduce bus bandwidth: algbw * 2(N-1)/N (NCCL convention)."""
    if N <= 1:
        return 0.0
    return nbytes / seconds * 2.0 * (N - 1) / N


# The paper's fitted parameters, context only.
PAPER_PS = CostModel(PS, 4223.8, 12.1, 290.8)
PAPER_RING = CostModel(RING, 4400.1, 59.6, 363.5)
