"""Seeded synthetic inputs for the BSN-TEM data-parallel step.

This is the ONLY module shared by the oracle side (tests) and the product side
(bench.py / smoke).  It holds none of the method's arithmetic: no convolution,
no loss, no reduction -- only random draws with the shapes, distributions and
structure of the paper's workload (ActivityNet-1.3 two-stream snippet features,
P:181-186; BSN-style temporal labels, reading R13).

Recipe:
  * features x ~ N(0, 1) i.i.d. float32, [B][T=100][Cin=400] (400 = 200 spatial
    + 200 temporal two-stream dims), from numpy.random.default_rng(seed)
    with seed = 1906064960 + 1000*rank + batch_idx.
  * labels [B][3][T] in [0, 1]: per video 1-3 action instances (uniform), length
    fraction U(0.05, 0.5), start U(0, 1 - len).  Channel 0 (actionness) =
    max over instances of the IoP of snippet [t/T, (t+1)/T] with the instance;
    channels 1/2 (start/end) = the same with a region of width
    max(0.1*len, 1/T) centred on the instance boundary.
  * parameters: torch-default-style U(-1/sqrt(fan_in), +1/sqrt(fan_in)) for each
    weight and bias, fan_in = Cin*3, C*3, C for conv1/2/3, flat order
    [W1, b1, W2, b2, W3, b3], zero-padded to any requested length.
  * PEM (BASELINE configs[4], reading R19): P = 128 proposals per video; BSP features
    [B][P][32] ~ U(0, 1) (BSN's BSP feature samples probability sequences, values in
    [0, 1]); IoU targets [B][P] = U(0, 1)^2 (skewed to low overlap, as dense proposal sets
    are); PEM parameters [W1p (512 x 32), b1p, w2p, b2p] ~ U(+-1/sqrt(fan_in)), fan_in 32, 512.
  * PGM (reading R24): the labels' instances in snippet units (instances()), and TEM-shaped
    probability sequences 0.05 + 0.8 * labels + U(0, 0.1) (tem_probabilities()).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 1906064960
T_DEFAULT, CIN_DEFAULT, C_DEFAULT, CO_DEFAULT = 100, 400, 512, 3
PEM_P, PEM_F, PEM_H = 128, 32, 512


def batch_seed(rank: int, batch_idx: int) -> int:
    return SEED_BASE + 1000 * int(rank) + int(batch_idx)


def features(B: int, T: int = T_DEFAULT, Cin: int = CIN_DEFAULT, *, rank: int = 0,
             batch_idx: int = 0) -> np.ndarray:
    rng = np.random.default_rng(batch_seed(rank, batch_idx))
    return rng.standard_normal((B, T, Cin), dtype=np.float32)


def _overlap_over_snippet(t0, t1, a, b):
    """Length of [t0,t1] ∩ [a,b] divided by the snippet length t1 - t0."""
    inter = np.clip(np.minimum(t1, b) - np.maximum(t0, a), 0.0, None)
    return inter / (t1 - t0)


def _instance_draws(B: int, rank: int, batch_idx: int):
    """Per video the list of (start, end, length) action instances in [0, 1] (labels' recipe)."""
    rng = np.random.default_rng(batch_seed(rank, batch_idx) + 7_000_000)
    out = []
    for _ in range(B):
        n_inst = int(rng.integers(1, 4))
        segs = []
        for _ in range(n_inst):
            ln = rng.uniform(0.05, 0.5)
            s = rng.uniform(0.0, 1.0 - ln)
            segs.append((s, s + ln, ln))
        out.append(segs)
    return out


GT_MAX = 3  # instances per video (labels' recipe draws 1-3)


def instances(B: int, T: int = T_DEFAULT, *, rank: int = 0, batch_idx: int = 0):
    """The ground-truth instances behind labels(B, T, rank, batch_idx), in snippet units
    (time * T): seg [B][GT_MAX][2] float32 (unused rows 0), count [B] int32."""
    seg = np.zeros((B, GT_MAX, 2), np.float32)
    cnt = np.zeros(B, np.int32)
    for v, segs in enumerate(_instance_draws(B, rank, batch_idx)):
        cnt[v] = len(segs)
        for i, (s, e, _) in enumerate(segs):
            seg[v, i] = (s * T, e * T)
    return seg, cnt


def tem_probabilities(B: int, T: int = T_DEFAULT, *, rank: int = 0, batch_idx: int = 0) -> np.ndarray:
    """TEM-output-shaped probability sequences [B][3][T] (actionness, start, end) for the PGM
    tests / bench: the labels of the same batch, scaled into [0.05, 0.85], plus U(0, 0.1)
    noise (a partly trained TEM: peaks near the true boundaries, spurious local maxima)."""
    lab = labels(B, T, rank=rank, batch_idx=batch_idx)
    rng = np.random.default_rng(batch_seed(rank, batch_idx) + 17_000_000)
    return (0.05 + 0.8 * lab + 0.1 * rng.random(lab.shape)).astype(np.float32)


def labels(B: int, T: int = T_DEFAULT, *, rank: int = 0, batch_idx: int = 0) -> np.ndarray:
    out = np.zeros((B, 3, T), dtype=np.float32)
    t0 = np.arange(T, dtype=np.float64) / T
    t1 = (np.arange(T, dtype=np.float64) + 1.0) / T
    for v, segs in enumerate(_instance_draws(B, rank, batch_idx)):
        for s, e, ln in segs:
            w = max(0.1 * ln, 1.0 / T)
            out[v, 0] = np.maximum(out[v, 0], _overlap_over_snippet(t0, t1, s, e))
            out[v, 1] = np.maximum(out[v, 1], _overlap_over_snippet(t0, t1, s - w / 2, s + w / 2))
            out[v, 2] = np.maximum(out[v, 2], _overlap_over_snippet(t0, t1, e - w / 2, e + w / 2))
    return out


def num_params(Cin: int = CIN_DEFAULT, C: int = C_DEFAULT, Co: int = CO_DEFAULT) -> int:
    return C * 3 * Cin + C + C * 3 * C + C + Co * C + Co


def init_params(Cin: int = CIN_DEFAULT, C: int = C_DEFAULT, Co: int = CO_DEFAULT, *,
                seed: int = SEED_BASE, pad_to: int | None = None) -> np.ndarray:
    rng = np.random.default_rng(seed + 99)
    parts = []
    for fan_in, shapes in ((Cin * 3, [(C * 3 * Cin,), (C,)]),
                           (C * 3, [(C * 3 * C,), (C,)]),
                           (C, [(Co * C,), (Co,)])):
        bound = 1.0 / np.sqrt(fan_in)
        for shp in shapes:
            parts.append(rng.uniform(-bound, bound, size=shp).astype(np.float32))
    flat = np.concatenate(parts)
    if pad_to is not None:
        assert pad_to >= flat.size
        flat = np.concatenate([flat, np.zeros(pad_to - flat.size, np.float32)])
    return flat


def bsp_features(B: int, P: int = PEM_P, F: int = PEM_F, *, rank: int = 0, batch_idx: int = 0) -> np.ndarray:
    rng = np.random.default_rng(batch_seed(rank, batch_idx) + 11_000_000)
    return rng.random((B, P, F), dtype=np.float32)


def iou_targets(B: int, P: int = PEM_P, *, rank: int = 0, batch_idx: int = 0) -> np.ndarray:
    rng = np.random.default_rng(batch_seed(rank, batch_idx) + 13_000_000)
    u = rng.random((B, P), dtype=np.float32)
    return (u * u).astype(np.float32)


def pem_num_params(F: int = PEM_F, H: int = PEM_H) -> int:
    return H * F + 2 * H + 1


def init_pem_params(F: int = PEM_F, H: int = PEM_H, *, seed: int = SEED_BASE) -> np.ndarray:
    rng = np.random.default_rng(seed + 199)
    b1 = 1.0 / np.sqrt(F)
    b2 = 1.0 / np.sqrt(H)
    parts = [rng.uniform(-b1, b1, size=H * F), rng.uniform(-b1, b1, size=H),
             rng.uniform(-b2, b2, size=H), rng.uniform(-b2, b2, size=1)]
    return np.concatenate(parts).astype(np.float32)


def gradients(N: int, K: int, *, seed: int = SEED_BASE, scale: float = 1e-3) -> np.ndarray:
    """Random per-rank gradient buffers [N][K] float32 (for allreduce-only tests/bench)."""
    rng = np.random.default_rng(seed + 5)
    return (rng.standard_normal((N, K), dtype=np.float32) * np.float32(scale)).astype(np.float32)


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) and return uint16 bit patterns.  Used to hand the
    c3 path its bf16 features (x is stored as bf16 once, at generation time)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)
