"""PGM oracle: BSN's proposal generation -- candidate boundaries, proposals and their
Boundary-Sensitive Proposal (BSP) features -- as the data path that feeds PEM (SURVEY 8(f)
NEXT #4; A5; reading R24 in DESIGN.md).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and bench.py's
reference legs, never by the product package.  Plain numpy / Python loops, written step by
step in the order of reading R24; integer decisions (candidate flags, the fp32 score and
the ranking) are taken in fp32, as the kernel takes them, and the BSP features and IoU
targets are computed in fp64.

The paper names the stage only ("generating a possibilities sequences and selecting
candidate proposals"; Fig. 1b); its steps follow BSN (Lin et al., 2018), the
paper's cited method, as stated in reading R24:
  1. candidates: t is a start candidate iff p_s[t] > fl32(0.9 * max p_s) or p_s has a strict
     local peak at t (0 < t < T-1, p_s[t] > p_s[t-1] and p_s[t] > p_s[t+1]); same for ends;
  2. proposals: every (t_s, t_e) of a start and an end candidate with t_s < t_e, score
     c = fl32(p_s[t_s] * p_e[t_e]);
  3. the first P proposals by (c descending, t_s ascending, t_e ascending);
  4. BSP feature (32): with d = t_e - t_s, n points at x_k = a + (k + 1/2)(b - a)/n of the
     actionness sequence p_a linearly interpolated (zero outside [0, T-1]) over the start
     region [t_s - d/5, t_s + d/5] (8), the proposal [t_s, t_e] (16) and the end region
     [t_e - d/5, t_e + d/5] (8);
  5. IoU target: max over ground-truth instances [g_s, g_e] (snippet units) of the IoU with
     the proposal's span [t_s + 1/2, t_e + 1/2] (snippet centres); 0 without instances.
"""
from __future__ import annotations

import numpy as np

N_START, N_CENTER, N_END = 8, 16, 8
F_BSP = N_START + N_CENTER + N_END


def candidates(p: np.ndarray) -> list[int]:
    """Step 1 for one probability sequence (fp32 comparisons)."""
    p = np.asarray(p, np.float32)
    T = p.size
    thr = np.float32(np.float32(0.9) * p.max()) if T else np.float32(0)
    out = []
    for t in range(T):
        high = p[t] > thr
        peak = 0 < t < T - 1 and p[t] > p[t - 1] and p[t] > p[t + 1]
        if high or peak:
            out.append(t)
    return out


def interp(pa: np.ndarray, x: float) -> float:
    """Step 4's sampling: linear interpolation of pa at x, pa zero outside [0, T-1]."""
    T = pa.size
    i = int(np.floor(x))
    f = x - i

    def at(j):
        return float(pa[j]) if 0 <= j < T else 0.0
    return (1.0 - f) * at(i) + f * at(i + 1)


def bsp_feature(pa: np.ndarray, ts: int, te: int) -> np.ndarray:
    d = float(te - ts)
    regions = ((ts - d / 5.0, ts + d / 5.0, N_START), (float(ts), float(te), N_CENTER),
               (te - d / 5.0, te + d / 5.0, N_END))
    f = []
    for a, b, n in regions:
        for k in range(n):
            f.append(interp(pa, a + (k + 0.5) * (b - a) / n))
    return np.asarray(f, np.float64)


def iou(ts: int, te: int, gt: np.ndarray, n_gt: int) -> float:
    s1, e1 = ts + 0.5, te + 0.5
    best = 0.0
    for g in range(n_gt):
        s2, e2 = float(gt[g][0]), float(gt[g][1])
        inter = max(0.0, min(e1, e2) - max(s1, s2))
        union = (e1 - s1) + (e2 - s2) - inter
        if union > 0:
            best = max(best, inter / union)
    return best


def pgm_video(prob: np.ndarray, gt: np.ndarray, n_gt: int, P: int):
    """One video: prob [3][T] fp32 (0 actionness, 1 start, 2 end; R4).  Returns
    (count, ts [P] int32 (-1 unused), te [P], features [P][32] f64, iou [P] f64)."""
    prob = np.asarray(prob, np.float32)
    pa, ps, pe = prob[0], prob[1], prob[2]
    S, E = candidates(ps), candidates(pe)
    props = []
    for a in S:
        for b in E:
            if a < b:
                props.append((np.float32(ps[a] * pe[b]), a, b))
    props.sort(key=lambda q: (-float(q[0]), q[1], q[2]))
    props = props[:P]
    n = len(props)
    ts = np.full(P, -1, np.int32)
    te = np.full(P, -1, np.int32)
    feat = np.zeros((P, F_BSP), np.float64)
    tgt = np.zeros(P, np.float64)
    for i, (_, a, b) in enumerate(props):
        ts[i], te[i] = a, b
        feat[i] = bsp_feature(pa, a, b)
        tgt[i] = iou(a, b, gt, n_gt)
    return n, ts, te, feat, tgt


def pgm(prob: np.ndarray, gt: np.ndarray, n_gt: np.ndarray, P: int):
    """Batch of videos: prob [B][3][T], gt [B][G][2], n_gt [B].  Returns dict of arrays
    count [B], ts/te [B][P], features [B][P][32], iou [B][P]."""
    B = prob.shape[0]
    out = {"count": np.zeros(B, np.int32), "ts": np.zeros((B, P), np.int32), "te": np.zeros((B, P), np.int32),
           "features": np.zeros((B, P, F_BSP)), "iou": np.zeros((B, P))}
    for v in range(B):
        n, ts, te, f, g = pgm_video(prob[v], gt[v], int(n_gt[v]), P)
        out["count"][v], out["ts"][v], out["te"][v], out["features"][v], out["iou"][v] = n, ts, te, f, g
    return out
