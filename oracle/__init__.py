"""CPU oracle for the BSN-TEM data-parallel step and the paper's ring allreduce.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_1906_06496_b200`` never imports it, and
the two share no code.

The arithmetic lives in ``tem_oracle.cpp`` (plain C++, fp64 ground truth, fp32
ring replay, ``-ffp-contract=off``); this module only builds it with g++ and
marshals numpy arrays through ctypes.  Every function cites the passage it
follows in the C++ source.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tem_oracle.cpp")
_LIB = os.path.join(_HERE, "libtem_oracle.so")
_lock = threading.Lock()
_lib = None

SUM, MEAN = 0, 1


def build(force: bool = False) -> str:
    """Compile tem_oracle.cpp -> libtem_oracle.so (plain g++, no fast math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
            "-fno-unsafe-math-optimizations", "-shared", "-fPIC", _SRC, "-o", tmp,
        ])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            i64, i32, f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_float
            P = ctypes.c_void_p
            L.orc_kpad.restype = i64
            L.orc_kpad.argtypes = [i64, i32, i32]
            for fn in (L.orc_scatter_schedule, L.orc_gather_schedule):
                fn.restype = i32
                fn.argtypes = [i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
            L.orc_ring_allreduce_f32.restype = i32
            L.orc_ring_allreduce_f32.argtypes = [P, i32, i64, i32, P]
            L.orc_ring_sgd_f32.restype = i32
            L.orc_ring_sgd_f32.argtypes = [P, P, i32, i64, i32, f32]
            L.orc_ring_chain_f32.restype = i32
            L.orc_ring_chain_f32.argtypes = [P, i32, i64, i32, P]
            L.orc_ps_allreduce_f32.restype = i32
            L.orc_ps_allreduce_f32.argtypes = [P, i32, i64, i32, P]
            L.orc_bf16_bits.restype = ctypes.c_uint16
            L.orc_bf16_bits.argtypes = [f32]
            L.orc_tem_num_params.restype = i64
            L.orc_tem_num_params.argtypes = [i32, i32, i32]
            L.orc_tem_fwd_bwd.restype = i32
            L.orc_tem_fwd_bwd.argtypes = [i32, i32, i32, i32, i32, i32, P, P, P, P, P, P, P]
            L.orc_tem_fwd_bwd_ex.restype = i32
            L.orc_tem_fwd_bwd_ex.argtypes = [i32, i32, i32, i32, i32, i32, P, P, P, P, P, P, P,
                                             P, i64, ctypes.c_double, ctypes.c_double, P, i64, P, P]
            L.orc_ring_adam_f32.restype = i32
            L.orc_ring_adam_f32.argtypes = [P, P, P, P, P, i32, i64, f32, f32, f32, f32]
            L.orc_ring_momentum_f32.restype = i32
            L.orc_ring_momentum_f32.argtypes = [P, P, P, i32, i64, f32, f32]
            L.orc_pem_num_params.restype = i64
            L.orc_pem_num_params.argtypes = [i32, i32]
            L.orc_pem_fwd_bwd.restype = i32
            L.orc_pem_fwd_bwd.argtypes = [i32, i32, i32, P, P, P, P, P, P, P, i64, ctypes.c_double, P, i64,
                                          P, P]
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------- partition / schedules
def kpad(K: int, N: int, V: int = 4) -> int:
    """K_pad = roundup(K, N*V)."""
    r = lib().orc_kpad(K, N, V)
    if r < 0:
        raise ValueError("invalid partition arguments")
    return int(r)


def scatter_schedule(rank: int, N: int, rnd: int):
    """send (n-i)%N, receive (n-i-1)%N."""
    s, r = ctypes.c_int(), ctypes.c_int()
    if lib().orc_scatter_schedule(rank, N, rnd, ctypes.byref(s), ctypes.byref(r)):
        raise ValueError("round out of range")
    return s.value, r.value


def gather_schedule(rank: int, N: int, rnd: int):
    """P:152 with reading R10: send (n+1-k)%N, receive (n-k)%N."""
    s, r = ctypes.c_int(), ctypes.c_int()
    if lib().orc_gather_schedule(rank, N, rnd, ctypes.byref(s), ctypes.byref(r)):
        raise ValueError("round out of range")
    return s.value, r.value


# --------------------------------------------------------------------------- ring / PS replay
def ring_allreduce(grads: np.ndarray, op: int = SUM):
    """Round-by-round ring replay.  grads: [N][K_pad] float32.

    Returns (out [N][K_pad] float32, sent_elems [N] int64)."""
    g = np.ascontiguousarray(grads, dtype=np.float32).copy()
    N, K_pad = g.shape
    sent = np.zeros(N, dtype=np.int64)
    if lib().orc_ring_allreduce_f32(_ptr(g), N, K_pad, op, _ptr(sent)):
        raise ValueError("invalid ring arguments")
    return g, sent


def ring_chain(grads: np.ndarray, op: int = SUM) -> np.ndarray:
    """Per-element chain form: [K_pad] float32."""
    g = np.ascontiguousarray(grads, dtype=np.float32)
    N, K_pad = g.shape
    out = np.empty(K_pad, dtype=np.float32)
    if lib().orc_ring_chain_f32(_ptr(g), N, K_pad, op, _ptr(out)):
        raise ValueError("invalid ring arguments")
    return out


def ring_sgd(grads: np.ndarray, params: np.ndarray, lr: float, op: int = MEAN) -> np.ndarray:
    """Ring allreduce + owner SGD (fma(-lr, gbar, w)) + gather of weights.

    grads [N][K_pad] f32; params [K_pad] f32 (identical on all ranks on entry).
    Returns params after the step, [N][K_pad] float32."""
    g = np.ascontiguousarray(grads, dtype=np.float32)
    N, K_pad = g.shape
    p = np.ascontiguousarray(np.broadcast_to(np.asarray(params, np.float32), (N, K_pad))).copy()
    if lib().orc_ring_sgd_f32(_ptr(g), _ptr(p), N, K_pad, op, float(lr)):
        raise ValueError("invalid ring arguments")
    return p


def ps_allreduce(grads: np.ndarray, op: int = SUM) -> np.ndarray:
    """Parameter-server comparator (ascending-rank sum)."""
    g = np.ascontiguousarray(grads, dtype=np.float32)
    N, K = g.shape
    out = np.empty(K, dtype=np.float32)
    if lib().orc_ps_allreduce_f32(_ptr(g), N, K, op, _ptr(out)):
        raise ValueError("invalid PS arguments")
    return out


def bf16_round(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (RNE bit rule) -> fp32, elementwise (reading R8)."""
    f = np.ascontiguousarray(a, dtype=np.float32).ravel()
    L = lib()
    bits = np.fromiter((L.orc_bf16_bits(float(v)) for v in f), dtype=np.uint32, count=f.size)
    return (bits << 16).view(np.float32).reshape(np.shape(a))


# --------------------------------------------------------------------------- TEM
def num_params(Cin: int = 400, C: int = 512, Co: int = 3) -> int:
    return int(lib().orc_tem_num_params(Cin, C, Co))


def tem_fwd_bwd(x, params, labels, lam=(1.0, 1.0, 1.0), prec: int = 0, C: int = 512,
                flips=(), kink_tau=0.0, kinks_cap: int = 4096, threads: int = 1):
    """BSN-TEM forward + weighted logistic loss + backward.

    x [B][T][Cin], params flat (fp32 values, any float dtype), labels [B][Co][T].
    prec 0 = fp64, 1 = bf16-operand emulation (reading R8).
    flips: indices layer*(B*T*C) + (b*T+t)*C + c of ReLU decisions to invert (reading R7b).
    kink_tau > 0: also report pre-activations with |a| <= kink_tau * sum|terms|; a pair
    (tau_a1, tau_a2) gives each layer its own band (reading R7b).
    threads > 1: the videos are split into contiguous sub-batches computed concurrently (the
    C call releases the GIL) and merged in sub-batch order -- see _tem_fwd_bwd_split.
    Returns dict(loss [1+Co] f64, z [B][T][Co] f64, grad [K] f64, kinks [n] int64)."""
    if threads > 1 and np.shape(x)[0] > 1:
        return _tem_fwd_bwd_split(x, params, labels, lam, prec, C, flips, kink_tau, kinks_cap, threads)
    x = np.ascontiguousarray(x, dtype=np.float64)
    B, T, Cin = x.shape
    labels = np.ascontiguousarray(labels, dtype=np.float64)
    Co = labels.shape[1]
    K = num_params(Cin, C, Co)
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64)[:K])
    assert p.size == K, (p.size, K)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    loss = np.zeros(1 + Co)
    z = np.zeros((B, T, Co))
    grad = np.zeros(K)
    fl = np.ascontiguousarray(np.sort(np.asarray(flips, dtype=np.int64)))
    tau1, tau2 = (kink_tau, kink_tau) if np.isscalar(kink_tau) else tuple(kink_tau)
    kinks = np.zeros(max(kinks_cap, 1), dtype=np.int64)
    nk = np.zeros(1, dtype=np.int64)
    dec = np.zeros(2 * B * T * C, dtype=np.uint8)
    rc = lib().orc_tem_fwd_bwd_ex(prec, B, T, Cin, C, Co, _ptr(x), _ptr(p), _ptr(labels), _ptr(lam),
                                  _ptr(loss), _ptr(z), _ptr(grad), _ptr(fl) if fl.size else None,
                                  int(fl.size), float(tau1), float(tau2), _ptr(kinks), int(kinks_cap), _ptr(nk),
                                  _ptr(dec))
    if rc:
        raise ValueError("invalid TEM arguments")
    n = int(nk[0])
    return {"loss": loss, "z": z, "grad": grad, "kinks": kinks[:min(n, kinks_cap)].copy(), "nkinks": n,
            "decisions": dec}


def _tem_fwd_bwd_split(x, params, labels, lam, prec, C, flips, kink_tau, kinks_cap, threads):
    """tem_fwd_bwd over contiguous sub-batches in parallel.  The loss is a per-video mean
    (L = (1/B) sum_v L_v, reading R6), so a sub-batch of b videos returns (1/b) sum over its
    videos and the whole batch is sum_c (b_c / B) * result_c, merged in sub-batch order (fp64:
    differs from the one-call result only by summation order).  ReLU-decision indices
    layer*(B*T*C) + (b*T+t)*C + c are translated between the batch and each sub-batch.
    prec = 1 rounds dA2 / dA1 to bf16 AFTER the 1/B factor of dz: the sub-batches are then
    equal with B/b a power of two, so the rescaling b/B is exact and commutes with rounding."""
    from concurrent.futures import ThreadPoolExecutor
    B, T, _ = np.shape(x)
    n = min(threads, B)
    if prec == 1:
        n = 1
        while 2 * n <= min(threads, B) and B % (2 * n) == 0:
            n *= 2
        if n == 1:
            return tem_fwd_bwd(x, params, labels, lam, prec, C, flips, kink_tau, kinks_cap)
    cuts = [B * i // n for i in range(n + 1)]
    BTC, fl = B * T * C, np.sort(np.asarray(flips, dtype=np.int64))
    layer, within = fl // BTC, fl % BTC

    def part(i):
        b0, b1 = cuts[i], cuts[i + 1]
        lo, hi = b0 * T * C, b1 * T * C
        m = (within >= lo) & (within < hi)
        sub = layer[m] * ((b1 - b0) * T * C) + (within[m] - lo)
        return tem_fwd_bwd(x[b0:b1], params, labels[b0:b1], lam, prec, C, sub, kink_tau, kinks_cap)
    with ThreadPoolExecutor(n) as ex:
        parts = list(ex.map(part, range(n)))
    loss = sum(((cuts[i + 1] - cuts[i]) / B) * parts[i]["loss"] for i in range(n))
    grad = sum(((cuts[i + 1] - cuts[i]) / B) * parts[i]["grad"] for i in range(n))
    z = np.concatenate([q["z"] for q in parts])
    dec = np.concatenate([q["decisions"].reshape(2, -1) for q in parts], axis=1).ravel()
    kinks, nk = [], 0
    for i, q in enumerate(parts):
        bsz = (cuts[i + 1] - cuts[i]) * T * C
        k = q["kinks"]
        kinks.append((k // bsz) * BTC + cuts[i] * T * C + k % bsz)
        nk += q["nkinks"]
    kinks = np.sort(np.concatenate(kinks)) if kinks else np.zeros(0, np.int64)
    return {"loss": loss, "z": z, "grad": grad, "kinks": kinks[:kinks_cap], "nkinks": nk, "decisions": dec}


def ring_adam(grads, params, m, v, scal, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """Ring mean + Adam owner update (reading R22).  grads [N][K_pad] f32; params, m, v [K_pad]
    f32 (one replica; every rank ends with the same params); scal [2] = (beta1^t, beta2^t) of the
    previous step, updated in place.  Returns (params', m', v', scal')."""
    g = np.ascontiguousarray(grads, dtype=np.float32)
    N, Kp = g.shape
    w = np.array(params, dtype=np.float32, copy=True)
    mm = np.array(m, dtype=np.float32, copy=True)
    vv = np.array(v, dtype=np.float32, copy=True)
    sc = np.array(scal, dtype=np.float32, copy=True)
    rc = lib().orc_ring_adam_f32(_ptr(g), _ptr(w), _ptr(mm), _ptr(vv), _ptr(sc), N, Kp, float(lr), float(beta1),
                                 float(beta2), float(eps))
    if rc:
        raise ValueError("invalid ring_adam arguments")
    return w, mm, vv, sc


def ring_momentum(grads, params, u, lr, mu):
    """Ring mean + heavy-ball momentum owner update (reading R23): u = fma(mu, u, gbar),
    w = fma(-lr, u, w).  grads [N][K_pad] f32; params, u [K_pad] f32.  Returns (params', u')."""
    g = np.ascontiguousarray(grads, dtype=np.float32)
    N, Kp = g.shape
    w = np.array(params, dtype=np.float32, copy=True)
    uu = np.array(u, dtype=np.float32, copy=True)
    if lib().orc_ring_momentum_f32(_ptr(g), _ptr(w), _ptr(uu), N, Kp, float(lr), float(mu)):
        raise ValueError("invalid ring_momentum arguments")
    return w, uu


# --------------------------------------------------------------------------- PEM
def pem_num_params(F: int = 32, H: int = 512) -> int:
    return int(lib().orc_pem_num_params(F, H))


def pem_fwd_bwd(f, params, g, flips=(), kink_tau: float = 0.0, kinks_cap: int = 4096):
    """BSN PEM forward + MSE-to-IoU loss + backward (configs[4], readings R19-R21), fp64.

    f [M][F] BSP features, params flat [W1 (H x F), b1 (H), w2 (H), b2], g [M] IoU targets.
    flips / kink_tau: ReLU decision overrides and ambiguity band, indices m*H + j (R7b).
    Returns dict(loss f64, y [M], grad [K_pem], kinks, nkinks, decisions [M*H] u8)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    M, F = f.shape
    Kp = None
    p = np.asarray(params, dtype=np.float64).ravel()
    # H from the parameter count: K = H*F + 2H + 1
    H = (p.size - 1) // (F + 2)
    Kp = pem_num_params(F, H)
    assert p.size == Kp, (p.size, Kp)
    p = np.ascontiguousarray(p)
    g = np.ascontiguousarray(g, dtype=np.float64).ravel()
    assert g.size == M
    loss = np.zeros(1)
    y = np.zeros(M)
    grad = np.zeros(Kp)
    fl = np.ascontiguousarray(np.sort(np.asarray(flips, dtype=np.int64)))
    kinks = np.zeros(max(kinks_cap, 1), dtype=np.int64)
    nk = np.zeros(1, dtype=np.int64)
    dec = np.zeros(max(M * H, 1), dtype=np.uint8)
    rc = lib().orc_pem_fwd_bwd(M, F, H, _ptr(f), _ptr(p), _ptr(g), _ptr(loss), _ptr(y), _ptr(grad),
                               _ptr(fl) if fl.size else None, int(fl.size), float(kink_tau), _ptr(kinks),
                               int(kinks_cap), _ptr(nk), _ptr(dec))
    if rc:
        raise ValueError("invalid PEM arguments")
    n = int(nk[0])
    return {"loss": float(loss[0]), "y": y, "grad": grad, "kinks": kinks[:min(n, kinks_cap)].copy(), "nkinks": n,
            "decisions": dec[:M * H]}


def pem_param_slices(F: int = 32, H: int = 512):
    """Flat PEM parameter order [W1p, b1p, w2p, b2p] (reading R21)."""
    sizes = [("W1p", H * F), ("b1p", H), ("w2p", H), ("b2p", 1)]
    out, off = {}, 0
    for name, n in sizes:
        out[name] = slice(off, off + n)
        off += n
    return out


def param_slices(Cin: int = 400, C: int = 512, Co: int = 3):
    """Flat gradient order [W1, b1, W2, b2, W3, b3] (SURVEY 8(c) layouts)."""
    sizes = [("W1", C * 3 * Cin), ("b1", C), ("W2", C * 3 * C), ("b2", C), ("W3", Co * C), ("b3", Co)]
    out, off = {}, 0
    for name, n in sizes:
        out[name] = slice(off, off + n)
        off += n
    return out


# --------------------------------------------------------------------------- PGM
from .proposals import pgm, pgm_video, candidates as pgm_candidates, bsp_feature, F_BSP  # noqa: E402,F401
