"""Thin Python binding of libtem.so (include/tem.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
behind the C ABI.  torch is used for device memory, streams and process groups
(symmetric-memory rendezvous for the peer heaps).  There is no fallback: if the
library cannot be loaded, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _build

TEM_OK, TEM_ERR_INVALID_ARG, TEM_ERR_PROTOCOL, TEM_ERR_TRANSPORT, TEM_ERR_CUDA, \
    TEM_ERR_NONFINITE, TEM_ERR_STATE = range(7)
TEM_SUM, TEM_MEAN = 0, 1
TEM_FP32, TEM_BF16 = 0, 1
TEM_EXCHANGE_RING, TEM_EXCHANGE_PS, TEM_EXCHANGE_TWOSHOT = 0, 1, 2
TEM_OPT_SGD, TEM_OPT_ADAM, TEM_OPT_MOMENTUM = 0, 1, 2
MAX_RANKS = 8

_P = ctypes.c_void_p


class tem_config(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32), ("world_size", ctypes.c_int32), ("device", ctypes.c_int32),
        ("local_ranks", ctypes.c_int32),
        ("batch_per_rank", ctypes.c_int32), ("seq_len", ctypes.c_int32),
        ("c_in", ctypes.c_int32), ("c_hidden", ctypes.c_int32), ("c_out", ctypes.c_int32),
        ("precision", ctypes.c_int32),
        ("lr", ctypes.c_float), ("loss_weight", ctypes.c_float * 3),
        ("peer_bufs", ctypes.POINTER(ctypes.c_void_p)), ("sym_bytes", ctypes.c_size_t),
        ("max_allreduce_elems", ctypes.c_int64),
        ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
        ("ring_channels", ctypes.c_int32), ("spin_timeout_ms", ctypes.c_int32),
        ("exchange", ctypes.c_int32),
        ("pem_proposals", ctypes.c_int32), ("pem_features", ctypes.c_int32), ("pem_hidden", ctypes.c_int32),
        ("optimizer", ctypes.c_int32), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float),
        ("momentum", ctypes.c_float), ("exchange_buckets", ctypes.c_int32), ("pgm_gt_max", ctypes.c_int32),
    ]


class TemError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{what}: {status_string(code)} ({code})")


_lib = None


def lib():
    """Load the in-tree libtem.so (building it with nvcc if stale).  Raises if it cannot."""
    global _lib
    if _lib is None:
        # TEM_DIAG_LIB=1 (scripts/probes only): the diagnostics build with kernel traces
        path = _build.build(diag=os.environ.get("TEM_DIAG_LIB") == "1")
        if os.environ.get("TEM_DIAG_LIB") == "1" and os.environ.get("TEM_DIAG_LIB_PATH"):
            path = os.environ["TEM_DIAG_LIB_PATH"]  # a diagnostics build variant (experiments)
        L = ctypes.CDLL(path)
        cp = ctypes.POINTER(tem_config)
        L.tem_num_params.restype = ctypes.c_int64
        L.tem_num_params.argtypes = [cp]
        L.tem_kpad.restype = ctypes.c_int64
        L.tem_kpad.argtypes = [cp, ctypes.c_int64]
        for f in (L.tem_workspace_bytes, L.tem_sym_bytes, L.tem_sym_user_offset, L.tem_sym_hdr_offset,
                  L.tem_sym_ll_offset):
            f.restype = ctypes.c_size_t
            f.argtypes = [cp]
        L.tem_ll_slot_lines.restype = ctypes.c_int64
        L.tem_ll_slot_lines.argtypes = [cp]
        L.tem_init.restype = ctypes.c_int
        L.tem_init.argtypes = [cp, _P, ctypes.POINTER(_P)]
        for f in (L.tem_step, L.tem_compute):
            f.restype = ctypes.c_int
            f.argtypes = [_P, _P, _P, _P, _P]
        for f in (L.tem_step_pem, L.tem_compute_pem, L.tem_step_pgm, L.tem_compute_pgm):
            f.restype = ctypes.c_int
            f.argtypes = [_P, _P, _P, _P, _P, _P, _P]
        L.tem_pem_relu_decisions.restype = ctypes.c_int
        L.tem_pem_relu_decisions.argtypes = [_P, ctypes.c_int32, _P, _P]
        L.tem_step_host.restype = ctypes.c_int
        L.tem_step_host.argtypes = [_P, _P, _P, _P, _P]
        L.tem_pgm.restype = ctypes.c_int
        L.tem_pgm.argtypes = [ctypes.c_int32] * 4 + [_P] * 9
        L.tem_step_pem_host.restype = ctypes.c_int
        L.tem_step_pem_host.argtypes = [_P, _P, _P, _P, _P, _P, _P]
        L.tem_exchange.restype = ctypes.c_int
        L.tem_exchange.argtypes = [_P, _P]
        for f in (L.ring_allreduce, L.ps_allreduce, L.twoshot_allreduce):
            f.restype = ctypes.c_int
            f.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int32, _P]
        L.tem_sync.restype = ctypes.c_int
        L.tem_sync.argtypes = [_P, _P, ctypes.POINTER(ctypes.c_int64)]
        L.tem_shutdown.restype = ctypes.c_int
        L.tem_shutdown.argtypes = [_P]
        for f in (L.tem_local_grad, L.tem_logits):
            f.restype = _P
            f.argtypes = [_P, ctypes.c_int32]
        for f in (L.tem_launches_per_step, L.tem_launches_per_exchange):
            f.restype = ctypes.c_int32
            f.argtypes = [_P]
        L.tem_status_string.restype = ctypes.c_char_p
        L.tem_status_string.argtypes = [ctypes.c_int32]
        L.tem_kernel_path.restype = ctypes.c_char_p
        L.tem_kernel_path.argtypes = [_P]
        L.tem_debug_buffer.restype = _P
        L.tem_debug_buffer.argtypes = [_P, ctypes.c_int32, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]
        L.tem_relu_decisions.restype = ctypes.c_int
        L.tem_relu_decisions.argtypes = [_P, ctypes.c_int32, _P, _P]
        L.tem_timing_slots.restype = ctypes.c_int32
        L.tem_timing_slots.argtypes = [_P]
        L.tem_timing_slot_name.restype = ctypes.c_char_p
        L.tem_timing_slot_name.argtypes = [_P, ctypes.c_int32]
        L.tem_timing_begin.restype = ctypes.c_int
        L.tem_timing_begin.argtypes = [_P, ctypes.c_int32]
        L.tem_timing_end.restype = ctypes.c_int
        L.tem_timing_end.argtypes = [_P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int32)]
        _lib = L
    return _lib


EXPORTS = ["tem_num_params", "tem_kpad", "tem_workspace_bytes", "tem_sym_bytes",
           "tem_sym_user_offset", "tem_init", "tem_step", "tem_compute", "tem_exchange",
           "tem_step_host", "ring_allreduce", "ps_allreduce", "tem_sync", "tem_shutdown",
           "tem_local_grad", "tem_logits", "tem_launches_per_step", "tem_launches_per_exchange",
           "tem_status_string", "tem_kernel_path", "tem_timing_slots", "tem_timing_slot_name",
           "tem_timing_begin", "tem_timing_end", "tem_relu_decisions", "tem_debug_buffer",
           "tem_step_pem", "tem_compute_pem", "tem_pem_relu_decisions", "twoshot_allreduce", "tem_step_pem_host", "tem_pgm", "tem_step_pgm", "tem_compute_pgm",
           "tem_sym_hdr_offset", "tem_sym_ll_offset", "tem_ll_slot_lines"]


def status_string(code: int) -> str:
    return lib().tem_status_string(int(code)).decode()


def _check(code: int, what: str):
    if code != TEM_OK:
        raise TemError(code, what)


def _stream_ptr(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


# ----------------------------------------------------------------------------- C-ABI mirrors
def tem_num_params(cfg: tem_config) -> int:
    return int(lib().tem_num_params(ctypes.byref(cfg)))


def tem_kpad(cfg: tem_config, K: int) -> int:
    return int(lib().tem_kpad(ctypes.byref(cfg), K))


def tem_workspace_bytes(cfg: tem_config) -> int:
    return int(lib().tem_workspace_bytes(ctypes.byref(cfg)))


def tem_sym_bytes(cfg: tem_config) -> int:
    return int(lib().tem_sym_bytes(ctypes.byref(cfg)))


def tem_sym_user_offset(cfg: tem_config) -> int:
    return int(lib().tem_sym_user_offset(ctypes.byref(cfg)))


def tem_init(cfg: tem_config, params_ptr: int) -> int:
    ctx = _P()
    _check(lib().tem_init(ctypes.byref(cfg), _P(params_ptr), ctypes.byref(ctx)), "tem_init")
    return ctx.value


def tem_step(ctx: int, x_ptr: int, labels_ptr: int, loss_ptr: int, stream=None):
    _check(lib().tem_step(_P(ctx), _P(x_ptr), _P(labels_ptr), _P(loss_ptr), _stream_ptr(stream)), "tem_step")


def tem_compute(ctx: int, x_ptr: int, labels_ptr: int, loss_ptr: int, stream=None):
    _check(lib().tem_compute(_P(ctx), _P(x_ptr), _P(labels_ptr), _P(loss_ptr), _stream_ptr(stream)),
           "tem_compute")


def tem_exchange(ctx: int, stream=None):
    _check(lib().tem_exchange(_P(ctx), _stream_ptr(stream)), "tem_exchange")


def tem_step_host(ctx: int, x_host_ptr: int, labels_host_ptr: int, loss_host_ptr: int, stream=None):
    _check(lib().tem_step_host(_P(ctx), _P(x_host_ptr), _P(labels_host_ptr), _P(loss_host_ptr),
                               _stream_ptr(stream)), "tem_step_host")


def ring_allreduce(ctx: int, buf_ptr: int, K: int, op: int = TEM_SUM, stream=None):
    _check(lib().ring_allreduce(_P(ctx), _P(buf_ptr), int(K), int(op), _stream_ptr(stream)), "ring_allreduce")


def ps_allreduce(ctx: int, buf_ptr: int, K: int, op: int = TEM_SUM, stream=None):
    _check(lib().ps_allreduce(_P(ctx), _P(buf_ptr), int(K), int(op), _stream_ptr(stream)), "ps_allreduce")


def twoshot_allreduce(ctx: int, buf_ptr: int, K: int, op: int = TEM_SUM, stream=None):
    _check(lib().twoshot_allreduce(_P(ctx), _P(buf_ptr), int(K), int(op), _stream_ptr(stream)), "twoshot_allreduce")


def tem_sync(ctx: int, stream=None):
    step = ctypes.c_int64(-1)
    code = lib().tem_sync(_P(ctx), _stream_ptr(stream), ctypes.byref(step))
    return int(code), int(step.value)


def tem_shutdown(ctx: int):
    _check(lib().tem_shutdown(_P(ctx)), "tem_shutdown")



def pgm(prob: torch.Tensor, gt: torch.Tensor, n_gt: torch.Tensor, P: int, stream=None) -> dict:
    """BSN proposal generation on the GPU (tem_pgm, reading R24).  prob [B][3][T] fp32, gt
    [B][G][2] fp32, n_gt [B] int32, all on one CUDA device.  Returns device tensors count [B],
    ts / te [B][P] int32, features [B][P][32], iou [B][P]."""
    B, _, T = prob.shape
    G = gt.shape[1]
    dev = prob.device
    out = {"count": torch.empty(B, dtype=torch.int32, device=dev),
           "ts": torch.empty(B, P, dtype=torch.int32, device=dev),
           "te": torch.empty(B, P, dtype=torch.int32, device=dev),
           "features": torch.empty(B, P, 32, dtype=torch.float32, device=dev),
           "iou": torch.empty(B, P, dtype=torch.float32, device=dev)}
    _check(lib().tem_pgm(B, T, G, P, _P(prob.data_ptr()), _P(gt.data_ptr()), _P(n_gt.data_ptr()),
                         _P(out["features"].data_ptr()), _P(out["iou"].data_ptr()), _P(out["ts"].data_ptr()),
                         _P(out["te"].data_ptr()), _P(out["count"].data_ptr()), _stream_ptr(stream)), "tem_pgm")
    return out


# ----------------------------------------------------------------------------- session helper
@dataclass
class SessionConfig:
    world_size: int = 1
    rank: int = 0
    local_ranks: int = 1
    batch_per_rank: int = 16
    seq_len: int = 100
    c_in: int = 400
    c_hidden: int = 512
    c_out: int = 3
    precision: int = TEM_FP32
    lr: float = 0.01
    loss_weight: Sequence[float] = (1.0, 1.0, 1.0)
    max_allreduce_elems: int = 0
    ring_channels: int = 0
    spin_timeout_ms: int = 0  # bound on a wait for a peer; 0 -> 20 s
    exchange: int = TEM_EXCHANGE_RING
    pem_proposals: int = 0  # > 0: joint TEM + PEM (configs[4]); params = [TEM | PEM]
    pem_features: int = 32
    pem_hidden: int = 512
    optimizer: int = TEM_OPT_SGD  # TEM_OPT_ADAM: owner-side Adam (reading R22)
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    momentum: float = 0.9  # TEM_OPT_MOMENTUM (reading R23)
    pgm_gt_max: int = 0  # > 0: PEM fed by PGM on the step's own TEM output (reading R24)
    exchange_buckets: int = 0  # 2: two-bucket exchange, the W2.. bucket overlapping conv1 wgrad (R25)


class TemSession:
    """Owns the device memory of one process's ranks and the library context.

    * world_size == local_ranks (N = 1, or the single-device emulation): every rank's
      heap is a plain device allocation on this GPU.
    * local_ranks == 1 and world_size > 1 (one process per GPU): the heap comes from
      torch symmetric memory; its rendezvous gives the peer pointers (NVLink P2P).
    * heap="ipc" (local_ranks == 1, world_size > 1): the heaps are plain device allocations
      whose CUDA IPC handles are exchanged over the process group (all_gather_object), each
      process mapping its peers' heaps -- where torch symmetric memory is unavailable, e.g.
      processes sharing one GPU (tests/test_gpu_symm.py).  Across GPUs each mapping opens a
      context on the peer's device.
    * virtual_peers=True (tests only; local_ranks == 1): every rank's heap is a plain
      allocation on this GPU and this process drives rank sc.rank alone; the test plays the
      other ranks by writing their headers and messages into the heaps (the wire protocol of
      include/tem.h) BEFORE the collective is launched, so no kernel ever waits on another.
    """

    def __init__(self, sc: SessionConfig, params: np.ndarray, device: int | None = None, group=None,
                 virtual_peers: bool = False, heap: str = "symm"):
        L = lib()
        self.sc = sc
        self.device = torch.cuda.current_device() if device is None else device
        self.dev = torch.device("cuda", self.device)
        cfg = tem_config()
        cfg.rank, cfg.world_size, cfg.device, cfg.local_ranks = sc.rank, sc.world_size, self.device, sc.local_ranks
        cfg.batch_per_rank, cfg.seq_len = sc.batch_per_rank, sc.seq_len
        cfg.c_in, cfg.c_hidden, cfg.c_out = sc.c_in, sc.c_hidden, sc.c_out
        cfg.precision, cfg.lr = sc.precision, sc.lr
        for i in range(3):
            cfg.loss_weight[i] = float(sc.loss_weight[i])
        cfg.max_allreduce_elems = sc.max_allreduce_elems
        cfg.ring_channels, cfg.spin_timeout_ms = sc.ring_channels, sc.spin_timeout_ms
        cfg.exchange = sc.exchange
        cfg.pem_proposals, cfg.pem_features, cfg.pem_hidden = sc.pem_proposals, sc.pem_features, sc.pem_hidden
        cfg.optimizer, cfg.beta1, cfg.beta2, cfg.eps = sc.optimizer, sc.beta1, sc.beta2, sc.eps
        cfg.momentum = sc.momentum
        cfg.pgm_gt_max = sc.pgm_gt_max
        cfg.exchange_buckets = sc.exchange_buckets
        self.K = tem_num_params(cfg)
        if self.K == 0:
            raise TemError(TEM_ERR_INVALID_ARG, "config")
        self.Kpad = tem_kpad(cfg, self.K)
        self.sym_bytes = tem_sym_bytes(cfg)
        self.user_off = tem_sym_user_offset(cfg)
        self.ws_bytes = tem_workspace_bytes(cfg)
        N = sc.world_size
        self._symm = None
        self.hdr_off = lib().tem_sym_hdr_offset(cfg)
        self.ll_off = lib().tem_sym_ll_offset(cfg)
        self.ll_lines = lib().tem_ll_slot_lines(cfg)
        if sc.local_ranks == N or virtual_peers:
            self.heaps = [torch.zeros(self.sym_bytes + 4096, dtype=torch.uint8, device=self.dev)
                          for _ in range(N)]
            ptrs = [(h.data_ptr() + 4095) // 4096 * 4096 for h in self.heaps]
            self.heap_off = [p - h.data_ptr() for p, h in zip(ptrs, self.heaps)]
        elif heap == "ipc":
            import torch.distributed as dist
            from torch.multiprocessing.reductions import reduce_tensor
            from . import dist as tdist
            grp = group if group is not None else dist.group.WORLD
            tdist.check_symmetric(sc, grp)
            t = torch.zeros(self.sym_bytes + 4096, dtype=torch.uint8, device=self.dev)
            off = (t.data_ptr() + 4095) // 4096 * 4096 - t.data_ptr()
            rebuild, args = reduce_tensor(t)
            objs = [None] * N
            dist.all_gather_object(objs, (args, off), group=grp)
            # every rank's heap as mapped in this process (peers: kept open for the session)
            self.heaps, self.heap_off = [], []
            for r, (a, o) in enumerate(objs):
                self.heaps.append(t if r == sc.rank else rebuild(*a))  # cudaIpcOpenMemHandle
                self.heap_off.append(off if r == sc.rank else o)
            ptrs = [h.data_ptr() + o for h, o in zip(self.heaps, self.heap_off)]
            torch.cuda.synchronize(self.dev)
            dist.barrier(group=grp)
        else:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            from . import dist as tdist
            grp = group if group is not None else dist.group.WORLD
            tdist.check_symmetric(sc, grp)  # equal K / shapes on every rank before any peer wait
            gname = grp.group_name
            if hasattr(symm_mem, "enable_symm_mem_for_group"):
                try:  # required on some torch versions, a no-op / deprecated on newer ones
                    symm_mem.enable_symm_mem_for_group(gname)
                except Exception:
                    pass
            t = symm_mem.empty(self.sym_bytes, dtype=torch.uint8, device=self.dev)
            t.zero_()
            hdl = symm_mem.rendezvous(t, gname)
            self._symm = (t, hdl)
            ptrs = list(hdl.buffer_ptrs)
            if any(p % 4096 for p in ptrs):
                raise TemError(TEM_ERR_INVALID_ARG, "symmetric heap not 4 KiB aligned")
            self.heaps = [t]
            self.heap_off = [0]
            torch.cuda.synchronize(self.dev)
            dist.barrier(group=grp)
        self._ptr_arr = (ctypes.c_void_p * N)(*ptrs)
        cfg.peer_bufs = ctypes.cast(self._ptr_arr, ctypes.POINTER(ctypes.c_void_p))
        cfg.sym_bytes = self.sym_bytes
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.dev)
        cfg.workspace, cfg.workspace_bytes = self.ws.data_ptr(), self.ws_bytes
        self.cfg = cfg
        p = np.zeros(self.Kpad, np.float32)
        p[: min(params.size, self.Kpad)] = np.asarray(params, np.float32)[: self.Kpad]
        pt = torch.from_numpy(p).to(self.dev)
        for l in range(sc.local_ranks):
            self.params(l).copy_(pt)
        if virtual_peers:
            for r in range(N):
                self._heap_of(r)[: 4 * self.Kpad].view(torch.float32).copy_(pt)
        torch.cuda.synchronize(self.dev)
        self.ctx = tem_init(cfg, ptrs[sc.rank])
        self.loss = torch.zeros(sc.local_ranks, 4, dtype=torch.float32, device=self.dev)
        # joint TEM + PEM: [local_ranks * 4 TEM losses | local_ranks PEM losses]
        self.loss_pem = torch.zeros(5 * sc.local_ranks, dtype=torch.float32, device=self.dev)

    # -- views into caller-owned memory
    def _heap(self, l: int) -> torch.Tensor:
        if len(self.heaps) > self.sc.local_ranks:  # virtual peers: local rank 0 is sc.rank
            l = self.sc.rank + l
        return self._heap_of(l)

    def _heap_of(self, r: int) -> torch.Tensor:
        """Heap of global rank r (emulation / virtual peers: all heaps live in this process;
        heap="ipc": the peers' heaps as mapped here)."""
        h = self.heaps[r]
        return h[self.heap_off[r]: self.heap_off[r] + self.sym_bytes]

    def params(self, l: int = 0) -> torch.Tensor:
        return self._heap(l)[: 4 * self.Kpad].view(torch.float32)

    def user(self, l: int = 0, K: int | None = None) -> torch.Tensor:
        n = self.Kpad if K is None else K
        return self._heap(l)[self.user_off: self.user_off + 4 * n].view(torch.float32)

    def _ws_view(self, ptr: int, nbytes: int) -> torch.Tensor:
        off = ptr - self.ws.data_ptr()
        return self.ws[off: off + nbytes]

    def local_grad(self, l: int = 0) -> torch.Tensor:
        ptr = lib().tem_local_grad(_P(self.ctx), l)
        return self._ws_view(ptr, 4 * self.Kpad).view(torch.float32)

    def logits(self, l: int = 0) -> torch.Tensor:
        ptr = lib().tem_logits(_P(self.ctx), l)
        B, T = self.sc.batch_per_rank, self.sc.seq_len
        return self._ws_view(ptr, 4 * B * T * 3).view(torch.float32).view(B, T, 3)

    def debug_buffer(self, name: str, l: int = 0):
        """Internal workspace tensor as a torch view (bf16/fp32 per the path), or None."""
        nb = ctypes.c_int64(0)
        ptr = lib().tem_debug_buffer(_P(self.ctx), l, name.encode(), ctypes.byref(nb))
        if not ptr:
            return None
        raw = self._ws_view(ptr, nb.value)
        if name == "h2" or name in ("pgm_prob", "pgm_feat", "pgm_iou"):
            return raw.view(torch.float32)
        if name in ("pgm_ts", "pgm_te", "pgm_count"):
            return raw.view(torch.int32)
        elem = 2 if self.kernel_path().startswith("tcgen05") or self.sc.precision == TEM_BF16 else 4
        return raw.view(torch.bfloat16 if elem == 2 else torch.float32)

    def relu_decisions(self, l: int = 0) -> torch.Tensor:
        B, T, C = self.sc.batch_per_rank, self.sc.seq_len, self.sc.c_hidden
        out = torch.zeros(2 * B * T * C, dtype=torch.uint8, device=self.dev)
        _check(lib().tem_relu_decisions(_P(self.ctx), l, _P(out.data_ptr()), _stream_ptr(None)),
               "tem_relu_decisions")
        return out

    # -- calls
    def step(self, x: torch.Tensor, labels: torch.Tensor, stream=None) -> torch.Tensor:
        tem_step(self.ctx, x.data_ptr(), labels.data_ptr(), self.loss.data_ptr(), stream)
        return self.loss

    def compute(self, x: torch.Tensor, labels: torch.Tensor, stream=None) -> torch.Tensor:
        tem_compute(self.ctx, x.data_ptr(), labels.data_ptr(), self.loss.data_ptr(), stream)
        return self.loss

    def step_pem(self, x: torch.Tensor, labels: torch.Tensor, bsp: torch.Tensor, iou: torch.Tensor, stream=None):
        """Joint TEM + PEM step (configs[4]); returns (tem_loss [local_ranks][4], pem_loss [local_ranks])."""
        _check(lib().tem_step_pem(_P(self.ctx), _P(x.data_ptr()), _P(labels.data_ptr()), _P(bsp.data_ptr()),
                                  _P(iou.data_ptr()), _P(self.loss_pem.data_ptr()), _stream_ptr(stream)), "tem_step_pem")
        n = self.sc.local_ranks
        return self.loss_pem[:4 * n].view(n, 4), self.loss_pem[4 * n:]

    def step_pgm(self, x: torch.Tensor, labels: torch.Tensor, gt: torch.Tensor, n_gt: torch.Tensor, stream=None):
        """Joint TEM + PGM + PEM step (pgm_gt_max > 0): PEM on PGM's proposals of this step's TEM
        output.  gt [local_ranks][B][G][2] fp32, n_gt [local_ranks][B] int32 (device)."""
        _check(lib().tem_step_pgm(_P(self.ctx), _P(x.data_ptr()), _P(labels.data_ptr()), _P(gt.data_ptr()),
                                  _P(n_gt.data_ptr()), _P(self.loss_pem.data_ptr()), _stream_ptr(stream)), "tem_step_pgm")
        n = self.sc.local_ranks
        return self.loss_pem[:4 * n].view(n, 4), self.loss_pem[4 * n:]

    def compute_pgm(self, x: torch.Tensor, labels: torch.Tensor, gt: torch.Tensor, n_gt: torch.Tensor, stream=None):
        _check(lib().tem_compute_pgm(_P(self.ctx), _P(x.data_ptr()), _P(labels.data_ptr()), _P(gt.data_ptr()),
                                     _P(n_gt.data_ptr()), _P(self.loss_pem.data_ptr()), _stream_ptr(stream)),
               "tem_compute_pgm")
        n = self.sc.local_ranks
        return self.loss_pem[:4 * n].view(n, 4), self.loss_pem[4 * n:]

    def compute_pem(self, x: torch.Tensor, labels: torch.Tensor, bsp: torch.Tensor, iou: torch.Tensor, stream=None):
        _check(lib().tem_compute_pem(_P(self.ctx), _P(x.data_ptr()), _P(labels.data_ptr()), _P(bsp.data_ptr()),
                                     _P(iou.data_ptr()), _P(self.loss_pem.data_ptr()), _stream_ptr(stream)),
               "tem_compute_pem")
        n = self.sc.local_ranks
        return self.loss_pem[:4 * n].view(n, 4), self.loss_pem[4 * n:]

    def pem_record_decisions(self):
        _check(lib().tem_pem_relu_decisions(_P(self.ctx), 0, None, None), "tem_pem_relu_decisions")

    def pem_relu_decisions(self, l: int = 0) -> torch.Tensor:
        M = self.sc.batch_per_rank * self.sc.pem_proposals
        out = torch.zeros(M * self.sc.pem_hidden, dtype=torch.uint8, device=self.dev)
        _check(lib().tem_pem_relu_decisions(_P(self.ctx), l, _P(out.data_ptr()), _stream_ptr(None)),
               "tem_pem_relu_decisions")
        return out

    def exchange(self, stream=None):
        tem_exchange(self.ctx, stream)

    def allreduce(self, K: int, op: int = TEM_SUM, stream=None):
        ring_allreduce(self.ctx, self.user(0).data_ptr(), K, op, stream)

    def ps_allreduce(self, K: int, op: int = TEM_SUM, stream=None):
        ps_allreduce(self.ctx, self.user(0).data_ptr(), K, op, stream)

    def twoshot_allreduce(self, K: int, op: int = TEM_SUM, stream=None):
        twoshot_allreduce(self.ctx, self.user(0).data_ptr(), K, op, stream)

    def sync(self, stream=None):
        return tem_sync(self.ctx, stream)

    def launches_per_step(self) -> int:
        return int(lib().tem_launches_per_step(_P(self.ctx)))

    def launches_per_exchange(self) -> int:
        return int(lib().tem_launches_per_exchange(_P(self.ctx)))

    def timing_begin(self, max_steps: int):
        _check(lib().tem_timing_begin(_P(self.ctx), int(max_steps)), "tem_timing_begin")

    def timing_end(self) -> tuple[dict, int]:
        n = int(lib().tem_timing_slots(_P(self.ctx)))
        arr = (ctypes.c_float * n)()
        steps = ctypes.c_int32(0)
        _check(lib().tem_timing_end(_P(self.ctx), arr, ctypes.byref(steps)), "tem_timing_end")
        names = [lib().tem_timing_slot_name(_P(self.ctx), k).decode() for k in range(n)]
        return {names[k]: float(arr[k]) for k in range(n)}, int(steps.value)

    def step_host(self, x_host: torch.Tensor, labels_host: torch.Tensor, loss_host: torch.Tensor, stream=None):
        tem_step_host(self.ctx, x_host.data_ptr(), labels_host.data_ptr(), loss_host.data_ptr(), stream)

    def step_pem_host(self, x_host: torch.Tensor, labels_host: torch.Tensor, bsp_host: torch.Tensor,
                      iou_host: torch.Tensor, loss_host: torch.Tensor, stream=None):
        """Joint step from host buffers (pinned); loss_host: 5 floats [4 TEM | PEM]."""
        _check(lib().tem_step_pem_host(_P(self.ctx), _P(x_host.data_ptr()), _P(labels_host.data_ptr()),
                                       _P(bsp_host.data_ptr()), _P(iou_host.data_ptr()), _P(loss_host.data_ptr()),
                                       _stream_ptr(stream)), "tem_step_pem_host")

    def kernel_path(self) -> str:
        return lib().tem_kernel_path(_P(self.ctx)).decode()

    def close(self):
        if getattr(self, "ctx", None):
            ctx, self.ctx = self.ctx, None
            tem_shutdown(ctx)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
