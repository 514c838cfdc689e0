#!/usr/bin/env python
"""bench.py -- data-parallel BSN-TEM training throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c1|c5] [--impl ours|reference]

One "step" = one pass of the whole hot path over one batch per
rank: conv1/conv2 forward, head + weighted logistic loss, backward, and the fused ring
allreduce + mean + SGD (tem_step through the C ABI).  N > 1 runs under torchrun, one
process per GPU (weak scaling: B per GPU fixed).  Rank 0 prints ONE JSON line.

Timing: W untimed warm-up steps; then K timed steps, each bracketed by CUDA events on the
launching stream, with a 256 MiB L2 flush (outside the events) between steps; barrier +
synchronize on both sides of the timed region; the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TEM train samples/sec at 1/2/4/8 B200; ring-allreduce bus GB/s vs NCCL"
UNIT = "samples/s"
# the fp32 path's arithmetic: fp32 inputs split x = hi + lo (bf16 each), products hi*hi + hi*lo +
# lo*hi on the tensor cores, fp32 accumulation (R16); the line's "parity" object
# carries its measured per-tensor error against the fp64 oracle
F32 = "f32 (bf16x3 split products, f32 accumulate)"
WORKLOADS = {
    "c1": dict(desc="configs[0]: BSN TEM (400->512->512->3 conv1d, T=100) one data-parallel SGD step, "
                    "batch 4/rank, fp32", B=4, prec=0, dtype=F32),
    "c2": dict(desc="configs[1]: BSN TEM fp32 training, batch 16/GPU, synthetic ActivityNet-shaped "
                    "features", B=16, prec=0, dtype=F32),
    "c3": dict(desc="configs[2]: BSN TEM bf16-operand/fp32-accumulate training, batch 256/GPU", B=256,
               prec=1, dtype="bf16 operands, f32 accumulate"),
    "c5": dict(desc="configs[4]: BSN TEM + PEM (proposal evaluation MLP 32->512->1 over 32-d BSP features) "
                    "joint data-parallel training, fp32, batch 16 videos/GPU x 128 proposals", B=16, prec=0,
               dtype=F32, pem=128),
    "c6": dict(desc="configs[4] with PGM: BSN TEM + PGM + PEM joint data-parallel training, fp32, batch 16 "
                    "videos/GPU; PEM trained on the 128 best proposals PGM generates from the step's own TEM "
                    "output (BSP features, IoU targets vs the ground-truth instances)", B=16, prec=0,
               dtype=F32, pem=128, pgm=3),
}
T, CIN, C = 100, 400, 512
# Algorithmic FLOPs per sample of each kernel (dense count incl. zero-pad taps).
FLOPS_PER_SAMPLE = {
    "conv1_fwd": 2 * T * C * 3 * CIN,      # 122.88 M
    "conv2_fwd": 2 * T * C * 3 * C,        # 157.29 M
    "conv2_dgrad": 2 * T * C * 3 * C,      # 157.29 M
    "conv2_wgrad": 2 * T * C * 3 * C,      # 157.29 M
    "conv1_wgrad": 2 * T * C * 3 * CIN,    # 122.88 M
    # fp32 persistent backward (bwd_kernel): conv2 DGRAD + conv2 WGRAD + conv1 WGRAD in one launch
    "backward": 2 * T * C * 3 * C * 2 + 2 * T * C * 3 * CIN,  # 437.46 M
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons polled through NVML every ~5 ms in a
    background thread; stats are taken over the samples inside [mark_start, mark_stop]."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period: float = 0.010):
        self.index = index
        self.period = period
        self.samples = []
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self._paused = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:
            self.ok = False

    def _reasons(self):
        nv = self.nv
        for fn in ("nvmlDeviceGetCurrentClocksEventReasons", "nvmlDeviceGetCurrentClocksThrottleReasons"):
            if hasattr(nv, fn):
                try:
                    return int(getattr(nv, fn)(self.h))
                except Exception:
                    pass
        return 0

    def _run(self):
        while not self._stop.is_set():
            if not self._paused.is_set():
                try:
                    sm = float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                    self.samples.append((time.perf_counter(), sm, self._reasons()))
                except Exception:
                    pass
            time.sleep(self.period)  # NVML calls take a driver lock: poll sparingly

    def pause(self, on: bool):
        """The NVML calls contend with the main thread's CUDA driver calls (measured: the
        host-buffer loop ran at 80 us/step with the sampler polling, 72 without), so the
        sampler is paused outside the device-timed region."""
        if on:
            self._paused.set()
        else:
            self._paused.clear()

    def start(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if not self.ok:
            return None
        time.sleep(0.02)
        self._stop.set()
        self.th.join(timeout=2)
        win = [x for x in self.samples if self.t0 is not None and self.t0 <= x[0] <= (self.t1 or 1e30)]
        if not win:  # timed region shorter than one poll: nearest samples around it
            win = sorted(self.samples, key=lambda x: abs(x[0] - (self.t0 or 0)))[:3]
        if not win:
            return None
        reasons = set()
        for _, _, r in win:
            for bit, nm in self.REASONS.items():
                if r & bit:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median([w[1] for w in win]), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(win), "source": "nvml"}


def bind_to_gpu_numa(index: int):
    """Run this rank on the CPU cores NVML reports as local to its GPU, so the pinned staging
    buffers of the end-to-end leg are first-touched on the GPU's NUMA node (host->device copies
    from the far node measured at half the bandwidth).  Returns the core count, or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        return None
    return None


def warm_until(step, n, torch, min_s: float = 0.05):
    """Run `n` steps, then more until >= min_s of continuous stepping has passed."""
    t0 = time.perf_counter()
    i = 0
    while i < n or time.perf_counter() - t0 < min_s:
        step(i)
        i += 1
        if i % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()


def host_info():
    """the host the CPU oracle ran on."""
    model = "?"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity_cores": len(os.sched_getaffinity(0)), "cpu_model": model}


def oracle_step(workload: dict, x, lab, p, threads: int, pp=None, extra=None):
    """One rank-step of the oracle as it stands: TEM fwd + loss + bwd over the videos (threaded
    over videos when threads > 1), PGM/PEM for the joint workloads, and the fp32 owner update
    replay of the K_pad-element vector at N = 1."""
    import numpy as np
    import datagen
    import oracle
    B = x.shape[0]
    ref = oracle.tem_fwd_bwd(x, p, lab, prec=workload["prec"], threads=threads)
    P = workload.get("pem", 0)
    if P and workload.get("pgm"):
        gt, n = extra
        prob = (1.0 / (1.0 + np.exp(-np.asarray(ref["z"], np.float64).reshape(B, T, 3)))).transpose(0, 2, 1)
        pg = oracle.pgm(prob.astype(np.float32), gt, n, P)
        oracle.pem_fwd_bwd(pg["features"].reshape(B * P, datagen.PEM_F), pp, pg["iou"].ravel())
    elif P:
        f, g = extra
        oracle.pem_fwd_bwd(f, pp, g)
    grad = np.zeros((1, oracle.kpad(ref["grad"].size, 1)), np.float32)
    grad[0, :ref["grad"].size] = ref["grad"]
    oracle.ring_sgd(grad, np.zeros(grad.shape[1], np.float32), 0.01)
    return ref


def workload_extra(workload, B, rank=0, batch_idx=0):
    import datagen
    P = workload.get("pem", 0)
    if P and workload.get("pgm"):
        return datagen.instances(B, rank=rank, batch_idx=batch_idx)
    if P:
        return (datagen.bsp_features(B, P, rank=rank, batch_idx=batch_idx).reshape(B * P, datagen.PEM_F),
                datagen.iou_targets(B, P, rank=rank, batch_idx=batch_idx).ravel())
    return None


def cpu_baseline(workload: dict, videos: int):
    """The oracle as it stands (plain C++, fp64 / bf16-emulated fp64) timed on a bounded sample of
    the same workload -- `videos` videos of one rank-step -- once on one core and once threaded
    over videos on every core this process may use."""
    import datagen
    import oracle
    oracle.lib()
    x = datagen.features(videos, rank=0, batch_idx=0)
    lab = datagen.labels(videos, rank=0, batch_idx=0)
    p = datagen.init_params()
    pp = datagen.init_pem_params() if workload.get("pem") else None
    extra = workload_extra(workload, videos)
    prec = "fp64" if workload["prec"] == 0 else "bf16-emulated fp64"
    what = (f"{videos} videos ({prec} fwd+loss+bwd, T=100, 400->512->512->3"
            + (f", + PEM over {workload['pem']} proposals each" if workload.get("pem") else "")
            + (", + PGM" if workload.get("pgm") else "") + ") + fp32 owner-update replay of the K_pad vector")
    cores = len(os.sched_getaffinity(0))
    out = {}
    for key, n in (("one", 1), ("all", cores)):
        t0 = time.perf_counter()
        oracle_step(workload, x, lab, p, n, pp, extra)
        dt = time.perf_counter() - t0
        out[key] = {"value": videos / dt, "unit": UNIT, "cores": n, "kind": "oracle",
                    "sample": f"{what}; {dt:.1f} s on {n} core(s)" + ("" if n == 1 else " (threaded over videos)")}
    return out


def run_reference(args, workload):
    """--impl reference: the CPU oracle as it stands on this arm's config, metric and unit (rank 0
    only): each step is one rank-step of the workload -- the whole batch of B videos (threaded
    over videos on every core this process may use), the joint modules, the owner update."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import datagen
    import oracle
    oracle.lib()
    p = datagen.init_params()
    B = workload["B"]
    x = datagen.features(B, rank=0, batch_idx=0)
    lab = datagen.labels(B, rank=0, batch_idx=0)
    pp = datagen.init_pem_params() if workload.get("pem") else None
    extra = workload_extra(workload, B)
    cores = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        oracle_step(workload, x, lab, p, cores, pp, extra)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(workload, x, lab, p, cores, pp, extra)
    dt = time.perf_counter() - t0
    v = B * args.steps / dt
    prec = "fp64" if workload["prec"] == 0 else "bf16-emulated fp64"
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": workload["desc"], "batch_per_gpu": B,
                                           "seq_len": T, "parallelism": f"dp{args.gpus}"},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": f"the whole {B}-video batch per step ({prec} C++ oracle threaded over "
                                      f"videos, + the fp32 owner-update replay), {args.steps} steps"},
           "host": host_info(),
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def parity_check(sess, workload, x, lab, extra_dev=None):
    """The timed path's numerics on one batch, for the record: per-tensor max|gpu - oracle| /
    max|oracle| of the gradient, logits and loss against the oracle (fp64, or bf16-emulated
    fp64 for configs[2]) at the current weights; ReLU decisions inside the oracle's rounding band
    follow the GPU (reading R7b)."""
    import numpy as np
    import torch
    import oracle
    B = x.shape[0]
    prec = workload["prec"]
    w = sess.params(0).cpu().numpy()[:sess.K].copy()
    xd = torch.from_numpy(x).cuda() if prec == 0 else None
    if prec == 1:
        import datagen
        xd = torch.from_numpy(datagen.to_bf16_bits(x).view(np.int16)).cuda()
    sess.compute(xd[None], torch.from_numpy(lab).cuda()[None])
    sess.sync()
    g = sess.local_grad(0).cpu().numpy()[:sess.K]
    z = sess.logits(0).cpu().numpy()
    loss = sess.loss[0].cpu().numpy()
    dec = sess.relu_decisions(0).cpu().numpy()
    cores = len(os.sched_getaffinity(0))
    taus = (2.0 ** -13, 2.0 ** -13) if prec == 0 else (2.0 ** -13, 2.0 ** -8)
    ref = oracle.tem_fwd_bwd(x, w, lab, prec=prec, kink_tau=taus, kinks_cap=1 << 24, threads=cores)
    diff = np.nonzero(dec != ref["decisions"])[0]
    inside = bool(np.all(np.isin(diff, ref["kinks"])))
    if diff.size:
        ref = oracle.tem_fwd_bwd(x, w, lab, prec=prec, flips=diff, threads=cores)
    err = {}
    for name, sl in oracle.param_slices().items():
        err[name] = float(np.abs(g[sl] - ref["grad"][sl]).max() / np.abs(ref["grad"][sl]).max())
    err["z"] = float(np.abs(z - ref["z"]).max() / np.abs(ref["z"]).max())
    err["loss"] = float(np.abs(loss - ref["loss"]).max() / np.abs(ref["loss"]).max())
    tol = 1e-4 if prec == 0 else 2e-2
    return {"rel_err": err, "tol": tol, "pass": all(v <= tol for v in err.values()) and inside,
            "relu_flips": int(diff.size), "relu_decisions": int(dec.size),
            "batch": f"{B} videos, pool batch 0, initial weights",
            "norm": "per tensor max|gpu-oracle| / max|oracle| (DESIGN.md R17)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pool", type=int, default=8, help="resident input batches per rank")
    ap.add_argument("--cpu-videos", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--exchange", default="ring", choices=["ring", "ps", "twoshot"],
                    help="gradient exchange: the paper's ring (default), the PS comparator, or the "
                         "NVSwitch two-shot (ring-identical bits, 2 phases)")
    ap.add_argument("--buckets", type=int, default=1, choices=[1, 2],
                    help="N > 1: 2 = two-bucket exchange, the W2.. bucket overlapping conv1 wgrad (reading R25)")
    ap.add_argument("--optimizer", default="sgd", choices=["sgd", "adam", "momentum"],
                    help="owner update: the paper's SGD (default), Adam (reading R22) or heavy-ball "
                         "momentum 0.9 (reading R23)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl)

    import numpy as np
    import torch
    import torch.distributed as dist
    import datagen
    from paper_1906_06496_b200 import tem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            print(json.dumps({"error": "run N>1 under torchrun (one process per GPU)"}))
            return 2
    numa_cores = bind_to_gpu_numa(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    B, prec = wl["B"], wl["prec"]
    P = wl.get("pem", 0)
    sc = tem.SessionConfig(world_size=world, rank=rank, local_ranks=1, batch_per_rank=B, precision=prec,
                           lr=args.lr, exchange={"ps": tem.TEM_EXCHANGE_PS, "twoshot": tem.TEM_EXCHANGE_TWOSHOT}.get(
                               args.exchange, tem.TEM_EXCHANGE_RING),
                           pem_proposals=P, pgm_gt_max=wl.get("pgm", 0), exchange_buckets=args.buckets,
                           optimizer={"adam": tem.TEM_OPT_ADAM, "momentum": tem.TEM_OPT_MOMENTUM}.get(
                               args.optimizer, tem.TEM_OPT_SGD))
    t_init0 = time.perf_counter()
    params0 = datagen.init_params() if not P else np.concatenate([datagen.init_params(), datagen.init_pem_params()])
    sess = tem.TemSession(sc, params0, device=local)
    t_init = time.perf_counter() - t_init0

    # resident input pool (HBM); rank r's shard of global batch k uses seeds (r, k)
    xs, labs, fs, gs = [], [], [], []
    for k in range(args.pool):
        x = datagen.features(B, rank=rank, batch_idx=k)
        lab = datagen.labels(B, rank=rank, batch_idx=k)
        if prec == 1:
            xs.append(torch.from_numpy(datagen.to_bf16_bits(x).view(np.int16)).to(dev))
        else:
            xs.append(torch.from_numpy(x).to(dev))
        labs.append(torch.from_numpy(lab).to(dev))
        if P and wl.get("pgm"):  # ground-truth instances and counts (PGM-fed PEM)
            seg, cnt = datagen.instances(B, rank=rank, batch_idx=k)
            fs.append(torch.from_numpy(seg).to(dev))
            gs.append(torch.from_numpy(cnt).to(dev))
        elif P:
            fs.append(torch.from_numpy(datagen.bsp_features(B, P, rank=rank, batch_idx=k)).to(dev))
            gs.append(torch.from_numpy(datagen.iou_targets(B, P, rank=rank, batch_idx=k)).to(dev))

    def do_step(i):
        j = i % args.pool
        if P and wl.get("pgm"):
            sess.step_pgm(xs[j], labs[j], fs[j], gs[j])
        elif P:
            sess.step_pem(xs[j], labs[j], fs[j], gs[j])
        else:
            sess.step(xs[j], labs[j])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    clocks = ClockSampler(local, float(os.environ.get("BENCH_NVML_MS", "10")) / 1e3)
    clocks.start()
    # the timed path's numerics for the record, at the initial weights (after hundreds of SGD steps
    # on the same pool the small tensors -- b3: a sum of dz that cancels as training converges --
    # lose relative precision, which says nothing about the kernels)
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not P:
        parity = parity_check(sess, wl, datagen.features(B, rank=0, batch_idx=0),
                              datagen.labels(B, rank=0, batch_idx=0))
    # W warm-up steps, continued until the GPU has been busy for >= 50 ms: measured on these
    # boxes, the first tens of ms of steps after an idle period run up to 35 % slower
    warm_until(do_step, args.warmup, torch)
    # host enqueue cost of one timed iteration (flush + events + graph replay), for the lead below
    t_h = time.perf_counter()
    for i in range(8):
        flush.zero_()
        do_step(i)
    host_us_per_step = (time.perf_counter() - t_h) / 8 * 1e6
    torch.cuda.synchronize()
    sm_hz = torch.cuda.get_device_properties(dev).clock_rate * 1e3 if hasattr(
        torch.cuda.get_device_properties(dev), "clock_rate") else 1.965e9
    code, _ = sess.sync()
    if code != 0:
        raise tem.TemError(code, "warmup")

    # ---------------- timed region (device value) ----------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    # launch-ahead: a device-side spin (outside every step's events) holds the stream while the
    # host enqueues the K steps, so a host-side hiccup while enqueueing (seen once: one 68 ms
    # step) cannot leave the GPU idle inside a timed step; the spin is sized from the host's
    # measured enqueue rate and capped at 0.5 s
    lead_ms = min(500.0, max(10.0, 3.0 * args.steps * host_us_per_step / 1e3))
    if hasattr(torch.cuda, "_sleep"):
        torch.cuda._sleep(int(lead_ms * 1e-3 * sm_hz))
    else:
        lead_ms = 0.0
    t_enq = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        do_step(i)  # CUDA-graph replay of the whole step
        ev[i][1].record(stream)
    enq_ms = (time.perf_counter() - t_enq) * 1e3
    torch.cuda.synchronize()
    clocks.mark_stop()
    barrier()
    clk = clocks.stop()
    code, _ = sess.sync()
    if code != 0:
        raise tem.TemError(code, "timed steps")
    step_ms = [a.elapsed_time(b) for a, b in ev]
    step_stats = {"min_us": min(step_ms) * 1e3, "median_us": statistics.median(step_ms) * 1e3,
                  "max_us": max(step_ms) * 1e3}
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    ms_per_step = total_ms / args.steps
    value = world * B * args.steps / (total_ms / 1e3)
    launches = sess.launches_per_step()

    # ---------------- instrumented pass: per-kernel durations (events around every kernel) ----
    n_inst = min(args.steps, 20)
    barrier()
    torch.cuda.synchronize()
    sess.timing_begin(n_inst)
    for i in range(n_inst):
        flush.zero_()
        do_step(i)
    torch.cuda.synchronize()
    slot_ms, nrec = sess.timing_end()
    code, _ = sess.sync()
    if code != 0:
        raise tem.TemError(code, "instrumented steps")

    # ---------------- end to end through the C ABI with host buffers ----------------
    e2e = None
    clocks.pause(True)
    if not args.no_e2e:
        if prec == 1:
            xh = [torch.from_numpy(datagen.to_bf16_bits(datagen.features(B, rank=rank, batch_idx=k)).view(np.int16)).pin_memory()
                  for k in range(2)]
        else:
            xh = [torch.from_numpy(datagen.features(B, rank=rank, batch_idx=k)).pin_memory() for k in range(2)]
        lh = [torch.from_numpy(datagen.labels(B, rank=rank, batch_idx=k)).pin_memory() for k in range(2)]
        loss_h = torch.zeros(4, dtype=torch.float32).pin_memory()
        if P:  # joint workload: tem_step_pem_host (copies, step, loss read-back)
            if wl.get("pgm"):  # PGM-fed: the extra host inputs are the instances and their counts
                fh = [torch.from_numpy(datagen.instances(B, rank=rank, batch_idx=k)[0]).pin_memory() for k in range(2)]
                gh = [torch.from_numpy(datagen.instances(B, rank=rank, batch_idx=k)[1]).pin_memory() for k in range(2)]
            else:
                fh = [torch.from_numpy(datagen.bsp_features(B, P, rank=rank, batch_idx=k)).pin_memory() for k in range(2)]
                gh = [torch.from_numpy(datagen.iou_targets(B, P, rank=rank, batch_idx=k)).pin_memory() for k in range(2)]
            loss_h = torch.zeros(5, dtype=torch.float32).pin_memory()

            def host_step(i):
                sess.step_pem_host(xh[i % 2], lh[i % 2], fh[i % 2], gh[i % 2], loss_h)
        else:
            def host_step(i):
                sess.step_host(xh[i % 2], lh[i % 2], loss_h)
        warm_until(host_step, max(2, args.warmup), torch)
        # One span over all K steps: the library copies step k+1's inputs on its copy stream while
        # step k computes, so per-step spans would not see the copies.  No L2 flush inside the
        # span (a flush between steps would hide copy time under a subtracted interval); every
        # step's inputs arrive fresh by H2D copy.
        e_beg, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e_beg.record(stream)
        for i in range(args.steps):
            host_step(i)
        e_end.record(stream)
        torch.cuda.synchronize()
        barrier()
        code, _ = sess.sync()
        if code != 0:
            raise tem.TemError(code, "e2e steps")
        span = e_beg.elapsed_time(e_end)
        t2 = torch.tensor([span], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        h2d = int(xh[0].numel() * xh[0].element_size() + lh[0].numel() * 4)
        if P:
            h2d += int(fh[0].numel() * fh[0].element_size() + gh[0].numel() * gh[0].element_size())
        e2e = {"value": world * B * args.steps / (float(t2.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(loss_h.numel() * 4),
               "api": "tem_step_pem_host" if P else "tem_step_host",
               "host_cores_bound": numa_cores,
               "timing": "one event span over the K steps (no L2 flush inside it); each step's H2D copies "
                         "run on the library's copy stream (double-buffered staging) beside the previous "
                         "step's compute, its loss D2H inside the step"}

    # ---------------- roofline of the dominant kernel ----------------
    peaks, peak_src = load_peaks()
    conv = {k: v for k, v in slot_ms.items() if k in FLOPS_PER_SAMPLE}
    dom = max(conv, key=conv.get) if nrec else None
    roof = None
    if dom:
        avg_s = conv[dom] / nrec / 1e3
        achieved = FLOPS_PER_SAMPLE[dom] * B / avg_s / 1e12
        kpath = sess.kernel_path()
        # the slot is one kernel timed alone for 20-40 us: the BURST bf16 peak applies
        # (B200_PROFILING.md), not the sustained one of a long back-to-back run
        key = "bf16_tflops"
        bf16 = peaks.get(key)
        # fp32 path: three bf16 products per fp32 MAC (hi*hi + hi*lo + lo*hi, R16)
        peak = bf16 if prec == 1 else bf16 / 3.0
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "peak_source": f"{key} (burst, {peak_src}: the slot is one isolated kernel)" +
                               ("" if prec == 1 else " / 3 (3 bf16 tensor-core products per fp32 MAC, DESIGN.md R16)")}
        tr = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr):
            try:
                t = json.load(open(tr)).get(f"{args.workload}/{kpath}/{dom}")
                roof["traffic"] = t
            except Exception:
                pass
        roof["share_of_step"] = conv[dom] / max(sum(slot_ms.values()), 1e-9)
        roof["timing"] = (f"kernel duration from an instrumented pass of {nrec} steps (CUDA events around "
                          f"every kernel on its stream, no graph, side branch serialised so each slot is one "
                          f"kernel alone; ~3-4 us event overhead per slot); value from {args.steps} "
                          f"graph-replayed steps")
        roof["slot_ms_per_step"] = {k: v / max(nrec, 1) for k, v in slot_ms.items()}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic (seeded ActivityNet-shaped features/labels, random-init weights)",
        "config": {"workload": wl["desc"], "batch_per_gpu": B, "global_batch": B * world, "seq_len": T,
                   "channels": "400->512->512->3", "parallelism": f"dp{world}",
                   "optimizer": args.optimizer,
                   **({"exchange_buckets": 2} if args.buckets == 2 and world > 1 else {}),
                   "exchange": ("N=1: owner update only" if world == 1 else
                                {"ps": "parameter server on rank 0 (KP1)",
                                 "twoshot": "NVSwitch two-shot allreduce + mean + SGD (ring-identical bits)"}.get(
                                     args.exchange, "fused ring allreduce + mean + SGD (KR1)")),
                   "l2": "flushed between timed steps (256 MiB write, outside the events)",
                   "launch_ahead": f"{lead_ms:.1f} ms device spin before the timed steps (outside the "
                                   f"events); the host enqueued the {args.steps} steps in {enq_ms:.1f} ms",
                   "warmup": f"{args.warmup} steps, continued until >= 50 ms of stepping",
                   "kernel_path": sess.kernel_path(),
                   **({"pem": f"{P} proposals/video, 32-d BSP features, MLP 32->512->1, gradient [TEM | PEM] "
                              f"= {sess.K} elements in one exchange"} if P else {}),
                   **({"pgm": "PEM inputs generated on the GPU each step by PGM (tem_pgm kernel) from the "
                              "step's own TEM probabilities: top-128 proposals, BSP features, IoU targets "
                              f"vs <= {wl['pgm']} instances/video (reading R24)"} if wl.get("pgm") else {})},
        "step_us": step_stats,
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "roofline": roof,
        "e2e": e2e,
        "clocks": clk,
        "t3_init_s": t_init,
        # P:163 training-time decomposition, per step, from the instrumented pass:
        # t1 = forward + backward (all kernels but the exchange), t2 = gradient exchange.
        "paper_metrics": {
            "t1_fwd_bwd_ms": sum(v for k, v in slot_ms.items() if not k.startswith("exchange")) / max(nrec, 1),
            "t2_exchange_ms": sum(v for k, v in slot_ms.items() if k.startswith("exchange")) / max(nrec, 1),
            "t3_setup_s": t_init,
            "epoch_videos": 9997,
            "epoch_time_s": 9997 / value,
        },
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(wl, args.cpu_videos)
        out["cpu_baseline"] = cb["one"]
        out["cpu_baseline_all_cores"] = cb["all"]
        out["host"] = host_info()
        if parity is not None:
            out["parity"] = parity
    if rank == 0:
        print(json.dumps(out), flush=True)
    sess.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
