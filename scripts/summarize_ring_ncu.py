#!/usr/bin/env python
"""Summarise an ncu CSV of `bench_ring.py --emulate N` (ring_kernel / twoshot_kernel launches,
metrics gpu__time_duration.sum, dram__bytes_read/write.sum, lts__t_bytes.sum):

    python scripts/summarize_ring_ncu.py N profiles/r02d_ring_ncu_emulated_N8.csv

bench_ring.py launches, per message size S (64 KiB .. max, plus 5,613,580 B), warmup + iters
ring launches, then warmup + iters two-shot launches; the last launch of each group is reported.
Algorithmic bytes: each rank sends 2(N-1)/N * S; the emulation runs all N
ranks on one GPU, so its traffic floor is N times one rank's, LL lines (ring) doubling the
wire bytes."""
import collections
import csv
import sys


def main():
    N = int(sys.argv[1])
    path = sys.argv[2]
    per = int(sys.argv[3]) if len(sys.argv) > 3 else 3  # launches per (impl, size)
    rows = list(csv.reader(line for line in open(path) if not line.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    items = list(d.values())
    sizes = sorted(set([1 << k for k in range(16, 25)] + [5613580]))
    print(f"N={N} emulated ranks (one cooperative launch on one B200); last launch of each group")
    print(f"{'bytes':>10} {'impl':>8} {'us':>8} {'DRAM MB':>8} {'L2 MB':>8} {'alg MB/rank':>11} {'alg x N GB/s':>12}")
    i = 0
    for S in sizes:
        for impl in ("ring", "twoshot"):
            if i + per > len(items):
                return
            m = items[i + per - 1]
            i += per
            t = m["gpu__time_duration.sum"] * 1e-9
            alg = 2 * (N - 1) / N * S
            dram = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / 1e6
            print(f"{S:>10} {impl:>8} {t * 1e6:>8.1f} {dram:>8.1f} {m['lts__t_bytes.sum'] / 1e6:>8.1f} "
                  f"{alg / 1e6:>11.2f} {alg * N / t / 1e9:>12.1f}")


if __name__ == "__main__":
    main()
