#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (committed evidence).

    python scripts/summarize_ncu.py launches <launches.csv> <out.txt>
    python scripts/summarize_ncu.py full <capture.ncu-rep> <out.txt> [--traffic-key PREFIX]

`launches`: per-kernel launch counts, mean device time (cold-cache, serialised under ncu) and
the share of the total.  `full`: per launch duration, DRAM bytes (read + write = the roofline
`traffic`), tensor-pipe utilisation, L2 / DRAM throughput, achieved occupancy.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__registers_per_thread", "l1tex__m_xbar2l1tex_read_bytes.sum"]


def to_us(v, unit):
    v = float(str(v).replace(",", ""))
    return {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3,
            "second": v * 1e6}.get(unit, v)


def to_bytes(v, unit):
    v = float(str(v).replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(unit, 1)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:90]].append(to_us(r[vi], r[ui]))
    # bench.py's own kernels (the L2 flush between steps, the launch-ahead spin before the timed
    # steps) run outside the step: listed, but not part of the share
    harness = lambda k: "FillFunctor<unsigned char>" in k or "spin_kernel" in k
    tot = sum(sum(v) for k, v in agg.items() if not harness(k))
    lines = [f"# ncu launch list ({os.path.basename(path)}): gpu__time_duration.sum, --clock-control none",
             "# cold-cache, serialised: compare SHARES, not absolute times; share = of the library's",
             "# kernels (bench.py's L2 flush and launch-ahead spin excluded, marked '-')", "",
             f"{'launches':>8} {'mean_us':>9} {'share':>7}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = "      -" if harness(k) else f"{100*sum(v)/tot:6.1f}%"
        lines.append(f"{len(v):8d} {sum(v)/len(v):9.2f} {share}  {k}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(path, out):
    raw = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(hdr)}
    lines = [f"# ncu --set full summary ({os.path.basename(path)}), --clock-control none", "",
             f"{'us':>8} {'DRAM_MB':>8} {'tensor%':>8} {'L2%':>6} {'DRAM%':>6} {'grid':>6} {'regs':>5} {'SMin_MB':>8}  kernel"]
    out_json = []
    for r in rows[2:]:
        def g(m, conv=None):
            i = idx.get(m)
            if i is None or r[i] in ("", "n/a"):
                return float("nan")
            return conv(r[i], units[i]) if conv else float(r[i].replace(",", ""))
        us = g("gpu__time_duration.sum", to_us)
        dr = (g("dram__bytes_read.sum", to_bytes) + g("dram__bytes_write.sum", to_bytes)) / 1e6
        sm_in = g("l1tex__m_xbar2l1tex_read_bytes.sum", to_bytes) / 1e6
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")[:80]
        lines.append(f"{us:8.1f} {dr:8.2f} {g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):8.1f} "
                     f"{g('lts__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
                     f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
                     f"{g('launch__grid_size'):6.0f} {g('launch__registers_per_thread'):5.0f} {sm_in:8.1f}  {name}")
        out_json.append({"kernel": name, "us": us, "dram_bytes": dr * 1e6, "sm_ingress_bytes": sm_in * 1e6,
                         "tensor_pct": g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")})
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(out_json, open(os.path.splitext(out)[0] + ".json", "w"), indent=1)
    print("\n".join(lines))


def details(path, out, kernel_regex):
    """The --page details sections (SOL, memory workload, occupancy, warp state, rules) of the LAST
    launch whose name matches kernel_regex (the steady-state step's launch)."""
    import re
    raw = subprocess.run([NCU, "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    ii, si, mi, ui, vi = (hdr.index(k) for k in ("ID", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    ki = hdr.index("Kernel Name")
    rows = [hdr] + [r for r in rows[1:] if len(r) > vi and re.search(kernel_regex, r[ki])]
    last = max(int(r[ii]) for r in rows[1:])
    sel = [r for r in rows[1:] if len(r) > vi and int(r[ii]) == last]
    lines = [f"# ncu --set full details ({os.path.basename(path)}), launch ID {last}: {sel[0][hdr.index('Kernel Name')]}",
             f"# grid {sel[0][hdr.index('Grid Size')]} block {sel[0][hdr.index('Block Size')]}, --clock-control none", ""]
    sec = None
    for r in sel:
        if r[si] != sec:
            sec = r[si]
            lines.append(f"## {sec}")
        if r[mi]:
            lines.append(f"  {r[mi]:<48} {r[vi]:>16} {r[ui]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    {"launches": launches, "full": full, "details": details}[sys.argv[1]](*sys.argv[2:])
