"""Summarise ncu reports (run here, no GPU needed).

    python tools/ncu_summary.py REPORT.ncu-rep [...]          # key metrics
    python tools/ncu_summary.py --sass REPORT.ncu-rep          # per-opcode mix + top stalls
    python tools/ncu_summary.py --launches launches.csv        # per-kernel share of a launch list
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, u))) for r in rows[2:]]


def summary(rep):
    for vals, units in raw(rep):
        print(f"== {rep}: {vals.get('Kernel Name', '')[:90]}")
        for k in KEYS:
            if k in vals:
                print(f"  {k:66s} {vals[k]:>18s} {units.get(k, '')}")
        if "dram__bytes_read.sum" in vals:
            def gb(k):
                v = float(vals[k].replace(",", ""))
                return v * (1e-3 if units[k] == "Mbyte" else 1.0 if units[k] == "Gbyte" else 1e-9)
            print(f"  {'dram read+write (GB)':66s} {gb('dram__bytes_read.sum') + gb('dram__bytes_write.sum'):18.3f}")


def sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stall = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(float(r[si] or 0) for r in data) or 1.0
    agg = defaultdict(lambda: [0.0, 0.0])
    for r in data:
        toks = r[1].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        agg[op][0] += float(r[ie] or 0)
        agg[op][1] += float(r[si] or 0)
    ti = sum(v[0] for v in agg.values()) or 1.0
    print(f"== {rep}: {ti:.3e} warp instructions, {tot:.0f} stall samples")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:20]:
        print(f"  {k:10s} inst {100 * v[0] / ti:5.1f}%   samples {100 * v[1] / tot:5.1f}%")
    st = defaultdict(float)
    for r in data:
        for i in stall:
            st[h[i]] += float(r[i] or 0)
    ts = sum(st.values()) or 1.0
    print("  stall reasons:", ", ".join(f"{k[6:]} {100 * v / ts:.1f}%"
                                       for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki][:70]][0] += 1
            agg[r[ki][:70]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:6d} {v[1] / 1e6:10.3f} ms {100 * v[1] / tot:5.1f}%  avg {v[1] / v[0] / 1e3:9.1f} us  {k}")


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--sass":
        for a in args[1:]:
            sass(a)
    elif args and args[0] == "--launches":
        launches(args[1])
    else:
        for a in args:
            summary(a)
