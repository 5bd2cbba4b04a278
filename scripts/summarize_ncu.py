"""Summarise ncu outputs into profiles/<round>/: launch-list shares and key --set full metrics.

usage: python scripts/summarize_ncu.py <launches.csv> <out.md> [<prof.ncu-rep> ...]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum"]


def launches(path):
    """Shares of one evaluate: the launch list is split at each keys_kernel (first kernel of
    an evaluation) and the last complete evaluation is reported."""
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    evals, cur = [], []
    for r in rows:
        name = r["Kernel Name"].split("(")[0].split("::")[-1]
        if name == "keys_kernel" and cur:
            evals.append(cur)
            cur = []
        cur.append((name, float(r["Metric Value"]) / 1e6))
    if cur:
        evals.append(cur)
    ev = evals[-1]
    agg = collections.OrderedDict()
    for name, ms in ev:
        agg[name] = agg.get(name, 0.0) + ms
    tot = sum(agg.values())
    out = ["| kernel | ms (sum of its launches) | share |", "|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        out.append(f"| {k} | {v:.3f} | {100 * v / tot:.1f}% |")
    out.append(f"| **total** ({len(ev)} launches in one evaluate) | {tot:.3f} | |")
    return "\n".join(out)


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append(f"### {r[hdr.index('Kernel Name')].split('(')[0].split('::')[-1]}")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"| {k} | {r[i]} {units[i]} |")
    return "\n".join(out)


if __name__ == "__main__":
    lc, dst, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    with open(dst, "w") as f:
        f.write("# ncu summary (cold-cache serialised launch list; shares, not absolutes)\n\n")
        f.write("## Launch list (one evaluate, c4 256^3, p=10, depth 6)\n\n")
        f.write(launches(lc) + "\n\n")
        f.write("## --set full (selected kernels)\n\n")
        for rep in reps:
            f.write(full(rep) + "\n\n")
    print(open(dst).read())
