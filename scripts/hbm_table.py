#!/usr/bin/env python3
"""HBM roofline table of one c4 evaluation from an ncu metrics CSV (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum per kernel): measured DRAM bytes and GB/s, and
for the memory-bound tree / translation passes the algorithmic bytes
and their fraction of the measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs).

    python scripts/hbm_table.py profiles/r2/ncu_dram_c4.csv [N=16777216] [p=10] [L=6]
"""
import collections
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path = sys.argv[1]
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
    p = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    L = int(sys.argv[4]) if len(sys.argv) > 4 else 6
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6553.9
    nc = (p + 1) ** 2
    cell = 3 * nc * 4  # bytes of one cell's expansion
    leaves = 8 ** L
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    k = collections.OrderedDict()
    for r in rows:
        d = k.setdefault(int(r["ID"]), {"name": r["Kernel Name"].split("(")[0]
                                        .replace("unnamed>::", "").replace("void ", "")})
        d[r["Metric Name"]] = float(r["Metric Value"])
    ids = sorted(k)
    evals, cur = [], []
    for i in ids:
        if k[i]["name"].startswith("keys_kernel") and cur:
            evals.append(cur)
            cur = []
        cur.append(i)
    evals.append(cur)
    last = evals[-1]
    # algorithmic bytes for the memory-bound passes (per launch)
    alg = {"keys_kernel": 20 * N, "radix_count": 4 * N, "radix_scatter": 16 * N,
           "leaf_ranges_kernel": 4 * N + 4 * (leaves + 1), "gather_kernel": 56 * N,
           "p2m_kernel<10>": 24 * N + leaves * cell}
    print(f"| kernel | ms | DRAM MB (ncu) | GB/s (ncu bytes) | algorithmic MB | algorithmic GB/s "
          f"| of {peak:.0f} GB/s |")
    print("|---|---|---|---|---|---|---|")
    seen = collections.Counter()
    for i in last:
        d = k[i]
        nm = d["name"]
        seen[nm] += 1
        t = d["gpu__time_duration.sum"] * 1e-9
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        a = alg.get(nm)
        if nm.startswith("translate_kernel<0>") and seen[nm] == 1:  # M2M, finest parent level
            a = leaves * cell + leaves // 8 * cell
        if nm.startswith("translate_kernel<1>") and seen[nm] == L:  # L2L into the leaf level
            a = leaves // 8 * cell + 2 * leaves * cell
        if nm.startswith("l2p_combine"):
            a = (24 + 24 + 4 + 24) * N + leaves * cell
        row = f"| {nm} | {t * 1e3:.3f} | {b / 1e6:.1f} | {b / t / 1e9:.0f} | "
        row += (f"{a / 1e6:.1f} | {a / t / 1e9:.0f} | {a / t / 1e9 / peak:.2f} |" if a else "— | — | — |")
        print(row)


if __name__ == "__main__":
    main()
