"""Summarise tree_bench.py JSON lines: ms, interaction counts and the achieved FP32 rate of the
treecode kernel at its algorithmic flop (M2P 96 (p+1)^2, P2P 69 per pair)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        d = json.loads(line)
        t, p = d["tree"], d["p"]
        fl = t["m2l"] * 96 * (p + 1) ** 2 + t["pairs"] * 69
        print(f"{d['field']:28s} theta {d['theta']:.1f}  fmm {d['fmm']['ms']:9.1f} ms  tree {t['ms']:9.1f} ms"
              f"  m2p {t['m2l']:.3g}  pairs {t['pairs']:.3g}  {fl / t['ms_p2p'] / 1e9:5.1f} TF/s"
              f" ({fl / t['ms_p2p'] / 1e9 / 74.4:.2f} of FP32)  |u_tree - u_fmm| {d['tree_vs_fmm_u']:.1e}")
