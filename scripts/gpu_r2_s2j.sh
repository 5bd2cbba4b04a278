#!/bin/bash
# round 2, session 2: treecode M2P with P2P sources as (delta, leaf index) float4 pairs: tests, timings
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tree.py -q -s > gpurun_out/s2j_tree.log 2>&1; echo "rc=$?" >> gpurun_out/s2j_tree.log
for a in "--config c2" "--config c3" "--clustered 1000000 --lam 1" "--clustered 1000000 --lam 1 --theta 0.7"; do
  timeout 300 python scripts/tree_bench.py $a --p 10 >> gpurun_out/s2j_tree_vs_fmm.jsonl 2>> gpurun_out/s2j_tree_vs_fmm.err
done
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:tree_kernel -c 1 -o gpurun_out/tree_s2j python scripts/tree_bench.py --config c2 --p 10 --reps 1 > gpurun_out/s2j_ncu_tree.log 2>&1
