#!/bin/bash
# round 2, session 2: treecode GPU tests + timing
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tree.py -q -s -x > gpurun_out/s2b_tree.log 2>&1; echo "rc=$?" >> gpurun_out/s2b_tree.log
timeout 300 python scripts/tree_bench.py --config c2 --p 10 > gpurun_out/s2b_tb.log 2>&1
timeout 300 python scripts/tree_bench.py --config c3 --p 10 >> gpurun_out/s2b_tb.log 2>&1
timeout 300 python scripts/tree_bench.py --clustered 1000000 --p 10 --lam 1 >> gpurun_out/s2b_tb.log 2>&1
