#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for m in cross sj; do
VFMM_P2P=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$m.log 2>&1
echo "$m $(grep -o '"p2p": [0-9.]*' gpurun_out/bench_$m.log)" >> gpurun_out/variants.log
done
timeout 900 python -m pytest tests -m gpu -q -x -k "near or fmm_vs_fmm or c4 or deterministic" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
