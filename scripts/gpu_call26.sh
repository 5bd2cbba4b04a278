#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/p2p_precision.py > gpurun_out/p2p_precision.log 2>&1; echo "rc=$?" >> gpurun_out/p2p_precision.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
VFMM_P2P=cross timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cross.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cross.log
